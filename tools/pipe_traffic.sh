# DRAM traffic of k_tpipe against k_tgemm + k_qfft on the same degree range (config 4, [300, 340))
export RING_MB=16384
for pipe in 1 0; do
  SLSHT_CUDA_TP_PIPE=$pipe SLSHT_CUDA_TP_NQG=16 SLSHT_CUDA_TP_FB=4 SLSHT_CUDA_NO_GRAPH=1 \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum \
      --clock-control none -k regex:"k_tpipe|k_tgemm|k_qfft" -c 6 --csv --log-file gpurun_out/pipe_traffic_$pipe.csv \
      python tools/range_time.py 4 300 340 1 > gpurun_out/pipe_traffic_$pipe.log 2>&1
done
