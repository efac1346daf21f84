# Degree-range timing of the two-pass path against SLSHT_CUDA_TP_KC (rows recomputed by k_qfft): gpurun -- bash tools/kc_check.sh
for kc in 0 2 4 6 8; do
  echo "== KC=$kc"
  SLSHT_CUDA_TP_KC=$kc python tools/range_time.py 4 300 400 3 2>&1 | tail -1
done
for kc in 0 4 8; do
  echo "== config 3 KC=$kc"
  SLSHT_CUDA_TP_KC=$kc python tools/range_time.py 3 150 200 3 2>&1 | tail -1
done
