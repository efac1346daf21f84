# k_tpipe timing sweeps (lean / k_qfft FFT items, timing switches SLSHT_CUDA_TP_EXP, config 3): gpurun -- bash tools/pipe_exp.sh
for fv in 1 0; do
echo "== FV=$fv"
SLSHT_CUDA_TP_FV=$fv SHAPES="13,16,3,4,1;10,16,4,4,1;13,16,3,8,1;13,8,3,8,1" timeout 300 python tools/pipe_check.py 4 300 400 2>&1
for e in 1 3; do
  echo "== FV=$fv EXP=$e"
  SLSHT_CUDA_TP_FV=$fv SLSHT_CUDA_TP_EXP=$e SHAPES="13,16,3,4,1;13,16,3,8,1" timeout 300 python tools/pipe_check.py 4 300 400 2>&1 | grep -v "^config"
done
done
echo "== config 3 (n = 65), FV=1"
SHAPES="0,0,0,0,0;0,16,3,4,1;0,24,3,4,1" timeout 300 python tools/pipe_check.py 3 150 200 2>&1
