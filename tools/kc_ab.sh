# A/B of SLSHT_CUDA_TP_KC under ncu (unthrottled, serialized launches) and in the bench (power cap)
for kc in 0 2; do
  SLSHT_CUDA_TP_KC=$kc ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_qfft|k_tgemm" --csv \
     --log-file gpurun_out/kc_ab_$kc.csv python tools/one_step.py 4 1 > /dev/null 2>&1
  python tools/launch_summary.py gpurun_out/kc_ab_$kc.csv "KC=$kc one_step 4" | grep "k_qfft\|k_tgemm"
done
for kc in 0 2 0 2; do SLSHT_CUDA_TP_KC=$kc timeout 600 python bench.py --no-cpu-baseline --steps 10 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('bench KC=$kc', d['ms_per_step'], d['stages_ms']['couple'], d['stages_ms']['qfft'], d['clocks']['sm_mhz'])
"; done
