SHAPES="13,16,3,4,1;13,16,4,4,2;10,16,4,4,2;10,16,4,4,1;7,16,6,4,2;10,12,4,4,2;10,16,4,8,2;10,16,5,4,3" timeout 300 python tools/pipe_check.py 4 300 400 2>&1
for shape in "13 16 3 4 1" "10 16 4 4 2"; do
  set -- $shape
  echo "== full bench, pipe ct=$1 nqg=$2 nslot=$3 fb=$4 lag=$5"
  SLSHT_CUDA_TP_PIPE=1 SLSHT_CUDA_TP_CT=$1 SLSHT_CUDA_TP_NQG=$2 SLSHT_CUDA_TP_NSLOT=$3 SLSHT_CUDA_TP_FB=$4 SLSHT_CUDA_TP_LAG=$5 timeout 600 python bench.py --no-cpu-baseline --steps 10 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(d['ms_per_step'], d['stages_ms'], d['clocks'], d['roundtrip_err'], d.get('digests_complete'))
    else: print(l.rstrip()[:300])
"
done
echo "== full bench, two-pass"
timeout 600 python bench.py --no-cpu-baseline --steps 10 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(d['ms_per_step'], d['stages_ms'], d['clocks'])
"
