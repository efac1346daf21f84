#!/usr/bin/env bash
# Regenerate the round's measurements on a B200 (run through gpurun from the repo root):
#   /usr/local/graft/bin/gpurun --timeout 3600 -- 'bash tools/refresh_profiles.sh r02'
# Bench lines of every BASELINE config and the reference arm, the default bench command's ncu
# launch list, and --set full captures of the coupling kernels; summaries via tools/*.py.
set -u
R=${1:-rXX}
O=gpurun_out
mkdir -p $O
for c in 1 2 3 4; do
  timeout 900 python bench.py --config $c --steps $([ $c -le 2 ] && echo 50 || echo 3) > $O/${R}_bench_config$c.json 2> $O/${R}_bench_config$c.err
done
timeout 1200 python bench.py --config 5 --steps 2 > $O/${R}_bench_config5.json 2> $O/${R}_bench_config5.err
timeout 600 python bench.py --impl reference --steps 3 > $O/${R}_bench_reference_config2.json 2> $O/${R}_bench_reference.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $O/${R}_launches_config2_raw.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
python tools/launch_summary.py $O/${R}_launches_config2_raw.csv "python bench.py --steps 2 --warmup 1" > $O/${R}_launches_config2.csv
ncu --set full --clock-control none --import-source on -k regex:k_couple_lines -c 1 \
    -o $O/${R}_couple_lines_config2 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
for c in "3 250 260" "4 500 510" "5 1000 1001"; do
  set -- $c
  ncu --set full --clock-control none --import-source on -k regex:"k_tgemm|k_qfft" -c 2 \
      -o $O/${R}_twopass_config$1 python tools/profile_shard.py $c > /dev/null 2>&1
done
echo done
