#!/usr/bin/env bash
# Round-2 measurements on a B200 (through gpurun, from the repo root):
#   /usr/local/graft/bin/gpurun --timeout 5400 -- 'bash tools/refresh_profiles_r02.sh'
set -u
cd "${GRAFT_REPO_ROOT:-.}"
R=r02
O=gpurun_out
mkdir -p $O
timeout 1200 python bench.py --steps 10 --warmup 3 > $O/${R}_bench_config4.json 2> $O/${R}_bench_config4.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/${R}_bench_reference_config4.json 2> $O/${R}_bench_reference.err
for c in 1 2; do
  timeout 900 python bench.py --config $c --steps 50 --warmup 5 > $O/${R}_bench_config$c.json 2> $O/${R}_bench_config$c.err
done
timeout 900 python bench.py --config 3 --steps 10 --warmup 3 > $O/${R}_bench_config3.json 2> $O/${R}_bench_config3.err
timeout 1800 python bench.py --config 5 --steps 2 --warmup 3 > $O/${R}_bench_config5.json 2> $O/${R}_bench_config5.err
# launch list of the default bench command (config 4)
timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
    --log-file $O/${R}_launches_config4_raw.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
python tools/launch_summary.py $O/${R}_launches_config4_raw.csv "python bench.py --steps 2 --warmup 1 --no-cpu-baseline" > $O/${R}_launches_config4.csv
# DRAM traffic of every coupling launch of one config-4 step (bench plan)
timeout 1800 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:"k_qfft|k_tgemm|k_modgemm" --csv --log-file $O/${R}_traffic_config4_raw.csv python tools/one_step.py 4 1 > /dev/null 2>&1
# full captures: the two coupling kernels and the modulated SHT at config 4, the line kernel at config 2
timeout 1800 ncu --set full --clock-control none --import-source on -k regex:"k_tgemm|k_qfft" -c 2 \
    -o $O/${R}_twopass_config4 python tools/profile_shard.py 4 500 510 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_modgemm -c 1 \
    -o $O/${R}_modgemm_config4 python tools/profile_shard.py 4 500 510 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_couple_lines -c 1 \
    -o $O/${R}_couple_lines_config2 python tools/one_step.py 2 1 > /dev/null 2>&1
echo done
