#!/usr/bin/env bash
# Run on the GPU box (gpurun): bench lines for every workload, the ncu launch
# list of the default bench, and ncu --set full captures of the top kernels.
# Usage: tools/collect_profiles.sh <tag>
set -u
TAG=${1:-r1}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $OUT/gpu.txt
python bench.py > $OUT/bench_c2.jsonl 2> $OUT/bench_c2.err
python bench.py --workload c1 --steps 2000 --warmup 20 > $OUT/bench_c1.jsonl 2>&1
python bench.py --workload c3 --steps 20 --warmup 3 --e2e-steps 2 > $OUT/bench_c3.jsonl 2>&1
python bench.py --workload c4 --steps 20 --warmup 3 --e2e-steps 2 > $OUT/bench_c4.jsonl 2>&1
python bench.py --workload c4 --enumeration full --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline > $OUT/bench_c4_full.jsonl 2>&1
python bench.py --workload c5 --steps 20 --warmup 3 --e2e-steps 2 --no-cpu-baseline > $OUT/bench_c5.jsonl 2>&1
python bench.py --workload c4 --enumeration dp --steps 50 --warmup 3 --e2e-steps 2 > $OUT/bench_c4_dp.jsonl 2>&1
python bench.py --workload f1 --steps 500 > $OUT/bench_f1.jsonl 2>&1
python bench.py --workload f2 --steps 500 > $OUT/bench_f2.jsonl 2>&1
python bench.py --workload f3 --steps 100 > $OUT/bench_f3.jsonl 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $OUT/launches_c2.csv \
    python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_hist_part|k_mid|k_label_part" -s 6 -c 3 \
    -o $OUT/prof_c2 python bench.py --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline > $OUT/ncu_c2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_search_rows" -s 1 -c 1 \
    -o $OUT/prof_c4full python bench.py --workload c4 --enumeration full --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline > $OUT/ncu_c4.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $OUT/launches_c4_dp.csv \
    python bench.py --workload c4 --enumeration dp --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_search_dp" -s 1 -c 1 \
    -o $OUT/prof_c4dp python bench.py --workload c4 --enumeration dp --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline > $OUT/ncu_c4dp.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 30 --csv --log-file $OUT/launches_f1.csv \
    python bench.py --workload f1 --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_tsallis2d" -s 3 -c 1 \
    -o $OUT/prof_f1 python bench.py --workload f1 --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > $OUT/ncu_f1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_morph" -s 4 -c 2 \
    -o $OUT/prof_f3 python bench.py --workload f3 --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > $OUT/ncu_f3.log 2>&1
ls -la $OUT
