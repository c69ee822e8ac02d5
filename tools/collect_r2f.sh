#!/usr/bin/env bash
# Round-2 evidence on the GPU box (gpurun): bench lines for every workload,
# the reference arm, ncu launch lists and compact exports (details / raw /
# hot SASS lines) of --set full captures of the dominant kernels.
# Final round-2 sweep: also the GPU test suite, smoke() and compute-sanitizer.
# Usage: tools/collect_r2f.sh <tag>     (writes gpurun_out/<tag>/)
set -u
TAG=${1:-r2}
OUT=gpurun_out/$TAG
mkdir -p $OUT /tmp/ncu
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $OUT/gpu.txt
nproc > $OUT/host.txt; lscpu | grep "Model name" >> $OUT/host.txt
timeout 2400 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $OUT/smoke.log 2>&1; echo "rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench_c5.jsonl 2> $OUT/bench_c5.err
timeout 600 python bench.py --workload c1 --steps 2000 --warmup 20 > $OUT/bench_c1.jsonl 2> $OUT/bench_c1.err
timeout 600 python bench.py --workload c2 --steps 2000 --warmup 20 > $OUT/bench_c2.jsonl 2> $OUT/bench_c2.err
timeout 900 python bench.py --workload c3 --steps 20 --warmup 3 --e2e-steps 2 > $OUT/bench_c3.jsonl 2> $OUT/bench_c3.err
timeout 900 python bench.py --workload c4 --steps 50 --warmup 3 --e2e-steps 2 > $OUT/bench_c4.jsonl 2> $OUT/bench_c4.err
timeout 600 python bench.py --workload c4 --shard tuples --steps 20 --warmup 3 > $OUT/bench_c4_tuples.jsonl 2> $OUT/bench_c4_tuples.err
timeout 600 python bench.py --workload c4 --enumeration dp --steps 50 --warmup 3 --e2e-steps 2 --no-cpu-baseline > $OUT/bench_c4_dp.jsonl 2>&1
timeout 600 python bench.py --workload c4 --enumeration full --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline > $OUT/bench_c4_full.jsonl 2>&1
timeout 600 python bench.py --workload f1 --steps 300 > $OUT/bench_f1.jsonl 2> $OUT/bench_f1.err
timeout 600 python bench.py --workload f2 --steps 300 > $OUT/bench_f2.jsonl 2> $OUT/bench_f2.err
timeout 600 python bench.py --workload f3 --steps 100 > $OUT/bench_f3.jsonl 2> $OUT/bench_f3.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 2 > $OUT/ref_c5.jsonl 2> $OUT/ref_c5.err
P="python tools/prof_run.py"
for w in c5 c4 c3 c2; do
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $OUT/launches_$w.csv \
      $P $w --reps 3 > /dev/null 2>&1
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $OUT/launches_c5_bench.csv \
    python bench.py --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
prof() {  # name kernel-regex args...
  name=$1; kre=$2; shift 2
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$kre -s 1 -c 1 -o /tmp/ncu/$name "$@" \
      > $OUT/ncu_$name.log 2>&1
  ncu -i /tmp/ncu/$name.ncu-rep --page details --csv > $OUT/details_$name.csv 2>/dev/null
  ncu -i /tmp/ncu/$name.ncu-rep --page raw --csv > $OUT/raw_$name.csv 2>/dev/null
  ncu -i /tmp/ncu/$name.ncu-rep --page source --csv --print-source sass > /tmp/ncu/src_$name.csv 2>/dev/null
  python tools/ncu_hot.py /tmp/ncu/src_$name.csv > $OUT/hot_$name.txt 2>&1
}
prof k2_c5 k_search_k2 $P c5 --reps 2
prof hist16_c5 k_hist16 $P c5 --reps 2
prof label_c5 k_label_flat $P c5 --reps 2
prof scanseed_c5 k_scan_seed $P c5 --reps 2
prof phi_c5 k_finalize_phi $P c5 --reps 2
prof tables_c4 k_tri_tables $P c4 --reps 2
prof tables_c3 k_tri_tables $P c3 --reps 2
prof tri_c4 k_search_tri $P c4 --reps 2
prof tri_c3 k_search_tri $P c3 --reps 2
prof hist_c2 k_hist_part $P c2 --reps 2
prof mid_c2 k_mid $P c2 --reps 2
timeout 1800 bash tools/sanitize.sh $OUT/sanitizer > $OUT/sanitize.log 2>&1; echo "rc=$?" >> $OUT/sanitize.log
du -sh $OUT
