mkdir -p gpurun_out/r2z
P="python tools/prof_run.py"
{ timeout 300 python tools/ab_prune.py c5 --reps 20; timeout 120 $P c4 --reps 6; timeout 120 $P c3 --reps 6; } > gpurun_out/r2z/times.txt 2>&1
for w in c5 c4 c3; do timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/r2z/launches_$w.csv $P $w --reps 2 > /dev/null 2>&1; done
timeout 600 python -m pytest tests/test_gpu_prune.py tests/test_gpu_tri.py -x -q > gpurun_out/r2z/pytest_prune.log 2>&1; echo "rc=$?" >> gpurun_out/r2z/pytest_prune.log
timeout 1500 python -m pytest tests/test_gpu_full_parity.py -x -q > gpurun_out/r2z/pytest_full.log 2>&1; echo "rc=$?" >> gpurun_out/r2z/pytest_full.log
for w in c3 c4; do timeout 300 python bench.py --workload $w --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/r2z/bench_$w.jsonl 2> gpurun_out/r2z/bench_$w.err; done
