export OUT=gpurun_out/r2zj
mkdir -p $OUT
for L in 1 2 3; do echo "== lanes $L"; TSA_SWEEP_LANES=$L timeout 300 python bench.py --workload c3 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['gpu_launches'])"; done > $OUT/sweep.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file $OUT/launches_c3.csv python bench.py --workload c3 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_full_parity.py -x -q -k "c3 or sweep" > $OUT/pytest_full.log 2>&1; echo "rc=$?" >> $OUT/pytest_full.log
tools/ncu_prof.sh c3 "c3 --reps 3" k_search_tri
