export OUT=gpurun_out/r2zl
mkdir -p $OUT
P="python tools/prof_run.py"
export TSA_LIB_PATH=build_ab/libtsa_cum.so
{ for w in c3 c4; do timeout 120 $P $w --reps 12 | tail -4; done; } > $OUT/times.txt 2>&1
for L in 4 6; do echo "== lanes $L"; TSA_SWEEP_LANES=$L timeout 300 python bench.py --workload c3 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'])"; done > $OUT/sweep.txt 2>&1
for w in c3 c4; do timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $OUT/launches_$w.csv $P $w --reps 2 > /dev/null 2>&1; done
timeout 900 python -m pytest tests/test_gpu_tri.py tests/test_gpu_prune.py tests/test_gpu_parity.py -x -q > $OUT/pytest_a.log 2>&1; echo "rc=$?" >> $OUT/pytest_a.log
timeout 1200 python -m pytest tests/test_gpu_full_parity.py -x -q -k "c3 or c4 or sweep" > $OUT/pytest_full.log 2>&1; echo "rc=$?" >> $OUT/pytest_full.log
