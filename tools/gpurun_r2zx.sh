export OUT=gpurun_out/r2zx
mkdir -p $OUT
P="python tools/prof_run.py"
for lib in build_ab/libtsa_cp0.so paper_2012_10684_b200/libtsa.so; do
  echo "== $lib"
  for w in c5 c4 c3 c2; do TSA_LIB_PATH=$lib timeout 120 $P $w --reps 12 | tail -3; done
  TSA_LIB_PATH=$lib timeout 300 python bench.py --workload c3 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3 sweep', d['ms_per_step'])"
  TSA_LIB_PATH=$lib timeout 300 python bench.py --steps 50 --warmup 3 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5 bench', d['ms_per_step'])"
done > $OUT/ab_cp.txt 2>&1
for w in c5 c4; do timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $OUT/launches_$w.csv $P $w --reps 2 > /dev/null 2>&1; done
timeout 2400 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
