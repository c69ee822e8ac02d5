export OUT=gpurun_out/r2zz6
mkdir -p $OUT
for lib in build_ab/libtsa_prev.so paper_2012_10684_b200/libtsa.so build_ab/libtsa_prev.so paper_2012_10684_b200/libtsa.so; do
  echo "== $lib"; TSA_LIB_PATH=$lib timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5 bench', d['ms_per_step'], d['kernels']['search']['ms'])"
done > $OUT/ab_stage.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $OUT/launches_c5.csv python tools/prof_run.py c5 --reps 2 > /dev/null 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $OUT/smoke.log 2>&1; echo "rc=$?" >> $OUT/smoke.log
