export OUT=gpurun_out/r2zz
mkdir -p $OUT
P="python tools/prof_run.py"
for lib in build_ab/libtsa_prev.so paper_2012_10684_b200/libtsa.so build_ab/libtsa_prev.so paper_2012_10684_b200/libtsa.so; do
  echo "== $lib"; TSA_LIB_PATH=$lib timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5 bench', d['ms_per_step'], d['kernels']['search']['ms'])"
done > $OUT/ab_rec.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $OUT/launches_c5.csv $P c5 --reps 2 > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_prune.py tests/test_gpu_parity.py -x -q > $OUT/pytest_a.log 2>&1; echo "rc=$?" >> $OUT/pytest_a.log
timeout 900 python -m pytest tests/test_gpu_full_parity.py -x -q -k "c5" > $OUT/pytest_full.log 2>&1; echo "rc=$?" >> $OUT/pytest_full.log
