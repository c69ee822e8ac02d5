export OUT=gpurun_out/r2zk
mkdir -p $OUT
P="python tools/prof_run.py"
# A: current in-tree lib (p2 from params), B: build_ab/libtsa_p2.so (p2 in shared)
for lib in paper_2012_10684_b200/libtsa.so build_ab/libtsa_p2.so; do
  echo "== $lib"
  for w in c2 c4 c5; do TSA_LIB_PATH=$lib timeout 120 $P $w --reps 12 | tail -4; done
  TSA_LIB_PATH=$lib timeout 120 $P c2 --reps 12 --pipeline staged | tail -3
done > $OUT/ab_p2.txt 2>&1
export TSA_LIB_PATH=build_ab/libtsa_p2.so
for L in 3 4 6; do echo "== lanes $L"; TSA_SWEEP_LANES=$L timeout 300 python bench.py --workload c3 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'])"; done > $OUT/sweep.txt 2>&1
for w in c2 c4 c5; do timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $OUT/launches_$w.csv $P $w --reps 2 > /dev/null 2>&1; done
timeout 900 python -m pytest tests/test_gpu_prune.py tests/test_gpu_parity.py tests/test_gpu_tri.py tests/test_gpu_dp.py tests/test_gpu_stream.py tests/test_gpu_hu.py -x -q > $OUT/pytest_a.log 2>&1; echo "rc=$?" >> $OUT/pytest_a.log
