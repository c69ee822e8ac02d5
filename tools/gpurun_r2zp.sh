export OUT=gpurun_out/r2zp
mkdir -p $OUT
P="python tools/prof_run.py"
for lib in paper_2012_10684_b200/libtsa.so build_ab/libtsa_q8.so; do echo "== $lib"; TSA_LIB_PATH=$lib timeout 120 $P c4 --reps 12 | tail -3; done > $OUT/ab_q.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $OUT/launches_c4.csv $P c4 --reps 2 > /dev/null 2>&1
TSA_LIB_PATH=build_ab/libtsa_q8.so timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $OUT/launches_c4_q8.csv $P c4 --reps 2 > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_tri.py tests/test_gpu_prune.py tests/test_gpu_dist.py -x -q > $OUT/pytest_a.log 2>&1; echo "rc=$?" >> $OUT/pytest_a.log
timeout 900 python -m pytest tests/test_gpu_full_parity.py -x -q -k "c4" > $OUT/pytest_full.log 2>&1; echo "rc=$?" >> $OUT/pytest_full.log
