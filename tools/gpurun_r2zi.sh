export OUT=gpurun_out/r2zi
mkdir -p $OUT
P="python tools/prof_run.py"
{ timeout 300 python tools/ab_prune.py c5 --reps 20 --var TSA_SPLIT_FINALIZE;
  for lc in 6 8; do echo "== TSA_LABEL_CTAS=$lc"; TSA_LABEL_CTAS=$lc timeout 300 python tools/ab_prune.py c5 --reps 20 --var TSA_SPLIT_FINALIZE | grep "=1"; done
  timeout 300 python tools/ab_prune.py c4 --reps 20 --var TSA_SPLIT_FINALIZE; } > $OUT/times.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $OUT/launches_c5.csv $P c5 --reps 2 > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_prune.py tests/test_gpu_parity.py tests/test_gpu_tri.py tests/test_gpu_dp.py -x -q > $OUT/pytest_a.log 2>&1; echo "rc=$?" >> $OUT/pytest_a.log
timeout 1500 python -m pytest tests/test_gpu_full_parity.py -x -q > $OUT/pytest_full.log 2>&1; echo "rc=$?" >> $OUT/pytest_full.log
