mkdir -p gpurun_out/r2y
{ timeout 300 python tools/ab_prune.py c5 --reps 20; timeout 120 python tools/ab_prune.py c5 --reps 10 --q 0.5;
  timeout 120 python tools/ab_prune.py c2 --reps 20 --pipeline staged; } > gpurun_out/r2y/ab.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_prune.py -x -q > gpurun_out/r2y/pytest_prune.log 2>&1; echo "rc=$?" >> gpurun_out/r2y/pytest_prune.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/r2y/launches_c5.csv python tools/prof_run.py c5 --reps 2 > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_full_parity.py -x -q -k "c5 or c2" > gpurun_out/r2y/pytest_full.log 2>&1; echo "rc=$?" >> gpurun_out/r2y/pytest_full.log
