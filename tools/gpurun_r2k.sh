mkdir -p gpurun_out/r2k
P="python tools/prof_run.py"
{ timeout 120 $P c5 --reps 4; for sl in 4 16 32; do timeout 120 $P c5 --pipeline overlap --hc $sl --reps 3 | tail -1; done
  timeout 120 $P c5 --pipeline staged --reps 3; timeout 120 $P c4 --reps 4; timeout 120 $P c3 --reps 4; } > gpurun_out/r2k/times.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r2k/launches_c4.csv $P c4 --reps 3 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r2k/launches_c3.csv $P c3 --reps 3 > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_overlap.py tests/test_gpu_tri.py tests/test_gpu_stream.py tests/test_gpu_parity.py -x -q > gpurun_out/r2k/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2k/pytest.log
