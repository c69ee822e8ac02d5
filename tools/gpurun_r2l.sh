mkdir -p gpurun_out/r2l
P="python tools/prof_run.py"
{ timeout 120 $P c5 --pipeline staged --reps 4; for sl in 2 4 8 16; do timeout 120 $P c5 --pipeline overlap --hc $sl --reps 3 | tail -1; done
  timeout 120 $P c5 --pipeline stream --reps 3 | tail -1; timeout 120 $P c2 --pipeline stream --reps 3 | tail -1; timeout 120 $P c2 --reps 3 | tail -1; } > gpurun_out/r2l/times.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r2l/launches_c5.csv $P c5 --pipeline staged --reps 3 > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_overlap.py tests/test_gpu_tri.py tests/test_gpu_stream.py tests/test_gpu_parity.py tests/test_gpu_dist.py -x -q > gpurun_out/r2l/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2l/pytest.log
