mkdir -p gpurun_out/r2m
P="python tools/prof_run.py"
{ timeout 120 $P c5 --reps 4; timeout 120 $P c4 --reps 4; timeout 120 $P c3 --reps 4; timeout 120 $P c2 --reps 3; } > gpurun_out/r2m/times.txt 2>&1
for w in c5 c4 c3; do timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r2m/launches_$w.csv $P $w --reps 3 > /dev/null 2>&1; done
timeout 900 python -m pytest tests/test_gpu_overlap.py tests/test_gpu_tri.py tests/test_gpu_stream.py tests/test_gpu_parity.py tests/test_gpu_dist.py -x -q > gpurun_out/r2m/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2m/pytest.log
