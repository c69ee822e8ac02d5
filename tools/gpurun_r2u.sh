mkdir -p gpurun_out/r2u
P="python tools/prof_run.py"
{ timeout 120 $P c5 --reps 4; timeout 120 $P c4 --reps 4; timeout 120 $P c3 --reps 4; } > gpurun_out/r2u/times.txt 2>&1
for w in c5 c4 c3; do timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r2u/launches_$w.csv $P $w --reps 3 > /dev/null 2>&1; done
M=gpu__time_duration.sum,sm__sass_thread_inst_executed_op_fp64_pred_on.sum,sm__inst_executed_pipe_fp64.sum,sm__inst_executed.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active
for w in c5 c4 c3; do timeout 300 ncu --metrics $M --clock-control none -k regex:"k_search" -c 2 --csv --log-file gpurun_out/r2u/fp64_$w.csv $P $w --reps 1 > /dev/null 2>&1; done
timeout 1200 python -m pytest tests/test_gpu_tri.py tests/test_gpu_parity.py tests/test_gpu_full_parity.py tests/test_gpu_stream.py tests/test_gpu_overlap.py -x -q > gpurun_out/r2u/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2u/pytest.log
