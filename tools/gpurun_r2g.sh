mkdir -p gpurun_out/r2g
P="python tools/prof_run.py"
{
timeout 120 $P c5 --pipeline staged --reps 4
TSA_LIB_PATH=$PWD/paper_2012_10684_b200/libtsa_k2b3.so timeout 120 $P c5 --pipeline staged --reps 4
timeout 120 $P c4 --reps 4
timeout 120 $P c3 --reps 4
timeout 120 $P c5 --pipeline stream --lag 32 --hc 4 --reps 3
} > gpurun_out/r2g/times.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/r2g/launches_c5.csv $P c5 --pipeline staged --reps 3 > /dev/null 2>&1
TSA_LIB_PATH=$PWD/paper_2012_10684_b200/libtsa_k2b3.so timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/r2g/launches_c5_b3.csv $P c5 --pipeline staged --reps 3 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r2g/launches_c4.csv $P c4 --reps 3 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r2g/launches_c3.csv $P c3 --reps 3 > /dev/null 2>&1
timeout 1200 python -m pytest tests/test_gpu_tri.py tests/test_gpu_parity.py tests/test_gpu_stream.py tests/test_gpu_full_parity.py tests/test_gpu_dist.py tests/test_gpu_bench_multirank.py -x -q > gpurun_out/r2g/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2g/pytest.log
