mkdir -p gpurun_out/r2b
nproc > gpurun_out/r2b/nproc.txt; lscpu | grep "Model name" >> gpurun_out/r2b/nproc.txt
timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_full_parity.py -x -q --durations=20 > gpurun_out/r2b/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2b/pytest.log
