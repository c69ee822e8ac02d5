mkdir -p gpurun_out/r2v
timeout 600 python bench.py --workload c3 --steps 20 --warmup 3 --e2e-steps 2 --no-cpu-baseline > gpurun_out/r2v/bench_c3.jsonl 2> gpurun_out/r2v/bench_c3.err
timeout 600 python bench.py --workload c1 --steps 2000 --warmup 20 --no-cpu-baseline > gpurun_out/r2v/bench_c1.jsonl 2> gpurun_out/r2v/bench_c1.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/r2v/launches_c3_sweep.csv python bench.py --workload c3 --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
timeout 1200 python -m pytest tests/test_gpu_full_parity.py tests/test_gpu_parity.py tests/test_gpu_tri.py -x -q > gpurun_out/r2v/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2v/pytest.log
