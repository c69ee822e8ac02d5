mkdir -p gpurun_out/r2d
timeout 600 python -m pytest tests/test_gpu_stream.py -x -q > gpurun_out/r2d/pytest_stream.log 2>&1; echo "rc=$?" >> gpurun_out/r2d/pytest_stream.log
timeout 300 python bench.py --steps 100 --e2e-steps 3 --no-cpu-baseline > gpurun_out/r2d/bench_c5.jsonl 2> gpurun_out/r2d/bench_c5.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/r2d/launches_c5.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_full_parity.py -x -q -k "c5" > gpurun_out/r2d/pytest_c5.log 2>&1; echo "rc=$?" >> gpurun_out/r2d/pytest_c5.log
