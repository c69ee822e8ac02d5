mkdir -p gpurun_out/r2e
timeout 300 python -m pytest tests/test_gpu_stream.py -x -q > gpurun_out/r2e/pytest_stream.log 2>&1; echo "rc=$?" >> gpurun_out/r2e/pytest_stream.log
timeout 900 python -m pytest tests/test_gpu_tri.py tests/test_gpu_parity.py tests/test_gpu_dp.py tests/test_gpu_dist.py -x -q > gpurun_out/r2e/pytest_parity.log 2>&1; echo "rc=$?" >> gpurun_out/r2e/pytest_parity.log
for w in c5 c3 c4; do timeout 300 python bench.py --workload $w --steps 50 --e2e-steps 2 --no-cpu-baseline > gpurun_out/r2e/bench_$w.jsonl 2> gpurun_out/r2e/bench_$w.err; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/r2e/launches_c5.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r2e/launches_c4.csv python bench.py --workload c4 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
