export OUT=gpurun_out/r2zz2
mkdir -p $OUT
timeout 2400 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $OUT/smoke.log 2>&1; echo "rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench_c5.jsonl 2> $OUT/bench_c5.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches_c5_bench.csv python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
timeout 600 python bench.py --workload c2 --steps 2000 --warmup 20 > $OUT/bench_c2.jsonl 2> $OUT/bench_c2.err
timeout 900 python bench.py --workload c3 --steps 20 --warmup 3 --e2e-steps 2 > $OUT/bench_c3.jsonl 2> $OUT/bench_c3.err
timeout 900 python bench.py --workload c4 --steps 50 --warmup 3 --e2e-steps 2 > $OUT/bench_c4.jsonl 2> $OUT/bench_c4.err
