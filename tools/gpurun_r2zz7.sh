export OUT=gpurun_out/r2zz7
mkdir -p $OUT
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $OUT/smoke.log 2>&1; echo "rc=$?" >> $OUT/smoke.log
timeout 900 python -m pytest tests/test_gpu_prune.py tests/test_gpu_parity.py tests/test_abi.py -q > $OUT/pytest_a.log 2>&1; echo "rc=$?" >> $OUT/pytest_a.log
timeout 600 python bench.py --steps 100 --warmup 5 > $OUT/bench_c5.jsonl 2> $OUT/bench_c5.err
