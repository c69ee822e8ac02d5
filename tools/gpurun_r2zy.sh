export OUT=gpurun_out/r2zy
mkdir -p $OUT
timeout 2400 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $OUT/smoke.log 2>&1; echo "rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench_c5.jsonl 2> $OUT/bench_c5.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/ref_c5.jsonl 2> $OUT/ref_c5.err
