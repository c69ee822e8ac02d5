export OUT=gpurun_out/r2zr
mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -x -q > $OUT/pytest_a.log 2>&1; echo "rc=$?" >> $OUT/pytest_a.log
for sl in 25 50; do timeout 300 python bench.py --workload c2 --steps 300 --warmup 5 --e2e-steps 10 --e2e-slab $sl --no-cpu-baseline > $OUT/bench_c2_slab$sl.jsonl 2>/dev/null; done
for sl in 13 25 50; do timeout 300 python bench.py --workload c5 --steps 20 --warmup 3 --e2e-steps 4 --e2e-slab $sl --no-cpu-baseline > $OUT/bench_c5_slab$sl.jsonl 2>/dev/null; done
for f in $OUT/bench_*.jsonl; do python -c "import json; d=json.loads(open('$f').read()); print('$f', d['value'], d['e2e']['value'])"; done > $OUT/e2e_summary.txt 2>&1
