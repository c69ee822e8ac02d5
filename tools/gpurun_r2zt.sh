export OUT=gpurun_out/r2zt
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_hu.py tests/test_gpu_prune.py tests/test_gpu_stream.py -x -q > $OUT/pytest_a.log 2>&1; echo "rc=$?" >> $OUT/pytest_a.log
timeout 900 python -m pytest tests/test_gpu_full_parity.py -x -q -k "c1 or c2" > $OUT/pytest_full.log 2>&1; echo "rc=$?" >> $OUT/pytest_full.log
timeout 300 python bench.py --workload c2 --steps 2000 --warmup 20 --no-cpu-baseline > $OUT/bench_c2.jsonl 2>/dev/null
timeout 300 python bench.py --workload f2 --steps 300 --no-cpu-baseline > $OUT/bench_f2.jsonl 2>/dev/null
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $OUT/launches_c2.csv python tools/prof_run.py c2 --reps 2 > /dev/null 2>&1
for f in $OUT/bench_*.jsonl; do python -c "import json; d=json.loads(open('$f').read()); print('$f', d['value'], d['ms_per_step'], d['e2e']['value'] if d.get('e2e') else None)"; done > $OUT/summary.txt 2>&1
