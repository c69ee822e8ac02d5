mkdir -p gpurun_out/r2c
timeout 600 python bench.py > gpurun_out/r2c/bench_default.jsonl 2> gpurun_out/r2c/bench_default.err
for w in c3 c4 c2; do timeout 400 python bench.py --workload $w --steps 50 > gpurun_out/r2c/bench_$w.jsonl 2> gpurun_out/r2c/bench_$w.err; done
timeout 300 python bench.py --workload c4 --shard tuples --steps 20 > gpurun_out/r2c/bench_c4_tuples.jsonl 2> gpurun_out/r2c/bench_c4_tuples.err
timeout 400 python bench.py --impl reference --steps 50 --warmup 5 > gpurun_out/r2c/ref_default.jsonl 2> gpurun_out/r2c/ref_default.err
