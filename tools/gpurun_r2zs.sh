export OUT=gpurun_out/r2zs
mkdir -p $OUT
for i in 1 2; do timeout 300 python tools/fused_trace.py c2 compact; done > $OUT/trace_c2.txt 2>&1
