export OUT=gpurun_out/r2zw
mkdir -p $OUT
timeout 300 python tools/scan_trace.py c5 > $OUT/scan_trace_c5.txt 2>&1
timeout 300 python tools/fused_trace.py c2 compact > $OUT/trace_c2.txt 2>&1
