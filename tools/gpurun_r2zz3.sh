export OUT=gpurun_out/r2zz3
mkdir -p $OUT
timeout 300 python tools/scan_trace.py c5 > $OUT/scan_trace_c5.txt 2>&1
