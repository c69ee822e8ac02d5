mkdir -p gpurun_out/r2f /tmp/ncu
P="python tools/prof_run.py"
for hc in 4 8 16; do for lag in 8 16 32; do timeout 120 $P c5 --pipeline stream --hc $hc --lag $lag --reps 3 2>&1 | tail -1; done; done > gpurun_out/r2f/stream_sweep.txt 2>&1
timeout 120 $P c5 --pipeline staged --reps 3 >> gpurun_out/r2f/stream_sweep.txt 2>&1
timeout 120 $P c4 --reps 3 >> gpurun_out/r2f/stream_sweep.txt 2>&1
timeout 120 $P c3 --reps 3 >> gpurun_out/r2f/stream_sweep.txt 2>&1
NCU="ncu --set full --import-source on --clock-control none"
prof() {  # name kernel-regex args...
  name=$1; kre=$2; shift 2
  timeout 900 $NCU -k regex:$kre -s 1 -c 1 -o /tmp/ncu/$name $P "$@" > gpurun_out/r2f/ncu_$name.log 2>&1
  ncu -i /tmp/ncu/$name.ncu-rep --page details --csv > gpurun_out/r2f/details_$name.csv 2>/dev/null
  ncu -i /tmp/ncu/$name.ncu-rep --page raw --csv > gpurun_out/r2f/raw_$name.csv 2>/dev/null
  ncu -i /tmp/ncu/$name.ncu-rep --page source --csv --print-source sass > /tmp/ncu/src_$name.csv 2>/dev/null
  python tools/ncu_hot.py /tmp/ncu/src_$name.csv > gpurun_out/r2f/hot_$name.txt 2>&1
}
prof tri_c4 k_search_tri c4 --reps 2
prof k2_c5 k_search_k2 c5 --pipeline staged --reps 2
prof h16_c5 k_hist16 c5 --pipeline staged --reps 2
prof stream_c5 k_stream c5 --pipeline stream --reps 2 --nz 300
du -sh gpurun_out
