mkdir -p gpurun_out/r2j /tmp/ncu
P="python tools/prof_run.py"
prof() {  # name kernel-regex args...
  name=$1; kre=$2; shift 2
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$kre -s 1 -c 1 -o /tmp/ncu/$name $P "$@" > gpurun_out/r2j/ncu_$name.log 2>&1
  ncu -i /tmp/ncu/$name.ncu-rep --page details --csv > gpurun_out/r2j/details_$name.csv 2>/dev/null
  ncu -i /tmp/ncu/$name.ncu-rep --page raw --csv > gpurun_out/r2j/raw_$name.csv 2>/dev/null
  ncu -i /tmp/ncu/$name.ncu-rep --page source --csv --print-source sass > /tmp/ncu/src_$name.csv 2>/dev/null
  python tools/ncu_hot.py /tmp/ncu/src_$name.csv > gpurun_out/r2j/hot_$name.txt 2>&1
}
prof tri4 k_search_tri c4 --reps 2
prof stream c5_stream k_stream c5 --pipeline stream --reps 2 --nz 300 2>/dev/null
prof st5 k_stream c5 --pipeline stream --reps 2 --nz 300
prof scan5 k_scan c5 --pipeline staged --reps 2
prof fin5 k_finalize c5 --pipeline staged --reps 2
