mkdir -p gpurun_out/r2r /tmp/ncu
P="python tools/prof_run.py"
prof() {
  name=$1; kre=$2; shift 2
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$kre -s 1 -c 1 -o /tmp/ncu/$name $P "$@" > gpurun_out/r2r/ncu_$name.log 2>&1
  ncu -i /tmp/ncu/$name.ncu-rep --page source --csv --print-source sass > /tmp/ncu/src_$name.csv 2>/dev/null
  python tools/ncu_hot.py /tmp/ncu/src_$name.csv > gpurun_out/r2r/hot_$name.txt 2>&1
  ncu -i /tmp/ncu/$name.ncu-rep --page raw --csv > gpurun_out/r2r/raw_$name.csv 2>/dev/null
}
prof tri4 k_search_tri c4 --reps 2
prof k2 k_search_k2 c5 --reps 2
