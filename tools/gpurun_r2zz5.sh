OUT=gpurun_out/r2zz5
mkdir -p $OUT /tmp/ncu
P="python tools/prof_run.py"
prof() {  # name kernel-regex args...
  name=$1; kre=$2; shift 2
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$kre -s 1 -c 1 -o /tmp/ncu/$name "$@" \
      > $OUT/ncu_$name.log 2>&1
  ncu -i /tmp/ncu/$name.ncu-rep --page details --csv > $OUT/details_$name.csv 2>/dev/null
  ncu -i /tmp/ncu/$name.ncu-rep --page raw --csv > $OUT/raw_$name.csv 2>/dev/null
  ncu -i /tmp/ncu/$name.ncu-rep --page source --csv --print-source sass > /tmp/ncu/src_$name.csv 2>/dev/null
  python tools/ncu_hot.py /tmp/ncu/src_$name.csv > $OUT/hot_$name.txt 2>&1
}
prof k2_c5 k_search_k2 $P c5 --reps 2
prof scanseed_c5 k_scan_seed $P c5 --reps 2
prof label_c5 k_label_flat $P c5 --reps 2
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches_c5_bench.csv python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
timeout 900 python bench.py > $OUT/bench_c5.jsonl 2> $OUT/bench_c5.err
