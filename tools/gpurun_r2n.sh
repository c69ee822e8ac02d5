mkdir -p gpurun_out/r2n /tmp/ncu
P="python tools/prof_run.py"
{ timeout 120 $P c4 --reps 4; timeout 120 $P c3 --reps 4; } > gpurun_out/r2n/times.txt 2>&1
for w in c4 c3; do timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r2n/launches_$w.csv $P $w --reps 3 > /dev/null 2>&1; done
prof() {  # name kernel-regex args...
  name=$1; kre=$2; shift 2
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$kre -s 1 -c 1 -o /tmp/ncu/$name $P "$@" > gpurun_out/r2n/ncu_$name.log 2>&1
  ncu -i /tmp/ncu/$name.ncu-rep --page details --csv > gpurun_out/r2n/details_$name.csv 2>/dev/null
  ncu -i /tmp/ncu/$name.ncu-rep --page raw --csv > gpurun_out/r2n/raw_$name.csv 2>/dev/null
  ncu -i /tmp/ncu/$name.ncu-rep --page source --csv --print-source sass > /tmp/ncu/src_$name.csv 2>/dev/null
  python tools/ncu_hot.py /tmp/ncu/src_$name.csv > gpurun_out/r2n/hot_$name.txt 2>&1
}
prof tri3 k_search_tri c3 --reps 2
prof tri4 k_search_tri c4 --reps 2
timeout 900 python -m pytest tests/test_gpu_tri.py tests/test_gpu_parity.py -x -q > gpurun_out/r2n/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2n/pytest.log
