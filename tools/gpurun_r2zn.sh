export OUT=gpurun_out/r2zn
mkdir -p $OUT
P="python tools/prof_run.py"
for lib in paper_2012_10684_b200/libtsa.so build_ab/libtsa_tt.so; do
  echo "== $lib"
  for w in c3 c4; do TSA_LIB_PATH=$lib timeout 120 $P $w --reps 12 | tail -3; done
  TSA_LIB_PATH=$lib timeout 300 python bench.py --workload c3 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3 sweep', d['ms_per_step'])"
done > $OUT/ab_tt.txt 2>&1
export TSA_LIB_PATH=build_ab/libtsa_tt.so
for w in c3 c4; do timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $OUT/launches_$w.csv $P $w --reps 2 > /dev/null 2>&1; done
timeout 900 python -m pytest tests/test_gpu_tri.py tests/test_gpu_prune.py tests/test_gpu_parity.py -x -q > $OUT/pytest_a.log 2>&1; echo "rc=$?" >> $OUT/pytest_a.log
timeout 1200 python -m pytest tests/test_gpu_full_parity.py -x -q -k "c3 or c4 or sweep" > $OUT/pytest_full.log 2>&1; echo "rc=$?" >> $OUT/pytest_full.log
tools/ncu_prof.sh c4 "c4 --reps 3" k_search_tri k_tri_tables
unset TSA_LIB_PATH
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_mid -s 2 -c 1 -f -o /tmp/ncu/mid python tools/prof_run.py c2 --reps 3 > /dev/null 2>&1
ncu -i /tmp/ncu/mid.ncu-rep --page source --csv --print-source cuda > $OUT/mid_cuda.csv 2>/dev/null
ncu -i /tmp/ncu/mid.ncu-rep --page details --csv > $OUT/mid_details.csv 2>/dev/null
