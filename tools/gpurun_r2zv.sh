export OUT=gpurun_out/r2zv
mkdir -p $OUT
P="python tools/prof_run.py"
for lib in paper_2012_10684_b200/libtsa.so build_ab/libtsa_sp2.so build_ab/libtsa_sp1.so; do
  echo "== $lib"
  for w in c3 c4; do TSA_LIB_PATH=$lib timeout 120 $P $w --reps 12 | tail -4; done
  TSA_LIB_PATH=$lib timeout 300 python bench.py --workload c3 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3 sweep', d['ms_per_step'])"
  TSA_LIB_PATH=$lib timeout 300 python bench.py --workload c4 --steps 50 --warmup 3 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c4 bench', d['ms_per_step'])"
done > $OUT/ab_seed.txt 2>&1
for lib in paper_2012_10684_b200/libtsa.so build_ab/libtsa_g16.so; do echo "== $lib"; TSA_LIB_PATH=$lib timeout 300 python tools/ab_prune.py c5 --reps 20 | grep median; done > $OUT/ab_grid.txt 2>&1
TSA_LIB_PATH=build_ab/libtsa_g16.so timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $OUT/launches_c5_g16.csv python tools/prof_run.py c5 --reps 2 > /dev/null 2>&1
