export OUT=gpurun_out/r2zo
mkdir -p $OUT
P="python tools/prof_run.py"
{ for w in c3 c4; do timeout 300 python tools/ab_prune.py $w --reps 20 --var TSA_TRI_STAGE; done
  for v in 1 0; do TSA_TRI_STAGE=$v timeout 300 python bench.py --workload c3 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3 sweep stage=$v', d['ms_per_step'])"; done; } > $OUT/ab_stage.txt 2>&1
for v in 1 0; do TSA_TRI_STAGE=$v timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $OUT/launches_c4_stage$v.csv $P c4 --reps 2 > /dev/null 2>&1; done
TSA_TRI_STAGE=0 timeout 900 python -m pytest tests/test_gpu_tri.py tests/test_gpu_prune.py -x -q > $OUT/pytest_a.log 2>&1; echo "rc=$?" >> $OUT/pytest_a.log
