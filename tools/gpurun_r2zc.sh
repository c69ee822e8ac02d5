export OUT=gpurun_out/r2zc
mkdir -p $OUT
P="python tools/prof_run.py"
{ timeout 300 python tools/ab_prune.py c5 --reps 20; timeout 120 $P c4 --reps 6; timeout 120 $P c3 --reps 6; } > $OUT/times.txt 2>&1
for w in c5 c4 c3; do timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $OUT/launches_$w.csv $P $w --reps 2 > /dev/null 2>&1; done
timeout 900 python -m pytest tests/test_gpu_prune.py tests/test_gpu_tri.py tests/test_gpu_parity.py -x -q > $OUT/pytest_a.log 2>&1; echo "rc=$?" >> $OUT/pytest_a.log
timeout 1500 python -m pytest tests/test_gpu_full_parity.py -x -q > $OUT/pytest_full.log 2>&1; echo "rc=$?" >> $OUT/pytest_full.log
tools/ncu_prof.sh c5 "c5 --reps 3" k_search_k2
tools/ncu_prof.sh c4 "c4 --reps 3" k_search_tri k_tri_tables
