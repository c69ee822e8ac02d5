export OUT=gpurun_out/r2zg
mkdir -p $OUT
P="python tools/prof_run.py"
{ timeout 300 python tools/ab_prune.py c5 --reps 20; } > $OUT/times.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $OUT/launches_c5.csv $P c5 --reps 2 > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_prune.py -x -q > $OUT/pytest_a.log 2>&1; echo "rc=$?" >> $OUT/pytest_a.log
tools/ncu_prof.sh c5 "c5 --reps 3" k_search_k2
