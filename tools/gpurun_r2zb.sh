export OUT=gpurun_out/r2zb
mkdir -p $OUT
P="python tools/prof_run.py"
{ timeout 120 $P c5 --reps 8; for hc in 2 4 8 16 32; do timeout 120 $P c5 --reps 8 --pipeline overlap --hc $hc; done; } > $OUT/overlap.txt 2>&1
tools/ncu_prof.sh c5 "c5 --reps 3" k_search_k2
ls -la $OUT
