export OUT=gpurun_out/r2za
mkdir -p $OUT
tools/ncu_prof.sh c4 "c4 --reps 3" k_search_tri k_tri_tables
tools/ncu_prof.sh c5 "c5 --reps 3" k_finalize k_k2_seed k_scan
tools/ncu_prof.sh c3 "c3 --reps 3" k_tri_tables
ls -la $OUT
