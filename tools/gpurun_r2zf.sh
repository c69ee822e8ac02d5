export OUT=gpurun_out/r2zf
mkdir -p $OUT
export TSA_LIB_PATH=build_ab/libtsa_ovl.so
P="python tools/prof_run.py"
{ timeout 100 $P c5 --reps 6;
  for lc in 2 3 4 6 8; do for sc in 1 2; do for G in 2 4; do
    echo "== label_ctas=$lc search_ctas=$sc G=$G"
    TSA_OVL_LABEL_CTAS=$lc TSA_OVL_SEARCH_CTAS=$sc timeout 100 $P c5 --reps 6 --pipeline overlap --hc $G | tail -3
  done; done; done; } > $OUT/overlap.txt 2>&1
