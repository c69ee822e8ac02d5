export OUT=gpurun_out/r2zq
mkdir -p $OUT
P="python tools/prof_run.py"
{ for lib in paper_2012_10684_b200/libtsa.so build_ab/libtsa_q32.so; do echo "== $lib"; TSA_LIB_PATH=$lib timeout 120 $P c4 --reps 12 | tail -3; done
  for ss in 1 2 4 8; do echo "== c3 ss=$ss"; TSA_TRI_SS=$ss timeout 120 $P c3 --reps 12 | tail -3; done
  for ss in 2 4 8; do echo "== c4 ss=$ss"; TSA_TRI_SS=$ss timeout 120 $P c4 --reps 12 | tail -3; done; } > $OUT/ab.txt 2>&1
