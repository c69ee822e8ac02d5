mkdir -p gpurun_out/r2f
P="python tools/prof_run.py"
# timings of the stream kernel under a few schedules, and the staged path
for hc in 4 8 16; do for lag in 8 16 32; do timeout 120 $P c5 --pipeline stream --hc $hc --lag $lag --reps 3 2>&1 | tail -1; done; done > gpurun_out/r2f/stream_sweep.txt 2>&1
timeout 120 $P c5 --pipeline staged --reps 3 >> gpurun_out/r2f/stream_sweep.txt 2>&1
timeout 120 $P c4 --reps 3 >> gpurun_out/r2f/stream_sweep.txt 2>&1
timeout 120 $P c3 --reps 3 >> gpurun_out/r2f/stream_sweep.txt 2>&1
NCU="ncu --set full --import-source on --clock-control none"
timeout 600 $NCU -k regex:k_search_tri -s 1 -c 1 -o gpurun_out/r2f/tri_c4 $P c4 --reps 2 > gpurun_out/r2f/ncu_tri.log 2>&1
timeout 600 $NCU -k regex:k_search_k2 -s 1 -c 1 -o gpurun_out/r2f/k2_c5 $P c5 --pipeline staged --reps 2 > gpurun_out/r2f/ncu_k2.log 2>&1
timeout 600 $NCU -k regex:k_hist16 -s 1 -c 1 -o gpurun_out/r2f/h16_c5 $P c5 --pipeline staged --reps 2 > gpurun_out/r2f/ncu_h16.log 2>&1
timeout 900 $NCU -k regex:k_stream -s 1 -c 1 -o gpurun_out/r2f/stream_c5 $P c5 --pipeline stream --reps 2 --nz 300 > gpurun_out/r2f/ncu_stream.log 2>&1
