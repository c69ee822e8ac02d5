mkdir -p gpurun_out/r2x
P="python tools/prof_run.py"
cat > /tmp/san_stream.py <<'PY'
import sys, os
sys.path.insert(0, os.getcwd())
import torch, phantom, paper_2012_10684_b200 as tsa
v5 = torch.from_numpy(phantom.make_volume(phantom.CONFIGS["c5"], nz=3, z_first=400)).cuda()
tsa.tsa_segment(v5, 4096, 2, 0.8, pipeline="stream")
tsa.tsa_segment(v5, 4096, 2, 0.8)
torch.cuda.synchronize(); print("ok")
PY
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python /tmp/san_stream.py > gpurun_out/r2x/racecheck_stream.log 2>&1; echo "racecheck exit=$?" >> gpurun_out/r2x/racecheck_stream.log
{ timeout 120 $P c5 --reps 4; timeout 120 $P c3 --reps 4; timeout 120 $P c4 --reps 4; } > gpurun_out/r2x/times.txt 2>&1
for w in c5 c3; do timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r2x/launches_$w.csv $P $w --reps 3 > /dev/null 2>&1; done
for sl in 10 20 30 50; do timeout 300 python bench.py --workload c2 --steps 200 --warmup 5 --e2e-steps 10 --e2e-slab $sl --no-cpu-baseline > gpurun_out/r2x/bench_c2_slab$sl.jsonl 2>/dev/null; done
for sl in 10 25 50; do timeout 300 python bench.py --workload c5 --steps 50 --warmup 3 --e2e-steps 4 --e2e-slab $sl --no-cpu-baseline > gpurun_out/r2x/bench_c5_slab$sl.jsonl 2>/dev/null; done
timeout 1200 python -m pytest tests/test_gpu_stream.py tests/test_gpu_full_parity.py tests/test_gpu_parity.py tests/test_gpu_tri.py -x -q > gpurun_out/r2x/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2x/pytest.log
