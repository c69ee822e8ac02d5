set -u
T=r1z
mkdir -p gpurun_out/$T
nvidia-smi > gpurun_out/$T/nvsmi.txt 2>&1
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/$T/gpu_tests.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/$T/smoke.log 2>&1
timeout 1500 bash tools/collect_profiles.sh $T
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/$T/ref_c2.jsonl 2>gpurun_out/$T/ref_c2.err
timeout 300 python bench.py --impl reference --workload f1 --steps 3 --warmup 3 > gpurun_out/$T/ref_f1.jsonl 2>gpurun_out/$T/ref_f1.err
for r in prof_c2 prof_c4full prof_c4dp prof_f1 prof_f3; do
  if [ -f gpurun_out/$T/$r.ncu-rep ]; then
    python tools/ncu_summary.py full gpurun_out/$T/$r.ncu-rep gpurun_out/$T/ncu_full_$r.md > /dev/null 2>&1
    ncu -i gpurun_out/$T/$r.ncu-rep --page raw --csv > gpurun_out/$T/raw_$r.csv 2>/dev/null
    rm -f gpurun_out/$T/$r.ncu-rep
  fi
done
for l in launches_c2 launches_c4_dp launches_f1; do
  python tools/ncu_summary.py launches gpurun_out/$T/$l.csv gpurun_out/$T/$l.md > /dev/null 2>&1
done
du -sh gpurun_out/$T
tail -2 gpurun_out/$T/gpu_tests.log
