mkdir -p gpurun_out/r2h
P="python tools/prof_run.py"
{ timeout 120 $P c4 --reps 4; timeout 120 $P c3 --reps 4; timeout 120 $P c4 --enumeration full --reps 2; } > gpurun_out/r2h/times.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r2h/launches_c4.csv $P c4 --reps 3 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r2h/launches_c3.csv $P c3 --reps 3 > /dev/null 2>&1
mkdir -p /tmp/ncu
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_search_tri -s 1 -c 1 -o /tmp/ncu/tri $P c4 --reps 2 > gpurun_out/r2h/ncu_tri.log 2>&1
ncu -i /tmp/ncu/tri.ncu-rep --page details --csv > gpurun_out/r2h/details_tri.csv 2>/dev/null
ncu -i /tmp/ncu/tri.ncu-rep --page raw --csv > gpurun_out/r2h/raw_tri.csv 2>/dev/null
ncu -i /tmp/ncu/tri.ncu-rep --page source --csv --print-source sass > /tmp/ncu/src_tri.csv 2>/dev/null
python tools/ncu_hot.py /tmp/ncu/src_tri.csv > gpurun_out/r2h/hot_tri.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_tri.py tests/test_gpu_parity.py tests/test_gpu_full_parity.py -x -q -k "tri or c3 or c4 or k3 or k4 or full or every or units or canonical" > gpurun_out/r2h/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2h/pytest.log
