mkdir -p gpurun_out/r2w
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2w/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2w/smoke.log
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r2w/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/r2w/pytest_gpu.log
timeout 2400 bash tools/sanitize.sh gpurun_out/r2w/sanitizer > /dev/null 2>&1
