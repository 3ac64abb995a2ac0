timeout 2400 python -m pytest tests -m gpu -q -s > gpurun_out/r2_gpu_full.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/r2_gpu_full.log
grep -E "^FAILED" gpurun_out/r2_gpu_full.log | head
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/r2_smoke.log
