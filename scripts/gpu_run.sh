timeout 300 python -m pytest tests -m gpu -q -x -k "small_cases or config_plan or (config_full_solve and tma and not 4)" > gpurun_out/gpu_tests19.log 2>&1; echo tests rc=$?; tail -1 gpurun_out/gpu_tests19.log; grep -E "Error|assert" gpurun_out/gpu_tests19.log | head
run() { timeout 120 python scripts/diag_launch.py $1 2>&1 | tail -1; }
for c in 5 3; do echo cfg $c; run $c; done
