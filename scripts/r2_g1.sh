set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -s -k "small_cases or many_hats or two_host or config_load or config_apply or config_unload or config_plan" > gpurun_out/r2_t1.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/r2_t1.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2_b1.log 2>&1; echo bench rc=$?
tail -1 gpurun_out/r2_b1.log | cut -c1-600
