timeout 300 python -m pytest tests -m gpu -q -x -k "not config5 and not config_full_solve" > gpurun_out/gpu_tests10.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/gpu_tests10.log
timeout 300 python -m pytest tests -m gpu -q -x -k "config_full_solve and tma and not 4" -s > gpurun_out/gpu_tests10b.log 2>&1; echo tests rc=$?; grep -E "config|passed|failed" gpurun_out/gpu_tests10b.log | tail -5
for c in 5 3 2; do timeout 200 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b10_c$c.json 2>&1; done
