timeout 300 python -m pytest tests -m gpu -q -x -k "not config5 and not config_full_solve" > gpurun_out/gpu_tests13.log 2>&1; echo tests rc=$?; tail -1 gpurun_out/gpu_tests13.log
timeout 300 python -m pytest tests -m gpu -q -x -k "config_full_solve and tma and (2 or 3)" -s 2>&1 | grep -E "config|passed|failed|Error" | tail -4
for c in 5 3; do timeout 200 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b13_c$c.json 2>&1; done
