timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "solve1d" 2>&1 | tail -3
timeout 300 python scripts/bench_1d.py > gpurun_out/fig1_1d.jsonl 2>&1; echo bench1d rc=$?; cat gpurun_out/fig1_1d.jsonl
