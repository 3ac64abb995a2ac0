timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_varcoef.py -x -q -k "apply or varcoef or pcg or imex or robin or errors" 2>&1 | tail -3
python scripts/bench_apply.py 2 3 4 5
python scripts/bench_pcg.py 2>/dev/null | tail -4 | cut -c1-300
