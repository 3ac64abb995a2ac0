timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_varcoef.py -x -q -k "apply or varcoef" 2>&1 | tail -2
python scripts/bench_apply.py 2 3 4 5
