timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "stress or (config_full and (2 or 4))" 2>&1 | tail -1
bash scripts/ab_cmp.sh 2 3
bash scripts/ab_cmp.sh 3 2
bash scripts/ab_cmp.sh 5 1
