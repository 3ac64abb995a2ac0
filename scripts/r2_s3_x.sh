timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "small_cases or stress or robin or mixed or many_hats or (config_full and (2 or 3))" 2>&1 | tail -2
bash scripts/ab_cmp.sh 5 2
bash scripts/ab_cmp.sh 3 2
bash scripts/ab_cmp.sh 4 1
