timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "small_cases or (config_full and 4) or stress" 2>&1 | tail -5
bash scripts/ab_env.sh 4 "HPFEM_NO_X2=1" "HPFEM_NO_X2=0"
