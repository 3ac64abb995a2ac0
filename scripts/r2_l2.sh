HPFEM_L2_KEEP=1 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "(config_full and (2 or 3)) or (small_cases and (17 or 20))" 2>&1 | tail -1
bash scripts/ab_env.sh 5 "HPFEM_L2_KEEP=0" "HPFEM_L2_KEEP=1" "HPFEM_L2_KEEP=0" "HPFEM_L2_KEEP=1"
bash scripts/ab_env.sh 3 "HPFEM_L2_KEEP=0" "HPFEM_L2_KEEP=1"
bash scripts/ab_env.sh 4 "HPFEM_L2_KEEP=0" "HPFEM_L2_KEEP=1"
