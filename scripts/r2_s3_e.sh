timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "small_cases or config_full or batched or robin or stress" 2>&1 | tail -3
bash scripts/ab_env.sh 5 "HPFEM_HATS_ASYNC=0 HPFEM_NO_HAT_SPLIT=1" "HPFEM_HATS_ASYNC=0" "HPFEM_HATS_ASYNC=1"
bash scripts/ab_env.sh 3 "HPFEM_HATS_ASYNC=0 HPFEM_NO_HAT_SPLIT=1" "HPFEM_HATS_ASYNC=0" "HPFEM_HATS_ASYNC=1"
bash scripts/ab_env.sh 4 "HPFEM_HATS_ASYNC=0 HPFEM_NO_HAT_SPLIT=1" "HPFEM_HATS_ASYNC=0" "HPFEM_HATS_ASYNC=1"
bash scripts/ab_env.sh 2 "HPFEM_HATS_ASYNC=0 HPFEM_NO_HAT_SPLIT=1" "HPFEM_HATS_ASYNC=0" "HPFEM_HATS_ASYNC=1"
