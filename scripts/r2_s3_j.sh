timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "small_cases and (19 or 20 or 21 or 22)" 2>&1 | tail -2
bash scripts/ab_env.sh 4 "HPFEM_NST_X=4" "HPFEM_NST_X=5" "HPFEM_NST_X=6" "HPFEM_NST_X=3"
