timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "small_cases and (19 or 20 or 21 or 22)" 2>&1 | tail -2
for nst in 3 4 2; do HPFEM_NST_X=$nst bash scripts/ab_cmp.sh 4 1; done
