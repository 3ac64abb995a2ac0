timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "small_cases or config_full or batched or robin or stress" 2>&1 | tail -3
bash scripts/ab_env.sh 5 "HPFEM_HATS_ASYNC=0" "HPFEM_HATS_ASYNC=1"
bash scripts/ab_env.sh 3 "HPFEM_HATS_ASYNC=0" "HPFEM_HATS_ASYNC=1"
export HPFEM_NO_GRAPH=1
python scripts/prof_solve.py 5 2 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_hats_rows_a|k_hats_cols_a" -s 2 -c 2 -o gpurun_out/s3_hatsa python scripts/prof_solve.py 5 2 > gpurun_out/s3_ncu_hatsa.log 2>&1; echo full rc=$?
python scripts/ncu_summary.py gpurun_out/s3_hatsa.ncu-rep
