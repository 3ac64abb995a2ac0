timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "small_cases or config_full or batched or robin or stress" 2>&1 | tail -3
bash scripts/ab_env.sh 5 "HPFEM_HATS_ASYNC=0" "HPFEM_HATS_ASYNC=2" "HPFEM_HATS_ASYNC=3"
bash scripts/ab_env.sh 3 "HPFEM_HATS_ASYNC=0" "HPFEM_HATS_ASYNC=2" "HPFEM_HATS_ASYNC=3"
bash scripts/ab_env.sh 4 "HPFEM_HATS_ASYNC=0" "HPFEM_HATS_ASYNC=2" "HPFEM_HATS_ASYNC=3"
export HPFEM_NO_GRAPH=1
python scripts/prof_solve.py 5 2 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_hats_rows_t" -s 2 -c 1 -o gpurun_out/s3_hatst python scripts/prof_solve.py 5 2 > gpurun_out/s3_ncu_hatst.log 2>&1; echo full rc=$?
python scripts/ncu_summary.py gpurun_out/s3_hatst.ncu-rep
