bash scripts/ab_env.sh 5 "HPFEM_NO_HAT_SPLIT=1 HPFEM_HATS_ASYNC=0" "HPFEM_NO_HAT_SPLIT=1 HPFEM_HATS_ASYNC=2" "HPFEM_NO_HAT_SPLIT=1 HPFEM_HATS_ASYNC=1"
export HPFEM_NO_GRAPH=1
python scripts/prof_solve.py 5 2 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_hats_rows_t" -s 1 -c 1 -o gpurun_out/s3_hatst5 python scripts/prof_solve.py 5 2 > gpurun_out/s3_ncu_hatst5.log 2>&1; echo full rc=$?
python scripts/ncu_summary.py gpurun_out/s3_hatst5.ncu-rep
python scripts/ncu_lines.py gpurun_out/s3_hatst5.ncu-rep k_hats_rows_t 40
