export HPFEM_NO_GRAPH=1
python scripts/prof_solve.py 5 2 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_hats_rows|k_hats_cols|k_hatrows_y|k_hatcols_x" -s 4 -c 4 -o gpurun_out/s3_hats5 python scripts/prof_solve.py 5 2 > gpurun_out/s3_ncu_hats.log 2>&1; echo full rc=$?
python scripts/ncu_summary.py gpurun_out/s3_hats5.ncu-rep
