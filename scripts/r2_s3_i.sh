export HPFEM_NO_GRAPH=1
python scripts/prof_solve.py 4 2 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_xstep_tma2" -s 2 -c 1 -o gpurun_out/s3_x2 python scripts/prof_solve.py 4 2 > gpurun_out/s3_ncu_x2.log 2>&1; echo full rc=$?
python scripts/ncu_summary.py gpurun_out/s3_x2.ncu-rep
python scripts/ncu_lines.py gpurun_out/s3_x2.ncu-rep k_xstep_tma2 25
