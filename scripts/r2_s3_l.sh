export HPFEM_NO_GRAPH=1
python scripts/prof_solve.py 5 2 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_ystep_tma|k_xstep_tma" -s 3 -c 2 -o gpurun_out/s3_xy5 python scripts/prof_solve.py 5 2 > gpurun_out/s3_ncu_xy5.log 2>&1; echo full rc=$?
python scripts/ncu_summary.py gpurun_out/s3_xy5.ncu-rep
python scripts/ncu_lines.py gpurun_out/s3_xy5.ncu-rep k_ystep_tma 40
