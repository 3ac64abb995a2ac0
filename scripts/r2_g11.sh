export HPFEM_NO_GRAPH=1
python scripts/prof_solve.py 4 2 > gpurun_out/ps4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_xstep_tma" -s 1 -c 1 -o gpurun_out/r2_x128 python scripts/prof_solve.py 4 2 > gpurun_out/ncu_x128.log 2>&1; echo ncu rc=$?
