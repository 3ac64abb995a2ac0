export HPFEM_NO_GRAPH=1
python scripts/prof_solve.py 5 2 > gpurun_out/ps.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_hats" -s 4 -c 2 -o gpurun_out/r2_hats python scripts/prof_solve.py 5 2 > gpurun_out/ncu_hats.log 2>&1; echo ncu rc=$?
tail -2 gpurun_out/ncu_hats.log
