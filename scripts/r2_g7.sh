export HPFEM_NO_GRAPH=1
python scripts/prof_solve.py 4 2 > gpurun_out/ps4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_bubbles" -s 2 -c 2 -o gpurun_out/r2_cfg4_ldg python scripts/prof_solve.py 4 2 > gpurun_out/ncu_c4.log 2>&1; echo ncu rc=$?
tail -1 gpurun_out/ncu_c4.log
