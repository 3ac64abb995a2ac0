export HPFEM_NO_GRAPH=1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_ystep_tma" -s 2 -c 1 -o gpurun_out/s2_ystep python scripts/yprof_run.py > gpurun_out/s2_ncu_y.log 2>&1; echo ncu rc=$?
tail -3 gpurun_out/s2_ncu_y.log
python scripts/ncu_hot.py gpurun_out/s2_ystep.ncu-rep k_ystep 0 40 > gpurun_out/s2_yhot.txt 2>&1; head -45 gpurun_out/s2_yhot.txt
