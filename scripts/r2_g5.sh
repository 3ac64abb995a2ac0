export HPFEM_NO_GRAPH=1
for lib in ab/base.so paper_2402_11299_b200/libhpfem_b200.so; do
  n=$(basename $lib .so)
  HPFEM_LIB_PATH=$lib python scripts/prof_solve.py 5 3 > gpurun_out/ps_$n.log 2>&1 && \
  HPFEM_LIB_PATH=$lib ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2_l5_$n.csv python scripts/prof_solve.py 5 3 > /dev/null 2>&1
  python scripts/launch_summary.py gpurun_out/r2_l5_$n.csv | head -12
done
