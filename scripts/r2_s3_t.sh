ncu --set full --clock-control none --import-source on -k regex:"k_apply2d" -s 2 -c 2 -o gpurun_out/s3_apply python scripts/bench_apply.py 5 > gpurun_out/s3_ncu_apply.log 2>&1; echo rc=$?
python scripts/ncu_summary.py gpurun_out/s3_apply.ncu-rep
python scripts/ncu_lines.py gpurun_out/s3_apply.ncu-rep k_apply2d_chain 14
