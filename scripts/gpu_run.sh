CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"tma|hatrows|hatcols|k_hats" -s 12 -c 6 -o gpurun_out/prof6_c5 $CMD > gpurun_out/ncu9.log 2>&1; echo ncu rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none -s 2938 -c 978 --csv --log-file gpurun_out/launches_c5_v6.csv $CMD > gpurun_out/ncu10.log 2>&1; echo ncu2 rc=$?
