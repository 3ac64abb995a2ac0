timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t31.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/t31.log
python bench.py > gpurun_out/b31_full.json 2> gpurun_out/b31_full.err; echo bench rc=$?
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum --clock-control none -s 2938 -c 978 --csv --log-file gpurun_out/launches_c5_v7.csv $CMD > gpurun_out/ncu31a.log 2>&1; echo ncu1 rc=$?
ncu --set full --clock-control none --import-source on -k regex:"tma|hatrows|hatcols|k_hats" -s 12 -c 6 -o gpurun_out/prof7_c5 $CMD > gpurun_out/ncu31b.log 2>&1; echo ncu2 rc=$?
