timeout 900 python -m pytest tests -m gpu -q -x -k "not config5 and not config_full_solve" > gpurun_out/gpu_tests3.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/gpu_tests3.log
for c in 5 4 3 2; do python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b2_c$c.json 2>&1; done
HPFEM_BUBBLE_KERNEL=reg python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b2reg_c5.json 2>&1
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_bubbles|k_hats" -s 4 -c 4 -o gpurun_out/prof2_c5 $CMD > gpurun_out/ncu4.log 2>&1; echo ncu rc=$?
