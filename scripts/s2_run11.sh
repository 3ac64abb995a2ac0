timeout 900 python -m pytest tests/test_gpu_varcoef.py -x -q > gpurun_out/s2_t11.log 2>&1; echo tests rc=$?
tail -2 gpurun_out/s2_t11.log
timeout 300 python scripts/bench_pcg.py --shapes 3:128 --fp64-peak 34.19 | cut -c1-400
timeout 300 python scripts/bench_burgers.py --shapes 9:128,36:128,72:64 | cut -c1-300
