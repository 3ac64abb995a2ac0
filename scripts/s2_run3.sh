timeout 900 python -m pytest tests/test_gpu_varcoef.py -x -q -s -k "imex or pcg_edge" > gpurun_out/s2_t3.log 2>&1; echo tests rc=$?
grep -v "^$" gpurun_out/s2_t3.log | tail -40
