timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -s -k "small_cases or config_full_solve or robin_cases" --deselect "tests/test_gpu_parity.py::test_config_full_solve[transposed-4]" > gpurun_out/r2_t9.log 2>&1; echo tests rc=$?; tail -1 gpurun_out/r2_t9.log
grep -E "case (19|20)|config 4" gpurun_out/r2_t9.log | head -12
bash scripts/ab_cmp.sh 4 1
