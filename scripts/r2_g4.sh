timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "small_cases or config_full_solve or robin_cases or many_hats or batched or mixed" --deselect "tests/test_gpu_parity.py::test_config_full_solve[small-4]" --deselect "tests/test_gpu_parity.py::test_config_full_solve[tma-4]" --deselect "tests/test_gpu_parity.py::test_config_full_solve[ldg-4]" > gpurun_out/r2_t4.log 2>&1; echo tests rc=$?; tail -1 gpurun_out/r2_t4.log
grep -E "config [123]" gpurun_out/r2_t4.log | head; grep "case 17\|case 18" gpurun_out/r2_t4.log | head -3
bash scripts/ab_cmp.sh 5 2
bash scripts/ab_cmp.sh 3 1
bash scripts/ab_cmp.sh 2 1
