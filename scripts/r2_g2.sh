timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "small_cases or config_full_solve or robin_cases" > gpurun_out/r2_t2.log 2>&1; echo tests rc=$?; tail -1 gpurun_out/r2_t2.log
bash scripts/ab_cmp.sh 5 2
bash scripts/ab_cmp.sh 3 1
