timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r02_gpu_tests_last.log 2>&1; echo tests rc=$?; tail -1 gpurun_out/r02_gpu_tests_last.log
