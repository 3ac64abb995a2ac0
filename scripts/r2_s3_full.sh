timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/s3_gpu_tests2.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/s3_gpu_tests2.log
