timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -s -k "robin" > gpurun_out/s2_t10.log 2>&1; echo tests rc=$?
grep -E "robin|passed|failed|Error|assert" gpurun_out/s2_t10.log | tail -25
