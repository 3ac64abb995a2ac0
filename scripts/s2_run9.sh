timeout 900 python -m pytest tests/test_gpu_varcoef.py -x -q > gpurun_out/s2_t9.log 2>&1; echo tests rc=$?
tail -2 gpurun_out/s2_t9.log
timeout 300 python scripts/bench_pcg.py > gpurun_out/s2_pcg2.jsonl; cut -c1-220 gpurun_out/s2_pcg2.jsonl
timeout 300 python scripts/bench_burgers.py --shapes 9:8,9:16,9:32 | cut -c1-200
