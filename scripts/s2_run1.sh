nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q -k "not config5" > gpurun_out/s2_tests.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/s2_tests.log
timeout 400 python bench.py --steps 5 --warmup 3 > gpurun_out/s2_bench.json 2> gpurun_out/s2_bench.err; echo bench rc=$?
tail -1 gpurun_out/s2_bench.json | cut -c1-600
