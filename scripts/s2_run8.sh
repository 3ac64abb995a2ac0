timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "not config5" > gpurun_out/s2_t8.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/s2_t8.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -s -k "small_cases and small" 2>&1 | grep "case" | head -20
for b in 1 32 1024; do
  timeout 300 python bench.py --config 1 --batch $b --steps 20 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('config 1 batch $b', round(d['ms_per_step'],3), 'ms', round(d['value'],1), d['unit'])"
done
timeout 300 python scripts/bench_pcg.py --shapes 1:8,1:16 | cut -c1-200
