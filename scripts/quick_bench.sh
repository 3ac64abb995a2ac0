timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['ms_per_step'],1), {k: round(v,1) for k,v in d['roofline']['per_kind_ms'].items()}, d['clocks']['sm_mhz'])"
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "small_cases or config_full" 2>&1 | tail -1
