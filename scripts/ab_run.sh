timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for c in 5 3; do
  timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('config $c', round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['roofline']['per_kind_ms'].items()}, d['clocks']['sm_mhz'])"
done
