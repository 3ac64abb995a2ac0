# quick A/B: parity subset, then config 5 and 3 timings with and without the knob in $1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "small_cases or config_full or batched or robin" 2>&1 | tail -1
for c in 5 3; do for v in 0 1; do
  env $1=$v timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('config $c $1=$v', round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['roofline']['per_kind_ms'].items()}, d['clocks']['sm_mhz'])"
done; done
