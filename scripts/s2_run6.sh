for s in 0 2 4 8; do
  HPFEM_HAT_SMS=$s timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('HAT_SMS=$s', round(d['ms_per_step'],1), d['roofline']['per_kind_ms'], d['clocks']['sm_mhz'])"
done
