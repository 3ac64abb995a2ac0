# A/B of environment knobs on one config: bash scripts/ab_env.sh CONFIG "ENV=V ..." "ENV=V ..." ...
c=$1; shift
for e in "$@"; do
  env $e timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());r=d['roofline'];print('config $c [$e]', round(d['ms_per_step'],2), {k: round(v,2) for k,v in r['per_kind_ms'].items()}, {k: round(v['avg_launch_ms']*1e3,1) for k,v in r['per_direction'].items()}, d['clocks']['sm_mhz'])"
done
