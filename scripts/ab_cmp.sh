# On the box: alternate base / new library runs of bench.py on config $1 (K reps each)
c=${1:-5}; k=${2:-2}; extra=${3:-}
for i in $(seq $k); do
  for lib in ab/base.so paper_2402_11299_b200/libhpfem_b200.so; do
    HPFEM_LIB_PATH=$lib timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline $extra 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('config $c $lib', round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['roofline']['per_kind_ms'].items()}, d['clocks']['sm_mhz'])"
  done
done
