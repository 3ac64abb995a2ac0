for k in 1 2; do
for lib in paper_2402_11299_b200/libhpfem_b200.so ab/SPB=1.so ab/NOBUF=1.so; do
  HPFEM_LIB_PATH=$lib timeout 300 python bench.py --config 5 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('config 5 $lib', round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['roofline']['per_kind_ms'].items()}, d['clocks']['sm_mhz'])"
done; done
