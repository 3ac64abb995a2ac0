timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "not config5" > gpurun_out/s2_t13.log 2>&1; echo tests rc=$?
tail -2 gpurun_out/s2_t13.log
for sp in 1 0 1; do
  HPFEM_Y_SPLIT=$sp timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('Y_SPLIT=$sp', round(d['ms_per_step'],1), d['roofline']['per_kind_ms'], d['clocks']['sm_mhz'])"
done
