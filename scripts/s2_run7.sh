timeout 900 python -m pytest tests -m gpu -x -q -k "not config5" > gpurun_out/s2_t7.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/s2_t7.log
for c in 1 2 3; do
 for g in 0 1; do
  HPFEM_NO_GRAPH=$g timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('config $c NO_GRAPH=$g', round(d['ms_per_step'],3), 'ms', round(d['value'],1), d['unit'], 'launches', d['gpu_launches'])"
 done
done
timeout 300 python scripts/bench_pcg.py --shapes 1:8,3:128 | cut -c1-300
