timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r2_bench5.json 2> gpurun_out/r2_bench5.err; echo bench rc=$?
tail -1 gpurun_out/r2_bench5.json | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print(d['value'], d['ms_per_step'], d['ms_per_step_median'], d['roofline']['frac'], d['roofline']['per_kind_ms'], d['e2e']['value'], d['clocks'])
print(json.dumps(d['cpu_baseline']))"
