timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "batched or reuse or two_host or iters_zero or stress" 2>&1 | tail -2
for c in 1 2; do timeout 600 python bench.py --config $c --batch 256 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1; done > gpurun_out/r02_batched.jsonl
timeout 600 python bench.py --config 3 --batch 32 --steps 5 --warmup 2 --no-cpu-baseline 2>/dev/null | tail -1 >> gpurun_out/r02_batched.jsonl
python -c "
import json
for l in open('gpurun_out/r02_batched.jsonl'):
    d=json.loads(l); print(d['config']['workload'][:8], round(d['ms_per_step'],3), round(d['value'],1), round(d['e2e']['value'],1))"
