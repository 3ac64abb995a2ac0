timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "solve1d" > gpurun_out/r2_t8.log 2>&1; echo tests rc=$?; tail -1 gpurun_out/r2_t8.log
timeout 300 python scripts/bench_1d.py > gpurun_out/r2_fig1.jsonl 2>&1; echo bench rc=$?
cat gpurun_out/r2_fig1.jsonl | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l)
    if 'summary' in d: print(d); continue
    print(d['n'], d['p'], d['N'], round(d['solve_ms_nrhs1'],3), round(d['solve_ms_nrhs1024'],3), round(d['roofline']['frac'],3))
"
