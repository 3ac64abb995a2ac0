timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -s -k "solve1d" 2>&1 | tail -32
for cl in 0 1; do echo "== CLUSTER=$cl"; HPFEM_1D_CLUSTER=$cl python scripts/bench_1d.py 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.strip()[:200]); continue
    if 'summary' in d: print(d)
    else: print(d['n'], d['p'], d['N'], 'nrhs1 %.3f ms' % d['solve_ms_nrhs1'], 'nrhs1024 %.3f ms' % d['solve_ms_nrhs1024'], 'frac %.3f' % d['roofline']['frac'])
"; done
