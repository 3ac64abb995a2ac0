for e in "HPFEM_PERSIST=0" "HPFEM_PERSIST_CTAS=1" "HPFEM_PERSIST_CTAS=2" "HPFEM_PERSIST=1"; do
env $e timeout 300 python bench.py --config 2 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('config 2 $e', round(d['ms_per_step'],3))"; done
