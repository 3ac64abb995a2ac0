timeout 600 python -m pytest tests -m gpu -x -q -k "not config5" > gpurun_out/t33.log 2>&1; echo tests rc=$?
tail -2 gpurun_out/t33.log
for h in 0 2 4 8; do
HPFEM_HAT_SMS=$h timeout 200 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('hat_sms $h', round(d['ms_per_step'],1), d['roofline']['per_kind_ms'])"
done
