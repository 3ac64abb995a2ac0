timeout 600 python -m pytest tests -m gpu -x -q -k "not config5" > gpurun_out/t32.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/t32.log
for c in 1 2 3; do
timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('cfg $c single', round(d['value'],1), 'solves/s', round(d['ms_per_step'],3),'ms', d['e2e']['value'])"
for b in 8 32; do
timeout 300 python bench.py --config $c --batch $b --steps 5 --warmup 2 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('cfg $c batch $b', round(d['value'],1), 'solves/s', round(d['ms_per_step'],3),'ms/step e2e', d['e2e']['value'])"
done; done
