timeout 400 python -m pytest tests -m gpu -x -q -k "not config5" > gpurun_out/t27.log 2>&1; echo tests rc=$?
tail -5 gpurun_out/t27.log
timeout 120 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b27.json 2>gpurun_out/b27.err
python -c "import json;d=json.loads(open('gpurun_out/b27.json').read().strip().splitlines()[-1]);print(round(d['ms_per_step'],1),d['roofline']['per_kind_ms'])"
ncu --metrics gpu__time_duration.sum --clock-control none -s 1500 -c 200 --csv --log-file gpurun_out/launches27.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu27.log 2>&1; echo ncu rc=$?
