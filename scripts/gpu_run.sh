timeout 600 python -m pytest tests -m gpu -x -q -k "not config5" > gpurun_out/t44.log 2>&1; echo tests rc=$?
tail -2 gpurun_out/t44.log
timeout 200 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['ms_per_step'],1), d['roofline']['per_kind_ms'], d['clocks'])"
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"step_tma" -s 6 -c 6 --csv --log-file gpurun_out/l44.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1; python scripts/launch_summary.py gpurun_out/l44.csv | sed -n 2,3p
