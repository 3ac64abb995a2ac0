export HPFEM_NO_GRAPH=1
python scripts/prof_solve.py 4 3 > gpurun_out/ps4.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2_l4.csv python scripts/prof_solve.py 4 3 > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/r2_l4.csv > gpurun_out/r2_l4.txt; head -20 gpurun_out/r2_l4.txt
timeout 300 python bench.py --config 4 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('config 4', round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['roofline']['per_kind_ms'].items()}, d['clocks']['sm_mhz'])"
