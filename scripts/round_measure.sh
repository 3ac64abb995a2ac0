# Round measurement (one B200): GPU tests, the default bench line, the ncu
# launch list of one step and one `ncu --set full` launch of each hot kernel.
# Usage: gpurun -- 'bash scripts/round_measure.sh TAG'
TAG=${1:-r01}
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_tests.log 2>&1; echo "tests rc=$?"
tail -2 gpurun_out/${TAG}_tests.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
tail -1 gpurun_out/${TAG}_bench.json | cut -c1-300
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo "ncu list rc=$?"
python scripts/launch_summary.py gpurun_out/${TAG}_launches.csv > gpurun_out/${TAG}_launches.txt 2>&1; head -14 gpurun_out/${TAG}_launches.txt
HPFEM_NO_GRAPH=1 timeout 1200 ncu --set full --import-source on --clock-control none \
  -k regex:"k_xstep_tma|k_ystep_tma|k_hats" -s 6 -c 4 -o gpurun_out/${TAG}_full python scripts/yprof_run.py > gpurun_out/${TAG}_ncu_full.log 2>&1; echo "ncu full rc=$?"
python scripts/ncu_summary.py gpurun_out/${TAG}_full.ncu-rep > gpurun_out/${TAG}_ncu.txt 2>&1; head -60 gpurun_out/${TAG}_ncu.txt
