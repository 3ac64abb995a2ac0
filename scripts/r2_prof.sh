# round-2 evidence run: debug-checks build, bench lines, ncu launch lists / full captures
set -o pipefail
HPFEM_LIB_PATH=ab/checks.so timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "small_cases or (config_full_solve and not 4) or robin_cases or many_hats or stress" > gpurun_out/r02_checks.log 2>&1; echo checks rc=$?; tail -1 gpurun_out/r02_checks.log
for c in 1 2 3 4; do timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1; done > gpurun_out/r02_configs1-4.jsonl; echo cfgs rc=$?
for c in 1 2; do timeout 600 python bench.py --config $c --batch 256 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1; done > gpurun_out/r02_batched.jsonl
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench_config5.json 2> gpurun_out/r02_bench_config5.err; echo bench5 rc=$?
export HPFEM_NO_GRAPH=1
python scripts/prof_solve.py 5 3 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02_config5_launches.csv python scripts/prof_solve.py 5 3 > /dev/null 2>&1; echo l5 rc=$?
python scripts/prof_solve.py 4 3 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02_config4_launches.csv python scripts/prof_solve.py 4 3 > /dev/null 2>&1; echo l4 rc=$?
python scripts/prof_solve.py 5 2 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_[xy]step_tma|k_hats_rows|k_hats_cols" -s 4 -c 4 -o gpurun_out/r02_config5_full python scripts/prof_solve.py 5 2 > gpurun_out/r02_ncu_full.log 2>&1; echo full rc=$?
