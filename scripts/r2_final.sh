# round-2 final evidence run (one B200): gpu tests with their printed parity numbers, bench lines, ncu launch lists / full captures
set -o pipefail
timeout 2400 python -m pytest tests -m gpu -q -s > gpurun_out/r02_gpu_tests_full.log 2>&1; echo tests rc=$?; tail -1 gpurun_out/r02_gpu_tests_full.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/r02_smoke.log
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench_config5.json 2> gpurun_out/r02_bench_config5.err; echo bench5 rc=$?
for c in 1 2 3 4; do timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1; done > gpurun_out/r02_configs1-4.jsonl; echo cfgs rc=$?
for c in 1 2; do timeout 600 python bench.py --config $c --batch 256 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1; done > gpurun_out/r02_batched.jsonl
timeout 600 python bench.py --config 3 --batch 32 --steps 5 --warmup 2 --no-cpu-baseline 2>/dev/null | tail -1 >> gpurun_out/r02_batched.jsonl
python scripts/bench_apply.py 2 3 4 5 > gpurun_out/r02_apply.jsonl 2>/dev/null
python scripts/bench_1d.py > gpurun_out/r02_fig1_1d.jsonl 2>/dev/null
python scripts/bench_pcg.py > gpurun_out/r02_pcg_table1.jsonl 2>/dev/null
python scripts/bench_burgers.py > gpurun_out/r02_burgers_imex.jsonl 2>/dev/null
export HPFEM_NO_GRAPH=1
python scripts/prof_solve.py 5 3 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02_config5_launches.csv python scripts/prof_solve.py 5 3 > /dev/null 2>&1; echo l5 rc=$?
python scripts/prof_solve.py 4 3 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02_config4_launches.csv python scripts/prof_solve.py 4 3 > /dev/null 2>&1; echo l4 rc=$?
python scripts/prof_solve.py 5 2 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_[xy]step_tma|k_hats_rows|k_hats_cols|k_hatrows_y|k_hatcols_x" -s 8 -c 8 -o gpurun_out/r02_config5_full python scripts/prof_solve.py 5 2 > gpurun_out/r02_ncu_full5.log 2>&1; echo full5 rc=$?
python scripts/prof_solve.py 4 2 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_[xy]step_tma|k_hats_rows|k_hats_cols" -s 6 -c 8 -o gpurun_out/r02_config4_full python scripts/prof_solve.py 4 2 > gpurun_out/r02_ncu_full4.log 2>&1; echo full4 rc=$?
python scripts/ncu_summary.py gpurun_out/r02_config5_full.ncu-rep > gpurun_out/r02_config5_ncu.txt
python scripts/ncu_summary.py gpurun_out/r02_config4_full.ncu-rep > gpurun_out/r02_config4_ncu.txt
for k in k_ystep_tma k_xstep_tma k_hats_rows k_hats_cols; do echo "== $k"; python scripts/ncu_lines.py gpurun_out/r02_config5_full.ncu-rep $k 12; done > gpurun_out/r02_config5_ncu_lines.txt 2>&1
rm -f gpurun_out/r02_config5_full.ncu-rep gpurun_out/r02_config4_full.ncu-rep  # (gpurun brings back at most 64 MiB)
python scripts/launch_summary.py gpurun_out/r02_config5_launches.csv > gpurun_out/r02_config5_launches.txt
python scripts/launch_summary.py gpurun_out/r02_config4_launches.csv > gpurun_out/r02_config4_launches.txt
