timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "small_cases or config_full_solve or robin or mixed or many_hats" --deselect "tests/test_gpu_parity.py::test_config_full_solve[transposed-4]" --deselect "tests/test_gpu_parity.py::test_config_full_solve[small-4]" --deselect "tests/test_gpu_parity.py::test_config_full_solve[tma-4]" > gpurun_out/r2_t14.log 2>&1; echo tests rc=$?; tail -1 gpurun_out/r2_t14.log
export HPFEM_NO_GRAPH=1
python scripts/prof_solve.py 5 3 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_l5b.csv python scripts/prof_solve.py 5 3 > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/r2_l5b.csv | grep -E "hat"
unset HPFEM_NO_GRAPH
bash scripts/ab_env.sh 5 "HPFEM_HAT_SMS=4" "HPFEM_HAT_SMS=0" "HPFEM_HAT_SMS=2"
bash scripts/ab_env.sh 4 "HPFEM_HAT_SMS=4" "HPFEM_HAT_SMS=0"
bash scripts/ab_env.sh 3 "HPFEM_HAT_SMS=4" "HPFEM_HAT_SMS=0"
