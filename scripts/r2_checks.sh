# debug-checks build (HPFEM_NVCC_EXTRA=-DHPFEM_CHECKS -> ab/checks.so): device traps on the ring / tile bookkeeping
# and a NaN-poisoned TMA ring; the substitute for compute-sanitizer, which is closed on this pool
HPFEM_LIB_PATH=ab/checks.so timeout 600 python scripts/sanitize_cases.py > gpurun_out/r02_checks_cases.log 2>&1; echo cases rc=$?; tail -4 gpurun_out/r02_checks_cases.log
HPFEM_LIB_PATH=ab/checks.so timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "small_cases or (config_full_solve and not 5) or robin_cases or many_hats or stress or solve1d" > gpurun_out/r02_checks.log 2>&1; echo checks rc=$?; tail -1 gpurun_out/r02_checks.log
