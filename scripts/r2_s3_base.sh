# session-3 baseline: gpu tests, then short bench lines for configs 2-5
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/s3_gpu_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/s3_gpu_tests.log
for c in 2 3 4 5; do bash scripts/ab_env.sh $c "HPFEM_X=0"; done
python scripts/bench_1d.py > gpurun_out/s3_1d.jsonl 2>&1; tail -12 gpurun_out/s3_1d.jsonl
