timeout 600 python scripts/bench_burgers.py > gpurun_out/s2_burgers.jsonl 2> gpurun_out/s2_burgers.err; echo rc=$?
cat gpurun_out/s2_burgers.jsonl; tail -3 gpurun_out/s2_burgers.err
