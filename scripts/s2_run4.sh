nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/dfma_peak scripts/micro/dfma_peak.cu && /tmp/dfma_peak | tee gpurun_out/s2_dfma.json
PK=$(python -c "import json;print(json.load(open('gpurun_out/s2_dfma.json'))['fp64_fma_tflops'])")
timeout 600 python scripts/bench_pcg.py --fp64-peak $PK > gpurun_out/s2_pcg.jsonl 2> gpurun_out/s2_pcg.err; echo pcg rc=$?
cat gpurun_out/s2_pcg.jsonl; tail -3 gpurun_out/s2_pcg.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s2_pcg_launches.csv python scripts/bench_pcg.py --reps 1 --shapes 3:128 > /dev/null 2>&1; echo ncu rc=$?
python scripts/launch_summary.py gpurun_out/s2_pcg_launches.csv | head -20
