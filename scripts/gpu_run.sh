for n in 3 4; do
HPFEM_NST_Y=$n timeout 120 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b30_$n.json 2>gpurun_out/b30_$n.err
python -c "import json;d=json.loads(open('gpurun_out/b30_$n.json').read().strip().splitlines()[-1]);print('nobuf1 nst $n', round(d['ms_per_step'],1),d['roofline']['per_kind_ms'])"
done
