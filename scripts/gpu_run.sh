timeout 400 python -m pytest tests -m gpu -x -q -k "not config5" > gpurun_out/t17.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/t17.log
for nx in 2 3 4 6; do
  HPFEM_NST_X=$nx HPFEM_NST_Y=$nx timeout 120 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b17_$nx.json 2>gpurun_out/b17_$nx.err
  python -c "import json;d=json.loads(open('gpurun_out/b17_$nx.json').read().strip().splitlines()[-1]);print('nst',$nx,round(d['ms_per_step'],1),d['roofline']['per_kind_ms'])"
done
