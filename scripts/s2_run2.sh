timeout 900 python -m pytest tests -m gpu -x -q -k "small_cases or mixed or lemma51 or solve1d or unload_small or errors" > gpurun_out/s2_t2.log 2>&1; echo tests rc=$?
tail -30 gpurun_out/s2_t2.log
