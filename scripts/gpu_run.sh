for v in h34 h42 h32; do
cp scripts/micro/lib_$v.so paper_2402_11299_b200/libhpfem_b200.so
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_hats" -s 40 -c 8 --csv --log-file gpurun_out/l43_$v.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
echo $v; python scripts/launch_summary.py gpurun_out/l43_$v.csv | sed -n 2,3p
done
