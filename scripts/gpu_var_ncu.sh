# ncu --set full of the timed decode kernel for each build_var variant (VARS) on one workload (ARGS)
mkdir -p gpurun_out/var_ncu
cp paper_2404_06359_b200/libmc.so /tmp/libmc_orig.so
NCU="ncu --set full --import-source on --clock-control none -k regex:mc_decode_kernel"
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --sustained-seconds 0"
for v in $VARS; do
  cp build_var/libmc_$v.so paper_2404_06359_b200/libmc.so
  timeout 600 $NCU -s 3 -c 1 -o gpurun_out/var_ncu/$v -f $B $ARGS > /dev/null 2>&1
done
cp /tmp/libmc_orig.so paper_2404_06359_b200/libmc.so
