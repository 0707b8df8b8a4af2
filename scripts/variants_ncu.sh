# ncu --set full capture of the timed decode kernel for each build_var/libmc_*.so (GPU box scratch copy)
mkdir -p gpurun_out
cp paper_2404_06359_b200/libmc.so /tmp/libmc_orig.so
for so in build_var/libmc_*.so; do
  name=$(basename $so .so); name=${name#libmc_}
  cp $so paper_2404_06359_b200/libmc.so
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:mc_decode_kernel -s 3 -c 1 \
     -o gpurun_out/prof_var_$name -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e ${BENCH_ARGS} > gpurun_out/ncu_var_$name.log 2>&1
  tail -1 gpurun_out/ncu_var_$name.log
done
cp /tmp/libmc_orig.so paper_2404_06359_b200/libmc.so
