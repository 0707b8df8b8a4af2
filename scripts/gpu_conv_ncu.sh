# ncu --set full of the timed decode kernel per build_var variant: cfg4 u8x4, cfg5 64/64
mkdir -p gpurun_out
cp paper_2404_06359_b200/libmc.so /tmp/libmc_orig.so
NCU="ncu --set full --import-source on --clock-control none -k regex:mc_decode_kernel"
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --sustained-seconds 0"
for v in ${VARS:-base cld}; do
  cp build_var/libmc_$v.so paper_2404_06359_b200/libmc.so
  timeout 600 $NCU -s 3 -c 1 -o gpurun_out/pv_u8_$v -f $B --index-format u8x4 > /dev/null 2>&1
  timeout 600 $NCU -s 4 -c 1 -o gpurun_out/pv_g64_$v -f python scripts/sweep_cfg5.py --out /tmp/x.jsonl --sizes 64x64 --bits 16 --steps 2 > /dev/null 2>&1
done
cp /tmp/libmc_orig.so paper_2404_06359_b200/libmc.so
