# ncu --set full of one cfg5 point (SIZE, BITS, INST instances) for each build_var variant in VARS
mkdir -p gpurun_out/var_ncu
cp paper_2404_06359_b200/libmc.so /tmp/libmc_orig.so
NCU="ncu --set full --import-source on --clock-control none -k regex:mc_decode_kernel"
for v in $VARS; do
  cp build_var/libmc_$v.so paper_2404_06359_b200/libmc.so
  timeout 900 $NCU -s 4 -c 1 -o gpurun_out/var_ncu/${v}_${SIZE}_b${BITS} -f python scripts/sweep_cfg5.py --out /tmp/x.jsonl --sizes $SIZE --bits $BITS --instances ${INST:-100} --steps 2 > /dev/null 2>&1
done
cp /tmp/libmc_orig.so paper_2404_06359_b200/libmc.so
