# like variants.sh but over several workloads: WORKLOADS="cfg4_city cfg3_sphere_nrm8" bash scripts/variants_wl.sh
mkdir -p gpurun_out
cp paper_2404_06359_b200/libmc.so /tmp/libmc_orig.so
for so in build_var/libmc_*.so; do
  cp $so paper_2404_06359_b200/libmc.so
  for w in ${WORKLOADS:-cfg4_city}; do
    timeout 300 python bench.py --workload $w --steps 30 --no-cpu-baseline --no-e2e ${BENCH_ARGS} 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$so', '$w', round(d['value'],2), round(d['roofline']['frac'],3), d['checksum']['error_bits'])"
  done
done
cp /tmp/libmc_orig.so paper_2404_06359_b200/libmc.so
