# A/B experiment: bench each build_var/libmc_*.so in place of libmc.so (GPU box scratch copy only)
mkdir -p gpurun_out
cp paper_2404_06359_b200/libmc.so /tmp/libmc_orig.so
for so in build_var/libmc_*.so; do
  cp $so paper_2404_06359_b200/libmc.so
  if [ -n "$RUN_TESTS" ]; then echo "$so tests: $(timeout 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -1)"; fi
  for rep in 1 2; do
    timeout 300 python bench.py --steps 30 --no-cpu-baseline --no-e2e ${BENCH_ARGS} 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$so', round(d['value'],2), round(d['roofline']['frac'],3), d['checksum']['error_bits'], d['checksum']['indices'])"
  done
done
cp /tmp/libmc_orig.so paper_2404_06359_b200/libmc.so
