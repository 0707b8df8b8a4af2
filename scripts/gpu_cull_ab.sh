# Culled decode: parity on the in-tree build and on build_var/libmc_fused.so, sanitizer, then
# A/B of build_var variants on --cull (GPU box scratch only).
set -x
timeout 900 python -m pytest tests/test_gpu_cull.py -q -x 2>&1 | tail -2
cp paper_2404_06359_b200/libmc.so /tmp/libmc_orig.so
cp build_var/libmc_fused.so paper_2404_06359_b200/libmc.so
timeout 900 python -m pytest tests/test_gpu_cull.py -q -x 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_sanitizer.py -q 2>&1 | tail -2
cp /tmp/libmc_orig.so paper_2404_06359_b200/libmc.so
timeout 900 python -m pytest tests/test_gpu_sanitizer.py -q 2>&1 | tail -2
for rep in 1 2; do for so in build_var/libmc_*.so; do
  cp $so paper_2404_06359_b200/libmc.so
  for w in "cull:--cull" "cullu8:--cull --index-format u8x4" "cull125:--cull --instances 125"; do
    wn=${w%%:*}; wa=${w#*:}
    timeout 300 python bench.py --steps 30 --no-cpu-baseline --no-e2e --sustained-seconds 0 $wa 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$so', '$wn', round(d['value'],2), round(d['ms_per_step']*1e3,1), 'us', d['cull']['visible_records'], d['checksum']['error_bits'])"
  done
done; done
cp /tmp/libmc_orig.so paper_2404_06359_b200/libmc.so
