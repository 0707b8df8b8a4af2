# GPU parity suite on the product build, the standard A/B of build_var variants, and the
# 100-instance cfg5 points 32/32 and 64/64 at b = 16, 20 for every variant.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/conv_tests.log 2>&1
echo "tests exit $?" >> gpurun_out/conv_tests.log
REPS=${REPS:-2} timeout 3000 bash scripts/variants_multi.sh > gpurun_out/conv_ab.log 2>&1
cp paper_2404_06359_b200/libmc.so /tmp/libmc_orig.so
for rep in 1 2; do
for so in build_var/libmc_*.so; do
  name=$(basename $so .so); cp $so paper_2404_06359_b200/libmc.so
  timeout 900 python scripts/sweep_cfg5.py --instances 100 --out gpurun_out/sw100_${name}_$rep.jsonl --sizes 32x32,64x64 --bits 16,20 --label $name > /dev/null 2>&1
done
done
cp /tmp/libmc_orig.so paper_2404_06359_b200/libmc.so
