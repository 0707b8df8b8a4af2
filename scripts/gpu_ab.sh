# Parity tests on one variant (build_var/libmc_$1.so), then the A/B bench of every variant.
# usage: bash scripts/gpu_ab.sh <variant-to-test> [REPS]
set -x
cp paper_2404_06359_b200/libmc.so /tmp/libmc_orig.so
cp build_var/libmc_$1.so paper_2404_06359_b200/libmc.so
timeout 900 python -m pytest tests/test_gpu_dispatch.py tests/test_gpu_parity.py tests/test_gpu_cull.py -q -x 2>&1 | tail -2
cp /tmp/libmc_orig.so paper_2404_06359_b200/libmc.so
REPS=${2:-2} bash scripts/variants_multi.sh
