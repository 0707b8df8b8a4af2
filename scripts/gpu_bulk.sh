set -x
cp paper_2404_06359_b200/libmc.so /tmp/libmc_orig.so
cp build_var/libmc_bulk.so paper_2404_06359_b200/libmc.so
timeout 1500 python -m pytest tests/test_gpu_dispatch.py tests/test_gpu_parity.py tests/test_gpu_cull.py tests/test_gpu_basic_u8x4.py -q -x 2>&1 | tail -3
timeout 600 compute-sanitizer --tool memcheck --leak-check no python tests/sanitize_decode.py --big 2>&1 | tail -2
cp /tmp/libmc_orig.so paper_2404_06359_b200/libmc.so
REPS=2 bash scripts/variants_multi.sh
