# Converged-control-flow A/B: GPU parity suite on the product build, then the variants
# bench (build_var/libmc_*.so) over the standard workloads.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/conv_tests.log 2>&1
echo "tests exit $?" >> gpurun_out/conv_tests.log
REPS=${REPS:-2} timeout 3000 bash scripts/variants_multi.sh > gpurun_out/conv_ab.log 2>&1
