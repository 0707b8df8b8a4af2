set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_cull.py tests/test_gpu_sanitizer.py -q -x > gpurun_out/tests_r2f.log 2>&1; tail -5 gpurun_out/tests_r2f.log
timeout 600 python bench.py --cull --no-cpu-baseline --no-e2e --sustained-seconds 0 > gpurun_out/bench_cull_r2f.json 2>/dev/null; cat gpurun_out/bench_cull_r2f.json
timeout 600 python bench.py --no-cpu-baseline --no-e2e --sustained-seconds 0 > gpurun_out/bench_r2f.json 2>/dev/null; cat gpurun_out/bench_r2f.json
