set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/tests_r2d.log 2>&1; tail -5 gpurun_out/tests_r2d.log
cp paper_2404_06359_b200/libmc.so /tmp/libmc_orig.so; cp build_var/libmc_gcopy.so paper_2404_06359_b200/libmc.so
compute-sanitizer --tool racecheck --print-limit 100 python tests/sanitize_decode.py > gpurun_out/racecheck_gcopy.log 2>&1; tail -3 gpurun_out/racecheck_gcopy.log
cp /tmp/libmc_orig.so paper_2404_06359_b200/libmc.so
timeout 900 python bench.py --no-e2e > gpurun_out/bench_r2d.json 2> gpurun_out/bench_r2d.err; cat gpurun_out/bench_r2d.json
timeout 600 python bench.py --instances 125 --no-cpu-baseline --no-e2e > gpurun_out/bench_shard8_r2d.json 2>/dev/null; cat gpurun_out/bench_shard8_r2d.json
