set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/tests_r2e.log 2>&1; tail -5 gpurun_out/tests_r2e.log
timeout 900 python bench.py > gpurun_out/bench_r2e.json 2> gpurun_out/bench_r2e.err; tail -2 gpurun_out/bench_r2e.err; cat gpurun_out/bench_r2e.json
timeout 600 python bench.py --instances 125 --no-cpu-baseline --no-e2e > gpurun_out/bench_shard8_r2e.json 2>/dev/null; cat gpurun_out/bench_shard8_r2e.json
timeout 1200 python scripts/sweep_cfg5.py --out gpurun_out/sweep_cfg5_r2e.jsonl --label r2e > /dev/null 2>&1; wc -l gpurun_out/sweep_cfg5_r2e.jsonl
bash scripts/prof_r2.sh r2e launches cfg4 shard8 > gpurun_out/prof_r2e.log 2>&1; tail -3 gpurun_out/prof_r2e.log
