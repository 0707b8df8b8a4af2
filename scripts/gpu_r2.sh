# Round-2 GPU pass: all GPU tests (incl. sanitizer / dispatch / multiproc), smoke, bench
# (default + weak), one strong-scaling shard proxy (1/8 of the city on one GPU).
# usage: bash scripts/gpu_r2.sh <tag>
set -x
TAG=${1:-r2}
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/tests_$TAG.log 2>&1; tail -30 gpurun_out/tests_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -3 gpurun_out/bench_$TAG.err; cat gpurun_out/bench_$TAG.json
timeout 600 python bench.py --no-graph --no-cpu-baseline --no-e2e > gpurun_out/bench_nograph_$TAG.json 2>/dev/null; cat gpurun_out/bench_nograph_$TAG.json
timeout 600 python bench.py --instances 125 --no-cpu-baseline --no-e2e > gpurun_out/bench_shard8_$TAG.json 2>/dev/null; cat gpurun_out/bench_shard8_$TAG.json
nproc; lscpu | grep "Model name"
