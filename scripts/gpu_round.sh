# Full GPU evidence pass: parity tests, smoke, default bench (with cpu_baseline + e2e),
# reference arm, ncu launch list of the bench command, one ncu --set full capture of the
# timed kernel.  usage: bash scripts/gpu_round.sh <tag>
set -x
TAG=${1:-r}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -2 gpurun_out/bench_$TAG.err; cat gpurun_out/bench_$TAG.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ref_$TAG.json 2> gpurun_out/ref_$TAG.err; cat gpurun_out/ref_$TAG.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:mc_decode_kernel -s 3 -c 1 \
   -o gpurun_out/prof_$TAG -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_$TAG.log 2>&1
nproc; lscpu | grep "Model name"
