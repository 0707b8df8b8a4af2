# quick GPU iteration: parity tests, a short bench, optionally one ncu --set full capture
# usage: bash scripts/gpu_quick.sh <tag> [ncu]
set -x
TAG=${1:-q}
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
timeout 600 python bench.py --steps 30 --no-cpu-baseline --no-e2e > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -2 gpurun_out/bench_$TAG.err; cat gpurun_out/bench_$TAG.json
if [ "$2" = "ncu" ]; then
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:mc_decode_kernel -s 3 -c 1 \
     -o gpurun_out/prof_$TAG -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_$TAG.log 2>&1
  tail -3 gpurun_out/ncu_$TAG.log
fi
