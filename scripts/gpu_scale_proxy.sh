# Strong-scaling proxy on one GPU: the per-rank workload of N = 1, 2, 4, 8 (1000 / N city
# instances, the same kernel and CUDA graph as bench.py) timed back to back, twice.
mkdir -p gpurun_out/scale_proxy
for rep in 1 2; do
for inst in 1000 500 250 125; do
  timeout 600 python bench.py --instances $inst --no-cpu-baseline --no-e2e > gpurun_out/scale_proxy/bench_i${inst}_r$rep.json 2>/dev/null
done
done
