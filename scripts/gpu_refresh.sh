# Refresh every measured line with the product build: codecs / index formats / VW / cull on
# cfg4, cfg1-3 lines, the full cfg5 sweep, and a torchrun (NCCL) single-rank bench.
# usage: bash scripts/gpu_refresh.sh <tag>
TAG=${1:-r}
mkdir -p gpurun_out/refresh
for args in "--codec 2" "--codec 1" "--codec 3" "--codec 2 --index-format u8x4" "--codec 1 --index-format u8x4" "--codec 3 --index-format u8x4" "--codec 2 --variable-widths" "--codec 1 --variable-widths" "--codec 2 --variable-widths --index-format u8x4" "--cull"; do
  tag=$(echo $args | tr -d ' -')
  timeout 600 python bench.py $args --steps 30 --no-cpu-baseline --no-e2e > gpurun_out/refresh/bench_$tag.json 2> gpurun_out/refresh/bench_$tag.err || tail -3 gpurun_out/refresh/bench_$tag.err
  python -c "import json; d=json.load(open('gpurun_out/refresh/bench_$tag.json')); print('$args', round(d['value'],2), 'Gtri/s', round(d['roofline']['achieved']), 'GB/s frac', round(d['roofline']['frac'],3), 'err', d['checksum']['error_bits'])"
done
for w in cfg1_grid cfg2_torus cfg3_sphere cfg3_sphere_nrm8; do
  timeout 600 python bench.py --workload $w --steps 30 > gpurun_out/refresh/bench_$w.json 2> gpurun_out/refresh/bench_$w.err || tail -5 gpurun_out/refresh/bench_$w.err
  python -c "import json; d=json.load(open('gpurun_out/refresh/bench_$w.json')); print('$w', round(d['value'],2), 'Gtri/s frac', round(d['roofline']['frac'],3), 'e2e', d['e2e']['value'] if d['e2e'] else None)"
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 10 --no-cpu-baseline > gpurun_out/refresh/bench_torchrun1.json 2> gpurun_out/refresh/bench_torchrun1.err || tail -5 gpurun_out/refresh/bench_torchrun1.err
cat gpurun_out/refresh/bench_torchrun1.json | cut -c1-300
rm -f gpurun_out/refresh/sweep_cfg5.jsonl
timeout 1500 python scripts/sweep_cfg5.py --label $TAG --out gpurun_out/refresh/sweep_cfg5.jsonl > /dev/null 2> gpurun_out/refresh/sweep.err || tail -5 gpurun_out/refresh/sweep.err
wc -l gpurun_out/refresh/sweep_cfg5.jsonl
