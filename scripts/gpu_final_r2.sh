# Round-2 final evidence pass (one GPU box): tests, smoke, bench lines, reference arm, the
# strong-scaling shard proxy, ncu captures, codec/config lines, cfg5 sweeps, power probe.
# usage: bash scripts/gpu_final_r2.sh <tag>
set -x
TAG=${1:-final}
OUT=gpurun_out/final_$TAG
mkdir -p $OUT
timeout 2400 python -m pytest tests -m gpu -q > $OUT/tests.log 2>&1; tail -3 $OUT/tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; cat $OUT/bench.json
timeout 900 python bench.py --steps 20 --warmup 5 > $OUT/bench_s20.json 2> $OUT/bench_s20.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_reference.json 2> $OUT/bench_reference.err; cat $OUT/bench_reference.json
timeout 600 python bench.py --instances 125 --no-cpu-baseline --no-e2e > $OUT/bench_shard8.json 2>/dev/null; cat $OUT/bench_shard8.json
python scripts/power_probe.py > $OUT/power_probe.json 2>/dev/null
bash scripts/gpu_codecs.sh $TAG > $OUT/codecs.log 2>&1; cp -r gpurun_out/codecs_$TAG $OUT/codecs; cat $OUT/codecs.log
timeout 1800 python scripts/sweep_cfg5.py --out $OUT/sweep_cfg5_10.jsonl --label $TAG > /dev/null 2>&1
timeout 2400 python scripts/sweep_cfg5.py --instances 100 --out $OUT/sweep_cfg5_100.jsonl --label ${TAG}100 > /dev/null 2>&1
bash scripts/prof_r2.sh $TAG launches cfg4 shard8 cfg4u8 cfg4vw cfg2 cfg5_32x32_b16 cfg5_64x64_b16 cfg5_64x126_b8 cfg5_64x126_b16 > $OUT/prof.log 2>&1
mv gpurun_out/profiles_$TAG $OUT/profiles; rm -f gpurun_out/*.ncu-rep
nproc; lscpu | grep "Model name"; nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv
