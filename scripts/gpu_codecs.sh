# cfg4 bench line per codec / index format / widths / culling, and the cfg1-cfg3 parity
# configs (L2 flushed); every line lands in gpurun_out/codecs_<tag>/.
# usage: bash scripts/gpu_codecs.sh <tag>
TAG=${1:-r2}
OUT=gpurun_out/codecs_$TAG
mkdir -p $OUT
for args in "--codec 2" "--codec 1" "--codec 3" "--codec 2 --index-format u8x4" "--codec 1 --index-format u8x4" \
            "--codec 3 --index-format u8x4" "--codec 2 --variable-widths" "--codec 1 --variable-widths" \
            "--codec 2 --variable-widths --index-format u8x4" "--cull" \
            "--workload cfg1_grid" "--workload cfg2_torus" "--workload cfg3_sphere" "--workload cfg3_sphere_nrm8"; do
  tag=$(echo $args | tr -d ' -')
  timeout 600 python bench.py $args --steps 30 --no-cpu-baseline --no-e2e --sustained-seconds 0 > $OUT/bench_$tag.json 2> $OUT/bench_$tag.err || tail -3 $OUT/bench_$tag.err
  python -c "import json; d=json.load(open('$OUT/bench_$tag.json')); print('$args', round(d['value'],2), 'Gtri/s', round(d['roofline']['achieved']), 'GB/s frac', round(d['roofline']['frac'],3), 'bits/tri', d['config']['compressed_bits_per_tri'], 'err', d['checksum']['error_bits'])"
done
