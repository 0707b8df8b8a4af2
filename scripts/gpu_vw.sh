mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
for args in "--codec 2" "--codec 2 --variable-widths" "--codec 1 --variable-widths" "--codec 2 --variable-widths --index-format u8x4"; do
  tag=$(echo $args | tr -d ' -')
  timeout 600 python bench.py $args --steps 30 --no-cpu-baseline --no-e2e > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err || tail -3 gpurun_out/bench_$tag.err
  python -c "import json; d=json.load(open('gpurun_out/bench_$tag.json')); print('$args', round(d['value'],2), 'Gtri/s', round(d['roofline']['achieved']), 'GB/s frac', round(d['roofline']['frac'],3), 'bpt', d['config']['compressed_bits_per_tri'], 'err', d['checksum']['error_bits'])"
done
