mkdir -p gpurun_out/fin
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/fin/bench.json 2> gpurun_out/fin/bench.err; cut -c1-200 gpurun_out/fin/bench.json
for args in "--codec 2 --index-format u8x4" "--codec 1 --index-format u8x4" "--codec 2 --variable-widths --index-format u8x4"; do
  tag=$(echo $args | tr -d ' -')
  timeout 600 python bench.py $args --steps 30 --no-cpu-baseline --no-e2e > gpurun_out/fin/bench_$tag.json 2> gpurun_out/fin/bench_$tag.err
  python -c "import json; d=json.load(open('gpurun_out/fin/bench_$tag.json')); print('$args', round(d['value'],2), 'Gtri/s', round(d['roofline']['achieved']), 'GB/s frac', round(d['roofline']['frac'],3), 'err', d['checksum']['error_bits'])"
done
