mkdir -p gpurun_out
for w in cfg3_sphere cfg3_sphere_nrm8; do
  timeout 300 python bench.py --workload $w --steps 30 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', round(d['value'],2), round(d['roofline']['achieved']), d['ms_per_step'])"
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:mc_decode_kernel -s 3 -c 1 -o gpurun_out/prof_$w -f python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
done
