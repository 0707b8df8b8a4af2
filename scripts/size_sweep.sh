# Kernel time vs launch size on the cfg4 city (strong-scaling shards): fixed cost per launch.
# usage: bash scripts/size_sweep.sh [extra bench args]
for n in 16 32 63 125 250 500 1000; do
  timeout 600 python bench.py --instances $n --steps 30 --no-cpu-baseline --no-e2e "$@" 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print($n, d['config']['meshlets_this_rank'], round(d['value'],2), round(d['ms_per_step']*1e3,2), round(d['step_ms']['median']*1e3,2), round(d['roofline']['frac'],3))"
done
