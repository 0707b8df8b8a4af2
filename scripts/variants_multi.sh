# A/B of build_var/libmc_*.so over several workloads (GPU box scratch only).
# usage: bash scripts/variants_multi.sh   (workload list below or WLS="name:args ..."; REPS=2; NOSWEEP=1
#        skips the cfg5 points)
mkdir -p gpurun_out
cp paper_2404_06359_b200/libmc.so /tmp/libmc_orig.so
B="python bench.py --steps 30 --no-cpu-baseline --no-e2e --sustained-seconds 0"
for rep in $(seq ${REPS:-2}); do
for so in build_var/libmc_*.so; do
  cp $so paper_2404_06359_b200/libmc.so
  name=$(basename $so .so)
  for w in ${WLS:-"cfg4:" "cfg4u8:--index-format u8x4" "shard8:--instances 125" "vw:--variable-widths"}; do
    wn=${w%%:*}; wa=${w#*:}; wa=${wa//,/ }
    timeout 300 $B $wa 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$name', '$wn', round(d['value'],2), round(d['roofline']['frac'],3), d['checksum']['error_bits'], 'step_ms', d.get('step_ms',{}).get('median'), 'mhz', d.get('clocks',{}).get('sm_mhz'), d.get('clocks',{}).get('reasons'))"
  done
  [ -n "$NOSWEEP" ] && continue
  timeout 900 python scripts/sweep_cfg5.py --instances ${SWEEP_INST:-100} --out /tmp/sw_$name.jsonl --sizes 32x32,64x64 --bits 16,10 --label $name > /dev/null 2>&1
  python -c "
import json
for l in open('/tmp/sw_$name.jsonl'):
    d=json.loads(l); print('$name', 'cfg5', d['vmax'], d['tmax'], d['bits'], round(d['gtri_s'],1), round(d['alg_gb_s']), d['error_bits'])"
  rm -f /tmp/sw_$name.jsonl
done
done
cp /tmp/libmc_orig.so paper_2404_06359_b200/libmc.so
