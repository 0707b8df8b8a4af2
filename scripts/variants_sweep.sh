# A/B of build_var/libmc_*.so on cfg5 points (scripts/sweep_cfg5.py); GPU box scratch only.
# usage: SIZES=32x32,64x64 BITS=16 bash scripts/variants_sweep.sh
mkdir -p gpurun_out
cp paper_2404_06359_b200/libmc.so /tmp/libmc_orig.so
for so in build_var/libmc_*.so; do
  cp $so paper_2404_06359_b200/libmc.so
  name=$(basename $so .so)
  timeout 600 python scripts/sweep_cfg5.py --out /tmp/sw_$name.jsonl --sizes ${SIZES:-32x32,64x64} --bits ${BITS:-16} --label $name > /dev/null 2>&1
  python -c "
import json
for l in open('/tmp/sw_$name.jsonl'):
    d=json.loads(l); print('$name', d['vmax'], d['tmax'], d['bits'], round(d['gtri_s'],1), round(d['alg_gb_s']), d['error_bits'])"
done
cp /tmp/libmc_orig.so paper_2404_06359_b200/libmc.so
