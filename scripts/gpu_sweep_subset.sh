# cfg5 subset sweep for each build_var/libmc_*.so (A/B of the T~ > 128 path)
# usage: SIZES=128x256,256x256 BITS=16,8 bash scripts/gpu_sweep_subset.sh
mkdir -p gpurun_out
cp paper_2404_06359_b200/libmc.so /tmp/libmc_orig.so
for so in build_var/libmc_*.so; do
  name=$(basename $so .so); name=${name#libmc_}
  cp $so paper_2404_06359_b200/libmc.so
  timeout 900 python scripts/sweep_cfg5.py --label $name --sizes ${SIZES:-128x256,256x256} --bits ${BITS:-16} --out gpurun_out/sweep_subset.jsonl 2>/dev/null \
    | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['label'], d['vmax'], d['tmax'], d['bits'], round(d['gtri_s'],2), round(d['alg_gb_s']), d['error_bits'])"
done
cp /tmp/libmc_orig.so paper_2404_06359_b200/libmc.so
