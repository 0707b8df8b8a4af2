# cfg5 points (SIZES x BITS at INST instances) for every build_var variant, REPS times interleaved
mkdir -p gpurun_out
cp paper_2404_06359_b200/libmc.so /tmp/libmc_orig.so
rm -f gpurun_out/swab_*.jsonl
for rep in $(seq ${REPS:-2}); do
for so in build_var/libmc_*.so; do
  name=$(basename $so .so); cp $so paper_2404_06359_b200/libmc.so
  timeout 900 python scripts/sweep_cfg5.py --instances ${INST:-100} --out gpurun_out/swab_${name}_$rep.jsonl --sizes ${SIZES:-32x32,64x64} --bits ${BITS:-16} --label $name > /dev/null 2>&1
done
done
cp /tmp/libmc_orig.so paper_2404_06359_b200/libmc.so
cat gpurun_out/swab_*.jsonl | python -c "
import json,sys
r={}
for l in sys.stdin:
    d=json.loads(l); r.setdefault((d['vmax'],d['tmax'],d['bits'],d['label']),[]).append(round(d['gtri_s'],1))
for k in sorted(r): print(k, r[k])"
