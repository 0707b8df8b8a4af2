# cfg5 sweep for each build_var/libmc_*.so, plus cfg1-3 bench lines with the product build
mkdir -p gpurun_out
cp paper_2404_06359_b200/libmc.so /tmp/libmc_orig.so
for so in build_var/libmc_*.so; do
  name=$(basename $so .so); name=${name#libmc_}
  cp $so paper_2404_06359_b200/libmc.so
  timeout 900 python scripts/sweep_cfg5.py --label $name --out gpurun_out/sweep_cfg5.jsonl > /dev/null 2> gpurun_out/sweep_$name.err || tail -5 gpurun_out/sweep_$name.err
done
cp /tmp/libmc_orig.so paper_2404_06359_b200/libmc.so
for w in cfg1_grid cfg2_torus cfg3_sphere; do
  timeout 600 python bench.py --workload $w --steps 30 > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err || tail -5 gpurun_out/bench_$w.err
done
wc -l gpurun_out/sweep_cfg5.jsonl
