# ncu --set full of the product build's timed decode kernel for a few workloads + line tables
mkdir -p gpurun_out/prof_now
NCU="ncu --set full --import-source on --clock-control none -k regex:mc_decode_kernel"
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --sustained-seconds 0"
for w in ${WLS:-"u32:" "u8:--index-format u8x4" "vw:--variable-widths"}; do
  n=${w%%:*}; a=${w#*:}
  timeout 600 $NCU -s 3 -c 1 -o gpurun_out/prof_now/$n -f $B $a > /dev/null 2>&1
  python scripts/ncu_lines.py gpurun_out/prof_now/$n.ncu-rep 1141049 60 > gpurun_out/prof_now/${n}_lines.txt 2>&1
done
