# Round-2 ncu captures (one --set full launch each) + the bench launch list; run on the GPU box.
# Summaries are written on the box (gpurun_out/profiles_<tag>/); only the cfg4 report is kept.
# usage: bash scripts/prof_r2.sh <tag> [names...]   (names: cfg4 cfg4u8 cfg4vw shard8 cfg2 cfg5_32x32_b16 ...)
set -x
TAG=${1:-r2}; shift
NAMES=${@:-"launches cfg4 cfg4u8 cfg4vw shard8 cfg2 cfg5_32x32_b16 cfg5_64x64_b16 cfg5_64x126_b8 cfg5_64x126_b16"}
OUT=gpurun_out/profiles_$TAG
mkdir -p $OUT
export MC_PROFILES_DIR=$OUT
NCU="ncu --set full --import-source on --clock-control none -k regex:mc_decode_kernel"
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
for name in $NAMES; do
  rep=gpurun_out/prof_${name}_$TAG
  case $name in
    launches) timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv \
                 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; continue;;
    cfg4) timeout 900 $NCU -s 3 -c 1 -o $rep -f $B > /dev/null 2>&1;;
    cfg4u8) timeout 900 $NCU -s 3 -c 1 -o $rep -f $B --index-format u8x4 > /dev/null 2>&1;;
    cfg4vw) timeout 900 $NCU -s 3 -c 1 -o $rep -f $B --variable-widths > /dev/null 2>&1;;
    shard8) timeout 900 $NCU -s 3 -c 1 -o $rep -f $B --instances 125 > /dev/null 2>&1;;
    cfg2) timeout 900 $NCU -s 3 -c 1 -o $rep -f $B --workload cfg2_torus > /dev/null 2>&1;;
    cfg5_*) pt=${name#cfg5_}; sz=${pt%_b*}; b=${pt##*_b}
            timeout 900 $NCU -s 4 -c 1 -o $rep -f python scripts/sweep_cfg5.py --out /tmp/x.jsonl --sizes $sz --bits $b --steps 2 > /dev/null 2>&1;;
  esac
  python scripts/ncu_summary.py $rep.ncu-rep round2_${name} $name 1 > /dev/null 2>&1
  python scripts/ncu_lines.py $rep.ncu-rep 1 60 > $OUT/round2_${name}_lines.txt 2>&1
  if [ "$name" != cfg4 ]; then rm -f $rep.ncu-rep; fi
done
ls -la $OUT gpurun_out/*.ncu-rep
