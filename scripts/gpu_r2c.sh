set -x
mkdir -p gpurun_out
compute-sanitizer --tool racecheck --print-limit 100 python tests/sanitize_decode.py > gpurun_out/racecheck_full.log 2>&1; grep -c "Race reported\|hazard" gpurun_out/racecheck_full.log; tail -3 gpurun_out/racecheck_full.log
compute-sanitizer --tool synccheck python tests/sanitize_decode.py > gpurun_out/synccheck_full.log 2>&1; tail -3 gpurun_out/synccheck_full.log
SIZES=32x32,64x64,64x126 BITS=16,8 bash scripts/variants_sweep.sh > gpurun_out/var_small.log 2>&1; cat gpurun_out/var_small.log
bash scripts/size_sweep.sh > gpurun_out/size_sweep.log 2>&1; cat gpurun_out/size_sweep.log
