set -x
mkdir -p gpurun_out
python scripts/power_probe.py > gpurun_out/power_probe.json 2>gpurun_out/power_probe.err; head -c 600 gpurun_out/power_probe.json
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/tests_r2g.log 2>&1; tail -3 gpurun_out/tests_r2g.log
timeout 1800 python scripts/sweep_cfg5.py --instances 100 --out gpurun_out/sweep_cfg5_100_r2g.jsonl --label r2g100 > /dev/null 2>&1; wc -l gpurun_out/sweep_cfg5_100_r2g.jsonl
bash scripts/prof_r2.sh r2g cfg5_64x126_b10 cfg5_64x126_b12 cfg4u8 cfg4vw > gpurun_out/prof_r2g.log 2>&1; rm -f gpurun_out/*.ncu-rep; ls gpurun_out/profiles_r2g
