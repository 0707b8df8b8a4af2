set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -8
timeout 900 python bench.py > gpurun_out/bench3.json 2> gpurun_out/bench3.err; tail -3 gpurun_out/bench3.err; cat gpurun_out/bench3.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ref3.json 2> gpurun_out/ref3.err; tail -2 gpurun_out/ref3.err; cat gpurun_out/ref3.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches3.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; grep -c mc_decode gpurun_out/launches3.csv
nproc; lscpu | grep "Model name"
