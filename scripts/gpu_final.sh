# final confirmation of the product build: GPU parity tests, smoke, default bench, cfg2 line
mkdir -p gpurun_out/fin
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/fin/bench.json 2> gpurun_out/fin/bench.err; cut -c1-200 gpurun_out/fin/bench.json
timeout 600 python bench.py --workload cfg2_torus --steps 30 > gpurun_out/fin/bench_cfg2_torus.json 2> gpurun_out/fin/bench_cfg2.err; cut -c1-200 gpurun_out/fin/bench_cfg2_torus.json
