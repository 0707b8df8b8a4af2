set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "decode_host" 2>&1 | tail -5
for c in 0 4 8 16 32 64; do
timeout 600 python bench.py --steps 10 --no-cpu-baseline --e2e-chunks $c 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($c, d['value'], d['e2e'])"
done
