# Parity tests, then the bench configs (no e2e).
set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for c in 1 2 3 5 4; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --cpu-seconds 0.05 2>&1 | tail -1 | python tools/benchline.py; done
python tools/trace_ring.py 24 2>&1 | tail -4
