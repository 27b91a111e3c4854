# One GPU round: parity tests, then the bench configs (no e2e).
set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
for c in 1 2 3 5 4; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --cpu-seconds 0.5 2>&1 | tail -1 | python tools/benchline.py; done
for d in 14 33; do for c in 2 5; do HOOD_RING=$d timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --cpu-seconds 0.5 2>&1 | tail -1 | python tools/benchline.py "R=$d"; done; done
