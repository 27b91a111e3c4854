set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
for c in 1 2 3 5 4; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-e2e 2>&1 | tail -2; done
