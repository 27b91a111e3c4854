# A/B: the working tree's library vs lib/libhood_b200_prev.so (the last commit's), config 4, alternating.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "stealing or config4 or acceptance_fixture" > gpurun_out/pytest_ab.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ab.log
: > gpurun_out/ab_prev.log
for r in 1 2 3; do
  timeout 300 python bench.py --config 4 --steps 10 --warmup 5 --cpu-seconds 0.01 --no-e2e 2>/dev/null | tail -1 | python tools/benchline.py | sed "s/^/new /" >> gpurun_out/ab_prev.log
  HOOD_B200_LIB=$PWD/paper_1203_5004_b200/lib/libhood_b200_prev.so timeout 300 python bench.py --config 4 --steps 10 --warmup 5 --cpu-seconds 0.01 --no-e2e 2>/dev/null | tail -1 | python tools/benchline.py | sed "s/^/prev /" >> gpurun_out/ab_prev.log
done
