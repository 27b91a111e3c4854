mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -k "stealing" > gpurun_out/pytest_steal.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_steal.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
python tools/steal_diag.py > gpurun_out/steal_diag.log 2>&1
: > gpurun_out/ab_steal.log
for r in 1 2 3; do for c in 4 2; do
  st=20; [ $c = 4 ] && st=10
  for t in 0 1; do HOOD_STEAL=$t timeout 300 python bench.py --config $c --steps $st --warmup 5 --cpu-seconds 0.01 --no-e2e 2>/dev/null | tail -1 | python tools/benchline.py | sed "s/^/steal=$t /" >> gpurun_out/ab_steal.log; done
done; done
