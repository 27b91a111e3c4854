# Experiment: single-instance builds on the register-light LEAN ring kernel
# with a smaller smem hood/queue (HC=48, PC=48: 4 CTAs/SM for double2 too).
mkdir -p gpurun_out
L48=$PWD/paper_1203_5004_b200/lib/libhood_b200_lean48_48.so
HOOD_LEAN_SINGLE=1 HOOD_B200_LIB=$L48 timeout 900 python -m pytest tests -m gpu -q -x -k "config or random_sizes or known_answers or finished_unit or graph" > gpurun_out/pytest_lean1.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_lean1.log
: > gpurun_out/ab_lean1.log
for r in 1 2; do for c in 4 2; do
  st=20; [ $c = 4 ] && st=10
  timeout 300 python bench.py --config $c --steps $st --warmup 5 --cpu-seconds 0.01 --no-e2e 2>/dev/null | tail -1 | python tools/benchline.py | sed "s/^/base /" >> gpurun_out/ab_lean1.log
  HOOD_LEAN_SINGLE=1 HOOD_B200_LIB=$L48 timeout 300 python bench.py --config $c --steps $st --warmup 5 --cpu-seconds 0.01 --no-e2e 2>/dev/null | tail -1 | python tools/benchline.py | sed "s/^/lean48 /" >> gpurun_out/ab_lean1.log
done; done
tail -2 gpurun_out/pytest_lean1.log
