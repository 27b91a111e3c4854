# Experiment: the ring kernel at 128 registers with a 48-corner smem hood and
# a 48-entry survivor queue (4 CTAs = 16 warps per SM for both storages).
mkdir -p gpurun_out
R=$PWD/paper_1203_5004_b200/lib/libhood_b200_r128.so
HOOD_B200_LIB=$R timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_r128.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r128.log
: > gpurun_out/ab_r128.log
for r in 1 2; do for c in 4 2 3 5 1; do
  st=20; [ $c = 4 ] && st=10
  timeout 300 python bench.py --config $c --steps $st --warmup 5 --cpu-seconds 0.01 --no-e2e 2>/dev/null | tail -1 | python tools/benchline.py | sed "s/^/base /" >> gpurun_out/ab_r128.log
  HOOD_B200_LIB=$R timeout 300 python bench.py --config $c --steps $st --warmup 5 --cpu-seconds 0.01 --no-e2e 2>/dev/null | tail -1 | python tools/benchline.py | sed "s/^/r128 /" >> gpurun_out/ab_r128.log
done; done
tail -2 gpurun_out/pytest_r128.log
