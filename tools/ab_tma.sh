# (Needs the commit that added HOOD_RING_TMA; the variant was removed after this A/B.)
# A/B of the ring kernel's fill: 8 cp.async (LDGSTS) per lane vs one TMA tile
# (UTMALDG + mbarrier) per warp and block; same box, alternating, 3 rounds.
mkdir -p gpurun_out
HOOD_RING_TMA=1 timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_tma.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_tma.log
: > gpurun_out/ab_tma.log
for r in 1 2 3; do
  for c in 2 5 4 3 1; do
    for t in 0 1; do
      st=20; [ $c = 4 ] && st=10
      HOOD_RING_TMA=$t timeout 300 python bench.py --config $c --steps $st --warmup 5 --cpu-seconds 0.01 --no-e2e 2>/dev/null | tail -1 | python tools/benchline.py | sed "s/^/tma=$t /" >> gpurun_out/ab_tma.log
    done
  done
done
tail -3 gpurun_out/pytest_gpu_tma.log
