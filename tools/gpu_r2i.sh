mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 --cpu-seconds 1 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
cat > /tmp/san.py <<'PY'
import numpy as np, torch, sys
sys.path.insert(0, '.')
from paper_1203_5004_b200 import hood as H, workloads as W
for p, L in [(W.grid_uniform(1 << 16, seed=1), 0), (W.arc(1 << 14), 0), (W.batched(64, 1024, seed=5), 1024), (W.gauss(1 << 18, seed=3), 0)]:
    r = H.build_hood(torch.as_tensor(p).cuda(), block_len=L)
    print(int(r.counts[0]))
t = torch.as_tensor(W.grid_uniform(1 << 12, seed=2).astype(np.float64)).cuda()
H.match_and_merge_block(t, 2)
print("ok")
PY
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python /tmp/san.py > gpurun_out/sanitizer_memcheck.log 2>&1; echo "rc=$?" >> gpurun_out/sanitizer_memcheck.log
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python /tmp/san.py > gpurun_out/sanitizer_racecheck.log 2>&1; echo "rc=$?" >> gpurun_out/sanitizer_racecheck.log
tail -3 gpurun_out/pytest_gpu.log
