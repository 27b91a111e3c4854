# batched arc-like instances: the transposed pass vs the fallback (timing only)
import os, sys, torch, numpy as np
sys.path.insert(0, os.getcwd())
from paper_1203_5004_b200 import hood as H, workloads as W
n_inst, L = 8192, 1024
x = (np.arange(L) + 0.5) / L
base = np.stack([x, 0.25 + x * (1 - x)], 1)
p = np.tile(base, (n_inst, 1)).astype(np.float32).astype(np.float64)
t = torch.as_tensor(p).float().cuda() if False else torch.as_tensor(p.astype(np.float32)).cuda()
corners = torch.empty_like(t); counts = torch.empty(n_inst, dtype=torch.int32, device="cuda")
for _ in range(3): H.build_hood_async(t, L, corners=corners, counts=counts)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(10): H.build_hood_async(t, L, corners=corners, counts=counts)
b.record(); torch.cuda.synchronize()
print("batched arc 8192 x 1024 float: %.1f us/build, hull %d" % (a.elapsed_time(b) * 100, int(counts[0])))
