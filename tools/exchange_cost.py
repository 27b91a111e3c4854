"""Cost of the multi-GPU exchange pieces on one GPU (world 1 NCCL group):
graph-captured build alone, + pack, + all-gather, + merge.

  python -m torch.distributed.run --nproc-per-node 1 --master-addr 127.0.0.1 tools/exchange_cost.py
"""
import os
import statistics
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1203_5004_b200 import hood as H  # noqa: E402
from paper_1203_5004_b200 import workloads as W  # noqa: E402

dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
dev = torch.device("cuda", 0)
pts = W.grid_uniform_torch(1 << 24, seed=2)
ctx = H.Context.get(0)
ctx.reserve(pts.shape[0])
corners = torch.empty_like(pts)
counts = torch.empty(1, dtype=torch.int32, device=dev)
CAP = 4096
W_ = dist.get_world_size()
rec = torch.zeros(CAP + 1, 2, dtype=torch.float64, device=dev)
gathered = torch.zeros(W_, CAP + 1, 2, dtype=torch.float64, device=dev)
final = torch.empty(W_ * CAP, 2, dtype=torch.float64, device=dev)
fcnt = torch.empty(1, dtype=torch.int32, device=dev)
flush = torch.empty(64 << 20, dtype=torch.int32, device=dev)


def stage(k):
    H.build_hood_async(pts, corners=corners, counts=counts)
    if k >= 1:
        H.pack_record(corners, counts, CAP, 0.0, rec=rec)
    if k >= 2:
        dist.all_gather_into_tensor(gathered.view(-1), rec.view(-1))
    if k >= 3:
        H.merge_records(gathered, out=final, out_count=fcnt)


for k, name in enumerate(["build", "+pack", "+all_gather", "+merge"]):
    stage(k)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        stage(k)
    ts = []
    for i in range(15):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(a.elapsed_time(b) * 1e3)
    print(f"{name:12s} {statistics.median(ts):7.1f} us")

# the merge of an 8-rank exchange, records prepared from 8 slabs on this GPU
recs8 = []
for g in range(8):
    p = W.grid_uniform_torch(1 << 24, seed=10 + g)
    rep = H.build_hood(p)
    recs8.append(H.pack_record(rep.corners, rep.counts, CAP, x_offset=float(g)))
recs8 = torch.stack(recs8)
out8 = torch.empty(8 * CAP, 2, dtype=torch.float64, device=dev)
H.merge_records(recs8, out=out8, out_count=fcnt)
torch.cuda.synchronize()
g8 = torch.cuda.CUDAGraph()
with torch.cuda.graph(g8):
    H.merge_records(recs8, out=out8, out_count=fcnt)
ts = []
for i in range(15):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    g8.replay()
    b.record()
    torch.cuda.synchronize()
    if i >= 3:
        ts.append(a.elapsed_time(b) * 1e3)
print(f"merge of 8 records ({int(recs8[:, 0, 0].sum())} corners -> {int(fcnt)}): {statistics.median(ts):.1f} us")
dist.destroy_process_group()
