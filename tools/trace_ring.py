"""In-kernel timeline of the ring kernel (globaltimer): first warp entry, last
prologue end, last warp exit, against the event-measured kernel time.

  python tools/trace_ring.py [log2n ... | b (batched 65536 x 1024) | g<log2n> (Gaussian double)]
"""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1203_5004_b200 import hood as H  # noqa: E402
from paper_1203_5004_b200 import workloads as W  # noqa: E402

L = H.library()
L.hood_internal_set_debug.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
ctx = H.Context.get(0)
trace = torch.zeros(1024 + 16 * 8192, dtype=torch.int64, device="cuda")
flush = torch.empty(64 << 20, dtype=torch.int32, device="cuda")
for lg in sys.argv[1:] or ["12", "16", "20", "22", "24"]:
    block = 0
    if lg == "b":
        pts, block = W.batched_torch(65536, 1024, seed=5), 1024
    elif lg.startswith("g"):
        pts = W.gauss_torch(1 << int(lg[1:]), seed=4)
    elif lg.startswith("a"):
        pts = W.arc_torch(1 << int(lg[1:]))
    else:
        pts = W.grid_uniform_torch(1 << int(lg), seed=2)
    n = pts.shape[0]
    tiny = pts[: 1 << 14].clone()
    tiny_out = torch.empty_like(tiny)
    tiny_cnt = torch.empty(1, dtype=torch.int32, device="cuda")
    corners = torch.empty_like(pts)
    counts = torch.empty(max(n // block, 1) if block else 1, dtype=torch.int32, device="cuda")
    for rep in range(4):
        trace.zero_()
        trace[0] = (1 << 63) - 1
        flush.zero_()
        if os.environ.get("TLBWARM"):  # one element per 2 MiB page of the input and output
            stride = (2 << 20) // pts.element_size()
            _ = pts.view(-1)[::stride].sum() + corners.view(-1)[::stride].sum()
        if os.environ.get("L2WARM"):
            _ = pts.sum()
        if os.environ.get("CODEWARM"):  # the same kernels on a tiny input: their code into L2
            H.build_hood_async(tiny, corners=tiny_out, counts=tiny_cnt)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for e in (a, b):
            e.record()
        L.hood_internal_set_debug(ctx.handle, 0, trace.data_ptr())
        if not os.environ.get("NOEV"):
            ctx.set_profile_events(a, b)
        H.build_hood_async(pts, block, corners=corners, counts=counts)
        ctx.set_profile_events(None, None)
        L.hood_internal_set_debug(ctx.handle, 0, None)
        torch.cuda.synchronize()
        t = trace[:64].cpu().tolist()
        fin0 = int(trace[7 * 64 + 30])
        fin1 = int(trace[7 * 64 + 31])
        finr = int(trace[7 * 64 + 29])
    print(f"log2n={lg}: event {a.elapsed_time(b)*1e3:7.1f} us; in-kernel: prologue done +{(t[2]-t[0])/1e3:6.1f} us, "
          f"last exit +{(t[1]-t[0])/1e3:6.1f} us" + (f", finalize starts +{(fin0 - t[0])/1e3:6.1f} us" if fin0 else "")
          + (f", ends +{(fin1 - t[0])/1e3:6.1f} us" if fin1 else "")
          + (f"; finalize CTA resident +{(finr - t[0])/1e3:6.1f} us" if finr else ""))
    w = trace[1024:1024 + 4 * 8192].view(-1, 4).cpu()
    cyc = trace[1024 + 4 * 8192:1024 + 8 * 8192].view(-1, 4).cpu()
    ex2 = trace[1024 + 8 * 8192:1024 + 12 * 8192].view(-1, 4).cpu()
    ex3 = trace[1024 + 12 * 8192:].view(-1, 4).cpu()
    keep = w[:, 0] > 0
    w = w[keep]
    cyc = cyc[keep]
    ex2 = ex2[keep]
    ex3 = ex3[keep]
    ent = (w[:, 0] - t[0]).double() / 1e3
    ext = (w[:, 1] - t[0]).double() / 1e3
    dur = ext - ent
    q = lambda v: " ".join(f"{float(v.quantile(x)):.1f}" for x in (0, 0.1, 0.5, 0.9, 1.0))
    print(f"   {len(w)} warps; entry q0/10/50/90/100: {q(ent)}; exit: {q(ext)}; duration: {q(dur)}")
    cnt = w[:, 3]
    if int(cnt.min()) > 1 << 40:  # per-warp prologue end (globaltimer) instead of counters
        pro = (cnt - t[0]).double() / 1e3
        print(f"   prologue end q0/10/50/90/100: {q(pro)}; exit - prologue end: {q(ext - pro)}")
        print(f"   corr(prologue end, exit) = {float(torch.corrcoef(torch.stack([pro, ext]))[0, 1]):.2f}")
    elif int(cnt.abs().sum()):
        cand = (cnt >> 32).double(); edge = ((cnt >> 16) & 0xffff).double(); many = (cnt & 0xffff).double()
        order = torch.argsort(dur)
        print("   fastest (sm, us, cand, edge, many):", [(int(w[i, 2]), round(float(dur[i]), 1), int(cand[i]), int(edge[i]), int(many[i])) for i in order[:8]])
        print("   slowest:", [(int(w[i, 2]), round(float(dur[i]), 1), int(cand[i]), int(edge[i]), int(many[i])) for i in order[-12:]])
        c = torch.corrcoef(torch.stack([dur, cand]))[0, 1]
        for nm, j in (("cand+many path", 0), ("flush", 1), ("land", 2)):
            v = cyc[:, j].double() / 1965.0
            print(f"   {nm}: mean {float(v.mean()):.1f} us/warp, corr with duration {float(torch.corrcoef(torch.stack([dur, v]))[0, 1]):.2f}; slowest warps: {[round(float(v[i]), 1) for i in order[-6:]]}")
        print(f"   mean cand {float(cand.mean()):.1f} many {float(many.mean()):.2f} edge {float(edge.mean()):.2f}; corr(duration, cand) = {float(c):.2f}")
        # duration by SM: mean over the SM's warps
        import collections
        bysm = collections.defaultdict(list)
        for i in range(len(w)):
            bysm[int(w[i, 2])].append(float(dur[i]))
        means = sorted((sum(v) / len(v), k) for k, v in bysm.items())
        print("   SM mean duration: fastest", [(k, round(m, 1)) for m, k in means[:5]], "slowest", [(k, round(m, 1)) for m, k in means[-5:]])
    if int(cyc[:, 0].abs().sum()) and int(cyc[:, 3].min()) > 1 << 40:  # STEAL kernel: steals per warp
        nst = cyc[:, 0]
        lt = (cyc[:, 1] - t[0]).double() / 1e3
        lk = cyc[:, 2]
        oe = (cyc[:, 3] - t[0]).double() / 1e3
        order = torch.argsort(ext)
        print(f"   steals per warp: mean {float(nst.double().mean()):.2f} max {int(nst.max())}; own range end q0/50/100: "
              f"{float(oe.min()):.1f} {float(oe.median()):.1f} {float(oe.max()):.1f}")
        re = (ex2[:, 0] - t[0]).double() / 1e3
        mg = ex2[:, 1].double() / 1e3
        print("   last 16 exits (exit, own range end, steals, last steal at, its blocks, last range's end, merge us):",
              [(round(float(ext[i]), 1), round(float(oe[i]), 1), int(nst[i]), round(float(lt[i]), 1) if int(nst[i]) else None,
                int(lk[i]), round(float(re[i]), 1), round(float(mg[i]), 1)) for i in order[-16:]])
        print(f"   merge time per warp: mean {float(mg.mean()):.2f} us, max {float(mg.max()):.1f}; warps that merged: {int((mg > 0).sum())}")
        rs = (ex2[:, 2] - t[0]).double() / 1e3
        rb = (ex2[:, 3] & 0xffffffff).double()
        rc = (ex2[:, 3] >> 32).double()
        per = (re - rs) / rb.clamp(min=1)
        th = nst > 0
        print(f"   last range: us per block, thieves q50/90 {float(per[th].median()):.2f} {float(per[th].quantile(0.9)):.2f}; "
              f"owners (unstolen last range) q50/90 {float(per[~th].median()):.2f} {float(per[~th].quantile(0.9)):.2f}")
        ok = (ex3[:, 3] > 0)
        if int(ok.sum()):
            tt = (ex3[ok].double() - t[0]) / 1e3
            en = ent[ok]
            r0 = (tt[:, 0] - en) / 128
            rr = [(tt[:, j + 1] - tt[:, j]) / 128 for j in range(3)]
            print(f"   us per block by phase (warps with >= 512 blocks, {int(ok.sum())}): blocks 0-127 {float(r0.median()):.3f}, "
                  + ", ".join(f"{128 * (j + 1)}-{128 * (j + 2) - 1} {float(r.median()):.3f}" for j, r in enumerate(rr))
                  + f"; at {float(tt[:, 3].median()):.0f} us")
            late = ok & (nst == 0) & (rb > 530)
            if int(late.sum()):
                t512 = (ex3[late][:, 3].double() - t[0]) / 1e3
                rl = (re[late] - t512) / (rb[late] - 512)
                print(f"   warps that never stole, blocks 512..end of their unit ({int(late.sum())}): "
                      f"{float(rl.median()):.3f} us per block (q90 {float(rl.quantile(0.9)):.3f}), ending at {float(re[late].median()):.0f} us")
        print(f"   last range: candidate blocks per block, thieves {float((rc[th] / rb[th].clamp(min=1)).mean()):.3f}, "
              f"owners {float((rc[~th] / rb[~th].clamp(min=1)).mean()):.3f}")
        print("   last 16 exits (range start, blocks, us/block):", [(round(float(rs[i]), 1), int(rb[i]), round(float(per[i]), 2)) for i in order[-16:]])
        print(f"   exit - last range end: q50 {float((ext - re).median()):.1f} q90 {float((ext - re).quantile(0.9)):.1f} max {float((ext - re).max()):.1f}")
        thief = nst > 0
        for nm, m in (("warps that stole", thief), ("warps that did not", ~thief)):
            if int(m.sum()):
                print(f"   {nm}: {int(m.sum())}, exit q50/90/100 {float(ext[m].median()):.1f} "
                      f"{float(ext[m].quantile(0.9)):.1f} {float(ext[m].max()):.1f}")
    import collections
    persm = collections.defaultdict(list)
    for i in range(len(w)):
        persm[int(w[i, 2])].append(float(ext[i]))
    smx = sorted((max(v), k) for k, v in persm.items())
    print("   per-SM last exit: min", smx[0], "median", smx[len(smx)//2], "max", smx[-3:])
    # which warps are slow: by warp-in-CTA, by CTA wave (blockIdx // SMs), by SM
    idx = torch.nonzero(keep).flatten()
    gw = idx.double()
    wic = (idx % 4)
    cta = idx // 4
    nsm = len(persm)
    wave = cta // max(nsm, 1)
    for nm, key in (("warp in CTA", wic), ("CTA wave", wave)):
        parts = []
        for k in sorted(set(key.tolist())):
            m = key == k
            parts.append(f"{k}: {float(dur[m].mean()):.1f}")
        print(f"   mean duration by {nm}: " + ", ".join(parts))
    if os.environ.get("DUMP"):
        torch.save({"w": w, "dur": dur, "ext": ext, "idx": idx}, os.environ["DUMP"])
