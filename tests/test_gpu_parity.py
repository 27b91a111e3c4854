"""GPU parity: libhood_b200.so (through the C-ABI) vs the pinned CPU oracle.

Bit-exact comparison of corner coordinates (corners are selections of input
points; hood_b200.h).  Golden vectors restate the reference's own tests with
file:line; the fixtures come from the reference itself (tests/golden/).
"""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

from paper_1203_5004_b200 import hood as H  # noqa: E402
from paper_1203_5004_b200 import workloads as W  # noqa: E402

R = (10.0, 0.0)
A, B, C, D = (0.1, 0.5), (0.2, 0.6), (0.6, 0.9), (0.7, 0.2)


def gpu_hull(pts, dtype=torch.float64, **kw):
    t = torch.as_tensor(np.asarray(pts), dtype=dtype).cuda().contiguous()
    return H.build_hood(t, **kw).hull.cpu().numpy()


def same(a, b):
    a = np.asarray(a)
    b = np.asarray(b, dtype=a.dtype)
    return a.shape == b.shape and np.array_equal(a, b)


# ------------------------------------------------------------ golden vectors

@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_known_answers(dtype):
    npd = np.float64 if dtype == torch.float64 else np.float32
    cases = [
        ([A, B, C, D], [A, B, C, D]),                                        # test_kernel.cpp:119-125
        ([(0.1, 0.9), (0.3, 0.3), (0.6, 0.25), (0.9, 0.8)], [(0.1, 0.9), (0.9, 0.8)]),  # :127-132
        ([A, B, (0.6, 0.1), (0.7, 0.2)], [A, B, (0.7, 0.2)]),                # :133-138
        ([(0.2, 0.4), (0.6, 0.3)], [(0.2, 0.4), (0.6, 0.3)]),                # :141-151
        ([(0.05, 0.5), (0.1, 0.45), (0.15, 0.35), (0.2, 0.2),
          (0.8, 0.2), (0.85, 0.35), (0.9, 0.45), (0.95, 0.5)], [(0.05, 0.5), (0.95, 0.5)]),  # :153-168
        ([(0.05, 0.05), (0.25, 0.09), (0.45, 0.1), (0.5, 0.05), (0.55, 0.3), (0.6, 0.35)],
         [(0.05, 0.05), (0.6, 0.35)]),                                         # :269-300
        ([(0.3, 0.4), (0.6, 0.2)], [(0.3, 0.4), (0.6, 0.2)]),                # test_driver.cpp:36-42
        ([(0.5, 0.5)], [(0.5, 0.5)]),
    ]
    for pts, want in cases:
        assert same(gpu_hull(pts, dtype), np.array(want, dtype=npd)), pts
    par = [(k / 9.0, (k / 9.0) * (1.0 - k / 9.0)) for k in range(1, 9)]   # test_driver.cpp:51-59
    assert same(gpu_hull(par, dtype), np.array(par, dtype=npd))
    s8 = [(0.0625, 0.05859375), (0.125, 0.109375), (0.1875, 0.15234375), (0.25, 0.1875),
          (0.3125, 0.21484375), (0.375, 0.234375), (0.4375, 0.24609375), (0.5, 0.25)]  # data/sample8.txt
    assert same(gpu_hull(s8, dtype), np.array(s8, dtype=npd))


def test_dyadic_degenerate_resolved_like_oracle(oracle_mod):
    """test_kernel.cpp:330-350: the reference kernel flags this collinear
    tangency; the oracle resolves it (collinear middle points dropped) and so
    does the GPU path, bit for bit."""
    pts = np.array([(0.0625, 0.25), (0.125, 0.4), (0.25, 0.5), (0.3125, 0.46875),
                    (0.5625, 0.3), (0.625, 0.3125), (0.6875, 0.28), (0.75, 0.2)])
    assert same(gpu_hull(pts), oracle_mod.upper_hull(pts))


def test_acceptance_fixture_sweep(golden):
    """acceptance.cpp:44-72 criterion 1 against hood::build_hood's own output."""
    g = golden("acceptance.npz")
    for n in [4, 8, 16, 32, 64, 128, 256, 512, 1024]:
        pts = g[f"pts_{n}"]
        for s in range(pts.shape[0]):
            k = int(g[f"count_{n}"][s])
            assert same(gpu_hull(pts[s]), g[f"hull_{n}"][s][:k]), (n, s)


def test_driver_fixture(golden):  # test_driver.cpp:61-70
    g = golden("driver.npz")
    for n in [4, 8, 32, 128, 256]:
        for s in range(8):
            k = int(g[f"count_{n}"][s])
            assert same(gpu_hull(g[f"pts_{n}"][s]), g[f"hull_{n}"][s][:k])


def test_raw_reference_fixture(golden):
    g = golden("raw.npz")
    for e in [11, 12, 13, 14]:
        n = 1 << e
        assert same(gpu_hull(g[f"uniform_pts_{n}"]), g[f"uniform_hull_{n}"])
    assert same(gpu_hull(W.grid_uniform(1 << 16, seed=1), torch.float32).astype(np.float64), g["grid65536_hull"])
    assert same(gpu_hull(W.gauss(1 << 16, seed=4)), g["gauss65536_hull"])


def test_per_round_blocks(golden, oracle_mod):
    """acceptance criterion 2 / test_driver.cpp:72-94: every round-r block is
    the hull of its interval -- the GPU batched mode with block_len = d."""
    g = golden("acceptance.npz")
    for n in [64, 128, 256]:
        for s in range(4):
            p = g[f"pts_{n}"][s]
            t = torch.as_tensor(p).cuda()
            for r, buf in enumerate(g[f"rounds_{n}"][s]):
                d = 4 << r
                if d < 8:
                    continue
                rep = H.build_hood(t, block_len=d, padded=True)
                assert same(rep.padded.cpu().numpy(), buf), (n, s, d)


# ------------------------------------------------------------ random / degenerate

@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_random_sizes(oracle_mod, dtype):
    rng = np.random.default_rng(11)
    npd = np.float64 if dtype == torch.float64 else np.float32
    for n in [1, 2, 3, 5, 15, 16, 17, 255, 256, 257, 1000, 4095, 4096, 4097, 8191, 20000, 65537, 300001,
              1 << 20]:
        x = np.sort(rng.random(n)).astype(npd)
        ok = np.concatenate([[True], np.diff(x) > 0])
        x, m = x[ok], int(ok.sum())
        p = np.stack([x, rng.random(m).astype(npd)], axis=1)
        assert same(gpu_hull(p, dtype), oracle_mod.upper_hull(p)), n


def test_lattice_degenerate(oracle_mod):
    """Exactly collinear triples everywhere (exact predicates): the strict hull
    must match the oracle's pop-on-collinear rule."""
    for seed in range(12):
        for n, span in [(500, 16), (5000, 64), (70000, 256), (300000, 4096)]:
            p = W.lattice(n, span, seed=seed)
            assert same(gpu_hull(p), oracle_mod.upper_hull(p)), (seed, n)
            p32 = p.astype(np.float32)
            if np.all(np.diff(p32[:, 0]) > 0):
                assert same(gpu_hull(p32, torch.float32), oracle_mod.upper_hull(p32)), (seed, n)


def test_concave_and_convex_shapes(oracle_mod):
    for n in [100, 5000, 70000, 1 << 18]:
        a = W.arc(n)
        assert same(gpu_hull(a), oracle_mod.upper_hull(a))
        cup = a.copy()
        cup[:, 1] = 1.0 - cup[:, 1]
        assert same(gpu_hull(cup), oracle_mod.upper_hull(cup))
        # arc with a dent: large hulls cut in the middle (global merge path)
        dent = a.copy()
        dent[n // 3: 2 * n // 3, 1] -= 0.2
        assert same(gpu_hull(dent), oracle_mod.upper_hull(dent))


# ------------------------------------------------------------ the five configs

def test_config1_grid_2p16(oracle_mod):
    p = W.grid_uniform(1 << 16, seed=1)
    assert same(gpu_hull(p, torch.float32), oracle_mod.upper_hull(p))


def test_config2_grid_2p24(oracle_mod):
    t = W.grid_uniform_torch(1 << 24, seed=2)
    got = H.build_hood(t).hull.cpu().numpy()
    assert same(got, oracle_mod.upper_hull(t.cpu().numpy()))


def test_config3_arc_2p22(oracle_mod):
    t = W.arc_torch(1 << 22)
    rep = H.build_hood(t)
    assert int(rep.counts[0]) == 1 << 22
    assert same(rep.hull.cpu().numpy(), oracle_mod.upper_hull(t.cpu().numpy()))


def test_config4_gauss_2p26(oracle_mod):
    t = W.gauss_torch(1 << 26, seed=4)
    got = H.build_hood(t).hull.cpu().numpy()
    assert same(got, oracle_mod.upper_hull(t.cpu().numpy()))


@pytest.mark.slow
def test_config4_gauss_2p28(oracle_mod):
    t = W.gauss_torch(1 << 28, seed=4)
    got = H.build_hood(t).hull.cpu().numpy()
    host = t.cpu().numpy()
    del t
    assert same(got, oracle_mod.upper_hull(host))


def test_config5_batched(oracle_mod):
    t = W.batched_torch(65536, 1024, seed=5)
    rep = H.build_hood(t, block_len=1024)
    host = t.cpu().numpy()
    slots, counts = oracle_mod.block_hulls(host, 1024)
    gc = rep.counts.cpu().numpy()
    assert np.array_equal(gc, counts)
    gs = rep.corners.cpu().numpy()
    mask = (np.arange(1024)[None, :] < counts[:, None]).reshape(-1)
    assert np.array_equal(gs[mask], slots[mask])


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("block", [8, 16, 64, 256, 1024, 4096, 1 << 14, 1 << 16])
def test_block_lengths(oracle_mod, dtype, block):
    n = 1 << 20
    if dtype == torch.float32 and block < 16:
        pytest.skip("float2 chunks are 16 points")
    p = W.batched(n // block, block, seed=block) if block <= (1 << 14) else None
    if p is None:
        p = np.concatenate([W.grid_uniform(block, seed=s) for s in range(n // block)])
    p = p.astype(np.float64 if dtype == torch.float64 else np.float32)
    t = torch.as_tensor(p).cuda()
    rep = H.build_hood(t, block_len=block)
    slots, counts = oracle_mod.block_hulls(p, block)
    assert np.array_equal(rep.counts.cpu().numpy(), counts)
    mask = (np.arange(block)[None, :] < counts[:, None]).reshape(-1)
    assert np.array_equal(rep.corners.cpu().numpy()[mask], slots[mask])


# ------------------------------------------------------------ boundary behaviour

def test_padded_output(oracle_mod):
    p = W.grid_uniform(1 << 16, seed=9)
    t = torch.as_tensor(p).cuda()
    rep = H.build_hood(t, padded=True)
    h = oracle_mod.upper_hull(p)
    pad = rep.padded.cpu().numpy()
    assert np.array_equal(pad[: len(h)], h)
    assert np.all(pad[len(h):, 0] == 10.0) and np.all(pad[len(h):, 1] == 0.0)


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_x_not_increasing_reported(dtype):
    for n, bad in [(8, 3), (5000, 4096), (5000, 4095), (1 << 20, 777777), (1 << 20, 1)]:
        x = np.linspace(0.1, 0.9, n)
        x[bad] = x[bad - 1]
        p = np.stack([x, np.full(n, 0.5)], axis=1)
        with pytest.raises(H.ValidationError) as ei:
            gpu_hull(p, dtype)
        assert ei.value.code == H.HOOD_ERR_X_NOT_INCREASING and ei.value.index == bad


def test_x_range_check():
    p = np.array([(0.1, 0.5), (1.2, 0.6)])
    assert same(gpu_hull(p), p)  # the raw path (oracle::upper_hull) accepts it
    with pytest.raises(H.ValidationError) as ei:
        gpu_hull(p, check_range=True)
    assert ei.value.code == H.HOOD_ERR_X_OUT_OF_RANGE and ei.value.index == 1


def test_invalid_block_len():
    t = torch.rand(100, 2, dtype=torch.float64).cuda()
    with pytest.raises(H.HoodError):
        H.build_hood(t, block_len=7)


def test_host_path(oracle_mod):
    for p in [W.grid_uniform(1 << 20, seed=3), W.gauss(1 << 20, seed=6), W.arc(1 << 16)]:
        out, counts = H.build_hood_host(np.ascontiguousarray(p))
        assert same(out[: counts[0]], oracle_mod.upper_hull(p))
    b = W.batched(256, 1024, seed=8)
    out, counts = H.build_hood_host(b, block_len=1024)
    slots, oc = oracle_mod.block_hulls(b, 1024)
    assert np.array_equal(counts, oc)


@pytest.mark.parametrize("G", [2, 4, 8, 64])
def test_merge_segments(oracle_mod, G):
    """The multi-GPU exchange step on one device: per-slab hoods, then the
    final merge (A10 shows slab hulls compose exactly)."""
    for maker in [lambda: W.gauss(1 << 20, seed=G), lambda: W.arc(1 << 14)]:
        p = maker()
        n = p.shape[0]
        slabs = np.array_split(p, G)
        stride = max(len(s) for s in slabs)
        seg = torch.zeros(G, stride, 2, dtype=torch.float64, device="cuda")
        cnt = torch.zeros(G, dtype=torch.int32, device="cuda")
        for g, s in enumerate(slabs):
            h = H.build_hood(torch.as_tensor(np.ascontiguousarray(s)).cuda()).hull
            seg[g, : h.shape[0]] = h
            cnt[g] = h.shape[0]
        out, c = H.merge_segments(seg, cnt)
        torch.cuda.synchronize()
        got = out[: int(c[0])].cpu().numpy()
        assert same(got, oracle_mod.upper_hull(p)), (G, n)


def test_graph_capture_replay(oracle_mod):
    p = W.grid_uniform(1 << 20, seed=12)
    t = torch.as_tensor(p).cuda()
    ctx = H.Context.get(0)
    ctx.reserve(t.shape[0])
    corners = torch.empty_like(t)
    counts = torch.empty(1, dtype=torch.int32, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        H.build_hood_async(t, corners=corners, counts=counts)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        H.build_hood_async(t, corners=corners, counts=counts)
    corners.zero_()
    g.replay()
    torch.cuda.synchronize()
    h = oracle_mod.upper_hull(p)
    assert int(counts[0]) == len(h)
    assert same(corners[: len(h)].cpu().numpy(), h)


@pytest.mark.parametrize("n", [1 << 20, 3000])
def test_error_record_reset_every_replay(n):
    """The error record is reset inside the build (a kernel the ring kernel
    follows programmatically): a replay after a bad one reports clean, a bad
    one after clean replays reports the right index."""
    x = np.linspace(0.1, 0.9, n)
    p = np.stack([x, np.sin(9 * x)], axis=1)
    t = torch.as_tensor(p).cuda()
    ctx = H.Context.get(0)
    corners = torch.empty_like(t)
    counts = torch.empty(1, dtype=torch.int32, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        H.build_hood_async(t, corners=corners, counts=counts)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        H.build_hood_async(t, corners=corners, counts=counts)
    bad = n // 3
    for rnd in range(3):
        t[bad, 0] = t[bad - 1, 0]
        g.replay()
        torch.cuda.synchronize()
        with pytest.raises(H.ValidationError) as ei:
            ctx.last_error()
        assert ei.value.index == bad
        t[bad, 0] = float(x[bad])
        g.replay()
        torch.cuda.synchronize()
        ctx.last_error()  # clean
        assert int(counts[0]) > 0
        bad = n - 1 - rnd


def test_cpp_dropin_binary():
    """tests/cpp/test_dropin.cpp: include/hood_b200.hpp from C++, the
    reference's Point2 layout, known answers + random sets + errors."""
    import os
    import subprocess
    from paper_1203_5004_b200 import build as Bd
    Bd.build()
    exe = os.path.join(os.path.dirname(Bd.SO), "test_dropin")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "OK" in r.stdout


def test_sharded_build_on_device(oracle_mod):
    """distributed.sharded_build with the CUDA build and merge, one rank over
    NCCL (the N>1 protocol is covered by tests/test_distributed.py on gloo)."""
    import os
    import socket
    import torch.distributed as dist
    from paper_1203_5004_b200 import distributed as Dz
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        p = W.grid_uniform(1 << 18, seed=31)
        res = Dz.sharded_build(torch.as_tensor(p).cuda(), x_offset=0.0)
        assert res.exchanges == 1
        assert same(res.hull.cpu().numpy(), oracle_mod.upper_hull(p))
        res = Dz.sharded_build(torch.as_tensor(W.arc(1 << 14)).cuda(), cap=256)
        assert res.exchanges == 2
        assert same(res.hull.cpu().numpy(), oracle_mod.upper_hull(W.arc(1 << 14)))
    finally:
        dist.destroy_process_group()


def test_merge_round_reference_pairs(golden):
    """hood_merge_round on the reference's random hood pairs
    (make_random_hood_pair, acceptance.cpp:79) against match_and_merge_block's
    merged windows (test_kernel.cpp:302-328), REMOTE padding included."""
    P = golden("pairs.npz")
    for d in sorted(set(int(x) for x in P["pq"][:, 0])):
        idx = [t for t in range(P["pq"].shape[0]) if int(P["pq"][t, 0]) == d]
        buf = np.concatenate([P["slots"][t][: 2 * d] for t in idx])
        want = np.concatenate([P["merged"][t][: 2 * d] for t in idx])
        got = H.merge_round(torch.as_tensor(buf).cuda(), d).cpu().numpy()
        assert same(got, want), d


def test_merge_round_reproduces_reference_rounds(golden):
    """Every round of the reference round loop (driver.cpp:20-43) on the
    acceptance sweep (acceptance.cpp:46-64): round r's input buffer -> the
    reference's round-r output buffer, all 8 sets of a size in one call."""
    A = golden("acceptance.npz")
    for N in [4, 8, 16, 32, 64, 128, 256]:
        pts, rounds = A[f"pts_{N}"], A[f"rounds_{N}"]
        cur = pts.reshape(-1, 2)
        for r in range(rounds.shape[1]):
            d = 2 ** (r + 1)
            got = H.merge_round(torch.as_tensor(np.ascontiguousarray(cur)).cuda(), d).cpu().numpy()
            want = rounds[:, r].reshape(-1, 2)
            assert same(got, want), (N, r)
            cur = want


def test_merge_round_float_storage_and_in_place(oracle_mod):
    """float2 slots, in-place (d_in == d_out), chained over all rounds from
    blocks of 2 up to one block: the last buffer holds the reference hull."""
    p = W.grid_uniform(1 << 12, seed=21).astype(np.float32)
    t = torch.as_tensor(p).cuda()
    d = 2
    while d < t.shape[0]:
        H.merge_round(t, d, out=t)
        d *= 2
    h = oracle_mod.upper_hull(p.astype(np.float64))
    got = t.cpu().numpy()
    assert same(got[: len(h)], h)
    assert np.all(got[len(h):, 0] == 10.0) and np.all(got[len(h):, 1] == 0.0)


@pytest.mark.parametrize("G", [1, 2, 8])
@pytest.mark.parametrize("shape", ["uniform", "arc"])
def test_pack_and_merge_records(oracle_mod, G, shape):
    """The multi-GPU exchange kernels on one GPU: G slab hoods packed into
    records (x shifted by the slab index, exact in double), stacked as the
    all-gather would, merged -- small totals take the one-warp hull in the
    gather kernel, large ones (arc) the finalize kernel."""
    cap = 4096
    recs, full = [], []
    for g in range(G):
        p = (W.grid_uniform(1 << 14, seed=40 + g) if shape == "uniform" else W.arc(1 << 10)).astype(np.float64)
        t = torch.as_tensor(p.astype(np.float32) if shape == "uniform" else p).cuda()
        rep = H.build_hood(t)
        recs.append(H.pack_record(rep.corners, rep.counts, cap, x_offset=float(g)))
        q = p.copy()
        q[:, 0] += g
        full.append(q)
    out, cnt = H.merge_records(torch.stack(recs))
    torch.cuda.synchronize()
    got = out[: int(cnt[0])].cpu().numpy()
    want = oracle_mod.upper_hull(np.concatenate(full))
    assert same(got, want), (G, shape)


def _shape_points(kind, n, rng):
    """x strictly increasing on the 2^-24 grid (float-exact); y by shape."""
    step = max((1 << 24) // n, 1)
    x = (np.arange(n, dtype=np.int64) * step + rng.integers(1, max(step, 2), size=n)) * 2.0 ** -24
    x = np.clip(x, 2.0 ** -24, 1 - 2.0 ** -24)
    x = np.maximum.accumulate(x)
    x = x + np.arange(n) * 0.0  # keep dtype
    if kind == "uniform":
        y = rng.integers(1, 1 << 24, size=n) * 2.0 ** -24
    elif kind == "sawtooth":
        y = ((np.arange(n) % 97) / 97.0 * 0.5 + 0.25)
    elif kind == "steps":
        y = np.floor(np.arange(n) / max(n // 16, 1)) / 32.0 + 0.1
    elif kind == "cap":
        t = x
        y = 0.2 + t * (1 - t) + rng.integers(0, 8, size=n) * 2.0 ** -24
    elif kind == "cup":
        t = x
        y = 0.8 - t * (1 - t)
    elif kind == "clusters":
        y = rng.choice([0.3, 0.5, 0.7], size=n) + rng.integers(0, 1 << 10, size=n) * 2.0 ** -24
    else:  # "ties": many equal y values
        y = rng.integers(0, 4, size=n) * 0.125 + 0.25
    y = np.round(y * 2 ** 24) / 2 ** 24
    pts = np.stack([x, y], axis=1)
    keep = np.concatenate([[True], np.diff(pts[:, 0]) > 0])
    return pts[keep]


@pytest.mark.parametrize("kind", ["uniform", "sawtooth", "steps", "cap", "cup", "clusters", "ties"])
def test_random_shapes_sizes_and_storages(oracle_mod, kind):
    """Randomised parity sweep: shapes with collinear runs, plateaus and ties,
    sizes across block/unit boundaries, float2 and double2 storage."""
    rng = np.random.default_rng(sum(map(ord, kind)))  # stable across processes
    for n in [3, 31, 512, 513, 4095, 4096, 70001, 1 << 18]:
        p = _shape_points(kind, n, rng)
        want = oracle_mod.upper_hull(p)
        for dt in (torch.float32, torch.float64):
            got = gpu_hull(p, dtype=dt)
            assert same(got, want), (kind, n, dt)


@pytest.mark.parametrize("L", [512, 1024, 4096, 1 << 14])
def test_batched_random_shapes(oracle_mod, L):
    rng = np.random.default_rng(L)
    inst = max((1 << 18) // L, 2)
    parts = []
    for i in range(inst):
        kind = ["uniform", "cap", "steps", "ties", "sawtooth"][i % 5]
        q = _shape_points(kind, L, rng)
        while q.shape[0] < L:  # duplicates removed: pad by re-drawing
            q = _shape_points(kind, L, rng)
        parts.append(q[:L])
    p = np.concatenate(parts)
    t = torch.as_tensor(p).cuda()
    rep = H.build_hood(t, block_len=L)
    c = rep.counts.cpu().numpy()
    corners = rep.corners.cpu().numpy()
    for i in range(inst):
        want = oracle_mod.upper_hull(parts[i])
        assert same(corners[i * L: i * L + c[i]], want), (L, i)
    # host path: one strided copy of the widest instance
    out, counts = H.build_hood_host(np.ascontiguousarray(p), block_len=L)
    for i in range(inst):
        assert same(out[i * L: i * L + counts[i]], corners[i * L: i * L + c[i]]), (L, i)


def test_c_abi_argument_errors():
    """The C-ABI rejects bad arguments with HOOD_ERR_INVALID_ARG (never a crash
    or a silent fallback) and keeps working afterwards."""
    import ctypes
    L = H.library()
    ctx = H.Context.get(0)
    t = torch.as_tensor(W.grid_uniform(1 << 12, seed=3)).cuda()
    out = torch.empty_like(t)
    cnt = torch.empty(1, dtype=torch.int32, device="cuda")
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    assert L.hood_build_f32(ctx.handle, t.data_ptr(), 0, 0, out.data_ptr(), cnt.data_ptr(), None, 0, s) == \
        H.HOOD_ERR_INVALID_ARG                                                      # n = 0
    assert L.hood_build_f32(ctx.handle, t.data_ptr(), t.shape[0], 3, out.data_ptr(), cnt.data_ptr(), None, 0, s) == \
        H.HOOD_ERR_INVALID_ARG                                                      # block_len not a power of two
    assert L.hood_build_f32(ctx.handle, t.data_ptr(), t.shape[0], 1 << 13, out.data_ptr(), cnt.data_ptr(), None,
                            0, s) == H.HOOD_ERR_INVALID_ARG                         # block_len does not divide n
    assert L.hood_merge_round_f32(ctx.handle, t.data_ptr(), t.shape[0], 3, out.data_ptr(), s) == \
        H.HOOD_ERR_INVALID_ARG                                                      # d not a power of two
    assert L.hood_merge_segments_f64(ctx.handle, None, None, 2, 4, None, None, s) == H.HOOD_ERR_INVALID_ARG
    assert L.hood_build_f32(None, t.data_ptr(), t.shape[0], 0, out.data_ptr(), cnt.data_ptr(), None, 0, s) != 0
    # still healthy
    rep = H.build_hood(t)
    assert rep.hull.shape[0] >= 2


def test_tiny_inputs(oracle_mod):
    for pts in [[(0.5, 0.5)], [(0.25, 0.1), (0.75, 0.9)], [(0.1, 0.2), (0.2, 0.1), (0.3, 0.2)]]:
        p = np.array(pts, dtype=np.float64)
        for dt in (torch.float32, torch.float64):
            assert same(gpu_hull(p, dtype=dt), oracle_mod.upper_hull(p)), (pts, dt)
        out, counts = H.build_hood_host(np.ascontiguousarray(p))
        assert same(out[: counts[0]], oracle_mod.upper_hull(p))


@pytest.mark.parametrize("G", [1, 3])
def test_build_multi_single_process(oracle_mod, G):
    """hood_build_multi (one context per device, P2P record copies to the
    first device): here G contexts share cuda:0 -- the copies are same-device
    but take the same code path."""
    slabs, full = [], []
    for g in range(G):
        p = W.grid_uniform(1 << 16, seed=70 + g)
        slabs.append(torch.as_tensor(p).cuda())
        q = p.astype(np.float64)
        q[:, 0] += g
        full.append(q)
    ctxs = [H.Context(0) for _ in range(G)]
    got = H.build_multi(slabs, contexts=ctxs, x_offsets=[float(g) for g in range(G)]).cpu().numpy()
    assert same(got, oracle_mod.upper_hull(np.concatenate(full)))
    # double storage, no offsets (slabs already in global coordinates)
    p = W.gauss(1 << 18, seed=9)
    parts = np.array_split(p, G)
    got = H.build_multi([torch.as_tensor(np.ascontiguousarray(x)).cuda() for x in parts], contexts=ctxs).cpu().numpy()
    assert same(got, oracle_mod.upper_hull(p))


def test_trace_file_matches_reference(golden, tmp_path):
    """write_trace: the reference's round loop on the GPU (hood_merge_round per
    round) with the CLI's on_round_begin trace writer (cli.cpp:108-118,
    163-169), byte-identical to the reference's own `hull` run."""
    from paper_1203_5004_b200 import io as IO
    g = golden("trace.npz")
    off, toff = g["pts_off"], g["trace_off"]
    blob = bytes(g["trace_blob"])
    for i in range(len(off) - 1):
        pts = g["pts"][off[i]:off[i + 1]]
        path = tmp_path / f"t{i}.trace"
        IO.write_trace(str(path), pts)
        assert path.read_bytes() == blob[toff[i]:toff[i + 1]], len(pts)


def test_finished_unit_counter_across_builds(oracle_mod):
    """The finalize of a single-instance build starts on a finished-unit
    counter that it resets for the next build: interleaved sizes (different
    unit counts), batched builds in between, and graph replays must all see a
    clean counter and produce the oracle's hood."""
    ctx = H.Context.get(0)
    sets = [W.grid_uniform(1 << 20, seed=31), W.gauss(1 << 22, seed=32), W.grid_uniform(1 << 18, seed=33)]
    ts = [torch.as_tensor(p).cuda() for p in sets]
    want = [oracle_mod.upper_hull(p) for p in sets]
    bat = torch.as_tensor(W.batched(256, 1024, seed=34)).cuda()
    for rnd in range(3):
        for t, w in zip(ts, want):
            assert same(H.build_hood(t).hull.cpu().numpy(), w)
            H.build_hood(bat, block_len=1024)
    t = ts[0]
    ctx.reserve(t.shape[0])
    corners = torch.empty_like(t)
    counts = torch.empty(1, dtype=torch.int32, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        H.build_hood_async(t, corners=corners, counts=counts)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        H.build_hood_async(t, corners=corners, counts=counts)
    for rnd in range(5):
        corners.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert same(corners[: int(counts[0])].cpu().numpy(), want[0])
        assert same(H.build_hood(ts[1]).hull.cpu().numpy(), want[1])


def test_bare_read_reference_kernel_runs():
    """bench.py's attainable-read reference (hood_internal_stream_read): it
    launches, reads the whole buffer and leaves it untouched."""
    import ctypes
    t = torch.rand(1 << 20, 2, device="cuda")
    before = t.clone()
    ctx = H.Context.get(0)
    s = torch.cuda.current_stream()
    rc = H.library().hood_internal_stream_read(ctx.handle, ctypes.c_void_p(t.data_ptr()),
                                               ctypes.c_longlong(t.numel() * 4), ctypes.c_void_p(s.cuda_stream))
    torch.cuda.synchronize()
    assert rc == 0 and torch.equal(t, before)
    assert H.library().hood_internal_stream_read(ctx.handle, None, ctypes.c_longlong(64), None) != 0


# ------------------------------------------------ round 2: seams and errors

def test_merge_round_scratch_reference_pairs(golden):
    """The pinpoint phase's scratch (kernel.cpp:101-112): after the round,
    scratch[start] = pindex and scratch[start+1] = qindex, the values the
    reference's match_and_merge_block leaves (test_kernel.cpp:302-328)."""
    P = golden("pairs.npz")
    for d in sorted(set(int(x) for x in P["pq"][:, 0])):
        idx = [t for t in range(P["pq"].shape[0]) if int(P["pq"][t, 0]) == d]
        buf = np.concatenate([P["slots"][t][: 2 * d] for t in idx])
        sc = torch.full((buf.shape[0],), -7, dtype=torch.int32, device="cuda")
        out = H.match_and_merge_block(torch.as_tensor(buf).cuda(), d, scratch=sc)
        got = sc.cpu().numpy().reshape(len(idx), 2 * d)[:, :2]
        want = np.stack([P["scratch01"][t] for t in idx]) + np.arange(len(idx))[:, None] * 2 * d
        assert np.array_equal(got, want), d
        assert same(out.cpu().numpy(), np.concatenate([P["merged"][t][: 2 * d] for t in idx])), d


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_merge_round_scratch_known_answers(dtype):
    """E1 (test_kernel.cpp:98-102): pindex 1, qindex 2; singletons
    (test_kernel.cpp:141-151): 0 and 2; stale corners (test_kernel.cpp:153-168)
    with its tangent (0, 3) -> slots 0 and 7."""
    cases = [([A, B, C, D], 2, (1, 2), [A, B, C, D]),
             ([(0.2, 0.4), R, (0.6, 0.3), R], 2, (0, 2), [(0.2, 0.4), (0.6, 0.3), R, R]),
             ([(0.05, 0.5), (0.1, 0.45), (0.15, 0.35), (0.2, 0.2),
               (0.8, 0.2), (0.85, 0.35), (0.9, 0.45), (0.95, 0.5)], 4, (0, 7),
              [(0.05, 0.5), (0.95, 0.5), R, R, R, R, R, R])]
    for slots, d, pq, merged in cases:
        t = torch.as_tensor(np.array(slots), dtype=dtype).cuda()
        sc = torch.zeros(t.shape[0], dtype=torch.int32, device="cuda")
        out = H.match_and_merge_block(t, d, scratch=sc)
        assert tuple(sc[:2].cpu().tolist()) == pq
        assert same(out.cpu().numpy(), np.array(merged, dtype=np.float64).astype(out.cpu().numpy().dtype))


def test_merge_round_flags_degenerate_tangent():
    """test_kernel.cpp:330-350: p2, p3 and q1 on one dyadic line -- the
    reference flags the block (DegenerateTangent or a pinpoint write-write
    conflict); hood_merge_round reports HOOD_ERR_DEGENERATE for block 0, and a
    clean pair next to it does not mask it."""
    deg = [(0.0625, 0.25), (0.125, 0.4), (0.25, 0.5), (0.3125, 0.46875),
           (0.5625, 0.3), (0.625, 0.3125), (0.6875, 0.28), (0.75, 0.2)]
    ok = [(0.1, 0.5), (0.2, 0.6), (0.6, 0.9), (0.7, 0.2), (0.75, 0.1), (0.8, 0.15), (0.85, 0.12), (0.9, 0.05)]
    for blocks, bad in [([deg], 0), ([ok, deg], 1), ([deg, ok], 0)]:
        t = torch.as_tensor(np.concatenate([np.array(b) for b in blocks])).cuda()
        with pytest.raises(H.HoodError) as ei:
            H.match_and_merge_block(t, 4)
        assert ei.value.code == H.HOOD_ERR_DEGENERATE and ei.value.index == bad
    H.match_and_merge_block(torch.as_tensor(np.array(ok)).cuda(), 4)  # clean: no error


def _triple_points(n, bad_i, seed):
    """x strictly increasing on the 2^-24 grid, y random; with bad_i >= 0 the
    triple (bad_i, bad_i+1, bad_i+2) is made exactly collinear."""
    rng = np.random.default_rng(seed)
    x = (np.arange(n) * 8 + rng.integers(1, 8, size=n)) * 2.0 ** -24 * (1 << 20) / n
    y = rng.integers(1 << 20, 1 << 23, size=n) * 2.0 ** -24
    if bad_i >= 0:
        y[bad_i + 2] = y[bad_i] + (y[bad_i + 1] - y[bad_i]) * (x[bad_i + 2] - x[bad_i]) / (x[bad_i + 1] - x[bad_i])
    return np.stack([x, y], axis=1)


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_check_triples_first_index(oracle_mod, dtype):
    """HOOD_FLAG_CHECK_TRIPLES: validate_points' consecutive-triple margin
    (hoodbuf.cpp:16-26, :59) fused into the build: the first degenerate i is
    reported, exactly the reference's double |orient| < 1e-9 on the stored
    values, and x errors win over triple errors (hoodbuf.cpp:48-58 first)."""
    import ctypes
    L = H.library()
    for n, bad in [(1 << 16, 40000), (1 << 16, 1), (1 << 20, 777777), (5000, 4097), (3000, 0)]:
        p = _triple_points(n, bad, seed=n + bad)
        t = torch.as_tensor(p, dtype=dtype).cuda()
        stored = t.double().cpu().numpy()
        xs, ys = stored[:, 0], stored[:, 1]
        det = (xs[1:-1] - xs[:-2]) * (ys[2:] - ys[:-2]) - (ys[1:-1] - ys[:-2]) * (xs[2:] - xs[:-2])
        first = int(np.nonzero(np.abs(det) < 1e-9)[0][0]) if np.any(np.abs(det) < 1e-9) else -1
        assert first >= 0
        with pytest.raises(H.ValidationError) as ei:
            H.build_hood(t, check_triples=True)
        assert ei.value.code == H.HOOD_ERR_DEGENERATE_TRIPLE and ei.value.index == first, (n, bad)
        # the host path and the reference validate_points agree on the index
        if O_ref_ok(oracle_mod) and dtype == torch.float64:
            r = oracle_mod.ref_validate_points(stored)
            if r != -1 and r[1][1] == r[1][0] + 1 and r[1][2] == r[1][0] + 2 and n > 64 and n & (n - 1) == 0:
                assert r[1][0] == first
        # without the flag the same points build fine (and match the oracle)
        assert same(H.build_hood(t).hull.cpu().numpy(), oracle_mod.upper_hull(stored))
    # an x error before the triple wins
    p = _triple_points(1 << 14, 100, seed=3)
    p[9000, 0] = p[8999, 0]
    with pytest.raises(H.ValidationError) as ei:
        H.build_hood(torch.as_tensor(p).cuda(), check_triples=True)
    assert ei.value.code == H.HOOD_ERR_X_NOT_INCREASING and ei.value.index == 9000
    # clean input passes with the flag on; batched instances never cross
    p = np.concatenate([_triple_points(1024, -1, seed=s) for s in range(64)])
    t = torch.as_tensor(p).cuda()
    stored = p
    ok = True
    for i in range(64):
        q = stored[i * 1024:(i + 1) * 1024]
        det = (q[1:-1, 0] - q[:-2, 0]) * (q[2:, 1] - q[:-2, 1]) - (q[1:-1, 1] - q[:-2, 1]) * (q[2:, 0] - q[:-2, 0])
        ok &= not np.any(np.abs(det) < 1e-9)
    if ok:
        H.build_hood(t, block_len=1024, check_triples=True)
    for L_ in (16, 1024):  # instance kernel (L < one ring block) and ring kernel
        q = _triple_points(1 << 14, -1, seed=L_)
        i0 = 3 * L_ - 2  # straddles instances 2|3: not a triple of either
        q[i0 + 2, 1] = q[i0, 1] + (q[i0 + 1, 1] - q[i0, 1]) * (q[i0 + 2, 0] - q[i0, 0]) / (q[i0 + 1, 0] - q[i0, 0])
        det_ok = True
        for b in range(q.shape[0] // L_):
            w = q[b * L_:(b + 1) * L_]
            dd = (w[1:-1, 0] - w[:-2, 0]) * (w[2:, 1] - w[:-2, 1]) - (w[1:-1, 1] - w[:-2, 1]) * (w[2:, 0] - w[:-2, 0])
            det_ok &= not np.any(np.abs(dd) < 1e-9)
        if det_ok:
            H.build_hood(torch.as_tensor(q).cuda(), block_len=L_, check_triples=True)


def O_ref_ok(oracle_mod):
    return oracle_mod.ref_available()


def test_record_capacity_is_reported_not_truncated(oracle_mod):
    """hood_pack_record / hood_merge_records with a slab hood larger than the
    record: HOOD_ERR_CAPACITY with the capacity needed, never a silently
    truncated global hood; hood_build_multi sizes its records itself and
    returns the oracle's hood."""
    arc = W.arc(1 << 12)
    t = torch.as_tensor(arc).cuda()
    ctx = H.Context.get(0)
    rep = H.build_hood(t)
    cap = 1000
    rec = H.pack_record(rep.corners, rep.counts, cap)
    H.merge_records(torch.stack([rec, rec]))
    with pytest.raises(H.CapacityError) as ei:
        ctx.last_error()
    assert ei.value.index == 1 << 12
    # a fresh build clears the record
    H.build_hood(t)
    # build_multi: two arc slabs (every point a corner) with cap far below
    halves = [torch.as_tensor(np.ascontiguousarray(h)).cuda() for h in np.array_split(arc, 2)]
    ctxs = [H.Context(0) for _ in range(2)]
    got = H.build_multi(halves, contexts=ctxs, cap=3000).cpu().numpy()
    assert same(got, oracle_mod.upper_hull(arc))
    with pytest.raises(H.CapacityError):
        H.build_multi(halves, contexts=ctxs, cap=100)


def test_contexts_per_thread_and_stream_order(oracle_mod):
    """Python contexts are per (device, thread); builds from two threads on
    two streams at once produce the oracle's hoods."""
    import threading
    sets = [W.grid_uniform(1 << 20, seed=80 + i) for i in range(2)]
    want = [oracle_mod.upper_hull(p) for p in sets]
    errs = []

    def work(i):
        try:
            s = torch.cuda.Stream()
            t = torch.as_tensor(sets[i]).cuda()
            for _ in range(20):
                with torch.cuda.stream(s):
                    rep = H.build_hood(t)
                if not same(rep.hull.cpu().numpy(), want[i]):
                    errs.append(i)
        except Exception as e:  # pragma: no cover
            errs.append(repr(e))
    th = [threading.Thread(target=work, args=(i,)) for i in range(2)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    assert not errs
    # one context, alternating streams: each build ordered after the last
    t = torch.as_tensor(sets[0]).cuda()
    streams = [torch.cuda.Stream() for _ in range(3)]
    outs = []
    for i in range(9):
        with torch.cuda.stream(streams[i % 3]):
            outs.append(H.build_hood_async(t))
    torch.cuda.synchronize()
    for r in outs:
        assert same(r.hull.cpu().numpy(), want[0])


def test_host_path_pageable_and_pinned(oracle_mod):
    """hood_build_host_* from pageable memory (staged by host threads through
    the context's pinned bounce buffers, many 16 MiB chunks) and from pinned
    memory (direct DMA) give the same hood as the oracle, single and batched;
    an x error in a late chunk still reports its exact index."""
    p = W.gauss(1 << 23, seed=44)  # 128 MiB of double2: 8 staged chunks
    want = oracle_mod.upper_hull(p)
    out, counts = H.build_hood_host(np.ascontiguousarray(p))
    assert same(out[: counts[0]], want)
    pin = torch.as_tensor(p).pin_memory()
    ctx = H.Context.get(0)
    o = torch.empty_like(pin).pin_memory()
    c = torch.zeros(1, dtype=torch.int32).pin_memory()
    assert H.build_hood_host_ptr(ctx, pin.data_ptr(), p.shape[0], True, o.data_ptr(), c.data_ptr()) == 0
    assert same(o[: int(c[0])].numpy(), want)
    b = W.batched(1 << 14, 1024, seed=45)  # 128 MiB float2, one launch after the last chunk
    out, counts = H.build_hood_host(np.ascontiguousarray(b), block_len=1024)
    for i in range(0, 1 << 14, 997):
        assert same(out[i * 1024: i * 1024 + counts[i]], oracle_mod.upper_hull(b[i * 1024:(i + 1) * 1024])), i
    q = p.copy()
    q[7_000_001, 0] = q[7_000_000, 0]
    with pytest.raises(H.ValidationError) as ei:
        H.build_hood_host(np.ascontiguousarray(q))
    assert ei.value.code == H.HOOD_ERR_X_NOT_INCREASING and ei.value.index == 7_000_001


# ------------------------------------------ adversarial near-degenerate doubles

def _adv_sets():
    import adversarial as A
    out = []
    for n in (1 << 10, 1 << 14, 1 << 18, 1 << 21):
        for sh in (0.0, -1.5, 1.5, 1e6):
            out.append((f"clusters n={n} shift={sh}", A.ulp_clusters(n, seed=n % 977 + int(sh) % 13, shift=sh)))
        out.append((f"tied top n={n}", A.tied_top(n, seed=n % 31)))
    return out


def plateau_tie_only(got, want):
    """True when got and want differ only in WHICH point of an equal-y run
    a few ulps wide in x is kept -- the one divergence the design admits on
    inputs outside the reference's collinearity contract (DESIGN.md section
    2.3): the reference's monotone chain pops the left end of such a plateau
    when fl(c1.x - s.x) == fl(c.x - s.x) against a FAR stack element s
    (geom.hpp:26-28 strict >), a rounding coincidence no local merge can see."""
    gs = {tuple(r) for r in np.asarray(got, dtype=np.float64)}
    ws = {tuple(r) for r in np.asarray(want, dtype=np.float64)}
    if len(gs) != len(ws):
        return False
    for p in gs ^ ws:
        other = ws if p in gs else gs
        if not any(q[1] == p[1] and abs(q[0] - p[0]) <= 8 * np.spacing(max(abs(p[0]), abs(q[0])))
                   for q in other - (gs & ws)):
            return False
    return True


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_adversarial_ulp_clusters_single(oracle_mod, dtype):
    """Clusters of 3-5 points within a few ulps (x by nextafter steps, y
    within +-3 ulps) at hull corners, points within an ulp of hull edges,
    plateaus, y < 0 and y > 1, a tied top, against the reference's
    oracle::upper_hull (oracle/_ref when built, else the pinned restatement):
    float storage bit for bit; double storage bit for bit except (at most)
    the plateau-tie choice, and nothing else."""
    import adversarial as A
    ref = oracle_mod.ref_upper_hull if oracle_mod.ref_available() else oracle_mod.upper_hull
    sets = _adv_sets() if dtype == torch.float64 else [
        (f"f32 clusters n={n}", A.ulp_clusters(n, seed=n % 101, dtype=np.float32)) for n in (1 << 10, 1 << 14, 1 << 18, 1 << 21)]
    bad, ties = [], []
    for name, p in sets:
        want = ref(p.astype(np.float64))
        got = gpu_hull(p, dtype=dtype).astype(np.float64)
        if not same(got, want):
            (ties if dtype == torch.float64 and plateau_tie_only(got, want) else bad).append(name)
    assert not bad, bad
    assert len(ties) <= len(sets) // 4, ties


def test_adversarial_ulp_clusters_batched(oracle_mod):
    """The same clusters inside batched 1024-point instances (the warp-level
    unit-end hull) and 2^16-point instances (ring units + finalize)."""
    import adversarial as A
    for L in (1024, 1 << 16):
        inst = 64 if L == 1024 else 8
        parts = []
        for i in range(inst):
            q = A.ulp_clusters(L - 5 * 40, seed=1000 + i, clusters=40, shift=(-1.5, 0.0, 1.5)[i % 3])
            q = q[:L]
            while q.shape[0] < L:  # pad on the right with low points
                q = np.concatenate([q, [[np.nextafter(q[-1, 0], 2.0), q[:, 1].min() - 1.0]]])
            parts.append(q)
        p = np.concatenate(parts)
        rep = H.build_hood(torch.as_tensor(p).cuda(), block_len=L)
        c = rep.counts.cpu().numpy()
        corners = rep.corners.cpu().numpy()
        ties = 0
        for i in range(inst):
            got, want = corners[i * L: i * L + c[i]], oracle_mod.upper_hull(parts[i])
            if not same(got, want):
                assert plateau_tie_only(got, want), (L, i)
                ties += 1
        assert ties <= inst // 4, (L, ties)


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_acceptance_full_sweep_100_seeds(golden, dtype):
    """acceptance.cpp:43-72 criterion 1, all 900 runs (100 seeds x n = 4 ..
    1024): each size's 100 point sets as one batched build (block_len = n)
    and as single builds (double only), against the reference build_hood's
    hull of every run.  float storage: the same sets rounded to float, against
    the oracle of the rounded points."""
    import oracle as O
    g = golden("acceptance.npz")
    for n in [4, 8, 16, 32, 64, 128, 256, 512, 1024]:
        pts, hulls, cnt = g[f"pts100_{n}"], g[f"hulls100_{n}"], g[f"count100_{n}"]
        off = np.concatenate([[0], np.cumsum(cnt)])
        flat = np.ascontiguousarray(pts.reshape(-1, 2))
        if n < 16:  # instances shorter than one 128-byte chunk row: single builds
            for s in range(100):
                p = pts[s] if dtype == torch.float64 else pts[s].astype(np.float32)
                if dtype == torch.float32 and not np.all(np.diff(p[:, 0]) > 0):
                    continue
                want = hulls[off[s]:off[s + 1]] if dtype == torch.float64 else O.upper_hull(p)
                assert same(gpu_hull(p, dtype=dtype), want), (n, s)
            continue
        if dtype == torch.float32:
            flat32 = flat.astype(np.float32)
            keep = all(np.all(np.diff(flat32[s * n:(s + 1) * n, 0]) > 0) for s in range(100))
            if not keep:
                continue  # float rounding merged two x of one set: not a valid float input
            rep = H.build_hood(torch.as_tensor(flat32).cuda(), block_len=n)
            c, corners = rep.counts.cpu().numpy(), rep.corners.cpu().numpy()
            for s in range(100):
                want = O.upper_hull(flat32[s * n:(s + 1) * n])
                assert same(corners[s * n: s * n + c[s]], want), (n, s)
            continue
        rep = H.build_hood(torch.as_tensor(flat).cuda(), block_len=n)
        c, corners = rep.counts.cpu().numpy(), rep.corners.cpu().numpy()
        for s in range(100):
            want = hulls[off[s]:off[s + 1]]
            assert same(corners[s * n: s * n + c[s]], want), (n, s)
            if s % 10 == 0:
                assert same(gpu_hull(pts[s]), want), (n, s)


# ----------------------------- the reference's own harness through the drop-in

DROPIN = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_dropin")


def _run_bin(name, timeout=600):
    import subprocess
    path = os.path.join(DROPIN, name)
    if not os.path.exists(path):
        pytest.skip(f"{path} not built (oracle/dropin/build_dropin.py needs the reference tree)")
    r = subprocess.run([path], capture_output=True, text=True, timeout=timeout)
    return r.returncode, r.stdout + r.stderr


def test_reference_acceptance_through_dropin():
    """proj/tests/acceptance.cpp, unmodified, linked against driver.cpp with
    the HOOD_USE_B200 binding (oracle/dropin):
    criteria 1-3 run the 900-run sweep with an on_round_end observer, i.e.
    the reference round loop with every round merged on the GPU
    (hood_merge_round_host_f64); criterion 8 builds through hood_build_host.
    Every criterion must come out exactly as it does for the unpatched
    reference (acceptance_ref) -- criterion 4 is a psim-kernel property the
    reference itself fails (sample corners stepping left, test_kernel.cpp
    "tangent corners can step left"), untouched by the drop-in."""
    rc_ref, out_ref = _run_bin("acceptance_ref")
    rc, out = _run_bin("acceptance")

    def verdicts(text):
        return {ln.split(":")[0].split()[-1]: ln.split()[0] for ln in text.splitlines()
                if ln.startswith(("PASS criterion", "FAIL criterion"))}
    got, want = verdicts(out), verdicts(out_ref)
    assert set(got) == {str(i) for i in range(1, 9)}, out
    assert got == want, (out, out_ref)
    for c in ("1", "2", "3", "5", "6", "7", "8"):
        assert got[c] == "PASS", out
    assert "900 runs" in out and "0 mismatches" in out


@pytest.mark.parametrize("name", ["test_driver", "test_cli"])
def test_reference_unit_tests_through_dropin(name):
    """proj/tests/test_driver.cpp (build_hood with and without observers,
    round_metrics formulas) and test_cli.cpp (cli::run -> build_hood, trace
    observer) against the drop-in, with a minimal doctest stand-in."""
    rc, out = _run_bin(name)
    assert rc == 0 and "0 failed" in out, out


# ------------------------------------------------------------- tail stealing

def _steal_lib():
    import ctypes
    L = H.library()
    L.hood_internal_set_debug.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
    L.hood_internal_steals.restype = ctypes.c_longlong
    L.hood_internal_steals.argtypes = [ctypes.c_void_p]
    return L


@pytest.mark.parametrize("shape", ["gauss26", "arc25", "dent25", "multi"])
def test_tail_stealing_parity(oracle_mod, shape):
    """Work stealing of unit tails (the STEAL ring kernel): with every odd
    warp held back 300 us (debug mode 4) the others steal from those units
    (up to three times each), the parts of each stolen unit are merged left
    to right by bridge + splice, and the hood is still the oracle's, bit for
    bit -- single builds, multi-instance builds and the chunked host path."""
    L = _steal_lib()
    ctx = H.Context.get(0)
    rng = np.random.default_rng(7)
    block = 0
    if shape == "gauss26":
        p = W.gauss(1 << 26, seed=62)
    elif shape == "arc25":
        p = W.arc(1 << 25)
    elif shape == "dent25":  # an arc with random dents: survivors everywhere, merge trees, bridges
        p = W.arc(1 << 25)
        k = rng.choice(p.shape[0], size=1 << 16, replace=False)
        p[k, 1] -= rng.random(k.size) * 1e-3
    else:
        p = np.concatenate([W.gauss(1 << 24, seed=63 + i) for i in range(4)])
        block = 1 << 24
    t = torch.as_tensor(p).cuda()
    L.hood_internal_steals(ctx.handle)
    L.hood_internal_set_debug(ctx.handle, 4, None)
    try:
        rep = H.build_hood(t, block_len=block)
        steals = L.hood_internal_steals(ctx.handle)
        if block:
            c, corners = rep.counts.cpu().numpy(), rep.corners.cpu().numpy()
            for i in range(p.shape[0] // block):
                assert same(corners[i * block: i * block + c[i]], oracle_mod.upper_hull(p[i * block:(i + 1) * block])), i
        else:
            got = rep.hull.cpu().numpy()
            assert same(got, oracle_mod.upper_hull(p)), shape
            if shape == "gauss26":  # the chunked host path with steals
                out, cnt = H.build_hood_host(np.ascontiguousarray(p))
                assert same(out[: cnt[0]], got)
    finally:
        L.hood_internal_set_debug(ctx.handle, 0, None)
    assert steals > 0, shape
    if not block:
        # several steals per unit (up to kStealParts - 1 = 3): more steals than
        # delayed units (every odd warp of 3 CTAs x 4 warps per SM), so
        # merges of three and four parts ran too
        assert steals > torch.cuda.get_device_properties(0).multi_processor_count * 6, (shape, steals)
    # and the normal mode after it: the claim words of the slowed build
    # never leak into the next one
    assert same(H.build_hood(t, block_len=block).counts.cpu().numpy(), rep.counts.cpu().numpy())


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_dented_and_noisy_arcs(oracle_mod, dtype):
    """Arc-like inputs with imperfections: every block has many survivors but
    not a concave chain (the warp merge tree + bridge_warp), unit hoods of
    thousands of corners with non-convex seams (the finalize's range-based
    merge tree and its one compaction).  Bit-exact against the oracle."""
    rng = np.random.default_rng(11)
    for n, dents, depth in [(1 << 20, 1 << 12, 1e-4), (1 << 20, 1 << 18, 1e-6), (3 << 18, 1 << 10, 1e-2)]:
        p = W.arc(n)
        if dtype == torch.float32:
            p = p.astype(np.float32).astype(np.float64)
            keep = np.concatenate([[True], np.diff(p[:, 0]) > 0])
            p = p[keep]
        k = rng.choice(p.shape[0], size=min(dents, p.shape[0] // 2), replace=False)
        p[k, 1] -= rng.random(k.size) * depth
        if dtype == torch.float32:
            p = p.astype(np.float32)
        want = oracle_mod.upper_hull(p.astype(np.float64))
        assert same(gpu_hull(p, dtype=dtype).astype(np.float64), want), (n, dents, depth)
