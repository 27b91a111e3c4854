"""Multi-rank slab sharding on CPU: world_size 2 and 4 over
gloo, the exchange protocol of paper_1203_5004_b200/distributed.py with the
device operations replaced by the oracle (the CUDA path is covered by the GPU
tests).  Checks the property the sharding relies on --
upper_hull(concat of slab hulls) == upper_hull(all points) -- through the real
record packing, all_gather, overflow re-exchange and merge."""
import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _slab(rank: int, n: int, arc: bool):
    from paper_1203_5004_b200 import workloads as W
    return W.arc(n) if arc else W.grid_uniform(n, seed=100 + rank)


def _global_slab(rank: int, world: int, n_global: int):
    """bench.py's split: rank's contiguous slab of ONE config-4-shaped set."""
    from paper_1203_5004_b200 import workloads as W
    from paper_1203_5004_b200.distributed import slab_range
    lo, hi = slab_range(n_global, world, rank)
    return W.gauss(n_global, seed=4)[lo:hi]


def _worker(rank, world, port, n, cap, arc, q, global_set=False):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import torch
    import torch.distributed as dist

    import oracle as O
    from paper_1203_5004_b200 import distributed as Dz

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        pts = _global_slab(rank, world, n) if global_set else _slab(rank, n, arc)

        def build_local(p):
            h = O.upper_hull(np.asarray(p, dtype=np.float64))
            return torch.from_numpy(h), len(h)

        def merge(segs, counts):
            cat = np.concatenate([segs[g, : int(counts[g])].numpy() for g in range(segs.shape[0])])
            return torch.from_numpy(O.upper_hull(cat))

        res = Dz.sharded_build(torch.from_numpy(pts), cap=cap, x_offset=0.0 if global_set else float(rank),
                               build_local=build_local, merge=merge)
        q.put((rank, res.hull.numpy(), res.slab_counts, res.exchanges))
    finally:
        dist.destroy_process_group()


def _run(world, n, cap, arc, global_set=False):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, n, cap, arc, q, global_set)) for r in range(world)]
    for p in ps:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    return sorted(out, key=lambda t: t[0])


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_uniform_matches_global_oracle(oracle_mod, world):
    n = 1 << 12
    out = _run(world, n, cap=4096, arc=False)
    full = np.concatenate([_slab(r, n, False).astype(np.float64) + np.array([r, 0.0]) for r in range(world)])
    want = oracle_mod.upper_hull(full)
    for rank, hull, counts, ex in out:
        assert ex == 1
        assert len(counts) == world
        np.testing.assert_array_equal(hull, want)


def test_sharded_overflow_takes_second_exchange(oracle_mod):
    # arc slabs: every point a corner, more than the record capacity
    world, n, cap = 2, 256, 64
    out = _run(world, n, cap=cap, arc=True)
    full = np.concatenate([_slab(r, n, True) + np.array([r, 0.0]) for r in range(world)])
    want = oracle_mod.upper_hull(full)
    for rank, hull, counts, ex in out:
        assert ex == 2
        assert max(counts) > cap
        np.testing.assert_array_equal(hull, want)


def test_pack_record_layout():
    import torch
    from paper_1203_5004_b200 import distributed as Dz
    h = torch.tensor([[0.25, 0.5], [0.5, 0.75]], dtype=torch.float32)
    rec = Dz.pack_record(h, 2, cap=4, x_offset=3.0)
    assert rec.shape == (5, 2) and rec.dtype == torch.float64
    assert rec[0, 0] == 2
    assert rec[1, 0] == 3.25 and rec[2, 1] == 0.75 and rec[3, 0] == 0


@pytest.mark.parametrize("world", [2, 4])
def test_bench_split_of_one_global_set(oracle_mod, world):
    """bench.py under torchrun: ONE global config-4-shaped set (Gaussian
    double2, x global) cut by slab_range into contiguous slabs, no x offset;
    every rank ends with the global set's hood."""
    from paper_1203_5004_b200 import workloads as W
    n = 1 << 14
    out = _run(world, n, cap=512, arc=False, global_set=True)
    want = oracle_mod.upper_hull(W.gauss(n, seed=4))
    for rank, hull, counts, ex in out:
        assert ex == 1 and len(counts) == world
        np.testing.assert_array_equal(hull, want)


def test_slab_range_partitions():
    from paper_1203_5004_b200.distributed import slab_range
    for n, world, block in [(1 << 28, 8, 0), (1 << 30, 8, 0), (1 << 28, 2, 0), (65536 * 1024, 4, 1024)]:
        rs = [slab_range(n, world, r, block) for r in range(world)]
        assert rs[0][0] == 0 and rs[-1][1] == n
        assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
        assert len({hi - lo for lo, hi in rs}) == 1
        if block:
            assert all(lo % block == 0 for lo, _ in rs)
    with pytest.raises(ValueError):
        slab_range(1000, 3, 0)
    with pytest.raises(ValueError):
        slab_range(1024 * 3, 2, 0, 1024)
