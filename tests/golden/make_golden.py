"""Generate the golden fixtures in tests/golden/ FROM THE REFERENCE ITSELF.

Run in the development container, where /root/reference exists:

    make -C oracle all ref && python tests/golden/make_golden.py

It loads oracle/_ref/libhoodref.so (the unmodified reference sources compiled
by oracle/Makefile, plus the extern "C" shim oracle/ref_shim.cpp) and records:

  acceptance.npz  acceptance.cpp:44-72 sweep (seed 0xACCE97 + s*1315423911 + n),
                  n = 4..1024, 8 seeds per size: the validated inputs, the
                  hood::build_hood hull, and (n <= 256) the REMOTE-padded buffer
                  after every round (on_round_end, acceptance criterion 2).
  driver.npz      test_driver.cpp:61-70 sets (seed 900 + 31*s + n).
  raw.npz         unvalidated uniform sets at n = 2^11..2^14 through the raw
                  reference round loop (driver.cpp:20-43 steps), plus the
                  reference upper_hull of the config generators at small n
                  (grid 2^16, arc 2^14, gauss 2^16, batched 64 x 1024).
  io.npz          the reference front end on fixed texts and arrays:
                  cli::parse_points (+ validate_points) outcomes, format_coord
                  strings, validate_points codes (cli.cpp:62-106,
                  hoodbuf.cpp:30-70), incl. tests/data/sample8.txt.
  trace.npz       the reference's own `hull` run (cli::run through
                  oracle/_ref/hood_ref_run) with a trace file: the run output
                  (points / hood sections) and the per-round trace
                  (cli.cpp:108-118, 144-190) for sample8.txt and random sets.
  pairs.npz       make_random_hood_pair(d, 0xC4C5 + t) windows (acceptance.cpp:79)
                  with the reference classify_g / classify_f tables and the
                  merged block of match_and_merge_block (test_kernel.cpp:302-328).

The fixtures are small (< 2 MB) and committed; the GPU box never needs the
reference tree.
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import oracle as O  # noqa: E402
from paper_1203_5004_b200 import workloads as W  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def acceptance():
    data = {}
    for n in [4, 8, 16, 32, 64, 128, 256, 512, 1024]:
        pts, hulls, counts, rounds = [], [], [], []
        for s in range(8):
            seed = 0xACCE97 + s * 1315423911 + n
            p = O.ref_make_random_point_set(n, seed)
            h, rb = O.ref_build_hood(p, rounds=(n <= 256))
            pad = np.zeros((n, 2))
            pad[:, 0] = 10.0
            pad[: len(h)] = h
            pts.append(p)
            hulls.append(pad)
            counts.append(len(h))
            if rb is not None:
                rounds.append(rb)
        data[f"pts_{n}"] = np.stack(pts)
        data[f"hull_{n}"] = np.stack(hulls)
        data[f"count_{n}"] = np.array(counts, dtype=np.int32)
        if rounds:
            data[f"rounds_{n}"] = np.stack(rounds)
        # the whole sweep: all 100 seeds (acceptance.cpp:43-47 kSeedsPerSize),
        # inputs + build_hood's hull (compact, concatenated)
        p100, h100, c100 = [], [], []
        for s in range(100):
            seed = 0xACCE97 + s * 1315423911 + n
            p = O.ref_make_random_point_set(n, seed)
            h, _ = O.ref_build_hood(p)
            assert np.array_equal(h, O.ref_upper_hull(p))  # criterion 1 on the reference itself
            p100.append(p)
            h100.append(h)
            c100.append(len(h))
        data[f"pts100_{n}"] = np.stack(p100)
        data[f"hulls100_{n}"] = np.concatenate(h100)
        data[f"count100_{n}"] = np.array(c100, dtype=np.int32)
    np.savez_compressed(os.path.join(OUT, "acceptance.npz"), **data)


def driver():
    data = {}
    for n in [4, 8, 32, 128, 256]:
        pts, hulls, counts = [], [], []
        for s in range(8):
            p = O.ref_make_random_point_set(n, 900 + 31 * s + n)
            h, _ = O.ref_build_hood(p)
            pad = np.zeros((n, 2))
            pad[:, 0] = 10.0
            pad[: len(h)] = h
            pts.append(p)
            hulls.append(pad)
            counts.append(len(h))
        data[f"pts_{n}"] = np.stack(pts)
        data[f"hull_{n}"] = np.stack(hulls)
        data[f"count_{n}"] = np.array(counts, dtype=np.int32)
    np.savez_compressed(os.path.join(OUT, "driver.npz"), **data)


def raw():
    data = {}
    rng = np.random.default_rng(20260)
    for e in [11, 12, 13, 14]:
        n = 1 << e
        x = np.sort(rng.random(n))
        assert np.all(np.diff(x) > 0)
        p = np.stack([x, rng.random(n)], axis=1)
        data[f"uniform_pts_{n}"] = p
        data[f"uniform_hull_{n}"] = O.ref_build_hood_raw(p)
        assert np.array_equal(data[f"uniform_hull_{n}"], O.ref_upper_hull(p))
    # Reference upper_hull of the config generators (inputs are regenerated
    # by the tests from (n, seed); only the hulls are stored).
    g = W.grid_uniform(1 << 16, seed=1)
    data["grid65536_hull"] = O.ref_upper_hull(g.astype(np.float64))
    a = W.arc(1 << 14)
    data["arc16384_count"] = np.array([len(O.ref_upper_hull(a))])
    gs = W.gauss(1 << 16, seed=4)
    data["gauss65536_hull"] = O.ref_upper_hull(gs)
    b = W.batched(64, 1024, seed=5)
    bo, bc = O.ref_block_hulls(b.astype(np.float64), 1024)
    data["batched64_counts"] = bc
    data["batched64_slots"] = np.concatenate([bo[i * 1024: i * 1024 + bc[i]] for i in range(64)])
    np.savez_compressed(os.path.join(OUT, "raw.npz"), **data)


def pairs():
    sizes = [2, 4, 8, 16, 32, 64]
    slots, pq, g_tab, f_tab, merged, scratch01 = [], [], [], [], [], []
    for t in range(120):
        d = sizes[t % 6]
        s, pc, qc = O.ref_make_random_hood_pair(d, 0xC4C5 + t)
        w = np.zeros((128, 2))
        w[:, 0] = 10.0
        w[: 2 * d] = s
        gt = np.full((64, 64), 9, dtype=np.int8)
        ft = np.full((64, 64), 9, dtype=np.int8)
        for i in range(pc):
            for j in range(d, 2 * d):
                gt[i, j - d] = O.ref().ref_classify_g(O._ptr(np.ascontiguousarray(s)), 2 * d, i, j, 0, d)
        for j in range(qc):
            for i in range(d):
                ft[i, j] = O.ref().ref_classify_f(O._ptr(np.ascontiguousarray(s)), 2 * d, i, d + j, 0, d)
        d1 = 1 << ((int(np.log2(d)) + 1) // 2)
        d2 = d // d1
        nh, sc = O.ref_merge_block(s, d1, d2)
        m = np.zeros((128, 2))
        m[:, 0] = 10.0
        m[: 2 * d] = nh
        slots.append(w)
        pq.append((d, pc, qc))
        g_tab.append(gt)
        f_tab.append(ft)
        merged.append(m)
        scratch01.append(sc[:2])
    np.savez_compressed(os.path.join(OUT, "pairs.npz"), slots=np.stack(slots), pq=np.array(pq, dtype=np.int32),
                        g=np.stack(g_tab), f=np.stack(f_tab), merged=np.stack(merged),
                        scratch01=np.stack(scratch01))


IO_TEXTS = [
    b"4\n0.1 0.5 # A\n0.2 0.6\n0.6 0.9\n0.7 0.2\n",            # E1, test_kernel.cpp:17-117
    b"# comment only line\n2\n0.25 0.1\n0.75 0.9\n",
    b"2 0.25 0.1 0.75 0.9",                                       # one line
    b"3\n0.1 0.2\n0.3",                                           # truncated
    b"2\n0.1 0.2\n0.3 0.4\n5\n",                                  # trailing input
    b"x\n",                                                       # bad count
    b"-1\n",                                                      # negative count
    b"2\n0.1 abc\n0.3 0.4\n",                                     # bad number
    b"99999999999\n",                                             # count out of range
    b"",                                                          # empty
    b"3\n0.1 0.2\n0.2 0.3\n0.3 0.5\n",                            # not a power of two
    b"4\n0.1 0.1\n0.2 0.2\n0.3 0.3\n0.4 0.5\n",                    # collinear triple
    b"4\n0.1 0.5\n0.1 0.6\n0.6 0.9\n0.7 0.2\n",                    # x not increasing
    b"4\n0 0.5\n0.2 0.6\n0.6 0.9\n0.7 0.2\n",                      # x out of range
    b"2\n1e-3 .5e0\n0x1p-1 0.25\n",                                # strtod forms
]


def io():
    texts = list(IO_TEXTS)
    sample = os.path.join(O.REF_ROOT, "tests", "data", "sample8.txt") if hasattr(O, "REF_ROOT") else \
        "/root/reference/proj/tests/data/sample8.txt"
    with open(sample, "rb") as f:
        texts.append(f.read())
    rng = np.random.default_rng(5)
    for n in (64, 128, 1024):
        p = O.ref_make_random_point_set(n, 77 + n)
        texts.append(O.ref_format_points(p))
        bad = p.copy()
        bad[n // 2, 0] = bad[n // 2 - 1, 0]  # x not increasing
        texts.append(O.ref_format_points(bad))
    kinds, lines, codes, ijks, pts = [], [], [], [], []
    for t in texts:
        r = O.ref_parse_points(t)
        kinds.append({"ok": 0, "parse": 1, "validation": 2}[r[0]])
        lines.append(r[1] if r[0] == "parse" else -1)
        codes.append(r[1] if r[0] == "validation" else -1)
        ijks.append(r[2] if r[0] == "validation" else (-1, -1, -1))
        pts.append(r[1] if r[0] == "ok" else np.zeros((0, 2)))
    # format_coord on awkward doubles
    vals = np.array([0.1, 0.5, 1.0 / 3.0, 2.0 ** -24, 1e-300, 123456789.125, 0.0, -0.0, 5e-324,
                     np.nextafter(1.0, 0.0)] + list(rng.random(50)), dtype=np.float64)
    coords = [O.ref_format_coord(v) for v in vals]
    # validate_points codes on random sets with planted defects
    varr, vres = [], []
    for t in range(24):
        n = [4, 8, 64, 128, 256][t % 5]
        p = O.ref_make_random_point_set(n, 900 + t)
        if t % 4 == 1:
            i = 1 + (t % (n - 2))
            p[i, 1] = p[i - 1, 1] + (p[i + 1, 1] - p[i - 1, 1]) * (p[i, 0] - p[i - 1, 0]) / (p[i + 1, 0] - p[i - 1, 0])
        elif t % 4 == 2:
            p[n // 2, 0] = p[n // 2 - 1, 0]
        elif t % 4 == 3:
            p = p[:-1]
        r = O.ref_validate_points(p)
        varr.append(np.concatenate([p, np.zeros((256 - len(p), 2))]))
        vres.append((len(p), -1, -1, -1, -1) if r == -1 else (len(p), r[0], *r[1]))
    def blob(items):
        off = np.cumsum([0] + [len(x) for x in items])
        return np.frombuffer(b"".join(items), dtype=np.uint8), off
    tb, to = blob(texts)
    cb, co = blob(coords)
    pcat = np.concatenate([p.reshape(-1, 2) for p in pts]) if pts else np.zeros((0, 2))
    poff = np.cumsum([0] + [len(p) for p in pts])
    np.savez_compressed(os.path.join(OUT, "io.npz"), text_blob=tb, text_off=to, kinds=np.array(kinds),
                        lines=np.array(lines), codes=np.array(codes), ijks=np.array(ijks), pts=pcat,
                        pts_off=poff, coord_vals=vals, coord_blob=cb, coord_off=co,
                        varr=np.stack(varr), vres=np.array(vres))


def trace():
    import subprocess
    import tempfile
    runner = os.path.join(ROOT, "oracle", "_ref", "hood_ref_run")
    sample = "/root/reference/proj/tests/data/sample8.txt"
    inputs = []
    with open(sample, "rb") as f:
        inputs.append(f.read())
    for n in (2, 4, 8, 16, 32, 64, 128, 256, 1024):
        for s in range(2):
            inputs.append(O.ref_format_points(O.ref_make_random_point_set(n, 4242 + 17 * s + n)))
    pts, outs, traces = [], [], []
    with tempfile.TemporaryDirectory() as td:
        for k, text in enumerate(inputs):
            src, tr = os.path.join(td, f"p{k}.txt"), os.path.join(td, f"p{k}.trace")
            with open(src, "wb") as f:
                f.write(text)
            r = subprocess.run([runner, src, tr], capture_output=True, check=True)
            outs.append(r.stdout)
            with open(tr, "rb") as f:
                traces.append(f.read())
            pts.append(O.ref_parse_points(text)[1])

    def blob(items):
        off = np.cumsum([0] + [len(x) for x in items])
        return np.frombuffer(b"".join(items), dtype=np.uint8), off
    ob, oo = blob(outs)
    tb, to = blob(traces)
    np.savez_compressed(os.path.join(OUT, "trace.npz"), pts=np.concatenate(pts),
                        pts_off=np.cumsum([0] + [len(p) for p in pts]), out_blob=ob, out_off=oo,
                        trace_blob=tb, trace_off=to)


if __name__ == "__main__":
    O.build(ref=True)
    acceptance()
    driver()
    raw()
    pairs()
    io()
    trace()
    for f in sorted(os.listdir(OUT)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(OUT, f)))
