"""TEST INFRASTRUCTURE ONLY -- ctypes loader for the parity oracle.

Two CPU libraries, both checkers, never the product:
  * ``_build/libhood_oracle.so`` -- the C restatement in hood_oracle.c
    (always buildable: plain gcc, no reference tree needed);
  * ``_ref/libhoodref.so`` -- the UNMODIFIED reference sources under
    /root/reference/proj/src compiled by ``make ref`` plus ref_shim.cpp.  It is
    built in the development container (where /root/reference exists) and
    travels to the GPU box as a prebuilt file; everything that uses it skips
    when it is absent.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline / --impl
reference) import this module.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libhood_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libhoodref.so")
REF_SRC = "/root/reference/proj"

_lock = threading.Lock()
_oracle = None
_ref = None

_i64 = ctypes.c_int64
_i32 = ctypes.c_int32
_p = ctypes.c_void_p


def build(ref: bool = True) -> None:
    """Compile the oracle (and, when the reference tree is present, oracle/_ref)."""
    subprocess.run(["make", "-s", "-C", HERE, "all"], check=True)
    if ref and os.path.isdir(REF_SRC):
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def lib():
    global _oracle
    with _lock:
        if _oracle is None:
            if not os.path.exists(ORACLE_SO):
                build(ref=False)
            L = ctypes.CDLL(ORACLE_SO)
            for name in ("oracle_upper_hull_f64", "oracle_upper_hull_f32"):
                getattr(L, name).restype = _i64
                getattr(L, name).argtypes = [_p, _i64, _p]
            for name in ("oracle_upper_hull_mt_f64", "oracle_upper_hull_mt_f32"):
                getattr(L, name).restype = _i64
                getattr(L, name).argtypes = [_p, _i64, ctypes.c_int, _p]
            for name in ("oracle_block_hulls_f64", "oracle_block_hulls_f32"):
                getattr(L, name).restype = None
                getattr(L, name).argtypes = [_p, _i64, _i64, _p, _p, ctypes.c_int]
            L.oracle_orient.restype = ctypes.c_double
            L.oracle_orient.argtypes = [_p, _p, _p]
            L.oracle_brute_tangent_to_right.restype = _i64
            L.oracle_brute_tangent_to_right.argtypes = [_p, _p, _i64]
            L.oracle_brute_common_tangent.restype = ctypes.c_int
            L.oracle_brute_common_tangent.argtypes = [_p, _i64, _p, _i64, _p, _p]
            for name in ("oracle_classify_g", "oracle_classify_f"):
                getattr(L, name).restype = ctypes.c_int
                getattr(L, name).argtypes = [_p] + [ctypes.c_int] * 4
            L.oracle_round_schedule.restype = ctypes.c_int
            L.oracle_round_schedule.argtypes = [ctypes.c_int, _p, ctypes.c_int]
            L.oracle_validate_points.restype = ctypes.c_int
            L.oracle_validate_points.argtypes = [_p, _i64, _p]
            _oracle = L
    return _oracle


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref():
    """The compiled reference (oracle/_ref).  Raises if it was never built."""
    global _ref
    with _lock:
        if _ref is None:
            if not os.path.exists(REF_SO):
                raise FileNotFoundError(f"{REF_SO} not built (make -C oracle ref)")
            L = ctypes.CDLL(REF_SO)
            L.ref_upper_hull.restype = _i64
            L.ref_upper_hull.argtypes = [_p, _i64, _p]
            L.ref_upper_hull_mt.restype = _i64
            L.ref_upper_hull_mt.argtypes = [_p, _i64, ctypes.c_int, _p]
            L.ref_block_hulls_mt.restype = None
            L.ref_block_hulls_mt.argtypes = [_p, _i64, _i64, ctypes.c_int, _p, _p]
            L.ref_make_random_point_set.restype = ctypes.c_int
            L.ref_make_random_point_set.argtypes = [ctypes.c_int, ctypes.c_uint64, _p]
            L.ref_build_hood.restype = _i64
            L.ref_build_hood.argtypes = [_p, _i64, _p, _p, _p]
            L.ref_build_hood_raw.restype = _i64
            L.ref_build_hood_raw.argtypes = [_p, _i64, _p]
            L.ref_merge_block.restype = ctypes.c_int
            L.ref_merge_block.argtypes = [_p, ctypes.c_int, ctypes.c_int, _p, _p]
            L.ref_make_random_hood_pair.restype = ctypes.c_int
            L.ref_make_random_hood_pair.argtypes = [ctypes.c_int, ctypes.c_uint64, _p, _p]
            if hasattr(L, "ref_parse_points"):
                L.ref_parse_points.restype = ctypes.c_int
                L.ref_parse_points.argtypes = [ctypes.c_char_p, _i64, _p, _i64, _p, _p, _p]
                L.ref_validate_points.restype = ctypes.c_int
                L.ref_validate_points.argtypes = [_p, _i64, _p]
                L.ref_format_coord.restype = ctypes.c_int
                L.ref_format_coord.argtypes = [ctypes.c_double, ctypes.c_char_p, ctypes.c_int]
            for name in ("ref_classify_g", "ref_classify_f"):
                getattr(L, name).restype = ctypes.c_int
                getattr(L, name).argtypes = [_p, _i64] + [ctypes.c_int] * 4
            _ref = L
    return _ref


# ---------------------------------------------------------------- helpers

def _as_pts(points: np.ndarray) -> np.ndarray:
    a = np.ascontiguousarray(points)
    assert a.ndim == 2 and a.shape[1] == 2 and a.dtype in (np.float32, np.float64)
    return a


def upper_hull(points: np.ndarray, threads: int = 1) -> np.ndarray:
    """oracle.cpp:7-20 on an (n, 2) float32/float64 array; corners keep dtype."""
    a = _as_pts(points)
    out = np.empty_like(a)
    L = lib()
    f32 = a.dtype == np.float32
    if threads > 1:
        fn = L.oracle_upper_hull_mt_f32 if f32 else L.oracle_upper_hull_mt_f64
        h = fn(_ptr(a), a.shape[0], threads, _ptr(out))
    else:
        fn = L.oracle_upper_hull_f32 if f32 else L.oracle_upper_hull_f64
        h = fn(_ptr(a), a.shape[0], _ptr(out))
    return out[:h].copy()


def block_hulls(points: np.ndarray, block: int, pad_remote: bool = False):
    """Hull of every consecutive block; returns (slots (n,2), counts)."""
    a = _as_pts(points)
    n = a.shape[0]
    out = np.zeros_like(a)
    counts = np.zeros((n + block - 1) // block, dtype=np.int32)
    fn = lib().oracle_block_hulls_f32 if a.dtype == np.float32 else lib().oracle_block_hulls_f64
    fn(_ptr(a), n, block, _ptr(out), _ptr(counts), int(pad_remote))
    return out, counts


def orient(r, p, q) -> float:
    r, p, q = (np.ascontiguousarray(v, dtype=np.float64) for v in (r, p, q))
    return lib().oracle_orient(_ptr(r), _ptr(p), _ptr(q))


def brute_tangent_to_right(p, hull) -> int:
    p = np.ascontiguousarray(p, dtype=np.float64)
    h = np.ascontiguousarray(hull, dtype=np.float64)
    return lib().oracle_brute_tangent_to_right(_ptr(p), _ptr(h), h.shape[0])


def brute_common_tangent(p, q):
    p = np.ascontiguousarray(p, dtype=np.float64)
    q = np.ascontiguousarray(q, dtype=np.float64)
    a = np.zeros(1, np.int64)
    b = np.zeros(1, np.int64)
    rc = lib().oracle_brute_common_tangent(_ptr(p), p.shape[0], _ptr(q), q.shape[0], _ptr(a), _ptr(b))
    if rc != 0:
        raise ValueError("common tangent is not unique")
    return int(a[0]), int(b[0])


def classify_g(hood, i, j, start, d) -> int:
    h = np.ascontiguousarray(hood, dtype=np.float64)
    return lib().oracle_classify_g(_ptr(h), i, j, start, d)


def classify_f(hood, i, j, start, d) -> int:
    h = np.ascontiguousarray(hood, dtype=np.float64)
    return lib().oracle_classify_f(_ptr(h), i, j, start, d)


def round_schedule(n: int):
    buf = np.zeros((64, 4), dtype=np.int32)
    c = lib().oracle_round_schedule(n, _ptr(buf), 64)
    return [tuple(int(v) for v in row) for row in buf[:c]]


def validate_points(points):
    a = np.ascontiguousarray(points, dtype=np.float64)
    bad = np.zeros(1, np.int64)
    code = lib().oracle_validate_points(_ptr(a), a.shape[0], _ptr(bad))
    return code, int(bad[0])


# ------------------------------------------------- reference (oracle/_ref)

def ref_upper_hull(points: np.ndarray, threads: int = 1) -> np.ndarray:
    a = np.ascontiguousarray(points, dtype=np.float64)
    out = np.empty_like(a)
    if threads > 1:
        h = ref().ref_upper_hull_mt(_ptr(a), a.shape[0], threads, _ptr(out))
    else:
        h = ref().ref_upper_hull(_ptr(a), a.shape[0], _ptr(out))
    return out[:h].copy()


def ref_block_hulls(points: np.ndarray, block: int, threads: int = 1):
    a = np.ascontiguousarray(points, dtype=np.float64)
    n = a.shape[0]
    out = np.zeros_like(a)
    counts = np.zeros((n + block - 1) // block, dtype=np.int32)
    ref().ref_block_hulls_mt(_ptr(a), n, block, threads, _ptr(out), _ptr(counts))
    return out, counts


def ref_make_random_point_set(n: int, seed: int) -> np.ndarray:
    out = np.zeros((n, 2), dtype=np.float64)
    if ref().ref_make_random_point_set(n, seed, _ptr(out)) != 0:
        raise RuntimeError("could not draw a valid point set")
    return out


def ref_build_hood(points: np.ndarray, rounds: bool = False):
    """hood::build_hood on a validated PointSet -> (hull, per-round slots | None)."""
    a = np.ascontiguousarray(points, dtype=np.float64)
    n = a.shape[0]
    out = np.empty_like(a)
    nr = max(int(np.log2(n)) - 1, 0)
    rbuf = np.zeros((nr, n, 2), dtype=np.float64) if rounds and nr else None
    conf = np.zeros(1, np.int64)
    h = ref().ref_build_hood(_ptr(a), n, _ptr(out), _ptr(rbuf) if rbuf is not None else None, _ptr(conf))
    if h < 0:
        raise RuntimeError({-1: "ValidationError", -2: "DegenerateTangent"}.get(h, "error"))
    return out[:h].copy(), rbuf


def ref_build_hood_raw(points: np.ndarray) -> np.ndarray:
    a = np.ascontiguousarray(points, dtype=np.float64)
    out = np.empty_like(a)
    h = ref().ref_build_hood_raw(_ptr(a), a.shape[0], _ptr(out))
    if h < 0:
        raise RuntimeError({-2: "DegenerateTangent"}.get(h, "error"))
    return out[:h].copy()


def ref_merge_block(slots: np.ndarray, d1: int, d2: int):
    a = np.ascontiguousarray(slots, dtype=np.float64)
    n = a.shape[0]
    newhood = np.zeros_like(a)
    scratch = np.zeros(n, dtype=np.int32)
    rc = ref().ref_merge_block(_ptr(a), d1, d2, _ptr(newhood), _ptr(scratch))
    if rc != 0:
        raise RuntimeError({-2: "DegenerateTangent"}.get(rc, "error"))
    return newhood, scratch


def ref_make_random_hood_pair(d: int, seed: int):
    slots = np.zeros((2 * d, 2), dtype=np.float64)
    pq = np.zeros(2, dtype=np.int32)
    if ref().ref_make_random_hood_pair(d, seed, _ptr(slots), _ptr(pq)) != 0:
        raise RuntimeError("could not draw a valid hood pair")
    return slots, int(pq[0]), int(pq[1])


# ---- reference front end (cli.cpp / hoodbuf.cpp via oracle/_ref) ----------

def ref_parse_points(text: bytes):
    """cli.cpp parse_points (+ validate_points): ('ok', pts) | ('parse', line) |
    ('validation', code, (i, j, k))."""
    L = ref()
    cnt, line = ctypes.c_int64(0), ctypes.c_int64(0)
    ijk = (ctypes.c_int64 * 3)()
    cap = 1 << 16
    out = np.empty((cap, 2))
    rc = L.ref_parse_points(text, len(text), _ptr(out), cap, ctypes.byref(cnt), ctypes.byref(line), ijk)
    if rc == 3:
        out = np.empty((int(cnt.value), 2))
        rc = L.ref_parse_points(text, len(text), _ptr(out), out.shape[0], ctypes.byref(cnt), ctypes.byref(line), ijk)
    if rc == 0:
        return ("ok", out[: int(cnt.value)].copy())
    if rc == 1:
        return ("parse", int(line.value))
    return ("validation", int(line.value), (int(ijk[0]), int(ijk[1]), int(ijk[2])))


def ref_validate_points(points):
    """hoodbuf.cpp validate_points: -1 ok, else (code, (i, j, k))."""
    a = np.ascontiguousarray(points, dtype=np.float64)
    ijk = (ctypes.c_int64 * 3)()
    c = ref().ref_validate_points(_ptr(a), a.shape[0], ijk)
    return -1 if c < 0 else (c, (int(ijk[0]), int(ijk[1]), int(ijk[2])))


def ref_format_coord(v: float) -> bytes:
    buf = ctypes.create_string_buffer(64)
    n = ref().ref_format_coord(float(v), buf, 64)
    return buf.raw[:n]


def ref_format_points(points) -> bytes:
    """write_point_set's layout (cli.cpp:101-106) over the reference's format_coord."""
    a = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 2)
    return (str(a.shape[0]) + "\n").encode() + b"".join(
        ref_format_coord(x) + b" " + ref_format_coord(y) + b"\n" for x, y in a)
