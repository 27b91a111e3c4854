"""Python binding of libhood_b200.so (ctypes over the C-ABI in include/hood_b200.h).

Mirrors the reference's hot-path interface (/root/reference/proj/include/hood/
driver.hpp:16-48, oracle.hpp:23):

    build_hood(points, ...)   -> BuildReport(hull, counts, ...)   driver.cpp:19-45
    upper_hull(points)        -> compact corners                   oracle.cpp:7-20
    ValidationError(code, i)  hoodbuf.hpp:18-32 (x_not_increasing, x_out_of_range)

Points are CUDA tensors of shape (n, 2), float32 (float2 storage) or float64
(double2 storage), x strictly increasing.  There is no CPU fallback: without
the compiled library (python -m paper_1203_5004_b200.build) or without a GPU
every call raises.
"""
from __future__ import annotations

import ctypes
import os
import threading
from dataclasses import dataclass, field
from typing import Optional

PKG = os.path.dirname(os.path.abspath(__file__))
SO = os.environ.get("HOOD_B200_LIB") or os.path.join(PKG, "lib", "libhood_b200.so")  # override: experiments

HOOD_OK = 0
HOOD_ERR_INVALID_ARG = 1
HOOD_ERR_X_NOT_INCREASING = 2
HOOD_ERR_X_OUT_OF_RANGE = 3
HOOD_ERR_DEGENERATE = 4
HOOD_ERR_CUDA = 5
HOOD_ERR_CAPACITY = 6
HOOD_ERR_NOT_POWER_OF_TWO = 7
HOOD_ERR_PARSE = 8
HOOD_ERR_DEGENERATE_TRIPLE = 9
HOOD_FLAG_CHECK_RANGE = 0x1
HOOD_FLAG_CHECK_TRIPLES = 0x2

EXPORTS = [
    "hood_create", "hood_destroy", "hood_reserve", "hood_build_f32", "hood_build_f64",
    "hood_build_host_f32", "hood_build_host_f64", "hood_merge_segments_f32", "hood_merge_segments_f64",
    "hood_last_error", "hood_last_launch_count", "hood_status_string", "hood_abi_version",
    "hood_set_profile_events", "hood_merge_round_f32", "hood_merge_round_f64",
    "hood_parse_points", "hood_format_points", "hood_validate_points",
    "hood_format_section", "hood_format_trace_round", "hood_write_trace_f64",
    "hood_pack_record_f32", "hood_pack_record_f64", "hood_merge_records",
    "hood_build_multi_f32", "hood_build_multi_f64",
    "hood_merge_round_scratch_f32", "hood_merge_round_scratch_f64", "hood_merge_round_host_f64",
]


class HoodError(RuntimeError):
    def __init__(self, code: int, message: str, index: int = -1):
        super().__init__(message)
        self.code = code
        self.index = index


class ValidationError(HoodError):
    """hoodbuf.hpp:18-32; .code is x_not_increasing / x_out_of_range, .i the index."""

    @property
    def i(self):
        return self.index


class _Err(ctypes.Structure):
    _fields_ = [("code", ctypes.c_int32), ("cuda_error", ctypes.c_int32), ("index", ctypes.c_int64)]


_lib = None
_lock = threading.Lock()


def library():
    """Load libhood_b200.so; raises (never falls back) when it is missing."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(SO):
                raise ImportError(f"{SO} is not built: run `python -m paper_1203_5004_b200.build`")
            L = ctypes.CDLL(SO)
            p, i64, i32, u32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_uint32
            L.hood_create.argtypes = [ctypes.POINTER(p), ctypes.c_int]
            L.hood_destroy.argtypes = [p]
            L.hood_reserve.argtypes = [p, i64, i64, ctypes.c_int]
            for nm in ("hood_build_f32", "hood_build_f64"):
                getattr(L, nm).argtypes = [p, p, i64, i64, p, p, p, u32, p]
            for nm in ("hood_build_host_f32", "hood_build_host_f64"):
                getattr(L, nm).argtypes = [p, p, i64, i64, p, p, u32]
            for nm in ("hood_merge_segments_f32", "hood_merge_segments_f64"):
                getattr(L, nm).argtypes = [p, p, p, i64, i64, p, p, p]
            for nm in ("hood_merge_round_f32", "hood_merge_round_f64"):
                getattr(L, nm).argtypes = [p, p, i64, i64, p, p]
            for nm in ("hood_merge_round_scratch_f32", "hood_merge_round_scratch_f64"):
                getattr(L, nm).argtypes = [p, p, i64, i64, p, p, p]
            for nm in ("hood_pack_record_f32", "hood_pack_record_f64"):
                getattr(L, nm).argtypes = [p, p, p, i64, ctypes.c_double, p, p]
            L.hood_merge_records.argtypes = [p, p, i64, i64, p, p, p]
            L.hood_merge_round_host_f64.argtypes = [p, p, i64, i64, p]
            for nm in ("hood_build_multi_f32", "hood_build_multi_f64"):
                getattr(L, nm).argtypes = [p, ctypes.c_int, p, p, p, p, p, i64]
            L.hood_last_error.argtypes = [p, ctypes.POINTER(_Err)]
            L.hood_last_launch_count.argtypes = [p]
            L.hood_set_profile_events.argtypes = [p, p, p]
            L.hood_status_string.restype = ctypes.c_char_p
            L.hood_status_string.argtypes = [ctypes.c_int]
            for nm in EXPORTS:
                fn = getattr(L, nm)
                if nm != "hood_status_string":
                    fn.restype = ctypes.c_int
            _lib = L
    return _lib


class CapacityError(HoodError):
    """A multi-GPU exchange record was too small: .index is the capacity needed."""


def _raise(code: int, index: int = -1):
    msg = library().hood_status_string(code).decode()
    if code in (HOOD_ERR_X_NOT_INCREASING, HOOD_ERR_X_OUT_OF_RANGE, HOOD_ERR_NOT_POWER_OF_TWO,
                HOOD_ERR_DEGENERATE_TRIPLE):
        raise ValidationError(code, f"point {index}: {msg}", index)
    if code == HOOD_ERR_CAPACITY:
        raise CapacityError(code, f"{msg}: {index} slots needed", index)
    raise HoodError(code, msg, index)


class Context:
    """One hood_ctx per (device, host thread) (hood_create / hood_destroy).

    A context's workspace is reused by every build it runs, so contexts are
    never shared between threads (ctypes releases the GIL during the calls);
    the C-ABI orders a build on another stream than the context's last one
    after it (include/hood_b200.h)."""

    _per_key: dict = {}
    _key_lock = threading.Lock()

    def __init__(self, device: int = 0):
        L = library()
        h = ctypes.c_void_p()
        rc = L.hood_create(ctypes.byref(h), device)
        if rc:
            _raise(rc)
        self.handle = h
        self.device = device

    @classmethod
    def get(cls, device: int) -> "Context":
        key = (device, threading.get_ident())
        with cls._key_lock:
            c = cls._per_key.get(key)
            if c is None:
                c = cls._per_key[key] = Context(device)
        return c

    def __del__(self):
        try:
            if getattr(self, "handle", None) is not None and _lib is not None:
                _lib.hood_destroy(self.handle)
        except Exception:
            pass

    def last_error(self, raise_on_error: bool = True) -> int:
        e = _Err()
        rc = library().hood_last_error(self.handle, ctypes.byref(e))
        if rc and raise_on_error:
            _raise(rc, e.index)
        return rc

    def last_launch_count(self) -> int:
        return library().hood_last_launch_count(self.handle)

    def set_profile_events(self, before=None, after=None):
        """torch.cuda.Event pair recorded around the slab kernel of later builds."""
        library().hood_set_profile_events(self.handle, before.cuda_event if before is not None else None,
                                          after.cuda_event if after is not None else None)

    def reserve(self, n: int, block_len: int = 0, f64: bool = False):
        rc = library().hood_reserve(self.handle, n, block_len, int(f64))
        if rc:
            _raise(rc)


@dataclass
class BuildReport:
    """driver.hpp:37-41 -- hull (compact, left to right) per instance."""
    corners: object                      # (n, 2) slots, instance i at [i*L, i*L+counts[i])
    counts: object                       # (instances,) int32
    block_len: int
    padded: Optional[object] = None      # HoodBuffer layout (corners then REMOTE)
    conflicts: int = 0                   # always 0: no audited races on the GPU path
    metrics: dict = field(default_factory=dict)

    @property
    def hull(self):
        """Instance 0's corners (the reference BuildReport::hull)."""
        return self.corners[: int(self.counts[0])]

    def instance(self, i: int):
        L = self.block_len
        return self.corners[i * L: i * L + int(self.counts[i])]


def _check_points(points):
    import torch
    if not isinstance(points, torch.Tensor) or not points.is_cuda:
        raise TypeError("points must be a CUDA tensor of shape (n, 2)")
    if points.dim() != 2 or points.shape[1] != 2 or points.dtype not in (torch.float32, torch.float64):
        raise TypeError("points must be (n, 2) float32 or float64")
    if not points.is_contiguous():
        raise TypeError("points must be contiguous")


def _flags(check_range: bool, check_triples: bool) -> int:
    return (HOOD_FLAG_CHECK_RANGE if check_range else 0) | (HOOD_FLAG_CHECK_TRIPLES if check_triples else 0)


def build_hood_async(points, block_len: int = 0, corners=None, counts=None, padded=None,
                     check_range: bool = False, stream=None, check_triples: bool = False) -> BuildReport:
    """Enqueue a build on `stream` (default: torch's current stream); no sync."""
    import torch
    _check_points(points)
    n = points.shape[0]
    L = n if block_len in (0, None) else int(block_len)
    inst = max(n // L, 1)
    dev = points.device.index if points.device.index is not None else torch.cuda.current_device()
    ctx = Context.get(dev)
    if corners is None:
        corners = torch.empty_like(points)
    if counts is None:
        counts = torch.empty(inst, dtype=torch.int32, device=points.device)
    if stream is None:
        stream = torch.cuda.current_stream(points.device)
    fn = library().hood_build_f64 if points.dtype == torch.float64 else library().hood_build_f32
    rc = fn(ctx.handle, points.data_ptr(), n, L, corners.data_ptr(), counts.data_ptr(),
            padded.data_ptr() if padded is not None else None,
            _flags(check_range, check_triples), ctypes.c_void_p(stream.cuda_stream))
    if rc:
        _raise(rc)
    return BuildReport(corners=corners, counts=counts, block_len=L, padded=padded)


def build_hood(points, block_len: int = 0, padded: bool = False, check_range: bool = False,
               check_triples: bool = False) -> BuildReport:
    """driver.cpp:19-45 drop-in: build, synchronize, raise ValidationError on bad input
    (check_range / check_triples add validate_points' x-range and consecutive-triple
    margin checks, hoodbuf.cpp:30-60, fused into the build)."""
    import torch
    pad = torch.empty_like(points) if padded else None
    rep = build_hood_async(points, block_len, padded=pad, check_range=check_range, check_triples=check_triples)
    Context.get(points.device.index if points.device.index is not None else torch.cuda.current_device()).last_error()
    return rep


def upper_hull(points):
    """oracle.cpp:7-20 semantics on the GPU: compact corners of one instance."""
    rep = build_hood(points)
    return rep.hull


def build_hood_host(points_np, block_len: int = 0, check_range: bool = False, device: int = 0,
                    check_triples: bool = False):
    """Host buffers in / out through hood_build_host_* (the e2e path).
    Returns (corners ndarray (n,2), counts ndarray)."""
    import numpy as np
    a = points_np
    if not (isinstance(a, np.ndarray) and a.ndim == 2 and a.shape[1] == 2 and a.flags.c_contiguous):
        raise TypeError("points must be a C-contiguous (n, 2) ndarray")
    n = a.shape[0]
    L = n if block_len in (0, None) else int(block_len)
    out = np.empty_like(a)
    counts = np.zeros(max(n // L, 1), dtype=np.int32)
    ctx = Context.get(device)
    fn = library().hood_build_host_f64 if a.dtype == np.float64 else library().hood_build_host_f32
    rc = fn(ctx.handle, a.ctypes.data, n, L, out.ctypes.data, counts.ctypes.data,
            _flags(check_range, check_triples))
    if rc:
        e = _Err()
        library().hood_last_error(ctx.handle, ctypes.byref(e))
        _raise(rc, e.index)
    return out, counts


def build_hood_host_ptr(ctx: Context, host_ptr: int, n: int, f64: bool, out_ptr: int, counts_ptr: int,
                        block_len: int = 0) -> int:
    """Raw-pointer host build (pinned buffers owned by the caller); returns status."""
    fn = library().hood_build_host_f64 if f64 else library().hood_build_host_f32
    return fn(ctx.handle, host_ptr, n, n if block_len in (0, None) else block_len, out_ptr, counts_ptr, 0)


def merge_segments(seg_pts, seg_counts, out=None, out_count=None, stream=None):
    """Final merge of G adjacent slab hoods: seg_pts (G, stride, 2), seg_counts (G,) int32."""
    import torch
    G, stride = seg_pts.shape[0], seg_pts.shape[1]
    dev = seg_pts.device.index if seg_pts.device.index is not None else torch.cuda.current_device()
    ctx = Context.get(dev)
    if out is None:
        out = torch.empty(G * stride, 2, dtype=seg_pts.dtype, device=seg_pts.device)
    if out_count is None:
        out_count = torch.empty(1, dtype=torch.int32, device=seg_pts.device)
    if stream is None:
        stream = torch.cuda.current_stream(seg_pts.device)
    fn = library().hood_merge_segments_f64 if seg_pts.dtype == torch.float64 else library().hood_merge_segments_f32
    rc = fn(ctx.handle, seg_pts.contiguous().data_ptr(), seg_counts.contiguous().data_ptr(), G, stride,
            out.data_ptr(), out_count.data_ptr(), ctypes.c_void_p(stream.cuda_stream))
    if rc:
        _raise(rc)
    return out, out_count


def pack_record(corners, count, cap: int, x_offset: float = 0.0, rec=None, stream=None):
    """Exchange record of a slab hood (hood_pack_record_*): (cap + 1, 2) float64,
    row 0 = (count, 0), rows 1.. = corners with x + x_offset.  count is a
    device int32 tensor (no host sync: graph-capturable)."""
    import torch
    dev = corners.device.index if corners.device.index is not None else torch.cuda.current_device()
    ctx = Context.get(dev)
    if rec is None:
        rec = torch.zeros(cap + 1, 2, dtype=torch.float64, device=corners.device)
    if stream is None:
        stream = torch.cuda.current_stream(corners.device)
    fn = library().hood_pack_record_f64 if corners.dtype == torch.float64 else library().hood_pack_record_f32
    rc = fn(ctx.handle, corners.data_ptr(), count.data_ptr(), cap, float(x_offset), rec.data_ptr(),
            ctypes.c_void_p(stream.cuda_stream))
    if rc:
        _raise(rc)
    return rec


def merge_records(recs, out=None, out_count=None, stream=None):
    """Global hood from G gathered records (G, cap + 1, 2) float64 (hood_merge_records)."""
    import torch
    G, cap = recs.shape[0], recs.shape[1] - 1
    dev = recs.device.index if recs.device.index is not None else torch.cuda.current_device()
    ctx = Context.get(dev)
    if out is None:
        out = torch.empty(G * cap, 2, dtype=torch.float64, device=recs.device)
    if out_count is None:
        out_count = torch.empty(1, dtype=torch.int32, device=recs.device)
    if stream is None:
        stream = torch.cuda.current_stream(recs.device)
    rc = library().hood_merge_records(ctx.handle, recs.contiguous().data_ptr(), G, cap, out.data_ptr(),
                                      out_count.data_ptr(), ctypes.c_void_p(stream.cuda_stream))
    if rc:
        _raise(rc)
    return out, out_count


def build_multi(slabs, contexts=None, x_offsets=None, cap: int = 4096):
    """Single-process multi-GPU build (hood_build_multi_*): slab g is a CUDA
    tensor on its own device (contexts[g] defaults to that device's context);
    returns the global hood on slabs[0]'s device, float64."""
    import torch
    G = len(slabs)
    ctxs = contexts or [Context.get(t.device.index if t.device.index is not None else 0) for t in slabs]
    arr_ctx = (ctypes.c_void_p * G)(*[c.handle.value if hasattr(c.handle, "value") else c.handle for c in ctxs])
    arr_pts = (ctypes.c_void_p * G)(*[t.data_ptr() for t in slabs])
    arr_n = (ctypes.c_int64 * G)(*[t.shape[0] for t in slabs])
    offs = (ctypes.c_double * G)(*(x_offsets if x_offsets is not None else [0.0] * G))
    dev0 = slabs[0].device
    out = torch.empty(G * cap, 2, dtype=torch.float64, device=dev0)
    cnt = torch.empty(1, dtype=torch.int32, device=dev0)
    fn = library().hood_build_multi_f64 if slabs[0].dtype == torch.float64 else library().hood_build_multi_f32
    torch.cuda.synchronize(dev0)
    rc = fn(arr_ctx, G, arr_pts, arr_n, offs, out.data_ptr(), cnt.data_ptr(), cap)
    if rc:
        _raise(rc)
    return out[: int(cnt.item())]


def merge_round(slots, d: int, out=None, stream=None, scratch=None):
    """One reference round on the GPU (driver.cpp:20-43, kernel.cpp:155-161):
    slots (n, 2) in HoodBuffer layout with blocks of d -> blocks of 2d.
    scratch: optional (n,) int32 CUDA tensor that receives the pinpoint
    phase's pindex / qindex at every pair window's first two slots
    (kernel.cpp:101-112).  Asynchronous: ctx.last_error() (or
    merge_round_checked) reports a degenerate tangent."""
    import torch
    if not isinstance(slots, torch.Tensor) or not slots.is_cuda or slots.dim() != 2 or slots.shape[1] != 2:
        raise TypeError("slots must be a CUDA tensor of shape (n, 2)")
    slots = slots.contiguous()
    dev = slots.device.index if slots.device.index is not None else torch.cuda.current_device()
    ctx = Context.get(dev)
    if out is None:
        out = torch.empty_like(slots)
    if stream is None:
        stream = torch.cuda.current_stream(slots.device)
    if scratch is None:
        fn = library().hood_merge_round_f64 if slots.dtype == torch.float64 else library().hood_merge_round_f32
        rc = fn(ctx.handle, slots.data_ptr(), slots.shape[0], int(d), out.data_ptr(),
                ctypes.c_void_p(stream.cuda_stream))
    else:
        if scratch.dtype != torch.int32 or scratch.numel() < slots.shape[0] or not scratch.is_cuda:
            raise TypeError("scratch must be an int32 CUDA tensor of n entries")
        fn = (library().hood_merge_round_scratch_f64 if slots.dtype == torch.float64
              else library().hood_merge_round_scratch_f32)
        rc = fn(ctx.handle, slots.data_ptr(), slots.shape[0], int(d), out.data_ptr(), scratch.data_ptr(),
                ctypes.c_void_p(stream.cuda_stream))
    if rc:
        _raise(rc)
    return out


def match_and_merge_block(slots, d: int, scratch=None):
    """kernel.cpp:175-187 on the GPU: merge the pair windows of slots (blocks
    of d), synchronize, raise HoodError(HOOD_ERR_DEGENERATE) (.index = the
    block) where the reference throws DegenerateTangent."""
    import torch
    out = merge_round(slots, d, scratch=scratch)
    dev = slots.device.index if slots.device.index is not None else torch.cuda.current_device()
    Context.get(dev).last_error()
    return out


def round_schedule(n: int):
    """driver.cpp:5-17: (r, d1, d2, d) of the log2(n)-1 reference rounds."""
    rounds, d1, d2, r = [], 2, 1, 1
    d = d1 * d2
    while d < n:
        rounds.append((r, d1, d2, d))
        if d1 > d2:
            d2 *= 2
        else:
            d1 *= 2
        r += 1
        d = d1 * d2
    return rounds
