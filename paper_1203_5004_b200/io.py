"""Point files and input validation (host side of the C-ABI, no GPU needed).

The reference's front end, restated natively in csrc/hood_host.cpp:
    parse_points(text)      cli.cpp:62-99  -> (n, 2) float64, raises ParseError
    read_points(path)       cli.cpp:56-60  (parse + validate_points)
    validate_points(points) hoodbuf.cpp:30-70 -> raises ValidationError
    format_points(points)   cli.cpp:101-106 write_point_set ("%.17g")
    write_point_set(path, points)
    format_section(label, points)      cli.cpp:47-52 (the run output's sections)
    format_run_output(points, hull)    cli.cpp:147, 183-184 ("points", "hood")
    format_trace_round(slots, d)       cli.cpp:108-118 write_trace_round
    write_trace(path, points)          the trace of build_hood (cli.cpp:163-169),
                                       the round loop run on the GPU
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import hood as H


class ParseError(ValueError):
    """cli.hpp ParseError: where:line: message."""

    def __init__(self, where: str, line: int, message: str = "parse error"):
        super().__init__(f"{where}:{line}: {message}")
        self.line = line


_VCODES = {H.HOOD_ERR_NOT_POWER_OF_TWO: "not_power_of_two", H.HOOD_ERR_X_OUT_OF_RANGE: "x_out_of_range",
           H.HOOD_ERR_X_NOT_INCREASING: "x_not_increasing", H.HOOD_ERR_DEGENERATE_TRIPLE: "degenerate_triple"}


def _lib():
    L = H.library()
    if not getattr(L, "_io_bound", False):
        p, i64 = ctypes.c_void_p, ctypes.c_int64
        L.hood_parse_points.argtypes = [p, i64, p, i64, ctypes.POINTER(i64), ctypes.POINTER(i64)]
        L.hood_format_points.argtypes = [p, i64, p, i64]
        L.hood_format_points.restype = i64
        L.hood_validate_points.argtypes = [p, i64, ctypes.POINTER(i64 * 3)]
        L.hood_format_section.argtypes = [ctypes.c_char_p, p, i64, p, i64]
        L.hood_format_section.restype = i64
        L.hood_format_trace_round.argtypes = [p, i64, i64, p, i64]
        L.hood_format_trace_round.restype = i64
        L.hood_write_trace_f64.argtypes = [p, p, i64, ctypes.c_char_p]
        L._io_bound = True
    return L


def parse_points(text, where: str = "<stream>") -> np.ndarray:
    """Raw points of a point file (no validation)."""
    data = text.encode() if isinstance(text, str) else bytes(text)
    L = _lib()
    count, line = ctypes.c_int64(0), ctypes.c_int64(0)
    rc = L.hood_parse_points(data, len(data), None, 0, ctypes.byref(count), ctypes.byref(line))
    if rc == H.HOOD_ERR_PARSE:
        raise ParseError(where, int(line.value))
    if rc not in (H.HOOD_OK, H.HOOD_ERR_CAPACITY):
        H._raise(rc)
    out = np.empty((int(count.value), 2), dtype=np.float64)
    rc = L.hood_parse_points(data, len(data), out.ctypes.data if out.size else None, out.shape[0],
                             ctypes.byref(count), ctypes.byref(line))
    if rc == H.HOOD_ERR_PARSE:
        raise ParseError(where, int(line.value))
    if rc:
        H._raise(rc)
    return out


def validate_points(points) -> np.ndarray:
    """hoodbuf.cpp:30-70; returns the points, raises hood.ValidationError."""
    a = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 2)
    ijk = (ctypes.c_int64 * 3)()
    rc = _lib().hood_validate_points(a.ctypes.data if a.size else None, a.shape[0], ctypes.byref(ijk))
    if rc:
        kind = _VCODES.get(rc, str(rc))
        e = H.ValidationError(rc, f"{kind} at point {int(ijk[0])}", int(ijk[0]))
        e.kind = kind
        e.ijk = (int(ijk[0]), int(ijk[1]), int(ijk[2]))
        raise e
    return a


def read_points(path: str) -> np.ndarray:
    with open(path, "rb") as f:
        return validate_points(parse_points(f.read(), path))


def format_points(points) -> str:
    a = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 2)
    L = _lib()
    n = L.hood_format_points(a.ctypes.data if a.size else None, a.shape[0], None, 0)
    buf = ctypes.create_string_buffer(int(n))
    L.hood_format_points(a.ctypes.data if a.size else None, a.shape[0], buf, n)
    return buf.raw[:n].decode()


def write_point_set(path: str, points) -> None:
    with open(path, "w") as f:
        f.write(format_points(points))


def _text(fn, *args) -> str:
    n = fn(*args, None, 0)
    if n < 0:
        raise ValueError("invalid arguments")
    buf = ctypes.create_string_buffer(int(n))
    fn(*args, buf, n)
    return buf.raw[:n].decode()


def format_section(label: str, points) -> str:
    """write_section (cli.cpp:47-52): "<label> <n>" then one line per point."""
    a = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 2)
    return _text(_lib().hood_format_section, label.encode(), a.ctypes.data if a.size else None, a.shape[0])


def format_run_output(points, hull, conflicts: int = 0) -> str:
    """The run output grammar (cli.cpp:147, 183-184): the points section, an
    optional "# conflicts" comment, then the hood section."""
    out = format_section("points", points)
    if conflicts:
        out += f"# conflicts {conflicts}\n"
    return out + format_section("hood", hull)


def format_trace_round(slots, d: int) -> str:
    """write_trace_round (cli.cpp:108-118) of a HoodBuffer layout (n slots,
    blocks of d, corners then REMOTE padding)."""
    a = np.ascontiguousarray(slots, dtype=np.float64).reshape(-1, 2)
    return _text(_lib().hood_format_trace_round, a.ctypes.data, a.shape[0], int(d))


def write_trace(path: str, points, device: int = 0) -> None:
    """The trace file of build_hood with the CLI's on_round_begin observer
    (cli.cpp:163-169): every round's HoodBuffer, then "0".  The round loop runs
    on the GPU (hood_merge_round per round)."""
    a = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 2)
    rc = _lib().hood_write_trace_f64(H.Context.get(device).handle, a.ctypes.data, a.shape[0], path.encode())
    if rc:
        H._raise(rc)
