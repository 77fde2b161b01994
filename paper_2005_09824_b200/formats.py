"""On-disk formats of the reference, for the CLI front-end.

* Text FST (`/root/reference/pkg/src/chainloss/fst_io.py:1-140`): parsed by the
  native ingestion code in ``libpaper_lfmmi.so`` (``lfmmi_fst_text_size`` /
  ``lfmmi_fst_text_parse``, host-only, no GPU needed) into a
  :class:`~.graph.ChainGraph`; serialised with 17 significant digits so the
  text round trip is exact.  Errors are :class:`FstParseError` (a
  ``ValueError``) carrying 1-based line numbers.
* PCTN arrays (`array_io.py:1-72`): ``PCTN`` magic, u32 version 1, u32 ndim
  (<= 4), u64 dims, little-endian float64 payload; bit-exact round trip.
"""

from __future__ import annotations

import ctypes
import math
import struct
from pathlib import Path

import numpy as np

from . import _backend
from .graph import ChainGraph

__all__ = ["FstParseError", "parse_fst_text", "serialize_fst_text", "read_array", "write_array"]


class FstParseError(ValueError):
    """Malformed text-FST input (messages carry 1-based line numbers)."""


_LIB = None


def _lib():
    global _LIB
    if _LIB is None:
        lib = ctypes.CDLL(_backend.core_library_path())
        lib.lfmmi_last_error.restype = ctypes.c_char_p
        I32, I64, SZ, P = ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t, ctypes.c_void_p
        lib.lfmmi_fst_text_size.argtypes = [ctypes.c_char_p, SZ, I32, ctypes.POINTER(I64),
                                            ctypes.POINTER(I64)]
        lib.lfmmi_fst_text_parse.argtypes = [ctypes.c_char_p, SZ, I32, I64, I64, P, P, P, P, P]
        lib.lfmmi_fst_text_size.restype = ctypes.c_int
        lib.lfmmi_fst_text_parse.restype = ctypes.c_int
        _LIB = lib
    return _LIB


def parse_fst_text(text: str, num_pdfs: int) -> ChainGraph:
    """Text FST -> :class:`ChainGraph` (fst_io.py:53-110 contract)."""
    if num_pdfs < 1:
        raise ValueError(f"num_pdfs must be >= 1, got {num_pdfs}")
    lib = _lib()
    data = text.encode("utf-8")
    ns, na = ctypes.c_int64(), ctypes.c_int64()
    rc = lib.lfmmi_fst_text_size(data, len(data), int(num_pdfs), ctypes.byref(ns), ctypes.byref(na))
    if rc:
        raise FstParseError(lib.lfmmi_last_error().decode())
    S, I = ns.value, na.value
    src = np.empty(I, np.uint32)
    dst = np.empty(I, np.uint32)
    pdf = np.empty(I, np.uint32)
    prob = np.empty(I, np.float64)
    finals = np.empty(S, np.float64)
    ptr = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    rc = lib.lfmmi_fst_text_parse(data, len(data), int(num_pdfs), S, I, ptr(src), ptr(dst),
                                  ptr(pdf), ptr(prob), ptr(finals))
    if rc:
        raise FstParseError(lib.lfmmi_last_error().decode())
    arcs = list(zip(src.tolist(), dst.tolist(), pdf.tolist(), prob.tolist()))
    return ChainGraph(arcs, S, int(num_pdfs), 0, finals)


def _weight(p: float) -> str:
    return f"{(-math.log(p) + 0.0):.17g}"


def serialize_fst_text(graph) -> str:
    """:class:`ChainGraph` -> text FST: arcs by source state with the initial
    state's block first, then final lines in state order (fst_io.py:118-140)."""
    states = [graph.initial_state] + [s for s in range(graph.num_states) if s != graph.initial_state]
    out = []
    for s in states:
        lo, hi = (int(x) for x in graph.forward_index[s])
        out += [f"{graph.forward_from[i]} {graph.forward_to[i]} {graph.forward_pdf[i] + 1} "
                f"{_weight(graph.forward_probs[i])}" for i in range(lo, hi)]
    out += [f"{s} {_weight(p)}" for s, p in enumerate(graph.final_probs) if p > 0.0]
    return "\n".join(out) + "\n"


_HDR = struct.Struct("<4sII")


def write_array(path, values) -> None:
    """Write ``values`` as float64 PCTN."""
    arr = np.asarray(values, dtype=np.float64, order="C")  # keeps 0-d arrays 0-d
    if arr.ndim > 4:
        raise ValueError(f"PCTN supports at most 4 dimensions, got {arr.ndim}")
    with open(path, "wb") as f:
        f.write(_HDR.pack(b"PCTN", 1, arr.ndim))
        f.write(struct.pack(f"<{arr.ndim}Q", *arr.shape))
        f.write(arr.astype("<f8", copy=False).tobytes())


def read_array(path) -> np.ndarray:
    """Read a PCTN file bit-exactly (ValueError on any malformation)."""
    data = Path(path).read_bytes()
    if len(data) < _HDR.size:
        raise ValueError(f"{path}: truncated header ({len(data)} bytes)")
    magic, version, ndim = _HDR.unpack_from(data)
    if magic != b"PCTN":
        raise ValueError(f"{path}: bad magic {magic!r}, expected b'PCTN'")
    if version != 1:
        raise ValueError(f"{path}: unsupported version {version}")
    if ndim > 4:
        raise ValueError(f"{path}: ndim {ndim} exceeds maximum 4")
    off = _HDR.size + 8 * ndim
    if len(data) < off:
        raise ValueError(f"{path}: truncated header (missing dims)")
    dims = struct.unpack_from(f"<{ndim}Q", data, _HDR.size)
    n = int(np.prod(dims, dtype=np.int64)) if ndim else 1
    need = off + 8 * n
    if len(data) < need:
        raise ValueError(f"{path}: truncated payload ({len(data) - off} of {8 * n} bytes)")
    if len(data) > need:
        raise ValueError(f"{path}: {len(data) - need} trailing bytes after payload")
    return np.reshape(np.frombuffer(data, dtype="<f8", count=n, offset=off).astype(np.float64),
                      tuple(dims))
