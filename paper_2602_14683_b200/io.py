"""Data ingestion and synthetic generation (reference include/ntf/io.hpp, src/io.cpp).

Thin wrappers over the C ABI (include/ntfg.h, csrc/io_api.cu):

* ``read_tensor`` / ``write_tensor`` -- CTF1 files, byte-exact with the
  reference (io.cpp:30-77).  ``device=...`` streams the payload straight into a
  CUDA tensor (pinned staging, fp64 -> fp32 on the device).
* ``read_coo`` -- the reference COO text grammar (io.cpp:87-142) returned as
  nonzeros ``(indices[nnz, N] int32, values[nnz] fp64, dims)`` for the sparse
  fits; ``coo_to_dense`` gives read_coo's dense result (duplicates +=, floor).
* ``write_trace`` -- "iter,time_s,loss" with %.17g (io.cpp:154-164).
* ``philox_uniforms`` / ``cp_factors`` / ``generate_cp_gamma`` -- the
  counter-based generator behind the BASELINE configs (new).
"""
from __future__ import annotations

import ctypes as C
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import _native as N
from .api import TraceRecord, _check, _dp, _u64, _UP, default_context

K_DEFAULT_ENTRY_BUDGET = 1 << 27  # io.hpp:19
STREAM_TRUTH, STREAM_INIT, STREAM_NOISE = 1, 2, 3


def _path(p) -> bytes:
    return str(p).encode()


def ctf1_shape(path, max_entries: int = K_DEFAULT_ENTRY_BUDGET) -> List[int]:
    order = C.c_uint32(0)
    dims = np.zeros(255, dtype=np.uint64)
    _check(N.load().ntfg_ctf1_header(_path(path), C.byref(order), dims.ctypes.data_as(_UP), 255, int(max_entries)))
    return [int(d) for d in dims[:order.value]]


def read_tensor(path, max_entries: int = K_DEFAULT_ENTRY_BUDGET, dtype: str = "f64", device=None):
    """read_tensor (io.cpp:46-77).  Host numpy array, or a CUDA tensor on
    ``device`` (int or torch.device) filled without a host copy."""
    dims = ctf1_shape(path, max_entries)
    code = 1 if dtype == "f32" else 0
    if device is None:
        out = np.empty(dims, dtype=np.float32 if code else np.float64)
        _check(N.load().ntfg_ctf1_read(None, _path(path), C.c_void_p(out.ctypes.data), code, 0, int(max_entries)))
        return out
    import torch
    dev = torch.device("cuda", device) if isinstance(device, int) else torch.device(device)
    out = torch.empty(dims, dtype=torch.float32 if code else torch.float64, device=dev)
    ctx = default_context(dev.index or 0)
    _check(N.load().ntfg_ctf1_read(ctx.h, _path(path), C.c_void_p(out.data_ptr()), code, 1, int(max_entries)))
    return out


def write_tensor(path, x) -> None:
    """write_tensor (io.cpp:30-44): fp64 LE payload (fp32 inputs widen exactly)."""
    try:
        import torch
        if isinstance(x, torch.Tensor):
            t = x.contiguous()
            code = 1 if t.dtype == torch.float32 else 0
            if t.dtype not in (torch.float32, torch.float64):
                t = t.double()
                code = 0
            dims = list(t.shape)
            ctx = default_context(t.device.index or 0) if t.is_cuda else None
            _check(N.load().ntfg_ctf1_write(ctx.h if ctx else None, _path(path), len(dims),
                                            _u64(dims).ctypes.data_as(_UP), C.c_void_p(t.data_ptr()), code,
                                            1 if t.is_cuda else 0))
            return
    except ImportError:
        pass
    a = np.asarray(x)
    a = np.ascontiguousarray(a, dtype=np.float32 if a.dtype == np.float32 else np.float64)
    _check(N.load().ntfg_ctf1_write(None, _path(path), a.ndim, _u64(list(a.shape)).ctypes.data_as(_UP),
                                    C.c_void_p(a.ctypes.data), 1 if a.dtype == np.float32 else 0, 0))


def read_coo(path, max_entries: int = 0) -> Tuple[np.ndarray, np.ndarray, List[int]]:
    """read_coo's grammar and errors (io.cpp:87-142) as nonzeros; duplicates
    are kept (the sparse fits and coo_to_dense accumulate them in order).
    max_entries = 0 disables the dense entry budget (the sparse path never
    materialises the dense tensor)."""
    lib = N.load()
    order = C.c_uint32(0)
    dims = np.zeros(8, dtype=np.uint64)
    nnz = C.c_uint64(0)
    _check(lib.ntfg_coo_text_read(_path(path), C.byref(order), dims.ctypes.data_as(_UP), 8, C.byref(nnz), None,
                                  None, 0, int(max_entries)))
    n = nnz.value
    idx = np.zeros((max(n, 1), order.value), dtype=np.int32)
    val = np.zeros(max(n, 1))
    _check(lib.ntfg_coo_text_read(_path(path), C.byref(order), dims.ctypes.data_as(_UP), 8, C.byref(nnz),
                                  C.c_void_p(idx.ctypes.data), _dp(val), n, int(max_entries)))
    return idx[:n], val[:n], [int(d) for d in dims[:order.value]]


def coo_to_dense(indices, values, dims, floor: Optional[float] = None) -> np.ndarray:
    """The dense tensor read_coo returns: zeros, ``+=`` per line, optional
    elementwise floor (io.cpp:136-141)."""
    dense = np.zeros(int(np.prod(dims)))
    lin = np.ravel_multi_index(tuple(np.asarray(indices, dtype=np.int64).T), tuple(dims))
    np.add.at(dense, lin, np.asarray(values, dtype=np.float64))  # unbuffered, in index order
    dense = dense.reshape(dims)
    return np.maximum(dense, floor) if floor is not None else dense


def write_trace(path, trace: Sequence[TraceRecord]) -> None:
    rows = (N.TraceRowC * max(len(trace), 1))()
    for i, t in enumerate(trace):
        rows[i].iter, rows[i].time_s, rows[i].loss = int(t.iter), float(t.time_s), float(t.loss)
    _check(N.load().ntfg_trace_write(_path(path), rows, len(trace)))


def read_trace(path) -> List[TraceRecord]:
    """read_trace (io.cpp:166-186)."""
    out = []
    with open(path) as f:
        if f.readline().rstrip("\n") != "iter,time_s,loss":
            raise ValueError("line 1: missing trace header")
        for line in f:
            if line.strip():
                a, b, c = line.strip().split(",")
                out.append(TraceRecord(int(a), float(b), float(c)))
    return out


# ---------------------------------------------------------------------------
# generator

def philox_uniforms(seed: int, stream: int, offset: int, n: int) -> np.ndarray:
    out = np.zeros(max(n, 1))
    _check(N.load().ntfg_philox_uniforms(int(seed), int(stream), int(offset), int(n), _dp(out)))
    return out[:n]


def cp_factors(dims, rank: int, seed: int, which: str = "init", eps: float = 1e-12) -> List[np.ndarray]:
    """which='truth': U[0,1) clamped to eps (random_matrix io.cpp:202-208);
    which='init': U[0.1, 1.1) (the BASELINE configs' init)."""
    dims = [int(d) for d in dims]
    out = np.zeros(sum(d * rank for d in dims))
    _check(N.load().ntfg_cp_factors_generate(len(dims), _u64(dims).ctypes.data_as(_UP), int(rank), int(seed),
                                             0 if which == "truth" else 1, float(eps), _dp(out)))
    fs, off = [], 0
    for d in dims:
        fs.append(out[off:off + d * rank].reshape(d, rank).copy())
        off += d * rank
    return fs


def generate_cp_gamma(dims, rank: int, seed: int, k: int = 10, theta: float = 0.1, rows=None,
                      dtype: str = "f32", device=0):
    """X = [[truth]] * Gamma(k, theta) for mode-0 rows ``rows = (row0, row1)``
    (default: all), generated in place on the device (BASELINE C2/C5 data)."""
    import torch
    dims = [int(d) for d in dims]
    r0, r1 = rows if rows is not None else (0, dims[0])
    dev = torch.device("cuda", device) if isinstance(device, int) else torch.device(device)
    x = torch.empty([r1 - r0] + dims[1:], dtype=torch.float32 if dtype == "f32" else torch.float64, device=dev)
    ctx = default_context(dev.index or 0)
    _check(N.load().ntfg_generate_cp_gamma(ctx.h, len(dims), _u64(dims).ctypes.data_as(_UP), int(rank), int(seed),
                                           int(k), float(theta), int(r0), int(r1), C.c_void_p(x.data_ptr()),
                                           1 if dtype == "f32" else 0))
    return x
