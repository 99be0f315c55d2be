"""ctypes binding of oracle/_ref/libntf_ref.so (the compiled, unmodified reference).

TEST INFRASTRUCTURE ONLY (see oracle/ntf_oracle.py header for who may import it).
Build with ``make -C oracle`` (needs /root/reference; the built .so travels to
the GPU box with the repo snapshot).  ``available()`` is False when the .so is
absent; callers then fall back to the NumPy restatement.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import List, Optional, Sequence, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "libntf_ref.so")
_lib = None

_P = C.POINTER(C.c_double)
_U = C.POINTER(C.c_uint64)


class RefError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code
        self.msg = msg


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(LIB_PATH)
        _lib.ntfref_last_error.restype = C.c_char_p
    return _lib


def _d(a: np.ndarray):
    return a.ctypes.data_as(_P)


def _u64(vals) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(vals, dtype=np.uint64))


def _check(code):
    if code != 0:
        raise RefError(code, lib().ntfref_last_error().decode())


def _cat(mats: Sequence[np.ndarray]) -> np.ndarray:
    return np.ascontiguousarray(np.concatenate([np.asarray(m, dtype=np.float64).ravel() for m in mats]))


def _split(flat: np.ndarray, shapes) -> List[np.ndarray]:
    out, off = [], 0
    for s in shapes:
        n = int(np.prod(s))
        out.append(flat[off:off + n].reshape(s).copy())
        off += n
    return out


def cp_fit(algo: str, x: np.ndarray, init: Sequence[np.ndarray], beta, eps=1e-12, inner_steps=3,
           max_iters=500, tol=0.0, extrapolate=False, extrap_cap=1.0, extrap_delta=1e-6):
    x = np.ascontiguousarray(x, dtype=np.float64)
    dims = _u64(x.shape)
    rank = init[0].shape[1]
    f = _cat(init)
    tt = np.zeros(max_iters + 1)
    tl = np.zeros(max_iters + 1)
    n = C.c_int(0)
    _check(lib().ntfref_cp_fit(C.c_int(0 if algo == "bcomm" else 1), C.c_int(x.ndim),
                               dims.ctypes.data_as(_U), _d(x), C.c_int(rank), _d(f),
                               C.c_double(beta), C.c_double(eps), C.c_int(inner_steps),
                               C.c_int(max_iters), C.c_double(tol), C.c_int(int(extrapolate)),
                               C.c_double(extrap_cap), C.c_double(extrap_delta), _d(tt), _d(tl),
                               C.byref(n)))
    return _split(f, [(d, rank) for d in x.shape]), tt[:n.value].copy(), tl[:n.value].copy()


def tucker_fit(algo: str, x: np.ndarray, core: np.ndarray, factors: Sequence[np.ndarray], beta,
               eps=1e-12, inner_steps=3, max_iters=500, tol=0.0, extrapolate=False,
               extrap_cap=1.0, extrap_delta=1e-6):
    x = np.ascontiguousarray(x, dtype=np.float64)
    dims = _u64(x.shape)
    ranks = _u64(core.shape)
    c = np.ascontiguousarray(core, dtype=np.float64).copy()
    f = _cat(factors)
    tt = np.zeros(max_iters + 1)
    tl = np.zeros(max_iters + 1)
    n = C.c_int(0)
    _check(lib().ntfref_tucker_fit(C.c_int(0 if algo == "bcomm" else 1), C.c_int(x.ndim),
                                   dims.ctypes.data_as(_U), _d(x), ranks.ctypes.data_as(_U), _d(c),
                                   _d(f), C.c_double(beta), C.c_double(eps), C.c_int(inner_steps),
                                   C.c_int(max_iters), C.c_double(tol), C.c_int(int(extrapolate)),
                                   C.c_double(extrap_cap), C.c_double(extrap_delta), _d(tt), _d(tl),
                                   C.byref(n)))
    return c, _split(f, list(zip(x.shape, core.shape))), tt[:n.value].copy(), tl[:n.value].copy()


def cp_time_outer(algo: str, x: np.ndarray, init: Sequence[np.ndarray], beta, steps, inner_steps=5,
                  eps=1e-12) -> Tuple[float, List[np.ndarray]]:
    x = np.ascontiguousarray(x, dtype=np.float64)
    dims = _u64(x.shape)
    rank = init[0].shape[1]
    f = _cat(init)
    sec = C.c_double(0.0)
    _check(lib().ntfref_cp_time_outer(C.c_int(0 if algo == "bcomm" else 1), C.c_int(x.ndim),
                                      dims.ctypes.data_as(_U), _d(x), C.c_int(rank), _d(f),
                                      C.c_double(beta), C.c_double(eps), C.c_int(inner_steps),
                                      C.c_int(steps), C.byref(sec)))
    return sec.value, _split(f, [(d, rank) for d in x.shape])


def cp_block_update(x, factors, mode, beta, eps=1e-12, anchor: Optional[np.ndarray] = None):
    x = np.ascontiguousarray(x, dtype=np.float64)
    rank = factors[0].shape[1]
    f = _cat(factors)
    a = None if anchor is None else np.ascontiguousarray(anchor, dtype=np.float64)
    _check(lib().ntfref_cp_block_update(C.c_int(x.ndim), _u64(x.shape).ctypes.data_as(_U), _d(x),
                                        C.c_int(rank), _d(f), C.c_int(mode),
                                        None if a is None else _d(a), C.c_double(beta), C.c_double(eps)))
    return _split(f, [(d, rank) for d in x.shape])


def cp_bcomm_sweep(x, factors, beta, eps=1e-12):
    x = np.ascontiguousarray(x, dtype=np.float64)
    rank = factors[0].shape[1]
    f = _cat(factors)
    _check(lib().ntfref_cp_bcomm_sweep(C.c_int(x.ndim), _u64(x.shape).ctypes.data_as(_U), _d(x),
                                       C.c_int(rank), _d(f), C.c_double(beta), C.c_double(eps)))
    return _split(f, [(d, rank) for d in x.shape])


def cp_jcomm_reference(x, factors, beta, eps=1e-12):
    x = np.ascontiguousarray(x, dtype=np.float64)
    rank = factors[0].shape[1]
    f = _cat(factors)
    p = np.zeros_like(x)
    q = np.zeros_like(x)
    _check(lib().ntfref_cp_jcomm_reference(C.c_int(x.ndim), _u64(x.shape).ctypes.data_as(_U), _d(x),
                                           C.c_int(rank), _d(f), C.c_double(beta), C.c_double(eps),
                                           _d(p), _d(q)))
    return p, q


def cp_jcomm_inner_update(x, ref, current, mode, beta, eps=1e-12):
    x = np.ascontiguousarray(x, dtype=np.float64)
    rank = ref[0].shape[1]
    r = _cat(ref)
    c = _cat(current)
    _check(lib().ntfref_cp_jcomm_inner_update(C.c_int(x.ndim), _u64(x.shape).ctypes.data_as(_U),
                                              _d(x), C.c_int(rank), _d(r), _d(c), C.c_int(mode),
                                              C.c_double(beta), C.c_double(eps)))
    return _split(c, [(d, rank) for d in x.shape])


def cp_jcomm_outer_step(x, factors, beta, inner_steps, eps=1e-12):
    x = np.ascontiguousarray(x, dtype=np.float64)
    rank = factors[0].shape[1]
    f = _cat(factors)
    _check(lib().ntfref_cp_jcomm_outer_step(C.c_int(x.ndim), _u64(x.shape).ctypes.data_as(_U), _d(x),
                                            C.c_int(rank), _d(f), C.c_double(beta),
                                            C.c_int(inner_steps), C.c_double(eps)))
    return _split(f, [(d, rank) for d in x.shape])


def cp_reconstruct(factors):
    dims = [a.shape[0] for a in factors]
    rank = factors[0].shape[1]
    out = np.zeros(dims)
    _check(lib().ntfref_cp_reconstruct(C.c_int(len(dims)), _u64(dims).ctypes.data_as(_U), C.c_int(rank),
                                       _d(_cat(factors)), _d(out)))
    return out


def cp_contract(t, factors, mode):
    t = np.ascontiguousarray(t, dtype=np.float64)
    rank = factors[mode].shape[1]
    out = np.zeros((t.shape[mode], rank))
    _check(lib().ntfref_cp_contract(C.c_int(t.ndim), _u64(t.shape).ctypes.data_as(_U), _d(t),
                                    C.c_int(rank), _d(_cat(factors)), C.c_int(mode), _d(out)))
    return out


def D_beta(x, xhat, beta):
    x = np.ascontiguousarray(x, dtype=np.float64).ravel()
    xh = np.ascontiguousarray(xhat, dtype=np.float64).ravel()
    out = C.c_double(0)
    _check(lib().ntfref_D_beta(C.c_uint64(x.size), _d(x), _d(xh), C.c_double(beta), C.byref(out)))
    return out.value


def tucker_reconstruct(core, factors):
    dims = [a.shape[0] for a in factors]
    out = np.zeros(dims)
    c = np.ascontiguousarray(core, dtype=np.float64)
    _check(lib().ntfref_tucker_reconstruct(C.c_int(len(dims)), _u64(dims).ctypes.data_as(_U),
                                           _u64(core.shape).ctypes.data_as(_U), _d(c),
                                           _d(_cat(factors)), _d(out)))
    return out


def tucker_step(kind, x, core, factors, mode=0, beta=1.0, inner=1, eps=1e-12, ref=None):
    x = np.ascontiguousarray(x, dtype=np.float64)
    c = np.ascontiguousarray(core, dtype=np.float64).copy()
    f = _cat(factors)
    rc = rf = None
    if ref is not None:
        rc = np.ascontiguousarray(ref[0], dtype=np.float64)
        rf = _cat(ref[1])
    _check(lib().ntfref_tucker_step(C.c_int(kind), C.c_int(x.ndim), _u64(x.shape).ctypes.data_as(_U),
                                    _d(x), _u64(core.shape).ctypes.data_as(_U),
                                    None if rc is None else _d(rc), None if rf is None else _d(rf),
                                    _d(c), _d(f), C.c_int(mode), C.c_double(beta), C.c_int(inner),
                                    C.c_double(eps)))
    return c, _split(f, list(zip(x.shape, core.shape)))


def rng_uniform(seed, stream, n):
    out = np.zeros(n)
    _check(lib().ntfref_rng_uniform(C.c_uint64(seed), C.c_uint64(stream), C.c_uint64(n), _d(out)))
    return out


def init_cp_factors(dims, rank, seed, eps=1e-12):
    out = np.zeros(int(sum(dims)) * rank)
    _check(lib().ntfref_init_cp_factors(C.c_int(len(dims)), _u64(dims).ctypes.data_as(_U), C.c_int(rank),
                                        C.c_uint64(seed), C.c_double(eps), _d(out)))
    return _split(out, [(d, rank) for d in dims])


# ---- I/O (reference io.cpp) ---------------------------------------------------

def write_tensor(path: str, x: np.ndarray) -> None:
    lib().ntfref_write_tensor.argtypes = [C.c_char_p, C.c_int, _U, _P]
    x = np.ascontiguousarray(x, dtype=np.float64)
    dims = _u64(x.shape)
    _check(lib().ntfref_write_tensor(path.encode(), x.ndim, dims.ctypes.data_as(_U), _d(x)))


def read_coo_dense(path: str, cap: int, floor: Optional[float] = None) -> np.ndarray:
    """read_coo through the shim, in a child interpreter that has not loaded
    NumPy (the reference's iostream parsing crashes inside a NumPy process
    here -- an environment quirk, not a reference behaviour)."""
    import json
    import subprocess
    import sys
    code = (
        "import ctypes as C, json, sys\n"
        f"l = C.CDLL({LIB_PATH!r})\n"
        f"out = (C.c_double * {cap})(); order = C.c_int(0); dims = (C.c_uint64 * 16)()\n"
        f"rc = l.ntfref_read_coo_dense({path.encode()!r}, {1 if floor is not None else 0}, "
        f"C.c_double({float(floor or 0.0)!r}), C.c_uint64({cap}), out, C.byref(order), dims)\n"
        "l.ntfref_last_error.restype = C.c_char_p\n"
        "print(json.dumps([rc, l.ntfref_last_error().decode(), order.value, list(dims)[:order.value], "
        "[float.hex(v) for v in out]]))\n")
    rc, msg, order, shape, vals = json.loads(subprocess.run([sys.executable, "-c", code], capture_output=True,
                                                            text=True, check=True).stdout)
    if rc != 0:
        raise RefError(rc, msg)
    n = int(np.prod(shape))
    return np.array([float.fromhex(v) for v in vals[:n]]).reshape(shape)


def write_trace(path: str, times, losses) -> None:
    lib().ntfref_write_trace.argtypes = [C.c_char_p, C.c_int, _P, _P]
    t = np.ascontiguousarray(times, dtype=np.float64)
    l = np.ascontiguousarray(losses, dtype=np.float64)
    _check(lib().ntfref_write_trace(path.encode(), len(t), _d(t), _d(l)))


def mu_unfold_cp_sweep(x, factors, beta, eps=1e-12):
    """The compiled reference's matricized sweep (unfold.cpp:109-135)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    f = _cat(factors)
    rank = np.shape(factors[0])[1]
    _check(lib().ntfref_mu_unfold_cp_sweep(C.c_int(x.ndim), _u64(x.shape).ctypes.data_as(_U), _d(x), C.c_int(rank),
                                           _d(f), C.c_double(beta), C.c_double(eps)))
    return _split(f, [np.shape(a) for a in factors])


def joint_surrogate_cp(theta, ref, x, beta, eps=1e-12):
    """reference oracle::eval_joint_surrogate_cp (oracle.cpp:215-243)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    rank = ref[0].shape[1]
    out = C.c_double(0)
    _check(lib().ntfref_joint_surrogate_cp(C.c_int(x.ndim), _u64(x.shape).ctypes.data_as(_U), _d(x), C.c_int(rank),
                                           _d(_cat(theta)), _d(_cat(ref)), C.c_double(beta), C.c_double(eps),
                                           C.byref(out)))
    return out.value


def joint_surrogate_tucker(theta, ref, x, beta, eps=1e-12):
    """reference oracle::eval_joint_surrogate_tucker (oracle.cpp:245-281); models are (core, factors)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    tc = np.ascontiguousarray(theta[0], dtype=np.float64)
    rc = np.ascontiguousarray(ref[0], dtype=np.float64)
    out = C.c_double(0)
    _check(lib().ntfref_joint_surrogate_tucker(C.c_int(x.ndim), _u64(x.shape).ctypes.data_as(_U), _d(x),
                                               _u64(rc.shape).ctypes.data_as(_U), _d(tc), _d(_cat(theta[1])),
                                               _d(rc), _d(_cat(ref[1])), C.c_double(beta), C.c_double(eps),
                                               C.byref(out)))
    return out.value


def scalar_minimizer(num, den, beta, floor=1e-12):
    """reference oracle::scalar_minimizer and jmm_scalar_objective at the minimizer (oracle.cpp:285-302)."""
    u, g = C.c_double(0), C.c_double(0)
    _check(lib().ntfref_scalar_minimizer(C.c_double(num), C.c_double(den), C.c_double(beta), C.c_double(floor),
                                         C.byref(u), C.byref(g)))
    return u.value, g.value
