"""Reference-facing API of the B200 MU engine (mirrors namespace ``ntf``).

Names, argument meaning and error behaviour follow the reference C++ solver
API (/root/reference/proj/include/ntf/{cp,tucker,tensor,divergence,config}.hpp);
every call goes through the C ABI of libntfg.so (include/ntfg.h).

Models are plain NumPy arrays: a CP model is a list of I_n x R fp64 factor
matrices; a Tucker model is ``(core, [factors])``.  The data tensor ``x`` is
either a NumPy array (host; copied to the device per call) or a CUDA torch
tensor (device resident, fp32 or fp64) -- the latter is what a benchmark or a
data-parallel rank passes to keep X in HBM.
"""
from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import _native as N


# ---------------------------------------------------------------------------
# errors (reference include/ntf/errors.hpp:10-43)

class NtfError(Exception):
    pass


class ShapeError(NtfError, ValueError):
    pass


class DomainError(NtfError, ArithmeticError):
    pass


class NumericalError(NtfError, RuntimeError):
    pass


class FormatError(NtfError, RuntimeError):
    pass


class CudaError(NtfError, RuntimeError):
    pass


class CommError(NtfError, RuntimeError):
    pass


_STATUS = {
    N.NtfgStatus.SHAPE: ShapeError,
    N.NtfgStatus.DOMAIN: DomainError,
    N.NtfgStatus.NUMERICAL: NumericalError,
    N.NtfgStatus.FORMAT: FormatError,
    N.NtfgStatus.CUDA: CudaError,
    N.NtfgStatus.COMM: CommError,
    N.NtfgStatus.OOM: CudaError,
    N.NtfgStatus.INTERNAL: NtfError,
}


def _check(status: int):
    if status != N.NtfgStatus.OK:
        raise _STATUS.get(status, NtfError)(N.last_error())


# ---------------------------------------------------------------------------
# config / results (reference config.hpp:18-39, cp.hpp:24-27, tucker.hpp:26-29)

F64 = 0
F32 = 1


@dataclass
class FitConfig:
    beta: float = 1.0
    rank: int = 1
    ranks: List[int] = field(default_factory=list)
    eps: float = 1e-12
    inner_steps: int = 3
    max_iters: int = 500
    tol: float = 0.0
    seed: int = 0
    extrapolate: bool = False
    extrap_cap: float = 1.0
    extrap_delta: float = 1e-6
    data_floor: Optional[float] = None
    # new fields (north star: device options as additions)
    precision: str = "f64"      # "f64" validation build or "f32" streaming
    use_graphs: bool = True

    def _c(self):
        ranks = np.ascontiguousarray(np.asarray(self.ranks, dtype=np.uint64))
        c = N.FitConfigC()
        c.beta = float(self.beta)
        c.rank = int(self.rank)
        c.ranks = ranks.ctypes.data_as(C.POINTER(C.c_uint64)) if ranks.size else None
        c.n_ranks = int(ranks.size)
        c.eps = float(self.eps)
        c.inner_steps = int(self.inner_steps)
        c.max_iters = int(self.max_iters)
        c.tol = float(self.tol)
        c.seed = int(self.seed)
        c.extrapolate = int(bool(self.extrapolate))
        c.extrap_cap = float(self.extrap_cap)
        c.extrap_delta = float(self.extrap_delta)
        c.has_data_floor = int(self.data_floor is not None)
        c.data_floor = float(self.data_floor) if self.data_floor is not None else 0.0
        c.precision = _prec(self.precision)
        c.use_graphs = int(bool(self.use_graphs))
        return c, ranks  # keep ranks alive


@dataclass
class TraceRecord:
    iter: int
    time_s: float
    loss: float


@dataclass
class CpFitResult:
    model: List[np.ndarray]
    trace: List[TraceRecord]


@dataclass
class TuckerFitResult:
    model: Tuple[np.ndarray, List[np.ndarray]]
    trace: List[TraceRecord]


@dataclass
class JcommCpReference:
    ref: List[np.ndarray]
    p: np.ndarray
    q: np.ndarray


@dataclass
class JcommTuckerReference:
    """reference tucker.hpp:59-63: the reference model and its P~/Q~."""
    ref: Tuple[np.ndarray, List[np.ndarray]]
    p: np.ndarray
    q: np.ndarray


def _prec(p) -> int:
    if p in ("f64", "fp64", "float64", F64, np.float64):
        return F64
    if p in ("f32", "fp32", "float32", F32, np.float32):
        return F32
    raise ValueError(f"unknown precision {p!r}")


def validate_fit_config(cfg: FitConfig) -> None:
    """config.cpp:7-18 via ntfg_validate_fit_config."""
    c, _keep = cfg._c()
    _check(N.load().ntfg_validate_fit_config(C.byref(c)))


# ---------------------------------------------------------------------------
# context

class Context:
    """Owns one ntfg_context (device, stream, cached buffers)."""

    def __init__(self, device: int = 0):
        lib = N.load()
        h = C.c_void_p()
        _check(lib.ntfg_context_create(int(device), C.byref(h)))
        self.h = h
        self.device = device
        self._allreduce_cb = None

    def close(self):
        if self.h:
            N.load().ntfg_context_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream_ptr: int):
        _check(N.load().ntfg_context_set_stream(self.h, C.c_void_p(stream_ptr)))

    def set_allreduce(self, fn):
        """fn(device_ptr:int, count:int, stream_ptr:int) -> None; sums in place across ranks."""
        if fn is None:
            self._allreduce_cb = None
            _check(N.load().ntfg_context_set_allreduce(self.h, N.ALLREDUCE_FN(), None))
            return

        def tramp(user, buf, count, stream):
            try:
                fn(C.cast(buf, C.c_void_p).value, int(count), stream or 0)
                return 0
            except Exception:  # reported as NTFG_ERR_COMM by the engine
                import traceback
                traceback.print_exc()
                return 1

        self._allreduce_cb = N.ALLREDUCE_FN(tramp)
        _check(N.load().ntfg_context_set_allreduce(self.h, self._allreduce_cb, None))

    def stats(self) -> dict:
        s = N.StatsC()
        _check(N.load().ntfg_context_stats(self.h, C.byref(s)))
        return {f: getattr(s, f) for f, _ in N.StatsC._fields_}

    def set_profiling(self, enabled: bool):
        _check(N.load().ntfg_context_set_profiling(self.h, int(bool(enabled))))

    def set_comm_buffer(self, ptr: int, capacity: int):
        _check(N.load().ntfg_context_set_comm_buffer(self.h, C.c_void_p(ptr), int(capacity)))

    def init_nccl(self, unique_id: bytes, nranks: int, rank: int):
        """Attach a native NCCL communicator (ntfg_context_init_nccl): sharded
        fits then allreduce on the context stream inside the CUDA graph."""
        if len(unique_id) != 128:
            raise ValueError("NCCL unique id must be 128 bytes")
        buf = C.create_string_buffer(bytes(unique_id), 128)
        _check(N.load().ntfg_context_init_nccl(self.h, C.cast(buf, C.c_void_p), int(nranks), int(rank)))

    def trim(self):
        _check(N.load().ntfg_context_trim(self.h))


_default = {}
_dlock = threading.Lock()


def nccl_unique_id() -> bytes:
    """ncclGetUniqueId through libntfg (rank 0 creates it, the caller broadcasts it)."""
    buf = C.create_string_buffer(128)
    _check(N.load().ntfg_nccl_unique_id(C.cast(buf, C.c_void_p)))
    return buf.raw


def default_context(device: int = 0) -> Context:
    with _dlock:
        c = _default.get((threading.get_ident(), device))
        if c is None:
            c = Context(device)
            _default[(threading.get_ident(), device)] = c
        return c


# ---------------------------------------------------------------------------
# marshalling helpers

_DP = C.POINTER(C.c_double)
_UP = C.POINTER(C.c_uint64)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _dp(a: np.ndarray):
    return a.ctypes.data_as(_DP)


def _u64(v) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(v, dtype=np.uint64))


def _cat(mats: Sequence[np.ndarray]) -> np.ndarray:
    return np.ascontiguousarray(np.concatenate([_f64(m).ravel() for m in mats]))


def _split(flat: np.ndarray, shapes) -> List[np.ndarray]:
    out, off = [], 0
    for s in shapes:
        n = int(np.prod(s))
        out.append(flat[off:off + n].reshape(s).copy())
        off += n
    return out


def _is_cuda_tensor(x) -> bool:
    try:
        import torch
        return isinstance(x, torch.Tensor) and x.is_cuda
    except ImportError:
        return False


def _x_arg(x):
    """(dims, pointer, dtype code, location, keepalive) for host or device X."""
    try:
        import torch
        if isinstance(x, torch.Tensor):
            if not x.is_contiguous():
                raise ShapeError("x must be contiguous")
            if x.dtype not in (torch.float32, torch.float64):
                raise ShapeError("x must be float32 or float64")
            loc = 1 if x.is_cuda else 0
            if x.is_cuda:
                # the engine reads X on its own stream: finish torch's pending
                # writes to it first (no cross-stream race on device inputs)
                torch.cuda.current_stream(x.device).synchronize()
            return (list(x.shape), C.c_void_p(x.data_ptr()), 1 if x.dtype == torch.float32 else 0,
                    loc, x)
    except ImportError:
        pass
    a = np.asarray(x)
    if a.dtype == np.float32:
        a = np.ascontiguousarray(a)
        return list(a.shape), C.c_void_p(a.ctypes.data), 1, 0, a
    a = _f64(a)
    return list(a.shape), C.c_void_p(a.ctypes.data), 0, 0, a


def _check_cp_model(factors, dims, op):
    if len(factors) == 0:
        raise ShapeError("CpFactors: at least one factor required")
    r = factors[0].shape[1] if np.ndim(factors[0]) == 2 else 0
    for a in factors:
        if np.ndim(a) != 2 or a.shape[1] != r:
            raise ShapeError("CpFactors: factors must share a column count")
        if a.shape[0] == 0 or r == 0:
            raise ShapeError("CpFactors: empty factor")
    if dims is not None:
        if len(factors) != len(dims):
            raise ShapeError(f"{op}: order mismatch")
        for a, d in zip(factors, dims):
            if a.shape[0] != d:
                raise ShapeError(f"{op}: factor rows do not match data dimension")
    return r


def _trace(rows, n) -> List[TraceRecord]:
    return [TraceRecord(int(rows[i].iter), float(rows[i].time_s), float(rows[i].loss)) for i in range(n)]


# ---------------------------------------------------------------------------
# CP fits (reference cp.hpp:48,76)

def _cp_fit(algo: int, x, init, cfg: FitConfig, ctx=None, shard=None) -> CpFitResult:
    ctx = ctx or default_context()
    dims, xp, xdt, xloc, keep = _x_arg(x)
    init = [_f64(a) for a in init]
    cfgc, keep_r = cfg._c()
    _check(N.load().ntfg_validate_fit_config(C.byref(cfgc)))
    r = _check_cp_model(init, dims, "bcomm_fit" if algo == 0 else "jcomm_fit")
    if r != cfg.rank:
        cfgc.rank = r  # the model's column count is authoritative (reference ignores cfg.rank)
    f = _cat(init)
    rows = (N.TraceRowC * (int(cfg.max_iters) + 1))()
    n = C.c_uint64(0)
    sh = None
    if shard is not None:
        sh = N.ShardC(int(shard[0]), int(shard[1]))
    _check(N.load().ntfg_cp_fit(ctx.h, C.byref(cfgc), algo, len(dims), _u64(dims).ctypes.data_as(_UP), xp,
                                xdt, xloc, C.byref(sh) if sh is not None else None, _dp(f), rows,
                                C.byref(n)))
    return CpFitResult(_split(f, [a.shape for a in init]), _trace(rows, n.value))


def bcomm_fit(x, init, cfg: FitConfig, ctx: Optional[Context] = None, shard=None) -> CpFitResult:
    """Block-MM CP fit (reference cp.cpp:244-269)."""
    return _cp_fit(0, x, init, cfg, ctx, shard)


def jcomm_fit(x, init, cfg: FitConfig, ctx: Optional[Context] = None, shard=None) -> CpFitResult:
    """Joint-MM CP fit (reference cp.cpp:271-298)."""
    return _cp_fit(1, x, init, cfg, ctx, shard)


def _cp_fit_coo(algo: int, indices, values, dims, init, cfg: FitConfig, ctx=None, shard=None) -> CpFitResult:
    ctx = ctx or default_context()
    dims = [int(d) for d in dims]
    init = [_f64(a) for a in init]
    cfgc, keep_r = cfg._c()
    _check(N.load().ntfg_validate_fit_config(C.byref(cfgc)))
    r = _check_cp_model(init, dims, "coo fit")
    if r != cfg.rank:
        cfgc.rank = r
    keep = []
    if _is_cuda_tensor(indices):
        import torch
        idx = indices.to(torch.int32).contiguous()
        val = values.contiguous()
        if idx.dim() != 2 or idx.shape[1] != len(dims) or val.numel() != idx.shape[0]:
            raise ShapeError("coo fit: indices must be [nnz, order] with one value per nonzero")
        keep += [idx, val]
        ip, vp, vdt, loc, nnz = C.c_void_p(idx.data_ptr()), C.c_void_p(val.data_ptr()), \
            (1 if val.dtype == torch.float32 else 0), 1, idx.shape[0]
        if val.dtype not in (torch.float32, torch.float64):
            raise ShapeError("coo fit: values must be float32 or float64")
    else:
        idx = np.ascontiguousarray(np.asarray(indices), dtype=np.int32)
        val = np.asarray(values)
        val = np.ascontiguousarray(val, dtype=np.float32 if val.dtype == np.float32 else np.float64)
        if idx.ndim != 2 or idx.shape[1] != len(dims) or val.size != idx.shape[0]:
            raise ShapeError("coo fit: indices must be [nnz, order] with one value per nonzero")
        keep += [idx, val]
        ip, vp, vdt, loc, nnz = C.c_void_p(idx.ctypes.data), C.c_void_p(val.ctypes.data), \
            (1 if val.dtype == np.float32 else 0), 0, idx.shape[0]
    f = _cat(init)
    rows = (N.TraceRowC * (int(cfg.max_iters) + 1))()
    n = C.c_uint64(0)
    sh = None if shard is None else N.ShardC(int(shard[0]), int(shard[1]))
    _check(N.load().ntfg_cp_fit_coo(ctx.h, C.byref(cfgc), algo, len(dims), _u64(dims).ctypes.data_as(_UP),
                                    int(nnz), ip, vp, vdt, loc, C.byref(sh) if sh is not None else None, _dp(f),
                                    rows, C.byref(n)))
    return CpFitResult(_split(f, [a.shape for a in init]), _trace(rows, n.value))


def bcomm_fit_coo(indices, values, dims, init, cfg: FitConfig, ctx: Optional[Context] = None,
                  shard=None) -> CpFitResult:
    """Block-MM CP fit of a sparse COO count tensor at beta = 1 (new; the
    reference densifies COO input, io.cpp:87-142, then runs bcomm_fit).
    shard = (global_dim0, slab_begin): this rank's nonzeros, i_0 rebased to
    its mode-0 slab (see dist.shard_coo)."""
    return _cp_fit_coo(0, indices, values, dims, init, cfg, ctx, shard)


def jcomm_fit_coo(indices, values, dims, init, cfg: FitConfig, ctx: Optional[Context] = None,
                  shard=None) -> CpFitResult:
    """Joint-MM CP fit of a sparse COO count tensor at beta = 1 (see bcomm_fit_coo)."""
    return _cp_fit_coo(1, indices, values, dims, init, cfg, ctx, shard)


def mu_unfold_cp_fit(x, init, cfg: FitConfig, ctx: Optional[Context] = None) -> CpFitResult:
    """Classical matricized MU baseline (reference unfold.cpp:187-197): explicit
    Khatri-Rao + unfolding + cuBLAS GEMMs, for the contraction-vs-unfolding
    comparison."""
    ctx = ctx or default_context()
    dims, xp, xdt, xloc, keep = _x_arg(x)
    init = [_f64(a) for a in init]
    cfgc, keep_r = cfg._c()
    _check(N.load().ntfg_validate_fit_config(C.byref(cfgc)))
    r = _check_cp_model(init, dims, "mu_unfold_cp_fit")
    cfgc.rank = r
    f = _cat(init)
    rows = (N.TraceRowC * (int(cfg.max_iters) + 1))()
    n = C.c_uint64(0)
    _check(N.load().ntfg_cp_mu_unfold_fit(ctx.h, C.byref(cfgc), len(dims), _u64(dims).ctypes.data_as(_UP), xp, xdt,
                                          xloc, _dp(f), rows, C.byref(n)))
    return CpFitResult(_split(f, [a.shape for a in init]), _trace(rows, n.value))


def mu_unfold_cp_sweep(f, x, beta: float, eps: float, precision: str = "f64", ctx=None) -> List[np.ndarray]:
    """mu_unfold_cp_sweep (reference unfold.cpp:109-135) on the GPU."""
    ctx = ctx or default_context()
    x = _f64(x)
    f = [_f64(a) for a in f]
    r = _check_cp_model(f, list(x.shape), "mu_unfold_cp_sweep")
    flat = _cat(f)
    _check(N.load().ntfg_cp_mu_unfold_sweep(ctx.h, _prec(precision), float(beta), float(eps), x.ndim,
                                            _u64(list(x.shape)).ctypes.data_as(_UP), _dp(x), r, _dp(flat)))
    return _split(flat, [a.shape for a in f])


def mu_unfold_tucker_fit(x, init, cfg: FitConfig, ctx: Optional[Context] = None) -> TuckerFitResult:
    """Classical matricized Tucker MU baseline (reference unfold.cpp:137-185,
    199-209): every mode product through an explicit unfolding + cuBLAS GEMM."""
    ctx = ctx or default_context()
    dims, xp, xdt, xloc, keep = _x_arg(x)
    core, fs = _check_tucker(init[0], init[1], dims, "mu_unfold_tucker_fit")
    cfgc, keep_r = cfg._c()
    _check(N.load().ntfg_validate_fit_config(C.byref(cfgc)))
    c = core.copy()
    f = _cat(fs)
    rows = (N.TraceRowC * (int(cfg.max_iters) + 1))()
    n = C.c_uint64(0)
    _check(N.load().ntfg_tucker_mu_unfold_fit(ctx.h, C.byref(cfgc), len(dims), _u64(dims).ctypes.data_as(_UP), xp,
                                              xdt, xloc, _dp(c), _dp(f), rows, C.byref(n)))
    return TuckerFitResult((c, _split(f, [a.shape for a in fs])), _trace(rows, n.value))


def mu_unfold_tucker_sweep(core, factors, x, beta: float, eps: float, precision: str = "f64", ctx=None):
    """mu_unfold_tucker_sweep (reference unfold.cpp:137-185) on the GPU."""
    ctx = ctx or default_context()
    x = _f64(x)
    core, fs = _check_tucker(core, factors, list(x.shape), "mu_unfold_tucker_sweep")
    c = core.copy()
    f = _cat(fs)
    _check(N.load().ntfg_tucker_mu_unfold_sweep(ctx.h, _prec(precision), float(beta), float(eps), x.ndim,
                                                _u64(list(x.shape)).ctypes.data_as(_UP),
                                                _u64(list(core.shape)).ctypes.data_as(_UP), _dp(x), _dp(c), _dp(f)))
    return c, _split(f, [a.shape for a in fs])


# ---------------------------------------------------------------------------
# CP step level (reference cp.hpp:30-74)

def cp_reconstruct(factors, precision="f64", ctx=None) -> np.ndarray:
    ctx = ctx or default_context()
    factors = [_f64(a) for a in factors]
    r = _check_cp_model(factors, None, "cp_reconstruct")
    dims = [a.shape[0] for a in factors]
    out = np.zeros(dims)
    _check(N.load().ntfg_cp_reconstruct(ctx.h, _prec(precision), len(dims), _u64(dims).ctypes.data_as(_UP),
                                        r, _dp(_cat(factors)), _dp(out)))
    return out


def cp_contract(t, factors, mode: int, precision="f64", ctx=None) -> np.ndarray:
    ctx = ctx or default_context()
    t = _f64(t)
    if len(factors) != t.ndim:
        raise ShapeError("cp_contract: expected one factor per mode")
    if mode >= t.ndim:
        raise ShapeError("cp_contract: mode out of range")
    r = np.shape(factors[mode])[1]
    fs = []
    for m, a in enumerate(factors):
        a = _f64(a)
        if m == mode:
            a = np.ones((t.shape[m], r))  # only its column count is consulted
        elif a.shape[0] != t.shape[m]:
            raise ShapeError("cp_contract: factor rows do not match tensor dimension")
        elif a.shape[1] != r:
            raise ShapeError("cp_contract: inconsistent column counts")
        fs.append(a)
    out = np.zeros((t.shape[mode], r))
    _check(N.load().ntfg_cp_contract(ctx.h, _prec(precision), t.ndim, _u64(t.shape).ctypes.data_as(_UP), _dp(t),
                                     r, _dp(_cat(fs)), mode, _dp(out)))
    return out


def cp_objective(x, factors, beta: float, precision="f64", ctx=None) -> float:
    """D_beta_mean(x, cp_reconstruct(f)) in one fused pass (reference cp.cpp:264,293)."""
    ctx = ctx or default_context()
    x = _f64(x)
    factors = [_f64(a) for a in factors]
    r = _check_cp_model(factors, list(x.shape), "cp_objective")
    out = C.c_double(0)
    _check(N.load().ntfg_cp_objective(ctx.h, _prec(precision), float(beta), x.ndim,
                                      _u64(x.shape).ctypes.data_as(_UP), _dp(x), r, _dp(_cat(factors)),
                                      C.byref(out)))
    return out.value


def D_beta(x, xhat, beta: float, ctx=None) -> float:
    """divergence.cpp:35-40."""
    ctx = ctx or default_context()
    x = _f64(x)
    xhat = _f64(xhat)
    if x.shape != xhat.shape:
        raise ShapeError("D_beta: shape mismatch")
    out = C.c_double(0)
    _check(N.load().ntfg_D_beta(ctx.h, float(beta), x.size, _dp(x), _dp(xhat), C.byref(out)))
    return out.value


def D_beta_mean(x, xhat, beta: float, ctx=None) -> float:
    """divergence.cpp:42-44."""
    return D_beta(x, xhat, beta, ctx) / float(np.asarray(x).size)


def cp_block_update_anchored(f, mode, anchor, x, beta, eps, precision="f64", ctx=None):
    ctx = ctx or default_context()
    x = _f64(x)
    f = [_f64(a) for a in f]
    r = _check_cp_model(f, list(x.shape), "cp_block_update")
    if mode >= len(f):
        raise ShapeError("cp_block_update: mode out of range")
    flat = _cat(f)
    a = None if anchor is None else _f64(anchor)
    if a is not None and a.shape != f[mode].shape:
        raise ShapeError("cp_block_update: anchor shape mismatch")
    _check(N.load().ntfg_cp_block_update(ctx.h, _prec(precision), float(beta), float(eps), x.ndim,
                                         _u64(x.shape).ctypes.data_as(_UP), _dp(x), r, _dp(flat), mode,
                                         None if a is None else _dp(a)))
    return _split(flat, [m.shape for m in f])


def bcomm_block_update(f, mode, x, beta, eps, precision="f64", ctx=None):
    """cp.cpp:125-129."""
    if mode >= len(f):
        raise ShapeError("bcomm_block_update: mode out of range")
    return cp_block_update_anchored(f, mode, None, x, beta, eps, precision, ctx)


def bcomm_sweep(f, x, beta, eps, precision="f64", ctx=None):
    """cp.cpp:131-135."""
    ctx = ctx or default_context()
    x = _f64(x)
    f = [_f64(a) for a in f]
    r = _check_cp_model(f, list(x.shape), "bcomm_sweep")
    flat = _cat(f)
    _check(N.load().ntfg_cp_bcomm_sweep(ctx.h, _prec(precision), float(beta), float(eps), x.ndim,
                                        _u64(x.shape).ctypes.data_as(_UP), _dp(x), r, _dp(flat)))
    return _split(flat, [m.shape for m in f])


def make_jcomm_reference(ref, x, beta, eps, precision="f64", ctx=None) -> JcommCpReference:
    """cp.cpp:202-208 (P~, Q~ returned to the host as the reference struct exposes them)."""
    ctx = ctx or default_context()
    x = _f64(x)
    ref = [_f64(a) for a in ref]
    r = _check_cp_model(ref, list(x.shape), "make_jcomm_reference")
    p = np.zeros(x.shape)
    q = np.zeros(x.shape)
    _check(N.load().ntfg_cp_jcomm_reference(ctx.h, _prec(precision), float(beta), float(eps), x.ndim,
                                            _u64(x.shape).ctypes.data_as(_UP), _dp(x), r, _dp(_cat(ref)),
                                            _dp(p), _dp(q)))
    return JcommCpReference([a.copy() for a in ref], p, q)


def jcomm_inner_update(current, ctx_ref: JcommCpReference, mode, beta, eps, precision="f64", ctx=None):
    """cp.cpp:210-229."""
    ctx = ctx or default_context()
    cur = [_f64(a) for a in current]
    if mode >= len(cur):
        raise ShapeError("jcomm_inner_update: mode out of range")
    p = _f64(ctx_ref.p)
    q = _f64(ctx_ref.q)
    r = _check_cp_model(cur, list(p.shape), "jcomm_inner_update")
    flat = _cat(cur)
    _check(N.load().ntfg_cp_jcomm_inner_update(ctx.h, _prec(precision), float(beta), float(eps), p.ndim,
                                               _u64(p.shape).ctypes.data_as(_UP), _dp(p), _dp(q), r,
                                               _dp(_cat(ctx_ref.ref)), _dp(flat), mode))
    return _split(flat, [m.shape for m in cur])


def jcomm_outer_step(f, x, beta, inner_steps, eps, precision="f64", ctx=None):
    """cp.cpp:231-240."""
    ctx = ctx or default_context()
    x = _f64(x)
    f = [_f64(a) for a in f]
    r = _check_cp_model(f, list(x.shape), "jcomm_outer_step")
    flat = _cat(f)
    _check(N.load().ntfg_cp_jcomm_outer_step(ctx.h, _prec(precision), float(beta), float(eps),
                                             int(inner_steps), x.ndim, _u64(x.shape).ctypes.data_as(_UP),
                                             _dp(x), r, _dp(flat)))
    return _split(flat, [m.shape for m in f])


# ---------------------------------------------------------------------------
# Tucker (reference tucker.hpp:38-84, tensor.hpp:105-130)

def _check_tucker(core, factors, dims, op):
    core = _f64(core)
    factors = [_f64(a) for a in factors]
    if len(factors) == 0:
        raise ShapeError("TuckerModel: at least one factor required")
    if core.ndim != len(factors):
        raise ShapeError("TuckerModel: core order does not match factor count")
    for n, a in enumerate(factors):
        if a.ndim != 2 or a.shape[1] != core.shape[n]:
            raise ShapeError("TuckerModel: factor columns do not match core dimension")
    if dims is not None:
        if len(dims) != len(factors):
            raise ShapeError(f"{op}: order mismatch")
        for a, d in zip(factors, dims):
            if a.shape[0] != d:
                raise ShapeError(f"{op}: factor rows do not match data dimension")
    return core, factors


def _tucker_fit(algo, x, init, cfg: FitConfig, ctx=None, shard=None) -> TuckerFitResult:
    ctx = ctx or default_context()
    dims, xp, xdt, xloc, keep = _x_arg(x)
    core, fs = _check_tucker(init[0], init[1], dims, "tucker_bcomm_fit" if algo == 0 else "tucker_jcomm_fit")
    cfgc, keep_r = cfg._c()
    _check(N.load().ntfg_validate_fit_config(C.byref(cfgc)))
    c = core.copy()
    f = _cat(fs)
    rows = (N.TraceRowC * (int(cfg.max_iters) + 1))()
    n = C.c_uint64(0)
    sh = None if shard is None else N.ShardC(int(shard[0]), int(shard[1]))
    _check(N.load().ntfg_tucker_fit(ctx.h, C.byref(cfgc), algo, len(dims), _u64(dims).ctypes.data_as(_UP), xp,
                                    xdt, xloc, C.byref(sh) if sh is not None else None, _dp(c), _dp(f),
                                    rows, C.byref(n)))
    return TuckerFitResult((c, _split(f, [a.shape for a in fs])), _trace(rows, n.value))


def tucker_bcomm_fit(x, init, cfg: FitConfig, ctx=None, shard=None) -> TuckerFitResult:
    """tucker.cpp:221-247."""
    return _tucker_fit(0, x, init, cfg, ctx, shard)


def tucker_jcomm_fit(x, init, cfg: FitConfig, ctx=None, shard=None) -> TuckerFitResult:
    """tucker.cpp:249-275."""
    return _tucker_fit(1, x, init, cfg, ctx, shard)


def tucker_reconstruct(core, factors, precision="f64", ctx=None) -> np.ndarray:
    ctx = ctx or default_context()
    core, factors = _check_tucker(core, factors, None, "tucker_reconstruct")
    dims = [a.shape[0] for a in factors]
    out = np.zeros(dims)
    _check(N.load().ntfg_tucker_reconstruct(ctx.h, _prec(precision), len(dims), _u64(dims).ctypes.data_as(_UP),
                                            _u64(core.shape).ctypes.data_as(_UP), _dp(core),
                                            _dp(_cat(factors)), _dp(out)))
    return out


def tucker_multimode_contract(t, factors, skip: Optional[int] = None, precision="f64", ctx=None):
    ctx = ctx or default_context()
    t = _f64(t)
    factors = [_f64(a) for a in factors]
    if len(factors) != t.ndim:
        raise ShapeError("tucker_multimode_contract: expected one factor per mode")
    if skip is not None and skip >= t.ndim:
        raise ShapeError("tucker_multimode_contract: skip mode out of range")
    shape = []
    for m, a in enumerate(factors):
        if skip is not None and m == skip:
            continue
        if a.shape[0] != t.shape[m]:
            raise ShapeError("tucker_multimode_contract: factor rows do not match dimension")
        shape.append(a.shape[1])
    if skip is not None:
        shape.append(t.shape[skip])
    cols = [a.shape[1] for a in factors]
    fs = [a if (skip is None or m != skip) else np.zeros((t.shape[m], a.shape[1])) for m, a in enumerate(factors)]
    out = np.zeros(shape)
    _check(N.load().ntfg_tucker_multimode_contract(ctx.h, _prec(precision), t.ndim,
                                                   _u64(t.shape).ctypes.data_as(_UP), _dp(t),
                                                   _u64(cols).ctypes.data_as(_UP), _dp(_cat(fs)),
                                                   -1 if skip is None else int(skip), _dp(out)))
    return out


def tucker_factor_contract(t, core, factors, mode: int, precision="f64", ctx=None) -> np.ndarray:
    ctx = ctx or default_context()
    t = _f64(t)
    core = _f64(core)
    if len(factors) != t.ndim:
        raise ShapeError("tucker_factor_contract: expected one factor per mode")
    if core.ndim != t.ndim:
        raise ShapeError("tucker_factor_contract: core order does not match tensor order")
    if mode >= t.ndim:
        raise ShapeError("tucker_factor_contract: mode out of range")
    fs = []
    for m, a in enumerate(factors):
        a = _f64(a)
        if m == mode:
            a = np.zeros((t.shape[m], core.shape[m]))
        elif a.shape[0] != t.shape[m] or a.shape[1] != core.shape[m]:
            raise ShapeError("tucker_factor_contract: factor shape mismatch")
        fs.append(a)
    out = np.zeros((t.shape[mode], core.shape[mode]))
    _check(N.load().ntfg_tucker_factor_contract(ctx.h, _prec(precision), t.ndim, _u64(t.shape).ctypes.data_as(_UP),
                                                _dp(t), _u64(core.shape).ctypes.data_as(_UP), _dp(core),
                                                _dp(_cat(fs)), mode, _dp(out)))
    return out


def tucker_objective(x, model, beta, precision="f64", ctx=None) -> float:
    ctx = ctx or default_context()
    x = _f64(x)
    core, fs = _check_tucker(model[0], model[1], list(x.shape), "tucker_objective")
    out = C.c_double(0)
    _check(N.load().ntfg_tucker_objective(ctx.h, _prec(precision), float(beta), x.ndim,
                                          _u64(x.shape).ctypes.data_as(_UP), _dp(x),
                                          _u64(core.shape).ctypes.data_as(_UP), _dp(core), _dp(_cat(fs)),
                                          C.byref(out)))
    return out.value


def _tucker_step(kind, model, x, beta, eps, mode=0, inner=1, ref=None, precision="f64", ctx=None):
    ctx = ctx or default_context()
    x = _f64(x)
    core, fs = _check_tucker(model[0], model[1], list(x.shape), "tucker_step")
    c = core.copy()
    f = _cat(fs)
    rc = rf = None
    if ref is not None:
        rcore, rfs = _check_tucker(ref[0], ref[1], list(x.shape), "tucker_step")
        rc, rf = rcore, _cat(rfs)
    _check(N.load().ntfg_tucker_step(ctx.h, _prec(precision), kind, float(beta), float(eps), int(inner), x.ndim,
                                     _u64(x.shape).ctypes.data_as(_UP), _dp(x),
                                     _u64(core.shape).ctypes.data_as(_UP),
                                     None if rc is None else _dp(rc), None if rf is None else _dp(rf),
                                     _dp(c), _dp(f), int(mode)))
    return c, _split(f, [a.shape for a in fs])


def block_core_update(m, x, beta, eps, precision="f64", ctx=None):
    """tucker.cpp:57-60."""
    return _tucker_step(0, m, x, beta, eps, precision=precision, ctx=ctx)


def block_factor_update(m, mode, x, beta, eps, precision="f64", ctx=None):
    """tucker.cpp:77-81."""
    if mode >= len(m[1]):
        raise ShapeError("block_factor_update: mode out of range")
    return _tucker_step(1, m, x, beta, eps, mode=mode, precision=precision, ctx=ctx)


def tucker_bcomm_sweep(m, x, beta, eps, precision="f64", ctx=None):
    """tucker.cpp:83-88."""
    return _tucker_step(2, m, x, beta, eps, precision=precision, ctx=ctx)


def jcomm_tucker_outer_step(m, x, beta, inner_steps, eps, precision="f64", ctx=None):
    """tucker.cpp:138-149."""
    if inner_steps < 1:
        raise DomainError("jcomm_tucker_outer_step: inner_steps must be >= 1")
    return _tucker_step(3, m, x, beta, eps, inner=inner_steps, precision=precision, ctx=ctx)


def make_jcomm_tucker_reference(ref, x, beta, eps, precision="f64", ctx=None) -> JcommTuckerReference:
    """tucker.cpp:92-98: P~/Q~ of the reference model, computed on the device."""
    ctx = ctx or default_context()
    x = _f64(x)
    core, fs = _check_tucker(ref[0], ref[1], list(x.shape), "make_jcomm_tucker_reference")
    p = np.zeros(x.shape)
    q = np.zeros(x.shape)
    _check(N.load().ntfg_tucker_jcomm_reference(ctx.h, _prec(precision), float(beta), float(eps), x.ndim,
                                                _u64(x.shape).ctypes.data_as(_UP), _dp(x),
                                                _u64(core.shape).ctypes.data_as(_UP), _dp(core), _dp(_cat(fs)),
                                                _dp(p), _dp(q)))
    return JcommTuckerReference((core.copy(), [a.copy() for a in fs]), p, q)


def _tucker_inner(cur, ctx_ref: JcommTuckerReference, block, beta, eps, precision, ctx):
    ctx = ctx or default_context()
    p, q = _f64(ctx_ref.p), _f64(ctx_ref.q)
    if p.shape != q.shape:
        raise ShapeError("jcomm_inner_update: P/Q shape mismatch")
    core, fs = _check_tucker(cur[0], cur[1], list(p.shape), "jcomm_inner_update")
    rcore, rfs = _check_tucker(ctx_ref.ref[0], ctx_ref.ref[1], list(p.shape), "jcomm_inner_update")
    c = core.copy()
    f = _cat(fs)
    _check(N.load().ntfg_tucker_jcomm_inner_update(ctx.h, _prec(precision), float(beta), float(eps), p.ndim,
                                                   _u64(p.shape).ctypes.data_as(_UP), _dp(p), _dp(q),
                                                   _u64(core.shape).ctypes.data_as(_UP), _dp(rcore),
                                                   _dp(_cat(rfs)), _dp(c), _dp(f), int(block)))
    return c, _split(f, [a.shape for a in fs])


def jcomm_inner_core_update(cur, ctx_ref: JcommTuckerReference, beta, eps, precision="f64", ctx=None):
    """tucker.cpp:100-114 (from the cached host P~/Q~)."""
    return _tucker_inner(cur, ctx_ref, -1, beta, eps, precision, ctx)


def jcomm_inner_factor_update(cur, ctx_ref: JcommTuckerReference, mode, beta, eps, precision="f64",
                              ctx=None):
    """tucker.cpp:116-136 (from the cached host P~/Q~)."""
    if mode >= len(cur[1]):
        raise ShapeError("jcomm_inner_factor_update: mode out of range")
    return _tucker_inner(cur, ctx_ref, int(mode), beta, eps, precision, ctx)


# ---------------------------------------------------------------------------
# BMMe step-level API (reference cp.hpp:80-110, tucker.hpp:88-106): factor-sized
# host arithmetic as in the reference; the fit drivers run it on the device.

@dataclass
class ExtrapolationState:
    previous: list
    t: float = 1.0
    alpha: float = 0.0
    cap: float = 1.0
    delta: float = 1e-6
    eps: float = 1e-12
    enabled: bool = False


def _pos_sq(cur, prev) -> float:
    cur, prev = np.asarray(cur, dtype=np.float64), np.asarray(prev, dtype=np.float64)
    if cur.shape != prev.shape:
        raise ShapeError("extrapolation: shape mismatch with recorded iterate")
    d = cur - prev
    d = d[d > 0.0]
    return float(np.sum(d * d))


def _blocks(model):
    """CP: list of factors; Tucker: (core, factors) -> [core] + factors."""
    if isinstance(model, tuple):
        return [model[0]] + list(model[1])
    return list(model)


def make_extrapolation_state(initial, enabled: bool, cap: float, delta: float, eps: float) -> ExtrapolationState:
    """CP factors or a Tucker (core, factors) model (make_tucker_extrapolation_state)."""
    prev = (np.array(initial[0], copy=True), [np.array(a, copy=True) for a in initial[1]]) \
        if isinstance(initial, tuple) else [np.array(a, copy=True) for a in initial]
    return ExtrapolationState(prev, cap=float(cap), delta=float(delta), eps=float(eps), enabled=bool(enabled))


make_tucker_extrapolation_state = make_extrapolation_state


def extrapolation_begin_iteration(st: ExtrapolationState, current) -> None:
    tn = 0.5 * (1.0 + np.sqrt(1.0 + 4.0 * st.t * st.t))
    an = (st.t - 1.0) / tn
    st.t = tn
    cur, prev = _blocks(current), _blocks(st.previous)
    if len(cur) != len(prev):
        raise ShapeError("extrapolation: order mismatch")
    sq = 0.0
    for a, b in zip(cur, prev):
        sq += _pos_sq(a, b)
    st.alpha = min(an, st.cap / (np.sqrt(sq) + st.delta))


def _inertial(cur, prev, alpha, eps):
    cur, prev = np.asarray(cur, dtype=np.float64), np.asarray(prev, dtype=np.float64)
    if cur.shape != prev.shape:
        raise ShapeError("extrapolate_block: shape mismatch with recorded iterate")
    d = cur - prev
    return np.maximum(cur + alpha * np.where(d > 0.0, d, 0.0), eps)


def extrapolate_block(current, st: ExtrapolationState, block: int) -> np.ndarray:
    """CP: factor `block`; Tucker state: factor `block` (the core is extrapolate_core)."""
    facs = st.previous[1] if isinstance(st.previous, tuple) else st.previous
    if block >= len(facs):
        raise ShapeError("extrapolate_block: block out of range")
    return _inertial(current, facs[block], st.alpha, st.eps)


def extrapolate_core(current, st: ExtrapolationState) -> np.ndarray:
    return _inertial(current, st.previous[0], st.alpha, st.eps)


def extrapolation_end_iteration(st: ExtrapolationState, iterate) -> None:
    st.previous = (np.array(iterate[0], copy=True), [np.array(a, copy=True) for a in iterate[1]]) \
        if isinstance(iterate, tuple) else [np.array(a, copy=True) for a in iterate]
