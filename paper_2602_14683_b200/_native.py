"""ctypes binding of libntfg.so (the C ABI declared in include/ntfg.h).

The CUDA library is the only compute path: if it is missing or no B200 is
visible, every call raises -- there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libntfg.so")


class NtfgStatus:
    OK = 0
    SHAPE = 1
    DOMAIN = 2
    NUMERICAL = 3
    FORMAT = 4
    CUDA = 5
    COMM = 6
    OOM = 7
    INTERNAL = 8


class FitConfigC(C.Structure):
    _fields_ = [
        ("beta", C.c_double),
        ("rank", C.c_uint64),
        ("ranks", C.POINTER(C.c_uint64)),
        ("n_ranks", C.c_uint32),
        ("eps", C.c_double),
        ("inner_steps", C.c_uint64),
        ("max_iters", C.c_uint64),
        ("tol", C.c_double),
        ("seed", C.c_uint64),
        ("extrapolate", C.c_int32),
        ("extrap_cap", C.c_double),
        ("extrap_delta", C.c_double),
        ("has_data_floor", C.c_int32),
        ("data_floor", C.c_double),
        ("precision", C.c_int32),
        ("use_graphs", C.c_int32),
    ]


class TraceRowC(C.Structure):
    _fields_ = [("iter", C.c_uint64), ("time_s", C.c_double), ("loss", C.c_double)]


class ShardC(C.Structure):
    _fields_ = [("global_dim0", C.c_uint64), ("slab_begin", C.c_uint64)]


class StatsC(C.Structure):
    _fields_ = [("kernel_launches", C.c_uint64), ("graph_launches", C.c_uint64),
                ("device_ms", C.c_double), ("recon_ms", C.c_double), ("recon_launches", C.c_uint64),
                ("contract_ms", C.c_double), ("contract_launches", C.c_uint64),
                ("other_ms", C.c_double), ("other_launches", C.c_uint64)]


ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_double), C.c_size_t, C.c_void_p)

_P = C.POINTER(C.c_double)
_U = C.POINTER(C.c_uint64)
_V = C.c_void_p

# name -> argtypes (restype is always ntfg_status == int)
_SIGS = {
    "ntfg_context_create": [C.c_int, C.POINTER(C.c_void_p)],
    "ntfg_context_destroy": [_V],
    "ntfg_context_set_stream": [_V, _V],
    "ntfg_context_set_allreduce": [_V, ALLREDUCE_FN, _V],
    "ntfg_context_stats": [_V, C.POINTER(StatsC)],
    "ntfg_context_trim": [_V],
    "ntfg_context_set_profiling": [_V, C.c_int],
    "ntfg_context_set_comm_buffer": [_V, _V, C.c_size_t],
    "ntfg_nccl_unique_id": [_V],
    "ntfg_context_init_nccl": [_V, _V, C.c_int32, C.c_int32],
    "ntfg_validate_fit_config": [C.POINTER(FitConfigC)],
    "ntfg_cp_fit": [_V, C.POINTER(FitConfigC), C.c_int32, C.c_uint32, _U, _V, C.c_int32, C.c_int32,
                    C.POINTER(ShardC), _P, C.POINTER(TraceRowC), _U],
    "ntfg_cp_fit_coo": [_V, C.POINTER(FitConfigC), C.c_int32, C.c_uint32, _U, C.c_uint64, _V, _V, C.c_int32,
                        C.c_int32, C.POINTER(ShardC), _P, C.POINTER(TraceRowC), _U],
    "ntfg_cp_mu_unfold_fit": [_V, C.POINTER(FitConfigC), C.c_uint32, _U, _V, C.c_int32, C.c_int32, _P,
                              C.POINTER(TraceRowC), _U],
    "ntfg_cp_mu_unfold_sweep": [_V, C.c_int32, C.c_double, C.c_double, C.c_uint32, _U, _P, C.c_uint64, _P],
    "ntfg_tucker_mu_unfold_fit": [_V, C.POINTER(FitConfigC), C.c_uint32, _U, _V, C.c_int32, C.c_int32, _P, _P,
                                  C.POINTER(TraceRowC), _U],
    "ntfg_tucker_mu_unfold_sweep": [_V, C.c_int32, C.c_double, C.c_double, C.c_uint32, _U, _U, _P, _P, _P],
    "ntfg_ctf1_header": [C.c_char_p, C.POINTER(C.c_uint32), _U, C.c_uint32, C.c_uint64],
    "ntfg_ctf1_read": [_V, C.c_char_p, _V, C.c_int32, C.c_int32, C.c_uint64],
    "ntfg_ctf1_write": [_V, C.c_char_p, C.c_uint32, _U, _V, C.c_int32, C.c_int32],
    "ntfg_coo_text_read": [C.c_char_p, C.POINTER(C.c_uint32), _U, C.c_uint32, _U, _V, _P, C.c_uint64,
                           C.c_uint64],
    "ntfg_trace_write": [C.c_char_p, C.POINTER(TraceRowC), C.c_uint64],
    "ntfg_philox_uniforms": [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, _P],
    "ntfg_cp_factors_generate": [C.c_uint32, _U, C.c_uint64, C.c_uint64, C.c_int32, C.c_double, _P],
    "ntfg_generate_cp_gamma": [_V, C.c_uint32, _U, C.c_uint64, C.c_uint64, C.c_uint32, C.c_double, C.c_uint64,
                               C.c_uint64, _V, C.c_int32],
    "ntfg_tucker_fit": [_V, C.POINTER(FitConfigC), C.c_int32, C.c_uint32, _U, _V, C.c_int32, C.c_int32,
                        C.POINTER(ShardC), _P, _P, C.POINTER(TraceRowC), _U],
    "ntfg_cp_reconstruct": [_V, C.c_int32, C.c_uint32, _U, C.c_uint64, _P, _P],
    "ntfg_cp_contract": [_V, C.c_int32, C.c_uint32, _U, _P, C.c_uint64, _P, C.c_uint32, _P],
    "ntfg_cp_objective": [_V, C.c_int32, C.c_double, C.c_uint32, _U, _P, C.c_uint64, _P, _P],
    "ntfg_cp_block_update": [_V, C.c_int32, C.c_double, C.c_double, C.c_uint32, _U, _P, C.c_uint64, _P,
                             C.c_uint32, _P],
    "ntfg_cp_bcomm_sweep": [_V, C.c_int32, C.c_double, C.c_double, C.c_uint32, _U, _P, C.c_uint64, _P],
    "ntfg_cp_jcomm_reference": [_V, C.c_int32, C.c_double, C.c_double, C.c_uint32, _U, _P, C.c_uint64,
                                _P, _P, _P],
    "ntfg_cp_jcomm_inner_update": [_V, C.c_int32, C.c_double, C.c_double, C.c_uint32, _U, _P, _P,
                                   C.c_uint64, _P, _P, C.c_uint32],
    "ntfg_cp_jcomm_outer_step": [_V, C.c_int32, C.c_double, C.c_double, C.c_uint64, C.c_uint32, _U, _P,
                                 C.c_uint64, _P],
    "ntfg_D_beta": [_V, C.c_double, C.c_uint64, _P, _P, _P],
    "ntfg_tucker_reconstruct": [_V, C.c_int32, C.c_uint32, _U, _U, _P, _P, _P],
    "ntfg_tucker_multimode_contract": [_V, C.c_int32, C.c_uint32, _U, _P, _U, _P, C.c_int32, _P],
    "ntfg_tucker_factor_contract": [_V, C.c_int32, C.c_uint32, _U, _P, _U, _P, _P, C.c_uint32, _P],
    "ntfg_tucker_objective": [_V, C.c_int32, C.c_double, C.c_uint32, _U, _P, _U, _P, _P, _P],
    "ntfg_tucker_jcomm_reference": [_V, C.c_int32, C.c_double, C.c_double, C.c_uint32, _U, _P, _U, _P, _P,
                                    _P, _P],
    "ntfg_tucker_jcomm_inner_update": [_V, C.c_int32, C.c_double, C.c_double, C.c_uint32, _U, _P, _P, _U, _P,
                                       _P, _P, _P, C.c_int32],
    "ntfg_tucker_step": [_V, C.c_int32, C.c_int32, C.c_double, C.c_double, C.c_uint64, C.c_uint32, _U,
                         _P, _U, _P, _P, _P, _P, C.c_uint32],
}

EXPORTED = ["ntfg_abi_version", "ntfg_last_error"] + list(_SIGS)

_lib = None
_lock = threading.Lock()


def load(path: str = LIB_PATH):
    """Load and type the library (no GPU needed); raises if it was not built."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(path):
                raise RuntimeError(
                    f"libntfg.so not found at {path}: build it with "
                    "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback exists)")
            lib = C.CDLL(path)
            lib.ntfg_abi_version.restype = C.c_int
            lib.ntfg_last_error.restype = C.c_char_p
            for name, args in _SIGS.items():
                fn = getattr(lib, name)
                fn.argtypes = args
                fn.restype = C.c_int
            _lib = lib
    return _lib


def last_error() -> str:
    return load().ntfg_last_error().decode(errors="replace")
