"""B200-native contraction-only beta-divergence MU engine (CP / Tucker, B-CoMM / J-CoMM).

The compute path is libntfg.so (hand-written sm_100a CUDA kernels behind the C
ABI in include/ntfg.h); this package is the Python mirror of the reference's
``ntf`` solver API on top of it.  See DESIGN.md.
"""
from .api import (  # noqa: F401
    CommError, Context, CpFitResult, CudaError, D_beta, D_beta_mean, DomainError, FitConfig,
    FormatError, JcommCpReference, JcommTuckerReference, NtfError, NumericalError, ShapeError,
    TraceRecord, TuckerFitResult, bcomm_block_update, bcomm_fit, bcomm_fit_coo, bcomm_sweep, block_core_update,
    block_factor_update, cp_block_update_anchored, cp_contract, cp_objective, cp_reconstruct,
    default_context, jcomm_fit, jcomm_fit_coo, jcomm_inner_core_update, jcomm_inner_factor_update,
    jcomm_inner_update, jcomm_outer_step, jcomm_tucker_outer_step, make_jcomm_reference,
    make_jcomm_tucker_reference, mu_unfold_cp_fit, mu_unfold_cp_sweep, mu_unfold_tucker_fit, mu_unfold_tucker_sweep, tucker_bcomm_fit, tucker_bcomm_sweep, tucker_factor_contract,
    tucker_jcomm_fit, tucker_multimode_contract, tucker_objective, tucker_reconstruct,
    nccl_unique_id, validate_fit_config, ExtrapolationState, make_extrapolation_state,
    make_tucker_extrapolation_state, extrapolation_begin_iteration, extrapolate_block, extrapolate_core,
    extrapolation_end_iteration)

__version__ = "0.1.0"
