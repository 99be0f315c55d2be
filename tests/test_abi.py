"""CPU checks of the drop-in boundary: libntfg.so loads without a GPU, exports
every entry point include/ntfg.h declares, validates configs on the host,
and the Python layer fails loudly (no CPU fallback) when no device exists."""
import os
import re

import numpy as np
import pytest

import paper_2602_14683_b200 as ntf
from paper_2602_14683_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared():
    src = open(os.path.join(ROOT, "include", "ntfg.h")).read()
    return sorted(set(re.findall(r"\b(ntfg_[A-Za-z0-9_]+)\s*\(", src)) - {"ntfg_allreduce_fn"})


def test_header_declarations_are_exported():
    lib = _native.load()
    names = declared()
    assert len(names) >= 25
    for n in names:
        assert hasattr(lib, n), n
    assert set(_native.EXPORTED) <= set(names) | {"ntfg_abi_version", "ntfg_last_error"}


def test_abi_version():
    assert _native.load().ntfg_abi_version() == 1


def test_config_validation_on_host():
    ntf.validate_fit_config(ntf.FitConfig(beta=1.5, rank=3))
    for bad in [dict(beta=2.0), dict(beta=-0.1), dict(eps=0.0), dict(inner_steps=0), dict(rank=0),
                dict(ranks=[2, 0]), dict(data_floor=0.0), dict(extrap_cap=-1.0), dict(extrap_delta=0.0)]:
        with pytest.raises(ntf.DomainError):
            ntf.validate_fit_config(ntf.FitConfig(**bad))


def test_no_silent_cpu_fallback_without_gpu():
    from tests.conftest import HAS_GPU
    if HAS_GPU:
        pytest.skip("device present")
    with pytest.raises(ntf.CudaError):
        ntf.Context(0)
    with pytest.raises(ntf.NtfError):
        ntf.bcomm_fit(np.ones((2, 2)), [np.ones((2, 1)), np.ones((2, 1))], ntf.FitConfig(max_iters=1))
