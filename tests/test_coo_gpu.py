"""Sparse COO path at beta = 1 (coo_kernels.cuh, K7): parity with the dense
fits of the densified tensor (oracle and GPU), duplicate accumulation, the
piece/segment machinery on Zipf-skewed modes, and the error contract.
SURVEY.md 8(c) "Sparse path": pinned by densifying small instances."""
import numpy as np
import pytest

import paper_2602_14683_b200 as ntf
from oracle import ntf_oracle as O

pytestmark = pytest.mark.gpu


def relm(a, b):
    return max(O.rel_err(u, v) for u, v in zip(a, b))


def init_for(dims, rank, seed):
    rng = np.random.default_rng(seed)
    return [0.1 + rng.random((d, rank)) for d in dims]


@pytest.mark.parametrize("algo", ["bcomm", "jcomm"])
@pytest.mark.parametrize("dims,nnz,rank", [((6, 5, 7), 60, 3), ((5, 4, 6, 3), 150, 4), ((9, 7), 20, 2)])
def test_coo_matches_dense_oracle(algo, dims, nnz, rank):
    idx, vals = O.coo_synthetic(dims, nnz, seed=1)
    x = O.coo_densify(idx, vals, dims)
    init = init_for(dims, rank, 2)
    cfg = ntf.FitConfig(beta=1.0, rank=rank, max_iters=15, inner_steps=3, precision="f64")
    fit = ntf.bcomm_fit_coo if algo == "bcomm" else ntf.jcomm_fit_coo
    res = fit(idx, vals, dims, init, cfg)
    ofit = O.bcomm_fit if algo == "bcomm" else O.jcomm_fit
    om, otr = ofit(x, init, O.FitConfig(beta=1.0, rank=rank, max_iters=15, inner_steps=3))
    assert relm(res.model, om) < 1e-9
    assert O.rel_err([t.loss for t in res.trace], [t[2] for t in otr]) < 1e-10


@pytest.mark.parametrize("algo", ["bcomm", "jcomm"])
def test_coo_zipf_matches_gpu_dense(algo):
    # heavy keys (> 256 nonzeros) exercise multi-piece segments
    dims = (30, 8, 120, 90)
    idx, vals = O.coo_synthetic(dims, 40000, seed=3, zipf_modes=(2, 3))
    counts = np.bincount(idx[:, 2], minlength=dims[2])
    assert counts.max() > 1000
    x = O.coo_densify(idx, vals, dims)
    init = init_for(dims, 6, 4)
    cfg = ntf.FitConfig(beta=1.0, rank=6, max_iters=10, inner_steps=3, precision="f64")
    fit_s = ntf.bcomm_fit_coo if algo == "bcomm" else ntf.jcomm_fit_coo
    fit_d = ntf.bcomm_fit if algo == "bcomm" else ntf.jcomm_fit
    a = fit_s(idx, vals, dims, init, cfg)
    b = fit_d(x, init, cfg)
    assert relm(a.model, b.model) < 1e-9
    assert O.rel_err([t.loss for t in a.trace], [t.loss for t in b.trace]) < 1e-10


def test_coo_rank_over_32_and_extrapolation():
    dims = (12, 10, 9)
    idx, vals = O.coo_synthetic(dims, 500, seed=5)
    x = O.coo_densify(idx, vals, dims)
    init = init_for(dims, 40, 6)
    cfg = ntf.FitConfig(beta=1.0, rank=40, max_iters=8, inner_steps=2, precision="f64", extrapolate=True)
    a = ntf.jcomm_fit_coo(idx, vals, dims, init, cfg)
    b = ntf.jcomm_fit(x, init, cfg)
    assert relm(a.model, b.model) < 1e-9
    assert O.rel_err([t.loss for t in a.trace], [t.loss for t in b.trace]) < 1e-10


def test_coo_duplicates_accumulate_in_order():
    dims = (4, 3, 5)
    idx, vals = O.coo_synthetic(dims, 40, seed=7)
    # same nonzeros, merged by hand in input order
    lin = np.ravel_multi_index(tuple(idx.T.astype(np.int64)), dims)
    merged = {}
    for j, v in zip(lin.tolist(), vals.tolist()):
        merged[j] = merged.get(j, 0.0) + v
    keys = sorted(merged)
    midx = np.array(np.unravel_index(keys, dims)).T.astype(np.int32)
    mval = np.array([merged[k] for k in keys])
    init = init_for(dims, 3, 8)
    cfg = ntf.FitConfig(beta=1.0, rank=3, max_iters=6, inner_steps=2, precision="f64")
    a = ntf.jcomm_fit_coo(idx, vals, dims, init, cfg)
    b = ntf.jcomm_fit_coo(midx[::-1].copy(), mval[::-1].copy(), dims, init, cfg)
    for u, v in zip(a.model, b.model):
        assert np.array_equal(u, v)
    assert [t.loss for t in a.trace] == [t.loss for t in b.trace]


def test_coo_device_inputs_match_host():
    import torch
    dims = (7, 6, 5)
    idx, vals = O.coo_synthetic(dims, 90, seed=9)
    init = init_for(dims, 4, 10)
    cfg = ntf.FitConfig(beta=1.0, rank=4, max_iters=5, inner_steps=2, precision="f64")
    a = ntf.jcomm_fit_coo(idx, vals, dims, init, cfg)
    b = ntf.jcomm_fit_coo(torch.from_numpy(idx).cuda(), torch.from_numpy(vals).float().cuda(), dims, init, cfg)
    assert relm(a.model, b.model) < 1e-12  # integer counts: fp32 values are exact


def test_coo_errors():
    dims = (4, 4, 4)
    idx, vals = O.coo_synthetic(dims, 10, seed=11)
    init = init_for(dims, 2, 12)
    with pytest.raises(ntf.DomainError):
        ntf.jcomm_fit_coo(idx, vals, dims, init, ntf.FitConfig(beta=0.5, rank=2, max_iters=2))
    bad = idx.copy()
    bad[0, 1] = 4
    with pytest.raises(ntf.ShapeError):
        ntf.jcomm_fit_coo(bad, vals, dims, init, ntf.FitConfig(beta=1.0, rank=2, max_iters=2))
    neg = vals.copy()
    neg[3] = -1.0
    with pytest.raises(ntf.DomainError):
        ntf.jcomm_fit_coo(idx, neg, dims, init, ntf.FitConfig(beta=1.0, rank=2, max_iters=2))
