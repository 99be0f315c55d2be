"""MU-unfold baseline on the GPU (unfold_api.cu; reference unfold.cpp:109-197):
against the compiled reference's matricized sweep, and acceptance criterion 2
(acceptance.cpp:104-132): 20 unfold sweeps == 20 contraction sweeps to 1e-10."""
import numpy as np
import pytest

import paper_2602_14683_b200 as ntf
from oracle import ntf_oracle as O
from oracle import ref as R

pytestmark = pytest.mark.gpu
EPS = 1e-12


def relm(a, b):
    return max(O.rel_err(u, v) for u, v in zip(a, b))


def problem(dims, rank, seed):
    rng = np.random.default_rng(seed)
    truth = [rng.random((d, rank)) for d in dims]
    x = O.cp_reconstruct(truth) * rng.gamma(10.0, 0.1, size=dims)
    return x, [0.1 + rng.random((d, rank)) for d in dims]


@pytest.mark.skipif(not R.available(), reason="compiled reference (oracle/_ref) not built")
@pytest.mark.parametrize("beta", [0.0, 0.5, 1.0, 1.5, 1.2])
@pytest.mark.parametrize("dims,rank", [((6, 5, 4), 2), ((5, 4, 3, 6), 3)])
def test_unfold_sweep_matches_compiled_reference(beta, dims, rank):
    x, f = problem(dims, rank, 1)
    got = ntf.mu_unfold_cp_sweep(f, x, beta, EPS)
    want = R.mu_unfold_cp_sweep(x, f, beta, EPS)
    assert relm(got, want) < 1e-12


@pytest.mark.parametrize("beta", [0.5, 1.0, 1.5])
def test_criterion2_unfold_equals_contraction(beta):
    x, _ = problem((6, 5, 4), 2, 0)
    a = [0.1 + np.random.default_rng(3).random((d, 2)) for d in (6, 5, 4)]
    b = [m.copy() for m in a]
    worst = 0.0
    for _ in range(20):
        a = ntf.bcomm_sweep(a, x, beta, EPS)
        b = ntf.mu_unfold_cp_sweep(b, x, beta, EPS)
        worst = max(worst, relm(a, b))
    assert worst <= 1e-10


@pytest.mark.parametrize("beta", [0.5, 1.0])
def test_unfold_fit_matches_bcomm_fit(beta):
    x, init = problem((16, 12, 10), 4, 2)
    cfg = ntf.FitConfig(beta=beta, rank=4, max_iters=15, precision="f64")
    a = ntf.mu_unfold_cp_fit(x, init, cfg)
    b = ntf.bcomm_fit(x, init, cfg)
    assert relm(a.model, b.model) < 1e-10
    assert O.rel_err([t.loss for t in a.trace], [t.loss for t in b.trace]) < 1e-10
    assert len(a.trace) == 16


def test_unfold_fit_fp32():
    x, init = problem((24, 16, 128), 8, 4)
    a = ntf.mu_unfold_cp_fit(x, init, ntf.FitConfig(beta=0.5, rank=8, max_iters=10, precision="f32"))
    b = ntf.mu_unfold_cp_fit(x, init, ntf.FitConfig(beta=0.5, rank=8, max_iters=10, precision="f64"))
    assert relm(a.model, b.model) < 1e-4
    assert O.rel_err([t.loss for t in a.trace], [t.loss for t in b.trace]) < 1e-5


# ---- Tucker MU-unfold (reference unfold.cpp:137-185) ---------------------------------

def tucker_problem(dims, ranks, seed):
    rng = np.random.default_rng(seed)
    core = rng.random(ranks)
    fs = [rng.random((d, j)) for d, j in zip(dims, ranks)]
    x = O.tucker_reconstruct(core, fs) * rng.gamma(10.0, 0.1, size=dims)
    init = (0.1 + rng.random(ranks), [0.1 + rng.random((d, j)) for d, j in zip(dims, ranks)])
    return x, init


@pytest.mark.parametrize("beta", [0.0, 0.5, 1.0, 1.5])
@pytest.mark.parametrize("dims,ranks", [((9, 7, 6), (3, 2, 4)), ((5, 4, 6, 3), (2, 3, 2, 2))])
def test_mu_unfold_tucker_sweep_equals_block_sweep(beta, dims, ranks):
    # the matricized sweep is the same MM map as the contraction-based block
    # sweep (core first, then factors ascending), up to summation order
    x, (core, fs) = tucker_problem(dims, ranks, 3)
    c1, f1 = ntf.mu_unfold_tucker_sweep(core, fs, x, beta, EPS)
    oc, of = O.tucker_bcomm_sweep((core, fs), x, beta, EPS)
    assert O.rel_err(c1, oc) < 1e-11
    assert max(O.rel_err(a, b) for a, b in zip(f1, of)) < 1e-11


@pytest.mark.parametrize("beta", [0.5, 1.0])
def test_mu_unfold_tucker_fit_matches_bcomm(beta):
    x, init = tucker_problem((10, 8, 6), (3, 3, 2), 5)
    cfg = ntf.FitConfig(beta=beta, rank=1, ranks=[3, 3, 2], max_iters=12)
    a = ntf.mu_unfold_tucker_fit(x, init, cfg)
    b = ntf.tucker_bcomm_fit(x, init, cfg)
    assert O.rel_err([t.loss for t in a.trace], [t.loss for t in b.trace]) < 1e-10
    assert O.rel_err(a.model[0], b.model[0]) < 1e-10
    f32 = ntf.mu_unfold_tucker_fit(x, init, ntf.FitConfig(beta=beta, rank=1, ranks=[3, 3, 2], max_iters=12,
                                                          precision="f32"))
    assert O.rel_err([t.loss for t in f32.trace], [t.loss for t in b.trace]) < 1e-5
