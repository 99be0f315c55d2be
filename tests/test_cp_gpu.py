"""CP parity tests: CUDA path (libntfg.so via the C ABI) vs the CPU oracle.

Mirrors the reference's own suites (tests/test_cp.cpp, test_tensor.cpp,
test_divergence.cpp) with the oracle (oracle/ntf_oracle.py, pinned to the
compiled reference in tests/test_oracle_pins.py) as the checker.
Tolerances: fp64 validation build 1e-10 (factors and trace, rel_err of
test_support.hpp:17-19); fp32 build 1e-4 factors / 1e-5 trace (north star).
"""
import numpy as np
import pytest

import paper_2602_14683_b200 as ntf
from oracle import ntf_oracle as O

pytestmark = pytest.mark.gpu
EPS = 1e-12
BETAS = [0.0, 0.5, 1.0, 1.5, 0.7]


def relerr_model(a, b):
    return max(O.rel_err(x, y) for x, y in zip(a, b))


def data(dims, seed):
    return O.random_tensor(dims, seed)


# ---- known answers (reference test_cp.cpp:22-58, test_tensor.cpp:108-125) -----

def test_cp_reconstruct_kat():
    ones = [np.ones((2, 3)), np.ones((2, 3))]
    assert np.all(ntf.cp_reconstruct(ones) == 3.0)
    r1 = [np.array([[1.0], [2.0]]), np.array([[3.0], [4.0]])]
    assert ntf.cp_reconstruct(r1).ravel().tolist() == [3.0, 4.0, 6.0, 8.0]
    f = O.random_cp_factors([4, 3, 2], 3, O.Rng(0, O.Rng.DATA), EPS)
    assert O.rel_err(ntf.cp_reconstruct(f), O.cp_reconstruct(f)) < 1e-14


def test_cp_contract_kat():
    t = np.arange(1, 9, dtype=np.float64).reshape(2, 2, 2)
    m = ntf.cp_contract(t, [np.zeros((2, 1)), np.ones((2, 1)), np.ones((2, 1))], 0)
    assert m[:, 0].tolist() == [10.0, 26.0]
    m3 = ntf.cp_contract(t, [np.zeros((2, 3)), np.ones((2, 3)), np.ones((2, 3))], 0)
    assert np.all(m3[0] == 10.0) and np.all(m3[1] == 26.0)
    with pytest.raises(ntf.ShapeError):
        ntf.cp_contract(t, [np.zeros((2, 1)), np.ones((2, 2)), np.ones((2, 1))], 0)


@pytest.mark.parametrize("order", [1, 2, 3, 4])
@pytest.mark.parametrize("rank", [1, 3, 10, 33])
def test_cp_contract_vs_oracle(order, rank):
    rng = np.random.default_rng(order * 100 + rank)
    dims = [int(d) for d in rng.integers(1, 7, size=order)]
    t = rng.random(dims)
    fs = [rng.random((d, rank)) + 0.05 for d in dims]
    for mode in range(order):
        got = ntf.cp_contract(t, fs, mode)
        assert O.rel_err(got, O.cp_contract(t, fs, mode)) < 1e-12


def test_block_update_scalar_problem():
    x = np.array([[2.0]])
    g = ntf.bcomm_block_update([np.ones((1, 1)), np.ones((1, 1))], 0, x, 1.0, EPS)
    assert g[0][0, 0] == 2.0
    assert ntf.cp_objective(x, g, 1.0) == 0.0


def test_block_update_fixed_point():
    x = np.array([[2.0]])
    g = ntf.bcomm_block_update([np.full((1, 1), 2.0), np.ones((1, 1))], 0, x, 1.0, EPS)
    assert g[0][0, 0] == 2.0
    xs, truth = O.synth_cp([4, 3, 2], 2, 5)
    for b in [0.5, 1.0, 1.5]:
        h = [a.copy() for a in truth]
        for n in range(3):
            h = ntf.bcomm_block_update(h, n, xs, b, EPS)
        assert relerr_model(h, truth) < 1e-13


# ---- single steps vs oracle ---------------------------------------------------------

@pytest.mark.parametrize("beta", BETAS)
@pytest.mark.parametrize("dims,rank", [((6,), 2), ((7, 5), 3), ((6, 5, 4), 2), ((5, 4, 3, 6), 4),
                                       ((20, 18, 16), 10), ((9, 11, 130), 17), ((3, 4, 5, 6, 2), 5)])
def test_block_update_vs_oracle(beta, dims, rank):
    x = data(list(dims), 11)
    f = O.init_cp_factors(list(dims), rank, 11, EPS)
    for mode in range(len(dims)):
        got = ntf.bcomm_block_update(f, mode, x, beta, EPS)
        want = O.bcomm_block_update(f, mode, x, beta, EPS)
        assert relerr_model(got, want) < 1e-12, (mode, relerr_model(got, want))


@pytest.mark.parametrize("beta", [0.0, 0.5, 1.0, 1.5])
@pytest.mark.parametrize("dims", [(7, 5), (6, 5, 4), (5, 4, 3, 6)])
@pytest.mark.parametrize("precision", ["f64", "f32"])
def test_first_joint_inner_equals_block_update_bitwise(beta, dims, precision):
    """reference test_cp.cpp:116-128 (bitwise in both builds: same kernels, same order)."""
    x = data(list(dims), 3)
    f = O.init_cp_factors(list(dims), 2, 3, EPS)
    ctx = ntf.make_jcomm_reference(f, x, beta, EPS, precision=precision)
    joint = ntf.jcomm_inner_update(f, ctx, 0, beta, EPS, precision=precision)
    block = ntf.bcomm_block_update(f, 0, x, beta, EPS, precision=precision)
    assert np.array_equal(joint[0], block[0])


@pytest.mark.parametrize("beta", BETAS)
def test_jcomm_reference_and_inner_update_vs_oracle(beta):
    dims = [6, 5, 4]
    x = data(dims, 8)
    ref = O.init_cp_factors(dims, 3, 8, EPS)
    ctx = ntf.make_jcomm_reference(ref, x, beta, EPS)
    o_ref, o_p, o_q = O.make_jcomm_reference(ref, x, beta, EPS)
    assert O.rel_err(ctx.p, o_p) < 1e-14 and O.rel_err(ctx.q, o_q) < 1e-14
    rng = O.Rng(30, O.Rng.DATA)
    cur = [a * (1.0 + 0.2 * rng.uniforms(a.size).reshape(a.shape)) for a in ref]
    for mode in range(3):
        got = ntf.jcomm_inner_update(cur, ctx, mode, beta, EPS)
        want = O.jcomm_inner_update(cur, (o_ref, o_p, o_q), mode, beta, EPS)
        assert relerr_model(got, want) < 1e-12


@pytest.mark.parametrize("beta", BETAS)
def test_jcomm_outer_step_vs_oracle(beta):
    dims = [8, 7, 6]
    x = data(dims, 19)
    f = O.init_cp_factors(dims, 3, 19, EPS)
    got = ntf.jcomm_outer_step(f, x, beta, 3, EPS)
    want = O.jcomm_outer_step(f, x, beta, 3, EPS)
    assert relerr_model(got, want) < 1e-12


# ---- fits ----------------------------------------------------------------------------

@pytest.mark.parametrize("algo", ["bcomm", "jcomm"])
@pytest.mark.parametrize("beta", BETAS)
def test_fit_f64_matches_oracle(algo, beta):
    dims = [12, 10, 9]
    x = data(dims, 4)
    init = O.init_cp_factors(dims, 3, 4, EPS)
    cfg = ntf.FitConfig(beta=beta, rank=3, max_iters=40, inner_steps=3)
    res = (ntf.bcomm_fit if algo == "bcomm" else ntf.jcomm_fit)(x, init, cfg)
    om, otr = (O.bcomm_fit if algo == "bcomm" else O.jcomm_fit)(x, init, O.FitConfig(beta=beta, rank=3, max_iters=40))
    assert len(res.trace) == 41
    assert relerr_model(res.model, om) < 1e-10
    assert O.rel_err([t.loss for t in res.trace], [t[2] for t in otr]) < 1e-10
    losses = [t.loss for t in res.trace]
    for a, b in zip(losses, losses[1:]):
        assert b <= a + 1e-12 * (1 + abs(a))
    times = [t.time_s for t in res.trace]
    assert times[0] == 0.0 and all(b >= a for a, b in zip(times, times[1:]))


@pytest.mark.parametrize("algo", ["bcomm", "jcomm"])
@pytest.mark.parametrize("beta", [0.0, 0.5, 1.0, 1.5])
def test_fit_f32_matches_oracle(algo, beta):
    dims = [24, 20, 16]
    rng = np.random.default_rng(7)
    truth = [rng.random((d, 4)) for d in dims]
    x = O.cp_reconstruct(truth) * rng.gamma(10.0, 0.1, size=dims)
    init = [0.1 + rng.random((d, 4)) for d in dims]
    cfg = ntf.FitConfig(beta=beta, rank=4, max_iters=30, inner_steps=5, precision="f32")
    res = (ntf.bcomm_fit if algo == "bcomm" else ntf.jcomm_fit)(x, init, cfg)
    ocfg = O.FitConfig(beta=beta, rank=4, max_iters=30, inner_steps=5)
    om, otr = (O.bcomm_fit if algo == "bcomm" else O.jcomm_fit)(x, init, ocfg)
    assert relerr_model(res.model, om) < 1e-4
    assert O.rel_err([t.loss for t in res.trace], [t[2] for t in otr]) < 1e-5


def test_graphs_and_eager_agree_bitwise():
    dims = [10, 9, 8]
    x = data(dims, 2)
    init = O.init_cp_factors(dims, 3, 2, EPS)
    a = ntf.jcomm_fit(x, init, ntf.FitConfig(beta=0.5, rank=3, max_iters=10, use_graphs=True))
    b = ntf.jcomm_fit(x, init, ntf.FitConfig(beta=0.5, rank=3, max_iters=10, use_graphs=False))
    for u, v in zip(a.model, b.model):
        assert np.array_equal(u, v)
    assert [t.loss for t in a.trace] == [t.loss for t in b.trace]


def test_stopping_rules():
    """reference test_cp.cpp:88-104, 149-157."""
    x, _ = O.synth_cp([4, 3, 2], 2, 1)
    init = O.init_cp_factors([4, 3, 2], 2, 1, EPS)
    r0 = ntf.bcomm_fit(x, init, ntf.FitConfig(beta=1.0, rank=2, max_iters=0))
    assert len(r0.trace) == 1 and r0.trace[0].iter == 0
    assert relerr_model(r0.model, init) == 0.0
    r1 = ntf.bcomm_fit(x, init, ntf.FitConfig(beta=1.0, rank=2, max_iters=50, tol=float("inf")))
    assert len(r1.trace) == 2
    j0 = ntf.jcomm_fit(x, init, ntf.FitConfig(rank=2, max_iters=0))
    assert len(j0.trace) == 1 and relerr_model(j0.model, init) == 0.0


@pytest.mark.parametrize("algo", ["bcomm", "jcomm"])
def test_tol_stop_matches_oracle(algo):
    dims = [8, 7, 6]
    x = data(dims, 5)
    init = O.init_cp_factors(dims, 2, 5, EPS)
    cfg = ntf.FitConfig(beta=1.5, rank=2, max_iters=200, tol=1e-4)
    res = (ntf.bcomm_fit if algo == "bcomm" else ntf.jcomm_fit)(x, init, cfg)
    om, otr = (O.bcomm_fit if algo == "bcomm" else O.jcomm_fit)(x, init, O.FitConfig(beta=1.5, rank=2, max_iters=200, tol=1e-4))
    assert len(res.trace) == len(otr)
    assert relerr_model(res.model, om) < 1e-10


def test_beta0_zero_data_names_data_floor():
    x = data([4, 3, 2], 1)
    x[0, 0, 0] = 0.0
    init = O.init_cp_factors([4, 3, 2], 2, 1, EPS)
    with pytest.raises(ntf.NumericalError, match="data-floor"):
        ntf.bcomm_fit(x, init, ntf.FitConfig(beta=0.0, rank=2, max_iters=3))


def test_config_validation():
    with pytest.raises(ntf.DomainError):
        ntf.validate_fit_config(ntf.FitConfig(beta=2.0))
    with pytest.raises(ntf.DomainError):
        ntf.validate_fit_config(ntf.FitConfig(eps=0.0))
    with pytest.raises(ntf.DomainError):
        ntf.validate_fit_config(ntf.FitConfig(inner_steps=0))
    x = data([4, 3, 2], 1)
    with pytest.raises(ntf.ShapeError):
        ntf.bcomm_fit(x, [np.ones((4, 2)), np.ones((3, 2))], ntf.FitConfig(rank=2, max_iters=1))


@pytest.mark.parametrize("algo", ["bcomm", "jcomm"])
def test_zero_cap_extrapolation_is_plain_path_bitwise(algo):
    """reference test_cp.cpp:218-234."""
    x, _ = O.synth_cp([6, 5, 4], 2, 4)
    init = O.init_cp_factors([6, 5, 4], 2, 4, EPS)
    plain = ntf.FitConfig(beta=1.5, rank=2, max_iters=20)
    capped = ntf.FitConfig(beta=1.5, rank=2, max_iters=20, extrapolate=True, extrap_cap=0.0)
    fit = ntf.bcomm_fit if algo == "bcomm" else ntf.jcomm_fit
    a = fit(x, init, plain)
    b = fit(x, init, capped)
    for u, v in zip(a.model, b.model):
        assert np.array_equal(u, v)
    assert [t.loss for t in a.trace] == [t.loss for t in b.trace]


@pytest.mark.parametrize("algo", ["bcomm", "jcomm"])
@pytest.mark.parametrize("beta", [0.5, 1.0])
def test_extrapolated_fit_matches_oracle(algo, beta):
    dims = [8, 7, 6]
    x = data(dims, 12)
    init = O.init_cp_factors(dims, 2, 12, EPS)
    cfg = ntf.FitConfig(beta=beta, rank=2, max_iters=25, extrapolate=True)
    res = (ntf.bcomm_fit if algo == "bcomm" else ntf.jcomm_fit)(x, init, cfg)
    om, otr = (O.bcomm_fit if algo == "bcomm" else O.jcomm_fit)(
        x, init, O.FitConfig(beta=beta, rank=2, max_iters=25, extrapolate=True))
    assert relerr_model(res.model, om) < 1e-10
    assert O.rel_err([t.loss for t in res.trace], [t[2] for t in otr]) < 1e-10


def test_D_beta_kats():
    """reference test_divergence.cpp:22-35, 79-87."""
    assert abs(ntf.D_beta([4.0], [1.0], 0.5) - 2.0) < 1e-14
    assert abs(ntf.D_beta([2.0], [1.0], 1.0) - (2 * np.log(2.0) - 1)) < 1e-14
    assert np.isinf(ntf.D_beta([0.0], [1.0], 0.0))
    assert ntf.D_beta([0.0], [1.5], 1.0) == 1.5
    with pytest.raises(ntf.DomainError):
        ntf.D_beta([1.0], [0.0], 1.0)
    x = np.full((2, 2), 2.0)
    assert abs(ntf.D_beta(x, np.ones((2, 2)), 1.0) - 4 * (2 * np.log(2.0) - 1)) < 1e-14
