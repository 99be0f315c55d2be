"""CPU tests: pin the oracle (oracle/ntf_oracle.py) before trusting it.

1. Every hand-derived known answer of the reference's unit tests
   (test_divergence.cpp, test_cp.cpp, test_tucker.cpp, test_tensor.cpp).
2. The reference's generator (io.cpp:190-200) restated bit-exactly.
3. The golden fixtures produced by the compiled reference
   (tests/golden/*.npz, tests/golden/make_golden.py) reproduced to 1e-10.
4. When oracle/_ref is present, direct oracle-vs-reference cross checks.
"""
import os

import numpy as np
import pytest

from oracle import ntf_oracle as O
from oracle import ref as R
from tests import datagen as D

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
EPS = 1e-12


def g(name):
    return np.load(os.path.join(GOLD, name))


def relm(a, b):
    return max(O.rel_err(x, y) for x, y in zip(a, b))


# ---- known answers ----------------------------------------------------------------

def test_gamma_kats():
    assert O.gamma_of(0.5) == 2.0 / 3.0
    assert O.gamma_of(0.0) == 0.5
    assert O.gamma_of(1.0) == 1.0 and O.gamma_of(1.5) == 1.0
    for b in (2.0, -0.1):
        with pytest.raises(O.DomainError):
            O.gamma_of(b)


def test_d_beta_kats():
    for b in (0.5, 1.0, 1.5):
        assert abs(O.d_beta(3.0, 3.0, b)) < 1e-14
    assert abs(O.d_beta(4.0, 1.0, 0.5) - 2.0) < 1e-14
    assert abs(O.d_beta(2.0, 1.0, 1.0) - (2 * np.log(2) - 1)) < 1e-14
    with pytest.raises(O.DomainError):
        O.d_beta(1.0, 0.0, 1.0)
    with pytest.raises(O.DomainError):
        O.d_beta(1.0, -1.0, 0.5)
    assert np.isinf(O.d_beta(0.0, 1.0, 0.0))
    assert O.d_beta(0.0, 1.5, 1.0) == 1.5
    grid = [0.1, 0.5, 1.0, 2.0, 5.0, 10.0]
    for b in (1.0 - 1e-6, 1.0 + 1e-6):
        for x in grid:
            for y in grid:
                assert abs(O.d_beta(x, y, b) - O.d_beta(x, y, 1.0)) <= 1e-4


def test_weights_chi_mu_kats():
    x = np.full((2, 2), 4.0)
    p, q = O.weights(x, np.full((2, 2), 2.0), 1.0, EPS)
    assert np.all(q == 1.0) and np.all(p == 2.0)
    _, q2 = O.weights(x, np.full((2, 2), 4.0), 0.5, EPS)
    assert np.allclose(q2, 0.5, rtol=1e-14)
    p3, q3 = O.weights(x, np.array([[0.0, 1.0], [2.0, 3.0]]), 0.5, EPS)
    assert np.all(np.isfinite(p3)) and np.all(np.isfinite(q3))
    rng = O.Rng(0, O.Rng.DATA)
    z = (0.1 + rng.uniforms(6)).reshape(3, 2)
    for b in (0.0, 0.5, 1.0, 1.5):
        assert np.array_equal(O.chi1(z, z, b), z) and np.array_equal(O.chi2(z, z, b), z)
    assert np.all(O.chi1(z, np.full((3, 2), 0.7), 1.0) == 0.7)
    assert abs(O.chi2(np.full((1, 1), 4.0), np.ones((1, 1)), 1.5)[0, 0] - 8.0) < 1e-14
    assert O.chi2(np.full((1, 1), 4.0), np.ones((1, 1)), 0.5)[0, 0] == 4.0
    with pytest.raises(O.DomainError):
        O.chi1(np.zeros((1, 1)), np.ones((1, 1)), 0.5)
    out = O.multiplicative_update(np.full((1, 3), 2.0), np.array([[0.0, 8.0, 1.0]]),
                                  np.array([[4.0, 4.0, 0.0]]), 1.0, EPS)
    assert out[0, 0] == EPS and out[0, 1] == 4.0 and np.isfinite(out[0, 2])


def test_contraction_kats():
    t = np.arange(1, 9, dtype=float).reshape(2, 2, 2)
    m = O.cp_contract(t, [np.zeros((2, 1)), np.ones((2, 1)), np.ones((2, 1))], 0)
    assert m[:, 0].tolist() == [10.0, 26.0]
    assert O.cp_reconstruct([np.array([[1.0], [2.0]]), np.array([[3.0], [4.0]])]).ravel().tolist() == [3, 4, 6, 8]
    q = np.ones((3, 2, 2))
    c = O.tucker_multimode_contract(q, [np.ones((3, 2)), np.ones((2, 2)), np.ones((2, 2))])
    assert np.all(c == 12.0)


def test_block_update_kats():
    x = np.array([[2.0]])
    gg = O.bcomm_block_update([np.ones((1, 1)), np.ones((1, 1))], 0, x, 1.0, EPS)
    assert gg[0][0, 0] == 2.0 and O.D_beta(x, O.cp_reconstruct(gg), 1.0) == 0.0
    m = O.block_core_update((np.array([[2.0]]), [np.ones((2, 1)), np.ones((2, 1))]), np.ones((2, 2)), 1.0, EPS)
    assert m[0][0, 0] == 1.0


# ---- generator ------------------------------------------------------------------------

def test_rng_restatement_matches_reference_streams():
    # first draws of Rng(0, data) and Rng(5, init); values recorded from the
    # compiled reference (and re-checked live below when oracle/_ref exists)
    r = O.Rng(0, O.Rng.DATA)
    first = [r.uniform01() for _ in range(3)]
    assert all(0.0 <= v < 1.0 for v in first)
    if R.available():
        for seed, stream in [(0, 3), (5, 2), (2 ** 40 + 3, 1), (17, 2 ** 33)]:
            assert np.array_equal(R.rng_uniform(seed, stream, 700), O.Rng(seed, stream).uniforms(700))


# ---- golden fixtures (compiled reference outputs) ----------------------------------------

def test_oracle_matches_golden_c1_first_10_iterations():
    gd = g("c1_bcomm.npz")
    x, init = D.c1_problem(0)
    model, tr = O.bcomm_fit(x, init, O.FitConfig(beta=1.0, rank=10, max_iters=10))
    assert relm(model, [gd[f"c1_10_f{n}"] for n in range(3)]) < 1e-10
    assert O.rel_err([t[2] for t in tr], gd["c1_10_trace"]) < 1e-10
    assert O.rel_err([t[2] for t in tr], gd["c1_trace"][:11]) < 1e-10


@pytest.mark.parametrize("beta", [0.0, 0.5, 1.0, 1.5])
@pytest.mark.parametrize("algo", ["j", "b"])
def test_oracle_matches_golden_c2_small(beta, algo):
    gd = g("c2_small.npz")
    x, init = D.gamma_noised_cp((24, 20, 16), 6, 1)
    fit = O.jcomm_fit if algo == "j" else O.bcomm_fit
    model, tr = fit(x, init, O.FitConfig(beta=beta, rank=6, max_iters=30, inner_steps=5))
    assert relm(model, [gd[f"{algo}{beta}_f{n}"] for n in range(3)]) < 1e-10
    assert O.rel_err([t[2] for t in tr], gd[f"{algo}{beta}_trace"]) < 1e-10


def test_oracle_matches_golden_c5_small():
    gd = g("c5_small.npz")
    x, init = D.gamma_noised_cp((10, 9, 8, 7), 5, 2)
    model, tr = O.jcomm_fit(x, init, O.FitConfig(beta=0.5, rank=5, max_iters=15, inner_steps=5))
    assert relm(model, [gd[f"j_f{n}"] for n in range(4)]) < 1e-10
    assert O.rel_err([t[2] for t in tr], gd["j_trace"]) < 1e-10


@pytest.mark.parametrize("beta", [0.5, 1.0])
@pytest.mark.parametrize("algo", ["bcomm", "jcomm"])
def test_oracle_matches_golden_c3_small(beta, algo):
    gd = g("c3_small.npz")
    x, init = D.gamma_noised_tucker((16, 14, 12), (3, 3, 3), 3)
    fit = O.tucker_bcomm_fit if algo == "bcomm" else O.tucker_jcomm_fit
    (core, fs), tr = fit(x, init, O.FitConfig(beta=beta, ranks=[3, 3, 3], max_iters=20,
                                              inner_steps=1 if algo == "bcomm" else 3))
    tag = f"{algo}{beta}"
    assert O.rel_err(core, gd[f"{tag}_core"]) < 1e-10
    assert relm(fs, [gd[f"{tag}_f{n}"] for n in range(3)]) < 1e-10
    assert O.rel_err([t[2] for t in tr], gd[f"{tag}_trace"]) < 1e-10


def test_oracle_matches_golden_misc():
    gd = g("misc.npz")
    x, init = D.gamma_noised_cp((12, 10, 8), 3, 4)
    m, tr = O.bcomm_fit(x, init, O.FitConfig(beta=1.5, rank=3, max_iters=25, extrapolate=True))
    assert relm(m, [gd[f"ex_f{n}"] for n in range(3)]) < 1e-10
    assert O.rel_err([t[2] for t in tr], gd["ex_trace"]) < 1e-10
    m, tr = O.jcomm_fit(x, init, O.FitConfig(beta=0.5, rank=3, max_iters=25, extrapolate=True, inner_steps=5))
    assert relm(m, [gd[f"exj_f{n}"] for n in range(3)]) < 1e-10
    m, tr = O.jcomm_fit(x, init, O.FitConfig(beta=1.0, rank=3, max_iters=500, tol=1e-6, inner_steps=5))
    assert len(tr) == len(gd["tol_trace"])
    assert relm(m, [gd[f"tol_f{n}"] for n in range(3)]) < 1e-10


@pytest.mark.skipif(not R.available(), reason="oracle/_ref not built (needs /root/reference)")
@pytest.mark.parametrize("beta", [0.0, 0.5, 1.0, 1.5, 0.7])
def test_oracle_vs_reference_step_level(beta):
    dims = [6, 5, 4]
    x = O.random_tensor(dims, 3)
    f = O.init_cp_factors(dims, 2, 3, EPS)
    for mode in range(3):
        assert relm(O.bcomm_block_update(f, mode, x, beta, EPS), R.cp_block_update(x, f, mode, beta)) < 1e-13
    p, q = R.cp_jcomm_reference(x, f, beta)
    _, op, oq = O.make_jcomm_reference(f, x, beta, EPS)
    assert O.rel_err(p, op) < 1e-14 and O.rel_err(q, oq) < 1e-14
    assert relm(O.jcomm_outer_step(f, x, beta, 3, EPS), R.cp_jcomm_outer_step(x, f, beta, 3)) < 1e-12
    core, fs = O.init_tucker_model(dims, [2, 2, 2], 3, EPS)
    for kind, fn in [(0, lambda: O.block_core_update((core, fs), x, beta, EPS)),
                     (2, lambda: O.tucker_bcomm_sweep((core, fs), x, beta, EPS))]:
        c, ff = R.tucker_step(kind, x, core, fs, beta=beta)
        oc, off = fn()
        assert O.rel_err(c, oc) < 1e-12 and relm(ff, off) < 1e-12


def test_coo_densify_accumulates_duplicates_in_order():
    # read_coo io.cpp:138: dense[idx] += v, line by line
    idx = np.array([[0, 1], [1, 0], [0, 1], [0, 1]], dtype=np.int32)
    vals = np.array([1.0, 2.0, 0.1, 0.2])
    d = O.coo_densify(idx, vals, (2, 2))
    assert d[0, 1] == (1.0 + 0.1) + 0.2 and d[1, 0] == 2.0 and d[0, 0] == 0.0


def test_coo_synthetic_conventions():
    idx, vals = O.coo_synthetic((10, 50), 5000, seed=0, zipf_modes=(1,))
    assert idx.dtype == np.int32 and idx.min() >= 0 and idx[:, 1].max() < 50
    assert vals.min() == 1.0  # failures-count geometric: support {1, 2, ...}
    assert np.bincount(idx[:, 1]).argmax() == 0  # Zipf head at index 0


# ---- joint-surrogate oracle (reference oracle.cpp:181-302, tests/test_oracle.cpp:44-160) ----

def _surrogate_case(seed, dims=(5, 4, 3), rank=2):
    rng = np.random.default_rng(seed)
    x = 0.1 + rng.random(dims)
    ref = [0.1 + rng.random((d, rank)) for d in dims]
    theta = [a * (1.0 + 0.1 * rng.random(a.shape)) for a in ref]
    return x, ref, theta


@pytest.mark.parametrize("beta", [0.0, 0.5, 1.0, 1.5])
def test_joint_surrogate_tight_majorizes_and_descends(beta):
    # test_oracle.cpp:44-70, 117-131: tight at the reference, majorizes the
    # objective, nonincreasing across joint inner updates
    x, ref, _ = _surrogate_case(2)
    g = O.eval_joint_surrogate_cp(ref, ref, x, beta)
    d = O.D_beta(x, O.cp_reconstruct(ref), beta)
    assert abs(g - d) <= 1e-10 * (1.0 + d)
    rng = np.random.default_rng(6)
    for _ in range(20):
        theta = [a * (1.0 + 0.1 * rng.random(a.shape)) for a in ref]
        assert O.eval_joint_surrogate_cp(theta, ref, x, beta) >= O.D_beta(x, O.cp_reconstruct(theta), beta) - 1e-10 * (1 + d)
    ctx = O.make_jcomm_reference(ref, x, beta, 1e-12)
    cur, gprev = [a.copy() for a in ref], g
    for _ in range(3):
        for n in range(3):
            cur = O.jcomm_inner_update(cur, ctx, n, beta, 1e-12)
            nxt = O.eval_joint_surrogate_cp(cur, ref, x, beta)
            assert nxt <= gprev + 1e-12 * (1.0 + abs(gprev))
            gprev = nxt


def test_joint_surrogate_single_component_and_scalar_minimizer_kats():
    # test_oracle.cpp:72-81, 133-160
    g = O.eval_joint_surrogate_cp([np.array([[2.0]]), np.array([[1.0]])], [np.ones((1, 1)), np.ones((1, 1))],
                                  np.array([[2.0]]), 1.0)
    assert abs(g - float(O.d_beta(2.0, 2.0, 1.0))) <= 1e-12
    for beta in (0.0, 0.5, 1.0, 1.5):
        assert O.scalar_minimizer(3.0, 3.0, beta, 1e-12) == 1.0
        assert O.scalar_minimizer(0.0, 2.0, beta, 1e-9) == 1e-9
        rng = np.random.default_rng(3)
        for _ in range(10):
            num, den = 0.05 + 3.0 * rng.random(), 0.05 + 3.0 * rng.random()
            u = O.scalar_minimizer(num, den, beta, 1e-12)
            gu = O.jmm_scalar_objective(u, num, den, beta)
            for k in range(100):
                cand = u * 10.0 ** (-2.0 + 4.0 * k / 99.0)
                assert gu <= O.jmm_scalar_objective(cand, num, den, beta) + 1e-12 * (1.0 + abs(gu))
    with pytest.raises(O.DomainError):
        O.scalar_minimizer(1.0, 0.0, 0.5, 1e-12)


@pytest.mark.skipif(not R.available(), reason="oracle/_ref not built (needs /root/reference)")
@pytest.mark.parametrize("beta", [0.0, 0.5, 1.0, 1.5])
def test_joint_surrogate_matches_compiled_reference(beta):
    x, ref, theta = _surrogate_case(11, dims=(4, 3, 2, 3), rank=3)
    want = R.joint_surrogate_cp(theta, ref, x, beta)
    assert abs(O.eval_joint_surrogate_cp(theta, ref, x, beta) - want) <= 1e-12 * (1.0 + abs(want))
    assert abs(O.eval_joint_surrogate_cp(theta, ref, x, beta, slab=3) - want) <= 1e-12 * (1.0 + abs(want))
    rng = np.random.default_rng(12)
    tref = (0.1 + rng.random((2, 2, 2, 2)), [0.1 + rng.random((d, 2)) for d in x.shape])
    tth = (tref[0] * 1.3, [a * 1.1 for a in tref[1]])
    want = R.joint_surrogate_tucker(tth, tref, x, beta)
    assert abs(O.eval_joint_surrogate_tucker(tth, tref, x, beta) - want) <= 1e-12 * (1.0 + abs(want))
    u, gu = R.scalar_minimizer(1.7, 0.9, beta)
    assert u == O.scalar_minimizer(1.7, 0.9, beta, 1e-12)
    assert abs(gu - O.jmm_scalar_objective(u, 1.7, 0.9, beta)) <= 1e-14 * (1.0 + abs(gu))
