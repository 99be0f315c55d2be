"""Tucker parity tests: CUDA path vs the CPU oracle (reference tests/test_tucker.cpp,
test_tensor.cpp:145-202, acceptance criterion 1).  Tolerances as in test_cp_gpu.py."""
import numpy as np
import pytest

import paper_2602_14683_b200 as ntf
from oracle import ntf_oracle as O

pytestmark = pytest.mark.gpu
EPS = 1e-12


def rel_model(a, b):
    return max([O.rel_err(a[0], b[0])] + [O.rel_err(x, y) for x, y in zip(a[1], b[1])])


def test_tucker_reconstruct_kats():
    core = O.random_tensor([2, 3], 5)
    assert np.array_equal(ntf.tucker_reconstruct(core, [np.eye(2), np.eye(3)]), core)
    ones = ntf.tucker_reconstruct(np.ones((1, 1)), [np.ones((3, 1)), np.ones((2, 1))])
    assert np.all(ones == 1.0)
    rng = O.Rng(4, O.Rng.DATA)
    fs = [O.random_cp_factors([3], 2, rng, EPS)[0], O.random_cp_factors([2], 3, rng, EPS)[0]]
    assert O.rel_err(ntf.tucker_reconstruct(core, fs), O.tucker_reconstruct(core, fs)) < 1e-14


@pytest.mark.parametrize("case", range(40))
def test_contractions_vs_oracle(case):
    """acceptance criterion 1 (orders 2-4, random small shapes)."""
    rng = np.random.default_rng(case)
    order = 2 + case % 3
    dims = [int(d) for d in rng.integers(1, 6, size=order)]
    ranks = [int(j) for j in rng.integers(1, 4, size=order)]
    mode = int(rng.integers(0, order))
    t = rng.random(dims)
    fs = [rng.random((d, j)) + 0.05 for d, j in zip(dims, ranks)]
    core = rng.random(ranks) + 0.05
    assert O.rel_err(ntf.tucker_multimode_contract(t, fs), O.tucker_multimode_contract(t, fs)) < 1e-12
    assert O.rel_err(ntf.tucker_multimode_contract(t, fs, skip=mode),
                     O.tucker_multimode_contract(t, fs, skip=mode)) < 1e-12
    assert O.rel_err(ntf.tucker_factor_contract(t, core, fs, mode),
                     O.tucker_factor_contract(t, core, fs, mode)) < 1e-12
    assert O.rel_err(ntf.tucker_reconstruct(core, fs), O.tucker_reconstruct(core, fs)) < 1e-12


def test_core_update_scalar_problem():
    x = np.ones((2, 2))
    m = (np.array([[2.0]]), [np.ones((2, 1)), np.ones((2, 1))])
    g = ntf.block_core_update(m, x, 1.0, EPS)
    assert g[0][0, 0] == 1.0
    assert ntf.tucker_objective(x, g, 1.0) == 0.0


def test_noiseless_optimum_unchanged():
    x, truth = O.synth_tucker([5, 4, 3], [2, 2, 2], 0)
    for b in [0.5, 1.0, 1.5]:
        m = ntf.block_core_update(truth, x, b, EPS)
        for n in range(3):
            m = ntf.block_factor_update(m, n, x, b, EPS)
        assert rel_model(m, truth) < 1e-12


@pytest.mark.parametrize("beta", [0.0, 0.5, 1.0, 1.5, 0.7])
def test_block_updates_vs_oracle(beta):
    x = O.random_tensor([6, 5, 4], 100)
    m = O.init_tucker_model([6, 5, 4], [2, 3, 2], 7, EPS)
    got = ntf.block_core_update(m, x, beta, EPS)
    assert rel_model(got, O.block_core_update(m, x, beta, EPS)) < 1e-12
    for n in range(3):
        got = ntf.block_factor_update(m, n, x, beta, EPS)
        assert rel_model(got, O.block_factor_update(m, n, x, beta, EPS)) < 1e-12


@pytest.mark.parametrize("beta", [0.0, 0.5, 1.0, 1.5])
@pytest.mark.parametrize("precision", ["f64", "f32"])
def test_first_joint_core_update_equals_block_bitwise(beta, precision):
    """reference test_tucker.cpp:83-94."""
    x = O.random_tensor([5, 4, 3], 5)
    m = O.init_tucker_model([5, 4, 3], [2, 2, 2], 5, EPS)
    ctx = ntf.make_jcomm_tucker_reference(m, x, beta, EPS, precision=precision)
    joint = ntf.jcomm_inner_core_update(m, ctx, beta, EPS, precision=precision)
    block = ntf.block_core_update(m, x, beta, EPS, precision=precision)
    assert np.array_equal(joint[0], block[0])


@pytest.mark.parametrize("beta", [0.0, 0.5, 1.0, 1.5])
def test_joint_inner_updates_vs_oracle(beta):
    x = O.random_tensor([6, 5, 4], 8)
    ref = O.init_tucker_model([6, 5, 4], [2, 3, 2], 8, EPS)
    rng = O.Rng(30, O.Rng.DATA)
    cur = (ref[0] * (1 + 0.2 * rng.uniforms(ref[0].size).reshape(ref[0].shape)),
           [a * (1 + 0.2 * rng.uniforms(a.size).reshape(a.shape)) for a in ref[1]])
    octx = O.make_jcomm_tucker_reference(ref, x, beta, EPS)
    ctx = ntf.make_jcomm_tucker_reference(ref, x, beta, EPS)
    # the cache is the reference's type: host P~/Q~ (tucker.hpp:59-63)
    assert O.rel_err(ctx.p, octx[1]) < 1e-12 and O.rel_err(ctx.q, octx[2]) < 1e-12
    got = ntf.jcomm_inner_core_update(cur, ctx, beta, EPS)
    assert rel_model(got, O.jcomm_inner_core_update(cur, octx, beta, EPS)) < 1e-12
    for n in range(3):
        got = ntf.jcomm_inner_factor_update(cur, ctx, n, beta, EPS)
        assert rel_model(got, O.jcomm_inner_factor_update(cur, octx, n, beta, EPS)) < 1e-12


@pytest.mark.parametrize("algo", ["bcomm", "jcomm"])
@pytest.mark.parametrize("beta", [0.0, 0.5, 1.0, 1.5])
def test_fit_f64_matches_oracle(algo, beta):
    dims, ranks = [9, 8, 7], [3, 2, 4]
    x = O.random_tensor(dims, 2000)
    init = O.init_tucker_model(dims, ranks, 1, EPS)
    cfg = ntf.FitConfig(beta=beta, ranks=ranks, max_iters=25, inner_steps=3)
    fit = ntf.tucker_bcomm_fit if algo == "bcomm" else ntf.tucker_jcomm_fit
    ofit = O.tucker_bcomm_fit if algo == "bcomm" else O.tucker_jcomm_fit
    res = fit(x, init, cfg)
    om, otr = ofit(x, init, O.FitConfig(beta=beta, ranks=ranks, max_iters=25, inner_steps=3))
    assert rel_model(res.model, om) < 1e-10
    assert O.rel_err([t.loss for t in res.trace], [t[2] for t in otr]) < 1e-10
    losses = [t.loss for t in res.trace]
    assert all(b <= a + 1e-12 * (1 + abs(a)) for a, b in zip(losses, losses[1:]))


@pytest.mark.parametrize("algo", ["bcomm", "jcomm"])
@pytest.mark.parametrize("beta", [0.5, 1.0])
def test_fit_f32_matches_oracle(algo, beta):
    dims, ranks = [32, 28, 24], [4, 4, 4]
    rng = np.random.default_rng(3)
    core = rng.random(ranks)
    fs = [rng.random((d, j)) for d, j in zip(dims, ranks)]
    x = O.tucker_reconstruct(core, fs) * rng.gamma(10.0, 0.1, size=dims)
    init = (0.1 + rng.random(ranks), [0.1 + rng.random((d, j)) for d, j in zip(dims, ranks)])
    cfg = ntf.FitConfig(beta=beta, ranks=ranks, max_iters=20, inner_steps=3, precision="f32")
    fit = ntf.tucker_bcomm_fit if algo == "bcomm" else ntf.tucker_jcomm_fit
    ofit = O.tucker_bcomm_fit if algo == "bcomm" else O.tucker_jcomm_fit
    res = fit(x, init, cfg)
    om, otr = ofit(x, init, O.FitConfig(beta=beta, ranks=ranks, max_iters=20, inner_steps=3))
    assert rel_model(res.model, om) < 1e-4
    assert O.rel_err([t.loss for t in res.trace], [t[2] for t in otr]) < 1e-5


def test_fit_drivers_stopping_and_recovery():
    """reference test_tucker.cpp:131-152 (reduced iteration count)."""
    dims, ranks = [20, 18, 16], [10, 9, 8]
    x, truth = O.synth_tucker(dims, ranks, 0)
    init = O.init_tucker_model(dims, ranks, 0, EPS)
    r0 = ntf.tucker_bcomm_fit(x, init, ntf.FitConfig(ranks=ranks, max_iters=0))
    assert len(r0.trace) == 1 and rel_model(r0.model, init) == 0.0
    r1 = ntf.tucker_bcomm_fit(x, init, ntf.FitConfig(ranks=ranks, max_iters=300))
    losses = [t.loss for t in r1.trace]
    assert all(b <= a + 1e-12 * (1 + abs(a)) for a, b in zip(losses, losses[1:]))
    assert losses[-1] <= 1e-2 * losses[0]
    r2 = ntf.tucker_jcomm_fit(x, init, ntf.FitConfig(ranks=ranks, max_iters=60, inner_steps=2))
    l2 = [t.loss for t in r2.trace]
    assert all(b <= a + 1e-12 * (1 + abs(a)) for a, b in zip(l2, l2[1:]))


@pytest.mark.parametrize("algo", ["bcomm", "jcomm"])
def test_zero_cap_extrapolation_bitwise(algo):
    """reference test_tucker.cpp:154-172."""
    x, _ = O.synth_tucker([6, 5, 4], [2, 2, 2], 9)
    init = O.init_tucker_model([6, 5, 4], [2, 2, 2], 9, EPS)
    fit = ntf.tucker_bcomm_fit if algo == "bcomm" else ntf.tucker_jcomm_fit
    a = fit(x, init, ntf.FitConfig(beta=1.0, ranks=[2, 2, 2], max_iters=15))
    b = fit(x, init, ntf.FitConfig(beta=1.0, ranks=[2, 2, 2], max_iters=15, extrapolate=True, extrap_cap=0.0))
    assert np.array_equal(a.model[0], b.model[0])
    for u, v in zip(a.model[1], b.model[1]):
        assert np.array_equal(u, v)


@pytest.mark.parametrize("algo", ["bcomm", "jcomm"])
def test_extrapolated_fit_matches_oracle(algo):
    dims, ranks = [7, 6, 5], [2, 3, 2]
    x = O.random_tensor(dims, 44)
    init = O.init_tucker_model(dims, ranks, 4, EPS)
    cfg = ntf.FitConfig(beta=0.5, ranks=ranks, max_iters=15, extrapolate=True)
    fit = ntf.tucker_bcomm_fit if algo == "bcomm" else ntf.tucker_jcomm_fit
    ofit = O.tucker_bcomm_fit if algo == "bcomm" else O.tucker_jcomm_fit
    res = fit(x, init, cfg)
    om, otr = ofit(x, init, O.FitConfig(beta=0.5, ranks=ranks, max_iters=15, extrapolate=True))
    assert rel_model(res.model, om) < 1e-10
    assert O.rel_err([t.loss for t in res.trace], [t[2] for t in otr]) < 1e-10


@pytest.mark.parametrize("dims,ranks", [([6], [3]), ([7, 5], [2, 3]), ([5, 4, 3, 4], [2, 2, 3, 2])])
def test_other_orders_vs_oracle(dims, ranks):
    x = O.random_tensor(dims, 77)
    init = O.init_tucker_model(dims, ranks, 77, EPS)
    for algo in ["bcomm", "jcomm"]:
        fit = ntf.tucker_bcomm_fit if algo == "bcomm" else ntf.tucker_jcomm_fit
        ofit = O.tucker_bcomm_fit if algo == "bcomm" else O.tucker_jcomm_fit
        res = fit(x, init, ntf.FitConfig(beta=1.5, ranks=ranks, max_iters=10, inner_steps=2))
        om, otr = ofit(x, init, O.FitConfig(beta=1.5, ranks=ranks, max_iters=10, inner_steps=2))
        assert rel_model(res.model, om) < 1e-10


# Mid-size shapes that take the tiled kernels (tucker_kernels.cuh: cp.async rowgemm with
# K % 32 == 0, split-b TTM with I_m >= 64 and J_m in {8, 16}, table-driven core pairing) and
# the tcgen05 reconstruction with fp32 outputs and a row table (rows % 128 == 0, K % 128 == 0).
def _tucker_problem(dims, ranks, seed):
    rng = np.random.default_rng(seed)
    core = rng.random(ranks)
    fs = [rng.random((d, j)) for d, j in zip(dims, ranks)]
    x = O.tucker_reconstruct(core, fs) * rng.gamma(10.0, 0.1, size=dims)
    init = (0.1 + rng.random(ranks), [0.1 + rng.random((d, j)) for d, j in zip(dims, ranks)])
    return x, init


@pytest.mark.parametrize("algo", ["bcomm", "jcomm"])
@pytest.mark.parametrize("beta", [0.5, 1.0, 1.5])
@pytest.mark.parametrize("dims,ranks", [((64, 72, 128), (8, 16, 16)), ((16, 64, 256), (5, 8, 12))])
def test_tucker_tiled_paths_match_oracle(algo, beta, dims, ranks):
    x, init = _tucker_problem(dims, ranks, 3)
    fit32 = ntf.tucker_bcomm_fit if algo == "bcomm" else ntf.tucker_jcomm_fit
    ofit = O.tucker_bcomm_fit if algo == "bcomm" else O.tucker_jcomm_fit
    om, otr = ofit(x, init, O.FitConfig(beta=beta, ranks=list(ranks), max_iters=4, inner_steps=2))
    olosses = [t[2] for t in otr]
    for prec, tf, tt in (("f64", 1e-10, 1e-10), ("f32", 1e-4, 1e-5)):
        res = fit32(x, init, ntf.FitConfig(beta=beta, ranks=list(ranks), max_iters=4, inner_steps=2, precision=prec))
        assert rel_model(res.model, om) < tf, prec
        assert O.rel_err([t.loss for t in res.trace], olosses) < tt, prec


def test_tucker_contractions_mid_size_vs_oracle():
    # the split-b TTM and the offset-table core pairing against the oracle's einsum chains
    rng = np.random.default_rng(9)
    dims, ranks = (64, 80, 96), (8, 16, 8)
    t = rng.random(dims)
    fs = [rng.random((d, j)) + 0.05 for d, j in zip(dims, ranks)]
    core = rng.random(ranks) + 0.05
    assert O.rel_err(ntf.tucker_multimode_contract(t, fs), O.tucker_multimode_contract(t, fs)) < 1e-12
    for mode in range(3):
        assert O.rel_err(ntf.tucker_factor_contract(t, core, fs, mode),
                         O.tucker_factor_contract(t, core, fs, mode)) < 1e-12
