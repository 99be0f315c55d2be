"""BMMe step-level API (reference cp.hpp:80-110, tucker.hpp:88-106).

CPU: the Python mirror's ExtrapolationState arithmetic against the oracle's
restatement (cp.cpp:167-198).  GPU: a hand-written extrapolated loop over the
device step functions equals the device fit drivers (reference
test_cp.cpp:169-234 style)."""
import numpy as np
import pytest

import paper_2602_14683_b200 as ntf
from oracle import ntf_oracle as O


def _model(seed, dims=(6, 5, 4), r=3):
    rng = np.random.default_rng(seed)
    return [0.1 + rng.random((d, r)) for d in dims]


def test_state_matches_oracle():
    a, b, c = _model(1), _model(2), _model(3)
    st = ntf.make_extrapolation_state(a, True, 1.0, 1e-6, 1e-12)
    ost = O.Extrapolation(a, True, 1.0, 1e-6, 1e-12)
    for cur in (b, c):
        ntf.extrapolation_begin_iteration(st, cur)
        ost.begin(cur)
        assert st.alpha == ost.alpha and st.t == ost.t
        for n in range(3):
            assert np.array_equal(ntf.extrapolate_block(cur[n], st, n), ost.block(cur[n], n))
        ntf.extrapolation_end_iteration(st, cur)
        ost.end(cur)


def test_zero_cap_pins_alpha():
    a, b = _model(4), _model(5)
    st = ntf.make_extrapolation_state(a, True, 0.0, 1e-6, 1e-12)
    ntf.extrapolation_begin_iteration(st, b)
    assert st.alpha == 0.0
    assert np.array_equal(ntf.extrapolate_block(b[1], st, 1), b[1])


def test_tucker_state_blocks():
    rng = np.random.default_rng(6)
    m0 = (0.1 + rng.random((2, 3, 2)), _model(7, r=2))
    m1 = (m0[0] * 1.1, [f * 1.05 for f in m0[1]])
    st = ntf.make_tucker_extrapolation_state(m0, True, 1.0, 1e-6, 1e-12)
    ost = O.Extrapolation([m0[0]] + list(m0[1]), True, 1.0, 1e-6, 1e-12)
    ntf.extrapolation_begin_iteration(st, m1)
    ost.begin([m1[0]] + list(m1[1]))
    assert st.alpha == ost.alpha
    assert np.array_equal(ntf.extrapolate_core(m1[0], st), ost.block(m1[0], 0))
    assert np.array_equal(ntf.extrapolate_block(m1[1][2], st, 2), ost.block(m1[1][2], 3))
    with pytest.raises(ntf.ShapeError):
        ntf.extrapolate_block(m1[1][0][:2], st, 0)


@pytest.mark.gpu
@pytest.mark.parametrize("beta", [0.5, 1.0])
def test_step_loop_equals_fit_bcomm(beta):
    x = O.random_tensor([6, 5, 4], 31)
    f = _model(8)
    cfg = ntf.FitConfig(beta=beta, rank=3, max_iters=4, extrapolate=True, extrap_cap=5.0)
    fit = ntf.bcomm_fit(x, f, cfg)
    st = ntf.make_extrapolation_state(f, True, cfg.extrap_cap, cfg.extrap_delta, cfg.eps)
    cur = [a.copy() for a in f]
    for _ in range(4):
        snap = [a.copy() for a in cur]
        ntf.extrapolation_begin_iteration(st, cur)
        for n in range(3):
            cur = ntf.cp_block_update_anchored(cur, n, ntf.extrapolate_block(cur[n], st, n), x, beta, cfg.eps)
        ntf.extrapolation_end_iteration(st, snap)
    assert max(O.rel_err(a, b) for a, b in zip(cur, fit.model)) < 1e-10


@pytest.mark.gpu
def test_step_loop_equals_fit_jcomm():
    x = O.random_tensor([6, 5, 4], 32)
    f = _model(9)
    cfg = ntf.FitConfig(beta=0.5, rank=3, max_iters=3, inner_steps=2, extrapolate=True, extrap_cap=5.0)
    fit = ntf.jcomm_fit(x, f, cfg)
    st = ntf.make_extrapolation_state(f, True, cfg.extrap_cap, cfg.extrap_delta, cfg.eps)
    cur = [a.copy() for a in f]
    for _ in range(3):
        snap = [a.copy() for a in cur]
        ntf.extrapolation_begin_iteration(st, cur)
        ref = [ntf.extrapolate_block(cur[n], st, n) for n in range(3)]
        cur = ntf.jcomm_outer_step(ref, x, 0.5, 2, cfg.eps)
        ntf.extrapolation_end_iteration(st, snap)
    assert max(O.rel_err(a, b) for a, b in zip(cur, fit.model)) < 1e-10
