"""Deterministic synthetic inputs for the BASELINE.json configs (test infrastructure).

Only NumPy's PCG64 bit stream (stable across NumPy versions) is used; the
distributions are derived here so fixtures regenerate bit-identically:
  uniforms  Generator(PCG64(seed)).random()
  Gamma(k, theta) for integer k = theta * sum_{i<k} -log(U_i)
  Poisson(mu) by sequential inversion of uniforms (vectorised)
"""
from __future__ import annotations

import numpy as np


def _gen(seed):
    return np.random.Generator(np.random.PCG64(seed))


def uniform(shape, seed):
    return _gen(seed).random(shape)


def gamma_int(shape, k: int, theta: float, seed):
    g = _gen(seed)
    acc = np.zeros(shape)
    for _ in range(k):
        acc -= np.log1p(-g.random(shape))  # -log(1-U), U in [0,1) -> finite
    return theta * acc


def poisson(mu: np.ndarray, seed):
    """Inversion: smallest k with CDF(k) > U."""
    u = _gen(seed).random(mu.shape)
    k = np.zeros(mu.shape, dtype=np.int64)
    p = np.exp(-mu)
    cdf = p.copy()
    active = u >= cdf
    kk = 0
    while np.any(active) and kk < 1000:
        kk += 1
        p = p * mu / kk
        cdf = cdf + p
        k = np.where(active, kk, k)
        active = active & (u >= cdf)
    return k


def cp_truth(dims, rank, seed):
    return [uniform((d, rank), seed * 1000 + n) for n, d in enumerate(dims)]


def init_u(dims, rank, seed):
    """Init ~ U[0.1, 1.1) (BASELINE.json configs)."""
    return [0.1 + uniform((d, rank), seed * 1000 + 500 + n) for n, d in enumerate(dims)]


def c1_problem(seed=0, dims=(100, 100, 100), rank=10):
    """configs[0]: X = Poisson([[A,B,C]] scaled to mean 5) + 1e-6, init U[0.1,1.1)."""
    from oracle import ntf_oracle as O
    truth = cp_truth(dims, rank, seed)
    m = O.cp_reconstruct(truth)
    m = m * (5.0 / m.mean())
    x = poisson(m, seed + 77).astype(np.float64) + 1e-6
    return x, init_u(dims, rank, seed)


def gamma_noised_cp(dims, rank, seed):
    """configs[1]/[4]: [[A,B,C]] * Gamma(10, 0.1)."""
    from oracle import ntf_oracle as O
    truth = cp_truth(dims, rank, seed)
    return O.cp_reconstruct(truth) * gamma_int(tuple(dims), 10, 0.1, seed + 99), init_u(dims, rank, seed)


def gamma_noised_tucker(dims, ranks, seed):
    """configs[2]: Tucker reconstruction * Gamma(10, 0.1); core/factors U[0,1)."""
    from oracle import ntf_oracle as O
    core = uniform(tuple(ranks), seed * 1000 + 900)
    fs = [uniform((d, j), seed * 1000 + n) for n, (d, j) in enumerate(zip(dims, ranks))]
    x = O.tucker_reconstruct(core, fs) * gamma_int(tuple(dims), 10, 0.1, seed + 99)
    icore = 0.1 + uniform(tuple(ranks), seed * 1000 + 950)
    ifs = [0.1 + uniform((d, j), seed * 1000 + 500 + n) for n, (d, j) in enumerate(zip(dims, ranks))]
    return x, (icore, ifs)
