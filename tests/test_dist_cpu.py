"""World-size-2 gloo tests of the data-parallel (mode-0 slab) host logic on CPU.

The engine's sharded step (cp_engine.cuh: local partial sums -> allreduce
hook -> identical MU on every rank; mode 0 local; beta = 1 mode-0 colsums
and the objective sum allreduced) is emulated here with the oracle's
per-slab arithmetic and the package's real torch.distributed hook
(paper_2602_14683_b200.dist.make_allreduce), then compared against the
unsharded oracle fit.  Replicated factors must come out bitwise identical on
both ranks.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import ntf_oracle as O
from paper_2602_14683_b200 import dist as D

EPS = 1e-12


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _slab_jcomm_outer(x_slab, f, beta, inner, allreduce, comm, i0_global):
    """One J-CoMM outer step with the engine's sharding (oracle arithmetic)."""
    ref = [a.copy() for a in f]
    pt, qt = O.weights(x_slab, O.cp_reconstruct(ref), beta, EPS)
    # objective of the incoming model: local sum -> allreduce
    comm[0] = float(np.sum(O.d_beta(x_slab, O.cp_reconstruct(ref), beta)))
    allreduce(0, 1, 0)
    loss = float(comm[0]) / (x_slab.size // x_slab.shape[0] * i0_global)
    cur = [a.copy() for a in f]
    n_modes = len(f)
    for _ in range(inner):
        for n in range(n_modes):
            t1 = [cur[m] if m == n else O.chi1(cur[m], ref[m], beta) for m in range(n_modes)]
            t2 = [cur[m] if m == n else O.chi2(cur[m], ref[m], beta) for m in range(n_modes)]
            num = O.cp_contract(pt, t1, n)
            if beta == 1.0:
                r = t2[0].shape[1]
                prod = np.ones(r)
                for m in range(n_modes):
                    if m == n:
                        continue
                    cs = t2[m].sum(axis=0)
                    if m == 0:  # slab-local rows of mode 0 -> allreduce
                        comm[:r] = torch.from_numpy(cs)
                        allreduce(0, r, 0)
                        cs = comm[:r].numpy().copy()
                    prod = prod * cs
                den = np.broadcast_to(prod, num.shape).copy()
            else:
                den = O.cp_contract(qt, t2, n)
            if n != 0:
                # packed [num | den] partials; the closed-form beta = 1 den is
                # already global (engine: phase-1 den = 0, colprod after)
                k = num.size
                comm[:k] = torch.from_numpy(num.ravel())
                comm[k:2 * k] = torch.from_numpy(den.ravel() if beta != 1.0 else np.zeros(k))
                allreduce(0, 2 * k, 0)
                num = comm[:k].numpy().reshape(num.shape).copy()
                if beta != 1.0:
                    den = comm[k:2 * k].numpy().reshape(den.shape).copy()
            cur[n] = O.multiplicative_update(ref[n], num, den, O.gamma_of(beta), EPS)
    return cur, loss


def _worker(rank, world, port, beta, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        dims = (10, 7, 6)
        rng = np.random.default_rng(5)
        truth = [rng.random((d, 3)) for d in dims]
        x = O.cp_reconstruct(truth) * rng.gamma(10.0, 0.1, size=dims)
        init = [0.1 + rng.random((d, 3)) for d in dims]
        r0, r1 = D.slab_rows(dims[0], world, rank)
        comm = torch.zeros(2 * max(dims) * 3 + 8, dtype=torch.float64)
        ar = D.make_allreduce(comm)
        f = D.shard_model(init, r0, r1)
        losses = []
        for _ in range(4):
            f, loss = _slab_jcomm_outer(x[r0:r1], f, beta, 2, ar, comm, dims[0])
            losses.append(loss)
        full0 = D.gather_mode0(f[0], dims[0])
        out[rank] = (full0, f[1], f[2], losses)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("beta", [0.5, 1.0])
def test_two_rank_slab_jcomm_matches_unsharded(beta):
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(world, port, beta, out), nprocs=world, join=True)
    dims = (10, 7, 6)
    rng = np.random.default_rng(5)
    truth = [rng.random((d, 3)) for d in dims]
    x = O.cp_reconstruct(truth) * rng.gamma(10.0, 0.1, size=dims)
    init = [0.1 + rng.random((d, 3)) for d in dims]
    model, trace = O.jcomm_fit(x, init, O.FitConfig(beta=beta, rank=3, max_iters=4, inner_steps=2))
    a, b = out[0], out[1]
    # replicated factors bitwise identical across ranks
    assert np.array_equal(a[1], b[1]) and np.array_equal(a[2], b[2])
    assert np.array_equal(a[0], b[0])
    for got, want in zip([a[0], a[1], a[2]], model):
        assert O.rel_err(got, want) < 1e-12
    # objective rows 0..3 (fused evaluation of the incoming model)
    assert O.rel_err(a[3], [t[2] for t in trace[:4]]) < 1e-12


def test_slab_rows_partition():
    for dim in (1, 7, 512):
        for world in (1, 2, 3, 8):
            spans = [D.slab_rows(dim, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == dim
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
    with pytest.raises(ValueError):
        D.slab_rows(8, 2, 2)
