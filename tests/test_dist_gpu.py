"""The engine's data-parallel path, executed.

* Two processes on cuda:0, gloo over 127.0.0.1 (tests/dist_worker.py): each
  rank runs the real sharded engine on its mode-0 slab -- slab-local partial
  sums -> allreduce hook -> identical MU on every rank, for
  CP B-CoMM / J-CoMM at every beta, with BMMe extrapolation (alpha over the
  whole model), the fp32 tcgen05 build, and Tucker (core and middle factors
  reduced).  Checked against the unsharded fit of the whole tensor: fp64 to
  1e-12, fp32 to 1e-6; replicated factors, the Tucker core and the trace
  bitwise identical across ranks.  The collective is a host call, so no
  kernel ever waits on another rank (B200_PROFILING.md: never spin across
  processes on one GPU).
* The native NCCL communicator (ntfg_context_init_nccl) with one rank: the
  sharded path with ncclAllReduce on the engine stream, CUDA graphs on.
"""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

import paper_2602_14683_b200 as ntf
from oracle import ntf_oracle as O

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
if HERE not in sys.path:
    sys.path.insert(0, HERE)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module")
def two_rank_results(tmp_path_factory):
    out = str(tmp_path_factory.mktemp("dist"))
    port = _free_port()
    procs = []
    for r in range(2):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE="2", LOCAL_RANK="0", MASTER_ADDR="127.0.0.1",
                   MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, os.path.join(HERE, "dist_worker.py"), out], env=env,
                                      stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True))
    logs = []
    for p in procs:
        try:
            o, _ = p.communicate(timeout=900)
        except subprocess.TimeoutExpired:
            p.kill()
            o, _ = p.communicate()
        logs.append(o)
    assert all(p.returncode == 0 for p in procs), "\n".join(logs)[-4000:]
    return [dict(np.load(os.path.join(out, f"rank{r}.npz"))) for r in range(2)]


def _unsharded(case):
    x, init, cfg, kind = case
    if kind == "coo":
        idx, val, dims = x
        fit = ntf.bcomm_fit_coo if cfg.algo == "bcomm" else ntf.jcomm_fit_coo
        r = fit(idx, val, dims, init, cfg)
        return None, r.model, np.array([t.loss for t in r.trace])
    if kind == "cp":
        fit = ntf.bcomm_fit if cfg.algo == "bcomm" else ntf.jcomm_fit
        r = fit(x.astype(np.float32) if cfg.precision == "f32" else x, init, cfg)
        return None, r.model, np.array([t.loss for t in r.trace])
    fit = ntf.tucker_bcomm_fit if cfg.algo == "bcomm" else ntf.tucker_jcomm_fit
    r = fit(x, init, cfg)
    return r.model[0], r.model[1], np.array([t.loss for t in r.trace])


import dist_cases as CASES  # noqa: E402


@pytest.mark.parametrize("name", sorted(CASES.cases()))
def test_sharded_engine_matches_unsharded(two_rank_results, name):
    case = CASES.cases()[name]
    r0, r1 = two_rank_results
    core, fs, trace = _unsharded(case)
    tol = 1e-6 if case[2].precision == "f32" else 1e-11
    # replicas: bitwise identical across ranks
    assert np.array_equal(r0[f"{name}/trace"], r1[f"{name}/trace"])
    for n in range(1, len(fs)):
        assert np.array_equal(r0[f"{name}/f{n}"], r1[f"{name}/f{n}"]), n
    if core is not None:
        assert np.array_equal(r0[f"{name}/core"], r1[f"{name}/core"])
        assert O.rel_err(r0[f"{name}/core"], core) < tol
    # against the unsharded fit of the whole tensor
    f0 = np.concatenate([r0[f"{name}/f0"], r1[f"{name}/f0"]], axis=0)
    assert O.rel_err(f0, fs[0]) < tol
    for n in range(1, len(fs)):
        assert O.rel_err(r0[f"{name}/f{n}"], fs[n]) < tol, n
    assert O.rel_err(r0[f"{name}/trace"], trace) < tol


@pytest.mark.parametrize("algo", ["bcomm", "jcomm"])
@pytest.mark.parametrize("beta", [0.5, 1.0])
def test_native_nccl_single_rank(algo, beta):
    ctx = ntf.Context(0)
    ctx.init_nccl(ntf.nccl_unique_id(), 1, 0)
    rng = np.random.default_rng(5)
    dims = (24, 20, 16)
    truth = [rng.random((d, 4)) for d in dims]
    x = np.einsum("ir,jr,kr->ijk", *truth) * rng.gamma(10.0, 0.1, size=dims)
    init = [0.1 + rng.random((d, 4)) for d in dims]
    cfg = ntf.FitConfig(beta=beta, rank=4, max_iters=5, inner_steps=2)
    fit = ntf.bcomm_fit if algo == "bcomm" else ntf.jcomm_fit
    got = fit(x, init, cfg, ctx=ctx, shard=(dims[0], 0))
    assert ctx.stats()["graph_launches"] > 0  # the collective lives inside the CUDA graph
    ref = fit(x, init, cfg)
    assert max(O.rel_err(a, b) for a, b in zip(got.model, ref.model)) < 1e-13
    assert O.rel_err([t.loss for t in got.trace], [t.loss for t in ref.trace]) < 1e-13
