"""One rank of the data-parallel engine test (tests/test_dist_gpu.py).

Launched twice (RANK 0/1, WORLD_SIZE 2, gloo over 127.0.0.1) on the SAME GPU:
each rank runs the real engine (libntfg.so) on its mode-0 slab with
``shard=(I0, row0)``; partial sums go through paper_2602_14683_b200.dist's
allreduce hook (host collective: no kernel ever waits on another rank, so
two processes on one device are safe).  Results are written to
OUT/rank{r}.npz for the parent test to compare against the unsharded fit.
"""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2602_14683_b200 as ntf  # noqa: E402
from paper_2602_14683_b200 import dist as D  # noqa: E402
import dist_cases as CASES  # noqa: E402


def main():
    out = sys.argv[1]
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    ctx = ntf.Context(0)
    D.attach(ctx, torch.device("cuda", 0), 1 << 16)
    res = {}
    for name, case in CASES.cases().items():
        x, init, cfg, kind = case
        if kind == "coo":
            idx, val, dims = x
            li, lv, (row0, row1) = D.shard_coo(idx, val, dims[0], world, rank)
            local = D.shard_model(init, row0, row1)
            fit = ntf.bcomm_fit_coo if cfg.algo == "bcomm" else ntf.jcomm_fit_coo
            r = fit(li, lv, [row1 - row0] + list(dims[1:]), local, cfg, ctx=ctx, shard=(dims[0], row0))
            for n, a in enumerate(r.model):
                res[f"{name}/f{n}"] = a
            res[f"{name}/trace"] = np.array([t.loss for t in r.trace])
            continue
        i0 = x.shape[0]
        row0, row1 = D.slab_rows(i0, world, rank)
        xs = np.ascontiguousarray(x[row0:row1])
        if kind == "cp":
            local = D.shard_model(init, row0, row1)
            fit = ntf.bcomm_fit if cfg.algo == "bcomm" else ntf.jcomm_fit
            r = fit(xs.astype(np.float32) if cfg.precision == "f32" else xs, local, cfg, ctx=ctx, shard=(i0, row0))
            for n, a in enumerate(r.model):
                res[f"{name}/f{n}"] = a
        else:
            core, fs = init
            fs = D.shard_model(fs, row0, row1)
            fit = ntf.tucker_bcomm_fit if cfg.algo == "bcomm" else ntf.tucker_jcomm_fit
            r = fit(xs, (core, fs), cfg, ctx=ctx, shard=(i0, row0))
            res[f"{name}/core"] = r.model[0]
            for n, a in enumerate(r.model[1]):
                res[f"{name}/f{n}"] = a
        res[f"{name}/trace"] = np.array([t.loss for t in r.trace])
    np.savez(os.path.join(out, f"rank{rank}.npz"), **res)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
