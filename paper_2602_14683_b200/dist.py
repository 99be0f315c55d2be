"""Data-parallel (mode-0 slab) fits over torch.distributed.

SURVEY.md 8(e): X is split into contiguous mode-0 slabs, one per rank; factor
A_0 is sharded the same way (each rank owns its rows), every other factor /
the Tucker core is replicated.  Per block update the engine sums its local
Num/Den partials (packed fp64) and calls the allreduce hook registered on the
context; every rank then applies the identical MU step, so replicas stay
bitwise identical.  Mode-0 updates need no collective; at beta = 1 the
closed-form denominator's mode-0 column sums are allreduced; the objective
sum is allreduced once per outer iteration.

The hook stages payloads through one caller-owned device buffer (``comm``)
so torch.distributed (NCCL on GPUs, gloo in the CPU tests) can operate on a
regular tensor.
"""
from __future__ import annotations

from typing import List, Optional, Sequence, Tuple

import numpy as np


def slab_rows(global_dim0: int, world: int, rank: int) -> Tuple[int, int]:
    """Rows [row0, row1) of mode 0 owned by `rank` (balanced contiguous split)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("invalid world/rank")
    return global_dim0 * rank // world, global_dim0 * (rank + 1) // world


def shard_model(init: Sequence[np.ndarray], row0: int, row1: int) -> List[np.ndarray]:
    """This rank's CP model: mode-0 factor rows sliced, the rest replicated."""
    out = [np.array(a, dtype=np.float64, copy=True) for a in init]
    out[0] = out[0][row0:row1].copy()
    return out


def make_allreduce(comm, group=None):
    """Returns fn(ptr, count, stream) summing comm[:count] across the group.

    The engine enqueues the copy into ``comm`` on ITS stream and then calls the
    hook; the collective is issued on that same stream (ExternalStream), so it
    is ordered after the copy-in and before the engine's copy-back.  CUDA
    buffers with a CPU-only backend (gloo) go through host memory."""
    import torch
    import torch.distributed as dist

    def allreduce(ptr, count, stream):
        dev = comm.device
        if dev.type == "cuda":
            s = torch.cuda.ExternalStream(stream, device=dev) if stream else torch.cuda.current_stream(dev)
            with torch.cuda.stream(s):
                if dist.get_backend(group) == "gloo":
                    s.synchronize()
                    host = comm[:count].cpu()
                    dist.all_reduce(host, op=dist.ReduceOp.SUM, group=group)
                    comm[:count].copy_(host)
                else:
                    dist.all_reduce(comm[:count], op=dist.ReduceOp.SUM, group=group)
        else:
            dist.all_reduce(comm[:count], op=dist.ReduceOp.SUM, group=group)

    return allreduce


def attach(ctx, device, capacity: int, group=None):
    """Registers the comm buffer + Python hook on an ntf Context; returns the
    buffer.  Works with any torch.distributed backend; graphs are off while a
    hook is set (see attach_nccl for the native path)."""
    import torch
    comm = torch.zeros(int(capacity), dtype=torch.float64, device=device)
    ctx.set_comm_buffer(comm.data_ptr(), comm.numel())
    ctx.set_allreduce(make_allreduce(comm, group))
    return comm


def attach_nccl(ctx, group=None):
    """Native path: rank 0 of ``group`` creates an NCCL unique id, it is
    broadcast over torch.distributed, and every rank attaches a communicator
    to its context (ntfg_context_init_nccl).  The engine then allreduces with
    ncclAllReduce on its own stream, inside the captured CUDA graph -- no
    Python runs per block update."""
    import torch.distributed as dist
    from . import api
    obj = [api.nccl_unique_id() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
    ctx.init_nccl(obj[0], dist.get_world_size(group), dist.get_rank(group))


def shard_coo(indices, values, global_dim0: int, world: int, rank: int):
    """Nonzero partition by mode-0 index ranges: this rank's
    nonzeros with i_0 rebased to its slab, plus (row0, row1)."""
    idx = np.asarray(indices)
    val = np.asarray(values)
    row0, row1 = slab_rows(global_dim0, world, rank)
    keep = (idx[:, 0] >= row0) & (idx[:, 0] < row1)
    local = idx[keep].astype(np.int32, copy=True)
    local[:, 0] -= row0
    return local, val[keep].copy(), (row0, row1)


def gather_mode0(local: np.ndarray, global_dim0: int, group=None) -> np.ndarray:
    """All-gathers the mode-0 factor slabs into the full I_0 x R matrix."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    r = local.shape[1]
    sizes = [slab_rows(global_dim0, world, q)[1] - slab_rows(global_dim0, world, q)[0] for q in range(world)]
    mx = max(sizes)
    buf = torch.zeros(mx, r, dtype=torch.float64)
    buf[: local.shape[0]] = torch.from_numpy(local)
    outs = [torch.zeros(mx, r, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(outs, buf, group=group)
    del rank
    return np.concatenate([outs[q][: sizes[q]].numpy() for q in range(world)], axis=0)


def sharded_cp_fit(algo: str, x_slab, init_full: Sequence[np.ndarray], cfg, ctx, group=None,
                   gather: bool = True):
    """Runs this rank's share of a CP fit; returns (full factors, trace)."""
    import torch.distributed as dist
    from . import api
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    i0 = init_full[0].shape[0]
    row0, row1 = slab_rows(i0, world, rank)
    local = shard_model(init_full, row0, row1)
    fit = api.bcomm_fit if algo == "bcomm" else api.jcomm_fit
    res = fit(x_slab, local, cfg, ctx=ctx, shard=(i0, row0))
    model = list(res.model)
    if gather:
        model[0] = gather_mode0(model[0], i0, group)
    return model, res.trace
