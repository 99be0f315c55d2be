import sys, os
sys.path.insert(0, '/root/repo')
import numpy as np
import torch
import paper_2602_14683_b200 as ntf
from oracle import ntf_oracle as O
rng = np.random.default_rng(7)
dims = (16, 8, 128); rank = 4
truth = [rng.random((d, rank)) for d in dims]
x = O.cp_reconstruct(truth) * rng.gamma(10.0, 0.1, size=dims)
f = [0.1 + rng.random((d, rank)) for d in dims]
beta = 0.5
mode = 2
a = ntf.bcomm_block_update(f, mode, x, beta, 1e-12, precision="f32")[mode]
ctx = ntf.make_jcomm_reference(f, x, beta, 1e-12, precision="f32")
b = ntf.jcomm_inner_update(f, ctx, mode, beta, 1e-12, precision="f32")[mode]
# P/Q from oracle in fp32 then split like the recon kernel
_, op, oq = O.make_jcomm_reference(f, x, beta, 1e-12)
def hilo(v):
    t = torch.tensor(v, dtype=torch.float32)
    hi = t.to(torch.bfloat16); lo = (t - hi.float()).to(torch.bfloat16)
    return (hi.double() + lo.double()).numpy()
ctx2 = ntf.JcommCpReference(ctx.ref, hilo(op), hilo(oq))
c = ntf.jcomm_inner_update(f, ctx2, mode, beta, 1e-12, precision="f32")[mode]
print("block vs inner", np.abs(a - b).max())
print("inner(ctx) vs inner(oracle hilo)", np.abs(b - c).max(), "P diff", np.abs(ctx.p - hilo(op)).max())
a2 = ntf.bcomm_block_update(f, mode, x, beta, 1e-12, precision="f32")[mode]
print("block again vs block", np.abs(a2 - a).max())
# does a B-CoMM block update on the same engine equal jcomm inner within a fit?  fit 1 iter L=1
os.environ["NTFG_DISABLE_TC"] = "1"
d = ntf.bcomm_block_update(f, mode, x, beta, 1e-12, precision="f32")[mode]
e = ntf.jcomm_inner_update(f, ctx, mode, beta, 1e-12, precision="f32")[mode]
print("notc block vs tc block", np.abs(d - a).max(), "notc inner(ctx hilo) vs tc inner", np.abs(e - b).max())
