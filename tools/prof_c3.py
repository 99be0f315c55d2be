"""One eager Tucker outer iteration on the C3 workload (256^3, core 16^3) for ncu captures.
usage: python tools/prof_c3.py [jcomm|bcomm] [beta] [iters]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2602_14683_b200 as ntf  # noqa: E402

algo = sys.argv[1] if len(sys.argv) > 1 else "jcomm"
beta = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 1
dims, ranks = (256, 256, 256), (16, 16, 16)
g = torch.Generator(device="cpu").manual_seed(0)
core = torch.rand(ranks, generator=g, dtype=torch.float64)
fs = [torch.rand(n, j, generator=g, dtype=torch.float64) for n, j in zip(dims, ranks)]
dev = torch.device("cuda", 0)
x = torch.einsum("abc,ia,jb,kc->ijk", core.to(dev), *[f.to(dev) for f in fs])
gc = torch.Generator(device=dev).manual_seed(7)
x = (x * torch._standard_gamma(torch.full(dims, 10.0, device=dev, dtype=torch.float64), generator=gc) * 0.1).float().contiguous()
rng = np.random.default_rng(1)
init = (0.1 + rng.random(ranks), [0.1 + rng.random((n, j)) for n, j in zip(dims, ranks)])
fit = ntf.tucker_bcomm_fit if algo == "bcomm" else ntf.tucker_jcomm_fit
cfg = ntf.FitConfig(beta=beta, ranks=list(ranks), inner_steps=3, max_iters=iters, precision="f32", use_graphs=False)
res = fit(x, init, cfg)
print("loss", res.trace[-1].loss, ntf.default_context().stats())
