"""A few eager sparse J-CoMM outer iterations on the C4 stand-in (for ncu captures).
usage: python tools/prof_c4.py [iters]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2602_14683_b200 as ntf  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 1
idx, vals, init = bench.c4_problem(0)
dev = torch.device("cuda", 0)
di, dv = torch.from_numpy(idx).to(dev), torch.from_numpy(vals).to(dev)
cfg = ntf.FitConfig(beta=1.0, rank=bench.C4_RANK, inner_steps=bench.C4_INNER, max_iters=iters, precision="f64",
                    use_graphs=False)
res = ntf.jcomm_fit_coo(di, dv, bench.C4_DIMS, init, cfg)
print("loss", res.trace[-1].loss, ntf.default_context().stats())
