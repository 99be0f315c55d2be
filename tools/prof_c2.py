"""One eager J-CoMM outer step on the C2 workload (for ncu captures).
usage: python tools/prof_c2.py [beta] [iters]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2602_14683_b200 as ntf  # noqa: E402

beta = float(sys.argv[1]) if len(sys.argv) > 1 else 0.5
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 1
x, init = bench.make_problem(bench.DIMS, bench.RANK, 0, 0, bench.DIMS[0], torch.device("cuda", 0))
torch.cuda.synchronize()
cfg = ntf.FitConfig(beta=beta, rank=bench.RANK, inner_steps=bench.INNER, max_iters=iters,
                    precision="f32", use_graphs=False)
res = ntf.jcomm_fit(x, init, cfg)
print("loss", res.trace[-1].loss, ntf.default_context().stats())
