"""One eager J-CoMM outer iteration on the C5 workload (for ncu captures).
usage: python tools/prof_c5.py [iters]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_14683_b200 as ntf  # noqa: E402
from paper_2602_14683_b200 import io as nio  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 1
dims = (256,) * 4
x = nio.generate_cp_gamma(dims, 64, seed=0)
init = nio.cp_factors(dims, 64, seed=1, which="init")
cfg = ntf.FitConfig(beta=0.5, rank=64, inner_steps=5, max_iters=iters, precision="f32", use_graphs=False)
res = ntf.jcomm_fit(x, init, cfg)
print("loss", res.trace[-1].loss, ntf.default_context().stats())
