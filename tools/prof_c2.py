"""One eager J-CoMM outer step on the C2 workload (for ncu captures).
usage: python tools/prof_c2.py [beta] [iters]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_14683_b200 as ntf  # noqa: E402
from paper_2602_14683_b200 import io as nio  # noqa: E402

beta = float(sys.argv[1]) if len(sys.argv) > 1 else 0.5
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 1
dims = (512,) * 3
x = nio.generate_cp_gamma(dims, 32, seed=0)
init = nio.cp_factors(dims, 32, seed=1, which="init")
cfg = ntf.FitConfig(beta=beta, rank=32, inner_steps=5, max_iters=iters, precision="f32", use_graphs=False)
res = ntf.jcomm_fit(x, init, cfg)
print("loss", res.trace[-1].loss, ntf.default_context().stats())
