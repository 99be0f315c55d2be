"""Small fp32 J-CoMM fits that run the tcgen05 kernels (tc_contract_kernel for
N = 16/32/64, recon_tc_kernel, recon_tile_kernel) for compute-sanitizer:
  compute-sanitizer --tool {memcheck,racecheck,synccheck} python tools/sanitize_small.py
Checks the results against the oracle as well (a sanitizer-clean wrong answer is no use)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2602_14683_b200 as ntf  # noqa: E402
from oracle import ntf_oracle as O  # noqa: E402

rng = np.random.default_rng(0)
for dims, rank in [((2, 128, 128), 8), ((3, 16, 128), 24), ((2, 2, 128, 128), 40)]:
    truth = [rng.random((d, rank)) for d in dims]
    x = (O.cp_reconstruct(truth) * rng.gamma(10.0, 0.1, size=dims)).astype(np.float32)
    init = [0.1 + rng.random((d, rank)) for d in dims]
    for beta in (0.5, 1.0):
        cfg = ntf.FitConfig(beta=beta, rank=rank, max_iters=2, inner_steps=2, precision="f32", use_graphs=False)
        got = ntf.jcomm_fit(x, init, cfg)
        om, otr = O.jcomm_fit(x.astype(np.float64), init, O.FitConfig(beta=beta, rank=rank, max_iters=2, inner_steps=2))
        err = max(O.rel_err(a, b) for a, b in zip(got.model, om))
        assert err < 1e-4, (dims, rank, beta, err)
        print("ok", dims, rank, beta, "%.2e" % err, flush=True)
print("sanitize_small done", ntf.default_context().stats()["kernel_launches"], "launches")
