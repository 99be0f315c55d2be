"""C5 (BASELINE configs[4]) on one GPU: dense 4-way CP 256^4 fp32 (17 GB), R=64,
beta=0.5, J-CoMM L=5.  Data generated in place on the device (Philox, same
generator as the io tests); prints one JSON line with outer it/s and the
per-kernel split.  usage: python tools/bench_c5.py [steps] [warmup] [dim]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2602_14683_b200 as ntf  # noqa: E402
from paper_2602_14683_b200 import io as nio  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
warm = int(sys.argv[2]) if len(sys.argv) > 2 else 1
d = int(sys.argv[3]) if len(sys.argv) > 3 else 256
dims, R, beta, L = (d, d, d, d), 64, 0.5, 5
t0 = time.time()
x = nio.generate_cp_gamma(dims, R, seed=0)
init = nio.cp_factors(dims, R, seed=1, which="init")
torch.cuda.synchronize()
tgen = time.time() - t0
ctx = ntf.default_context(0)
cfg = lambda it: ntf.FitConfig(beta=beta, rank=R, inner_steps=L, max_iters=it, precision="f32")
ntf.jcomm_fit(x, init, cfg(warm), ctx=ctx)
res = ntf.jcomm_fit(x, init, cfg(steps), ctx=ctx)
st = ctx.stats()
ms = st["device_ms"] / steps
ctx.set_profiling(True)
ntf.jcomm_fit(x, init, cfg(1), ctx=ctx)
pst = ctx.stats()
ctx.set_profiling(False)
E = x.numel()
alg = 4.0 * E * (1 + 2 + 2 * L * 4)  # X read + P~,Q~ write + 2 planes-pairs read per inner block update
print(json.dumps({"workload": "C5 256^4 R=64 beta=0.5 J-CoMM L=5", "dims": dims, "outer_it_per_s": 1e3 / ms,
                  "ms_per_step": ms, "loss": [t.loss for t in res.trace], "gen_s": tgen,
                  "alg_bytes_per_outer": alg, "alg_GBps": alg / (ms * 1e-3) / 1e9,
                  "recon_ms": pst["recon_ms"], "contract_ms": pst["contract_ms"],
                  "contract_launches": pst["contract_launches"],
                  "contract_avg_ms": pst["contract_ms"] / max(1, pst["contract_launches"]),
                  "device_ms_prof": pst["device_ms"], "launches": st["kernel_launches"]}))
