"""Role ablation of the tensor-core contraction on the C2 workload: per-launch
contract time with B producers / MMAs / epilogue work switched off
(NTFG_TC_ABLATE bits, set per subprocess).  Timing only -- results are wrong.
usage: python tools/tc_ablate.py [beta]"""
import json
import os
import subprocess
import sys

if len(sys.argv) > 2:  # child
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import paper_2602_14683_b200 as ntf
    beta = float(sys.argv[1])
    if os.environ.get("WORKLOAD") == "c5":  # 4-way CP, R = 64 (C5 shape; dim from C5_DIM, default 256)
        from paper_2602_14683_b200 import io as nio
        d = int(os.environ.get("C5_DIM", "256"))
        x = nio.generate_cp_gamma((d,) * 4, 64, seed=0)
        init = nio.cp_factors((d,) * 4, 64, seed=1, which="init")
        cfg = ntf.FitConfig(beta=beta, rank=64, inner_steps=5, max_iters=1, precision="f32", use_graphs=False)
    else:
        from paper_2602_14683_b200 import io as nio
        x = nio.generate_cp_gamma((512,) * 3, 32, seed=0)
        init = nio.cp_factors((512,) * 3, 32, seed=1, which="init")
        cfg = ntf.FitConfig(beta=beta, rank=32, inner_steps=5, max_iters=3, precision="f32", use_graphs=False)
    ctx = ntf.default_context()
    ctx.set_profiling(True)
    try:
        ntf.jcomm_fit(x, init, cfg)
    except Exception as e:  # ablated runs can trip the domain checks
        print("#", type(e).__name__, str(e)[:80], file=sys.stderr)
    print(json.dumps(ctx.stats()))
else:
    beta = sys.argv[1] if len(sys.argv) > 1 else "0.5"
    variants = [(b, None) for b in [0, 1, 2, 4, 6, 3, 7]] + [(0, "100000"), (0, "4"), (0, "64")]
    for bits, seg in variants:
        env = dict(os.environ, NTFG_TC_ABLATE=str(bits))
        if seg:
            env["NTFG_TC_SEG"] = seg
        out = subprocess.run([sys.executable, __file__, beta, "child"], env=env, capture_output=True, text=True)
        line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-300:]
        try:
            st = json.loads(line)
            print(os.environ.get("WORKLOAD", "c2"), bits, "seg", seg, "contract_ms/launch %.4f" % (st["contract_ms"] / max(st["contract_launches"], 1)),
                  "recon_ms", round(st["recon_ms"], 3))
        except Exception:
            print(bits, line)
