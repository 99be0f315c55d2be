"""Generates tests/golden/*.npz from the COMPILED REFERENCE (oracle/_ref, built
from the unmodified /root/reference sources by oracle/Makefile).

Run here (the container that has /root/reference):  python tests/golden/make_golden.py
Inputs are regenerated at test time from tests/datagen.py (stable PCG64
stream), so the fixtures hold only seeds, small inits and the reference's
outputs (factors + objective traces).
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle import ref as R  # noqa: E402
import datagen as D  # noqa: E402


def save(name, **arrs):
    np.savez_compressed(os.path.join(HERE, name), **arrs)
    print("wrote", name, {k: np.shape(v) for k, v in arrs.items()})


def cp_block(tag, x, init, algo, beta, iters, inner=5, **kw):
    f, tt, tl = R.cp_fit(algo, x, init, beta, max_iters=iters, inner_steps=inner, **kw)
    out = {f"{tag}_trace": tl}
    for n, a in enumerate(f):
        out[f"{tag}_f{n}"] = a
    return out


def main():
    assert R.available(), "build oracle/_ref first: make -C oracle"
    # configs[0] (C1): the full reference-runnable config, 200 B-CoMM iterations
    x, init = D.c1_problem(0)
    out = cp_block("c1", x, init, "bcomm", 1.0, 200)
    out.update(cp_block("c1_10", x, init, "bcomm", 1.0, 10))
    save("c1_bcomm.npz", **out)

    # configs[1] (C2) shape family, reduced: 24x20x16, R=6, J-CoMM L=5, 30 outer, all betas
    x, init = D.gamma_noised_cp((24, 20, 16), 6, 1)
    out = {}
    for b in (0.0, 0.5, 1.0, 1.5):
        out.update(cp_block(f"j{b}", x, init, "jcomm", b, 30))
        out.update(cp_block(f"b{b}", x, init, "bcomm", b, 30))
    save("c2_small.npz", **out)

    # configs[4] (C5) family, reduced: 4-way 10x9x8x7, R=5, beta=0.5, J-CoMM L=5
    x, init = D.gamma_noised_cp((10, 9, 8, 7), 5, 2)
    save("c5_small.npz", **cp_block("j", x, init, "jcomm", 0.5, 15))

    # configs[2] (C3) family, reduced: Tucker 16x14x12, core 3x3x3, beta in {0.5, 1}
    x, (core, fs) = D.gamma_noised_tucker((16, 14, 12), (3, 3, 3), 3)
    out = {}
    for b in (0.5, 1.0):
        for algo, inner in (("bcomm", 1), ("jcomm", 3)):
            c, f, tt, tl = R.tucker_fit(algo, x, core, fs, b, max_iters=20, inner_steps=inner)
            tag = f"{algo}{b}"
            out[f"{tag}_core"] = c
            out[f"{tag}_trace"] = tl
            for n, a in enumerate(f):
                out[f"{tag}_f{n}"] = a
    save("c3_small.npz", **out)

    # extrapolation (BMMe) + tol stop, reference semantics
    x, init = D.gamma_noised_cp((12, 10, 8), 3, 4)
    out = cp_block("ex", x, init, "bcomm", 1.5, 25, extrapolate=True)
    out.update(cp_block("exj", x, init, "jcomm", 0.5, 25, extrapolate=True))
    out.update(cp_block("tol", x, init, "jcomm", 1.0, 500, tol=1e-6))
    save("misc.npz", **out)
    io_fixtures()


COO_TEXT = """
dims: 3 4 2

0 1 1 2.5
2 3 0 1
0 1 1 0.25
1 0 1 4
2 3 0 1e-3
0 0 0 0
"""


def io_fixtures():
    """CTF1 bytes, COO densify and trace CSV written by the compiled reference."""
    x = np.array([-0.0, 5e-324, 1e308, np.pi, 1.0 / 3.0, 2.0 ** -1074, -1.5, 7.0, 0.1, 1e-300, 123456789.0,
                  2.0 ** 52 + 1.0]).reshape(3, 2, 2)
    R.write_tensor(os.path.join(HERE, "ref_small.ctf1"), x)
    with open(os.path.join(HERE, "coo_small.txt"), "w") as f:
        f.write(COO_TEXT)
    dense = R.read_coo_dense(os.path.join(HERE, "coo_small.txt"), 64)
    floored = R.read_coo_dense(os.path.join(HERE, "coo_small.txt"), 64, floor=0.5)
    R.write_trace(os.path.join(HERE, "ref_trace.csv"), [0.0, 0.125, 1.0 / 3.0], [np.pi, 1e-17, 2.0 / 3.0])
    save("io_small.npz", ctf1_values=x, coo_dense=dense, coo_dense_floor=floored)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "io":
        io_fixtures()
    else:
        main()
