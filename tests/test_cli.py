"""ntf-cli: the reference command-line front end (tools/ntf_main.cpp) over the
drop-in library.  CPU: the binary builds, the usage / format exit-code
contract (1 usage, 3 format).  GPU: synth-cp -> fit -> trace CSV / model
files / bench CSV end to end, checked against the oracle run from the same
reference-RNG initialisation (init stream) and the same data."""
import os
import subprocess

import numpy as np
import pytest

from oracle import ntf_oracle as O
from paper_2602_14683_b200 import io as nio

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_2602_14683_b200", "lib", "ntf-cli")


def run(*args):
    return subprocess.run([CLI, *map(str, args)], capture_output=True, text=True, timeout=600)


def test_cli_built():
    assert os.access(CLI, os.X_OK)
    r = run("--help")
    assert r.returncode == 0 and "synth-cp" in r.stdout


@pytest.mark.parametrize("args,code", [
    ((), 1),
    (("frobnicate",), 1),
    (("fit", "--bogus", "1"), 1),
    (("fit", "--input"), 1),
    (("fit", "--input", "/nonexistent/x.ctf"), 3),
    (("fit", "--input", "x.ctf", "--beta", "2.5"), 1),
    (("fit", "--input", "x.ctf", "--algo", "sgd"), 1),
    (("synth-cp", "--rank", "2", "--out", "x.ctf"), 1),
    (("bench", "--input", "x.ctf", "--algos", "bcomm", "--out", "b.csv"), 1),
])
def test_cli_exit_codes(args, code, tmp_path):
    r = subprocess.run([CLI, *args], capture_output=True, text=True, cwd=tmp_path, timeout=60)
    assert r.returncode == code, (r.returncode, r.stderr)
    if code:
        assert r.stderr.startswith("error") or "usage" in r.stderr


def test_cli_bad_ctf1_is_format_error(tmp_path):
    bad = tmp_path / "bad.ctf"
    bad.write_bytes(b"CTF1\x02" + b"\x00" * 3)  # truncated header
    r = run("fit", "--input", bad)
    assert r.returncode == 3, r.stderr


@pytest.mark.gpu
@pytest.mark.parametrize("algo", ["bcomm", "jcomm"])
def test_cli_synth_fit_matches_oracle(algo, tmp_path):
    x_path, tr_path, pre = tmp_path / "x.ctf", tmp_path / "t.csv", tmp_path / "m"
    r = run("synth-cp", "--dims", "12,10,8", "--rank", "3", "--seed", "4", "--out", x_path)
    assert r.returncode == 0, r.stderr
    x = nio.read_tensor(str(x_path))
    xo, _ = O.synth_cp([12, 10, 8], 3, 4)
    assert np.allclose(x, xo, rtol=1e-13, atol=0)
    r = run("fit", "--input", x_path, "--algo", algo, "--beta", "0.5", "--rank", "3", "--max-iters", "15",
            "--inner", "2", "--seed", "7", "--trace", tr_path, "--out", pre)
    assert r.returncode == 0, r.stderr
    assert r.stdout.startswith("iters 15 final_loss")
    init = O.init_cp_factors([12, 10, 8], 3, 7, 1e-12)
    fit = O.bcomm_fit if algo == "bcomm" else O.jcomm_fit
    om, otr = fit(x, init, O.FitConfig(beta=0.5, rank=3, max_iters=15, inner_steps=2))
    trace = nio.read_trace(str(tr_path))
    assert [t.iter for t in trace] == list(range(16))
    assert O.rel_err([t.loss for t in trace], [t[2] for t in otr]) < 1e-10
    for n in range(3):
        got = nio.read_tensor(str(pre) + f".factor{n}.ctf")
        assert O.rel_err(got, om[n]) < 1e-10


@pytest.mark.gpu
def test_cli_bench_csv_and_numerical_exit(tmp_path):
    x_path, out = tmp_path / "x.ctf", tmp_path / "b.csv"
    assert run("synth-cp", "--dims", "8,6,5", "--rank", "2", "--out", x_path).returncode == 0
    r = run("bench", "--input", x_path, "--algos", "bcomm,jcomm,mu-unfold", "--seeds", "1,2", "--rank", "2",
            "--max-iters", "4", "--out", out)
    assert r.returncode == 0, r.stderr
    lines = out.read_text().splitlines()
    assert lines[0] == "algo,seed,iter,time_s,loss"
    assert len(lines) == 1 + 3 * 2 * 4
    assert {ln.split(",")[0] for ln in lines[1:]} == {"bcomm", "jcomm", "mu-unfold"}
    # beta = 0 on data with exact zeros: NumericalError naming --data-floor -> exit 2
    z = tmp_path / "z.ctf"
    xz = np.ones((4, 3, 2))
    xz[0, 0, 0] = 0.0
    nio.write_tensor(str(z), xz)
    r = run("fit", "--input", z, "--beta", "0", "--rank", "1", "--max-iters", "2")
    assert r.returncode == 2 and "data-floor" in r.stderr, (r.returncode, r.stderr)
    r = run("fit", "--input", z, "--beta", "0", "--rank", "1", "--max-iters", "2", "--data-floor", "1e-3")
    assert r.returncode == 0, r.stderr
