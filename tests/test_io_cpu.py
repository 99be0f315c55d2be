"""Ingestion/generation through the C ABI on the host (no GPU needed):
CTF1 byte-exact interchange with files written by the compiled reference,
the read_coo grammar and its line-numbered errors, trace CSV, and the
Philox generator against its NumPy restatement (oracle) and the published
Philox4x32-10 known answer.  Reference: io.cpp:30-186."""
import os

import numpy as np
import pytest

import paper_2602_14683_b200 as ntf
from paper_2602_14683_b200 import io as nio
from oracle import ntf_oracle as O

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def test_ctf1_reads_reference_file_bit_exact():
    want = np.load(os.path.join(GOLD, "io_small.npz"))["ctf1_values"]
    got = nio.read_tensor(os.path.join(GOLD, "ref_small.ctf1"))
    assert got.shape == want.shape
    assert got.tobytes() == want.tobytes()  # -0.0 and subnormals included
    assert nio.ctf1_shape(os.path.join(GOLD, "ref_small.ctf1")) == [3, 2, 2]


def test_ctf1_write_reproduces_reference_bytes(tmp_path):
    want = open(os.path.join(GOLD, "ref_small.ctf1"), "rb").read()
    x = np.load(os.path.join(GOLD, "io_small.npz"))["ctf1_values"]
    p = tmp_path / "ours.ctf1"
    nio.write_tensor(p, x)
    assert open(p, "rb").read() == want


def test_ctf1_fp32_round_trip_and_scalar(tmp_path):
    x = (np.arange(24, dtype=np.float32) / 7).reshape(2, 3, 4)
    p = tmp_path / "f.ctf1"
    nio.write_tensor(p, x)
    assert os.path.getsize(p) == 5 + 8 * 3 + 8 * 24
    assert np.array_equal(nio.read_tensor(p), x.astype(np.float64))
    assert np.array_equal(nio.read_tensor(p, dtype="f32"), x)
    s = tmp_path / "s.ctf1"
    nio.write_tensor(s, np.array([2.5]))
    assert os.path.getsize(s) == 21  # test_io.cpp:42-60: 21-byte scalar


@pytest.mark.parametrize("blob,msg", [
    (b"XXXX\x01" + b"\x01" + b"\x00" * 7 + b"\x00" * 8, "bad magic"),
    (b"CTF1\x00", "zero tensor order"),
    (b"CTF1\x02" + b"\x01" + b"\x00" * 7, "truncated header"),
    (b"CTF1\x01" + b"\x00" * 8, "zero dimension"),
    (b"CTF1\x01" + b"\x02" + b"\x00" * 7 + b"\x00" * 8, "truncated payload"),
    (b"CTF1\x01" + b"\x01" + b"\x00" * 7 + b"\x00" * 9, "trailing bytes"),
])
def test_ctf1_malformed(tmp_path, blob, msg):
    p = tmp_path / "bad.ctf1"
    p.write_bytes(blob)
    with pytest.raises(ntf.FormatError, match=msg):
        nio.read_tensor(p)


def test_ctf1_entry_budget(tmp_path):
    p = tmp_path / "big.ctf1"
    p.write_bytes(b"CTF1\x02" + (1 << 14).to_bytes(8, "little") + (1 << 14).to_bytes(8, "little"))
    with pytest.raises(ntf.FormatError, match="entry budget"):
        nio.read_tensor(p, max_entries=1 << 27)


def test_coo_text_matches_reference_densify():
    g = np.load(os.path.join(GOLD, "io_small.npz"))
    idx, val, dims = nio.read_coo(os.path.join(GOLD, "coo_small.txt"))
    assert dims == [3, 4, 2] and idx.shape == (6, 3)
    assert np.array_equal(nio.coo_to_dense(idx, val, dims), g["coo_dense"])
    assert np.array_equal(nio.coo_to_dense(idx, val, dims, floor=0.5), g["coo_dense_floor"])
    assert np.array_equal(O.coo_densify(idx, val, dims), g["coo_dense"])


@pytest.mark.parametrize("text,msg", [
    ("0 1 2\n", "line 1: expected `dims: I1 I2 ... IN`"),
    ("dims: 2 0\n", "line 1: dimensions must be positive"),
    ("dims: 2 2\n0 5 1.0\n", "line 2: index out of range for mode 2"),
    ("dims: 2 2\n\n0 1\n", "line 3: malformed or missing value"),
    ("dims: 2 2\n0 1 1.0 7\n", "line 2: trailing tokens after value"),
    ("dims: 2 2\n0 1 -1.0\n", "line 2: negative value"),
    ("dims: 2 2\n0 x 1\n", "line 2: malformed entry line"),
    ("\n\n", "missing `dims:` header"),
])
def test_coo_text_errors(tmp_path, text, msg):
    p = tmp_path / "c.txt"
    p.write_text(text)
    with pytest.raises(ntf.FormatError, match=msg.replace("`", ".").replace("(", ".")):
        nio.read_coo(p)


def test_trace_csv_matches_reference_bytes(tmp_path):
    p = tmp_path / "t.csv"
    tr = [ntf.TraceRecord(0, 0.0, np.pi), ntf.TraceRecord(1, 0.125, 1e-17), ntf.TraceRecord(2, 1.0 / 3.0, 2.0 / 3.0)]
    nio.write_trace(p, tr)
    assert open(p).read() == open(os.path.join(GOLD, "ref_trace.csv")).read()
    back = nio.read_trace(p)
    assert [(t.iter, t.time_s, t.loss) for t in back] == [(t.iter, t.time_s, t.loss) for t in tr]


def test_philox_known_answer():
    # Philox4x32-10, counter 0, key 0 (Random123 known-answer vector)
    z = np.zeros(1, dtype=np.uint64)
    out = O.philox4x32_10((z, z, z, z), (0, 0))
    assert [int(w[0]) for w in out] == [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]


def test_philox_library_matches_restatement():
    for seed, stream, off in ((0, 1, 0), (12345, 3, 7), (2 ** 40 + 3, 2, 2 ** 33 + 1)):
        a = nio.philox_uniforms(seed, stream, off, 1001)
        b = O.philox_uniforms(seed, stream, off, 1001)
        assert np.array_equal(a, b)
        assert a.min() >= 0.0 and a.max() < 1.0


def test_cp_factors_generator_matches_restatement():
    for which in ("truth", "init"):
        a = nio.cp_factors((5, 4, 3), 3, 9, which)
        b = O.philox_cp_factors((5, 4, 3), 3, 9, which)
        for u, v in zip(a, b):
            assert np.array_equal(u, v)
