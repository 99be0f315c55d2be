"""Device-side ingestion and generation: CTF1 streamed into device memory
(fp64 -> fp32 on the device), device tensors written byte-exact, and the
in-place C2/C5 generator against the NumPy restatement."""
import os

import numpy as np
import pytest

from paper_2602_14683_b200 import io as nio
from oracle import ntf_oracle as O

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def test_ctf1_device_read_matches_host():
    want = np.load(os.path.join(GOLD, "io_small.npz"))["ctf1_values"]
    d64 = nio.read_tensor(os.path.join(GOLD, "ref_small.ctf1"), device=0)
    assert d64.is_cuda and d64.cpu().numpy().tobytes() == want.tobytes()
    d32 = nio.read_tensor(os.path.join(GOLD, "ref_small.ctf1"), device=0, dtype="f32")
    assert np.array_equal(d32.cpu().numpy(), want.astype(np.float32))


def test_ctf1_device_large_multi_chunk(tmp_path):
    import torch
    # > one 32 MiB staging chunk, both halves of the double buffer used
    x = torch.rand(3, 1000, 3000, dtype=torch.float64, device="cuda")
    p = tmp_path / "big.ctf1"
    nio.write_tensor(p, x)
    assert os.path.getsize(p) == 5 + 24 + 8 * x.numel()
    back = nio.read_tensor(p, device=0, max_entries=0)
    assert torch.equal(back, x)
    back32 = nio.read_tensor(p, device=0, dtype="f32", max_entries=0)
    assert torch.equal(back32, x.float())
    host = nio.read_tensor(p, max_entries=0)
    assert np.array_equal(host, x.cpu().numpy())
    x32 = x.float()
    nio.write_tensor(p, x32)
    assert np.array_equal(nio.read_tensor(p, max_entries=0), x32.cpu().numpy().astype(np.float64))


@pytest.mark.parametrize("dims,rank,rows", [((12, 10, 8), 4, None), ((9, 6, 5, 4), 3, (3, 7))])
def test_generate_cp_gamma_matches_restatement(dims, rank, rows):
    g = nio.generate_cp_gamma(dims, rank, seed=5, rows=rows, dtype="f64").cpu().numpy()
    want = O.philox_cp_gamma(dims, rank, 5, rows=rows)
    assert g.shape == want.shape
    assert O.rel_err(g, want) < 1e-13
    g32 = nio.generate_cp_gamma(dims, rank, seed=5, rows=rows, dtype="f32").cpu().numpy()
    assert np.max(np.abs(g32 - want) / np.abs(want)) < 1e-6
    # gamma(10, 0.1) noise has mean 1
    noise = g / O.cp_reconstruct(O.philox_cp_factors(dims, rank, 5, "truth"))[slice(*(rows or (0, dims[0])))]
    assert abs(noise.mean() - 1.0) < 0.1


def test_generate_slabs_tile_the_full_tensor():
    full = nio.generate_cp_gamma((10, 7, 6), 3, seed=2, dtype="f32").cpu().numpy()
    parts = [nio.generate_cp_gamma((10, 7, 6), 3, seed=2, rows=r, dtype="f32").cpu().numpy()
             for r in ((0, 3), (3, 4), (4, 10))]
    assert np.array_equal(np.concatenate(parts), full)
