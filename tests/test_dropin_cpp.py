"""The drop-in C++ API: a reference-style caller (tests/cpp/dropin_test.cpp)
compiled against include/ntf/*.hpp and linked to libntf_b200.so -> libntfg.so.
CPU part: headers + library export the reference's ntf:: symbols.
GPU part: the program runs its checks on the B200."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2602_14683_b200", "lib")
SRC = os.path.join(ROOT, "tests", "cpp", "dropin_test.cpp")


def _build(tmp_path):
    exe = str(tmp_path / "dropin_test")
    r = subprocess.run(["g++", "-std=c++20", "-O1", "-I" + os.path.join(ROOT, "include"), SRC, "-L" + LIB,
                        "-lntf_b200", "-lntfg", "-Wl,-rpath," + LIB, "-o", exe], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_dropin_compiles_and_links(tmp_path):
    if not os.path.exists(os.path.join(LIB, "libntf_b200.so")):
        pytest.skip("native libraries not built")
    _build(tmp_path)
    syms = subprocess.run(["nm", "-DC", "--defined-only", os.path.join(LIB, "libntf_b200.so")],
                          capture_output=True, text=True).stdout
    for name in ["ntf::bcomm_fit", "ntf::jcomm_fit", "ntf::tucker_bcomm_fit", "ntf::tucker_jcomm_fit",
                 "ntf::bcomm_block_update", "ntf::cp_block_update_anchored", "ntf::bcomm_sweep",
                 "ntf::make_jcomm_reference", "ntf::jcomm_inner_update", "ntf::jcomm_outer_step",
                 "ntf::block_core_update", "ntf::block_factor_update", "ntf::tucker_bcomm_sweep",
                 "ntf::make_jcomm_tucker_reference", "ntf::jcomm_inner_core_update",
                 "ntf::jcomm_inner_factor_update", "ntf::jcomm_tucker_outer_step", "ntf::cp_reconstruct",
                 "ntf::D_beta", "ntf::D_beta_mean", "ntf::validate_fit_config",
                 "ntf::make_extrapolation_state", "ntf::extrapolation_begin_iteration", "ntf::extrapolate_block",
                 "ntf::extrapolation_end_iteration", "ntf::make_tucker_extrapolation_state",
                 "ntf::extrapolate_core"]:
        assert name + "(" in syms, name


@pytest.mark.gpu
def test_dropin_program_passes_on_gpu(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ALL PASS" in r.stdout, r.stdout + r.stderr
