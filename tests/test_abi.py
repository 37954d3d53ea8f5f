"""CPU checks of the C-ABI boundary: libslb.so builds for sm_100a, loads without a GPU, and
exports every function include/slb.h declares; host-only entry points behave as documented."""
import ctypes
import math
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "slb.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[A-Za-z_][A-Za-z0-9_ ]*?[\s\*]+(slb_[a-z0-9_]+)\s*\(", src, flags=re.M)
    return sorted(set(names))


@pytest.fixture(scope="module")
def lib():
    from paper_2310_00889_b200 import build
    build.build()
    from paper_2310_00889_b200._native import lib as L
    return L()


def test_header_declares_the_path(lib):
    names = declared_functions()
    for must in ["slb_upsample", "slb_farfield_laplace_dl", "slb_farfield_stokes_sldl",
                 "slb_nearcorr_apply", "slb_matvec"]:
        assert must in names


def test_every_declared_symbol_is_exported(lib):
    from paper_2310_00889_b200._native import DECLARED
    names = declared_functions()
    raw = ctypes.CDLL(os.path.join(ROOT, "paper_2310_00889_b200", "libslb.so"))
    for n in names:
        assert hasattr(raw, n), n
    assert set(names) <= set(DECLARED), set(names) - set(DECLARED)


def test_sm100a_cubin_present():
    import subprocess
    so = os.path.join(ROOT, "paper_2310_00889_b200", "libslb.so")
    out = subprocess.run(["cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_host_entry_points(lib):
    assert lib.slb_abi_version() == 2
    assert lib.slb_eta_cfie(0.05) == pytest.approx(1 / (2 * 0.05 * math.log(20)), rel=1e-15)
    assert math.isnan(lib.slb_eta_cfie(0.0)) and math.isnan(lib.slb_eta_cfie(1.5))
    # argument validation happens before any CUDA call
    st = lib.slb_upsample(1, 10, 11, 20, 24, 3, None, None, None)   # odd nt
    assert st == 1 and b"even" in lib.slb_last_error()
    st = lib.slb_nearcorr_apply(4, 2, 3, 120, None, None, None, None, None, None)
    assert st == 1


def test_eta_matches_input_generator(lib):
    from synth.configs import eta_cfie_input
    for rho in (0.035, 0.05, 0.02, 1e-2, 1e-4):
        assert lib.slb_eta_cfie(rho) == pytest.approx(eta_cfie_input(rho), rel=1e-15)
