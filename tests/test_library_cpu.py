"""CPU-side checks of the C-ABI library (no GPU calls): it builds for sm_100a, loads, exports every
symbol include/rsvd.h declares, and its pure host functions agree with the oracle's tables."""
import ctypes
import os
import re
import subprocess

import pytest

import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "rsvd.h")


@pytest.fixture(scope="module")
def libpath():
    from paper_1804_07531_b200 import build

    return build.build()


def declared_symbols():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(rsvd_[a-z_0-9]+)\s*\(", txt)))


def test_header_declares_abi():
    syms = declared_symbols()
    for s in ["rsvd_subspace", "rsvd_block_krylov", "rsvd_single_pass", "rsvd_create", "rsvd_comm_init"]:
        assert s in syms


def test_library_exports_every_declared_symbol(libpath):
    out = subprocess.run(["nm", "-D", "--defined-only", libpath], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (rsvd_\w+)", out))
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing
    lib = ctypes.CDLL(libpath)
    for s in declared_symbols():
        getattr(lib, s)


def test_binding_export_list_matches_header():
    from paper_1804_07531_b200 import rsvd

    assert sorted(rsvd.EXPORTS) == declared_symbols()


def test_sm100a_code_only(libpath):
    out = subprocess.run(["cuobjdump", "--list-elf", libpath], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_sass_uses_dmma_and_tma(libpath):
    """The view kernels are FP64 tensor-core (DMMA) kernels fed by TMA (UTMALDG)."""
    sass = subprocess.run(["cuobjdump", "-sass", libpath], capture_output=True, text=True).stdout
    assert "DMMA" in sass
    assert "UTMALDG" in sass


def test_recommend_input_matches_oracle(libpath):
    lib = ctypes.CDLL(libpath)
    for goal in range(4):
        for v in range(2, 9):
            assert lib.rsvd_recommend_input(goal, v) == O.recommend_input(goal, v)


def test_strerror_and_version(libpath):
    lib = ctypes.CDLL(libpath)
    lib.rsvd_strerror.restype = ctypes.c_char_p
    assert lib.rsvd_strerror(0) == b"ok"
    assert lib.rsvd_strerror(-1) == b"invalid argument"
    assert lib.rsvd_version() >= 100


def test_create_without_device_fails_cleanly(libpath):
    import torch

    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    lib = ctypes.CDLL(libpath)
    h = ctypes.c_void_p()
    rc = lib.rsvd_create(ctypes.byref(h), 0, None)
    assert rc == -3 and not h.value


def test_product_package_never_imports_oracle():
    """The product path must not route through the oracle (no CPU fallback)."""
    pkg = os.path.join(ROOT, "paper_1804_07531_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f


def test_rsvd_plan_matches_oracle():
    """Host-only ABI call (no GPU): rsvd_plan against the oracle's plans."""
    import oracle as O
    from paper_1804_07531_b200 import rsvd

    for k in range(1, 15):
        for T in range(2 * k + 6, 2 * k + 60, 3):
            for scheme, f in ((rsvd.RSVD_PLAN_FLAT, O.plan_flat), (rsvd.RSVD_PLAN_DECAY, O.plan_decay),
                              (rsvd.RSVD_PLAN_RAPID, O.plan_rapid)):
                l1, l2 = f(k, T)
                assert rsvd.plan(scheme, k, T) == (l1, k + l2, l1)
            for alpha in (0.0, 0.3, 0.5, 1.0):
                l1, l2, lc = O.plan_balanced(k, T, alpha)
                assert rsvd.plan(rsvd.RSVD_PLAN_BALANCED, k, T, alpha) == (l1, k + l2, lc)
    for bad in ((rsvd.RSVD_PLAN_FLAT, 5, 15, 0.5), (rsvd.RSVD_PLAN_BALANCED, 5, 24, 1.5), (7, 5, 24, 0.5),
                (rsvd.RSVD_PLAN_DECAY, 0, 24, 0.5)):
        with pytest.raises(rsvd.RsvdError):
            rsvd.plan(*bad)
