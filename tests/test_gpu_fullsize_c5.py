"""C5 at full size (fp32 100000 x 100000, 40 GB; tcgen05 3xTF32 views), element-wise against the
oracle (north_star: all five configs).

A is built on the GPU (synth.make_matrix_torch) and its fp32 bytes are copied back once (widened
to fp64, exactly); the oracle runs in fp64 on those values over row panels (oracle.PanelOp), with
the same Omega.  BASELINE C5's runs: subspace iteration and block Krylov (v = 2, 3 and Krylov 3, 4:
the final Krylov core is 500 wide).  Tolerances (north_star, fp32): sigma 1e-4 relative,
projectors 1e-3, residual within 1e-3 relative of the oracle's.
"""
import os

import numpy as np
import pytest
import torch

import oracle as O
import synth as S

pytestmark = pytest.mark.gpu

PANEL = 4096


@pytest.fixture(scope="module")
def ctx():
    from paper_1804_07531_b200 import build, rsvd

    build.build()
    c = rsvd.Context(0)
    yield c
    c.close()


def host64(t):
    return t.detach().cpu().numpy().astype(np.float64)


def _host_mem_available():
    try:
        import psutil

        return psutil.virtual_memory().available
    except Exception:
        return os.sysconf("SC_AVPHYS_PAGES") * os.sysconf("SC_PAGE_SIZE")


@pytest.fixture(scope="module")
def c5():
    free, _ = torch.cuda.mem_get_info()
    if free < 60e9:
        pytest.skip(f"C5 needs ~60 GB of free device memory, have {free / 1e9:.0f}")
    if _host_mem_available() < 100e9:
        pytest.skip("C5's oracle needs ~100 GB of host memory for the copied-back A (in fp64)")
    cfg = S.CONFIGS["C5"]
    dev = torch.device("cuda", 0)
    A = S.make_matrix_torch(cfg, dev, panel_rows=2048)
    Om = S.gaussian_test_matrix_torch(cfg.n, cfg.l, cfg, S.ROLE_OMEGA, dev)
    torch.cuda.synchronize()
    # the fp32 bytes, widened to fp64 (exact) on the device panel by panel: the oracle then runs
    # its fp64 views straight on BLAS (no per-view host upcast)
    Ah = np.empty((cfg.m, cfg.n), dtype=np.float64)
    for r0 in range(0, cfg.m, PANEL):
        Ah[r0:r0 + PANEL] = A[r0:r0 + PANEL].double().cpu().numpy()
    yield cfg, A, Ah, Om
    del A, Ah
    torch.cuda.empty_cache()


@pytest.mark.parametrize("alg,v", [("subspace", 2), ("subspace", 3), ("krylov", 3), ("krylov", 4)])
def test_c5_vs_oracle(ctx, c5, alg, v):
    cfg, A, Ah, Om = c5
    fn = ctx.subspace if alg == "subspace" else ctx.block_krylov
    U, s, V, info = fn(A, cfg.k, cfg.p, v, Om)
    assert U.dtype == torch.float32 and info.views == v
    U, s, V = host64(U), host64(s), host64(V)
    Uo, so, Vo, _ = O.svd_of(Ah, alg, cfg.k, cfg.p, v=v, Omega=host64(Om), panel_rows=PANEL)
    assert np.max(np.abs(s - so) / so) <= 1e-4
    assert O.projector_distance(U, Uo) <= 1e-3
    assert O.projector_distance(V, Vo) <= 1e-3
    r, ro = O.residual_fro(Ah, U, s, V, panel=PANEL), O.residual_fro(Ah, Uo, so, Vo, panel=PANEL)
    assert abs(r - ro) <= 1e-3 * ro
    # any size: orthonormal factors (fp32 outputs)
    np.testing.assert_allclose(U.T @ U, np.eye(cfg.k), atol=2e-5)
    np.testing.assert_allclose(V.T @ V, np.eye(cfg.k), atol=2e-5)
