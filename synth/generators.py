"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO arithmetic of the randomized-SVD method (no views, no QR of a
sketch, no SVD of a core).  It only draws random numbers and assembles the test
matrices whose recipes are stated in BASELINE.json ``configs`` and in the paper's
experiments section (§8.1).  Both the oracle (``oracle/``)
and the CUDA path (``paper_1804_07531_b200``) receive the *same bytes* produced
here; neither side imports the other.

Seeding: every array is drawn from NumPy PCG64 keyed by
``SeedSequence([1804, 7531, config_id, role, *extra])``.
Roles: 0 = U/X factor, 1 = V/Y factor, 2 = noise G, 3 = Omega (range test matrix,
paper Omega_r), 4 = Phi (co-range test matrix, paper Omega_c, P:667b),
5 = Omega_m (test matrix for the transposed input), 6 = misc test draws.

Large configs (C3 full size and up) can be built on a CUDA device with torch
(``make_matrix_torch``); the recipe is the same formula with torch's generator, so
the bytes differ from the NumPy ones.  Parity at those sizes compares the GPU
result with oracle computations on bytes copied back from the device.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

SEED_BASE = (1804, 7531)

ROLE_U, ROLE_V, ROLE_NOISE, ROLE_OMEGA, ROLE_PHI, ROLE_OMEGA_M, ROLE_MISC = range(7)


def rng(config_id: int, role: int, *extra: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([*SEED_BASE, config_id, role, *extra])))


def gaussian(shape, config_id: int, role: int, *extra: int, dtype=np.float64, order="C") -> np.ndarray:
    """i.i.d. N(0,1) entries (paper randn), drawn in fp64 then cast once."""
    g = rng(config_id, role, *extra).standard_normal(size=shape)
    return np.asarray(g, dtype=dtype, order=order)


def orthonormal_columns(rows: int, cols: int, config_id: int, role: int) -> np.ndarray:
    """Haar-distributed orthonormal columns: Q of qr(Gaussian) with diag(R) made >= 0.

    This is input construction (BASELINE.json configs: "Haar-random U,V (QR of seeded
    Gaussian)"), not the method's own QR.
    """
    g = gaussian((rows, cols), config_id, role)
    q, r = np.linalg.qr(g)
    s = np.sign(np.diag(r))
    s[s == 0] = 1.0
    return q * s


# ---------------------------------------------------------------- spectra (closed forms)

def sigma_c1(N: int) -> np.ndarray:
    """C1: sigma_i = 1 for i <= 10, (i-9)^-2 after (1-based i).  PolyFast-like (rho=2)."""
    i = np.arange(1, N + 1, dtype=np.float64)
    return np.where(i <= 10, 1.0, np.maximum(i - 9.0, 1.0) ** -2.0)


def sigma_c2(N: int) -> np.ndarray:
    """C2: sigma_i = 1 for i <= 20, 10^(-0.25 (i-20)) after.  ExpSlow-like (theta=0.25)."""
    i = np.arange(1, N + 1, dtype=np.float64)
    return np.where(i <= 20, 1.0, 10.0 ** (-0.25 * (i - 20.0)))


def sigma_c4(R: int) -> np.ndarray:
    """C4: sigma_i = i^-1.5, i = 1..R (R = 500)."""
    return np.arange(1, R + 1, dtype=np.float64) ** -1.5


def sigma_c5(R: int) -> np.ndarray:
    """C5: sigma_i = exp(-i/100), i = 1..R (R = 1000)."""
    return np.exp(-np.arange(1, R + 1, dtype=np.float64) / 100.0)


# paper test matrices, n = 1000, R = 10
def paper_poly(n: int = 1000, R: int = 10, rho: float = 1.0) -> np.ndarray:
    """diag(1,...,1 (R times), 2^-rho, 3^-rho, ..., (n-R+1)^-rho)."""
    tail = np.arange(2, n - R + 2, dtype=np.float64) ** (-rho)
    return np.concatenate([np.ones(R), tail])


def paper_exp(n: int = 1000, R: int = 10, theta: float = 0.25) -> np.ndarray:
    """diag(1,...,1 (R times), 10^-theta, 10^-2theta, ..., 10^-(n-R)theta)."""
    tail = 10.0 ** (-theta * np.arange(1, n - R + 1, dtype=np.float64))
    return np.concatenate([np.ones(R), tail])


def paper_lowrank_noise(n: int = 1000, R: int = 10, eta: float = 1e-2, seed_extra: int = 0) -> np.ndarray:
    """diag(1..1 (R), 0..0) + sqrt(eta R / (2 n^2)) (G + G^T)."""
    G = gaussian((n, n), 100, ROLE_NOISE, seed_extra)
    A = math.sqrt(eta * R / (2.0 * n * n)) * (G + G.T)
    A[np.arange(R), np.arange(R)] += 1.0
    return A


# ---------------------------------------------------------------- BASELINE.json configs

@dataclass(frozen=True)
class Config:
    name: str
    cid: int
    m: int
    n: int
    k: int
    p: int
    dtype: str          # "f64" | "f32"
    kind: str           # "haar" | "lowrank_noise"
    rank: int = 0       # for lowrank_noise
    noise: float = 0.0  # absolute noise scale
    l2_factor: int = 2  # single-pass l2 = 2 (k+p)   (SURVEY c-6)
    runs: dict = field(default_factory=dict)

    @property
    def l(self) -> int:
        return self.k + self.p

    @property
    def l2(self) -> int:
        return self.l2_factor * self.l

    @property
    def np_dtype(self):
        return np.float64 if self.dtype == "f64" else np.float32

    @property
    def itemsize(self) -> int:
        return 8 if self.dtype == "f64" else 4


CONFIGS = {
    "C1": Config("C1", 1, 200, 200, 10, 10, "f64", "haar",
                 runs=dict(subspace=[2, 3, 4], krylov=[2, 3, 4], single_pass=True)),
    "C2": Config("C2", 2, 4000, 4000, 20, 10, "f64", "haar",
                 runs=dict(subspace=[2, 3, 4, 5, 6], krylov=[3, 4, 5], single_pass=True)),
    "C3": Config("C3", 3, 20000, 8000, 50, 20, "f64", "lowrank_noise", rank=50,
                 noise=math.sqrt(1e-4 / 8000.0),
                 runs=dict(subspace=[2, 3, 4, 5], krylov=[2, 3, 4, 5], single_pass=True)),
    "C4": Config("C4", 4, 50000, 200000, 100, 20, "f64", "lowrank_noise", rank=500, noise=1e-8,
                 runs=dict(krylov=[3], single_pass=True, normal=[3])),
    "C5": Config("C5", 5, 100000, 100000, 200, 50, "f32", "lowrank_noise", rank=1000, noise=1e-6,
                 runs=dict(subspace=[2, 3, 4, 5, 6, 7], krylov=[3, 4, 5])),
}


def config_sigma(cfg: Config, N: int) -> np.ndarray:
    """Singular values of the noise-free part, length N (zeros past the rank)."""
    if cfg.name == "C1":
        return sigma_c1(N)
    if cfg.name == "C2":
        return sigma_c2(N)
    out = np.zeros(N)
    if cfg.name == "C3":
        s = np.ones(cfg.rank)
    elif cfg.name == "C4":
        s = sigma_c4(cfg.rank)
    else:
        s = sigma_c5(cfg.rank)
    r = min(N, cfg.rank)
    out[:r] = s[:r]
    return out


def make_matrix(cfg: Config, m: int | None = None, n: int | None = None) -> np.ndarray:
    """The config's A (row-major, C order), optionally at a reduced shape (same recipe).

    haar:           A = U diag(sigma) V^T, U (m x N), V (n x N) Haar, N = min(m, n)
    lowrank_noise:  A = X diag(sigma) Y^T + noise * G, X, Y orthonormalised Gaussian of rank R
    """
    m = cfg.m if m is None else m
    n = cfg.n if n is None else n
    if cfg.kind == "haar":
        N = min(m, n)
        U = orthonormal_columns(m, N, cfg.cid, ROLE_U)
        V = orthonormal_columns(n, N, cfg.cid, ROLE_V)
        A = (U * config_sigma(cfg, N)) @ V.T
    else:
        R = min(cfg.rank, m, n)
        X = orthonormal_columns(m, R, cfg.cid, ROLE_U)
        Y = orthonormal_columns(n, R, cfg.cid, ROLE_V)
        A = (X * config_sigma(cfg, R)) @ Y.T
        A += cfg.noise * gaussian((m, n), cfg.cid, ROLE_NOISE)
    return np.ascontiguousarray(A.astype(cfg.np_dtype))


def gaussian_test_matrix(rows: int, width: int, cfg: Config, role: int, *extra: int) -> np.ndarray:
    """Gaussian test matrix (Omega: role 3, Phi: role 4), stored column-major (rows x width, F order):
    each of the ``width`` test vectors is contiguous, the layout the C ABI takes."""
    g = gaussian((width, rows), cfg.cid, role, *extra)
    return np.asarray(g.T.astype(cfg.np_dtype), order="F")


def exact_rank_matrix(m: int, n: int, sigma: np.ndarray, seed: int) -> np.ndarray:
    """A = X diag(sigma) Y^T with X, Y Haar orthonormal (m x r, n x r); exact rank r = len(sigma)."""
    r = len(sigma)
    X = orthonormal_columns(m, r, 200 + seed, ROLE_U)
    Y = orthonormal_columns(n, r, 200 + seed, ROLE_V)
    return np.ascontiguousarray((X * sigma) @ Y.T)


def exact_rank_factors(m: int, n: int, r: int, seed: int):
    X = orthonormal_columns(m, r, 200 + seed, ROLE_U)
    Y = orthonormal_columns(n, r, 200 + seed, ROLE_V)
    return X, Y


def random_gaussian_matrix(m: int, n: int, seed: int, dtype=np.float64) -> np.ndarray:
    return gaussian((m, n), 300, ROLE_MISC, seed, dtype=dtype)


def integer_matrix(m: int, n: int, lo: int, hi: int, seed: int, dtype=np.float64, order="C") -> np.ndarray:
    """Integer-valued entries in [lo, hi]; every partial sum of products stays exact in fp64
    (|sum| < 2^53), so a view computed in any summation order is bit-exact."""
    g = rng(400, ROLE_MISC, seed).integers(lo, hi + 1, size=(m, n))
    return np.asarray(g.astype(dtype), order=order)


# ---------------------------------------------------------------- torch (device) builders

def srft_matrix(n: int, s: int, seed: int) -> np.ndarray:
    """A subsampled randomized Fourier transform test matrix Phi = D F P (n x s) for real A
    (P:806-812): D = diag of Rademacher signs, F = the orthonormal DCT-II matrix (n x n), P = s
    columns of I_n sampled without replacement.  Random test matrices are inputs of the method
    (reading R3): this only draws one; it is materialised dense (the GPU applies it as a dense
    test matrix in the same view).  Columns are orthonormal (F orthogonal)."""
    if not (1 <= s <= n):
        raise ValueError("need 1 <= s <= n")
    from scipy.fft import dct
    g = np.random.default_rng(np.random.SeedSequence([0x5A7F, seed]))
    d = g.choice(np.array([-1.0, 1.0]), size=n)
    cols = np.sort(g.choice(n, size=s, replace=False))
    F = dct(np.eye(n), type=2, norm="ortho", axis=0)   # F[:, j] = DCT-II of e_j
    return (d[:, None] * F)[:, cols]


NOISE_PANEL = 2048   # rows per seeded noise panel of the device-built matrices


def make_matrix_torch(cfg: Config, device, m: int | None = None, n: int | None = None,
                      panel_rows: int = NOISE_PANEL, seed_offset: int = 0, row0: int = 0, rows: int | None = None):
    """Same recipe as ``make_matrix`` built on a CUDA device with torch's Philox generator
    (for the multi-GB configs).  Haar factors use torch.linalg.qr of a Gaussian; this is input
    construction, not the method.  Returns a row-major torch tensor of cfg's dtype.

    row0 / rows select a row block [row0, row0 + rows) of the m x n matrix (a rank's shard): the
    noise is drawn in fixed panels of NOISE_PANEL rows, each from its own seed, and the factors are
    built whole, so the block's bytes equal those rows of the full matrix for any sharding.
    (panel_rows is accepted for compatibility; the noise panel grid is fixed.)"""
    import torch

    m = cfg.m if m is None else m
    n = cfg.n if n is None else n
    rows = m - row0 if rows is None else rows
    tdt = torch.float64 if cfg.dtype == "f64" else torch.float32
    gen = torch.Generator(device=device)
    base = (SEED_BASE[0] * 1_000_003 + SEED_BASE[1]) * 101 + cfg.cid * 7 + seed_offset

    def orth(nrows, cols, role):
        gen.manual_seed(base * 13 + role)
        g = torch.randn(nrows, cols, generator=gen, device=device, dtype=torch.float64)
        q, r = torch.linalg.qr(g)
        s = torch.sign(torch.diagonal(r))
        s[s == 0] = 1.0
        return q * s

    if cfg.kind == "haar":
        N = min(m, n)
        U = orth(m, N, ROLE_U)[row0:row0 + rows]
        V = orth(n, N, ROLE_V)
        sig = torch.as_tensor(config_sigma(cfg, N), device=device)
        return ((U * sig) @ V.T).to(tdt).contiguous()
    R = min(cfg.rank, m, n)
    Xs = orth(m, R, ROLE_U)[row0:row0 + rows] * torch.as_tensor(config_sigma(cfg, R), device=device)
    Y = orth(n, R, ROLE_V)
    A = torch.empty(rows, n, dtype=tdt, device=device)
    P = NOISE_PANEL
    for p0 in range((row0 // P) * P, row0 + rows, P):       # global noise panels overlapping the block
        gen.manual_seed(base * 13 + ROLE_NOISE + 1_000_003 * (p0 // P + 1))
        G = torch.randn(min(P, m - p0), n, generator=gen, device=device, dtype=torch.float64)
        a0, a1 = max(p0, row0), min(p0 + P, row0 + rows, m)
        blk = Xs[a0 - row0:a1 - row0] @ Y.T
        blk += cfg.noise * G[a0 - p0:a1 - p0]
        A[a0 - row0:a1 - row0] = blk.to(tdt)
        del blk, G
    return A


def gaussian_test_matrix_torch(rows: int, width: int, cfg: Config, role: int, device, seed_offset: int = 0):
    """Gaussian test matrix on device, column-major (returned as the transposed view of a
    width x rows row-major tensor, so each test vector is contiguous)."""
    import torch

    tdt = torch.float64 if cfg.dtype == "f64" else torch.float32
    gen = torch.Generator(device=device)
    gen.manual_seed(((SEED_BASE[0] * 1_000_003 + SEED_BASE[1]) * 101 + cfg.cid * 7 + seed_offset) * 13 + role)
    g = torch.randn(width, rows, generator=gen, device=device, dtype=torch.float64).to(tdt)
    return g.T  # rows x width, column-major view
