"""Input generators (synth/): the device builder's row blocks equal the rows of the full matrix for
any sharding (the multi-GPU bench builds each rank's shard on its own GPU), and the recipe's
construction values (no method arithmetic here)."""
import numpy as np
import torch

import synth as S
from paper_1804_07531_b200.sharding import shard_rows


def test_row_blocks_equal_rows_of_full_matrix():
    cfg = S.CONFIGS["C4"]
    m, n = 5000, 700                                 # not a multiple of the 2048-row noise panel
    dev = torch.device("cpu")
    full = S.make_matrix_torch(cfg, dev, m, n)
    for world in (2, 3, 8):
        parts = []
        for r in range(world):
            sh = shard_rows(m, world, r, align=128)
            parts.append(S.make_matrix_torch(cfg, dev, m, n, row0=sh.row0, rows=sh.m_local))
        assert torch.equal(torch.cat(parts), full)


def test_device_builder_recipe():
    """X diag(sigma) Y^T + noise G: the noise-free part has exactly the config's singular values."""
    cfg = S.CONFIGS["C5"]
    dev = torch.device("cpu")
    A = S.make_matrix_torch(cfg, dev, 1200, 1100).double().numpy()
    s = np.linalg.svd(A, compute_uv=False)
    sig = S.sigma_c5(cfg.rank)
    noise = cfg.noise * (np.sqrt(1200) + np.sqrt(1100)) * 1.1
    assert np.all(np.abs(s[:50] - sig[:50]) <= noise + 1e-6 * sig[0])   # fp32 rounding of A
