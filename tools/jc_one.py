"""One cluster Jacobi (core SVD) launch of width w for ncu: python tools/jc_one.py [w]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1804_07531_b200 import build, rsvd  # noqa: E402

build.build()
w = int(sys.argv[1]) if len(sys.argv) > 1 else 250
rng = np.random.default_rng(3)
m = 4 * w + 200
U, _ = np.linalg.qr(rng.standard_normal((m, m)))
V, _ = np.linalg.qr(rng.standard_normal((m, m)))
s = np.exp(-np.arange(m) / (w / 2.5)) + 1e-6
R = np.linalg.qr(((U * s) @ V.T) @ rng.standard_normal((m, w)))[1]
M = torch.from_numpy(np.ascontiguousarray(R)).cuda().t()
ctx = rsvd.Context(0)
for _ in range(2):
    ctx.core_svd(M, flags=rsvd.RSVD_CORE_NO_J)
torch.cuda.synchronize()
print("ok", flush=True)
