"""CholeskyQR2 time and accuracy by width (k_chol_fused vs RSVD_CHOL_OLD=1):
python tools/orth_cmp.py rows w..."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1804_07531_b200 import build, rsvd  # noqa: E402

build.build()
rows = int(sys.argv[1])
ctx = rsvd.Context(0)
for w in [int(x) for x in sys.argv[2:]]:
    g = torch.Generator(device="cuda")
    g.manual_seed(1)
    Y = (torch.randn(w, rows, generator=g, device="cuda", dtype=torch.float64) *
         torch.logspace(0, -6, w, device="cuda", dtype=torch.float64)[:, None]).t()
    for _ in range(3):
        Q, R, info = ctx.orth(Y)
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        Q, R, info = ctx.orth(Y)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    orth = (Q.t() @ Q - torch.eye(w, device="cuda", dtype=torch.float64)).abs().max().item()
    res = ((Q @ R - Y).norm() / Y.norm()).item()
    print(f"rows={rows} w={w:4d} {os.environ.get('RSVD_CHOL_OLD', '0')} orth_ms={ts[len(ts) // 2]:.3f} "
          f"|QtQ-I|={orth:.2e} |QR-Y|/|Y|={res:.2e} deficient={info.rank_deficient_cols}", flush=True)
