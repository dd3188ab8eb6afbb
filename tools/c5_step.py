"""One C5-shaped fp32 SVD call (after one warm-up) for ncu launch lists.
usage: python tools/c5_step.py [subspace|krylov] [v] [m] [n]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

from paper_1804_07531_b200 import rsvd

alg = sys.argv[1] if len(sys.argv) > 1 else "subspace"
v = int(sys.argv[2]) if len(sys.argv) > 2 else 2
m = int(sys.argv[3]) if len(sys.argv) > 3 else 100000
n = int(sys.argv[4]) if len(sys.argv) > 4 else 100000
ctx = rsvd.Context(0)
A = torch.empty(m, n, dtype=torch.float32, device="cuda")
for r0 in range(0, m, 8192):
    A[r0:r0 + 8192].normal_()
Om = torch.randn(250, n, dtype=torch.float32, device="cuda").t()
fn = ctx.subspace if alg == "subspace" else ctx.block_krylov
for i in range(2):
    U, s, V, info = fn(A, 200, 50, v, Om)
    torch.cuda.synchronize()
print("ok", info.kernel_launches)
