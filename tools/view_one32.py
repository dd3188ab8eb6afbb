"""One fp32 (tcgen05 3xTF32) view launch pair on a C5-shaped slab (for ncu --set full)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_1804_07531_b200 import rsvd
m = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
n = int(sys.argv[2]) if len(sys.argv) > 2 else 100000
w = int(sys.argv[3]) if len(sys.argv) > 3 else 250
ctx = rsvd.Context(0)
A = torch.randn(m, n, dtype=torch.float32, device="cuda")
X = torch.randn(w, n, dtype=torch.float32, device="cuda").t()
Y = torch.randn(w, m, dtype=torch.float32, device="cuda").t()
for _ in range(2):
    ctx.view(A, X, trans=False, flags=rsvd.RSVD_NO_GRAPH)
    ctx.view(A, Y, trans=True, flags=rsvd.RSVD_NO_GRAPH)
torch.cuda.synchronize()
print("ok")
