import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_1804_07531_b200 import rsvd
m, n, w, trans = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
ctx = rsvd.Context(0)
A = torch.randn(m, n, dtype=torch.float64, device="cuda")
X = torch.randn(w, n if trans == 0 else m, dtype=torch.float64, device="cuda").t()
for _ in range(3):
    Y, info = ctx.view(A, X, trans=bool(trans), flags=rsvd.RSVD_NO_GRAPH)
torch.cuda.synchronize()
print("ok")
