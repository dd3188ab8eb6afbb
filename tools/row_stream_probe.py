"""Single pass over the rows (rsvd_row_stream) vs Alg. 2 with v = 2 (rsvd_subspace): device time
(CUDA events, graph replay, L2 flushed before each rep) at C2 and C3.  Run under ncu with
dram__bytes_read.sum to see the view kernels read A once (row stream) vs twice (subspace)."""
import json, os, statistics, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import synth as S
from paper_1804_07531_b200 import rsvd

ctx = rsvd.Context(0)
dev = torch.device("cuda", 0)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
reps = int(os.environ.get("REPS", "5"))
for name in (sys.argv[1:] or ["C2", "C3"]):
    cfg = S.CONFIGS[name]
    A = S.make_matrix_torch(cfg, dev)
    Om = S.gaussian_test_matrix_torch(cfg.n, cfg.l, cfg, S.ROLE_OMEGA, dev)
    out = {"config": name}
    for alg, fn in (("row_stream", lambda: ctx.row_stream(A, cfg.k, cfg.p, Om)),
                    ("subspace_v2", lambda: ctx.subspace(A, cfg.k, cfg.p, 2, Om))):
        fn()
        ts = []
        for _ in range(reps):
            flush.zero_()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        out[alg + "_ms"] = statistics.median(ts)
    print(json.dumps(out), flush=True)
