"""RSVD_ASYNC: calls enqueue only and rsvd_wait completes them; three contexts on three streams
run concurrently and give bitwise the results of the synchronous calls."""
import numpy as np
import pytest
import torch

import synth as S

pytestmark = pytest.mark.gpu


def colmajor_dev(a):
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a).T)).cuda().t()


def test_async_concurrent_equals_sync():
    from paper_1804_07531_b200 import build, rsvd

    build.build()
    cfg = S.CONFIGS["C2"]
    A = torch.from_numpy(S.make_matrix(cfg)).cuda()
    Om = colmajor_dev(S.gaussian_test_matrix(cfg.n, cfg.l, cfg, S.ROLE_OMEGA))
    Phi = colmajor_dev(S.gaussian_test_matrix(cfg.m, cfg.l2, cfg, S.ROLE_PHI))
    streams = [torch.cuda.current_stream()] + [torch.cuda.Stream() for _ in range(2)]
    ctxs = [rsvd.Context(0, stream=s) for s in streams]
    calls = [lambda c, f: c.subspace(A, cfg.k, cfg.p, 3, Om, flags=f),
             lambda c, f: c.block_krylov(A, cfg.k, cfg.p, 4, Om, flags=f),
             lambda c, f: c.single_pass(A, cfg.k, cfg.p, cfg.l2, Om, Phi, flags=f)]
    ref = [[t.cpu().numpy() for t in fn(ctxs[0], 0)[:3]] for fn in calls]
    for rep in range(2):  # capture, then graph replay
        outs = []
        for c, s, fn in zip(ctxs, streams, calls):
            s.wait_stream(torch.cuda.current_stream())
            outs.append(fn(c, rsvd.RSVD_ASYNC))
        for c, o in zip(ctxs, outs):
            info = c.wait(o[3])
            assert info.status == 0
        torch.cuda.synchronize()
        for o, r in zip(outs, ref):
            for a, b in zip(o[:3], r):
                assert np.array_equal(a.cpu().numpy(), b)
    # a pending call blocks the context until rsvd_wait
    o = calls[0](ctxs[0], rsvd.RSVD_ASYNC)
    with pytest.raises(rsvd.RsvdError) as e:
        calls[0](ctxs[0], 0)
    assert e.value.code == -7
    ctxs[0].wait(o[3])
    for c in ctxs:
        c.close()


def test_sm_limit_same_results():
    """rsvd_set_sm_limit only resizes the persistent grids (reduction splits): results agree with the
    full-GPU context to rounding and with the oracle; n < 1 is an argument error."""
    import numpy as np
    import torch

    import oracle as O
    import synth as S
    from paper_1804_07531_b200 import build, rsvd

    build.build()
    cfg = S.CONFIGS["C2"]
    A = torch.from_numpy(S.make_matrix(cfg)).cuda()
    Om_h = S.gaussian_test_matrix(cfg.n, cfg.l, cfg, S.ROLE_OMEGA)
    Om = torch.from_numpy(np.ascontiguousarray(Om_h.T)).cuda().t()
    full, capped = rsvd.Context(0), rsvd.Context(0)
    capped.set_sm_limit(20)
    assert capped.sm_count == 20
    U0, s0, V0, _ = full.block_krylov(A, cfg.k, cfg.p, 4, Om)
    U1, s1, V1, _ = capped.block_krylov(A, cfg.k, cfg.p, 4, Om)
    s0, s1 = s0.cpu().numpy(), s1.cpu().numpy()
    assert np.max(np.abs(s1 - s0) / s0) <= 1e-12
    assert O.projector_distance(U1.cpu().numpy(), U0.cpu().numpy()) <= 1e-11
    Uo, so, Vo, _ = O.svd_of(A.cpu().numpy(), "krylov", cfg.k, cfg.p, v=4, Omega=Om_h)
    assert np.max(np.abs(s1 - so) / so) <= 1e-10
    with pytest.raises(rsvd.RsvdError):
        capped.set_sm_limit(0)
    capped.set_sm_limit(10_000)
    assert capped.sm_count == full.sm_count
    full.close()
    capped.close()
