"""Symmetric (upper-triangle) vs full-matrix matvec on the configs: agreement, L2-flushed
matvec time, PCG iterations per second (development aid; `python tools/symv_probe.py 1 2 5`)."""
import ctypes as C
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_09204_b200 import screenbem as S  # noqa: E402

cfgs = [int(a) for a in sys.argv[1:]] or [1, 2, 3, 4, 5]
ctx = S.Context(0)
ctx.timers(True)
L_ = S.lib()
for cfg in cfgs:
    pair = S.make_config(cfg)
    fine, coarse = S.inflate(pair.fine, validate=False), S.inflate(pair.coarse)
    W = S.assemble_W(fine, ctx=ctx)
    n = W.n
    L = S.assemble_rhs(fine, S.config_g(cfg), ctx=ctx)
    prec = S.build_preconditioner(W, S.partition_dofs(pair, fine), S.build_prolongation(pair, coarse, fine))
    x = np.random.default_rng(0).standard_normal(n)
    ldp = (n + 31) // 32 * 32
    dx, dy = C.c_void_p(), C.c_void_p()
    S._check(L_.sbg_device_alloc(ctx.h, 8 * ldp, C.byref(dx)))
    S._check(L_.sbg_device_alloc(ctx.h, 8 * ldp, C.byref(dy)))
    S._check(L_.sbg_memcpy_h2d(ctx.h, dx, x.ctypes.data_as(C.c_void_p), 8 * n))
    out = {}
    for form in ("full", "symmetric"):
        ctx.matvec_form = form
        y = W.matvec(x)
        for _ in range(3):
            S._check(L_.sbg_matvec_device(ctx.h, W.h, dx, dy, 1))
        ctx.reset_timers()
        for _ in range(20):
            ctx.l2_flush()
            S._check(L_.sbg_matvec_device(ctx.h, W.h, dx, dy, 1))
        ms, cnt = ctx.timer("gemv_f64")
        rep = S.pcg(W, prec, L, 1e-8)
        ctx.reset_timers()
        t0 = time.perf_counter()
        reps = 5
        for _ in range(reps):
            rep = S.pcg(W, prec, L, 1e-8)
        wall = (time.perf_counter() - t0) / reps
        pms = ctx.timer("pcg")[0] / reps
        out[form] = (y, rep)
        print(f"cfg {cfg} n {n} {form:9s}: matvec {1e3 * ms / cnt:8.1f} us (L2 flushed)  pcg {rep.iterations} it "
              f"{pms:.3f} ms = {rep.iterations / pms * 1e3:.0f} it/s (wall {wall * 1e3:.3f} ms)", flush=True)
    (yf, rf), (ys, rs) = out["full"], out["symmetric"]
    print(f"cfg {cfg}: max|y_sym - y_full| / max|y| = {np.abs(ys - yf).max() / np.abs(yf).max():.2e}; "
          f"pcg x rel diff {np.linalg.norm(rs.solution - rf.solution) / np.linalg.norm(rf.solution):.2e}", flush=True)
    L_.sbg_device_free(dx)
    L_.sbg_device_free(dy)
    del W, prec
    ctx.matvec_form = "symmetric"
