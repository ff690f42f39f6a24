"""Quick timing probe: assembly / matvec / preconditioner / PCG per config (development aid)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2310_09204_b200 import screenbem as S

ctx = S.Context(0)
ctx.timers(True)
cfgs = [int(c) for c in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["1", "2", "3"])]
for cfg in cfgs:
    pair = S.make_config(cfg)
    fine = S.inflate(pair.fine, validate=False)
    coarse = S.inflate(pair.coarse)
    nf = pair.fine.nf
    for rep in range(2):
        ctx.reset_timers()
        t0 = time.time()
        W = S.assemble_W(fine, ctx=ctx)
        ctx.synchronize()
        t1 = time.time()
        names = ["far_tiles", "near", "near_leaves", "sauter", "classify", "local_scatter", "mirror"]
        tm = {n: ctx.timer(n)[0] for n in names}
    npairs = nf * (nf + 1) // 2
    print(f"cfg{cfg}: nf={nf} n={fine.n} assemble wall {1e3*(t1-t0):.1f} ms -> {npairs/(t1-t0):.3e} pairs/s; "
          + " ".join(f"{k}={v:.2f}ms" for k, v in tm.items()), W.stats, flush=True)
    g = S.config_g(cfg)
    L = S.assemble_rhs(fine, g, ctx=ctx)
    t0 = time.time()
    P = S.build_prolongation(pair, coarse, fine)
    part = S.partition_dofs(pair, fine)
    t1 = time.time()
    ctx.reset_timers()
    prec = S.build_preconditioner(W, part, P)
    ctx.synchronize()
    t2 = time.time()
    print(f"   host partition+prolong {1e3*(t1-t0):.1f} ms; build_prec wall {1e3*(t2-t1):.1f} ms "
          f"(cholesky {ctx.timer('cholesky')[0]:.2f} ms, coarse {ctx.timer('coarse_galerkin')[0]:.2f} ms)", flush=True)
    ctx.reset_timers()
    t0 = time.time()
    rep = S.pcg(W, prec, L, 1e-8)
    t1 = time.time()
    gm, gc = ctx.timer("gemv_f64")
    pm, pc = ctx.timer("precond_apply")
    n = fine.n
    ld = (n + 31) // 32 * 32
    gb = 8.0 * n * ld / 1e9
    print(f"   pcg {rep.iterations} it in {1e3*(t1-t0):.1f} ms wall; gemv {gm/max(gc,1)*1e3:.1f} us/launch "
          f"({gb/max(gm/max(gc,1)/1e3,1e-12):.0f} GB/s incl padding), precond apply {pm/max(pc,1)*1e3:.1f} us; kappa {rep.kappa_estimate:.3f}",
          flush=True)
