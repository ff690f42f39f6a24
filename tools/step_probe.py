"""Wall-clock breakdown of one solve step (assemble, rhs, preconditioner, PCG) with a
synchronize after each call (development aid; bench.py is the measurement)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_09204_b200 import screenbem as S  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
ratio = int(sys.argv[2]) if len(sys.argv) > 2 else (8 if cfg == 5 else 0)
ctx = S.Context(0)
ctx.timers(True)
pair = S.make_config(cfg, ratio)
fine, coarse = S.inflate(pair.fine, validate=False), S.inflate(pair.coarse)
part, P = S.partition_dofs(pair, fine), S.build_prolongation(pair, coarse, fine)
g = S.config_g(cfg)
plan = S.AssemblyPlan(fine, ctx=ctx)
W = prec = None
for rep in range(6):
    ctx.reset_timers()
    t = [time.perf_counter()]
    W = plan.run(W)
    ctx.synchronize()
    t.append(time.perf_counter())
    L = S.assemble_rhs(fine, g, ctx=ctx)
    t.append(time.perf_counter())
    if os.environ.get("FREE_FIRST"):
        prec = None
    t.append(time.perf_counter())
    prec = S.build_preconditioner(W, part, P)
    ctx.synchronize()
    t.append(time.perf_counter())
    res = S.pcg(W, prec, L, 1e-8)
    t.append(time.perf_counter())
    d = [1e3 * (b - a) for a, b in zip(t, t[1:])]
    dev = {k: round(ctx.timer(k)[0], 2) for k in ("assemble_W", "build_preconditioner", "cholesky", "block_inverse",
                                                   "coarse_galerkin", "pcg")}
    print(f"rep {rep}: assemble {d[0]:.1f}  rhs {d[1]:.1f}  free prec {d[2]:.1f}  build prec {d[3]:.1f}  "
          f"pcg {d[4]:.1f} ms wall ({res.iterations} it); device {dev}; pool (reserved, used) GB "
          f"{tuple(round(x / 1e9, 2) for x in ctx.pool_stats())}", flush=True)

# end-to-end pieces of S.assemble_W(host mesh) + W.download()
for rep in range(3):
    ctx.reset_timers()
    t = [time.perf_counter()]
    mesh = S.SurfaceMesh(pair.fine.vertices, pair.fine.facets)
    im = S.inflate(mesh, validate=False)
    t.append(time.perf_counter())
    pl = S.AssemblyPlan(im, ctx=ctx)
    ctx.synchronize()
    t.append(time.perf_counter())
    W2 = pl.run(None)
    ctx.synchronize()
    t.append(time.perf_counter())
    Wh = W2.download()
    t.append(time.perf_counter())
    d = [1e3 * (b - a) for a, b in zip(t, t[1:])]
    gbs = Wh.nbytes / (d[3] * 1e-3) / 1e9
    print(f"e2e rep {rep}: inflate {d[0]:.1f}  plan {d[1]:.1f}  run {d[2]:.1f}  download {d[3]:.1f} ms "
          f"({gbs:.1f} GB/s); device assemble_W {ctx.timer('assemble_W')[0]:.1f} ms, near {ctx.timer('near')[0]:.1f}, "
          f"far {ctx.timer('far_tiles')[0]:.1f}", flush=True)
    del W2, Wh, pl

# download into a fresh array vs a reused (already faulted) one
W3 = plan.run(None)
buf = None
for rep in range(3):
    t0 = time.perf_counter()
    a = W3.download()
    t1 = time.perf_counter()
    buf = W3.download(out=buf if buf is not None else a)
    t2 = time.perf_counter()
    print(f"download fresh {a.nbytes / (t1 - t0) / 1e9:.1f} GB/s, reused {a.nbytes / (t2 - t1) / 1e9:.1f} GB/s", flush=True)
