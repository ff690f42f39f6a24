"""eval_DL throughput (development aid): the config-c solution's double-layer potential on an
n x n grid of [-2, 2]^2 in z = 0 (masked within 1e-3 of the screen) plus a plane of points at
z = 0.05, on the device (fast and exact_far forms), and the CPU restatement on a point sample.
`python tools/dl_probe.py 5 64`"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_09204_b200 import screenbem as S  # noqa: E402
from oracle import oracle as O  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
ng = int(sys.argv[2]) if len(sys.argv) > 2 else 64
ctx = S.Context(0)
ctx.timers(True)
pair = S.make_config(cfg)
res = S.solve(pair, S.config_g(cfg), 1e-8, ctx=ctx)
im = S.inflate(pair.fine, validate=False)
v = res.report.solution
g = S.make_cartesian_grid(pair.fine, -2, 2, ng, ng, 1e-3, ctx=ctx).points
lift = g.copy()
lift[:, 2] = 0.05
pts = np.concatenate([g, lift])
nf = len(pair.fine.facets)
for exact in (False, True):
    qc = S.QuadratureConfig(exact_far=exact)
    S.eval_DL(v, im, pts[:64], qc, ctx=ctx)
    ctx.reset_timers()
    t0 = time.perf_counter()
    u = S.eval_DL(v, im, pts, qc, ctx=ctx)
    wall = time.perf_counter() - t0
    ms = ctx.timer("eval_dl")[0]
    pairs = len(pts) * nf
    print(f"cfg {cfg} exact_far={exact}: {len(pts)} points x {nf} facets: device {ms:.2f} ms, wall {wall * 1e3:.2f} ms, "
          f"{pairs / (ms * 1e-3):.3e} point-facet pairs/s, {pairs * 36 / (ms * 1e-3):.3e} rule evaluations/s", flush=True)
    if exact:
        ue = u
    else:
        uf = u
print("fast vs exact: max |diff| / max |U| = %.2e" % (np.abs(uf - ue).max() / np.abs(ue).max()))
# CPU restatement on a sample of points (all host threads)
om = O.Mesh(pair.fine.vertices, pair.fine.facets)
oim = O.inflate(om, validate=False)
k = 32
sel = np.linspace(0, len(pts) - 1, k).astype(int)
t0 = time.perf_counter()
uo = O.eval_DL(v, oim, pts[sel])
tc = time.perf_counter() - t0
print(f"oracle: {k} points in {tc:.2f} s on {os.cpu_count()} threads = {k * nf / tc:.3e} pairs/s; "
      f"exact_far device == oracle on the sample: {np.array_equal(ue[sel], uo)}")
