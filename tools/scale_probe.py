"""Beyond the BASELINE configs: a flat screen with m x m cells (default 256: 131 072 triangles,
65 025 DOFs, a 33.8 GB W) through assembly, preconditioner and PCG — checks the 64-bit
indexing and the memory layout at sizes the configs do not reach (development aid)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2310_09204_b200 import screenbem as S  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 256
r = int(sys.argv[2]) if len(sys.argv) > 2 else 16
ctx = S.Context(0)
ctx.timers(True)
pair = S.make_panels(0, m, r)
fine, coarse = S.inflate(pair.fine, validate=False), S.inflate(pair.coarse)
nf = pair.fine.nf
print(f"m={m}: {nf} triangles, {fine.n} DOFs, W {8.0 * fine.n * fine.n / 1e9:.1f} GB", flush=True)
part, P = S.partition_dofs(pair, fine), S.build_prolongation(pair, coarse, fine)
plan = S.AssemblyPlan(fine, ctx=ctx)
W = plan.run(None)
ctx.synchronize()
ctx.reset_timers()
W = plan.run(W)
ctx.synchronize()
t_asm = ctx.timer("assemble_W")[0]
print(f"assembly {t_asm:.1f} ms = {nf * (nf + 1) / 2 / (t_asm * 1e-3):.3e} tri-pairs/s; far {ctx.timer('far_tiles')[0]:.1f} "
      f"near {ctx.timer('near')[0]:.1f} sauter {ctx.timer('sauter')[0]:.1f}; symmetry defect {W.symmetry_defect()}",
      flush=True)
L = S.assemble_rhs(fine, [0.0, 0.0, 1.0], ctx=ctx)
ctx.reset_timers()
prec = S.build_preconditioner(W, part, P)
rep = S.pcg(W, prec, L, 1e-8)
print(f"build_preconditioner {ctx.timer('build_preconditioner')[0]:.1f} ms, PCG {rep.iterations} it in "
      f"{ctx.timer('pcg')[0]:.1f} ms, converged {rep.converged}, kappa_lanczos {rep.kappa_estimate:.3f}, "
      f"|x| {np.linalg.norm(rep.solution):.6e}; pool {[round(v / 1e9, 1) for v in ctx.pool_stats()]} GB", flush=True)
# the solution of the same problem on the coarser config-5 mesh scaled: sanity only (energy positive)
print("energy", float(L @ rep.solution))
