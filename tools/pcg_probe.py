"""PCG timing with a fresh vs a reused preconditioner (graph capture cost), development aid."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_09204_b200 import screenbem as S  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
ctx = S.Context(0)
ctx.timers(True)
pair = S.make_config(cfg)
fine, coarse = S.inflate(pair.fine, validate=False), S.inflate(pair.coarse)
part, P = S.partition_dofs(pair, fine), S.build_prolongation(pair, coarse, fine)
W = S.assemble_W(fine, ctx=ctx)
L = S.assemble_rhs(fine, S.config_g(cfg), ctx=ctx)
for fresh in (True, True, False, False, False):
    if fresh or "prec" not in dir():
        prec = S.build_preconditioner(W, part, P)
    ctx.reset_timers()
    t0 = time.perf_counter()
    rep = S.pcg(W, prec, L, 1e-8)
    t1 = time.perf_counter()
    print(f"fresh={fresh}: {rep.iterations} it, device {ctx.timer('pcg')[0]:.3f} ms, wall {1e3 * (t1 - t0):.3f} ms",
          flush=True)
