"""Build the config-5 (H/h 8) preconditioner twice and report device phase times
(development aid for the factorisation kernels)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_09204_b200 import screenbem as S  # noqa: E402

ratio = int(sys.argv[1]) if len(sys.argv) > 1 else 8
KEYS = ("build_preconditioner", "cholesky", "block_inverse", "inv_lower", "inv_lauum", "coarse_galerkin")
ctx = S.Context(0)
ctx.timers(True)
pair = S.make_config(5, ratio)
fine, coarse = S.inflate(pair.fine, validate=False), S.inflate(pair.coarse)
part, P = S.partition_dofs(pair, fine), S.build_prolongation(pair, coarse, fine)
W = S.assemble_W(fine, ctx=ctx)
for rep in range(3):
    ctx.reset_timers()
    prec = S.build_preconditioner(W, part, P)
    print({k: round(ctx.timer(k)[0], 2) for k in KEYS}, flush=True)
    del prec

# rebuild while the previous preconditioner is still alive (the bench's step pattern)
old = S.build_preconditioner(W, part, P)
for rep in range(3):
    ctx.reset_timers()
    new = S.build_preconditioner(W, part, P)
    print("keep-alive", {k: round(ctx.timer(k)[0], 2) for k in KEYS}, flush=True)
    old = new
