"""One config's PCG, solved `reps` times after a warm-up (development aid: a launch list of
the PCG kernels under ncu; `python tools/pcg_probe.py 2 3`)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_09204_b200 import screenbem as S  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
ctx = S.Context(0)
pair = S.make_config(cfg)
fine, coarse = S.inflate(pair.fine, validate=False), S.inflate(pair.coarse)
W = S.assemble_W(fine, ctx=ctx)
L = S.assemble_rhs(fine, S.config_g(cfg), ctx=ctx)
prec = S.build_preconditioner(W, S.partition_dofs(pair, fine), S.build_prolongation(pair, coarse, fine))
for _ in range(reps):
    rep = S.pcg(W, prec, L, 1e-8)
print("iterations", rep.iterations)
