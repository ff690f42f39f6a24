"""Small end-to-end run for compute-sanitizer (memcheck / racecheck / synccheck):
config 1 assembly -> RHS -> preconditioner -> PCG, the near-field path of the C ABI's
pair_integrals, the row-panel PCG, and a preconditioner whose blocks span more than one
panel of tiles (WB of 580 DOFs = 10 tiles: panel steps, the look-ahead far update on the
second stream, the L^-1 row steps and LAUUM).

    compute-sanitizer --tool memcheck python tools/sanitize_probe.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402  (checker only)
from paper_2310_09204_b200 import screenbem as S  # noqa: E402

ctx = S.Context(0)
res = S.solve(S.make_config(1), [0.0, 0.0, 1.0], 1e-8, ctx=ctx)
assert res.report.converged
m = S.make_builtin("bowtie:1")
f, g = np.tril_indices(m.nf)
S.pair_integrals(m, f, g, ctx=ctx)
rows = S.row_ranges(res.W.n, 2)[1]
rep = S.pcg_rows(res.W, res.prec, res.rhs, rows,
                 lambda d_p, d_y, n, stream: S.matvec_rows_device(res.W, d_p, d_y, 0, rows[0]), 1e-8)
assert rep.iterations == res.report.iterations
W0 = O.random_spd(640, 5)
faces = {0: list(range(0, 60))}
wb = list(range(60, 640))
for mode in ("inverse", "trsv"):
    prec = S.build_preconditioner(S.GalerkinMatrix.from_host(W0, ctx), S.DofPartition.create(faces, wb),
                                  S.Prolongation.empty(640), mode)
    z = prec.apply(O.normal_draws(3, 640))
    zo = O.build_preconditioner(W0, O.partition_from(faces, wb), O.empty_prolongation(640)).apply(
        O.normal_draws(3, 640))
    assert np.abs(z - zo).max() <= 1e-10 * np.abs(zo).max(), mode
print("sanitize probe ok")
