"""Generates the committed golden fixtures of tests/golden/ from the CPU restatement
(oracle/, itself pinned against the reference's known-answer tests and recorded numbers,
tests/test_oracle_pins.py).  Re-run only when the oracle changes:

    python tests/golden/make_golden.py

Fixtures (small, seeded, deterministic):
  cfg1.npz    config 1 (flat 16x16, H/h 8): DOF count, W (225x225), RHS for g = (0,0,1),
              partition (face ids/ptr/dofs, wire-basket), prolongation (CSC), preconditioned
              PCG to 1e-8 (iterations, solution, residual history), condition numbers.
  bowtie2.npz bow-tie refined twice (3-D junction geometry): pair integrals of every class on
              all facet pairs, W, RHS for g = (0.3, -0.2, 1).
  recorded.json  numbers the reference itself recorded (proj/test_output.txt:31-32).
"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_2310_09204_b200 import screenbem as S  # noqa: E402  (host-side config generator only)


def cfg1():
    pair = S.make_config(1)
    opair = O.LevelPair(O.Mesh(pair.coarse.vertices, pair.coarse.facets),
                        O.Mesh(pair.fine.vertices, pair.fine.facets), pair.parent)
    fine, coarse = O.inflate(opair.fine), O.inflate(opair.coarse)
    W = O.assemble_W(fine, workers=1)
    L = O.assemble_rhs(fine, [0.0, 0.0, 1.0])
    part = O.partition_dofs(opair, fine)
    R = O.build_prolongation(opair, coarse, fine)
    prec = O.build_preconditioner(W, part, R)
    rep = O.pcg(W, prec, L, 1e-8)
    lmin, lmax, kap = O.condition_number(W, prec)
    kraw = O.condition_number(W)[2]
    np.savez_compressed(os.path.join(HERE, "cfg1.npz"), vertices=np.asarray(pair.fine.vertices),
                        facets=np.asarray(pair.fine.facets), n=fine.n, W=W, rhs=L,
                        face_ids=part.face_ids, face_ptr=part.face_ptr, face_dofs=part.face_dofs,
                        wirebasket=part.wirebasket, R_col_ptr=R.col_ptr, R_row=R.row_idx, R_val=R.val,
                        pcg_iterations=rep.iterations, pcg_solution=rep.solution,
                        pcg_history=rep.residual_history, kappa_prec=kap, lambda_min=lmin, lambda_max=lmax,
                        kappa_unprec=kraw)


def bowtie2():
    m = S.make_builtin("bowtie:2")
    om = O.Mesh(m.vertices, m.facets)
    f, g = np.tril_indices(om.nf)
    I = O.pair_integrals(om, f, g, workers=1)
    im = O.inflate(om)
    W = O.assemble_W(im, workers=1)
    L = O.assemble_rhs(im, [0.3, -0.2, 1.0])
    np.savez_compressed(os.path.join(HERE, "bowtie2.npz"), vertices=np.asarray(m.vertices),
                        facets=np.asarray(m.facets), pair_f=f.astype(np.int32), pair_g=g.astype(np.int32),
                        pair_I=I, W=W, rhs=L)


def recorded():
    rec = {"source": "reference proj/test_output.txt:31-32 (acceptance.cpp:175-221, test_assemble.cpp:246-258)",
           "bowtie_Hh16": {"dofs": 465, "kappa_prec_2dp": 6.93, "kappa_unprec_2dp": 12.96},
           "W_vs_adaptive_oracle_worst_rel": 1.31e-09}
    with open(os.path.join(HERE, "recorded.json"), "w") as fh:
        json.dump(rec, fh, indent=1)


if __name__ == "__main__":
    cfg1()
    bowtie2()
    recorded()
    print("golden fixtures written to", HERE)
