"""W x on one config's assembled W, `reps` times (development aid: ncu captures of the
matvec kernels; `python tools/matvec_probe.py 5 3`)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_09204_b200 import screenbem as S  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
ctx = S.Context(0)
pair = S.make_config(cfg)
W = S.assemble_W(S.inflate(pair.fine, validate=False), ctx=ctx)
x = np.random.default_rng(0).standard_normal(W.n)
for _ in range(reps):
    y = W.matvec(x)
print("n", W.n, "|y|", float(np.abs(y).max()))
