"""Full-W parity report (device vs oracle) for a config: norm-relative and per-entry worst
errors for the fast and the exact far-field paths (development aid; numbers go to DESIGN.md)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_2310_09204_b200 import screenbem as S  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
ctx = S.Context(0)
pair = S.make_config(cfg)
im = S.inflate(pair.fine, validate=False)
Wo = O.assemble_W(O.inflate(O.Mesh(pair.fine.vertices, pair.fine.facets), validate=False),
                  workers=os.cpu_count() or 1)
scale = np.abs(Wo).max()
for exact in (False, True):
    Wg = S.assemble_W(im, S.QuadratureConfig(exact_far=exact), ctx=ctx).download()
    err = np.abs(Wg - Wo)
    rel = err / np.maximum(np.abs(Wo), 1e-300)
    slack = err / (1e-10 * np.abs(Wo) + 1e-13 * scale)
    print(f"config {cfg} exact_far={exact}: max|dW|/max|W| = {err.max() / scale:.3e}, "
          f"max per-entry rel = {rel.max():.3e} (at |W_ij|/max|W| = {np.abs(Wo).flat[rel.argmax()] / scale:.2e}), "
          f"worst use of the per-entry bound = {slack.max():.3e}, bitwise-equal entries = {(Wg == Wo).mean():.4f}",
          flush=True)
