"""Where the e2e time of bench.py goes (development aid): S.assemble_W(host InflatedMesh,
out=page-locked buffer) per run, wall clock split into the plan build (host timers), the
device assembly, the band patch and the rest.

    python tools/e2e_probe.py [--config 5] [--runs 8]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_09204_b200 import screenbem as S  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--runs", type=int, default=8)
    ap.add_argument("--bench-like", action="store_true")
    args = ap.parse_args()
    ctx = S.Context(0)
    ctx.timers(True)
    pair = S.make_config(args.config)
    im = S.inflate(S.SurfaceMesh(pair.fine.vertices, pair.fine.facets), validate=False)
    buf = S.pinned_empty((im.n, im.n))
    keep = []
    if "--bench-like" in sys.argv:  # what else bench.py holds while it times the e2e runs
        fine = S.inflate(pair.fine, validate=False)
        coarse = S.inflate(pair.coarse)
        Wm = S.AssemblyPlan(fine, ctx=ctx).run()
        keep = [Wm, S.build_preconditioner(Wm, S.partition_dofs(pair, fine), S.build_prolongation(pair, coarse, fine))]
        Wh = S.assemble_W(im, ctx=ctx).download()  # the pageable-destination record run
        del Wh
    keys = ("plan_total", "plan_curl_wait", "plan_singular_wait", "plan_sync", "assemble_W", "near", "far_tiles",
            "near_leaves", "band_patch")
    for r in range(args.runs):
        ctx.reset_timers()
        t0 = time.perf_counter()
        W = S.assemble_W(im, ctx=ctx, out=buf)
        t1 = time.perf_counter()
        tm = {k: round(ctx.timer(k)[0], 2) for k in keys}
        print(f"run {r}: wall {1e3 * (t1 - t0):8.2f} ms  " + " ".join(f"{k}={v}" for k, v in tm.items()), flush=True)
        del W


if __name__ == "__main__":
    main()
