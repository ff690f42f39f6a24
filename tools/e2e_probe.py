"""Where the e2e time of bench.py goes (development aid): S.assemble_W(host InflatedMesh)
+ W.download(), split into plan build (host), assembly kernels and the download, wall
clock and device timers, best of several runs.

    python tools/e2e_probe.py [--config 2] [--runs 6]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_09204_b200 import screenbem as S  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--runs", type=int, default=6)
    args = ap.parse_args()
    ctx = S.Context(0)
    ctx.timers(True)
    pair = S.make_config(args.config, 8 if args.config == 5 else 0)
    im = S.inflate(S.SurfaceMesh(pair.fine.vertices, pair.fine.facets), validate=False)
    rows = []
    for r in range(args.runs):
        ctx.reset_timers()
        t0 = time.perf_counter()
        plan = S.AssemblyPlan(im, ctx=ctx)
        t1 = time.perf_counter()
        W = plan.run()
        ctx.synchronize()
        t2 = time.perf_counter()
        Wh = W.download()
        t3 = time.perf_counter()
        ctx.reset_timers()
        t4 = time.perf_counter()
        W2 = S.assemble_W(im, ctx=ctx)
        Wh2 = W2.download()
        t5 = time.perf_counter()
        tm = {k: ctx.timer(k)[0] for k in ("plan_total", "plan_morton", "plan_curl_wait", "plan_upload_curls", "plan_blocks", "plan_curls", "plan_tiles", "plan_singular", "plan_singular_wait", "plan_sync", "assemble_W")}
        rows.append((t1 - t0, t2 - t1, t3 - t2, t5 - t4, tm))
        del W, Wh, W2, Wh2, plan
    for p, a, d, e, tm in rows:
        print(f"plan {1e3 * p:7.2f} ms  run {1e3 * a:7.2f} ms  download {1e3 * d:7.2f} ms  | one-call e2e "
              f"{1e3 * e:7.2f} ms  timers " + " ".join(f"{k}={v:.2f}" for k, v in tm.items()), flush=True)


if __name__ == "__main__":
    main()
