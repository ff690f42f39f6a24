"""Host plan-build timers of the one-shot assemble_W at config 5 (development aid; the scopes nest:
plan_total > plan_curls > plan_tiles > plan_singular)."""
import os, sys, time
sys.path.insert(0, '/root/repo')
from paper_2310_09204_b200 import screenbem as S
ctx = S.Context(0); ctx.timers(True)
pair = S.make_config(5)
im = S.inflate(S.SurfaceMesh(pair.fine.vertices, pair.fine.facets), validate=False)
buf = S.pinned_empty((im.n, im.n))
keys = ["plan_total","plan_curls","plan_morton","plan_tiles","plan_singular","plan_singular_wait","plan_sync","plan_upload_curls","plan_blocks","plan_curl_wait"]
for r in range(4):
    ctx.reset_timers()
    t0 = time.perf_counter()
    W = S.assemble_W(im, ctx=ctx, out=buf)
    t1 = time.perf_counter()
    print(f"run {r}: wall {1e3*(t1-t0):.1f}", {k: round(ctx.timer(k)[0], 2) for k in keys})
    del W
