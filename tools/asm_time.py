"""Device time of the assembly phases for one config (development aid for A/B builds:
SBG_LIB_PATH=scratch/<variant>.so python tools/asm_time.py 5).  Median of 5 runs after one
warm-up; the timers are the library's CUDA-event phase timers."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_09204_b200 import screenbem as S  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
ctx = S.Context(0)
ctx.timers(True)
fine = S.inflate(S.make_config(cfg).fine, validate=False)
plan = S.AssemblyPlan(fine, ctx=ctx)
W = plan.run()
names = ("assemble_W", "far_tiles", "near_leaves", "sauter", "near_classify")
rows = {k: [] for k in names}
for _ in range(5):
    ctx.reset_timers()
    W = plan.run(W)
    ctx.synchronize()
    for k in names:
        rows[k].append(ctx.timer(k)[0])
tag = os.path.basename(os.environ.get("SBG_LIB_PATH", "in-tree"))
print(f"cfg {cfg} [{tag}] " + " ".join(f"{k} {statistics.median(v):.2f}" for k, v in rows.items()))
