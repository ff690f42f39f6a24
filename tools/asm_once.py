"""Assemble one config twice (warm-up + measured) — small command for ncu launch lists."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_09204_b200 import screenbem as S
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
ctx = S.Context(0)
pair = S.make_config(cfg)
fine = S.inflate(pair.fine, validate=False)
plan = S.AssemblyPlan(fine, ctx=ctx)
W = plan.run()
W = plan.run(W)
ctx.synchronize()
print("ok", W.stats)
