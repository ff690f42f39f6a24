"""Wall-clock time to solution through S.solve (host mesh pair in, host x out) — the bench's
tts_e2e, repeated (development aid).  python tools/tts_probe.py [config] [runs]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_09204_b200 import screenbem as S  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
runs = int(sys.argv[2]) if len(sys.argv) > 2 else 4
ctx = S.Context(0)
pair = S.make_config(cfg)
g = S.config_g(cfg)
for r in range(runs):
    t0 = time.perf_counter()
    res = S.solve(pair, g, ctx=ctx)
    x = res.report.solution
    t1 = time.perf_counter()
    print(f"run {r}: {1e3 * (t1 - t0):.1f} ms, {res.report.iterations} iterations", flush=True)
    del res
