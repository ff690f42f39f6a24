"""Matvec per-launch time with the L2 flushed before each launch (as bench.py measures it)
for configs 1-3 (development aid; W symmetric random).

    python tools/matvec_probe.py [--configs 1,2,3] [--reps 30]
"""
import argparse
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2310_09204_b200 import screenbem as S  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3")
    ap.add_argument("--reps", type=int, default=30)
    args = ap.parse_args()
    ctx = S.Context(0)
    ctx.timers(True)
    for cfg in [int(c) for c in args.configs.split(",")]:
        n = S.inflate(S.make_config(cfg).fine, validate=False).n
        A = np.random.default_rng(cfg).standard_normal((n, n))
        W = S.GalerkinMatrix.from_host(A + A.T, ctx)  # symmetric, as W (the column-sum form relies on it)
        del A
        ldp = (n + 31) // 32 * 32
        dx, dy = C.c_void_p(), C.c_void_p()
        S._check(S.lib().sbg_device_alloc(ctx.h, 8 * ldp, C.byref(dx)))
        S._check(S.lib().sbg_device_alloc(ctx.h, 8 * ldp, C.byref(dy)))
        xh = np.zeros(ldp)
        xh[:n] = np.random.default_rng(7).standard_normal(n)
        S._check(S.lib().sbg_memcpy_h2d(ctx.h, dx, xh.ctypes.data_as(C.c_void_p), 8 * ldp))
        for _ in range(3):
            S._check(S.lib().sbg_matvec_device(ctx.h, W.h, dx, dy, 1))
        if n <= 13000:
            yh = np.zeros(n)
            S._check(S.lib().sbg_memcpy_d2h(ctx.h, yh.ctypes.data_as(C.c_void_p), dy, 8 * n))
            ref = W.download() @ xh[:n]
            err = np.abs(yh - ref).max() / np.abs(ref).max()
            assert err < 1e-13, (cfg, err)
        ctx.reset_timers()
        for _ in range(args.reps):
            ctx.l2_flush()
            S._check(S.lib().sbg_matvec_device(ctx.h, W.h, dx, dy, 1))
        ms, cnt = ctx.timer("gemv_f64")
        us = 1e3 * ms / cnt
        print(f"config {cfg} n {n} tma {os.environ.get('SBG_GEMV_TMA', '0')}: {us:.2f} us, "
              f"{(8.0 * n * n + 16.0 * n) / (us * 1e-6) / 1e9:.0f} GB/s", flush=True)
        S.lib().sbg_device_free(dx)
        S.lib().sbg_device_free(dy)


if __name__ == "__main__":
    main()
