"""Config 5 subdomain sweep (BASELINE.json configs[4]): 160x160 flat screen, H/h in
{8, 16, 20, 40}: PCG iterations, PCG iterations/s, preconditioner applies/s, matvec
GB/s, preconditioner build time and the spectral condition numbers (device Lanczos,
condition_number(W, prec) and condition_number(W)).  One JSON line per ratio, and a
markdown table with --md PATH.

    python tools/sweep_cfg5.py [--ratios 8,16,20,40] [--md profiles/r01_cfg5_sweep.md]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C  # noqa: E402

import numpy as np  # noqa: E402

from paper_2310_09204_b200 import screenbem as S  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ratios", default="8,16,20,40")
    ap.add_argument("--md", default=None)
    ap.add_argument("--no-kappa", action="store_true")
    args = ap.parse_args()
    ratios = [int(r) for r in args.ratios.split(",")]
    ctx = S.Context(0)
    ctx.timers(True)
    rows = []
    W = raw = None
    for ratio in ratios:
        pair = S.make_config(5, ratio)
        fine, coarse = S.inflate(pair.fine, validate=False), S.inflate(pair.coarse)
        part, P = S.partition_dofs(pair, fine), S.build_prolongation(pair, coarse, fine)
        if W is None:  # the fine mesh (and W) is the same for every ratio
            ctx.reset_timers()
            W = S.assemble_W(fine, ctx=ctx)
            asm_ms = ctx.timer("assemble_W")[0]
            L = S.assemble_rhs(fine, S.config_g(5), ctx=ctx)
            if not args.no_kappa:
                t0 = time.perf_counter()
                raw = S.condition_number(W)
                raw_s = time.perf_counter() - t0
        S.build_preconditioner(W, part, P)  # warm (first-touch pool growth)
        ctx.reset_timers()
        prec = S.build_preconditioner(W, part, P)
        build_ms = ctx.timer("build_preconditioner")[0]
        S.pcg(W, prec, L, 1e-8)  # warm
        ctx.reset_timers()
        rep = S.pcg(W, prec, L, 1e-8)
        pcg_ms = ctx.timer("pcg")[0]
        # matvec / apply per launch with the L2 flushed (as bench.py)
        n = fine.n
        ldp = (n + 31) // 32 * 32
        dx, dy = C.c_void_p(), C.c_void_p()
        S._check(S.lib().sbg_device_alloc(ctx.h, 8 * ldp, C.byref(dx)))
        S._check(S.lib().sbg_device_alloc(ctx.h, 8 * ldp, C.byref(dy)))
        xh = np.random.default_rng(0).standard_normal(n)
        S._check(S.lib().sbg_memcpy_h2d(ctx.h, dx, xh.ctypes.data_as(C.c_void_p), 8 * n))
        ctx.reset_timers()
        for _ in range(10):
            ctx.l2_flush()
            S._check(S.lib().sbg_matvec_device(ctx.h, W.h, dx, dy, 1))
            # the 5 GB matvec leaves only clean lines of W in L2 (an explicit flush right
            # before the apply would leave 256 MB of dirty lines to write back during it)
            S._check(S.lib().sbg_apply_preconditioner_device(ctx.h, prec.h, dx, dy, 1))
        gm, gc = ctx.timer("gemv_f64")
        am, ac = ctx.timer("precond_apply")
        S.lib().sbg_device_free(dx)
        S.lib().sbg_device_free(dy)
        row = {"H/h": ratio, "dofs": n, "faces": len(part.face_ids), "wirebasket": len(part.wirebasket),
               "coarse": P.cols, "iterations": rep.iterations, "converged": rep.converged,
               "pcg_ms": pcg_ms, "pcg_iters_per_s": rep.iterations / (pcg_ms * 1e-3),
               "matvec_us": 1e3 * gm / gc, "matvec_gbs": (8.0 * n * n + 16.0 * n) / (gm / gc * 1e-3) / 1e9,
               "apply_us": 1e3 * am / ac, "applies_per_s": 1e3 / (am / ac),
               "apply_factor_gbs": prec.factor_bytes() / (am / ac * 1e-3) / 1e9, "factor_mb": prec.factor_bytes() / 1e6,
               "build_preconditioner_ms": build_ms, "assemble_W_ms": asm_ms,
               "kappa_lanczos_pcg": rep.kappa_estimate}
        if not args.no_kappa:
            t0 = time.perf_counter()
            sp = S.condition_number(W, prec)
            row.update({"kappa_prec": sp.kappa, "lambda_min": sp.lambda_min, "lambda_max": sp.lambda_max,
                        "lanczos_steps": sp.iterations, "kappa_s": time.perf_counter() - t0,
                        "kappa_unprec": raw.kappa, "kappa_unprec_steps": raw.iterations,
                        "kappa_unprec_s": raw_s})
        rows.append(row)
        print(json.dumps(row), flush=True)
        del prec
    if args.md:
        with open(args.md, "w") as f:
            f.write("# Config 5 subdomain sweep (160x160 flat screen, 51 200 triangles, 25 281 DOFs), 1 B200\n\n")
            f.write("Produced by `python tools/sweep_cfg5.py --md ...` on the GPU box; device times from CUDA events;\n"
                    "matvec timed per launch with the L2 flushed before it, the apply right after it; build\n"
                    "time is the second build (the first grows the device memory pool).\n"
                    "kappa_prec / kappa_unprec: `condition_number` (device Lanczos, W inner product, full\n"
                    "reorthogonalisation, extreme Ritz residuals <= 1e-10 |theta|; reference schwarz.hpp:150-190).\n\n")
            f.write("| H/h | faces x size | WB | coarse | PCG it | PCG it/s | matvec GB/s | apply us | build ms "
                    "| apply GB/s | kappa_prec | kappa_unprec |\n|---:|---|---:|---:|---:|---:|---:|---:|---:|---:|---:|---:|\n")
            for r in rows:
                fs = f"{r['faces']} x {(r['dofs'] - r['wirebasket']) // max(r['faces'], 1)}"
                f.write(f"| {r['H/h']} | {fs} | {r['wirebasket']} | {r['coarse']} | {r['iterations']} | "
                        f"{r['pcg_iters_per_s']:.0f} | {r['matvec_gbs']:.0f} | {r['apply_us']:.1f} | "
                        f"{r['build_preconditioner_ms']:.1f} | {r['apply_factor_gbs']:.0f} | "
                        f"{r.get('kappa_prec', float('nan')):.3f} | "
                        f"{r.get('kappa_unprec', float('nan')):.1f} |\n")
            f.write("\nRaw rows:\n\n```\n" + "\n".join(json.dumps(r) for r in rows) + "\n```\n")


if __name__ == "__main__":
    main()
