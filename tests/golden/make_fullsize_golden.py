"""Generates the full-size pipeline fixtures tests/golden/full_cfg{3,4,5}.npz from the CPU
restatement (oracle/, pinned by tests/test_oracle_pins.py).  The oracle's whole pipeline
runs here, on the oracle-assembled W, exactly as the reference's cmd_solve does
(inc/experiments.hpp:130-145): assemble_W -> assemble_rhs -> partition_dofs /
build_prolongation -> build_preconditioner -> pcg to 1e-8 from x0 = 0.  Meshes come from the
oracle's own Appendix-A generator (oracle.make_config), never from the product library.

    python tests/golden/make_fullsize_golden.py [cfg ...]      # default: 3 4 5

Config 5 assembles a 5.1 GB W on the host (per-worker dense partials, run_partitioned
semantics: workers are capped by RAM) and factors an 8481-DOF wire-basket block on one
thread: about 40 minutes on 8 cores.  Each fixture holds, per config:
  n, max_abs_W, diag (W_ii), probe (seeded v, normal_draws(23, n)), Wv = W v, absWv = |W| |v|
  (a checksum of the whole matrix: every entry enters; the second vector scales the test
  tolerance per row), and per H/h ratio r in the config's list:
  rhs_r, x_r (PCG solution), iters_r, hist_r (residual history), kappa_r (Lanczos estimate).
"""
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from oracle import oracle as O  # noqa: E402

RATIOS = {3: [12], 4: [8], 5: [8, 16, 20, 40]}
PROBE_SEED = 23


def workers_for(n: int) -> int:
    cores = os.cpu_count() or 1
    ram = os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES")
    # per-worker partials (inc/assemble.hpp:92-96) + the result, within ~60% of RAM
    return max(1, min(cores, int(0.6 * ram // (8 * n * n)) - 1))


def run(cfg: int):
    t0 = time.time()
    base = O.make_config(cfg, RATIOS[cfg][0])
    fine = O.inflate(base.fine, validate=False)
    n = fine.n
    w = workers_for(n)
    print(f"cfg {cfg}: n = {n}, assembling with {w} workers", flush=True)
    W = O.assemble_W(fine, workers=w)
    print(f"  assemble_W {time.time() - t0:.0f} s", flush=True)
    v = O.normal_draws(PROBE_SEED, n)
    out = {"n": n, "max_abs_W": np.abs(W).max(), "diag": np.ascontiguousarray(np.diag(W)), "probe": v,
           "Wv": W @ v, "absWv": np.abs(W) @ np.abs(v), "ratios": np.array(RATIOS[cfg], dtype=np.int32)}
    g = O.config_g(cfg)
    L = O.assemble_rhs(fine, g)
    for r in RATIOS[cfg]:
        t1 = time.time()
        pair = O.make_config(cfg, r)
        coarse = O.inflate(pair.coarse)
        prec = O.build_preconditioner(W, O.partition_dofs(pair, fine), O.build_prolongation(pair, coarse, fine))
        t2 = time.time()
        rep = O.pcg(W, prec, L, 1e-8)
        assert rep.converged
        print(f"  H/h {r}: build_preconditioner {t2 - t1:.0f} s, pcg {rep.iterations} it {time.time() - t2:.0f} s, "
              f"kappa {rep.kappa_estimate:.3f}", flush=True)
        out.update({f"rhs_{r}": L, f"x_{r}": rep.solution, f"iters_{r}": rep.iterations,
                    f"hist_{r}": rep.residual_history, f"kappa_{r}": rep.kappa_estimate})
        del prec
    del W
    np.savez_compressed(os.path.join(HERE, f"full_cfg{cfg}.npz"), **out)
    print(f"cfg {cfg} done in {time.time() - t0:.0f} s", flush=True)


if __name__ == "__main__":
    for c in [int(a) for a in sys.argv[1:]] or [3, 4, 5]:
        run(c)
