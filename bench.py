"""Benchmark of the B200 screenbem hot path (driver contract).

A step is one pass of the hot path over the config's synthetic mesh: assemble_W,
assemble_rhs, build_preconditioner and PCG to 1e-8 (inc/experiments.hpp:130-145).
Default workload: config 5 (flat 160x160, 25 281 DOFs, 5.1 GB W) at H/h 8 — the largest
BASELINE config, which fits one B200.
  value : assembly triangle-pairs/s (nf(nf+1)/2 per assembly) with the mesh-derived
          data resident in HBM (AssemblyPlan built before the timed region),
          device time from CUDA events, max over ranks;
  e2e   : the same metric through the public assemble_W call (host mesh in, host W
          out: plan build + H2D + kernels + D2H of the n x n matrix), the drop-in for
          the reference's assemble_W (inc/assemble.hpp:72-139); median over runs;
  tts_e2e_ms: time to solution through the public API, host mesh pair -> host x
          (inflate, partition, prolongation, plan, assembly, RHS, preconditioner, PCG);
  extras: PCG iterations/s, matvec GB/s (HBM roofline), preconditioner applies/s,
          per-phase device times.
--gpus N without a launcher re-executes itself under torch.distributed.run with N ranks
(one GPU each).  N > 1 assembles ONE W across the ranks (strong scaling) unless
--replicas.  --impl reference times the CPU restatement of the reference's assemble_W
(oracle/, all host threads, run_partitioned semantics) on an unbiased sample of the pair
space; it never loads the product library.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "assembly tri-pairs/s; PCG iters/s & matvec GB/s vs HBM peak (fp64, 1 B200)"
UNIT = "tri-pairs/s"
CFG_NAMES = {1: "flat 16x16 (512 tri)", 2: "flat 64x64 (8192 tri)", 3: "T-junction 3x48x48 (13824 tri)",
             4: "triple cross 3x64x64 (24576 tri)", 5: "flat 160x160 (51200 tri)"}
DEFAULT_RATIO = {1: 8, 2: 16, 3: 12, 4: 8, 5: 8}   # BASELINE.json configs (H/h)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--exact-far", action="store_true",
                    help="far pairs bitwise like the CPU restatement (SURVEY Appendix B parity-gate path)")
    ap.add_argument("--clocks", default="nvml", choices=["nvml", "smi", "off"],
                    help="clock/throttle sampler during the timed region (nvml: in-process NVML queries)")
    ap.add_argument("--no-cpu-phases", action="store_true",
                    help="skip the CPU restatement's setup/preconditioner/PCG timings")
    ap.add_argument("--cpu-phases-max-n", type=int, default=8000)
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--ratio", type=int, default=0, help="H/h (default: the config's, 8 for config 5)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="target CPU sample length")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: functional check of the N>1 paths (ranks may share one GPU; not a timing)")
    ap.add_argument("--replicas", action="store_true",
                    help="N>1: N independent replicas of the whole step (weak scaling) instead of one W "
                         "assembled across the ranks")
    ap.add_argument("--shard", action="store_true", help="(default for N>1) one W across the ranks")
    ap.add_argument("--tts-runs", type=int, default=3, help="time-to-solution runs (median reported)")
    ap.add_argument("--dl-grid", type=int, default=64,
                    help="eval_DL of the solution on an n x n grid of [-2,2]^2 (z = 0 and z = 0.05); 0: skip")
    return ap.parse_args()


def dist_env():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(
        os.environ.get("LOCAL_RANK", "0"))


def reduce_max(values, dist=None, device="cpu"):
    """Element-wise max over ranks (the timing contract: max over ranks of device times).
    NCCL on the GPU box (device cuda:LOCAL_RANK), gloo on CPU (tests/test_distributed.py)."""
    if dist is None:
        return list(values)
    import torch
    t = torch.tensor(list(values), dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(v) for v in t]


def allreduce_sum_(t, dist, rdev: str):
    """In-place sum over ranks of a partial W (the --shard reduction): NCCL on the device
    tensor, or through host memory for gloo (tests/test_distributed.py, functional runs)."""
    if rdev == "cpu" and t.device.type != "cpu":
        h = t.cpu()
        dist.all_reduce(h)
        t.copy_(h)
    else:
        dist.all_reduce(t)


# --------------------------------------------------------------------------- clocks
class NvmlSampler:
    """SM clock + throttle reasons sampled every 20 ms during the timed region through
    in-process NVML (the nvidia-smi loop contends for the driver with the timed step)."""
    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20, "sw_power_cap": 0x4}

    def __init__(self, device: int):
        self.device, self.rows, self.stop, self.t = device, [], threading.Event(), None

    def __enter__(self):
        try:
            import pynvml as N
            N.nvmlInit()
            h = N.nvmlDeviceGetHandleByIndex(self.device)
            self.mx = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)
            reasons_fn = getattr(N, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                N.nvmlDeviceGetCurrentClocksThrottleReasons

            def run():
                while True:
                    try:
                        sm = N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)
                        r = reasons_fn(h)
                        self.rows.append((sm, r))
                    except Exception:
                        pass
                    if self.stop.wait(0.02):
                        break
            self.t = threading.Thread(target=run, daemon=True)
            self.t.start()
        except Exception:
            self.t = None
        return self

    def __exit__(self, *a):
        self.stop.set()
        if self.t:
            self.t.join(timeout=2)
            try:
                import pynvml as N
                N.nvmlShutdown()
            except Exception:
                pass

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = sorted(r[0] for r in self.rows)
        reasons = sorted({k for _, bits in self.rows for k, m in self.REASONS.items() if bits & m})
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": self.mx, "reasons": reasons, "samples": len(self.rows),
                "source": "NVML"}


class NullSampler:
    def __init__(self, device: int):
        pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        pass

    def summary(self):
        return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled (--clocks off)"]}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device, self.rows, self.proc = device, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = sorted(float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit())
        mx = max((float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()), default=None)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(self.rows)}


# --------------------------------------------------------------------------- CPU restatement (oracle)
def host_ram_bytes() -> int:
    try:
        with open("/proc/meminfo") as f:
            for line in f:
                if line.startswith("MemAvailable:"):
                    return int(line.split()[1]) * 1024
    except Exception:
        pass
    return os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES")


def config_dict(cfg: int, ratio: int, nf: int, n: int) -> dict:
    """The workload, identical in both arms (the driver compares them)."""
    return {"workload": f"config {cfg}: {CFG_NAMES[cfg]}, H/h {ratio}", "triangles": nf, "dofs": n,
            "tri_pairs": nf * (nf + 1) // 2, "h_ratio": ratio, "pcg_tol": 1e-8}


class CpuAssembly:
    """The reference's assemble_W restated in oracle/ on the host cores (all threads, RAM
    permitting: each worker holds a dense n x n partial, inc/assemble.hpp:92-96), timed
    on an unbiased bounded sample of the pair space (oracle.AssemblySampler):
      t_full = t_call + (npairs / k) * t_loop(k systematically sampled pairs)
    t_call = the per-call work with no pairs (partials allocated and zeroed in their
    threads, worker-ordered sum, mirror), measured once; t_loop = the pair loop over the
    sample split into contiguous per-worker chunks as run_partitioned splits the full
    range (common.hpp:31-59).  value = npairs / t_full.  Meshes come from the oracle's
    own config generator: the product library is never loaded."""

    def __init__(self, cfg: int, ratio: int, target_s: float):
        from oracle import oracle as O
        pair = O.make_config(cfg, ratio)
        self.im = O.inflate(pair.fine, validate=False)
        self.nf, self.n = pair.fine.nf, self.im.n
        self.npairs = self.nf * (self.nf + 1) // 2
        cores = os.cpu_count() or 1
        cap = max(1, int(0.8 * host_ram_bytes() // max(8 * self.n * self.n, 1)))
        self.workers = max(1, min(cores, cap))
        self.sampler = O.AssemblySampler(self.im, self.workers)
        self.t_call = self.sampler.fixed()
        # calibrate the per-pair cost on a small sample, then size the timed sample
        k0 = min(self.npairs, max(2000 * self.workers, 20000))
        t0 = self.sampler.run(O.systematic_pair_sample(self.nf, k0, seed=1))
        self.k = int(min(self.npairs, max(k0, target_s * k0 / max(t0, 1e-9))))
        self.idx = O.systematic_pair_sample(self.nf, self.k, seed=0)
        self.loops = []

    def step(self, timed: bool = True, short: bool = False) -> float:
        if short:  # untimed warm-up on a small sample
            from oracle import oracle as O
            return self.sampler.run(O.systematic_pair_sample(self.nf, min(self.k, 20000), seed=2))
        t = self.sampler.run(self.idx)
        if timed:
            self.loops.append(t)
        return t

    def summary(self) -> dict:
        loop = sum(self.loops) / len(self.loops)
        t_full = self.t_call + self.npairs / self.k * loop
        return {"value": self.npairs / t_full, "unit": UNIT, "cores": self.workers, "kind": "port",
                "sample": (f"oracle assemble_W pair loop on {self.k} of {self.npairs} pairs (systematic sample of the "
                           f"reference pair order, seeded offset) {loop:.1f} s/step on {self.workers} threads, plus the "
                           f"per-call work (partials, ordered sum, mirror) {self.t_call:.2f} s, measured once; "
                           f"value = npairs / (t_call + npairs/k * t_loop) = full assemble_W {t_full:.1f} s"),
                "seconds_full_estimate": t_full, "seconds_loop": loop, "seconds_call": self.t_call,
                "pairs_sampled": self.k, "workers_ram_cap": self.workers < (os.cpu_count() or 1)}


def cpu_assembly_sample(cfg: int, ratio: int, target_s: float):
    """one timed sample (our arm's cpu_baseline leg)"""
    ca = CpuAssembly(cfg, ratio, target_s)
    ca.step()
    return ca.summary()


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip() + f" ({os.cpu_count()} logical CPUs)"
    except Exception:
        pass
    return f"unknown ({os.cpu_count()} logical CPUs)"


def cpu_phases(cfg: int, ratio: int, W_host=None, max_n: int = 8000):
    """The reference's other phases on the CPU restatement, single-threaded as in the
    reference (Eigen without OpenMP): setup (inflate both levels, partition_dofs,
    build_prolongation), build_preconditioner, one preconditioner apply, and PCG to
    1e-8 on W_host (the GPU-assembled matrix when given, else the oracle's own full
    assembly on all host threads, timed as assembly_s).  Skipped above max_n DOFs
    (the WB Cholesky and dense coarse product take minutes at config 5)."""
    import numpy as np

    from oracle import oracle as O
    t0 = time.perf_counter()
    opair = O.make_config(cfg, ratio)
    fine, coarse = O.inflate(opair.fine, validate=False), O.inflate(opair.coarse)
    part, R = O.partition_dofs(opair, fine), O.build_prolongation(opair, coarse, fine)
    out = {"setup_s": time.perf_counter() - t0, "dofs": fine.n}
    if fine.n > max_n:
        out["skipped"] = f"n = {fine.n} > {max_n}: single-threaded WB Cholesky and dense coarse product take minutes"
        return out
    if W_host is None:
        t0 = time.perf_counter()
        W_host = O.assemble_W(fine, workers=os.cpu_count() or 1)
        out["assembly_s"] = time.perf_counter() - t0
        out["assembly_workers"] = os.cpu_count() or 1
    t0 = time.perf_counter()
    prec = O.build_preconditioner(W_host, part, R)
    out["build_preconditioner_s"] = time.perf_counter() - t0
    xv = O.normal_draws(5, fine.n)
    t0 = time.perf_counter()
    O.matvec(W_host, xv, reps=3)
    mv = (time.perf_counter() - t0) / 3
    out["matvec_s"] = mv
    out["matvec_gbs"] = 8.0 * fine.n * fine.n / mv / 1e9
    r = O.normal_draws(17, fine.n)
    t0 = time.perf_counter()
    for _ in range(3):
        prec.apply(r)
    out["precond_apply_s"] = (time.perf_counter() - t0) / 3
    L = O.assemble_rhs(fine, O.config_g(cfg))
    t0 = time.perf_counter()
    rep = O.pcg(W_host, prec, L, 1e-8)
    dt = time.perf_counter() - t0
    out["cpu_model"] = cpu_model()
    out.update({"pcg_s": dt, "pcg_iterations": rep.iterations,
                "pcg_iters_per_s": rep.iterations / dt if dt > 0 else None, "threads": 1,
                "matrix": "GPU-assembled W (downloaded)" if "assembly_s" not in out else "oracle assemble_W"})
    del np
    return out


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:  # the reference is the CPU path: rank 0 alone runs and prints it
        return
    cfg = args.config
    ratio = args.ratio or DEFAULT_RATIO[cfg]
    # each timed step: the pair loop over the same unbiased sample, sized so the whole run
    # stays within a few minutes
    per_step = max(3.0, min(args.cpu_seconds, 150.0 / max(args.steps, 1)))
    ca = CpuAssembly(cfg, ratio, per_step)
    for _ in range(args.warmup):
        ca.step(timed=False, short=True)
    for _ in range(args.steps):
        ca.step()
    cb = ca.summary()
    v = cb["value"]
    phases = None
    if not args.no_cpu_phases:
        try:
            phases = cpu_phases(cfg, ratio, None, max_n=args.cpu_phases_max_n)
        except Exception as e:  # pragma: no cover
            phases = {"failed": str(e)}
    cb["phases"] = phases
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(ca.loops) / len(ca.loops),
            "higher_is_better": True, "scaling": "strong" if args.gpus > 1 and not args.replicas else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_dict(cfg, ratio, ca.nf, ca.n),
            "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample", "phases")},
            "cpu_model": cpu_model(),
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- ours
def matvec_traffic(cfg: int):
    """DRAM bytes per matvec launch from the committed ncu capture for this config (or None)."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02_traffic.json")) as f:
            e = json.load(f)["gemv_f64"].get(str(cfg))
        return None if e is None else e["dram_read"] + e["dram_write"]
    except Exception:
        return None


def kernel_traffic(kernel: str, cfg: int):
    """DRAM bytes per step of an assembly kernel (summed over its launches in one step) from
    the committed ncu --set full capture for this config (or None)."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02_traffic.json")) as f:
            e = json.load(f)[kernel].get(str(cfg))
        return None if e is None else int(sum(e["dram_bytes_per_step"]))
    except Exception:
        return None


def kernel_pipe(kernel: str, cfg: int):
    """ncu's FP64-pipe activity of an assembly kernel (fraction of active cycles) and its FP64
    instructions per evaluation, from the committed capture for this config (or None)."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02_traffic.json")) as f:
            e = json.load(f)[kernel].get(str(cfg))
        return None if e is None or "fp64_pipe_active" not in e else {
            "fp64_pipe_active_ncu": e["fp64_pipe_active"], "fp64_instr_per_eval": e.get("fp64_instr_per_eval"),
            "source": e.get("source")}
    except Exception:
        return None


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


def run_ours(args):
    import numpy as np

    from paper_2310_09204_b200 import screenbem as S
    rank, world, local = dist_env()
    dist = None
    if world > 1:
        import torch
        import torch.distributed as dist
        if args.dist_backend == "gloo":  # functional check of the N>1 paths; ranks may share a GPU
            local = local % torch.cuda.device_count()
        torch.cuda.set_device(local)
        dist.init_process_group(args.dist_backend)
    ctx = S.Context(local)
    rdev = "cpu" if args.dist_backend == "gloo" else f"cuda:{local}"

    def allreduce_(t):
        allreduce_sum_(t, dist, rdev)
    ctx.timers(True)
    cfg = args.config
    ratio = args.ratio or DEFAULT_RATIO[cfg]
    pair = S.make_config(cfg, ratio)
    fine = S.inflate(pair.fine, validate=cfg <= 3)
    coarse = S.inflate(pair.coarse)
    part = S.partition_dofs(pair, fine)
    P = S.build_prolongation(pair, coarse, fine)
    g = S.config_g(cfg)
    nf, n = pair.fine.nf, fine.n
    npairs = nf * (nf + 1) // 2
    qcfg = S.QuadratureConfig(exact_far=args.exact_far)
    # the e2e runs' destination: a page-locked host buffer allocated once, up front (as the
    # inputs of a step come from pinned memory; the pageable-destination time is reported
    # beside it)
    try:
        Wbuf = S.pinned_empty((n, n))
        dest = "page-locked host buffer allocated once"
    except Exception:  # not enough page-lockable host memory: a pageable buffer, reused
        Wbuf = np.empty((n, n))
        Wbuf.fill(0.0)
        dest = "pageable host buffer allocated (and touched) once"
    plan = S.AssemblyPlan(fine, qcfg, ctx=ctx)
    plan_ms = {k: round(ctx.timer(k)[0], 3) for k in ("plan_total", "plan_curls", "plan_tiles", "plan_singular")}

    shard = world > 1 and not args.replicas

    def assemble(plan, W):
        """the timed assembly: the whole W, or this rank's shard + the all-reduce of the
        partial W over NCCL (in place on W's device storage, through __cuda_array_interface__)"""
        if not shard:
            return plan.run(W)
        import torch
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record()  # legacy stream; the context stream is a blocking stream
        W = plan.run(W, shard=(rank, world))
        # W is symmetric: only its upper triangle (n (n + 1) / 2 doubles, half of W) is summed
        if "packed" not in packed_buf:
            packed_buf["packed"] = torch.empty(n * (n + 1) // 2, dtype=torch.float64, device=f"cuda:{local}")
        packed = packed_buf["packed"]
        W.pack_upper(packed.data_ptr())
        allreduce_(packed)
        W.unpack_upper(packed.data_ptr())
        ev[1].record()
        ev[1].synchronize()
        shard_ms.append(ev[0].elapsed_time(ev[1]))
        return W

    shard_ms = []
    packed_buf = {}

    # --shard: the PCG runs by row panels — this rank's rows of each W p, then
    # one all-gather of W p per iteration over NCCL on the PCG stream
    rows = S.row_ranges(n, world)[rank] if shard else None
    exchange = (S.allgather_exchange(dist, rank, world, n, device=f"cuda:{local}", host_staging=(rdev == "cpu"))
                if shard else None)
    # the stop decision of the row-panel PCG is collective (every rank enqueues the same
    # all-gathers even if its state differs in the last bits)
    agree = S.allreduce_agree(dist, device=None if rdev == "cpu" else rdev) if shard else None

    def rhs():
        L = S.assemble_rhs(fine, g, ctx=ctx)
        if shard:  # the RHS is assembled with fp64 atomics: take rank 0's on every rank
            import torch
            t = torch.from_numpy(L)
            if rdev != "cpu":
                t = t.to(rdev)
            dist.broadcast(t, 0)
            L = t.cpu().numpy()
        return L

    def step(W):
        W = assemble(plan, W)
        L = rhs()
        prec = S.build_preconditioner(W, part, P)
        rep = S.pcg_rows(W, prec, L, rows, exchange, 1e-8, agree=agree) if shard else S.pcg(W, prec, L, 1e-8)
        return W, prec, rep

    W = None
    for _ in range(args.warmup):
        ctx.l2_flush()
        W, prec, rep = step(W)
    ctx.synchronize()
    ctx.reset_timers()
    launches0 = S.launch_count()
    iters = []
    if dist:
        dist.barrier()
    sampler = {"nvml": NvmlSampler, "smi": ClockSampler, "off": NullSampler}[args.clocks]
    with sampler(local) as clocks:
        for _ in range(args.steps):
            ctx.l2_flush()
            ctx.begin("step")
            W, prec, rep = step(W)
            ctx.end()
            iters.append(rep.iterations)
        ctx.synchronize()
    launches = S.launch_count() - launches0
    tm = {k: ctx.timer(k) for k in ("step", "assemble_W", "far_tiles", "near", "near_leaves", "sauter", "classify",
                                     "local_scatter", "mirror", "near_classify", "build_preconditioner", "cholesky",
                                     "block_inverse", "coarse_galerkin", "pcg", "gemv_f64", "precond_apply", "inv_alloc",
                                     "inv_lower", "inv_lauum")}
    # per-step totals (a phase may run several launches per step, e.g. one near level each)
    ms = {k: v[0] / args.steps for k, v in tm.items()}
    launches_per_step = {k: v[1] / args.steps for k, v in tm.items()}
    t_asm = ms["assemble_W"] * 1e-3
    if shard:  # shard compute + all-reduce, per step
        t_asm = sum(shard_ms[-args.steps:]) / args.steps * 1e-3
    step_ms = ms["step"]
    t_asm, step_ms = reduce_max([t_asm, step_ms], dist, rdev)
    value = (1 if shard else world) * npairs / t_asm
    stats = dict(W.stats)
    if shard:  # a shard does not separate its far count: total far pairs (exact) / world
        import torch
        loc = torch.tensor([sum(stats[k] for k in ("identical", "edge", "vertex", "near_pairs"))],
                           dtype=torch.float64, device=rdev)
        dist.all_reduce(loc)
        stats["far_pairs"] = int(round((npairs - float(loc[0])) / world))
        stats["far_pairs_estimated"] = True
    # ---- dominant-kernel roofline (FP64 pipe): SURVEY.md §8d 20 flop per tensor-rule evaluation
    fp64_peak = S.fp64_peak_tflops(ctx)
    far_ms, near_ms = ms["far_tiles"], ms["near_leaves"]
    far_flop = 20.0 * 256 * stats["far_pairs"]
    near_flop = 20.0 * 1296 * stats["near_leaves"]
    dom = ("far_tiles", far_flop, far_ms) if far_ms >= near_ms else ("near_leaves", near_flop, near_ms)
    achieved = dom[1] / (dom[2] * 1e-3) / 1e12 if dom[2] > 0 else 0.0
    pipe = kernel_pipe(dom[0], cfg)
    # ---- matvec (HBM) and preconditioner applies, L2 flushed between launches
    ctx.reset_timers()
    import ctypes as C
    dx = C.c_void_p()
    dy = C.c_void_p()
    ldp = (n + 31) // 32 * 32
    S._check(S.lib().sbg_device_alloc(ctx.h, 8 * ldp, C.byref(dx)))
    S._check(S.lib().sbg_device_alloc(ctx.h, 8 * ldp, C.byref(dy)))
    xh = np.random.default_rng(0).standard_normal(n)
    S._check(S.lib().sbg_memcpy_h2d(ctx.h, dx, xh.ctypes.data_as(C.c_void_p), 8 * n))
    for _ in range(3):
        S._check(S.lib().sbg_matvec_device(ctx.h, W.h, dx, dy, 1))
    ctx.reset_timers()
    reps = 20
    for _ in range(reps):
        ctx.l2_flush()
        S._check(S.lib().sbg_matvec_device(ctx.h, W.h, dx, dy, 1))
        S._check(S.lib().sbg_apply_preconditioner_device(ctx.h, prec.h, dx, dy, 1))
    gm, gc = ctx.timer("gemv_f64")
    am, ac = ctx.timer("precond_apply")
    matvec_s = gm / gc * 1e-3
    # algorithmic bytes of the context's matvec form (symmetric: the upper triangle, x, y and
    # the partial sums; linalg.cu gemv_bytes)
    mb = C.c_double()
    S._check(S.lib().sbg_matvec_bytes(ctx.h, W.h, C.byref(mb)))
    matvec_bytes = mb.value
    matvec_gbs = matvec_bytes / matvec_s / 1e9
    peaks = load_peaks()
    hbm_peak = peaks.get("hbm_gbs") or 6650.0
    # the full-matrix form beside it (every stored entry of the dense W read once,
    # 8 n^2 + 16 n bytes; the symmetric form above reads half of them and is reported separately)
    form0 = ctx.matvec_form
    full_s = full_bytes = None
    if form0 == "symmetric":
        ctx.matvec_form = "full"
        for _ in range(3):
            S._check(S.lib().sbg_matvec_device(ctx.h, W.h, dx, dy, 1))
        ctx.reset_timers()
        for _ in range(reps):
            ctx.l2_flush()
            S._check(S.lib().sbg_matvec_device(ctx.h, W.h, dx, dy, 1))
        fm, fc = ctx.timer("gemv_f64")
        full_s = fm / fc * 1e-3
        S._check(S.lib().sbg_matvec_bytes(ctx.h, W.h, C.byref(mb)))
        full_bytes = mb.value
        ctx.matvec_form = form0
    S.lib().sbg_device_free(dx)
    S.lib().sbg_device_free(dy)
    # ---- e2e: public assemble_W with host mesh in, host W out
    e2e_times, e2e_parts = [], []
    h2d = 0
    # the reference arm times assemble_W on an inflated mesh; so does this one: the host-side
    # InflatedMesh is the call's input, everything from there to the host copy of W is timed
    im2 = S.inflate(S.SurfaceMesh(pair.fine.vertices, pair.fine.facets), validate=False)
    pageable_ms = None
    import gc
    gc.collect()
    gc.disable()  # no cyclic-GC pauses inside the timed e2e / time-to-solution runs
    for it in range(1 + max(args.steps, 4)):  # first run warms the host paths; median over the rest
        ctx.reset_timers()
        t0 = time.perf_counter()
        ctx.begin("e2e")
        if shard:
            W2 = assemble(S.AssemblyPlan(im2, qcfg, ctx=ctx), None)
            W2.download(out=Wbuf)
        else:  # the host copy comes with the call (overlapped with the near field into pinned memory)
            W2 = S.assemble_W(im2, qcfg, ctx=ctx, out=Wbuf)
        h2d = int(W2.stats["h2d_bytes"])
        ctx.end()
        ctx.synchronize()
        e2e_times.append(ctx.timer("e2e")[0] * 1e-3)
        e2e_parts.append({k: round(ctx.timer(k)[0], 1) for k in ("assemble_W", "far_tiles", "near_leaves", "band_patch",
                                                                  "w_copy", "plan_total")})
        del W2
    del Wbuf
    runs = sorted(e2e_times[1:] if len(e2e_times) > 1 else e2e_times)
    e2e_t = runs[len(runs) // 2]
    e2e_min = runs[0]
    e2e_t, e2e_min = reduce_max([e2e_t, e2e_min], dist, rdev)
    # ---- time to solution through the public API: host MeshLevelPair -> host x
    # (inflate both levels, partition_dofs, build_prolongation, assemble_W with its plan,
    # assemble_rhs, build_preconditioner, pcg to 1e-8, the solution copied to the host)
    tts = []
    if not shard:
        hpair = S.MeshLevelPair(S.SurfaceMesh(pair.coarse.vertices, pair.coarse.facets),
                                S.SurfaceMesh(pair.fine.vertices, pair.fine.facets), pair.parent)
        for it in range(1 + max(args.tts_runs, 1)):
            ctx.synchronize()
            t0 = time.perf_counter()
            res = S.solve(hpair, g, 1e-8, qcfg, ctx=ctx)
            x = res.report.solution
            dt = time.perf_counter() - t0
            if it:  # the first run warms the host paths
                tts.append(dt * 1e3)
            tts_iters = res.report.iterations
            xsol = x
            del res, x
        tts_runs = [round(t, 2) for t in tts]
        tts.sort()
    # ---- the next adjacent compute: eval_DL (potential.hpp:104-138) of the
    # solution on the reference's evaluation grid, device-timed; the CPU restatement beside it on
    # a point sample (the cpu_baseline leg)
    dl = None
    if not shard and args.dl_grid > 0:
        fm = S.SurfaceMesh(pair.fine.vertices, pair.fine.facets)
        gpts = S.make_cartesian_grid(fm, -2.0, 2.0, args.dl_grid, args.dl_grid, 1e-3, ctx=ctx).points
        lift = gpts.copy()
        lift[:, 2] = 0.05
        dpts = np.concatenate([gpts, lift])
        S.eval_DL(xsol, im2, dpts[:128], qcfg, ctx=ctx)
        dl_ms = []
        for _ in range(3):
            ctx.reset_timers()
            S.eval_DL(xsol, im2, dpts, qcfg, ctx=ctx)
            dl_ms.append(ctx.timer("eval_dl")[0])
        dl_ms.sort()
        nfac = len(pair.fine.facets)
        nrule = (qcfg.far_order + 2) ** 2
        dpairs = len(dpts) * nfac
        dl = {"points": len(dpts), "facets": nfac, "ms": dl_ms[1], "ms_runs": [round(t, 3) for t in dl_ms],
              "point_facet_pairs_per_s": dpairs / (dl_ms[1] * 1e-3),
              "rule_evaluations_per_s": dpairs * nrule / (dl_ms[1] * 1e-3),
              "what": f"eval_DL of the PCG solution on the {args.dl_grid}x{args.dl_grid} grid of [-2,2]^2 in z = 0 "
                      "(points within 1e-3 of the screen masked) and the same points at z = 0.05; device time of "
                      "sbg_eval_dl (H2D of points and density, the on-screen check, the kernels, D2H), median of 3"}
        if rank == 0 and world == 1 and not args.no_cpu_baseline:
            try:
                from oracle import oracle as O
                oim = O.inflate(O.Mesh(pair.fine.vertices, pair.fine.facets), validate=False)
                sel = np.linspace(0, len(dpts) - 1, 64).astype(int)
                t0 = time.perf_counter()
                O.eval_DL(xsol, oim, dpts[sel], O.QuadratureConfig(far_order=qcfg.far_order))
                tc = time.perf_counter() - t0
                dl["cpu_baseline"] = {"point_facet_pairs_per_s": len(sel) * nfac / tc, "cores": os.cpu_count() or 1,
                                      "kind": "port", "sample": f"{len(sel)} of the points, oracle eval_DL"}
            except Exception as e:  # pragma: no cover - reported, not fatal
                dl["cpu_baseline"] = {"failed": str(e)}
    gc.enable()
    # one assembly into a fresh pageable numpy array, for the record (last: the 5 GB of fresh
    # pageable memory it faults in and frees does not run beside the timed e2e/tts runs)
    ctx.reset_timers()
    ctx.begin("e2e")
    W2 = S.assemble_W(im2, ctx=ctx) if not shard else assemble(S.AssemblyPlan(im2, qcfg, ctx=ctx), None)
    Wh = W2.download()
    ctx.end()
    ctx.synchronize()
    pageable_ms = ctx.timer("e2e")[0]
    del W2, Wh
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_assembly_sample(cfg, ratio, args.cpu_seconds)
            cpu = {k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample")}
            if not args.no_cpu_phases:
                ph = cpu_phases(cfg, ratio, W.download() if n <= args.cpu_phases_max_n else None,
                                max_n=args.cpu_phases_max_n)
                if "pcg_s" in ph and cpu.get("value"):
                    # setup + full assembly at the sampled rate + preconditioner + PCG
                    ph["time_to_solution_s_est"] = (ph["setup_s"] + npairs / cpu["value"] + ph["build_preconditioner_s"]
                                                    + ph["pcg_s"])
                cpu["phases"] = ph
        except Exception as e:  # pragma: no cover
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "port", "sample": f"failed: {e}"}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True, "scaling": "strong" if shard else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_dict(cfg, ratio, nf, n),
            "parallelism": (f"assembly sharded x{world} (NCCL all-reduce of W's packed upper triangle), preconditioner "
                            f"replicated, PCG by "
                            f"row panels (NCCL all-gather of W p per iteration)") if shard
            else (f"replicas x{world}" if world > 1 else "single GPU"),
            "l2": "flushed (256 MiB write + 256 MiB read: cold L2 with clean lines) before every timed step and "
                  "every matvec launch",
            "far_field": "exact (IEEE, oracle order)" if args.exact_far else "fast (distance expansion + refined rsqrt)",
            "roofline": {"bound": "fp64", "kernel": dom[0], "achieved": achieved, "peak": fp64_peak,
                         "unit": "TFLOP/s", "frac": achieved / fp64_peak if fp64_peak else None,
                         "traffic": kernel_traffic(dom[0], cfg),
                         "traffic_note": "DRAM bytes per step (all launches of the kernel in one step) from "
                                         "profiles/r02_traffic.json; the kernel is FP64-bound, so the bytes only "
                                         "show it re-reads nothing (leaf list, geometry and W updates)",
                         "peak_source": "DFMA loop measured by bench.py on this GPU (MEASURED_PEAKS.json has no fp64)",
                         "flop_convention": "20 flop per tensor-rule kernel evaluation (SURVEY.md §8d), fixed "
                                            "regardless of the implementation; an evaluation issues 7 FP64 "
                                            "instructions (14 flop) on flat panels, 8 otherwise, so frac exceeds the "
                                            "FP64-pipe activity and can exceed 1: frac_issued counts the issued "
                                            "instructions (2 flop each) against the same DFMA peak",
                         "pipe": pipe,
                         "achieved_issued": achieved * 2.0 * pipe["fp64_instr_per_eval"] / 20.0
                         if pipe and pipe.get("fp64_instr_per_eval") else None,
                         "frac_issued": achieved * 2.0 * pipe["fp64_instr_per_eval"] / 20.0 / fp64_peak
                         if pipe and pipe.get("fp64_instr_per_eval") and fp64_peak else None,
                         "ms_per_step": dom[2], "launches_per_step": launches_per_step[dom[0]],
                         "achieved_other": {"kernel": ("near_leaves" if dom[0] == "far_tiles" else "far_tiles"),
                                            "tflops": (near_flop / (near_ms * 1e-3) / 1e12 if dom[0] == "far_tiles"
                                                       else far_flop / (far_ms * 1e-3) / 1e12)
                                            if min(far_ms, near_ms) > 0 else None}},
            "roofline_matvec": {"bound": "hbm", "kernel": "gemv_f64", "achieved": matvec_gbs, "peak": hbm_peak,
                                "unit": "GB/s", "frac": matvec_gbs / hbm_peak, "traffic": matvec_traffic(cfg),
                                "form": ctx.matvec_form, "bytes_per_launch": matvec_bytes,
                                "bytes_full_matrix": 8.0 * n * n + 16.0 * n, "us_per_launch": matvec_s * 1e6,
                                "peak_source": ("of measured: MEASURED_PEAKS.json hbm_gbs (a copy; a read-only "
                                                "stream can exceed it)") if peaks.get("hbm_gbs") else "of fallback",
                                "peak_nominal": 7700.0, "frac_nominal": matvec_gbs / 7700.0,
                                "full_form": None if full_s is None else {
                                    "bytes_per_launch": full_bytes, "us_per_launch": full_s * 1e6,
                                    "achieved": full_bytes / full_s / 1e9, "unit": "GB/s",
                                    "frac": full_bytes / full_s / 1e9 / hbm_peak,
                                    "frac_nominal": full_bytes / full_s / 1e9 / 7700.0,
                                    "what": "every entry of the dense W read once (8 n^2 + 16 n bytes), L2 flushed"}},
            "pcg": {"iterations": iters[-1], "iters_per_s": iters[-1] / (ms["pcg"] * 1e-3) if ms["pcg"] else None,
                    "ms": ms["pcg"], "kappa_lanczos": rep.kappa_estimate,
                    "precond_applies_per_s": 1e3 / (am / ac) if ac else None, "precond_apply_us": 1e3 * am / ac if ac else None,
                    "precond_factor_bytes": prec.factor_bytes()},
            "time_to_solution_ms": step_ms,
            "eval_dl": dl,
            "tts_e2e_ms": tts[len(tts) // 2] if tts else None,
            "tts_e2e": ({"ms_median": tts[len(tts) // 2], "ms_min": tts[0], "runs": len(tts), "pcg_iterations": tts_iters,
                         "ms_runs": tts_runs,
                         "what": "S.solve(host MeshLevelPair, g): inflate (fine + coarse), partition_dofs, "
                                 "build_prolongation, assemble_W (plan build, H2D, kernels), assemble_rhs, "
                                 "build_preconditioner, pcg to 1e-8, solution on the host; wall clock"}
                        if tts else None),
            "phases_ms": {k: round(v, 4) for k, v in ms.items()},
            "phase_launches_per_step": launches_per_step,
            "plan_build_ms_host": plan_ms,
            "assembly_stats": stats,
            "e2e": {"value": (1 if shard else world) * npairs / e2e_t, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": 8 * n * n, "ms": e2e_t * 1e3, "ms_min": e2e_min * 1e3,
                    "runs": len(e2e_times) - 1 if len(e2e_times) > 1 else 1, "statistic": "median",
                    "ms_runs": [round(1e3 * t, 2) for t in (e2e_times[1:] if len(e2e_times) > 1 else e2e_times)],
                    "ms_runs_parts": e2e_parts[1:] if len(e2e_parts) > 1 else e2e_parts,
                    "ms_pageable_destination": pageable_ms,
                    "what": "S.assemble_W(host InflatedMesh, out=buf): plan build (host), H2D, kernels, D2H of the "
                            f"n x n W into a {dest} — streamed out while the near field is integrated, then the "
                            "band of entries the near/singular pairs touched copied again (sbg_assemble_w_host); "
                            "the reference arm times assemble_W on an inflated mesh the same way"},
            "gpu_launches": launches,
            "clocks": clocks.summary(),
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def launch_ranks(args) -> int:
    """`bench.py --gpus N` started without a launcher: re-execute under
    torch.distributed.run with N ranks on this node (one GPU each, 127.0.0.1 rendezvous),
    NCCL's init lines left on so the communicator size is visible in the log."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd, env=env).returncode


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "0"))
    if args.gpus > 1 and world == 0:
        sys.exit(launch_ranks(args))
    if world and world != args.gpus:
        sys.exit(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
