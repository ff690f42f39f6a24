"""Load balance of the sharded assembly (bench.py --shard), measured on one GPU: each
shard (rank r of N) is assembled alone and timed with CUDA events; the max over ranks is
the compute part of an N-GPU assembly (the NCCL all-reduce of the partial W comes on top).

    python tools/shard_probe.py [--config 5] [--worlds 2,4,8]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_09204_b200 import screenbem as S  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--worlds", default="2,4,8")
    args = ap.parse_args()
    ctx = S.Context(0)
    ctx.timers(True)
    pair = S.make_config(args.config, 8 if args.config == 5 else 0)
    im = S.inflate(pair.fine, validate=False)
    plan = S.AssemblyPlan(im, ctx=ctx)
    W = plan.run()
    W = plan.run(W)
    ctx.reset_timers()
    W = plan.run(W)
    full = ctx.timer("assemble_W")[0]
    out = {"config": args.config, "full_ms": full, "worlds": {}}
    for world in [int(w) for w in args.worlds.split(",")]:
        ts = []
        for r in range(world):
            plan.run(W, shard=(r, world))  # warm (first use of this shard's buffers)
            ctx.reset_timers()
            plan.run(W, shard=(r, world))
            ts.append(ctx.timer("assemble_W")[0])
        out["worlds"][world] = {"max_ms": max(ts), "mean_ms": sum(ts) / world, "min_ms": min(ts),
                                "imbalance": max(ts) / (sum(ts) / world),
                                "compute_speedup": full / max(ts), "per_rank_ms": ts}
        print(json.dumps({world: out["worlds"][world]}), flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
