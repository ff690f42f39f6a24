"""Summaries of ncu output for profiles/ (run here, on the CPU side, on reports
brought back from the B200 box).

  python tools/ncu_summary.py launches <launches.csv> <out.md>   # per-kernel share of device time
  python tools/ncu_summary.py report <prof.ncu-rep> <out.md>     # key metrics + stall reasons per launch
"""
import collections
import csv
import subprocess
import sys

UNIT = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "second": 1e3, "s": 1e3}


def launches(path, out):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.OrderedDict()
    for r in rows[hdr + 1:]:
        if len(r) <= vi or not r[vi]:
            continue
        name = r[ki].split("(")[0].split("::")[-1].split("<")[0]
        ms = float(r[vi].replace(",", "")) * UNIT.get(r[ui], 1e-6)
        a = agg.setdefault(name, [0.0, 0])
        a[0] += ms
        a[1] += 1
    tot = sum(v[0] for v in agg.values())
    with open(out, "w") as f:
        f.write(f"# ncu launch list summary: `{path}`\n\n")
        f.write("Per-launch device time (`gpu__time_duration.sum`, `--clock-control none`; ncu serialises and "
                "cold-starts every launch, so compare shares, not absolute times).\n\n")
        f.write(f"Total profiled device time: {tot:.3f} ms over {sum(v[1] for v in agg.values())} launches\n\n")
        f.write("| kernel | launches | total ms | share |\n|---|---:|---:|---:|\n")
        for k, v in sorted(agg.items(), key=lambda x: -x[1][0]):
            f.write(f"| `{k}` | {v[1]} | {v[0]:.3f} | {100 * v[0] / tot:.1f}% |\n")
    print(open(out).read())


UNITB = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}

WANT = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "FP64 pipe inst % of peak (active)"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe cycles active %"),
    ("sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active", "DMMA subpipe %"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("dram__bytes_read.sum", "DRAM bytes read"),
    ("dram__bytes_write.sum", "DRAM bytes write"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
]


def report(path, out):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h = rows[0]
    units = {h[i]: rows[1][i] for i in range(min(len(h), len(rows[1])))}
    # one launch per kernel: the longest (the representative large launch)
    best = {}
    for v in rows[2:]:
        d = {h[i]: v[i] for i in range(min(len(h), len(v)))}
        name = d.get("Kernel Name", "?").split("(")[0]
        try:
            dur = float(d.get("gpu__time_duration.sum", "0").replace(",", ""))
        except ValueError:
            dur = 0.0
        if name not in best or dur > best[name][0]:
            best[name] = (dur, d)
    allrows = []
    for v in rows[2:]:
        d = {h[i]: v[i] for i in range(min(len(h), len(v)))}
        allrows.append(d)
    with open(out, "w") as f:
        f.write(f"# ncu --set full summary: `{path}`\n\n")
        f.write("Every captured launch (in launch order):\n\n| # | kernel | duration | FP64 pipe % | DRAM read + write |\n"
                "|---:|---|---:|---:|---:|\n")
        for i, d in enumerate(allrows):
            def num(k):
                try:
                    return float(d.get(k, "nan").replace(",", ""))
                except ValueError:
                    return float("nan")
            rw = num("dram__bytes_read.sum") * UNITB.get(units.get("dram__bytes_read.sum"), 1) + \
                num("dram__bytes_write.sum") * UNITB.get(units.get("dram__bytes_write.sum"), 1)
            f.write(f"| {i} | `{d.get('Kernel Name', '?').split('(')[0].split('::')[-1]}` | "
                    f"{d.get('gpu__time_duration.sum', '?')} {units.get('gpu__time_duration.sum', '')} | "
                    f"{num('sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active'):.1f} | {rw / 1e6:.2f} MB |\n")
        f.write("\n")
        f.write("One launch per kernel (the longest captured); `--clock-control none`, cold caches and "
                "serialised launches, so durations are not the live ones.\n\n")
        for _, d in sorted(best.values(), key=lambda x: -x[0]):
            f.write(f"## `{d.get('Kernel Name', '?')[:120]}`\n\n| metric | value |\n|---|---:|\n")
            for key, label in WANT:
                if key in d:
                    f.write(f"| {label} (`{key}`) | {d[key]} {units.get(key, '')} |\n")
            stalls = []
            for k, val in d.items():
                if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
                    try:
                        stalls.append((float(val), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
                    except ValueError:
                        pass
            if stalls:
                f.write("\nTop stall reasons (warp cycles per issued instruction):\n\n")
                for val, name in sorted(stalls, reverse=True)[:6]:
                    f.write(f"- {name}: {val:.2f}\n")
            f.write("\n")
    print(open(out).read())


if __name__ == "__main__":
    {"launches": launches, "report": report}[sys.argv[1]](sys.argv[2], sys.argv[3])
