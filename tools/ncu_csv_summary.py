"""Markdown summary of an `ncu --page raw --csv` export (one row per profiled launch), for
profiles/: the metrics the roofline discussion cites, per launch, and the top stall reasons.
The .ncu-rep files themselves stay on the box (gpurun brings back at most 64 MiB).

    python tools/ncu_csv_summary.py <raw.csv[.gz]> <title> > profiles/<name>.md
"""
import csv
import gzip
import sys

KEYS = [("duration", "gpu__time_duration.sum", "us"),
        ("FP64 pipe % (active)", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "%"),
        ("FP64 inst % (active)", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "%"),
        ("DMMA subpipe % (active)", "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", "%"),
        ("issue slots busy %", "smsp__issue_active.avg.pct_of_peak_sustained_active", "%"),
        ("achieved occupancy %", "sm__warps_active.avg.pct_of_peak_sustained_active", "%"),
        ("DRAM read", "dram__bytes_read.sum", "B"),
        ("DRAM write", "dram__bytes_write.sum", "B"),
        ("DRAM throughput %", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "%"),
        ("registers/thread", "launch__registers_per_thread", ""),
        ("grid", "launch__grid_size", ""),
        ("block", "launch__block_size", "")]


BYTES = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
TIME_US = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6}


def fmt(v, unit, src_unit=""):
    try:
        x = float(v.replace(",", ""))
    except (ValueError, AttributeError):
        return v
    if x != x:
        return "n/a (not collected)"
    if unit == "B":
        return f"{x * BYTES.get(src_unit, 1.0) / 1e6:.3f} MB"
    if unit == "us":
        return f"{x:.1f}"
    if unit == "%":
        return f"{x:.1f}"
    return f"{x:.0f}"


def main(path, title):
    op = gzip.open if path.endswith(".gz") else open
    rows = list(csv.reader(op(path, "rt")))
    hdr, units = rows[0], rows[1]
    data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]
    print(f"# {title}\n")
    print(f"Source: `{path}` (`ncu --set full --clock-control none`, exported with `--page raw --csv`). "
          "ncu replays each launch with cold caches and serialised launches: durations are not the live ones; "
          "the pipe utilisations and DRAM bytes are the kernel's own.\n")
    dur_unit = units[hdr.index("gpu__time_duration.sum")] if "gpu__time_duration.sum" in hdr else "ns"
    for d in data:
        name = d.get("Kernel Name", "?")
        short = name.split("(")[0].replace("(anonymous namespace)::", "").replace("void ", "")
        print(f"## `{short}` (ID {d.get('ID', '?')})\n")
        print("| metric | value |\n|---|---:|")
        for label, key, unit in KEYS:
            if key not in d:
                continue
            v = d[key]
            if key == "gpu__time_duration.sum":
                x = float(v.replace(",", "")) * TIME_US.get(dur_unit, 1e-3)
                print(f"| {label} (us) | {x:.1f} |")
                continue
            print(f"| {label} | {fmt(v, unit, units[hdr.index(key)])} |")
        stalls = []
        for k, v in d.items():
            if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
                try:
                    stalls.append((float(v), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        if stalls:
            print("\nTop stalls (warp cycles per issued instruction): " +
                  ", ".join(f"{n} {v:.2f}" for v, n in stalls[:5]) + "\n")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else sys.argv[1])
