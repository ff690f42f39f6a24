"""Aggregate an ncu `--metrics gpu__time_duration.sum --csv` launch list by kernel, from the
last launch of `start` (default k_pcg_init) on: count, total and mean duration per kernel."""
import collections
import csv
import sys


def main(path, start="k_pcg_init"):
    rows = list(csv.DictReader(l for l in open(path) if not l.startswith("==")))
    names = [r["Kernel Name"] for r in rows]
    idx = [i for i, nm in enumerate(names) if start in nm]
    sel = rows[idx[-1]:] if idx else rows
    agg = collections.OrderedDict()
    for r in sel:
        nm = r["Kernel Name"].split("(")[0].replace("sbg::", "").replace("(anonymous namespace)::", "")
        v = float(r["Metric Value"].replace(",", ""))
        us = v / 1000 if r["Metric Unit"] in ("nsecond", "ns") else v * 1000 if r["Metric Unit"] in ("msecond", "ms") else v
        a = agg.setdefault(nm, [0, 0.0])
        a[0] += 1
        a[1] += us
    tot = sum(a[1] for a in agg.values())
    print(f"| kernel | launches | total us | us/launch | share |\n|---|---|---|---|---|")
    for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"| `{k}` | {c} | {t:.1f} | {t / c:.2f} | {100 * t / tot:.1f}% |")
    print(f"| total | {sum(a[0] for a in agg.values())} | {tot:.1f} | | |")


if __name__ == "__main__":
    main(*sys.argv[1:])
