"""Summaries for profiles/ from the outputs of tools/profile_r02b.sh (the same command list serves the later capture sets) and the per-config bench
runs brought back in gpurun_out/ (run here, on the CPU side):

    python tools/write_r02b_profiles.py [tag]   (default tag r02c)
"""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")
TAG = sys.argv[1] if len(sys.argv) > 1 else "r02c"  # the capture set's name in profiles/


def last_json(path):
    return json.loads(open(path).read().strip().splitlines()[-1])


def main():
    # bench lines
    for c in (1, 2, 3, 4, 5):
        src = os.path.join(G, "final_bench_cfg5.json" if c == 5 else f"bench_cfg{c}.json")
        if os.path.exists(src):
            json.dump(last_json(src), open(os.path.join(P, f"{TAG}_bench_cfg{c}.json"), "w"), indent=1)
    d5 = json.load(open(os.path.join(P, f"{TAG}_bench_cfg5.json")))
    stats = d5["assembly_stats"]
    evals = {"far": stats["far_pairs"] * 256.0, "near": stats["near_leaves"] * 1296.0}
    # config-5 far/near metrics
    rows = [r for r in csv.reader(open(os.path.join(G, "asm5_metrics.csv"))) if len(r) > 10]
    h = rows[0]
    ik, im, iv, iu = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    m = {}
    for r in rows[1:]:
        m.setdefault("far" if "k_far_tiles" in r[ik] else "near", {})[r[im]] = (r[iv].replace(",", ""), r[iu])
    names = [("gpu__time_duration.sum", "duration"),
             ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe % (active)"),
             ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
             ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
             ("dram__bytes_read.sum", "DRAM read"), ("dram__bytes_write.sum", "DRAM write"),
             ("smsp__inst_executed.sum", "warp instructions executed"),
             ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "shared-load wavefronts"),
             ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "shared-load bank conflicts"),
             ("launch__registers_per_thread", "registers/thread"), ("launch__grid_size", "grid"),
             ("launch__block_size", "block")]
    out = [f"# Config-5 assembly kernels — ncu metrics capture ({TAG}: flat-plane evaluation, two-stage contraction, "
           "padded leaf staging, 7-instruction evaluation)", "",
           "`ncu --metrics <list below> --clock-control none -k regex:'k_far_tiles|k_near_leaves' --launch-skip 2 "
           "-c 2 --csv python tools/asm_once.py 5` (`tools/profile_r02b.sh`; the second assembly's launches). ncu "
           "serialises launches and starts them cold; the pipe utilisations, instruction counts and DRAM bytes are "
           "the kernels' own.", "", "| metric | k_far_tiles<16,0> | k_near_leaves |", "|---|---:|---:|"]
    for key, lab in names:
        a, b = m["far"].get(key, ("", "")), m["near"].get(key, ("", ""))
        out.append(f"| {lab} (`{key}`) | {a[0]} {a[1]} | {b[0]} {b[1]} |")
    ipe = {k: float(m[k]["smsp__inst_executed.sum"][0]) * 32 / evals[k] for k in ("far", "near")}
    out += ["", f"Thread instructions per kernel evaluation: far tiles {ipe['far']:.2f}, near leaves {ipe['near']:.2f} "
            f"(evaluations: far {evals['far']:.4g} = 256 per far pair, near {evals['near']:.4g} = 1296 per leaf). "
            "The flat evaluation is 7 FP64 instructions + MUFU.RSQ64H + its zero low word + a share of the "
            "shared-memory loads and loop overhead; the rest is per-tile / per-leaf setup, classification, the "
            "contraction and the flush."]
    open(os.path.join(P, f"{TAG}_ncu_cfg5_asm.md"), "w").write("\n".join(out) + "\n")
    # traffic / pipe json
    tj = os.path.join(P, "r02_traffic.json")
    t = json.load(open(tj))
    for k, name in (("far", "far_tiles"), ("near", "near_leaves")):
        t[name]["5"] = {"kernel": "k_far_tiles<16, 0>" if k == "far" else "k_near_leaves", "launches_per_step": 1,
                        "dram_bytes_per_step": [int(float(m[k]["dram__bytes_read.sum"][0]) +
                                                    float(m[k]["dram__bytes_write.sum"][0]))],
                        "fp64_pipe_active": round(float(
                            m[k]["sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"][0]) / 100, 4),
                        "fp64_instr_per_eval": 7, "source": "profiles/" + TAG + "_ncu_cfg5_asm.md"}
    json.dump(t, open(tj, "w"), indent=1)
    # launch list, config-2 full capture, SASS
    tools = os.path.join(ROOT, "tools")
    subprocess.run([sys.executable, os.path.join(tools, "ncu_summary.py"), "launches",
                    os.path.join(G, "launches_cfg5.csv"), os.path.join(P, f"{TAG}_launches_bench_cfg5.md")],
                   check=True, capture_output=True)
    lp = os.path.join(P, f"{TAG}_launches_bench_cfg5.md")
    lines = open(lp).read().splitlines()
    lines[0] = ("# ncu launch list summary: `SBG_PCG_GRAPH=0 ncu --metrics gpu__time_duration.sum --clock-control "
                "none python bench.py --steps 2 --warmup 1 --no-cpu-baseline --tts-runs 1 --dl-grid 0` (config 5, "
                "final r02 code; the PCG loop on the stream so its kernels are listed)")
    open(lp, "w").write("\n".join(lines) + "\n")
    subprocess.run([sys.executable, os.path.join(tools, "ncu_summary.py"), "report",
                    os.path.join(G, "asm2_full.ncu-rep"), os.path.join(P, f"{TAG}_ncu_full_cfg2_asm.md")],
                   check=True, capture_output=True)
    with open(os.path.join(P, f"{TAG}_sass.md"), "w") as f:
        subprocess.run([sys.executable, os.path.join(tools, "sass_summary.py")], check=True, stdout=f,
                       stderr=subprocess.DEVNULL)
    print("written")


if __name__ == "__main__":
    main()
