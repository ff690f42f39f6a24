"""bench.py keeps the driver contract: one JSON line with the required keys (the reference
arm on the CPU here, our arm on a B200 with `-m gpu`)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_bench(*args, timeout=900):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_reference_arm_json_line():
    d = run_bench("--impl", "reference", "--config", "1", "--steps", "1", "--warmup", "0", "--cpu-seconds", "1",
                  "--no-cpu-phases")
    assert d["impl"] == "reference"
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["value"] > 0 and d["unit"] == "tri-pairs/s" and d["higher_is_better"] is True
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["config"] == {"workload": "config 1: flat 16x16 (512 tri), H/h 8", "triangles": 512, "dofs": 225,
                           "tri_pairs": 131328, "h_ratio": 8, "pcg_tol": 1e-8}


def test_reference_arm_never_loads_the_product_library():
    """the reference arm runs the oracle alone: meshes from the oracle's own config
    generator, the assembly sample from oracle.AssemblySampler"""
    code = ("import sys, bench; sys.argv = ['bench.py', '--impl', 'reference', '--config', '1', '--steps', '1', "
            "'--warmup', '0', '--cpu-seconds', '1']; bench.main(); "
            "assert 'paper_2310_09204_b200.screenbem' not in sys.modules, 'product imported'; "
            "maps = open('/proc/self/maps').read(); assert 'libscreenbem_b200' not in maps, 'product mapped'")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]


def test_cpu_sample_is_unbiased():
    """the systematic pair sample covers the reference pair order evenly: the fraction of
    sampled pairs in any contiguous slice of the order matches the slice's share"""
    from oracle import oracle as O
    nf = 51200
    total = nf * (nf + 1) // 2
    idx = O.systematic_pair_sample(nf, 100000)
    assert len(idx) == 100000 and (idx[1:] > idx[:-1]).all() and idx[0] >= 0 and idx[-1] < total
    for lo, hi in [(0, total // 10), (total // 2, total // 2 + total // 7), (total - total // 20, total)]:
        share = ((idx >= lo) & (idx < hi)).mean()
        assert abs(share - (hi - lo) / total) < 2e-4


@pytest.mark.gpu
def test_our_arm_json_line():
    d = run_bench("--config", "1", "--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--tts-runs", "1")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["steps"] == 3 and d["warmup"] == 3 and d["n_gpus"] == 1 and d["dtype"] == "f64"
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in d["roofline"], k
    assert 0 < d["roofline"]["frac"] < 1.2
    for k in ("value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"):
        assert k in d["e2e"], k
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0
    assert "workload" in d["config"]
    assert d["tts_e2e_ms"] > 0 and d["e2e"]["statistic"] == "median" and d["e2e"]["ms_min"] <= d["e2e"]["ms"]
    # the full-matrix matvec is reported beside the context's (symmetric) form: 8 n^2 + 16 n bytes
    mv = d["roofline_matvec"]
    n = d["config"]["dofs"]
    assert mv["bound"] == "hbm" and mv["full_form"]["bytes_per_launch"] == 8.0 * n * n + 16.0 * n
    assert mv["full_form"]["us_per_launch"] > 0 and mv["full_form"]["achieved"] > 0


@pytest.mark.gpu
def test_our_arm_two_ranks_one_command():
    """`bench.py --gpus 2` launches two ranks itself; N > 1 assembles ONE W across them
    (strong scaling).  gloo lets both ranks share the box's one GPU (functional check,
    not a timing)."""
    d = run_bench("--gpus", "2", "--dist-backend", "gloo", "--config", "1", "--steps", "2", "--warmup", "3",
                  "--no-cpu-baseline", "--clocks", "off")
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and d["pcg"]["iterations"] > 0
