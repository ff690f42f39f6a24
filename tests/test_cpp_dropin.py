"""The C++ drop-in header (include/screenbem/gpu.hpp) compiles against the C ABI;
on a B200 the example runs the cmd_solve hot path and matches the Python path."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2310_09204_b200", "_lib")


def build_example(tmp_path):
    exe = str(tmp_path / "dropin")
    cmd = ["g++", "-std=c++17", "-O2", "-Wall", "-Wextra", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "tools", "cpp_dropin_example.cpp"), "-L", LIBDIR, "-lscreenbem_b200",
           f"-Wl,-rpath,{LIBDIR}", "-o", exe]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_cpp_dropin_compiles_and_links(tmp_path):
    build_example(tmp_path)


def test_cpp_dropin_validation_error_maps_to_exit_2(tmp_path):
    exe = build_example(tmp_path)
    r = subprocess.run([exe, "9"], capture_output=True, text=True, timeout=300)
    # unknown config -> ValidationError (exit 2) before any device work, or no device (exit 4)
    assert r.returncode in (2, 4), (r.returncode, r.stderr)


@pytest.mark.gpu
def test_cpp_dropin_runs_cfg1(tmp_path):
    exe = build_example(tmp_path)
    r = subprocess.run([exe, "1"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    assert "dofs 225" in r.stdout and "converged 1" in r.stdout
    from paper_2310_09204_b200 import screenbem as S
    res = S.solve(S.make_config(1), [0.0, 0.0, 1.0], 1e-8)
    assert f"iterations {res.report.iterations}" in r.stdout
    kp = float(r.stdout.split("kappa_prec")[1].split()[0])
    assert kp == pytest.approx(S.condition_number(res.W, res.prec).kappa, rel=1e-8)
    assert float(r.stdout.split("shard_sum_rel")[1].split()[0]) <= 1e-13
    # row-panel PCG through the C++ header: the same iterations, the default pcg's solution to
    # the PCG tolerance, and bitwise the solution of pcg with the full-matrix form (row kernel)
    assert f"rows_iterations {res.report.iterations}" in r.stdout
    assert float(r.stdout.split("rows_max_dx_rel")[1].split()[0]) <= 1e-8
    assert float(r.stdout.split("rows_max_dx_full")[1].split()[0]) == 0.0
    # eval_DL / make_cartesian_grid through the header, against the Python path
    import numpy as np
    g = S.make_cartesian_grid(S.make_config(1).fine, -2.0, 2.0, 9, 9, 0.05)
    U = S.eval_DL(res.report.solution, S.inflate(S.make_config(1).fine), g)
    assert f"dl_points {len(g)}" in r.stdout
    assert float(r.stdout.split("dl_sum")[1].split()[0]) == pytest.approx(float(np.sum(U)), rel=1e-9, abs=1e-14)


@pytest.mark.gpu
def test_cpp_dropin_field_rhs_and_energy_history_cfg2(tmp_path):
    """Config 2 through the C++ header with a non-constant Neumann field g(x)
    (std::function<Vec3(const Vec3&)>, inc/assemble.hpp:143-145) and pcg's exact-solution
    energy history (inc/pcg.hpp:33-35, 48-53): RHS, iterations, solution and the energy
    history against the oracle's pipeline on the same matrix."""
    import numpy as np
    from oracle import oracle as O
    exe = build_example(tmp_path)
    out = str(tmp_path / "field.bin")
    r = subprocess.run([exe, "2", out], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    raw = open(out, "rb").read()
    n, iters, ne = np.frombuffer(raw[:12], dtype=np.int32)
    vals = np.frombuffer(raw[12:], dtype=np.float64)
    L, x, energy, exact = vals[:n], vals[n:2 * n], vals[2 * n:2 * n + ne], vals[2 * n + ne:3 * n + ne]
    assert n == 3969 and ne == iters + 1

    def g(p):
        return [0.3 + p[1] * p[0], -0.2 * p[0] + np.sin(3.0 * p[1]), 1.0 + 0.5 * np.sqrt(p[0] ** 2 + p[1] ** 2 + p[2] ** 2)]
    pair = O.make_config(2)
    fine, coarse = O.inflate(pair.fine), O.inflate(pair.coarse)
    Lo = O.assemble_rhs(fine, g)
    np.testing.assert_allclose(L, Lo, rtol=1e-12, atol=1e-14 * np.abs(Lo).max())
    from paper_2310_09204_b200 import screenbem as S
    W = S.assemble_W(S.inflate(S.make_config(2).fine)).download()
    prec = O.build_preconditioner(W, O.partition_dofs(pair, fine), O.build_prolongation(pair, coarse, fine))
    rep = O.pcg(W, prec, Lo, 1e-8, exact=exact)
    assert abs(int(iters) - rep.iterations) <= 1
    assert np.linalg.norm(x - rep.solution) <= 1e-8 * np.linalg.norm(rep.solution)
    k = min(len(energy), len(rep.energy_error_history))
    np.testing.assert_allclose(energy[:k], rep.energy_error_history[:k], rtol=1e-6,
                               atol=1e-9 * rep.energy_error_history[0])
    assert (np.diff(energy) <= energy[:-1] * 1e-10).all()  # monotone (tests/test_pcg.cpp:95-98)
