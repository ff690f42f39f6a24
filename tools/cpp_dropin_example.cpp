// The reference's cmd_solve hot path (inc/experiments.hpp:130-145) written against
// the C++ drop-in header screenbem/gpu.hpp.  Built and run by tests/test_cpp_dropin.py.
//   g++ -std=c++17 -I include tools/cpp_dropin_example.cpp -L paper_2310_09204_b200/_lib -lscreenbem_b200
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "screenbem/gpu.hpp"

namespace sb = screenbem::gpu;

// row-panel PCG exchange of "rank 1 of 2", emulated in one process: the other panel's
// rows of W p are computed here on the same stream (a real run all-gathers them over NCCL)
struct Emul {
    sbg_ctx* ctx;
    const sbg_matrix* W;
    int lo, hi;
};
static int emulated_exchange(void* user, const double* d_p, double* d_y, int, void*)
{
    const Emul* e = static_cast<const Emul*>(user);
    return sbg_matvec_rows_device(e->ctx, e->W, d_p, d_y, e->lo, e->hi);
}

// the reference's Neumann data as a field (inc/assemble.hpp:143-145 takes a
// std::function<Vec3(const Vec3&)>); a smooth non-constant g
static sb::Vec3 field_g(const sb::Vec3& x)
{
    return sb::Vec3(0.3 + x.y() * x.x(), -0.2 * x.x() + std::sin(3.0 * x.y()), 1.0 + 0.5 * x.norm());
}

// `dropin <cfg> <out.bin>`: the pipeline with the field g and pcg's exact-solution energy
// history (pcg.hpp:33-35); writes n, iterations, L, x, energy history for the test to check
// against the oracle
static int field_run(int cfg, const char* path)
{
    sb::Context ctx(0);
    sb::MeshLevelPair pair = sb::make_config(cfg);
    sb::InflatedMesh fine = sb::inflate(pair.fine());
    sb::InflatedMesh coarse = sb::inflate(pair.coarse());
    sb::GalerkinMatrix W = sb::assemble_W(ctx, fine);
    const std::vector<double> L = sb::assemble_rhs(ctx, fine, field_g);
    sb::SchwarzPreconditioner P =
        sb::build_preconditioner(ctx, W, sb::partition_dofs(pair, fine), sb::build_prolongation(pair, coarse, fine));
    const sb::PcgReport tight = sb::pcg(ctx, W, &P, L, 1e-13);
    const sb::PcgReport rep = sb::pcg(ctx, W, &P, L, 1e-8, 0, &tight.solution);
    std::FILE* f = std::fopen(path, "wb");
    if (!f) return 4;
    const int hdr[3] = {W.rows(), rep.iterations, (int)rep.energy_error_history.size()};
    std::fwrite(hdr, sizeof(int), 3, f);
    std::fwrite(L.data(), sizeof(double), L.size(), f);
    std::fwrite(rep.solution.data(), sizeof(double), rep.solution.size(), f);
    std::fwrite(rep.energy_error_history.data(), sizeof(double), rep.energy_error_history.size(), f);
    std::fwrite(tight.solution.data(), sizeof(double), tight.solution.size(), f);
    std::fclose(f);
    std::printf("field dofs %d iterations %d energy_len %d\n", hdr[0], hdr[1], hdr[2]);
    return rep.converged ? 0 : 3;
}

int main(int argc, char** argv)
{
    const int cfg = argc > 1 ? std::atoi(argv[1]) : 1;
    try {
        if (argc > 2) return field_run(cfg, argv[2]);
        sb::Context ctx(0);
        sb::MeshLevelPair pair = sb::make_config(cfg);
        sb::InflatedMesh fine = sb::inflate(pair.fine());
        sb::InflatedMesh coarse = sb::inflate(pair.coarse());
        sb::GalerkinMatrix W = sb::assemble_W(ctx, fine);
        const double g[3] = {0.0, 0.0, 1.0};
        const std::vector<double> L = sb::assemble_rhs(ctx, fine, g);
        sb::SchwarzPreconditioner P =
            sb::build_preconditioner(ctx, W, sb::partition_dofs(pair, fine), sb::build_prolongation(pair, coarse, fine));
        const sb::PcgReport rep = sb::pcg(ctx, W, &P, L, 1e-8);
        std::printf("dofs %d iterations %d converged %d kappa %.4f\n", W.rows(), rep.iterations, (int)rep.converged,
                    rep.kappa_estimate);
        const sb::SpectrumResult sp = sb::condition_number(ctx, W, P);  // schwarz.hpp:185-190
        std::printf("kappa_prec %.8f\n", sp.kappa);
        // two shards of a multi-GPU assembly sum to W (here both on this GPU)
        const std::vector<double> Wh = W.download();
        std::vector<double> Ws = sb::assemble_W_shard(ctx, fine, 0, 2).download();
        const std::vector<double> W1 = sb::assemble_W_shard(ctx, fine, 1, 2).download();
        double dmax = 0.0, wmax = 0.0;
        for (size_t k = 0; k < Wh.size(); ++k) {
            dmax = std::max(dmax, std::fabs(Ws[k] + W1[k] - Wh[k]));
            wmax = std::max(wmax, std::fabs(Wh[k]));
        }
        std::printf("shard_sum_rel %.3e\n", dmax / wmax);
        const int half = (W.rows() + 1) / 2;
        Emul em{ctx.get(), W.get(), 0, half};
        const sb::PcgReport rr = sb::pcg_rows(ctx, W, &P, L, half, W.rows(), emulated_exchange, &em, 1e-8);
        // against the default pcg (symmetric matvec) to the PCG tolerance, and bitwise against
        // pcg with the full-matrix form, whose row kernel the panels share
        ctx.set_matvec_form(1);
        const sb::PcgReport rf = sb::pcg(ctx, W, &P, L, 1e-8);
        ctx.set_matvec_form(0);
        double xd = 0.0, xf = 0.0, xn = 0.0;
        for (size_t k = 0; k < rr.solution.size(); ++k) {
            xd = std::max(xd, std::fabs(rr.solution[k] - rep.solution[k]));
            xf = std::max(xf, std::fabs(rr.solution[k] - rf.solution[k]));
            xn = std::max(xn, std::fabs(rep.solution[k]));
        }
        std::printf("rows_iterations %d rows_max_dx_rel %.3e rows_max_dx_full %.3e\n", rr.iterations, xd / xn, xf);
        // the solution's double-layer potential on the reference's evaluation grid (potential.hpp)
        const sb::EvaluationGrid grid = sb::make_cartesian_grid(ctx, pair.fine(), -2.0, 2.0, 9, 9, 0.05);
        const std::vector<double> U = sb::eval_DL(ctx, rep.solution, fine, grid);
        double us = 0.0;
        for (double u : U) us += u;
        std::printf("dl_points %d dl_sum %.17g\n", (int)grid.points.size(), us);
        return rep.converged ? 0 : 3;
    } catch (const screenbem::ValidationError& e) {
        std::fprintf(stderr, "validation error: %s\n", e.what());
        return 2;
    } catch (const screenbem::NumericalError& e) {
        std::fprintf(stderr, "numerical error: %s\n", e.what());
        return 3;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 4;
    }
}
