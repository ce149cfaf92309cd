// ORACLE / TEST INFRASTRUCTURE ONLY: the drop-in check of include/sdc_gpu.hpp.
//
// Builds a coupled system with the reference's own assembly, solves it with
// the reference's CPU path (td_bgs(Uzawa(AMG), AMG) + pd_gmres wired as
// bench.cpp:121-182) and with the GPU path through the adapter, and also runs
// the reference's own sdc::pd_gmres with the GPU preconditioner plugged in as
// an sdc::Preconditioner.  Compiled by `make -C oracle adapter`, run by
// tests/test_gpu_adapter.py on a GPU box.
#include <cmath>
#include <cstdio>
#include <stdexcept>

#include "sdc/assembly.hpp"
#include "sdc/krylov.hpp"
#include "sdc/precond.hpp"
#include "sdc_gpu.hpp"

using namespace sdc;

static double rel_l2(const std::vector<double>& x, const std::vector<double>& y) {
    double num = 0.0, den = 0.0;
    for (size_t i = 0; i < x.size(); ++i) {
        num += (x[i] - y[i]) * (x[i] - y[i]);
        den += y[i] * y[i];
    }
    return std::sqrt(num / den);
}

int main(int argc, char** argv) {
    const int n = argc > 1 ? std::atoi(argv[1]) : 16;
    ScenarioConfig cfg;
    cfg.cells_per_unit_square = n;
    cfg.permeability = 1e-2;
    cfg.alpha_bj = 1.0;
    cfg.kinematic_viscosity = 1.0;
    cfg.density = 1.0;
    cfg.dt = std::numeric_limits<double>::infinity();
    cfg.t_end = 1.0;
    cfg.dp_max = 1.0;
    StaggeredGrid g;
    g.cells_per_unit = n;
    g.h = 1.0 / n;
    g.ff = StokesBox{n, n, g.h};
    g.pm = DarcyBox{n, n, g.h};
    CoupledSystem sys = assemble_monolithic(g, cfg, {}, 1.0);
    const double tol = 1e-8 * norm2(sys.rhs);

    // reference CPU path (bench.cpp:121-182)
    const int n_v = sys.pv_v.size(), n_pff = sys.pv_pff.size(), n_ppm = sys.pv_ppm.size(), n_ff = sys.td_ff.size();
    auto d_block = ground_dof(submatrix(sys.matrix, n_ff, sys.n_total(), n_ff, sys.n_total()));
    std::vector<int> comps(n_v, 0);
    for (int k = g.ff.n_u(); k < n_v; ++k) comps[k] = 1;
    UzawaConfig ucfg;
    ucfg.amg.components = comps;
    auto first = std::make_shared<UzawaPreconditioner>(submatrix(sys.matrix, 0, n_v, 0, n_v),
                                                       submatrix(sys.matrix, 0, n_v, n_v, n_ff),
                                                       submatrix(sys.matrix, n_v, n_ff, 0, n_v), ucfg);
    auto pm = std::make_shared<AmgPreconditioner>(d_block);
    BlockPreconditioner cpu_p(BlockPrecondKind::td_bgs, sys.matrix, n_v, n_pff, n_ppm, first, pm);
    RestartController fixed50;
    fixed50.m_init = fixed50.m_min = fixed50.m_max = fixed50.current_m = 50;
    auto cpu = pd_gmres(LinearOperator::from_matrix(sys.matrix), &cpu_p, sys.rhs, tol, 400, fixed50);

    // GPU path through the adapter
    sdc_gpu::Context ctx;
    sdc_gpu::Matrix A(ctx, sys.matrix);
    auto gpu_p = sdc_gpu::td_bgs(A, sys);
    auto gpu = sdc_gpu::pd_gmres(A, gpu_p.get(), sys.rhs, tol, 400, fixed50);
    const double d1 = rel_l2(gpu.x, cpu.x);
    std::printf("cpu iterations %d, gpu iterations %d, rel diff %.3e, omega cpu %.6e gpu %.6e\n",
                cpu.report.iterations, gpu.report.iterations, d1, first->omega(), gpu_p->omega());

    // the reference's own Krylov driver with the GPU preconditioner plugged in
    auto mixed = pd_gmres(LinearOperator::from_matrix(sys.matrix), gpu_p.get(), sys.rhs, tol, 400, fixed50);
    const double d2 = rel_l2(mixed.x, cpu.x);
    std::printf("reference pd_gmres + GPU preconditioner: iterations %d, rel diff %.3e, applications %lld\n",
                mixed.report.iterations, d2, static_cast<long long>(gpu_p->applications()));

    // the GPU operator behind the reference's LinearOperator
    auto op = A.op();
    std::vector<double> y(sys.n_total()), y_ref(sys.n_total());
    op.apply(sys.rhs, y);
    spmv(sys.matrix, sys.rhs, y_ref);
    const bool spmv_exact = y == y_ref;

    // exception mapping
    bool threw = false;
    try {
        std::vector<double> bad(3, 1.0);
        sdc_gpu::pd_gmres(A, gpu_p.get(), bad, tol, 10, fixed50);
    } catch (const std::invalid_argument&) {
        threw = true;
    }

    const int it_ref = cpu.report.iterations;
    const bool ok = cpu.report.converged && gpu.report.converged && mixed.report.converged &&
                    std::abs(gpu.report.iterations - it_ref) <= std::max(1.0, 0.05 * it_ref) && d1 <= 1e-6 &&
                    d2 <= 1e-6 && spmv_exact && threw;
    std::printf("spmv bitwise %d, dimension error -> std::invalid_argument %d\n%s\n", spmv_exact, threw,
                ok ? "ADAPTER OK" : "ADAPTER FAILED");
    return ok ? 0 : 1;
}
