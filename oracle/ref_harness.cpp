// ORACLE / TEST INFRASTRUCTURE ONLY.
//
// C-ABI shim over the UNMODIFIED reference library `sdcore`, compiled from
// /root/reference/proj/core/src by oracle/Makefile into oracle/_ref/.
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// --impl reference leg may load the resulting library.  It is the checker,
// never the product: nothing in paper_2108_13229_b200/ links against it.
//
// Every entry point forwards to the reference's public API; the wiring of the
// block preconditioner mirrors MonolithicDriver::build_preconditioner
// (proj/core/src/bench.cpp:121-182) with AmgOptions.max_levels exposed,
// because SURVEY.md §8(d) makes the AMG depth a per-config parity input.
// The n x n free-flow box follows SURVEY.md §8(d) (build_grid would make it
// n x 3n, proj/core/src/grid.cpp:65).

#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "sdc/assembly.hpp"
#include "sdc/krylov.hpp"
#include "sdc/lu.hpp"
#include "sdc/precond.hpp"
#include "sdc/sparse.hpp"

using namespace sdc;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::runtime_error& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 3;
    }
}

SparseMatrix from_csr(int n_rows, int n_cols, const int* rp, const int* ci, const double* v) {
    SparseMatrix m(n_rows, n_cols);
    m.row_offsets.assign(rp, rp + n_rows + 1);
    const int nnz = rp[n_rows];
    m.col_indices.assign(ci, ci + nnz);
    m.values.assign(v, v + nnz);
    return m;
}

struct SystemHandle {
    CoupledSystem sys;
};

// Everything a td_* solve needs, kept alive together.
struct MatrixHandle {
    SparseMatrix a;
};

struct HierHandle {
    AMGHierarchy h;
};

struct PrecondHandle {
    std::shared_ptr<const Preconditioner> p;
};

struct TdHandle {
    SparseMatrix a;                         // the monolithic matrix (owned copy)
    std::shared_ptr<UzawaPreconditioner> uz;
    std::shared_ptr<Preconditioner> pm;
    std::shared_ptr<BlockPreconditioner> block;
    HierHandle v_h;                         // same deterministic setup as inside uz
    HierHandle d_h;
    double setup_seconds = 0.0;
};

void copy_csr(const SparseMatrix& m, int* rp, int* ci, double* v) {
    if (rp) std::memcpy(rp, m.row_offsets.data(), sizeof(int) * (m.n_rows + 1));
    if (ci) std::memcpy(ci, m.col_indices.data(), sizeof(int) * m.nnz());
    if (v) std::memcpy(v, m.values.data(), sizeof(double) * m.nnz());
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---------------------------------------------------------------------------
// system assembly (reference assemble_monolithic, n x n free-flow box)

int ref_system_new(int n, double permeability, double alpha_bj, double nu, double rho,
                   double dt, double t_end, double dp_max, double t, const double* v_prev,
                   void** out) {
    return guarded([&] {
        ScenarioConfig cfg;
        cfg.cells_per_unit_square = n;
        cfg.permeability = permeability;
        cfg.alpha_bj = alpha_bj;
        cfg.kinematic_viscosity = nu;
        cfg.density = rho;
        cfg.dt = dt;
        cfg.t_end = t_end;
        cfg.dp_max = dp_max;
        StaggeredGrid g;
        g.cells_per_unit = n;
        g.h = 1.0 / n;
        g.ff = StokesBox{n, n, g.h};
        g.pm = DarcyBox{n, n, g.h};
        std::vector<double> vp;
        if (v_prev) vp.assign(v_prev, v_prev + g.n_vel());
        auto* h = new SystemHandle{assemble_monolithic(g, cfg, vp, t)};
        *out = h;
    });
}

void ref_system_sizes(void* hs, int* n, long long* nnz, int* n_u, int* n_vel, int* n_pff,
                      int* n_ppm) {
    auto* h = static_cast<SystemHandle*>(hs);
    *n = h->sys.n_total();
    *nnz = h->sys.matrix.nnz();
    *n_u = h->sys.grid.ff.n_u();
    *n_vel = h->sys.grid.n_vel();
    *n_pff = h->sys.grid.n_pff();
    *n_ppm = h->sys.grid.n_ppm();
}

void ref_system_copy(void* hs, int* rp, int* ci, double* v, double* rhs) {
    auto* h = static_cast<SystemHandle*>(hs);
    copy_csr(h->sys.matrix, rp, ci, v);
    if (rhs) std::memcpy(rhs, h->sys.rhs.data(), sizeof(double) * h->sys.rhs.size());
}

void ref_system_free(void* hs) { delete static_cast<SystemHandle*>(hs); }

// ---------------------------------------------------------------------------
// partitioned pieces (coupling.cpp:218-242): the standalone Stokes system with
// Dirichlet interface velocities and the Darcy system with Dirichlet interface
// pressures, on the n x n boxes, with the traces that close the loop.

static ScenarioConfig scenario_of(int n, double permeability, double alpha_bj, double nu, double rho, double dt,
                                  double t_end, double dp_max) {
    ScenarioConfig cfg;
    cfg.cells_per_unit_square = n;
    cfg.permeability = permeability;
    cfg.alpha_bj = alpha_bj;
    cfg.kinematic_viscosity = nu;
    cfg.density = rho;
    cfg.dt = dt;
    cfg.t_end = t_end;
    cfg.dp_max = dp_max;
    return cfg;
}

// matrix handle + rhs of assemble_stokes(StokesBox{n,n,h}, ..., &v_gamma)
int ref_stokes_new(int n, double permeability, double alpha_bj, double nu, double rho, double dt, double t_end,
                   double dp_max, double t, const double* v_prev, const double* v_gamma, void** mat_out,
                   double* rhs_out) {
    return guarded([&] {
        const ScenarioConfig cfg = scenario_of(n, permeability, alpha_bj, nu, rho, dt, t_end, dp_max);
        const StokesBox box{n, n, 1.0 / n};
        StokesBcs bcs;
        bcs.left = StokesSideBc::pressure_bc(cfg.inflow_pressure(t));
        bcs.right = StokesSideBc::pressure_bc(0.0);
        bcs.top = StokesSideBc::wall();
        std::vector<double> vp;
        if (v_prev) vp.assign(v_prev, v_prev + box.n_vel());
        std::vector<double> vg(v_gamma, v_gamma + n);
        auto sys = assemble_stokes(box, FlowParams::from(cfg), vp, bcs, &vg);
        std::memcpy(rhs_out, sys.rhs.data(), sizeof(double) * sys.rhs.size());
        *mat_out = new MatrixHandle{std::move(sys.matrix)};
    });
}

// matrix handle + rhs of assemble_darcy(DarcyBox{n,n,h}, K/mu, {}, &p_gamma)
int ref_darcy_new(int n, double k_over_mu, const double* p_gamma, void** mat_out, double* rhs_out) {
    return guarded([&] {
        const DarcyBox box{n, n, 1.0 / n};
        std::vector<double> pg(p_gamma, p_gamma + n);
        auto sys = assemble_darcy(box, k_over_mu, DarcyBcs{}, &pg);
        std::memcpy(rhs_out, sys.rhs.data(), sizeof(double) * sys.rhs.size());
        *mat_out = new MatrixHandle{std::move(sys.matrix)};
    });
}

int ref_stokes_pressure_trace(int n, double mu, const double* solution, double* trace) {
    return guarded([&] {
        const StokesBox box{n, n, 1.0 / n};
        auto tr = stokes_pressure_trace(box, mu, std::span<const double>(solution, box.n_total()));
        std::memcpy(trace, tr.data(), sizeof(double) * tr.size());
    });
}

int ref_darcy_velocity_trace(int n, double k_over_mu, const double* p, const double* p_gamma, double* trace) {
    return guarded([&] {
        const DarcyBox box{n, n, 1.0 / n};
        auto tr = darcy_velocity_trace_dirichlet(box, k_over_mu, std::span<const double>(p, box.n_p()),
                                                 std::span<const double>(p_gamma, n));
        std::memcpy(trace, tr.data(), sizeof(double) * tr.size());
    });
}

// UzawaPreconditioner(v, b, c, cfg) on a Stokes matrix (the CouplingDriver's
// Stokes-side preconditioner, coupling.cpp:115-138) and AmgPreconditioner on a
// Darcy matrix (coupling.cpp:140-146), as opaque handles usable with
// ref_pd_gmres / ref_bicgstab (precond kinds 3 and 4).
int ref_uzawa_stokes_new(void* mat, int n, int max_levels, void** out) {
    return guarded([&] {
        const SparseMatrix& a = static_cast<MatrixHandle*>(mat)->a;
        const StokesBox box{n, n, 1.0 / n};
        const int n_vel = box.n_vel(), nt = box.n_total();
        UzawaConfig ucfg;
        ucfg.mode = UzawaConfig::Mode::inexact;
        ucfg.amg.max_levels = max_levels;
        ucfg.amg.components.assign(n_vel, 0);
        for (int k = box.n_u(); k < n_vel; ++k) ucfg.amg.components[k] = 1;
        *out = new PrecondHandle{std::make_shared<UzawaPreconditioner>(
            submatrix(a, 0, n_vel, 0, n_vel), submatrix(a, 0, n_vel, n_vel, nt), submatrix(a, n_vel, nt, 0, n_vel),
            ucfg)};
    });
}

int ref_amg_precond_new(void* mat, int max_levels, void** out) {
    return guarded([&] {
        AmgOptions o;
        o.max_levels = max_levels;
        *out = new PrecondHandle{std::make_shared<AmgPreconditioner>(static_cast<MatrixHandle*>(mat)->a, o)};
    });
}

void ref_precond_free(void* p) { delete static_cast<PrecondHandle*>(p); }

// ILU(0) (precond.cpp:13-87) of a matrix, and a plain apply of any precond handle.
int ref_ilu0_new(void* mat, void** out) {
    return guarded([&] {
        *out = new PrecondHandle{std::make_shared<Ilu0Preconditioner>(static_cast<MatrixHandle*>(mat)->a)};
    });
}

int ref_precond_apply(void* p, const double* r, double* z) {
    return guarded([&] {
        const auto& pc = static_cast<PrecondHandle*>(p)->p;
        const int n = pc->rows();
        pc->apply(std::span<const double>(r, n), std::span<double>(z, n));
    });
}


// Interface traces of a monolithic solution (assembly.cpp:382-428).
int ref_system_traces(void* hs, const double* x, double* p_ff_gamma, double* v_pm_gamma) {
    return guarded([&] {
        auto* h = static_cast<SystemHandle*>(hs);
        std::span<const double> sx(x, h->sys.n_total());
        auto st = extract_interface_traces(h->sys, sx);
        std::memcpy(p_ff_gamma, st.p_ff_gamma.data(), sizeof(double) * st.p_ff_gamma.size());
        std::memcpy(v_pm_gamma, st.v_pm_gamma.data(), sizeof(double) * st.v_pm_gamma.size());
    });
}

// ---------------------------------------------------------------------------
// sparse kernels (sparse.cpp)

int ref_spmv(int n_rows, int n_cols, const int* rp, const int* ci, const double* v,
             const double* x, double* y) {
    return guarded([&] {
        auto a = from_csr(n_rows, n_cols, rp, ci, v);
        spmv(a, std::span<const double>(x, n_cols), std::span<double>(y, n_rows));
    });
}

int ref_spmv_add(int n_rows, int n_cols, const int* rp, const int* ci, const double* v,
                 const double* x, double* y, double alpha) {
    return guarded([&] {
        auto a = from_csr(n_rows, n_cols, rp, ci, v);
        spmv_add(a, std::span<const double>(x, n_cols), std::span<double>(y, n_rows), alpha);
    });
}

int ref_sor_sweep(int n, const int* rp, const int* ci, const double* v, double* z,
                  const double* r, double omega) {
    return guarded([&] {
        auto a = from_csr(n, n, rp, ci, v);
        sor_sweep(a, std::span<double>(z, n), std::span<const double>(r, n), omega);
    });
}

void ref_random_vector(int n, unsigned seed, double* out) {
    // same generator family as the reference tests' random_vector
    // (tests/support/dense_oracles.hpp:202-208): mt19937 + uniform(-1, 1)
    std::mt19937 rng(seed);
    std::uniform_real_distribution<double> val(-1.0, 1.0);
    for (int i = 0; i < n; ++i) out[i] = val(rng);
}

// Random diagonally dominant matrix in the manner of the reference tests'
// random_dominant (tests/support/dense_oracles.hpp:177-200).
int ref_random_dominant(int n, double density, unsigned seed, int symmetric, void** out) {
    return guarded([&] {
        std::mt19937 rng(seed);
        std::uniform_real_distribution<double> val(-1.0, 1.0);
        std::uniform_real_distribution<double> coin(0.0, 1.0);
        std::vector<double> d(static_cast<std::size_t>(n) * n, 0.0);
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j)
                if (i != j && coin(rng) < density) d[i * (std::size_t)n + j] = val(rng);
        if (symmetric)
            for (int i = 0; i < n; ++i)
                for (int j = 0; j < i; ++j) d[i * (std::size_t)n + j] = d[j * (std::size_t)n + i];
        for (int i = 0; i < n; ++i) {
            double s = 0.0;
            for (int j = 0; j < n; ++j)
                if (j != i) s += std::abs(d[i * (std::size_t)n + j]);
            d[i * (std::size_t)n + i] = s + 1.0 + std::abs(val(rng));
        }
        CooBuilder b(n, n);
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j)
                if (d[i * (std::size_t)n + j] != 0.0) b.add(i, j, d[i * (std::size_t)n + j]);
        *out = new MatrixHandle{b.finalize()};
    });
}

int ref_matrix_new(int n_rows, int n_cols, const int* rp, const int* ci, const double* v,
                   void** out) {
    return guarded([&] { *out = new MatrixHandle{from_csr(n_rows, n_cols, rp, ci, v)}; });
}

void ref_matrix_sizes(void* m, int* n_rows, int* n_cols, long long* nnz) {
    auto* h = static_cast<MatrixHandle*>(m);
    *n_rows = h->a.n_rows;
    *n_cols = h->a.n_cols;
    *nnz = h->a.nnz();
}

void ref_matrix_copy(void* m, int* rp, int* ci, double* v) {
    copy_csr(static_cast<MatrixHandle*>(m)->a, rp, ci, v);
}

void ref_matrix_free(void* m) { delete static_cast<MatrixHandle*>(m); }

int ref_ground_dof(void* m, int dof, void** out) {
    return guarded([&] {
        *out = new MatrixHandle{ground_dof(static_cast<MatrixHandle*>(m)->a, dof)};
    });
}

// ---------------------------------------------------------------------------
// AMG hierarchy (precond.cpp:189-259)

int ref_amg_setup(void* m, int max_levels, double theta, int coarse_threshold,
                  const int* components, void** out) {
    return guarded([&] {
        const auto& a = static_cast<MatrixHandle*>(m)->a;
        AmgOptions o;
        o.max_levels = max_levels;
        o.strength_theta = theta;
        o.coarse_threshold = coarse_threshold;
        if (components) o.components.assign(components, components + a.n_rows);
        *out = new HierHandle{amg_setup(a, o)};
    });
}

int ref_hier_num_levels(void* h) { return (int)static_cast<HierHandle*>(h)->h.levels.size(); }

void ref_hier_level_sizes(void* h, int lev, int* n, long long* nnz, int* n_coarse) {
    const auto& L = static_cast<HierHandle*>(h)->h.levels[lev];
    *n = L.a.n_rows;
    *nnz = L.a.nnz();
    *n_coarse = L.n_coarse;
}

void ref_hier_level_copy(void* h, int lev, int* rp, int* ci, double* v, int* agg) {
    const auto& L = static_cast<HierHandle*>(h)->h.levels[lev];
    copy_csr(L.a, rp, ci, v);
    if (agg && !L.aggregate_of.empty())
        std::memcpy(agg, L.aggregate_of.data(), sizeof(int) * L.aggregate_of.size());
}

void ref_hier_coarse_lu_sizes(void* h, int* n, long long* nnz_l, long long* nnz_u) {
    const auto& f = static_cast<HierHandle*>(h)->h.coarse_lu;
    *n = f.rows();
    *nnz_l = f.lower.nnz();
    *nnz_u = f.upper.nnz();
}

void ref_hier_coarse_lu_copy(void* h, int* l_rp, int* l_ci, double* l_v, int* u_rp, int* u_ci,
                             double* u_v, int* perm) {
    const auto& f = static_cast<HierHandle*>(h)->h.coarse_lu;
    copy_csr(f.lower, l_rp, l_ci, l_v);
    copy_csr(f.upper, u_rp, u_ci, u_v);
    if (perm) std::memcpy(perm, f.row_permutation.data(), sizeof(int) * f.row_permutation.size());
}

int ref_hier_vcycle(void* h, const double* r, double* z) {
    return guarded([&] {
        const auto& hh = static_cast<HierHandle*>(h)->h;
        auto out = amg_vcycle_apply(hh, std::span<const double>(r, hh.finest_rows()));
        std::memcpy(z, out.data(), sizeof(double) * out.size());
    });
}

void ref_hier_free(void* h) { delete static_cast<HierHandle*>(h); }

int ref_lu_solve_dense_check(void* m, const double* b, double* x) {
    // factor + solve of an arbitrary matrix with the reference sparse LU (lu.cpp)
    return guarded([&] {
        const auto& a = static_cast<MatrixHandle*>(m)->a;
        auto f = lu_factor(a);
        auto y = lu_solve(f, std::span<const double>(b, a.n_rows));
        std::memcpy(x, y.data(), sizeof(double) * y.size());
    });
}

// ---------------------------------------------------------------------------
// td_* block preconditioner wired as MonolithicDriver::build_preconditioner
// (bench.cpp:121-182): D' = ground_dof(A[pm,pm]); V labels u=0 / v=1;
// UzawaConfig{inexact, amg = v_amg}; BlockPreconditioner(kind, A, ...).
// kind: 0 = td_bj, 1 = td_bgs, 2 = td_bj with ILU(0) on D', 3 = td_bgs with ILU(0).

int ref_td_new(int n, const int* rp, const int* ci, const double* v, int n_u, int n_vel,
               int n_pff, int n_ppm, int kind, int v_max_levels, int d_max_levels, void** out) {
    return guarded([&] {
        auto t0 = std::chrono::steady_clock::now();
        auto* h = new TdHandle;
        h->a = from_csr(n, n, rp, ci, v);
        const int n_ff = n_vel + n_pff;
        if (n_ff + n_ppm != n) throw std::invalid_argument("ref_td_new: partition mismatch");
        auto d_block = ground_dof(submatrix(h->a, n_ff, n, n_ff, n));
        std::vector<int> comps(n_vel, 0);
        for (int k = n_u; k < n_vel; ++k) comps[k] = 1;
        AmgOptions v_amg;
        v_amg.components = comps;
        v_amg.max_levels = v_max_levels;
        AmgOptions d_amg;
        d_amg.max_levels = d_max_levels;
        auto v_block = submatrix(h->a, 0, n_vel, 0, n_vel);
        auto b_block = submatrix(h->a, 0, n_vel, n_vel, n_ff);
        auto c_block = submatrix(h->a, n_vel, n_ff, 0, n_vel);
        UzawaConfig ucfg;
        ucfg.amg = v_amg;
        h->uz = std::make_shared<UzawaPreconditioner>(v_block, b_block, c_block, ucfg);
        // kind 2 / 3: td_bj / td_bgs with ILU(0) on D' (bench.cpp:156-172, td_*_uzawa_ilu0)
        if (kind >= 2)
            h->pm = std::make_shared<Ilu0Preconditioner>(d_block);
        else
            h->pm = std::make_shared<AmgPreconditioner>(d_block, d_amg);
        h->block = std::make_shared<BlockPreconditioner>(
            kind % 2 == 0 ? BlockPrecondKind::td_bj : BlockPrecondKind::td_bgs, h->a, n_vel, n_pff,
            n_ppm, h->uz, h->pm);
        h->setup_seconds =
            std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        // deterministic: identical to the hierarchies inside uz / pm
        h->v_h.h = amg_setup(v_block, v_amg);
        h->d_h.h = amg_setup(d_block, d_amg);
        *out = h;
    });
}

double ref_td_omega(void* p) { return static_cast<TdHandle*>(p)->uz->omega(); }
double ref_td_setup_seconds(void* p) { return static_cast<TdHandle*>(p)->setup_seconds; }

// Borrowed views of the two hierarchies (do not free).
void* ref_td_v_hier(void* p) {
    auto* h = static_cast<TdHandle*>(p);
    return reinterpret_cast<void*>(&h->v_h);
}
void* ref_td_d_hier(void* p) {
    auto* h = static_cast<TdHandle*>(p);
    return reinterpret_cast<void*>(&h->d_h);
}

int ref_td_apply(void* p, const double* r, double* z) {
    return guarded([&] {
        auto* h = static_cast<TdHandle*>(p);
        const int n = h->block->rows();
        h->block->apply(std::span<const double>(r, n), std::span<double>(z, n));
    });
}

int ref_uzawa_apply(void* p, const double* r, double* z) {
    return guarded([&] {
        auto* h = static_cast<TdHandle*>(p);
        const int n = h->uz->rows();
        h->uz->apply(std::span<const double>(r, n), std::span<double>(z, n));
    });
}

void ref_td_free(void* p) { delete static_cast<TdHandle*>(p); }

// ---------------------------------------------------------------------------
// Krylov solvers (krylov.cpp). precond_kind: 0 none, 1 td handle, 2 hierarchy
// (AMG V-cycle as the preconditioner).

namespace {

struct HierPrecond final : public Preconditioner {
    const AMGHierarchy* h;
    explicit HierPrecond(const AMGHierarchy* hh) : h(hh) {}
    int rows() const override { return h->finest_rows(); }
    void do_apply(std::span<const double> r, std::span<double> z) const override {
        auto x = amg_vcycle_apply(*h, r);
        std::copy(x.begin(), x.end(), z.begin());
    }
};

void fill_report(const SolveReport& rep, int* iters, double* final_res, int* converged,
                 double* wall, double* hist, int hist_cap, int* hist_len) {
    *iters = rep.iterations;
    *final_res = rep.final_residual;
    *converged = rep.converged ? 1 : 0;
    *wall = rep.wall_time;
    *hist_len = (int)rep.residual_history.size();
    if (hist)
        for (int i = 0; i < hist_cap && i < (int)rep.residual_history.size(); ++i)
            hist[i] = rep.residual_history[i];
}

}  // namespace

int ref_pd_gmres(void* mat, int precond_kind, void* precond, const double* b, double tol_abs,
                 int max_restarts, int m_init, int m_min, int m_step, int m_max, double* x,
                 int* iters, double* final_res, int* converged, double* wall, double* hist,
                 int hist_cap, int* hist_len) {
    return guarded([&] {
        const auto& a = static_cast<MatrixHandle*>(mat)->a;
        RestartController c;
        c.m_init = c.current_m = m_init;
        c.m_min = m_min;
        c.m_step = m_step;
        c.m_max = m_max;
        std::unique_ptr<HierPrecond> hp;
        const Preconditioner* p = nullptr;
        if (precond_kind == 1) p = static_cast<TdHandle*>(precond)->block.get();
        if (precond_kind == 2) {
            hp = std::make_unique<HierPrecond>(&static_cast<HierHandle*>(precond)->h);
            p = hp.get();
        }
        if (precond_kind == 3) p = static_cast<PrecondHandle*>(precond)->p.get();
        auto res = pd_gmres(LinearOperator::from_matrix(a), p,
                            std::span<const double>(b, a.n_rows), tol_abs, max_restarts, c);
        std::memcpy(x, res.x.data(), sizeof(double) * res.x.size());
        fill_report(res.report, iters, final_res, converged, wall, hist, hist_cap, hist_len);
    });
}

int ref_bicgstab(void* mat, int precond_kind, void* precond, const double* b, double tol_abs,
                 int max_iters, double* x, int* iters, double* final_res, int* converged,
                 double* wall, double* hist, int hist_cap, int* hist_len) {
    return guarded([&] {
        const auto& a = static_cast<MatrixHandle*>(mat)->a;
        std::unique_ptr<HierPrecond> hp;
        const Preconditioner* p = nullptr;
        if (precond_kind == 1) p = static_cast<TdHandle*>(precond)->block.get();
        if (precond_kind == 2) {
            hp = std::make_unique<HierPrecond>(&static_cast<HierHandle*>(precond)->h);
            p = hp.get();
        }
        if (precond_kind == 3) p = static_cast<PrecondHandle*>(precond)->p.get();
        auto res = bicgstab(LinearOperator::from_matrix(a), p,
                            std::span<const double>(b, a.n_rows), tol_abs, max_iters);
        std::memcpy(x, res.x.data(), sizeof(double) * res.x.size());
        fill_report(res.report, iters, final_res, converged, wall, hist, hist_cap, hist_len);
    });
}

int ref_power_iteration(void* mat, double tol_rel, int max_iters, unsigned seed, double* value,
                        int* iterations, int* converged) {
    return guarded([&] {
        const auto& a = static_cast<MatrixHandle*>(mat)->a;
        auto r = power_iteration(LinearOperator::from_matrix(a), tol_rel, max_iters, seed);
        *value = r.value;
        *iterations = r.iterations;
        *converged = r.converged ? 1 : 0;
    });
}

}  // extern "C"
