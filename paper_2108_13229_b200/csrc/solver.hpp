// Device-resident objects behind the C-ABI handles: matrices (the
// LinearOperator of operator.hpp:18-28), preconditioners (the Preconditioner
// contract of operator.hpp:34-62) and the Krylov drivers (krylov.cpp).
#pragma once

#include <atomic>
#include <cmath>
#include <memory>
#include <vector>

#include "coarse.hpp"
#include "common.hpp"
#include "gs.cuh"
#include "kernels.cuh"
#include "setup.hpp"

namespace sdg {

// device right-hand side of the monolithic system (assemble.cu), bitwise setup.cpp's
void launch_assemble_rhs(Context& c, const sdg_scenario& sc, const double* v_prev, double* rhs);
int64_t assemble_matrix_device(Context& c, const sdg_scenario& sc, const double* k_cell_dev, int* rowptr_dev,
                               int* col_dev, double* val_dev, int64_t capacity);

struct BiWork;     // krylov.cu: cached BiCGSTAB workspace + captured iteration graph
struct GmresWork;  // krylov.cu: cached GMRES basis / workspace + captured Arnoldi-step graphs

// A device CSR plus its host copy (setup extracts blocks from it) and, on
// demand, the Gauss-Seidel level schedule.
struct Matrix {
    CtxPtr ctx;
    HostCsr host;
    DevCsr dev;
    // lazily built for sdg_sor_sweep
    bool sched_ready = false;
    DevBuf<int> lvl_ptr, lvl_rows;
    int n_levels = 0;

    std::shared_ptr<BiWork> bi_work;
    std::shared_ptr<GmresWork> gm_work;

    Matrix(CtxPtr c, HostCsr h);
    void ensure_schedule();
};
using MatrixPtr = std::shared_ptr<Matrix>;

class Precond {
public:
    explicit Precond(CtxPtr c) : ctx_(std::move(c)) {}
    virtual ~Precond() = default;
    virtual int rows() const = 0;
    // Preconditioner::apply (operator.hpp:40-43): counts, then applies on
    // the context stream; r and z are distinct device vectors.
    void apply(const double* r, double* z) {
        applications_.fetch_add(1, std::memory_order_relaxed);
        do_apply(r, z);
    }
    int64_t applications() const { return applications_.load(std::memory_order_relaxed); }
    // a captured graph that contains k applies was replayed
    void add_applications(int64_t k) { applications_.fetch_add(k, std::memory_order_relaxed); }
    // setup-time applies (BlockPrecond interface split) that are not counted
    void apply_uncounted(const double* r, double* z) { do_apply(r, z); }
    virtual int64_t setup_memory_doubles() const { return 0; }
    virtual int64_t work_per_apply() const { return 0; }
    virtual double omega() const { return std::nan(""); }
    double setup_seconds = 0.0;
    Context& ctx() const { return *ctx_; }
    CtxPtr ctx_ptr() const { return ctx_; }

protected:
    virtual void do_apply(const double* r, double* z) = 0;
    CtxPtr ctx_;

private:
    std::atomic<int64_t> applications_{0};
};
using PrecondPtr = std::shared_ptr<Precond>;

class IdentityPrecond final : public Precond {
public:
    IdentityPrecond(CtxPtr c, int n) : Precond(std::move(c)), n_(n) {}
    int rows() const override { return n_; }

protected:
    void do_apply(const double* r, double* z) override;

private:
    int n_;
};

// ILU(0) (precond.hpp:18-30, precond.cpp:13-87): factors from the host
// restatement (setup.cpp ilu0_factor, bitwise the reference's); each apply is
// the unit-lower forward solve and the upper backward solve as two sweeps of
// the Gauss-Seidel lower-solve machinery: L + I as it is, U with its rows and
// columns reversed (its strict upper part becomes a lower triangle, 1/u_ii the
// scaling), so the structured 5-point D' runs both on the multi-SM wavefront.
class Ilu0Precond final : public Precond {
public:
    Ilu0Precond(CtxPtr c, const HostCsr& a);
    int rows() const override { return n_; }
    int64_t setup_memory_doubles() const override { return nnz_; }
    int64_t work_per_apply() const override { return 2 * nnz_; }

protected:
    void do_apply(const double* r, double* z) override;

private:
    int n_ = 0;
    int64_t nnz_ = 0;
    GsPlan lower_, upper_rev_;
    DevBuf<double> y_, t_;
};

// Aggregation AMG, V(1,1) (precond.hpp:101-120, precond.cpp:233-259).
class AmgPrecond final : public Precond {
public:
    AmgPrecond(CtxPtr c, const HostCsr& a, const AmgOpts& o);
    int rows() const override { return n_rows_; }
    int64_t setup_memory_doubles() const override;
    int64_t work_per_apply() const override;
    int num_levels() const { return static_cast<int>(levels_.size()); }
    int level_rows(int l) const { return levels_[l].a.n_rows; }
    int64_t level_nnz(int l) const { return levels_[l].a.nnz; }
    // the finest level's post-smoother: its plan (null unless it is a walk
    // that can record a mark) and the event recorded once its packed b values
    // are final (BlockPrecond's early interface correction)
    const GsPlan* markable_post_plan() const {
        return !levels_.empty() && levels_[0].fast && num_levels() > 1 && levels_[0].gs.can_mark() ? &levels_[0].gs
                                                                                                    : nullptr;
    }
    cudaEvent_t post_mark = nullptr;
    // the finest level's smoother runs the multi-SM wavefront (gs_wave.cu)
    bool finest_wave() const { return !levels_.empty() && levels_[0].fast && num_levels() > 1 && levels_[0].gs.wave; }
    // some coarse level's smoother runs the multi-SM lattice (gs_lattice.cu), itself or in a label block
    bool coarse_lattice() const {
        for (size_t l = 1; l + 1 < levels_.size(); ++l) {
            const GsPlan& g = levels_[l].gs;
            if (!levels_[l].fast) continue;
            if (g.lattice) return true;
            for (const auto& p : g.parts)
                if (p->lattice) return true;
        }
        return false;
    }

protected:
    void do_apply(const double* r, double* z) override;

private:
    struct Level {
        DevCsr a;
        DevBuf<int> lvl_ptr, lvl_rows;
        int n_sched = 0;
        DevBuf<int> agg;
        DevBuf<int> pt_ptr, pt_rows;
        int n_coarse = 0;
        DevBuf<double> zt;      // z + P zc before post-smoothing (bitwise path)
        DevBuf<double> r, z;    // this level's rhs / solution (levels >= 1)
        GsPlan gs;              // fast smoother plan
        bool fast = false;
    };
    void vcycle(int lev, const double* r, double* z);
    void factor_coarse(const HostCsr& coarse);

    int n_rows_ = 0;
    bool exact_ = false;  // SDG_GS_EXACT=1: bitwise smoother path throughout
    std::vector<Level> levels_;
    int n_c_ = 0;
    CoarseSolver coarse_;  // direct solve of the coarsest matrix (coarse.hpp)
};

// Inexact Uzawa sweep (precond.cpp:264-299).
class UzawaPrecond final : public Precond {
public:
    UzawaPrecond(CtxPtr c, const HostCsr& v, const HostCsr& b, const HostCsr& cm,
                 const AmgOpts& amg, double power_tol, int power_max, unsigned seed,
                 double omega_override);
    int rows() const override { return n_v_ + n_p_; }
    double omega() const override { return omega_; }
    int64_t setup_memory_doubles() const override {
        return inner_->setup_memory_doubles() + b_.nnz + c_.nnz;
    }
    int64_t work_per_apply() const override { return inner_->work_per_apply() + c_.nnz + n_p_; }
    const AmgPrecond& inner() const { return *inner_; }
    AmgPrecond& inner_mut() { return *inner_; }

protected:
    void do_apply(const double* r, double* z) override;

private:
    int n_v_, n_p_;
    DevCsr b_, c_;
    std::shared_ptr<AmgPrecond> inner_;
    double omega_ = 1.0;
};

// td_* / pv_* block combinators (precond.cpp:304-363).
class BlockPrecond final : public Precond {
public:
    BlockPrecond(CtxPtr c, int kind, const HostCsr& matrix, int n_v, int n_pff, int n_ppm,
                 PrecondPtr first, PrecondPtr pm);
    int rows() const override { return n_v_ + n_pff_ + n_ppm_; }
    double omega() const override { return first_->omega(); }
    int64_t setup_memory_doubles() const override;
    int64_t work_per_apply() const override;
    const PrecondPtr& first() const { return first_; }
    const PrecondPtr& pm() const { return pm_; }
    bool interface_split() const { return n_gamma_ > 0; }
    bool early_correction() const { return early_ev_ != nullptr; }

protected:
    void do_apply(const double* r, double* z) override;

private:
    int kind_;
    int n_v_, n_pff_, n_ppm_;
    PrecondPtr first_, pm_;
    DevCsr c_prime_, c_, c1_prime_;
    DevBuf<double> tmp_;
    // td_bgs interface split (setup_interface_split)
    void setup_interface_split(const HostCsr& cp);
    int n_gamma_ = 0;
    DevCsr c_gamma_;               // the interface rows of C'
    DevBuf<double> w_gamma_;       // (C' z_ff) on those rows
    DevBuf<double> k_gamma_;       // P_D' e_g for every interface row g, column-major
    // early correction: w and z_pm -= K w on the side stream as soon as the
    // Uzawa V-cycle's finest post-smoother has its packed b (setup_early_w)
    void setup_early_w(const HostCsr& matrix);
    void tune_early();  // early or late, timed at setup
    cudaEvent_t early_ev_ = nullptr;
    const GsPlan* early_plan_ = nullptr;

public:
    ~BlockPrecond() override;
};

// Krylov drivers on device vectors; host control flow mirrors krylov.cpp.
struct SolveOut {
    int iterations = 0;
    bool converged = false;
    double final_residual = 0.0;
    std::vector<double> history;
    double device_ms = 0.0;
    bool breakdown = false;  // repeated BiCGSTAB breakdown, reported instead of thrown
};

struct Restart {
    int m_init = 3, m_min = 3, m_step = 5, m_max = 53, current_m = 3;
    double previous_rate = 0.0;
    bool has_rate_sample = false;
    double alpha_p = -3.0, alpha_d = 5.0, stall_threshold = 0.05;
    void update(double rate);  // krylov.cpp:37-45
};

SolveOut pd_gmres(Matrix& a, Precond* p, const double* b_dev, double* x_dev, double tol_abs,
                  int max_restarts, Restart ctrl);
// throw_on_breakdown = false: a repeated breakdown ends the solve with
// out.breakdown set and x holding the last iterate (warm-started drivers).
SolveOut bicgstab(Matrix& a, Precond* p, const double* b_dev, double* x_dev, double tol_abs,
                  int max_iters, bool throw_on_breakdown = true);

// Row-major explicit inverse of a (small, coarsest-level) matrix: dense LU on
// the device (cuSOLVER getrf) + getrs against I.  Throws SDG_ESINGULAR.

struct PowerOut {
    double value = 0.0;
    bool converged = false;
    int iterations = 0;
};
// power_iteration (krylov.cpp:307-339) on a device operator y = op(x).
template <class Op>
PowerOut power_iteration(Context& c, int n, Op&& op, double tol_rel, int max_iters, unsigned seed);

}  // namespace sdg
