// Device preconditioners: AMG V(1,1), inexact Uzawa, td_*/pv_* block
// combinators.  Setup (aggregation, Galerkin, schedules) is host C++
// (setup.cpp); the coarse factorization is the nested-dissection block
// elimination of coarse.hpp (explicit inverses of small dense blocks computed
// on the device), so each coarse solve is a few fully parallel batched
// products instead of two sequential triangular solves (SURVEY.md §7 hard
// part 2: at the reference's 3 levels the coarse factor is ~58% dense).
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <string>

#include "launch.cuh"
#include "power.cuh"
#include "solver.hpp"

namespace sdg {

// ---------------------------------------------------------------------------
// context / matrix

Context::Context(int dev) : device(dev) {
    SDG_CUDA(cudaSetDevice(dev));
    SDG_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
    SDG_CUDA(cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev));
    pinned = std::make_unique<PinnedBuf>(64 * 1024);
    for (auto& e : step_ev) SDG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    if (const char* e = std::getenv("SDG_PDL")) pdl = e[0] != '0';
}

Context::~Context() {
    for (auto& r : prof) {
        cudaEventDestroy(r.a);
        cudaEventDestroy(r.b);
    }
    for (auto e : event_pool) cudaEventDestroy(e);
    for (auto e : step_ev)
        if (e) cudaEventDestroy(e);
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
    if (side) cudaStreamDestroy(side);
    if (stream) cudaStreamDestroy(stream);
}

void Context::side_begin() {
    if (!side) {
        int lo = 0, hi = 0;
        SDG_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        SDG_CUDA(cudaStreamCreateWithPriority(&side, cudaStreamNonBlocking, hi));
        SDG_CUDA(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
        SDG_CUDA(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming));
    }
    if (main_stream) fail(SDG_EINVAL, "side_begin: already on the side stream");
    SDG_CUDA(cudaEventRecord(ev_fork, stream));
    SDG_CUDA(cudaStreamWaitEvent(side, ev_fork, 0));
    main_stream = stream;
    stream = side;
}

void Context::side_continue(cudaEvent_t after) {
    if (!side) fail(SDG_EINVAL, "side_continue: no side stream yet");
    if (main_stream) fail(SDG_EINVAL, "side_continue: already on the side stream");
    SDG_CUDA(cudaStreamWaitEvent(side, after, 0));
    main_stream = stream;
    stream = side;
}

void Context::side_end() {
    if (!main_stream) fail(SDG_EINVAL, "side_end: not on the side stream");
    SDG_CUDA(cudaEventRecord(ev_join, side));
    stream = main_stream;
    main_stream = nullptr;
}

void Context::side_join() { SDG_CUDA(cudaStreamWaitEvent(stream, ev_join, 0)); }

cudaEvent_t Context::take_event() {
    if (!event_pool.empty()) {
        cudaEvent_t e = event_pool.back();
        event_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    SDG_CUDA(cudaEventCreate(&e));
    return e;
}

void Context::drain_profile() {
    if (prof.empty()) return;
    SDG_CUDA(cudaStreamSynchronize(stream));
    for (auto& r : prof) {
        float ms = 0.f;
        SDG_CUDA(cudaEventElapsedTime(&ms, r.a, r.b));
        prof_ms[r.family] += ms;
        prof_launches[r.family] += 1;
        prof_bytes[r.family] += r.bytes;
        event_pool.push_back(r.a);
        event_pool.push_back(r.b);
    }
    prof.clear();
}

Matrix::Matrix(CtxPtr c, HostCsr h) : ctx(std::move(c)), host(std::move(h)) {
    host.check();
    dev.upload(host, ctx->stream);
    // the operator SpMV of the Krylov drivers streams A once per apply: give
    // it the coalesced SELL-32 copy (SDG_SELL=0 keeps the CSR kernel)
    const char* e = std::getenv("SDG_SELL");
    if (!(e && e[0] == '0') && host.n_rows >= 4096) dev.build_sell(host, ctx->stream);
}

void Matrix::ensure_schedule() {
    if (sched_ready) return;
    if (host.n_rows != host.n_cols) fail(SDG_EDIM, "sor_sweep: matrix must be square");
    require_diagonal(host, "sor_sweep");
    LevelSchedule s = lower_schedule(host);
    lvl_ptr.upload(s.lvl_ptr, ctx->stream);
    lvl_rows.upload(s.lvl_rows, ctx->stream);
    n_levels = s.n_levels();
    sched_ready = true;
}

void IdentityPrecond::do_apply(const double* r, double* z) { launch_copy(*ctx_, z, r, n_); }

// ---------------------------------------------------------------------------
// ILU(0)

namespace {
__global__ void k_reverse(int n, const double* __restrict__ x, double* __restrict__ y) {
    pdl_begin();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) y[i] = x[n - 1 - i];
}
void launch_reverse(Context& c, int n, const double* x, double* y) {
    ProfScope ps_(c, PF_VEC, 16.0 * n);
    if (n == 0) return;
    launch_k(c, k_reverse, (n + 255) / 256, 256, 0, n, x, y);
    c.count();
}
}  // namespace

Ilu0Precond::Ilu0Precond(CtxPtr c, const HostCsr& a) : Precond(std::move(c)), n_(a.n_rows) {
    auto t0 = std::chrono::steady_clock::now();
    Context& cx = *ctx_;
    HostCsr lo, up;
    ilu0_factor(a, lo, up);
    nnz_ = lo.nnz() + up.nnz();
    const int n = n_;
    // L + I (unit diagonal: the lower solve's 1/d is 1)
    HostCsr ml(n, n);
    for (int i = 0; i < n; ++i) {
        for (int k = lo.rp[i]; k < lo.rp[i + 1]; ++k) {
            ml.ci.push_back(lo.ci[k]);
            ml.v.push_back(lo.v[k]);
        }
        ml.ci.push_back(i);
        ml.v.push_back(1.0);
        ml.rp[i + 1] = static_cast<int>(ml.ci.size());
    }
    // U reversed: row i' = n-1-i holds U's row i with columns n-1-j, sorted ascending
    HostCsr mu(n, n);
    for (int ip = 0; ip < n; ++ip) {
        const int i = n - 1 - ip;
        for (int k = up.rp[i + 1] - 1; k >= up.rp[i]; --k) {  // descending j = ascending n-1-j
            mu.ci.push_back(n - 1 - up.ci[k]);
            mu.v.push_back(up.v[k]);
        }
        mu.rp[ip + 1] = static_cast<int>(mu.ci.size());
    }
    lower_.build(ml, {}, cx.stream, 0, false);
    upper_rev_.build(mu, {}, cx.stream, 0, false);
    y_.resize(std::max(n, 1));
    t_.resize(std::max(n, 1));
    cx.sync();
    setup_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// precond.cpp:73-87: y = L^{-1} r (unit lower), z = U^{-1} y, the backward
// solve as a forward one on the reversed U
void Ilu0Precond::do_apply(const double* r, double* z) {
    Context& cx = *ctx_;
    launch_gs_prep_pre(cx, lower_, r);
    launch_gs_lower(cx, lower_, y_.get());
    launch_reverse(cx, n_, y_.get(), t_.get());
    launch_gs_prep_pre(cx, upper_rev_, t_.get());
    launch_gs_lower(cx, upper_rev_, y_.get());
    launch_reverse(cx, n_, y_.get(), z);
}

// ---------------------------------------------------------------------------
// AMG

AmgPrecond::AmgPrecond(CtxPtr c, const HostCsr& a, const AmgOpts& o) : Precond(std::move(c)) {
    auto t0 = std::chrono::steady_clock::now();
    Context& cx = *ctx_;
    // aggregation on the host (a sequential greedy pass), Galerkin products on the device
    const char* ge = std::getenv("SDG_GALERKIN");
    const bool host_product = ge && ge[0] == 'h';
    std::vector<HostLevel> hl = build_hierarchy(
        a, o,
        host_product ? GalerkinFn{}
                     : GalerkinFn{[&cx](const HostCsr& m, const std::vector<int>& agg, int nc) {
                           return galerkin_device(cx, m, agg, nc);
                       }});
    n_rows_ = a.n_rows;
    const char* ex = std::getenv("SDG_GS_EXACT");
    exact_ = ex && ex[0] == '1';
    levels_.resize(hl.size());
    for (size_t l = 0; l < hl.size(); ++l) {
        Level& L = levels_[l];
        const HostCsr& A = hl[l].a;
        L.a.upload(A, cx.stream);
        if (l > 0) {
            L.r.resize(A.n_rows);
            L.z.resize(A.n_rows);
        }
        if (l + 1 < hl.size()) {
            require_diagonal(A, "sor_sweep");
            LevelSchedule s = lower_schedule(A);
            L.lvl_ptr.upload(s.lvl_ptr, cx.stream);
            L.lvl_rows.upload(s.lvl_rows, cx.stream);
            L.n_sched = s.n_levels();
            L.agg.upload(hl[l].aggregate_of, cx.stream);
            std::vector<int> ptr, rows;
            aggregate_transpose(hl[l].aggregate_of, hl[l].n_coarse, ptr, rows);
            L.pt_ptr.upload(ptr, cx.stream);
            L.pt_rows.upload(rows, cx.stream);
            L.n_coarse = hl[l].n_coarse;
            L.zt.resize(A.n_rows);
            if (!exact_) {
                L.gs.tune = &cx;
                L.gs.build(A, hl[l].components, cx.stream, 0, /*allow_merge=*/true);
                L.fast = L.gs.usable;
            }
        }
    }
    factor_coarse(hl.back().a);
    cx.sync();
    setup_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

void AmgPrecond::factor_coarse(const HostCsr& coarse) {
    n_c_ = coarse.n_rows;
    coarse_.build(*ctx_, coarse);
}

int64_t AmgPrecond::setup_memory_doubles() const {
    int64_t s = coarse_.doubles() + coarse_.sparse_entries();
    for (const auto& l : levels_) s += l.a.nnz;
    return s;
}

int64_t AmgPrecond::work_per_apply() const {
    int64_t s = coarse_.doubles() + coarse_.sparse_entries();
    for (const auto& l : levels_) s += 5 * l.a.nnz;
    return s;
}

void AmgPrecond::vcycle(int lev, const double* r, double* z) {
    Context& cx = *ctx_;
    if (lev + 1 == num_levels()) {
        coarse_.solve(cx, r, z);
        return;
    }
    Level& L = levels_[lev];
    Level& C = levels_[lev + 1];
    // the next level's pre-smoother input is seeded by the restriction
    const GsPlan* seed = (lev + 2 < num_levels() && C.fast && !C.gs.merged) ? &C.gs : nullptr;
    if (L.fast) {
        if (lev == 0 || L.gs.merged) launch_gs_prep_pre(cx, L.gs, r);  // else seeded by the restriction
        launch_gs_lower(cx, L.gs, z);
        launch_restrict_warp(cx, L.a, L.pt_ptr.get(), L.pt_rows.get(), L.n_coarse, r, z, C.r.get(), seed);
        vcycle(lev + 1, C.r.get(), C.z.get());
        launch_gs_prep_post(cx, L.gs, r, z, C.z.get(), L.agg.get());  // fused prolongation
        launch_gs_lower(cx, L.gs, z, lev == 0 ? post_mark : nullptr);
        return;
    }
    launch_gs_levels(cx, L.a, L.lvl_ptr.get(), L.lvl_rows.get(), L.n_sched, r, nullptr, z, 1.0);
    launch_restrict_warp(cx, L.a, L.pt_ptr.get(), L.pt_rows.get(), L.n_coarse, r, z, C.r.get(), seed);
    vcycle(lev + 1, C.r.get(), C.z.get());
    launch_prolong(cx, L.a.n_rows, L.agg.get(), z, C.z.get(), L.zt.get());
    launch_gs_levels(cx, L.a, L.lvl_ptr.get(), L.lvl_rows.get(), L.n_sched, r, L.zt.get(), z, 1.0);
}

void AmgPrecond::do_apply(const double* r, double* z) { vcycle(0, r, z); }

// ---------------------------------------------------------------------------
// Uzawa

UzawaPrecond::UzawaPrecond(CtxPtr c, const HostCsr& v, const HostCsr& b, const HostCsr& cm,
                           const AmgOpts& amg, double power_tol, int power_max, unsigned seed,
                           double omega_override)
    : Precond(std::move(c)), n_v_(v.n_rows), n_p_(cm.n_rows) {
    auto t0 = std::chrono::steady_clock::now();
    if (v.n_rows != v.n_cols || b.n_rows != n_v_ || cm.n_cols != n_v_ || b.n_cols != cm.n_rows)
        fail(SDG_EDIM, "uzawa: inconsistent block dimensions");
    Context& cx = *ctx_;
    inner_ = std::make_shared<AmgPrecond>(ctx_, v, amg);
    b_.upload(b, cx.stream);
    c_.upload(cm, cx.stream);
    if (!std::isnan(omega_override)) {
        omega_ = omega_override;
    } else {
        // omega = 1 / lambda_max(C Vtilde^{-1} B) (precond.cpp:274-286)
        DevBuf<double> t1(n_v_), t2(n_v_);
        auto schur = [&](const double* x, double* y) {
            launch_spmv(cx, b_, x, t1.get());
            inner_->apply(t1.get(), t2.get());
            launch_spmv(cx, c_, t2.get(), y);
        };
        PowerOut est = power_iteration(cx, n_p_, schur, power_tol, power_max, seed);
        omega_ = (std::abs(est.value) > 1e-300) ? 1.0 / est.value : 1.0;
    }
    cx.sync();
    setup_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

void UzawaPrecond::do_apply(const double* r, double* z) {
    inner_->apply(r, z);
    launch_uzawa_pressure(*ctx_, c_, z, r + n_v_, omega_, z + n_v_);
}

// ---------------------------------------------------------------------------
// block combinators

BlockPrecond::BlockPrecond(CtxPtr c, int kind, const HostCsr& matrix, int n_v, int n_pff,
                           int n_ppm, PrecondPtr first, PrecondPtr pm)
    : Precond(std::move(c)), kind_(kind), n_v_(n_v), n_pff_(n_pff), n_ppm_(n_ppm),
      first_(std::move(first)), pm_(std::move(pm)) {
    const int n = n_v_ + n_pff_ + n_ppm_;
    if (matrix.n_rows != n || matrix.n_cols != n)
        fail(SDG_EDIM, "block preconditioner: partition does not cover the matrix");
    if (kind_ < SDG_TD_BJ || kind_ > SDG_PV_BGS) fail(SDG_EINVAL, "block preconditioner: bad kind");
    const int n_ff = n_v_ + n_pff_;
    const bool td = kind_ == SDG_TD_BJ || kind_ == SDG_TD_BGS;
    const int first_rows = td ? n_ff : n_v_;
    if (first_ && first_->rows() != first_rows)
        fail(SDG_EDIM, "block preconditioner: first sub-block size mismatch");
    if (pm_ && pm_->rows() != n_ppm_)
        fail(SDG_EDIM, "block preconditioner: pm sub-block size mismatch");
    if (!first_ || !pm_) fail(SDG_EDIM, "block preconditioner: missing sub-preconditioner");
    Context& cx = *ctx_;
    if (kind_ == SDG_TD_BGS) {
        const HostCsr cp = submatrix(matrix, n_ff, n, 0, n_ff);
        c_prime_.upload(cp, cx.stream);
        setup_interface_split(cp);
        if (n_gamma_ > 0) setup_early_w(matrix);
    }
    if (kind_ == SDG_PV_BGS) {
        c_.upload(submatrix(matrix, n_v_, n_ff, 0, n_v_), cx.stream);
        c1_prime_.upload(submatrix(matrix, n_ff, n, 0, n_v_), cx.stream);
    }
    tmp_.resize(std::max(n_ppm_, 1));
    cx.sync();
    if (early_ev_) tune_early();
}

// Early or late interface correction?  Both are the same arithmetic (bitwise);
// which is faster depends on what the GEMV's stream of K does to the
// post-smoother it overlaps: at c2 (K = 33 MB, in L2) and c4 (K = 8 GB, the
// GEMV far longer than the smoother) early wins, at c3 (K = 1 GB, GEMV and
// wavefront about equally long) the GEMV's CTAs fill the SMs before the
// wavefront's CTAs find room and late wins (c3 solve 208.6 ms early, 203.4 ms
// late; c4 55.9 s early, 57.8 s late; c2 76.5 ms early, 79.6 ms late).  So, like
// the smoother plans, the choice is timed at setup: twice ten applies each way.
// SDG_TD_EARLY=1 keeps early without timing, =0 never sets it up.
void BlockPrecond::tune_early() {
    const char* e = std::getenv("SDG_TD_EARLY");
    if (e && e[0] == '1') return;
    auto* uz = dynamic_cast<UzawaPrecond*>(first_.get());
    if (!uz) return;
    Context& cx = *ctx_;
    const int n = n_v_ + n_pff_ + n_ppm_;
    DevBuf<double> r(n), z(n);
    launch_fill(cx, r.get(), 1.0, n);
    cudaEvent_t a, b;
    SDG_CUDA(cudaEventCreate(&a));
    SDG_CUDA(cudaEventCreate(&b));
    auto timed = [&] {
        for (int k = 0; k < 3; ++k) do_apply(r.get(), z.get());
        SDG_CUDA(cudaEventRecord(a, cx.stream));
        for (int k = 0; k < 10; ++k) do_apply(r.get(), z.get());
        SDG_CUDA(cudaEventRecord(b, cx.stream));
        SDG_CUDA(cudaEventSynchronize(b));
        float ms = 0.f;
        cudaEventElapsedTime(&ms, a, b);
        return ms / 10.f;
    };
    // early, late, early, late: alternate so that a drift of the clocks or of the
    // caches does not favour one side (the two differ by only 1-4 % of an apply)
    cudaEvent_t ev = early_ev_;
    const GsPlan* plan = early_plan_;
    auto set_early = [&](bool on) {
        early_ev_ = on ? ev : nullptr;
        early_plan_ = on ? plan : nullptr;
        uz->inner_mut().post_mark = on ? ev : nullptr;
    };
    float t_early = 0.f, t_late = 0.f;
    for (int rep = 0; rep < 2; ++rep) {
        set_early(true);
        t_early += 0.5f * timed();
        set_early(false);
        t_late += 0.5f * timed();
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    // early must win by 1 %: in the captured solve it gains a little less than in
    // these eagerly launched applies (c3: 0.5-1.5 % apart here, late 2.5 % faster there)
    const bool keep = t_early < 0.99f * t_late;
    set_early(keep);
    if (!keep) cudaEventDestroy(ev);
    if (std::getenv("SDG_DEBUG"))
        std::fprintf(stderr, "[sdg td_bgs] interface correction: early %.1f us, late %.1f us per apply -> %s\n",
                     1e3 * t_early, 1e3 * t_late, keep ? "early" : "late");
}

// td_bgs: z_pm = P_D'(r_pm - C' z_ff).  P_D' (one AMG V-cycle from zero:
// Gauss-Seidel sweeps, restriction, coarse solve, prolongation) is linear, and
// C' is nonzero only in the interface rows G of the porous block, so
//   z_pm = P_D' r_pm - K w,   K = P_D' restricted to the columns G,  w = (C' z_ff)_G.
// P_D' r_pm does not wait for the free-flow solve: it runs on the side stream
// while the Uzawa V-cycle runs on the main one; after the join one GEMV with
// the precomputed K (|G| applies of P_D' at setup) finishes the block.  Equal
// to precond.cpp:339-345 in exact arithmetic.  Used when K fits kSplitBudget
// bytes and streaming it is modelled at < 70 % of one measured P_D' apply;
// SDG_TD_SPLIT=0 disables, =1 skips the time test.
void BlockPrecond::setup_interface_split(const HostCsr& cp) {
    constexpr double kSplitBudget = 16.0 * 1024 * 1024 * 1024;  // bytes of K at most
    constexpr double kGemvBytesPerSec = 5.0e12;                  // K streamed once per apply
    const char* e = std::getenv("SDG_TD_SPLIT");
    if (e && e[0] == '0') return;
    std::vector<int> rows;
    for (int i = 0; i < cp.n_rows; ++i)
        if (cp.rp[i + 1] > cp.rp[i]) rows.push_back(i);
    const int m = static_cast<int>(rows.size());
    const double kbytes = static_cast<double>(n_ppm_) * m * 8.0;
    if (m == 0 || kbytes > kSplitBudget || m > kColmajorMaxGamma) return;
    Context& cx = *ctx_;
    // worth it only when streaming K costs clearly less than the porous
    // V-cycle it takes off the critical path: time one apply
    {
        DevBuf<double> x(n_ppm_), y(n_ppm_);
        launch_fill(cx, x.get(), 1.0, n_ppm_);
        pm_->apply_uncounted(x.get(), y.get());  // warm-up (plans, caches)
        cudaEvent_t a, b;
        SDG_CUDA(cudaEventCreate(&a));
        SDG_CUDA(cudaEventCreate(&b));
        SDG_CUDA(cudaEventRecord(a, cx.stream));
        pm_->apply_uncounted(x.get(), y.get());
        SDG_CUDA(cudaEventRecord(b, cx.stream));
        SDG_CUDA(cudaEventSynchronize(b));
        float ms = 0.f;
        cudaEventElapsedTime(&ms, a, b);
        cudaEventDestroy(a);
        cudaEventDestroy(b);
        const bool force = e && e[0] == '1';
        if (!force && kbytes / kGemvBytesPerSec > 0.7e-3 * ms) return;
    }
    HostCsr cg(m, cp.n_cols);
    for (int k = 0; k < m; ++k) {
        const int i = rows[k];
        for (int q = cp.rp[i]; q < cp.rp[i + 1]; ++q) {
            cg.ci.push_back(cp.ci[q]);
            cg.v.push_back(cp.v[q]);
        }
        cg.rp[k + 1] = static_cast<int>(cg.ci.size());
    }
    c_gamma_.upload(cg, cx.stream);
    w_gamma_.resize(m);
    k_gamma_.resize(static_cast<size_t>(n_ppm_) * m);
    DevBuf<double> unit(n_ppm_), one(1);
    one.upload(std::vector<double>{1.0}, cx.stream);
    for (int k = 0; k < m; ++k) {  // column k of K = P_D' e_{rows[k]}
        launch_fill(cx, unit.get(), 0.0, n_ppm_);
        SDG_CUDA(cudaMemcpyAsync(unit.get() + rows[k], one.get(), sizeof(double), cudaMemcpyDeviceToDevice,
                                 cx.stream));
        pm_->apply_uncounted(unit.get(), k_gamma_.get() + static_cast<size_t>(k) * n_ppm_);
    }
    cx.sync();
    n_gamma_ = m;
}

// Early interface correction.  w = (C' z_ff)_G reads z_v only in the columns
// of C' (the interface velocities v(i,0), assembly.cpp:142-149, 274-275).
// When those rows have no lower entries in V, the finest post-smoother of the
// Uzawa V-cycle gives them z = b = (r - U z_old)/d, which sits in the walk's
// packed buffer before the walk starts, and nothing after the V-cycle changes
// z_v (precond.cpp:296-298 only writes z_p).  So w and z_pm -= K w run on the
// side stream from the post-smoother's mark on, overlapping its walk, instead
// of after the join.  w is summed in the order of launch_spmv (bitwise equal).
void BlockPrecond::setup_early_w(const HostCsr& matrix) {
    const char* e = std::getenv("SDG_TD_EARLY");
    if (e && e[0] == '0') return;
    auto* uz = dynamic_cast<UzawaPrecond*>(first_.get());
    if (!uz) return;
    AmgPrecond& amg = uz->inner_mut();
    const GsPlan* plan = amg.markable_post_plan();
    if (!plan || amg.post_mark) return;
    // the premise is checked on the matrix the post-smoother's plan was built
    // from (the Uzawa's own V, level 0 of its AMG), not on the block of
    // `matrix`: the two need not be equal for an arbitrary Uzawa handle
    if (plan->n != n_v_ || plan->row_has_lower.size() != static_cast<size_t>(n_v_)) return;
    const HostCsr cp = submatrix(matrix, n_v_ + n_pff_, matrix.n_rows, 0, n_v_ + n_pff_);
    for (int i = 0; i < cp.n_rows; ++i)
        for (int q = cp.rp[i]; q < cp.rp[i + 1]; ++q) {
            const int j = cp.ci[q];
            if (j >= n_v_) return;                 // C' reads a free-flow pressure
            if (plan->row_has_lower[j]) return;    // z_v(j) depends on the lower solve
        }
    SDG_CUDA(cudaEventCreateWithFlags(&early_ev_, cudaEventDisableTiming));
    amg.post_mark = early_ev_;
    early_plan_ = plan;
}

BlockPrecond::~BlockPrecond() {
    if (early_ev_) {
        if (auto* uz = dynamic_cast<UzawaPrecond*>(first_.get()))
            if (uz->inner_mut().post_mark == early_ev_) uz->inner_mut().post_mark = nullptr;
        cudaEventDestroy(early_ev_);
    }
}

int64_t BlockPrecond::setup_memory_doubles() const {
    return first_->setup_memory_doubles() + pm_->setup_memory_doubles() + c_prime_.nnz + c_.nnz +
           c1_prime_.nnz + static_cast<int64_t>(n_ppm_) * n_gamma_;
}

int64_t BlockPrecond::work_per_apply() const {
    return first_->work_per_apply() + pm_->work_per_apply() + c_prime_.nnz + c_.nnz +
           c1_prime_.nnz;
}

void BlockPrecond::do_apply(const double* r, double* z) {
    Context& cx = *ctx_;
    const int n_ff = n_v_ + n_pff_;
    switch (kind_) {
    case SDG_TD_BJ:
        first_->apply(r, z);
        pm_->apply(r + n_ff, z + n_ff);
        break;
    case SDG_TD_BGS:  // precond.cpp:339-345
        if (n_gamma_ > 0) {  // see setup_interface_split
            // fork unless this apply is itself running on the side stream
            // (a td_bgs nested in another one): then the same split, in order
            const bool fork = cx.main_stream == nullptr;
            if (fork) cx.side_begin();
            try {
                pm_->apply(r + n_ff, z + n_ff);
            } catch (...) {
                if (fork) {
                    cx.side_end();
                    cx.side_join();
                }
                throw;
            }
            if (fork) cx.side_end();
            first_->apply(r, z);
            if (fork && early_ev_) {  // see setup_early_w
                cx.side_continue(early_ev_);
                try {
                    launch_spmv_packed(cx, c_gamma_, early_plan_->bidx.get(), early_plan_->packed.get(),
                                       w_gamma_.get());
                    launch_colmajor_gemv_sub(cx, n_ppm_, n_gamma_, k_gamma_.get(), w_gamma_.get(), z + n_ff);
                } catch (...) {
                    cx.side_end();
                    cx.side_join();
                    throw;
                }
                cx.side_end();
                cx.side_join();
                break;
            }
            launch_spmv(cx, c_gamma_, z, w_gamma_.get());
            if (fork) cx.side_join();
            launch_colmajor_gemv_sub(cx, n_ppm_, n_gamma_, k_gamma_.get(), w_gamma_.get(), z + n_ff);
            break;
        }
        first_->apply(r, z);
        launch_spmv_add(cx, c_prime_, z, r + n_ff, tmp_.get(), -1.0);
        pm_->apply(tmp_.get(), z + n_ff);
        break;
    case SDG_PV_BJ:
        first_->apply(r, z);
        launch_copy(cx, z + n_v_, r + n_v_, n_pff_);
        pm_->apply(r + n_ff, z + n_ff);
        break;
    case SDG_PV_BGS:
        first_->apply(r, z);
        launch_spmv_add(cx, c_, z, r + n_v_, z + n_v_, -1.0);
        launch_spmv_add(cx, c1_prime_, z, r + n_ff, tmp_.get(), -1.0);
        pm_->apply(tmp_.get(), z + n_ff);
        break;
    }
}

}  // namespace sdg
