// Internal plumbing of libsdgpu.so: errors, device buffers, the per-handle
// context (device + stream), host/device CSR.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "sdg.h"

namespace sdg {

// Internal exception carrying an SDG_* code; the C-ABI layer converts it to
// a return code + thread-local message.
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(int code, const std::string& msg) { throw Error(code, msg); }

#define SDG_CUDA(call)                                                                    \
    do {                                                                                  \
        cudaError_t e_ = (call);                                                          \
        if (e_ != cudaSuccess)                                                            \
            ::sdg::fail(e_ == cudaErrorMemoryAllocation ? SDG_ENOMEM : SDG_ECUDA,        \
                        std::string(#call) + ": " + cudaGetErrorString(e_));              \
    } while (0)

// Owning device allocation.
template <class T>
class DevBuf {
public:
    DevBuf() = default;
    explicit DevBuf(std::size_t n) { resize(n); }
    ~DevBuf() { release(); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p_(o.p_), n_(o.n_) { o.p_ = nullptr; o.n_ = 0; }
    DevBuf& operator=(DevBuf&& o) noexcept {
        if (this != &o) {
            release();
            p_ = o.p_;
            n_ = o.n_;
            o.p_ = nullptr;
            o.n_ = 0;
        }
        return *this;
    }
    void resize(std::size_t n) {
        release();
        if (n) SDG_CUDA(cudaMalloc(&p_, n * sizeof(T)));
        n_ = n;
    }
    void release() {
        if (p_) cudaFree(p_);
        p_ = nullptr;
        n_ = 0;
    }
    T* get() const { return p_; }
    std::size_t size() const { return n_; }
    void upload(const T* h, std::size_t n, cudaStream_t s) {
        if (n) SDG_CUDA(cudaMemcpyAsync(p_, h, n * sizeof(T), cudaMemcpyHostToDevice, s));
    }
    void upload(const std::vector<T>& h, cudaStream_t s) {
        if (h.size() != n_) resize(h.size());
        upload(h.data(), h.size(), s);
    }

private:
    T* p_ = nullptr;
    std::size_t n_ = 0;
};

// Pinned host scratch for small device->host status reads.
class PinnedBuf {
public:
    explicit PinnedBuf(std::size_t bytes) : n_(bytes) { SDG_CUDA(cudaMallocHost(&p_, bytes)); }
    ~PinnedBuf() {
        if (p_) cudaFreeHost(p_);
    }
    PinnedBuf(const PinnedBuf&) = delete;
    PinnedBuf& operator=(const PinnedBuf&) = delete;
    template <class T>
    T* as() const { return static_cast<T*>(p_); }
    std::size_t bytes() const { return n_; }

private:
    void* p_ = nullptr;
    std::size_t n_ = 0;
};

// Kernel families for the live profiler (sdg_context_profile).
enum ProfFamily {
    PF_SPMV = 0,      // operator SpMV over the SELL-32 copy (incl. spmv_add, residual)
    PF_GS,            // Gauss-Seidel sweeps
    PF_RESTRICT,      // fused residual + restriction
    PF_PROLONG,       // prolongation
    PF_COARSE,        // dense coarse solve
    PF_UZAWA,         // Uzawa pressure step
    PF_ORTHO,         // GMRES multi-dot / multi-axpy / lincomb / scale
    PF_BICG,          // fused BiCGSTAB update + reduction kernels
    PF_VEC,           // copies, fills, axpy, dots
    PF_SETUP,         // setup-only kernels
    PF_GSPREP,        // smoother prep (upper part, fused prolongation)
    PF_SPMV_BLOCK,    // CSR SpMV of the blocks (C', Uzawa B / C) and small operators
    PF_GS_WAVE,       // Gauss-Seidel lower solve of the structured finest levels (multi-SM wavefront)
    PF_IFACE,         // td_bgs interface correction z_pm -= K w (column-major GEMV)
    PF_GS_LATTICE,    // Gauss-Seidel lower solve of the aggregated coarse levels (multi-SM lattice)
    PF_COUNT
};

// One device + one stream.  Every handle created from a context enqueues on
// its stream, so calls through one context are ordered like the reference's
// single-threaded calls.
struct Context {
    int device = 0;
    int num_sms = 148;
    cudaStream_t stream = nullptr;
    std::atomic<int64_t> launches{0};
    std::unique_ptr<PinnedBuf> pinned;   // status words, small host reads
    bool pdl = true;                     // programmatic dependent launch (launch.cuh; SDG_PDL=0 off)

    // live profiler: CUDA events bracketing every launch of a family
    struct ProfRec {
        int family;
        cudaEvent_t a, b;
        double bytes;
    };
    bool profiling = false;
    std::vector<ProfRec> prof;
    std::vector<cudaEvent_t> event_pool;
    int64_t prof_launches[PF_COUNT] = {};
    double prof_ms[PF_COUNT] = {};
    double prof_bytes[PF_COUNT] = {};
    cudaEvent_t take_event();
    void drain_profile();  // folds recorded events into the per-family sums

    // A second stream for work that overlaps the main one (BlockPrecond
    // td_bgs).  side_begin: side waits for everything issued on `stream` so
    // far and launches go to side; side_end: launches go back to the main
    // stream (no wait); side_join: the main stream waits for the side work.
    // Events only, so this also works under graph capture.
    cudaStream_t side = nullptr, main_stream = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    cudaEvent_t step_ev[2] = {nullptr, nullptr};  // GMRES: Arnoldi read-back done (krylov.cu)
    void side_begin();
    void side_continue(cudaEvent_t after);  // like side_begin, but side waits for `after` only
    void side_end();
    void side_join();

    // Device staging of the host-pointer solve entry points (b and x), kept
    // across calls: a cudaMalloc / cudaFree pair per call cost up to 130 ms on
    // the GPU box (cudaFree synchronises the device and unmaps; measured with
    // scripts/e2e_probe.py), which is end-to-end time of every host-pointer solve.
    DevBuf<double> stage_b, stage_x;
    void stage(std::size_t n) {
        if (stage_b.size() < n) stage_b.resize(n);
        if (stage_x.size() < n) stage_x.resize(n);
    }

    explicit Context(int dev);
    ~Context();
    void sync() { SDG_CUDA(cudaStreamSynchronize(stream)); }
    void count(int n = 1) { launches.fetch_add(n, std::memory_order_relaxed); }
};

// RAII: when profiling, records an event before and after the launch(es)
// issued in its scope, tagged with the launch's algorithmic bytes.
class ProfScope {
public:
    ProfScope(Context& c, int family, double bytes) : c_(c) {
        if (!c_.profiling) return;
        rec_.family = family;
        rec_.bytes = bytes;
        rec_.a = c_.take_event();
        rec_.b = c_.take_event();
        cudaEventRecord(rec_.a, c_.stream);
        on_ = true;
    }
    ~ProfScope() {
        if (!on_) return;
        cudaEventRecord(rec_.b, c_.stream);
        c_.prof.push_back(rec_);
        if (c_.prof.size() >= 4096) c_.drain_profile();
    }

private:
    Context& c_;
    Context::ProfRec rec_{};
    bool on_ = false;
};

using CtxPtr = std::shared_ptr<Context>;

// Host CSR, same invariants as the reference SparseMatrix (sparse.hpp:17-46):
// row_offsets of length n_rows+1, strictly increasing columns per row.
struct HostCsr {
    int n_rows = 0;
    int n_cols = 0;
    std::vector<int> rp{0};
    std::vector<int> ci;
    std::vector<double> v;

    HostCsr() = default;
    HostCsr(int r, int c) : n_rows(r), n_cols(c), rp(r + 1, 0) {}
    int64_t nnz() const { return static_cast<int64_t>(v.size()); }
    void check() const;  // throws SDG_EDIM on structural violations
};

// Device CSR.
struct DevCsr {
    int n_rows = 0;
    int n_cols = 0;
    int64_t nnz = 0;
    DevBuf<int> rp;
    DevBuf<int> ci;
    DevBuf<double> v;

    // optional SELL-32 copy for the operator SpMV (build_sell, kernels.cu):
    // slice s of 32 rows stores entry t of its lane-l row at sell_off[s] + 32 t + l
    bool sell = false;
    int64_t sell_entries = 0;
    DevBuf<int> sell_off, sell_len, sell_ci;
    DevBuf<double> sell_v;

    void upload(const HostCsr& h, cudaStream_t s) {
        n_rows = h.n_rows;
        n_cols = h.n_cols;
        nnz = h.nnz();
        rp.upload(h.rp, s);
        ci.upload(h.ci, s);
        v.upload(h.v, s);
    }
    void build_sell(const HostCsr& h, cudaStream_t s);  // kernels.cu
};

}  // namespace sdg
