// Device kernels of the hot path.  See kernels.cuh for the contracts.
#include "kernels.cuh"
#include "launch.cuh"
#include "rowdot.cuh"

#include <algorithm>
#include <string>

namespace sdg {

namespace {

constexpr int kThreads = 256;
constexpr int kGsThreads = 1024;
constexpr int kMaxDotVecs = 64;

inline int blocks_for(int64_t n, int threads = kThreads) {
    int64_t b = (n + threads - 1) / threads;
    return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(b, 1 << 30)));
}

__device__ __forceinline__ double warp_sum(double x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
}

// Block-wide sum of NV values; result valid in thread 0.  Fixed tree ->
// deterministic for a fixed block size.
template <int NV>
__device__ __forceinline__ void block_sum(double (&acc)[NV]) {
    __shared__ double sm[NV][32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nwarps = (blockDim.x + 31) >> 5;
#pragma unroll
    for (int v = 0; v < NV; ++v) acc[v] = warp_sum(acc[v]);
    if (lane == 0)
#pragma unroll
        for (int v = 0; v < NV; ++v) sm[v][warp] = acc[v];
    __syncthreads();
    if (warp == 0) {
#pragma unroll
        for (int v = 0; v < NV; ++v) {
            double x = lane < nwarps ? sm[v][lane] : 0.0;
            acc[v] = warp_sum(x);
        }
    }
    __syncthreads();
}

// Stores this block's NV partials; returns true in the block that arrives
// last, after folding all partials (block order fixed) into acc (thread 0).
template <int NV>
__device__ bool finish_reduce(double (&acc)[NV], double* partials, unsigned* ticket) {
    __shared__ bool am_last;
    block_sum<NV>(acc);
    if (threadIdx.x == 0) {
#pragma unroll
        for (int v = 0; v < NV; ++v) partials[blockIdx.x * NV + v] = acc[v];
        __threadfence();
        const unsigned t = atomicAdd(ticket, 1u);
        am_last = (t == gridDim.x - 1);
    }
    __syncthreads();
    if (!am_last) return false;
    __threadfence();
#pragma unroll
    for (int v = 0; v < NV; ++v) acc[v] = 0.0;
    for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x)
#pragma unroll
        for (int v = 0; v < NV; ++v) acc[v] += __ldcg(partials + b * NV + v);
    block_sum<NV>(acc);
    if (threadIdx.x == 0) *ticket = 0u;
    return true;
}

// ---------------------------------------------------------------------------
// sparse kernels

// BITWISE: sparse.cpp:81-90 / 98-108
__global__ void k_spmv(int n, const int* __restrict__ rp, const int* __restrict__ ci,
                       const double* __restrict__ v, const double* __restrict__ x,
                       const double* __restrict__ y_in, double* __restrict__ y, double alpha,
                       int add) {
    pdl_begin();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double sum = 0.0;
    row_fold<8>(ci, v, rp[i], rp[i + 1], [&](int j) { return x[j]; },
                [&](double a, double xv) { sum = __dadd_rn(sum, __dmul_rn(a, xv)); });
    y[i] = add ? __dadd_rn(y_in[i], __dmul_rn(alpha, sum)) : sum;
}

// k_spmv (add = 0) with x[j] = packed[bidx[j]] (BlockPrecond::setup_early_w)
__global__ void k_spmv_packed(int n, const int* __restrict__ rp, const int* __restrict__ ci,
                              const double* __restrict__ v, const int* __restrict__ bidx,
                              const double* __restrict__ packed, double* __restrict__ y) {
    pdl_begin();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double sum = 0.0;
    row_fold<8>(ci, v, rp[i], rp[i + 1], [&](int j) { return packed[bidx[j]]; },
                [&](double a, double xv) { sum = __dadd_rn(sum, __dmul_rn(a, xv)); });
    y[i] = sum;
}

// BITWISE: sparse.cpp:81-90 / 98-108 over the SELL-32 copy (DevCsr::build_sell):
// one thread per row still sums its entries in column order, but lane l of a
// warp reads entry t of row 32 s + l at off + 32 t + l, so every value/column
// load of the warp is one contiguous 256 B / 128 B segment (the CSR kernel
// above reads at the row stride).  Values and columns are streamed (evict
// first) so x stays in L1/L2 for the gathers; three entries per step keep
// independent loads in flight.
__global__ void __launch_bounds__(256) k_spmv_sell(int n, const int* __restrict__ off, const int* __restrict__ len,
                                                   const double* __restrict__ sv, const int* __restrict__ sc,
                                                   const double* __restrict__ x, const double* __restrict__ y_in,
                                                   double* __restrict__ y, double alpha, int add) {
    pdl_begin();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int L = len[i];
    const double* pv = sv + off[i >> 5] + (i & 31);
    const int* pc = sc + off[i >> 5] + (i & 31);
    double sum = 0.0;
    int t = 0;
    for (; t + 3 <= L; t += 3) {
        const double v0 = __ldcs(pv + 32 * t), v1 = __ldcs(pv + 32 * (t + 1)), v2 = __ldcs(pv + 32 * (t + 2));
        const int c0 = __ldcs(pc + 32 * t), c1 = __ldcs(pc + 32 * (t + 1)), c2 = __ldcs(pc + 32 * (t + 2));
        const double x0 = __ldg(x + c0), x1 = __ldg(x + c1), x2 = __ldg(x + c2);
        sum = __dadd_rn(sum, __dmul_rn(v0, x0));
        sum = __dadd_rn(sum, __dmul_rn(v1, x1));
        sum = __dadd_rn(sum, __dmul_rn(v2, x2));
    }
    for (; t < L; ++t) sum = __dadd_rn(sum, __dmul_rn(__ldcs(pv + 32 * t), __ldg(x + __ldcs(pc + 32 * t))));
    y[i] = add ? __dadd_rn(y_in[i], __dmul_rn(alpha, sum)) : sum;
}

// z[i] -= sum_k K[k n + i] w[k]  (K column-major n x m, w staged in shared
// memory).  The sum of a row is four interleaved chains a_c over the columns
// k = c (mod 4) (the tail m mod 4 columns continue a_0), folded as
// (a0 + a1) + (a2 + a3).  Warp c of a group of four computes chain c for 32
// consecutive rows (every load instruction reads 256 contiguous bytes of one
// column), 8 loads in flight per lane, and the fold goes through shared
// memory in the same association, so the result does not depend on the
// launch shape.  (An 8-way column split with a different fold changed the
// BiCGSTAB count at c2 by rounding alone; one lane per row with 4 loads in
// flight left the GEMV latency-bound: 27 us for 33 MB at c2.)
template <bool STREAM>
__device__ __forceinline__ double ld_k(const double* p) {
    return STREAM ? __ldcs(p) : __ldg(p);
}

constexpr int kGemvRowBlocks = 2;  // 32-row blocks per CTA (4 warps each)

template <bool STREAM>  // STREAM: K too large to stay in L2, read once per apply (evict first)
__global__ void __launch_bounds__(128 * kGemvRowBlocks)
    k_colmajor_gemv_sub(int n, int m, const double* __restrict__ kmat, const double* __restrict__ w,
                        double* __restrict__ z) {
    pdl_begin();
    extern __shared__ double ws[];
    __shared__ double part[4 * kGemvRowBlocks][32];
    for (int k = threadIdx.x; k < m; k += blockDim.x) ws[k] = w[k];
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int c = warp & 3, rb = warp >> 2;
    const int i = (blockIdx.x * kGemvRowBlocks + rb) * 32 + lane;
    double a = 0.0;
    if (i < n) {
        const double* col = kmat + i;
        const int m4 = m & ~3;
        int k = c;
        constexpr int U = 8;
        for (; k + 4 * (U - 1) < m4; k += 4 * U) {
            double v[U];
#pragma unroll
            for (int j = 0; j < U; ++j) v[j] = ld_k<STREAM>(col + static_cast<size_t>(k + 4 * j) * n);
#pragma unroll
            for (int j = 0; j < U; ++j) a = fma(v[j], ws[k + 4 * j], a);
        }
        for (; k < m4; k += 4) a = fma(ld_k<STREAM>(col + static_cast<size_t>(k) * n), ws[k], a);
        if (c == 0)
            for (k = m4; k < m; ++k) a = fma(ld_k<STREAM>(col + static_cast<size_t>(k) * n), ws[k], a);
    }
    part[warp][lane] = a;
    __syncthreads();
    if (c == 0 && i < n) {
        const double* p = &part[4 * rb][lane];
        z[i] -= (p[0] + p[32]) + (p[64] + p[96]);
    }
}

// BITWISE: precond.cpp:92-108 (sor_sweep), one CTA walking the level
// schedule.  Lower neighbours (j < i) read the new iterate, upper ones the
// old, in the reference's column order; the division order of
// `(1 - omega) * z + omega * s / diag` is kept.
__global__ void __launch_bounds__(kGsThreads)
k_gs_levels(const int* __restrict__ rp, const int* __restrict__ ci, const double* __restrict__ v,
            const int* __restrict__ lvl_ptr, const int* __restrict__ lvl_rows, int n_levels,
            const double* __restrict__ r, const double* z_old, double* z_new, double omega) {
    pdl_begin();
    for (int l = 0; l < n_levels; ++l) {
        const int b = lvl_ptr[l], e = lvl_ptr[l + 1];
        for (int idx = b + threadIdx.x; idx < e; idx += blockDim.x) {
            const int i = lvl_rows[idx];
            double s = r[i];
            double diag = 0.0;
            const int ke = rp[i + 1];
            for (int k = rp[i]; k < ke; ++k) {
                const int j = ci[k];
                const double a = v[k];
                if (j == i) {
                    diag = a;
                } else {
                    const double zj = j < i ? z_new[j] : (z_old ? z_old[j] : 0.0);
                    s = __dsub_rn(s, __dmul_rn(a, zj));
                }
            }
            const double zi = z_old ? z_old[i] : 0.0;
            z_new[i] = __dadd_rn(__dmul_rn(1.0 - omega, zi), __ddiv_rn(__dmul_rn(omega, s), diag));
        }
        __syncthreads();
    }
}

// BITWISE: precond.cpp:241-244
__global__ void k_resid_restrict(int n_coarse, const int* __restrict__ pt_ptr,
                                 const int* __restrict__ pt_rows, const int* __restrict__ rp,
                                 const int* __restrict__ ci, const double* __restrict__ v,
                                 const double* __restrict__ r, const double* __restrict__ z,
                                 double* __restrict__ rc) {
    pdl_begin();
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= n_coarse) return;
    double acc = 0.0;
    const int qe = pt_ptr[c + 1];
    for (int q = pt_ptr[c]; q < qe; ++q) {
        const int i = pt_rows[q];
        double sum = 0.0;
        const int ke = rp[i + 1];
        for (int k = rp[i]; k < ke; ++k) sum = __dadd_rn(sum, __dmul_rn(v[k], z[ci[k]]));
        acc = __dadd_rn(acc, __dadd_rn(r[i], __dmul_rn(-1.0, sum)));
    }
    rc[c] = acc;
}

// BITWISE: precond.cpp:247
__global__ void k_prolong(int n, const int* __restrict__ agg, const double* __restrict__ z,
                          const double* __restrict__ zc, double* __restrict__ out) {
    pdl_begin();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = __dadd_rn(z[i], zc[agg[i]]);
}

// y = Ainv x, one warp per row.
__global__ void k_dense_gemv(int n, const double* __restrict__ a, const double* __restrict__ x,
                             double* __restrict__ y) {
    pdl_begin();
    const int warps = blockDim.x >> 5;
    const int row = blockIdx.x * warps + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (row >= n) return;
    const double* ar = a + static_cast<size_t>(row) * n;
    // four independent accumulators keep four loads in flight per lane
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int j = lane;
    for (; j + 96 < n; j += 128) {
        s0 = fma(__ldg(ar + j), __ldg(x + j), s0);
        s1 = fma(__ldg(ar + j + 32), __ldg(x + j + 32), s1);
        s2 = fma(__ldg(ar + j + 64), __ldg(x + j + 64), s2);
        s3 = fma(__ldg(ar + j + 96), __ldg(x + j + 96), s3);
    }
    for (; j < n; j += 32) s0 = fma(__ldg(ar + j), __ldg(x + j), s0);
    double s = warp_sum((s0 + s1) + (s2 + s3));
    if (lane == 0) y[row] = s;
}

// The same GEMV with WPR warps per row (a fixed-order fold of their partial
// sums): small coarse inverses live in L2, where one warp per row leaves too
// few loads in flight (c2: 1,407 rows -> 1.2 TB/s).
template <int WPR>
__global__ void k_dense_gemv_split(int n, const double* __restrict__ a, const double* __restrict__ x,
                                   double* __restrict__ y) {
    pdl_begin();
    __shared__ double red[32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int row = blockIdx.x * ((blockDim.x >> 5) / WPR) + warp / WPR;
    const int part = warp % WPR;
    double s = 0.0;
    if (row < n) {
        const double* ar = a + static_cast<size_t>(row) * n;
        const int chunk = (n + WPR - 1) / WPR;
        const int c0 = part * chunk, c1 = min(n, c0 + chunk);
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
        int j = c0 + lane;
        for (; j + 96 < c1; j += 128) {
            s0 = fma(__ldg(ar + j), __ldg(x + j), s0);
            s1 = fma(__ldg(ar + j + 32), __ldg(x + j + 32), s1);
            s2 = fma(__ldg(ar + j + 64), __ldg(x + j + 64), s2);
            s3 = fma(__ldg(ar + j + 96), __ldg(x + j + 96), s3);
        }
        for (; j < c1; j += 32) s0 = fma(__ldg(ar + j), __ldg(x + j), s0);
        s = warp_sum((s0 + s1) + (s2 + s3));
    }
    if (lane == 0) red[warp] = s;
    __syncthreads();
    if (row < n && part == 0 && lane == 0) {
        double t = red[warp];
#pragma unroll
        for (int q = 1; q < WPR; ++q) t += red[warp + q];
        y[row] = t;
    }
}

// BITWISE: precond.cpp:296-298
__global__ void k_uzawa_p(int n, const int* __restrict__ rp, const int* __restrict__ ci,
                          const double* __restrict__ v, const double* __restrict__ zv,
                          const double* __restrict__ r_p, double omega, double* __restrict__ z_p) {
    pdl_begin();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double sum = 0.0;
    row_fold<8>(ci, v, rp[i], rp[i + 1], [&](int j) { return zv[j]; },
                [&](double a, double x) { sum = __dadd_rn(sum, __dmul_rn(a, x)); });
    z_p[i] = __dmul_rn(omega, __dsub_rn(sum, r_p[i]));
}

__global__ void k_copy(int64_t n, double* __restrict__ d, const double* __restrict__ s) {
    pdl_begin();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        d[i] = s[i];
}

__global__ void k_fill(int64_t n, double* __restrict__ d, double val) {
    pdl_begin();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        d[i] = val;
}

__global__ void k_csr_to_dense(int n, const int* __restrict__ rp, const int* __restrict__ ci,
                               const double* __restrict__ v, double* __restrict__ dense) {
    pdl_begin();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    for (int k = rp[i]; k < rp[i + 1]; ++k) dense[static_cast<size_t>(i) * n + ci[k]] = v[k];
}

__global__ void k_set_identity(int n, double* dense) {
    pdl_begin();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) dense[static_cast<size_t>(i) * n + i] = 1.0;
}

// ---------------------------------------------------------------------------
// Krylov vector kernels

// Block b owns elements [b*chunk, min(n,(b+1)*chunk)); warp w dots vectors
// w, w+8, ... of X against y over that chunk.
// out[v] = X[v] . y for v < k.  One 1024-thread block per SM owns a chunk of
// rows; its threads walk the chunk once per group of kDotGroup vectors with
// that many independent accumulators, two rows per step (16 loads in flight
// per thread), and fold them in a fixed order.  The last block folds the
// per-block partials one vector per warp (deterministic, no block barriers).
constexpr int kDotGroup = 8;
constexpr int kDotThreads = 1024;

__global__ void __launch_bounds__(kDotThreads) k_multidot(int64_t n, int k, const double* __restrict__ X,
                                                          int64_t ldx, const double* __restrict__ y, int64_t chunk,
                                                          double* partials, unsigned* ticket,
                                                          double* __restrict__ out) {
    pdl_begin();
    __shared__ bool am_last;
    __shared__ double red[kDotThreads / 32][kMaxDotVecs];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    const int64_t b0 = blockIdx.x * chunk;
    const int64_t b1 = min(n, b0 + chunk);
    // no block barrier between groups: a warp that has finished a group's rows
    // folds its accumulators and starts the next group's loads while the other
    // warps are still streaming (one barrier at the end, same fold order)
    for (int g0 = 0; g0 < k; g0 += kDotGroup) {
        double acc[kDotGroup];
#pragma unroll
        for (int g = 0; g < kDotGroup; ++g) acc[g] = 0.0;
        const int ng = min(kDotGroup, k - g0);
        int64_t i = b0 + threadIdx.x;
        for (; i + blockDim.x < b1; i += 2 * blockDim.x) {
            const double y0 = __ldg(y + i), y1 = __ldg(y + i + blockDim.x);
            double x0[kDotGroup], x1[kDotGroup];
#pragma unroll
            for (int g = 0; g < kDotGroup; ++g) {
                x0[g] = g < ng ? __ldcs(X + (g0 + g) * ldx + i) : 0.0;
                x1[g] = g < ng ? __ldcs(X + (g0 + g) * ldx + i + blockDim.x) : 0.0;
            }
#pragma unroll
            for (int g = 0; g < kDotGroup; ++g) acc[g] = fma(x1[g], y1, fma(x0[g], y0, acc[g]));
        }
        if (i < b1) {
            const double y0 = __ldg(y + i);
#pragma unroll
            for (int g = 0; g < kDotGroup; ++g)
                if (g < ng) acc[g] = fma(__ldcs(X + (g0 + g) * ldx + i), y0, acc[g]);
        }
#pragma unroll
        for (int g = 0; g < kDotGroup; ++g) {
            const double t = warp_sum(acc[g]);
            if (lane == 0 && g < ng) red[warp][g0 + g] = t;
        }
    }
    __syncthreads();
    if (threadIdx.x < k) {
        double t = 0.0;
        for (int w = 0; w < nwarps; ++w) t += red[w][threadIdx.x];
        partials[blockIdx.x * kMaxDotVecs + threadIdx.x] = t;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned t = atomicAdd(ticket, 1u);
        am_last = (t == gridDim.x - 1);
    }
    __syncthreads();
    if (!am_last) return;
    __threadfence();
    for (int vv = warp; vv < k; vv += nwarps) {
        double s = 0.0;
        for (int b = lane; b < (int)gridDim.x; b += 32) s += __ldcg(partials + b * kMaxDotVecs + vv);
        s = warp_sum(s);
        if (lane == 0) out[vv] = s;
    }
    __syncthreads();
    if (threadIdx.x == 0) *ticket = 0u;
}

template <bool NORM>
__global__ void k_multi_axpy(int64_t n, int k, const double* __restrict__ X, int64_t ldx,
                             const double* __restrict__ h, double* __restrict__ w,
                             double* partials, unsigned* ticket, double* out) {
    pdl_begin();
    __shared__ double hs[kMaxDotVecs];
    if (threadIdx.x < k) hs[threadIdx.x] = h[threadIdx.x];
    __syncthreads();
    double acc[1] = {0.0};
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        double wi = w[i];
#pragma unroll 8
        for (int vv = 0; vv < k; ++vv) wi = fma(-hs[vv], __ldg(X + vv * ldx + i), wi);
        w[i] = wi;
        if (NORM) acc[0] = fma(wi, wi, acc[0]);
    }
    if (NORM) {
        if (finish_reduce<1>(acc, partials, ticket) && threadIdx.x == 0) out[0] = sqrt(acc[0]);  // ||w||, not its square
    }
}

// BITWISE: reference `scale(vi, 1.0 / wn)` (krylov.cpp:115-117)
__global__ void k_scale_by_inv(int64_t n, const double* __restrict__ src,
                               const double* __restrict__ den, double* __restrict__ dst) {
    pdl_begin();
    const double d = *den;
    if (!(d > 0.0)) return;
    const double inv = 1.0 / d;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = __dmul_rn(src[i], inv);
}

// BITWISE: krylov.cpp:153-154 (fill + axpy loop, sequential in v)
__global__ void k_lincomb(int64_t n, int k, const double* __restrict__ X, int64_t ldx,
                          const double* __restrict__ y, double* __restrict__ w) {
    pdl_begin();
    __shared__ double ys[kMaxDotVecs];
    if (threadIdx.x < k) ys[threadIdx.x] = y[threadIdx.x];
    __syncthreads();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int vv = 0; vv < k; ++vv) s = __dadd_rn(s, __dmul_rn(ys[vv], X[vv * ldx + i]));
        w[i] = s;
    }
}

__global__ void k_add_inplace(int64_t n, double* __restrict__ x, const double* __restrict__ z) {
    pdl_begin();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        x[i] = __dadd_rn(x[i], z[i]);
}

__global__ void k_axpy_dev(int64_t n, const double* __restrict__ alpha,
                           const double* __restrict__ x, double* __restrict__ y) {
    pdl_begin();
    const double a = *alpha;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        y[i] = __dadd_rn(y[i], __dmul_rn(a, x[i]));
}

__global__ void k_dot(int64_t n, const double* __restrict__ x, const double* __restrict__ y,
                      double* partials, unsigned* ticket, double* out) {
    pdl_begin();
    double acc[1] = {0.0};
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        acc[0] = fma(x[i], y[i], acc[0]);
    if (finish_reduce<1>(acc, partials, ticket) && threadIdx.x == 0) out[0] = acc[0];
}

// BITWISE: krylov.cpp:337
__global__ void k_div_scalar(int64_t n, const double* __restrict__ y, const double* __restrict__ yn,
                             double* __restrict__ x) {
    pdl_begin();
    const double d = *yn;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        x[i] = __ddiv_rn(y[i], d);
}

// ---------------------------------------------------------------------------
// BiCGSTAB (krylov.cpp:240-283); element updates keep the reference's
// expression order, reductions are deterministic tree sums.

__global__ void k_bi_p(int64_t n, BiState* st, const double* __restrict__ r,
                       const double* __restrict__ v, double* __restrict__ p) {
    pdl_begin();
    if (st->flag) return;
    const double rho_new = st->rho_new;
    if (fabs(rho_new) < 1e-300) {
        if (blockIdx.x == 0 && threadIdx.x == 0) st->flag = BI_BREAK_RHO;
        return;
    }
    const double beta = __dmul_rn(__ddiv_rn(rho_new, st->rho), __ddiv_rn(st->alpha, st->omega));
    const double om = st->omega;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        p[i] = __dadd_rn(r[i], __dmul_rn(beta, __dsub_rn(p[i], __dmul_rn(om, v[i]))));
}

__global__ void k_bi_rv(int64_t n, BiState* st, const double* __restrict__ rhat,
                        const double* __restrict__ v, double* partials, unsigned* ticket) {
    pdl_begin();
    double acc[1] = {0.0};
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        acc[0] = fma(rhat[i], v[i], acc[0]);
    if (finish_reduce<1>(acc, partials, ticket) && threadIdx.x == 0) {
        if (st->flag) return;
        st->rv = acc[0];
        if (fabs(acc[0]) < 1e-300)
            st->flag = BI_BREAK_RV;
        else
            st->alpha = st->rho_new / acc[0];
    }
}

__global__ void k_bi_s(int64_t n, BiState* st, const double* __restrict__ r,
                       const double* __restrict__ v, double* __restrict__ s, double* partials,
                       unsigned* ticket) {
    pdl_begin();
    const int flag = st->flag;  // uniform for the whole launch
    double acc[1] = {0.0};
    if (!flag) {
        const double alpha = st->alpha;
        for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
             i += (int64_t)gridDim.x * blockDim.x) {
            const double si = __dsub_rn(r[i], __dmul_rn(alpha, v[i]));
            s[i] = si;
            acc[0] = fma(si, si, acc[0]);
        }
    }
    if (finish_reduce<1>(acc, partials, ticket) && threadIdx.x == 0) {
        if (flag) return;
        st->sn = sqrt(acc[0]);
        if (st->sn <= st->tol) st->flag = BI_S_CONV;
    }
}

__global__ void k_bi_t(int64_t n, BiState* st, const double* __restrict__ t,
                       const double* __restrict__ s, double* partials, unsigned* ticket) {
    pdl_begin();
    const int flag = st->flag;
    double acc[2] = {0.0, 0.0};
    if (!flag) {
        for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
             i += (int64_t)gridDim.x * blockDim.x) {
            const double ti = t[i];
            acc[0] = fma(ti, ti, acc[0]);
            acc[1] = fma(ti, s[i], acc[1]);
        }
    }
    if (finish_reduce<2>(acc, partials, ticket) && threadIdx.x == 0) {
        if (flag) return;
        st->tt = acc[0];
        st->ts = acc[1];
        if (acc[0] == 0.0) {
            st->flag = BI_BREAK_TT;
            return;
        }
        const double om = acc[1] / acc[0];
        if (fabs(om) < 1e-300)
            st->flag = BI_BREAK_OMEGA;
        else
            st->omega = om;
    }
}

__global__ void k_bi_xr(int64_t n, BiState* st, const double* __restrict__ phat,
                        const double* __restrict__ shat, const double* __restrict__ s,
                        const double* __restrict__ t, const double* __restrict__ rhat,
                        double* __restrict__ x, double* __restrict__ r, double* partials,
                        unsigned* ticket) {
    pdl_begin();
    const int flag = st->flag;
    double acc[2] = {0.0, 0.0};
    if (!flag) {
        const double alpha = st->alpha, om = st->omega;
        for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
             i += (int64_t)gridDim.x * blockDim.x) {
            x[i] = __dadd_rn(x[i], __dadd_rn(__dmul_rn(alpha, phat[i]), __dmul_rn(om, shat[i])));
            const double ri = __dsub_rn(s[i], __dmul_rn(om, t[i]));
            r[i] = ri;
            acc[0] = fma(ri, ri, acc[0]);
            acc[1] = fma(rhat[i], ri, acc[1]);
        }
    }
    if (finish_reduce<2>(acc, partials, ticket) && threadIdx.x == 0) {
        if (flag) return;
        st->rho = st->rho_new;
        st->rn = sqrt(acc[0]);
        st->rho_new = acc[1];
    }
}

__global__ void k_bi_rho(int64_t n, BiState* st, const double* __restrict__ rhat,
                         const double* __restrict__ r, double* partials, unsigned* ticket) {
    pdl_begin();
    double acc[1] = {0.0};
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        acc[0] = fma(rhat[i], r[i], acc[0]);
    if (finish_reduce<1>(acc, partials, ticket) && threadIdx.x == 0) st->rho_new = acc[0];
}

__global__ void k_bi_x_alpha(int64_t n, const BiState* st, const double* __restrict__ phat,
                             double* __restrict__ x) {
    pdl_begin();
    const double a = st->alpha;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        x[i] = __dadd_rn(x[i], __dmul_rn(a, phat[i]));
}

}  // namespace

// ---------------------------------------------------------------------------
// launchers

int reduce_blocks(int n, int num_sms) {
    const int want = (n + 4 * kThreads - 1) / (4 * kThreads);
    return std::max(1, std::min(want, 2 * num_sms));
}

void ReduceWs::init(int blocks, int vals, cudaStream_t s) {
    max_blocks = blocks;
    max_vals = vals;
    partials.resize(static_cast<size_t>(blocks) * vals);
    ticket.resize(1);
    SDG_CUDA(cudaMemsetAsync(ticket.get(), 0, sizeof(unsigned), s));
}

static inline int stride_blocks(Context& c, int64_t n) {
    const int64_t want = (n + kThreads - 1) / kThreads;
    return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(want, 8LL * c.num_sms)));
}

#define SDG_LAUNCHED(ctx)                                                  \
    do {                                                                   \
        (ctx).count();                                                     \
        cudaError_t e_ = cudaGetLastError();                               \
        if (e_ != cudaSuccess)                                             \
            ::sdg::fail(SDG_ECUDA, std::string(__func__) + ": " + cudaGetErrorString(e_)); \
    } while (0)

void launch_spmv_packed(Context& c, const DevCsr& a, const int* bidx, const double* packed, double* y) {
    ProfScope ps_(c, PF_SPMV_BLOCK, 12.0 * a.nnz + 4.0 * (a.n_rows + 1) + 12.0 * a.n_cols + 8.0 * a.n_rows);
    if (a.n_rows == 0) return;
    launch_k(c, k_spmv_packed, blocks_for(a.n_rows), kThreads, 0, a.n_rows, a.rp.get(), a.ci.get(), a.v.get(), bidx,
             packed, y);
    SDG_LAUNCHED(c);
}

void launch_spmv(Context& c, const DevCsr& a, const double* x, double* y) {
    ProfScope ps_(c, a.sell ? PF_SPMV : PF_SPMV_BLOCK,
                  12.0 * a.nnz + 4.0 * (a.n_rows + 1) + 8.0 * a.n_cols + 8.0 * a.n_rows);
    if (a.n_rows == 0) return;
    if (a.sell) {
        launch_k(c, k_spmv_sell, (a.n_rows + 255) / 256, 256, 0, a.n_rows, a.sell_off.get(), a.sell_len.get(),
                 a.sell_v.get(), a.sell_ci.get(), x, static_cast<const double*>(nullptr), y, 0.0, 0);
        SDG_LAUNCHED(c);
        return;
    }
    launch_k(c, k_spmv, blocks_for(a.n_rows), kThreads, 0, a.n_rows, a.rp.get(), a.ci.get(),
                                                            a.v.get(), x, nullptr, y, 0.0, 0);
    SDG_LAUNCHED(c);
}

void launch_spmv_add(Context& c, const DevCsr& a, const double* x, const double* y_in,
                     double* y_out, double alpha) {
    ProfScope ps_(c, a.sell ? PF_SPMV : PF_SPMV_BLOCK,
                  12.0 * a.nnz + 4.0 * (a.n_rows + 1) + 8.0 * a.n_cols + 16.0 * a.n_rows);
    if (a.n_rows == 0) return;
    if (a.sell) {
        launch_k(c, k_spmv_sell, (a.n_rows + 255) / 256, 256, 0, a.n_rows, a.sell_off.get(), a.sell_len.get(),
                 a.sell_v.get(), a.sell_ci.get(), x, y_in, y_out, alpha, 1);
        SDG_LAUNCHED(c);
        return;
    }
    launch_k(c, k_spmv, blocks_for(a.n_rows), kThreads, 0, a.n_rows, a.rp.get(), a.ci.get(),
                                                            a.v.get(), x, y_in, y_out, alpha, 1);
    SDG_LAUNCHED(c);
}

void launch_gs_levels(Context& c, const DevCsr& a, const int* lvl_ptr, const int* lvl_rows,
                      int n_levels, const double* r, const double* z_old, double* z_new,
                      double omega) {
    ProfScope ps_(c, PF_GS, 12.0 * a.nnz + 4.0 * (a.n_rows + 1) + (z_old ? 24.0 : 16.0) * a.n_rows + 4.0 * a.n_rows + 4.0 * (n_levels + 1));
    if (a.n_rows == 0) return;
    launch_k(c, k_gs_levels, 1, kGsThreads, 0, a.rp.get(), a.ci.get(), a.v.get(), lvl_ptr,
                                                lvl_rows, n_levels, r, z_old, z_new, omega);
    SDG_LAUNCHED(c);
}

void launch_resid_restrict(Context& c, const DevCsr& a, const int* pt_ptr, const int* pt_rows,
                           int n_coarse, const double* r, const double* z, double* rc) {
    ProfScope ps_(c, PF_RESTRICT, 12.0 * a.nnz + 4.0 * (a.n_rows + 1) + 16.0 * a.n_rows + 4.0 * a.n_rows + 4.0 * (n_coarse + 1) + 8.0 * n_coarse);
    if (n_coarse == 0) return;
    launch_k(c, k_resid_restrict, blocks_for(n_coarse, 128), 128, 0, 
        n_coarse, pt_ptr, pt_rows, a.rp.get(), a.ci.get(), a.v.get(), r, z, rc);
    SDG_LAUNCHED(c);
}

void launch_prolong(Context& c, int n, const int* agg, const double* z, const double* zc,
                    double* out) {
    ProfScope ps_(c, PF_PROLONG, 20.0 * n + 8.0 * n);
    if (n == 0) return;
    launch_k(c, k_prolong, blocks_for(n), kThreads, 0, n, agg, z, zc, out);
    SDG_LAUNCHED(c);
}

void launch_colmajor_gemv_sub(Context& c, int n, int m, const double* kmat, const double* w, double* z) {
    ProfScope ps_(c, PF_IFACE, 8.0 * n * m + 8.0 * m + 16.0 * n);
    if (n == 0 || m == 0) return;
    const size_t smem = static_cast<size_t>(m) * 8;
    // w is staged in shared memory: raise the dynamic limit once per instantiation
    // (callers keep m <= kColmajorMaxGamma, setup_interface_split)
    if (m > kColmajorMaxGamma) fail(SDG_EINVAL, "colmajor_gemv_sub: too many interface columns");
    static const bool attr = [] {
        const int lim = kColmajorMaxGamma * 8;
        SDG_CUDA(cudaFuncSetAttribute(k_colmajor_gemv_sub<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, lim));
        SDG_CUDA(cudaFuncSetAttribute(k_colmajor_gemv_sub<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, lim));
        return true;
    }();
    (void)attr;
    if (8.0 * n * m > 40e6)
        launch_k(c, k_colmajor_gemv_sub<true>, (n + 32 * kGemvRowBlocks - 1) / (32 * kGemvRowBlocks), 128 * kGemvRowBlocks, smem, n, m, kmat, w, z);
    else
        launch_k(c, k_colmajor_gemv_sub<false>, (n + 32 * kGemvRowBlocks - 1) / (32 * kGemvRowBlocks), 128 * kGemvRowBlocks, smem, n, m, kmat, w, z);
    SDG_LAUNCHED(c);
}

void launch_dense_gemv(Context& c, int n, const double* ainv, const double* x, double* y) {
    ProfScope ps_(c, PF_COARSE, 8.0 * n * (double)n + 16.0 * n);
    if (n == 0) return;
    const int warps = kThreads / 32;
    // enough warps in flight for the L2-resident case: up to 8 per row
    const int want = (4 * c.num_sms * 32 + n - 1) / std::max(n, 1);
    const int wpr = want >= 8 ? 8 : want >= 4 ? 4 : want >= 2 ? 2 : 1;
    if (wpr == 1) {
        launch_k(c, k_dense_gemv, (n + warps - 1) / warps, kThreads, 0, n, ainv, x, y);
    } else {
        const int rows_per_block = warps / wpr;
        const int grid = (n + rows_per_block - 1) / rows_per_block;
        if (wpr == 8) launch_k(c, k_dense_gemv_split<8>, grid, kThreads, 0, n, ainv, x, y);
        if (wpr == 4) launch_k(c, k_dense_gemv_split<4>, grid, kThreads, 0, n, ainv, x, y);
        if (wpr == 2) launch_k(c, k_dense_gemv_split<2>, grid, kThreads, 0, n, ainv, x, y);
    }
    SDG_LAUNCHED(c);
}

void launch_uzawa_pressure(Context& c, const DevCsr& cm, const double* z_v, const double* r_p,
                           double omega, double* z_p) {
    ProfScope ps_(c, PF_UZAWA, 12.0 * cm.nnz + 4.0 * (cm.n_rows + 1) + 8.0 * cm.n_cols + 16.0 * cm.n_rows);
    if (cm.n_rows == 0) return;
    launch_k(c, k_uzawa_p, blocks_for(cm.n_rows), kThreads, 0, cm.n_rows, cm.rp.get(), cm.ci.get(),
                                                                cm.v.get(), z_v, r_p, omega, z_p);
    SDG_LAUNCHED(c);
}

void launch_copy(Context& c, double* dst, const double* src, int64_t n) {
    ProfScope ps_(c, PF_VEC, 16.0 * n);
    if (n == 0 || dst == src) return;
    launch_k(c, k_copy, stride_blocks(c, n), kThreads, 0, n, dst, src);
    SDG_LAUNCHED(c);
}

void launch_fill(Context& c, double* dst, double v, int64_t n) {
    ProfScope ps_(c, PF_VEC, 8.0 * n);
    if (n == 0) return;
    launch_k(c, k_fill, stride_blocks(c, n), kThreads, 0, n, dst, v);
    SDG_LAUNCHED(c);
}

void launch_csr_to_dense(Context& c, const DevCsr& a, double* dense) {
    ProfScope ps_(c, PF_SETUP, 12.0 * a.nnz);
    if (a.n_rows == 0) return;
    launch_k(c, k_csr_to_dense, blocks_for(a.n_rows), kThreads, 0, a.n_rows, a.rp.get(),
                                                                    a.ci.get(), a.v.get(), dense);
    SDG_LAUNCHED(c);
}

void launch_set_identity(Context& c, int n, double* dense) {
    ProfScope ps_(c, PF_SETUP, 8.0 * n);
    if (n == 0) return;
    launch_k(c, k_set_identity, blocks_for(n), kThreads, 0, n, dense);
    SDG_LAUNCHED(c);
}

void launch_multidot(Context& c, ReduceWs& ws, int64_t n, int k, const double* X, int64_t ldx,
                     const double* y, double* out) {
    ProfScope ps_(c, PF_ORTHO, 8.0 * (k + 1) * (double)n);
    if (k <= 0) return;
    if (k > kMaxDotVecs || ws.max_vals < kMaxDotVecs) fail(SDG_EINVAL, "multidot: too many vectors");
    // one block per SM, fewer when the rows are few
    int nb = static_cast<int>(std::min<int64_t>(c.num_sms, (n + 4 * kDotThreads - 1) / (4 * kDotThreads)));
    nb = std::max(1, std::min(nb, ws.max_blocks));
    const int64_t chunk = std::max<int64_t>(1, (n + nb - 1) / nb);
    nb = static_cast<int>((n + chunk - 1) / chunk);
    if (nb < 1) nb = 1;
    launch_k(c, k_multidot, nb, kDotThreads, 0, n, k, X, ldx, y, chunk, ws.partials.get(), ws.ticket.get(), out);
    SDG_LAUNCHED(c);
}

void launch_multi_axpy(Context& c, int64_t n, int k, const double* X, int64_t ldx,
                       const double* h, double* w) {
    ProfScope ps_(c, PF_ORTHO, 8.0 * (k + 2) * (double)n);
    if (k <= 0) return;
    launch_k(c, k_multi_axpy<false>, stride_blocks(c, n), kThreads, 0, n, k, X, ldx, h, w,
                                                                       nullptr, nullptr, nullptr);
    SDG_LAUNCHED(c);
}

void launch_multi_axpy_norm2(Context& c, ReduceWs& ws, int64_t n, int k, const double* X,
                             int64_t ldx, const double* h, double* w, double* out) {
    ProfScope ps_(c, PF_ORTHO, 8.0 * (k + 2) * (double)n);
    // as many blocks as the plain multi_axpy (the norm fold reads one partial per block)
    const int nb = std::min(stride_blocks(c, n), ws.max_blocks);
    launch_k(c, k_multi_axpy<true>, nb, kThreads, 0, n, k, X, ldx, h, w, ws.partials.get(),
                                                      ws.ticket.get(), out);
    SDG_LAUNCHED(c);
}

void launch_scale_by_inv(Context& c, int64_t n, const double* src, const double* den, double* dst) {
    ProfScope ps_(c, PF_ORTHO, 16.0 * n);
    launch_k(c, k_scale_by_inv, stride_blocks(c, n), kThreads, 0, n, src, den, dst);
    SDG_LAUNCHED(c);
}

void launch_lincomb(Context& c, int64_t n, int k, const double* X, int64_t ldx, const double* y,
                    double* w) {
    ProfScope ps_(c, PF_ORTHO, 8.0 * (k + 1) * (double)n);
    if (k > kMaxDotVecs) fail(SDG_EINVAL, "lincomb: too many vectors");
    launch_k(c, k_lincomb, stride_blocks(c, n), kThreads, 0, n, k, X, ldx, y, w);
    SDG_LAUNCHED(c);
}

void launch_add_inplace(Context& c, int64_t n, double* x, const double* z) {
    ProfScope ps_(c, PF_VEC, 24.0 * n);
    launch_k(c, k_add_inplace, stride_blocks(c, n), kThreads, 0, n, x, z);
    SDG_LAUNCHED(c);
}

void launch_axpy_dev(Context& c, int64_t n, const double* alpha, const double* x, double* y) {
    ProfScope ps_(c, PF_VEC, 24.0 * n);
    launch_k(c, k_axpy_dev, stride_blocks(c, n), kThreads, 0, n, alpha, x, y);
    SDG_LAUNCHED(c);
}

static inline int red_blocks(Context& c, ReduceWs& ws, int64_t n) {
    return std::min(reduce_blocks(static_cast<int>(std::min<int64_t>(n, 1 << 30)), c.num_sms),
                    ws.max_blocks);
}

void launch_norm2sq(Context& c, ReduceWs& ws, int64_t n, const double* x, double* out) {
    ProfScope ps_(c, PF_VEC, 8.0 * n);
    launch_k(c, k_dot, red_blocks(c, ws, n), kThreads, 0, n, x, x, ws.partials.get(),
                                                           ws.ticket.get(), out);
    SDG_LAUNCHED(c);
}

void launch_dot(Context& c, ReduceWs& ws, int64_t n, const double* x, const double* y, double* out) {
    ProfScope ps_(c, PF_VEC, 16.0 * n);
    launch_k(c, k_dot, red_blocks(c, ws, n), kThreads, 0, n, x, y, ws.partials.get(),
                                                           ws.ticket.get(), out);
    SDG_LAUNCHED(c);
}

void launch_div_scalar(Context& c, int64_t n, const double* y, const double* yn, double* x) {
    ProfScope ps_(c, PF_VEC, 16.0 * n);
    launch_k(c, k_div_scalar, stride_blocks(c, n), kThreads, 0, n, y, yn, x);
    SDG_LAUNCHED(c);
}

void launch_bi_p(Context& c, int64_t n, BiState* st, const double* r, const double* v, double* p) {
    ProfScope ps_(c, PF_BICG, 32.0 * n);
    launch_k(c, k_bi_p, stride_blocks(c, n), kThreads, 0, n, st, r, v, p);
    SDG_LAUNCHED(c);
}

void launch_bi_rv(Context& c, ReduceWs& ws, int64_t n, BiState* st, const double* rhat,
                  const double* v) {
    ProfScope ps_(c, PF_BICG, 16.0 * n);
    launch_k(c, k_bi_rv, red_blocks(c, ws, n), kThreads, 0, n, st, rhat, v, ws.partials.get(),
                                                             ws.ticket.get());
    SDG_LAUNCHED(c);
}

void launch_bi_s(Context& c, ReduceWs& ws, int64_t n, BiState* st, const double* r,
                 const double* v, double* s) {
    ProfScope ps_(c, PF_BICG, 24.0 * n);
    launch_k(c, k_bi_s, red_blocks(c, ws, n), kThreads, 0, n, st, r, v, s, ws.partials.get(),
                                                            ws.ticket.get());
    SDG_LAUNCHED(c);
}

void launch_bi_t(Context& c, ReduceWs& ws, int64_t n, BiState* st, const double* t,
                 const double* s) {
    ProfScope ps_(c, PF_BICG, 16.0 * n);
    launch_k(c, k_bi_t, red_blocks(c, ws, n), kThreads, 0, n, st, t, s, ws.partials.get(),
                                                            ws.ticket.get());
    SDG_LAUNCHED(c);
}

void launch_bi_xr(Context& c, ReduceWs& ws, int64_t n, BiState* st, const double* phat,
                  const double* shat, const double* s, const double* t, const double* rhat,
                  double* x, double* r) {
    ProfScope ps_(c, PF_BICG, 64.0 * n);
    launch_k(c, k_bi_xr, red_blocks(c, ws, n), kThreads, 0, n, st, phat, shat, s, t, rhat, x, r,
                                                             ws.partials.get(), ws.ticket.get());
    SDG_LAUNCHED(c);
}

void launch_bi_rho(Context& c, ReduceWs& ws, int64_t n, BiState* st, const double* rhat,
                   const double* r) {
    ProfScope ps_(c, PF_BICG, 16.0 * n);
    launch_k(c, k_bi_rho, red_blocks(c, ws, n), kThreads, 0, n, st, rhat, r, ws.partials.get(),
                                                              ws.ticket.get());
    SDG_LAUNCHED(c);
}

void launch_bi_x_alpha(Context& c, int64_t n, BiState* st, const double* phat, double* x) {
    ProfScope ps_(c, PF_BICG, 24.0 * n);
    launch_k(c, k_bi_x_alpha, stride_blocks(c, n), kThreads, 0, n, st, phat, x);
    SDG_LAUNCHED(c);
}

void DevCsr::build_sell(const HostCsr& h, cudaStream_t s) {
    const int n = h.n_rows;
    const int ns = (n + 31) / 32;
    std::vector<int> off(ns + 1, 0), len(n);
    for (int sl = 0; sl < ns; ++sl) {
        int w = 0;
        for (int i = 32 * sl; i < std::min(n, 32 * sl + 32); ++i) {
            len[i] = h.rp[i + 1] - h.rp[i];
            w = std::max(w, len[i]);
        }
        if (static_cast<int64_t>(off[sl]) + 32LL * w >= (1LL << 31)) fail(SDG_EINVAL, "sell: too many entries");
        off[sl + 1] = off[sl] + 32 * w;
    }
    std::vector<double> v(off[ns], 0.0);
    std::vector<int> c(off[ns], 0);
    for (int i = 0; i < n; ++i)
        for (int k = h.rp[i]; k < h.rp[i + 1]; ++k) {
            const size_t q = static_cast<size_t>(off[i / 32]) + 32 * (k - h.rp[i]) + (i % 32);
            v[q] = h.v[k];
            c[q] = h.ci[k];
        }
    sell_off.upload(off, s);
    sell_len.upload(len, s);
    sell_v.upload(v, s);
    sell_ci.upload(c, s);
    sell_entries = off[ns];
    SDG_CUDA(cudaStreamSynchronize(s));  // host staging vectors die here
    sell = true;
}

}  // namespace sdg
