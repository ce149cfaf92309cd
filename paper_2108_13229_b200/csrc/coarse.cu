// Device side of the coarse direct solve (coarse.hpp): batched Gauss-Jordan
// inversion, the setup of the nested-dissection blocks and the solve phases.
#include <algorithm>
#include <cstdlib>
#include <string>

#include "coarse.hpp"
#include "kernels.cuh"
#include "launch.cuh"

namespace sdg {

namespace {

#define SDG_CHECK_LAUNCH(ctx)                                                                    \
    do {                                                                                         \
        (ctx).count();                                                                           \
        cudaError_t e_ = cudaGetLastError();                                                     \
        if (e_ != cudaSuccess) ::sdg::fail(SDG_ECUDA, std::string(__func__) + ": " + cudaGetErrorString(e_)); \
    } while (0)

// ---------------------------------------------------------------------------
// batched in-place Gauss-Jordan with partial pivoting.  Step k of every
// matrix of the batch: k_gj_pivot picks the pivot row p (largest |a_ik|,
// i >= k, lowest i on ties) and saves what the update overwrites -- the
// scaled pivot row, the old row k and column k after the swap -- and
// k_gj_elim updates the whole matrix from those copies, so no thread reads
// an element another one writes.  After the last step the column swaps are
// undone in reverse order (k_gj_colfix).

struct GjDev {
    double* a;
    int n;
};

constexpr int kGjThreads = 256;

__global__ void __launch_bounds__(kGjThreads)
k_gj_pivot(const GjDev* __restrict__ items, int k, int ld, double* __restrict__ rowbuf, double* __restrict__ rowold,
           double* __restrict__ colbuf, int* __restrict__ piv, int* __restrict__ singular) {
    pdl_begin();
    const GjDev it = items[blockIdx.x];
    const int n = it.n;
    if (k >= n) return;
    const double* a = it.a;
    __shared__ double sv[kGjThreads / 32];
    __shared__ int si[kGjThreads / 32];
    __shared__ int sp;
    double best = -1.0;
    int bi = k;
    for (int i = k + threadIdx.x; i < n; i += blockDim.x) {
        const double v = fabs(a[static_cast<size_t>(i) * n + k]);
        if (v > best) {
            best = v;
            bi = i;
        }
    }
    for (int o = 16; o; o >>= 1) {
        const double ov = __shfl_down_sync(0xffffffffu, best, o);
        const int oi = __shfl_down_sync(0xffffffffu, bi, o);
        if (ov > best || (ov == best && oi < bi)) {
            best = ov;
            bi = oi;
        }
    }
    if ((threadIdx.x & 31) == 0) {
        sv[threadIdx.x >> 5] = best;
        si[threadIdx.x >> 5] = bi;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < kGjThreads / 32; ++w)
            if (sv[w] > best || (sv[w] == best && si[w] < bi)) {
                best = sv[w];
                bi = si[w];
            }
        sp = bi;
        piv[static_cast<size_t>(blockIdx.x) * ld + k] = bi;
        if (!(best > 0.0)) singular[blockIdx.x] = 1;
    }
    __syncthreads();
    const int p = sp;
    double d = a[static_cast<size_t>(p) * n + k];
    if (d == 0.0) d = 1.0;  // flagged above; keep the arithmetic finite
    double* rb = rowbuf + static_cast<size_t>(blockIdx.x) * ld;
    double* ro = rowold + static_cast<size_t>(blockIdx.x) * ld;
    double* cb = colbuf + static_cast<size_t>(blockIdx.x) * ld;
    const double akk = a[static_cast<size_t>(k) * n + k];
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
        ro[j] = a[static_cast<size_t>(k) * n + j];
        rb[j] = j == k ? 1.0 / d : a[static_cast<size_t>(p) * n + j] / d;
        cb[j] = j == p ? akk : a[static_cast<size_t>(j) * n + k];
    }
}

// tile of 64 columns x 32 rows per block
__global__ void __launch_bounds__(kGjThreads)
k_gj_elim(const GjDev* __restrict__ items, int k, int ld, const double* __restrict__ rowbuf,
          const double* __restrict__ rowold, const double* __restrict__ colbuf, const int* __restrict__ piv) {
    pdl_begin();
    const int b = blockIdx.z;
    const GjDev it = items[b];
    const int n = it.n;
    if (k >= n) return;
    const int j = blockIdx.x * 64 + (threadIdx.x & 63);
    const int i0 = blockIdx.y * 32 + (threadIdx.x >> 6) * 8;
    if (j >= n || i0 >= n) return;
    const size_t off = static_cast<size_t>(b) * ld;
    const int p = piv[off + k];
    const double rj = rowbuf[off + j];
    const double oj = rowold[off + j];
#pragma unroll
    for (int r = 0; r < 8; ++r) {
        const int i = i0 + r;
        if (i >= n) break;
        double* e = it.a + static_cast<size_t>(i) * n + j;
        if (i == k) {
            *e = rj;
            continue;
        }
        double src = i == p ? oj : *e;
        if (j == k) src = 0.0;
        *e = fma(-colbuf[off + i], rj, src);
    }
}

__global__ void k_gj_colfix(const GjDev* __restrict__ items, int ld, const int* __restrict__ cperm) {
    extern __shared__ double row[];
    const GjDev it = items[blockIdx.y];
    const int n = it.n;
    const int i = blockIdx.x;
    if (i >= n) return;
    double* a = it.a + static_cast<size_t>(i) * n;
    for (int j = threadIdx.x; j < n; j += blockDim.x) row[j] = a[j];
    __syncthreads();
    const int* c = cperm + static_cast<size_t>(blockIdx.y) * ld;
    for (int j = threadIdx.x; j < n; j += blockDim.x) a[j] = row[c[j]];
}

// ---------------------------------------------------------------------------
// setup kernels of the nested-dissection blocks (P A P^T in CSR: rp, ci, v)

// dense copies of the leaves' diagonal blocks into the (zeroed) pool
__global__ void k_nd_densify_leaves(int n, const NdNodeDev* __restrict__ nodes, const int* __restrict__ leaf_of,
                                    const int* __restrict__ rp, const int* __restrict__ ci,
                                    const double* __restrict__ v, double* __restrict__ pool) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int id = leaf_of[i];
    if (id < 0) return;
    const NdNodeDev nd = nodes[id];
    const int nl = nd.hi - nd.lo;
    double* row = pool + nd.inv + static_cast<long long>(i - nd.lo) * nl;
    for (int k = rp[i]; k < rp[i + 1]; ++k) {
        const int j = ci[k];
        if (j >= nd.lo && j < nd.hi) row[j - nd.lo] = v[k];
    }
}

// right-hand sides A_IS of the internal nodes of one depth, column-major n x m (zeroed before)
__global__ void k_nd_fill_rhs(int n, const NdNodeDev* __restrict__ nodes, const int* __restrict__ node_of,
                              const int* __restrict__ rp, const int* __restrict__ ci, const double* __restrict__ v,
                              double* __restrict__ x) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int id = node_of[i];
    if (id < 0) return;
    const NdNodeDev nd = nodes[id];
    for (int k = rp[i]; k < rp[i + 1]; ++k) {
        const int j = ci[k];
        if (j >= nd.mid && j < nd.hi) x[static_cast<size_t>(j - nd.mid) * n + i] = v[k];
    }
}

// W of the nodes of one depth out of the solved right-hand sides (row-major |I| x |S| per node)
__global__ void k_nd_store_w(int n, const NdNodeDev* __restrict__ nodes, const int* __restrict__ node_of,
                             const double* __restrict__ y, double* __restrict__ pool) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int c = blockIdx.y;
    if (i >= n) return;
    const int id = node_of[i];
    if (id < 0) return;
    const NdNodeDev nd = nodes[id];
    const int ns = nd.hi - nd.mid;
    if (c < ns) pool[nd.w + static_cast<long long>(i - nd.lo) * ns + c] = y[static_cast<size_t>(c) * n + i];
}

// Sc = A_SS - A_SI W per node of one depth, into the node's inverse slot
__global__ void k_nd_schur(const int* __restrict__ ids, const NdNodeDev* __restrict__ nodes,
                           const int* __restrict__ rp, const int* __restrict__ ci, const double* __restrict__ v,
                           double* __restrict__ pool) {
    const NdNodeDev nd = nodes[ids[blockIdx.x]];
    const int ns = nd.hi - nd.mid;
    const long long total = static_cast<long long>(ns) * ns;
    const double* w = pool + nd.w;
    for (long long e = blockIdx.y * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<long long>(gridDim.y) * blockDim.x) {
        const int s = static_cast<int>(e / ns), c = static_cast<int>(e % ns);
        const int row = nd.mid + s;
        double acc = 0.0;
        for (int k = rp[row]; k < rp[row + 1]; ++k) {
            const int j = ci[k];
            if (j >= nd.mid && j < nd.hi) {
                if (j - nd.mid == c) acc += v[k];
            } else if (j >= nd.lo && j < nd.mid) {
                acc = fma(-v[k], w[static_cast<long long>(j - nd.lo) * ns + c], acc);
            }
        }
        pool[nd.inv + e] = acc;
    }
}

// ---------------------------------------------------------------------------
// solve phases.  u: right-hand side(s), y: work / solution in the new
// numbering, both column-major with leading dimension ld; blockIdx.y is the
// column.  perm != nullptr: u (and xout) are in the original numbering.

constexpr int kNdThreads = 256;

__device__ __forceinline__ double warp_sum(double a) {
#pragma unroll
    for (int o = 16; o; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    return a;
}

// leaves: y_L = inv(A_LL) u_L, one warp per row
__global__ void __launch_bounds__(kNdThreads)
k_nd_leaf(int n, const NdNodeDev* __restrict__ nodes, const int* __restrict__ leaf_of,
          const double* __restrict__ pool, const double* __restrict__ u, const int* __restrict__ perm,
          double* __restrict__ y, long long ld) {
    pdl_begin();
    const int row = blockIdx.x * (kNdThreads / 32) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (row >= n) return;
    const int id = leaf_of[row];
    if (id < 0) return;
    const NdNodeDev nd = nodes[id];
    const int nl = nd.hi - nd.lo;
    const double* __restrict__ m = pool + nd.inv + static_cast<long long>(row - nd.lo) * nl;
    const double* __restrict__ uc = u + blockIdx.y * ld;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    int c = lane;
    if (perm) {
        const int* __restrict__ pc = perm + nd.lo;
        for (; c + 96 < nl; c += 128) {
            const double m0 = __ldcs(m + c), m1 = __ldcs(m + c + 32), m2 = __ldcs(m + c + 64), m3 = __ldcs(m + c + 96);
            a0 = fma(m0, uc[pc[c]], a0);
            a1 = fma(m1, uc[pc[c + 32]], a1);
            a2 = fma(m2, uc[pc[c + 64]], a2);
            a3 = fma(m3, uc[pc[c + 96]], a3);
        }
        for (; c < nl; c += 32) a0 = fma(__ldcs(m + c), uc[pc[c]], a0);
    } else {
        const double* __restrict__ ul = uc + nd.lo;
        for (; c + 96 < nl; c += 128) {
            const double m0 = m[c], m1 = m[c + 32], m2 = m[c + 64], m3 = m[c + 96];
            a0 = fma(m0, ul[c], a0);
            a1 = fma(m1, ul[c + 32], a1);
            a2 = fma(m2, ul[c + 64], a2);
            a3 = fma(m3, ul[c + 96], a3);
        }
        for (; c < nl; c += 32) a0 = fma(m[c], ul[c], a0);
    }
    const double s = warp_sum((a0 + a1) + (a2 + a3));
    if (lane == 0) y[blockIdx.y * ld + row] = s;
}

// separators of one depth: t = u_S - A_SI y_I (every part computes all of t),
// then x_S = inv(Sc) t for the part's rows.  blockIdx.x = node * parts + part.
__global__ void __launch_bounds__(1024)
k_nd_sep(const int* __restrict__ ids, int parts, const NdNodeDev* __restrict__ nodes, const int* __restrict__ rp,
         const int* __restrict__ ci, const double* __restrict__ v, const double* __restrict__ pool,
         const double* __restrict__ u, const int* __restrict__ perm, double* __restrict__ y, long long ld,
         double* __restrict__ xout) {
    extern __shared__ double t[];
    pdl_begin();
    const NdNodeDev nd = nodes[ids[blockIdx.x / parts]];
    const int part = blockIdx.x % parts;
    const int ns = nd.hi - nd.mid;
    const double* __restrict__ uc = u + blockIdx.y * ld;
    double* __restrict__ yc = y + blockIdx.y * ld;
    // eight lanes per separator row: the row's entries are loaded side by side
    // (a thread per row would chain one L2 round trip per entry)
    const int sub = threadIdx.x & 7, grp = threadIdx.x >> 3, ngrp = blockDim.x >> 3;
    for (int s0 = 0; s0 < ns; s0 += ngrp) {
        const int s = s0 + grp;
        const bool valid = s < ns;
        const int row = nd.mid + (valid ? s : 0);
        double acc = 0.0;
        if (valid) {
            const int ke = rp[row + 1];
            for (int k = rp[row] + sub; k < ke; k += 8) {
                const int j = ci[k];
                if (j >= nd.lo && j < nd.mid) acc = fma(-v[k], yc[j], acc);
            }
        }
        acc += __shfl_xor_sync(0xffffffffu, acc, 4);
        acc += __shfl_xor_sync(0xffffffffu, acc, 2);
        acc += __shfl_xor_sync(0xffffffffu, acc, 1);
        if (valid && sub == 0) t[s] = (perm ? uc[perm[row]] : uc[row]) + acc;
    }
    __syncthreads();
    const int per = (ns + parts - 1) / parts;
    const int r_end = min(ns, (part + 1) * per);
    const int lane = threadIdx.x & 31;
    const double* __restrict__ inv = pool + nd.inv;
    for (int r = part * per + (threadIdx.x >> 5); r < r_end; r += blockDim.x >> 5) {
        const double* __restrict__ m = inv + static_cast<long long>(r) * ns;
        double a0 = 0.0, a1 = 0.0;
        int c = lane;
        for (; c + 32 < ns; c += 64) {
            a0 = fma(m[c], t[c], a0);
            a1 = fma(m[c + 32], t[c + 32], a1);
        }
        if (c < ns) a0 = fma(m[c], t[c], a0);
        const double s = warp_sum(a0 + a1);
        if (lane == 0) {
            yc[nd.mid + r] = s;
            if (xout) xout[perm[nd.mid + r]] = s;
        }
    }
}

// interiors of one depth: y_I -= W x_S, one warp per row
__global__ void __launch_bounds__(kNdThreads)
k_nd_down(int n, const NdNodeDev* __restrict__ nodes, const int* __restrict__ node_of,
          const double* __restrict__ pool, const int* __restrict__ perm, double* __restrict__ y, long long ld,
          double* __restrict__ xout) {
    pdl_begin();
    const int row = blockIdx.x * (kNdThreads / 32) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (row >= n) return;
    const int id = node_of[row];
    if (id < 0) return;
    const NdNodeDev nd = nodes[id];
    const int ns = nd.hi - nd.mid;
    const double* __restrict__ w = pool + nd.w + static_cast<long long>(row - nd.lo) * ns;
    double* __restrict__ yc = y + blockIdx.y * ld;
    const double* __restrict__ xs = yc + nd.mid;
    double a0 = 0.0, a1 = 0.0;
    int c = lane;
    for (; c + 32 < ns; c += 64) {
        const double w0 = __ldcs(w + c), w1 = __ldcs(w + c + 32);
        a0 = fma(w0, xs[c], a0);
        a1 = fma(w1, xs[c + 32], a1);
    }
    if (c < ns) a0 = fma(__ldcs(w + c), xs[c], a0);
    const double s = warp_sum(a0 + a1);
    if (lane == 0) {
        const double val = yc[row] - s;
        yc[row] = val;
        if (xout) xout[perm[row]] = val;
    }
}

// x[perm[i]] = y[i]: only when the root has no separator (disconnected halves)
__global__ void k_nd_scatter(int n, const int* __restrict__ perm, const double* __restrict__ y,
                             double* __restrict__ xout) {
    pdl_begin();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) xout[perm[i]] = y[i];
}

int env_int(const char* name, int dflt) {
    const char* e = std::getenv(name);
    return e && *e ? std::atoi(e) : dflt;
}

}  // namespace

// ---------------------------------------------------------------------------

void batched_inverse(Context& cx, const std::vector<GjItem>& items, const char* what) {
    std::vector<GjDev> host;
    int nmax = 0;
    for (const auto& it : items)
        if (it.n > 0) {
            host.push_back({it.a, it.n});
            nmax = std::max(nmax, it.n);
        }
    const int nb = static_cast<int>(host.size());
    if (nb == 0) return;
    if (nb > 65535) fail(SDG_EINVAL, "batched_inverse: too many blocks in one batch");
    if (static_cast<size_t>(nmax) * 8 > 220 * 1024)
        fail(SDG_ENOMEM, std::string(what) + ": dense block of " + std::to_string(nmax) + " rows is too large to invert");
    DevBuf<GjDev> dev(nb);
    SDG_CUDA(cudaMemcpyAsync(dev.get(), host.data(), sizeof(GjDev) * nb, cudaMemcpyHostToDevice, cx.stream));
    const size_t ld = nmax;
    DevBuf<double> rowbuf(nb * ld), rowold(nb * ld), colbuf(nb * ld);
    DevBuf<int> piv(nb * ld), sing(nb), cperm(nb * ld);
    SDG_CUDA(cudaMemsetAsync(sing.get(), 0, sizeof(int) * nb, cx.stream));
    const dim3 egrid((nmax + 63) / 64, (nmax + 31) / 32, nb);
    for (int k = 0; k < nmax; ++k) {
        launch_k(cx, k_gj_pivot, nb, kGjThreads, 0, dev.get(), k, nmax, rowbuf.get(), rowold.get(), colbuf.get(),
                 piv.get(), sing.get());
        launch_k(cx, k_gj_elim, egrid, kGjThreads, 0, dev.get(), k, nmax, rowbuf.get(), rowold.get(), colbuf.get(),
                 piv.get());
        cx.count(2);
    }
    std::vector<int> hsing(nb), hpiv(nb * ld);
    SDG_CUDA(cudaMemcpyAsync(hsing.data(), sing.get(), sizeof(int) * nb, cudaMemcpyDeviceToHost, cx.stream));
    SDG_CUDA(cudaMemcpyAsync(hpiv.data(), piv.get(), sizeof(int) * nb * ld, cudaMemcpyDeviceToHost, cx.stream));
    cx.sync();
    {
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) fail(SDG_ECUDA, std::string("batched_inverse: ") + cudaGetErrorString(e));
    }
    for (int b = 0; b < nb; ++b)
        if (hsing[b]) fail(SDG_ESINGULAR, std::string(what) + ": matrix is singular, zero pivot column");
    // undo the row exchanges on the columns, last exchange first
    std::vector<int> hc(nb * ld, 0);
    for (int b = 0; b < nb; ++b) {
        int* c = hc.data() + b * ld;
        const int* p = hpiv.data() + b * ld;
        const int n = host[b].n;
        for (int j = 0; j < n; ++j) c[j] = j;
        for (int k = n - 1; k >= 0; --k) std::swap(c[k], c[p[k]]);
    }
    SDG_CUDA(cudaMemcpyAsync(cperm.get(), hc.data(), sizeof(int) * nb * ld, cudaMemcpyHostToDevice, cx.stream));
    static const bool attr = [] {
        SDG_CUDA(cudaFuncSetAttribute(k_gj_colfix, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
        return true;
    }();
    (void)attr;
    k_gj_colfix<<<dim3(nmax, nb), 256, static_cast<size_t>(nmax) * 8, cx.stream>>>(dev.get(), nmax, cperm.get());
    SDG_CHECK_LAUNCH(cx);
    cx.sync();
}

void CoarseSolver::build(Context& cx, const HostCsr& a) {
    if (a.n_rows != a.n_cols) fail(SDG_EDIM, "lu_factor: matrix must be square");
    n_ = a.n_rows;
    pool_.release();
    if (n_ == 0) return;
    const char* mode = std::getenv("SDG_COARSE");
    const bool force_dense = mode && mode[0] == 'd';
    const bool force_nd = mode && mode[0] == 'n';
    if (!force_dense && (n_ >= kNdMinRows || force_nd)) {
        try {
            build_nd(cx, a);
            if (!dense_) return;
        } catch (const Error& e) {
            if (e.code != SDG_ESINGULAR) throw;
            // a singular diagonal block of a regular (indefinite) matrix: pivot over the whole matrix instead
        }
    }
    build_dense(cx, a);
}

void CoarseSolver::build_dense(Context& cx, const HostCsr& a) {
    dense_ = true;
    tree_ = NdTree{};
    const size_t nn = static_cast<size_t>(n_) * n_;
    DevCsr dc;
    dc.upload(a, cx.stream);
    pool_.resize(nn);
    SDG_CUDA(cudaMemsetAsync(pool_.get(), 0, nn * sizeof(double), cx.stream));
    launch_csr_to_dense(cx, dc, pool_.get());
    batched_inverse(cx, {{pool_.get(), n_}}, "lu_factor");
}

void CoarseSolver::build_nd(Context& cx, const HostCsr& a) {
    const int leaf_rows = std::max(32, env_int("SDG_ND_LEAF", kNdLeafRows));
    tree_ = nd_order(a, leaf_rows, 24);
    if (tree_.nodes.size() == 1) {  // nothing to split
        dense_ = true;
        return;
    }
    dense_ = false;
    const int n = n_;
    const int depths = tree_.max_depth;  // internal nodes live at depths 0 .. max_depth - 1
    // pool layout + per-depth tables
    std::vector<NdNodeDev> hn(tree_.nodes.size());
    std::vector<int> leaf_of(n, -1);
    std::vector<std::vector<int>> node_of(depths, std::vector<int>(n, -1)), ids(depths);
    long long off = 0;
    max_s_.assign(depths, 0);
    bytes_sep_.assign(depths, 0.0);
    bytes_down_.assign(depths, 0.0);
    bytes_leaf_ = 0;
    for (size_t id = 0; id < tree_.nodes.size(); ++id) {
        const NdNode& nd = tree_.nodes[id];
        NdNodeDev& d = hn[id];
        d.lo = nd.lo;
        d.mid = nd.mid;
        d.hi = nd.hi;
        d.pad = 0;
        d.inv = off;
        d.w = 0;
        if (nd.leaf()) {
            const long long nl = nd.hi - nd.lo;
            off += nl * nl;
            bytes_leaf_ += 8.0 * nl * nl + 24.0 * nl;
            for (int i = nd.lo; i < nd.hi; ++i) leaf_of[i] = static_cast<int>(id);
        } else {
            const long long ni = nd.mid - nd.lo, ns = nd.hi - nd.mid;
            off += ns * ns;
            d.w = off;
            off += ni * ns;
            ids[nd.depth].push_back(static_cast<int>(id));
            max_s_[nd.depth] = std::max<int>(max_s_[nd.depth], static_cast<int>(ns));
            bytes_sep_[nd.depth] += 8.0 * ns * ns + 40.0 * ns;
            bytes_down_[nd.depth] += 8.0 * ni * ns + 16.0 * ni;
            for (int i = nd.lo; i < nd.mid; ++i) node_of[nd.depth][i] = static_cast<int>(id);
        }
    }
    const HostCsr ap = permute_symmetric(a, tree_.perm);
    ap_.upload(ap, cx.stream);
    nodes_.resize(hn.size());
    SDG_CUDA(cudaMemcpyAsync(nodes_.get(), hn.data(), sizeof(NdNodeDev) * hn.size(), cudaMemcpyHostToDevice, cx.stream));
    perm_.upload(tree_.perm, cx.stream);
    leaf_of_.upload(leaf_of, cx.stream);
    node_of_.clear();
    node_of_.resize(depths);
    ids_.clear();
    ids_.resize(depths);
    n_ids_.assign(depths, 0);
    for (int d = 0; d < depths; ++d) {
        node_of_[d].upload(node_of[d], cx.stream);
        n_ids_[d] = static_cast<int>(ids[d].size());
        if (n_ids_[d]) ids_[d].upload(ids[d], cx.stream);
    }
    pool_.resize(static_cast<size_t>(off));
    SDG_CUDA(cudaMemsetAsync(pool_.get(), 0, static_cast<size_t>(off) * sizeof(double), cx.stream));
    y_.resize(n);
    cx.sync();  // the host staging vectors above go out of scope below

    // leaves
    k_nd_densify_leaves<<<(n + 255) / 256, 256, 0, cx.stream>>>(n, nodes_.get(), leaf_of_.get(), ap_.rp.get(),
                                                                 ap_.ci.get(), ap_.v.get(), pool_.get());
    SDG_CHECK_LAUNCH(cx);
    std::vector<GjItem> batch;
    for (size_t id = 0; id < tree_.nodes.size(); ++id)
        if (tree_.nodes[id].leaf()) batch.push_back({pool_.get() + hn[id].inv, tree_.nodes[id].hi - tree_.nodes[id].lo});
    batched_inverse(cx, batch, "coarse solve (leaf block)");

    // internal nodes, deepest first: W = inv(A_II) A_IS through the phases below, then Sc and its inverse
    for (int d = depths - 1; d >= 0; --d) {
        if (!n_ids_[d]) continue;
        const int m = max_s_[d];
        if (m == 0) continue;  // empty separators (disconnected halves): nothing to store
        DevBuf<double> x(static_cast<size_t>(n) * m), y(static_cast<size_t>(n) * m);
        SDG_CUDA(cudaMemsetAsync(x.get(), 0, sizeof(double) * n * m, cx.stream));
        SDG_CUDA(cudaMemsetAsync(y.get(), 0, sizeof(double) * n * m, cx.stream));
        k_nd_fill_rhs<<<(n + 255) / 256, 256, 0, cx.stream>>>(n, nodes_.get(), node_of_[d].get(), ap_.rp.get(),
                                                               ap_.ci.get(), ap_.v.get(), x.get());
        SDG_CHECK_LAUNCH(cx);
        run_phases(cx, d, x.get(), nullptr, y.get(), nullptr, m);
        k_nd_store_w<<<dim3((n + 255) / 256, m), 256, 0, cx.stream>>>(n, nodes_.get(), node_of_[d].get(), y.get(),
                                                                       pool_.get());
        SDG_CHECK_LAUNCH(cx);
        const int chunks = std::max(1, std::min(64, (m * m + 4095) / 4096));
        k_nd_schur<<<dim3(n_ids_[d], chunks), 256, 0, cx.stream>>>(ids_[d].get(), nodes_.get(), ap_.rp.get(),
                                                                    ap_.ci.get(), ap_.v.get(), pool_.get());
        SDG_CHECK_LAUNCH(cx);
        batch.clear();
        for (int id : ids[d]) batch.push_back({pool_.get() + hn[id].inv, tree_.nodes[id].hi - tree_.nodes[id].mid});
        batched_inverse(cx, batch, "coarse solve (separator block)");
    }
    cx.sync();
}

void CoarseSolver::run_phases(Context& cx, int above, const double* u, const int* perm, double* y, double* xout,
                              int m) {
    const int n = n_;
    const long long ld = n;
    const int rows_per_block = kNdThreads / 32;
    const dim3 rgrid((n + rows_per_block - 1) / rows_per_block, m);
    static const bool attr = [] {
        SDG_CUDA(cudaFuncSetAttribute(k_nd_sep, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        return true;
    }();
    (void)attr;
    {
        ProfScope ps(cx, m == 1 ? PF_COARSE : PF_SETUP, bytes_leaf_);
        launch_k(cx, k_nd_leaf, rgrid, kNdThreads, 0, n, nodes_.get(), leaf_of_.get(), pool_.get(), u, perm, y, ld);
        SDG_CHECK_LAUNCH(cx);
    }
    bool wrote_out = false;
    for (int d = tree_.max_depth - 1; d > above; --d) {
        if (!n_ids_[d] || !max_s_[d]) continue;
        double* xo = d == 0 ? xout : nullptr;
        wrote_out = wrote_out || xo;
        const int parts = std::max(1, (max_s_[d] + 63) / 64);
        if (static_cast<size_t>(max_s_[d]) * 8 > 200 * 1024) fail(SDG_ENOMEM, "coarse solve: separator too wide");
        {
            ProfScope ps(cx, m == 1 ? PF_COARSE : PF_SETUP, bytes_sep_[d]);
            launch_k(cx, k_nd_sep, dim3(n_ids_[d] * parts, m), 1024, static_cast<size_t>(max_s_[d]) * 8, ids_[d].get(),
                     parts, nodes_.get(), ap_.rp.get(), ap_.ci.get(), ap_.v.get(), pool_.get(), u, perm, y, ld, xo);
            SDG_CHECK_LAUNCH(cx);
        }
        {
            ProfScope ps(cx, m == 1 ? PF_COARSE : PF_SETUP, bytes_down_[d]);
            launch_k(cx, k_nd_down, rgrid, kNdThreads, 0, n, nodes_.get(), node_of_[d].get(), pool_.get(), perm, y, ld,
                     xo);
            SDG_CHECK_LAUNCH(cx);
        }
    }
    if (xout && !wrote_out) {
        ProfScope ps(cx, PF_COARSE, 20.0 * n);
        launch_k(cx, k_nd_scatter, (n + 255) / 256, 256, 0, n, perm, static_cast<const double*>(y), xout);
        SDG_CHECK_LAUNCH(cx);
    }
}

void CoarseSolver::solve(Context& cx, const double* r, double* z) {
    if (n_ == 0) return;
    if (dense_) {
        launch_dense_gemv(cx, n_, pool_.get(), r, z);
        return;
    }
    run_phases(cx, -1, r, perm_.get(), y_.get(), z, 1);
}

}  // namespace sdg
