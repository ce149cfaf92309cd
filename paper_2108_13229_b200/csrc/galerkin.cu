// Device Galerkin product of the aggregation hierarchy (galerkin_product,
// precond.cpp:177-185): A_c = P^T A P for the piecewise-constant prolongation
// of an aggregation, A_c(c, c') = sum of a_ik over fine entries with
// agg[i] = c, agg[col_k] = c'.  The reference builds it through its
// CooBuilder (stable sort, duplicates summed in insertion order: fine rows
// ascending, row entries ascending); one thread per coarse row walks its
// aggregate's fine rows in that order and keeps the row's distinct coarse
// columns in a small local table, so every sum runs in the reference's order
// and the result is bitwise the host product (setup.cpp galerkin).
#include <algorithm>

#include "launch.cuh"
#include "setup.hpp"
#include "solver.hpp"

namespace sdg {

namespace {

constexpr int kGalCap = 128;  // distinct coarse columns per coarse row the kernels hold

// FILL = false: counts the distinct columns of every coarse row (cnt[c], or
// kGalCap + 1 on overflow); FILL = true: writes columns (ascending) and values
template <bool FILL>
__global__ void k_galerkin(int nc, const int* __restrict__ pt_ptr, const int* __restrict__ pt_rows,
                           const int* __restrict__ rp, const int* __restrict__ ci, const double* __restrict__ v,
                           const int* __restrict__ agg, int* __restrict__ cnt, const int* __restrict__ crp,
                           int* __restrict__ cci, double* __restrict__ cv) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= nc) return;
    int cols[kGalCap];
    double acc[kGalCap];
    int m = 0;
    bool overflow = false;
    for (int q = pt_ptr[c]; q < pt_ptr[c + 1]; ++q) {
        const int i = pt_rows[q];
        for (int k = rp[i]; k < rp[i + 1]; ++k) {
            const int cc = agg[ci[k]];
            int at = -1;
            for (int e = 0; e < m; ++e)
                if (cols[e] == cc) at = e;
            if (at < 0) {
                if (m == kGalCap) {
                    overflow = true;
                    continue;
                }
                at = m++;
                cols[at] = cc;
                acc[at] = 0.0;
            }
            if (FILL) acc[at] = __dadd_rn(acc[at], v[k]);
        }
    }
    if (!FILL) {
        cnt[c] = overflow ? kGalCap + 1 : m;
        return;
    }
    // ascending columns (insertion sort of the small table)
    for (int e = 1; e < m; ++e) {
        const int kc = cols[e];
        const double kv = acc[e];
        int f = e - 1;
        while (f >= 0 && cols[f] > kc) {
            cols[f + 1] = cols[f];
            acc[f + 1] = acc[f];
            --f;
        }
        cols[f + 1] = kc;
        acc[f + 1] = kv;
    }
    const int base = crp[c];
    for (int e = 0; e < m; ++e) {
        cci[base + e] = cols[e];
        cv[base + e] = acc[e];
    }
}

}  // namespace

// The coarse matrix of `a` under `agg` (n_coarse aggregates), computed on the
// device and returned on the host (the next aggregation pass runs there).
// Falls back to the host product when a coarse row has more than kGalCap
// distinct columns.
HostCsr galerkin_device(Context& cx, const HostCsr& a, const std::vector<int>& agg, int n_coarse) {
    if (n_coarse == 0 || a.nnz() == 0) return galerkin(a, agg, n_coarse);
    std::vector<int> ptr, rows;
    aggregate_transpose(agg, n_coarse, ptr, rows);
    DevCsr da;
    da.upload(a, cx.stream);
    DevBuf<int> d_agg, d_ptr, d_rows, d_cnt(n_coarse);
    d_agg.upload(agg, cx.stream);
    d_ptr.upload(ptr, cx.stream);
    d_rows.upload(rows, cx.stream);
    const int grid = (n_coarse + 127) / 128;
    k_galerkin<false><<<grid, 128, 0, cx.stream>>>(n_coarse, d_ptr.get(), d_rows.get(), da.rp.get(), da.ci.get(),
                                                   da.v.get(), d_agg.get(), d_cnt.get(), nullptr, nullptr, nullptr);
    cx.count();
    std::vector<int> cnt(n_coarse);
    SDG_CUDA(cudaMemcpyAsync(cnt.data(), d_cnt.get(), sizeof(int) * n_coarse, cudaMemcpyDeviceToHost, cx.stream));
    cx.sync();
    HostCsr c(n_coarse, n_coarse);
    for (int i = 0; i < n_coarse; ++i) {
        if (cnt[i] > kGalCap) return galerkin(a, agg, n_coarse);
        c.rp[i + 1] = c.rp[i] + cnt[i];
    }
    const int nnz = c.rp[n_coarse];
    DevBuf<int> d_crp, d_cci(std::max(nnz, 1));
    DevBuf<double> d_cv(std::max(nnz, 1));
    d_crp.upload(c.rp, cx.stream);
    k_galerkin<true><<<grid, 128, 0, cx.stream>>>(n_coarse, d_ptr.get(), d_rows.get(), da.rp.get(), da.ci.get(),
                                                  da.v.get(), d_agg.get(), nullptr, d_crp.get(), d_cci.get(), d_cv.get());
    cx.count();
    c.ci.resize(nnz);
    c.v.resize(nnz);
    SDG_CUDA(cudaMemcpyAsync(c.ci.data(), d_cci.get(), sizeof(int) * nnz, cudaMemcpyDeviceToHost, cx.stream));
    SDG_CUDA(cudaMemcpyAsync(c.v.data(), d_cv.get(), sizeof(double) * nnz, cudaMemcpyDeviceToHost, cx.stream));
    cx.sync();
    {
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) fail(SDG_ECUDA, std::string("galerkin_device: ") + cudaGetErrorString(e));
    }
    return c;
}

}  // namespace sdg
