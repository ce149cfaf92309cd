// Ordered CSR row sums with the row's loads issued up front.
//
// Thread-per-row kernels over short rows (5-20 entries) are bound by the
// chain  ci[k] -> x[ci[k]]  when each entry's loads wait for the previous
// entry's add.  Here the column indices and values of C entries are loaded
// together (predicated), then their C gathers, and only then are they folded,
// in column order, by the caller's functor: one round trip per C entries, and
// the same arithmetic sequence as the plain loop.
#pragma once

namespace sdg {

// f(a_k, x_{ci[k]}) for k = k0 .. k1-1 in order; xg(j) returns the gathered
// value for column j (a plain x[j], or e.g. z[j] + zc[agg[j]]).
template <int C, typename G, typename F>
__device__ __forceinline__ void row_fold(const int* __restrict__ ci, const double* __restrict__ v, int k0, int k1,
                                         G&& xg, F&& f) {
    for (int k = k0; k < k1; k += C) {
        int c[C];
        double a[C], xv[C];
#pragma unroll
        for (int j = 0; j < C; ++j) {
            const bool ok = k + j < k1;
            c[j] = ok ? __ldg(ci + k + j) : 0;
            a[j] = ok ? __ldg(v + k + j) : 0.0;
        }
#pragma unroll
        for (int j = 0; j < C; ++j) xv[j] = k + j < k1 ? xg(c[j]) : 0.0;
#pragma unroll
        for (int j = 0; j < C; ++j)
            if (k + j < k1) f(a[j], xv[j]);
    }
}

}  // namespace sdg
