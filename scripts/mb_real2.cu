// Dev harness: the production single-CTA walk (plan + kernel) on a synthetic
// nx x nx 5-point lower triangle, timed with CUDA events.  Feature knock-outs
// with -DSDG_WALK_EXP=mask (see gs_walk.cu).
#define private public
#include "../paper_2108_13229_b200/csrc/gs_walk.cu"

#include <cmath>
#include <vector>

using namespace sdg;

int main(int argc, char** argv) {
    const int nx = argc > 1 ? atoi(argv[1]) : 160, n = nx * nx;
    HostCsr a(n, n);
    std::vector<double> dinv(n, 0.25);
    std::vector<int> nlow(n, 0);
    for (int j = 0; j < nx; ++j)
        for (int i = 0; i < nx; ++i) {
            const int r = j * nx + i;
            if (j > 0) { a.ci.push_back(r - nx); a.v.push_back(-1.0); nlow[r]++; }
            if (i > 0) { a.ci.push_back(r - 1); a.v.push_back(-1.0); nlow[r]++; }
            a.ci.push_back(r); a.v.push_back(4.0);
            a.rp[r + 1] = static_cast<int>(a.ci.size());
        }
    cudaStream_t s;
    cudaStreamCreate(&s);
    GsPlan g;
    if (!g.build_walk(a, dinv, nlow, 2, s)) { printf("plan failed\n"); return 1; }
    std::vector<int> bidx(n);
    cudaMemcpy(bidx.data(), g.bidx.get(), n * 4, cudaMemcpyDeviceToHost);
    std::vector<double> pk(g.packed.size());
    cudaMemcpy(pk.data(), g.packed.get(), pk.size() * 8, cudaMemcpyDeviceToHost);
    for (int i = 0; i < n; ++i) pk[bidx[i]] = 0.25 * (1.0 + 1e-3 * (i % 7));
    cudaMemcpy(g.packed.get(), pk.data(), pk.size() * 8, cudaMemcpyHostToDevice);
    double* z;
    cudaMalloc(&z, n * 8);
    WalkPair wa{};
    wa.a[0] = WalkArgs{g.meta.get(), g.walk_iss.get(), reinterpret_cast<const unsigned char*>(g.packed.get()),
                       g.n_levels, g.walk_chunks, g.ring, g.walk_meta_bytes, g.walk_chunk_bytes, g.walk_zbytes, z,
                       0, 0, 0, nullptr};
    const auto kern = walk_kernel(g.walk_r2, g.walk_r8, g.walk_kw);
    printf("plan: warps %d rows/thread %d+%d levels %d\n", g.nthreads / 32 - 1, g.walk_r2, g.walk_r8, g.n_levels);
    for (int r = 0; r < 3; ++r) kern<<<1, g.nthreads, g.smem, s>>>(wa);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, s);
    for (int r = 0; r < 20; ++r) kern<<<1, g.nthreads, g.smem, s>>>(wa);
    cudaEventRecord(e1, s);
    cudaError_t e = cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    std::vector<double> hz(n), zc(n);
    cudaMemcpy(hz.data(), z, n * 8, cudaMemcpyDeviceToHost);
    double maxd = 0;
    int nbad = 0, first_bad = -1;
    for (int i = 0; i < n; ++i) {
        double acc = 0.25 * (1.0 + 1e-3 * (i % 7));
        for (int k = a.rp[i]; k < a.rp[i + 1]; ++k)
            if (a.ci[k] < i) acc += 0.25 * zc[a.ci[k]];
        zc[i] = acc;
        maxd = std::max(maxd, std::abs(acc - hz[i]) / std::abs(acc));
        if (std::abs(acc - hz[i]) > 1e-12 * std::abs(acc)) {
            if (first_bad < 0) first_bad = i;
            if (nbad < 24) printf("bad row %d (%d,%d) got %.6f want %.6f\n", i, i % nx, i / nx, hz[i], acc);
            ++nbad;
        }
    }
    if (nbad) printf("mismatches %d first at row %d (got %g want %g)\n", nbad, first_bad, hz[first_bad], zc[first_bad]);
#ifdef SDG_WALK_TRACE
    {
        std::vector<long long> tr(1024 * 16 * 4);
        cudaMemcpyFromSymbol(tr.data(), g_walk_trace, tr.size() * 8);
        const int nw = g.nthreads / 32;
        std::vector<double> arr(nw, 0), solve(nw, 0), fetch(nw, 0), topoff(nw, 0), arroff(nw, 0);
        double rel = 0, spread = 0;
        int m = 0;
        for (int L = 5; L + 1 < g.n_levels && L < 1000; ++L, ++m) {
            long long amax = 0, amin = 1LL << 62, rmin = 1LL << 62;
            for (int w = 0; w < nw; ++w) {
                const long long* t = &tr[(L * 16 + w) * 4];
                const long long* tn = &tr[((L + 1) * 16 + w) * 4];
                amax = std::max(amax, t[2]);
                amin = std::min(amin, t[2]);
                rmin = std::min(rmin, tn[0]);
                arr[w] += t[2] - t[0];
                if (w > 0) { solve[w] += t[1] - t[0]; fetch[w] += t[2] - t[1]; }
            }
            long long tmin = 1LL << 62;
            for (int w = 0; w < nw; ++w) tmin = std::min(tmin, tr[(L * 16 + w) * 4]);
            for (int w = 0; w < nw; ++w) {
                topoff[w] += tr[(L * 16 + w) * 4] - tmin;
                arroff[w] += tr[(L * 16 + w) * 4 + 2] - tmin;
            }
            rel += rmin - amax;
            spread += amax - amin;
        }
        printf("per level: last arrival -> first release %.0f, arrival spread %.0f\n", rel / m, spread / m);
        for (int w = 0; w < nw; ++w)
            printf("  warp %d: top->arrive %.0f (solve %.0f fetch %.0f) top offset %.0f arrive offset %.0f\n", w,
                   arr[w] / m, solve[w] / m, fetch[w] / m, topoff[w] / m, arroff[w] / m);
    }
#endif
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("nx %d levels %d threads %d: %.2f us/launch, %.0f cycles/level, rel err %.1e (%s)\n",
           nx, g.n_levels, g.nthreads, ms / 20 * 1e3, ms / 20 * 1e-3 * clk * 1e3 / g.n_levels, maxd,
           cudaGetErrorString(e));
    return 0;
}
