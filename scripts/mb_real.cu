// Dev harness: the production k_gs_walk kernel on a synthetic nx x ny 5-point
// lower triangle (all rows K2), timed with its own per-level trace.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr
//      -Ipaper_2108_13229_b200/csrc -Iinclude scripts/mb_real.cu -o scripts/mb_real
#include "../paper_2108_13229_b200/csrc/gs_walk.cu"

#include <vector>

using namespace sdg;

int main(int argc, char** argv) {
    const int nx = argc > 1 ? atoi(argv[1]) : 160, ny = nx;
    const int dbg = argc > 2 ? atoi(argv[2]) : 0;
    const int nl = nx + ny - 1;
    std::vector<int> lptr(nl + 1, 0), pos(nx * ny);
    for (int j = 0; j < ny; ++j)
        for (int i = 0; i < nx; ++i) lptr[i + j + 1]++;
    for (int q = 0; q < nl; ++q) lptr[q + 1] += lptr[q];
    std::vector<int> fill(lptr.begin(), lptr.end() - 1);
    for (int j = 0; j < ny; ++j)
        for (int i = 0; i < nx; ++i) pos[j * nx + i] = fill[i + j]++;
    int ring = 64;
    while (ring < 3 * nx) ring <<= 1;
    const int zero = ring, dummy = ring + 1;
    std::vector<unsigned char> pk(static_cast<size_t>(nx) * ny * 48);
    std::vector<int4> meta(nl), iss(nl);
    const int R = 160 * 1024;
    int cur = 0;
    for (int q = 0; q < nl; ++q) {
        const int rows = lptr[q + 1] - lptr[q], sz = rows * 48;
        if (cur + sz > R) cur = 0;
        meta[q] = make_int4(cur, rows, 0, lptr[q]);
        iss[q] = make_int4(lptr[q] * 48 / 16, sz, 0, q < 6 ? -1 : q - 6);
        cur += sz;
    }
    for (int j = 0; j < ny; ++j)
        for (int i = 0; i < nx; ++i) {
            const int p = pos[j * nx + i];
            unsigned char* rec = pk.data() + static_cast<size_t>(p) * 48;
            double* d = reinterpret_cast<double*>(rec);
            int* n = reinterpret_cast<int*>(rec);
            d[0] = 1.0;
            n[2] = j * nx + i;
            n[3] = dummy;
            d[2] = i > 0 ? -0.25 : 0.0;
            d[3] = j > 0 ? -0.25 : 0.0;
            n[8] = i > 0 ? (pos[j * nx + i - 1] & (ring - 1)) : zero;
            n[9] = j > 0 ? (pos[(j - 1) * nx + i] & (ring - 1)) : zero;
        }
    int4 *dm, *di;
    unsigned char* dp;
    double* z;
    long long* tr;
    cudaMalloc(&dm, nl * 16);
    cudaMalloc(&di, nl * 16);
    cudaMalloc(&dp, pk.size());
    cudaMalloc(&z, nx * ny * 8);
    cudaMalloc(&tr, nl * 8);
    cudaMemcpy(dm, meta.data(), nl * 16, cudaMemcpyHostToDevice);
    cudaMemcpy(di, iss.data(), nl * 16, cudaMemcpyHostToDevice);
    cudaMemcpy(dp, pk.data(), pk.size(), cudaMemcpyHostToDevice);
    const int tab = (nl * 16 + 15) / 16 * 16, zb = ((ring + 2) * 8 + 15) / 16 * 16;
    const size_t smem = 32 * 8 + 2 * tab + zb + R;
    cudaFuncSetAttribute(k_gs_walk, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    WalkArgs a{dm, di, dp, nl, ring, tab, zb, z, tr, dbg};
    const int threads = 32 + (nx + 31) / 32 * 32;
    for (int r = 0; r < 3; ++r) k_gs_walk<<<1, threads, smem>>>(a);
    cudaError_t e = cudaDeviceSynchronize();
    {
        WalkArgs b = a;
        b.trace = nullptr;
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        k_gs_walk<<<1, threads, smem>>>(b);
        cudaEventRecord(e0);
        for (int r = 0; r < 10; ++r) k_gs_walk<<<1, threads, smem>>>(b);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        int clk;
        cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
        printf("no-trace: %.2f us per launch, %.1f cycles/level at %d MHz\n", ms * 100, ms / 10 * 1e-3 * clk * 1e3 / nl,
               clk / 1000);
    }
    std::vector<long long> h(nl);
    cudaMemcpy(h.data(), tr, nl * 8, cudaMemcpyDeviceToHost);
    std::vector<double> hz(nx * ny);
    cudaMemcpy(hz.data(), z, nx * ny * 8, cudaMemcpyDeviceToHost);
    // CPU check
    std::vector<double> zc(nx * ny);
    double maxd = 0;
    for (int j = 0; j < ny; ++j)
        for (int i = 0; i < nx; ++i) {
            double acc = 1.0;
            if (i > 0) acc = fma(-0.25, zc[j * nx + i - 1], acc);
            if (j > 0) acc = fma(-0.25, zc[(j - 1) * nx + i], acc);
            zc[j * nx + i] = acc;
            maxd = std::max(maxd, std::abs(acc - hz[j * nx + i]));
        }
    printf("nx %d dbg %d threads %d: %.1f cycles/level, max diff %.2e (%s)\n", nx, dbg, threads,
           (double)(h[nl - 1] - h[0]) / (nl - 1), maxd, cudaGetErrorString(e));
    return 0;
}
