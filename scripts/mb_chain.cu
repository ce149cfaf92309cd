// Dev micro-benchmark: the bare per-level chain of the walk for one warp:
// two shared gathers of values written by other lanes in the previous level,
// two dependent DFMAs, a shared store, warp sync.  Variants isolate each part.
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k_chain(int levels, long long* out, double* sink) {
    __shared__ double z[2048];
    const int t = threadIdx.x;
    for (int i = t; i < 2048; i += 32) z[i] = 1e-3 * i;
    __syncwarp();
    int w = t, s0 = (t + 31) & 31, s1 = (t + 1) & 31;
    double acc = 0.0;
    long long t0 = clock64();
    for (int L = 0; L < levels; ++L) {
        const int base = (L & 31) * 64, nb = ((L + 1) & 31) * 64;
        double z0, z1;
        if (MODE == 3) {  // no gathers: chain through registers only
            z0 = acc;
            z1 = acc;
        } else {
            z0 = z[base + s0];
            z1 = z[base + s1];
        }
        acc = fma(0.25, z1, fma(0.25, z0, 1.0));
        if (MODE != 2) z[nb + w] = acc;  // MODE 2: no store (gathers read stale values)
        if (MODE == 0) __syncwarp();
        if (MODE == 1) asm volatile("bar.warp.sync 0xffffffff;" ::: "memory");
        if (MODE == 4) asm volatile("bar.sync 1, 32;" ::: "memory");
    }
    long long t1 = clock64();
    if (t == 0) out[MODE] = t1 - t0;
    sink[t] = acc;
}

int main() {
    long long* d;
    double* sink;
    cudaMalloc(&d, 64);
    cudaMalloc(&sink, 32 * 8);
    const int L = 20000;
    const char* names[] = {"__syncwarp", "bar.warp.sync", "no store", "register chain (no smem)",
                           "bar.sync 1,32"};
    k_chain<0><<<1, 32>>>(L, d, sink);
    k_chain<1><<<1, 32>>>(L, d, sink);
    k_chain<2><<<1, 32>>>(L, d, sink);
    k_chain<3><<<1, 32>>>(L, d, sink);
    k_chain<4><<<1, 32>>>(L, d, sink);
    for (int rep = 0; rep < 2; ++rep) {
        k_chain<0><<<1, 32>>>(L, d, sink);
        k_chain<1><<<1, 32>>>(L, d, sink);
        k_chain<2><<<1, 32>>>(L, d, sink);
        k_chain<3><<<1, 32>>>(L, d, sink);
        k_chain<4><<<1, 32>>>(L, d, sink);
    }
    long long h[5];
    cudaMemcpy(h, d, 40, cudaMemcpyDeviceToHost);
    for (int m = 0; m < 5; ++m) printf("%-28s %6.1f cycles/level\n", names[m], (double)h[m] / L);
    return 0;
}
