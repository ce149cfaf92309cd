// Dev micro-benchmark: what makes a level of the single-CTA walk cost what it
// costs.  Variants of a 2-term level loop (gather from a smem ring, FMA,
// ring store, barrier) with: a large dynamic smem allocation; next-level
// records prefetched from smem; a 1-thread producer warp.
#include <cstdio>
#include <cuda_runtime.h>

template <int REC, int PROD>
__global__ void k_var(int levels, int width, long long* out, double* sink) {
    extern __shared__ __align__(16) unsigned char sm[];
    double* ring = reinterpret_cast<double*>(sm);            // 4096 doubles
    int4* rec = reinterpret_cast<int4*>(sm + 4096 * 8);       // records: levels x width (s0, s1, b lo, b hi)
    const int t = threadIdx.x - 32;
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) ring[i] = 1.0 + i * 1e-6;
    if (REC)
        for (int i = threadIdx.x; i < 64 * width; i += blockDim.x) {
            const int tt = i % width;
            rec[i] = make_int4((tt * 7) & 4095, (tt * 7 + 1) & 4095, 0, 0x3ff00000);
        }
    __syncthreads();
    long long t0 = clock64();
    int s0 = (t * 7) & 4095, s1 = (t * 7 + 1) & 4095;
    double b = 1.0;
    int4 nx = make_int4(0, 0, 0, 0);
    volatile int sinkp = 0;
    for (int l = 0; l < levels; ++l) {
        if (t >= 0 && t < width) {
            const double z0 = ring[s0], z1 = ring[s1];
            if (REC) nx = rec[((l + 1) & 63) * width + t];
            const double acc = fma(0.2, z1, fma(0.3, z0, b));
            ring[(l * width + t) & 4095] = acc * 1e-3;
            if (REC) {
                s0 = (nx.x + l) & 4095;
                s1 = (nx.y + l) & 4095;
                b = __hiloint2double(nx.w, nx.z);
            } else {
                s0 = (s0 + width) & 4095;
                s1 = (s1 + width) & 4095;
            }
        } else if (PROD && threadIdx.x == 0) {
            sinkp = sinkp + 1;
        }
        __syncthreads();
    }
    if (threadIdx.x == 32) out[0] = clock64() - t0;
    if (threadIdx.x == 32) sink[0] = ring[5] + sinkp;
}

int main() {
    long long* d;
    double* sink;
    cudaMalloc(&d, 64);
    cudaMalloc(&sink, 64);
    const int levels = 4000;
    auto run = [&](auto kern, const char* name, int width, size_t smem) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        const int threads = 32 + (width + 31) / 32 * 32;
        long long h = 0;
        for (int r = 0; r < 2; ++r) kern<<<1, threads, smem>>>(levels, width, d, sink);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        printf("%-28s width %3d smem %6zu: %6.1f cycles/level (%s)\n", name, width, smem, (double)h / levels,
               cudaGetErrorString(e));
    };
    for (int width : {64, 160, 352}) {
        const size_t small = 4096 * 8 + 64 * width * 16;
        run(k_var<0, 0>, "ring only", width, small);
        run(k_var<0, 0>, "ring only, 227KB smem", width, 227 * 1024);
        run(k_var<1, 0>, "records", width, small);
        run(k_var<1, 0>, "records, 227KB smem", width, 227 * 1024);
        run(k_var<1, 1>, "records + producer", width, small);
    }
    return 0;
}
