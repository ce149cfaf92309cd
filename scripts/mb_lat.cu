// Dev micro-benchmark: dependent-latency of the operations on the GS critical
// path (DFMA, DADD, LDS, STS->LDS, shfl, bar.sync, named barrier) on B200.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_lat(long long* out, double* sink, int n) {
    __shared__ double s[1024];
    __shared__ int si[1024];
    const int t = threadIdx.x;
    for (int i = t; i < 1024; i += blockDim.x) {
        s[i] = 1.0 + i * 1e-9;
        si[i] = (i + 1) & 1023;
    }
    __syncthreads();
    double x = sink[0];
    long long t0, t1;
    // DFMA chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) x = fma(x, 0.999999, 1e-7);
    t1 = clock64();
    if (t == 0) out[0] = t1 - t0;
    // DADD chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) x = x + 1e-7;
    t1 = clock64();
    if (t == 0) out[1] = t1 - t0;
    // DMUL chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) x = x * 1.0000001;
    t1 = clock64();
    if (t == 0) out[2] = t1 - t0;
    // LDS pointer chase (int)
    int p = t & 1023;
    t0 = clock64();
    for (int i = 0; i < n; ++i) p = si[p];
    t1 = clock64();
    if (t == 0) out[3] = t1 - t0;
    // LDS.64 dependent (double load indexed by previous value)
    double y = 0.0;
    t0 = clock64();
    for (int i = 0; i < n; ++i) y = s[(int)y & 1023] - 1.0;
    t1 = clock64();
    if (t == 0) out[4] = t1 - t0;
    // STS then LDS same address (store -> load forwarding through smem)
    t0 = clock64();
    for (int i = 0; i < n; ++i) {
        s[t] = x;
        __syncwarp();
        x = s[t] * 1.0;
    }
    t1 = clock64();
    if (t == 0) out[5] = t1 - t0;
    // shfl chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) x = __shfl_sync(0xffffffffu, x, (t + 1) & 31);
    t1 = clock64();
    if (t == 0) out[6] = t1 - t0;
    // bar.sync
    t0 = clock64();
    for (int i = 0; i < n; ++i) __syncthreads();
    t1 = clock64();
    if (t == 0) out[7] = t1 - t0;
    // integer add chain (loop overhead reference)
    int q = t;
    t0 = clock64();
    for (int i = 0; i < n; ++i) q = q * 3 + 1;
    t1 = clock64();
    if (t == 0) out[8] = t1 - t0;
    sink[1 + t] = x + y + p + q;
}

int main() {
    long long* d;
    double* sink;
    cudaMalloc(&d, 16 * 8);
    cudaMalloc(&sink, 4096 * 8);
    cudaMemset(sink, 0, 4096 * 8);
    const char* names[] = {"DFMA", "DADD", "DMUL", "LDS.32 chase", "LDS.64 dep", "STS->LDS", "SHFL", "BAR(threads)", "IMAD"};
    const int n = 4096;
    for (int th : {32, 128, 384, 512}) {
        k_lat<<<1, th>>>(d, sink, n);
        k_lat<<<1, th>>>(d, sink, n);
        long long h[16];
        cudaMemcpy(h, d, 9 * 8, cudaMemcpyDeviceToHost);
        printf("threads %d:", th);
        for (int k = 0; k < 9; ++k) printf("  %s %.1f", names[k], (double)h[k] / n);
        printf("  (%s)\n", cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
