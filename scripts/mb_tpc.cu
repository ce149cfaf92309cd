// Does a CTA's shared-memory / TMA streaming rate drop when the other SM of its
// TPC runs the same kind of kernel?  One CTA per SM (200 KB dynamic smem),
// each streams `iters` x 16 KB bulk copies global -> shared and reads them back.
// Variants: 1 CTA; 2 CTAs in a cluster (same TPC in practice); 2 CTAs as a
// plain grid; a cluster of 4 using ranks 0 and 2 only.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__global__ void stream(const char* src, size_t src_bytes, int iters, int active_mask, double* out, int* smids) {
    extern __shared__ __align__(128) char sm[];
    unsigned rank = 0;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    if (!((active_mask >> rank) & 1) && active_mask != 0) return;
    __shared__ __align__(8) unsigned long long bar;
    const int tid = threadIdx.x;
    if (tid == 0) {
        asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        unsigned s; asm volatile("mov.u32 %0, %%smid;" : "=r"(s)); smids[blockIdx.x] = s;
    }
    __syncthreads();
    double acc = 0.0;
    unsigned phase = 0;
    const unsigned chunk = 16384;
    for (int it = 0; it < iters; ++it) {
        if (tid == 0) {
            const char* g = src + ((size_t)(it * 7 + blockIdx.x * 3) * chunk) % (src_bytes - chunk);
            asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(chunk));
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(smem_u32(sm + (it & 7) * chunk)), "l"(g), "r"(chunk), "r"(smem_u32(&bar)) : "memory");
        }
        unsigned done = 0;
        while (!done)
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                         : "=r"(done) : "r"(smem_u32(&bar)), "r"(phase) : "memory");
        phase ^= 1;
        const double* d = reinterpret_cast<const double*>(sm + (it & 7) * chunk);
        for (int k = tid; k < (int)(chunk / 8); k += blockDim.x) acc += d[k];
        __syncthreads();
    }
    if (acc == 12345.0) out[0] = acc;
}

int main() {
    const size_t bytes = 256u << 20;
    char* src; cudaMalloc(&src, bytes); cudaMemset(src, 0, bytes);
    double* out; cudaMalloc(&out, 8);
    int* smids; cudaMalloc(&smids, 64);
    const size_t smem = 200 * 1024;
    cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(stream, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    const int iters = 2000;
    struct V { const char* name; int grid, cluster, mask; } vs[] = {
        {"1 CTA", 1, 1, 0}, {"2 CTAs, cluster 2", 2, 2, 0}, {"2 CTAs, plain grid", 2, 1, 0},
        {"cluster 4, ranks 0+2 active", 4, 4, 0x5}, {"cluster 4, all active", 4, 4, 0}};
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (auto& v : vs) {
        float best = 1e9;
        int sid[4] = {-1, -1, -1, -1};
        for (int rep = 0; rep < 3; ++rep) {
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = v.grid; cfg.blockDim = 256; cfg.dynamicSmemBytes = smem;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = v.cluster; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
            cfg.attrs = at; cfg.numAttrs = 1;
            cudaEventRecord(a);
            cudaError_t e = cudaLaunchKernelEx(&cfg, stream, (const char*)src, bytes, iters, v.mask, out, smids);
            cudaEventRecord(b); cudaEventSynchronize(b);
            if (e != cudaSuccess) { printf("%s: %s\n", v.name, cudaGetErrorString(e)); break; }
            float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
            cudaMemcpy(sid, smids, sizeof(int) * v.grid, cudaMemcpyDeviceToHost);
        }
        printf("%-30s %8.1f us  (%.1f GB/s per active CTA)  sms %d %d %d %d\n", v.name, best * 1e3,
               iters * 16384.0 / (best * 1e-3) / 1e9, sid[0], sid[1], v.grid > 2 ? sid[2] : -1, v.grid > 3 ? sid[3] : -1);
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
