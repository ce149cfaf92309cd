// Do two single-CTA, whole-SM (big dynamic smem) kernels on two streams run
// concurrently?  Variants: plain launches, PDL attribute, a fork/join through
// events, and many-CTA kernels in between on the main stream.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void spin(long long cycles, int* out) {
    extern __shared__ int sm[];
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    long long t0 = clock64();
    int acc = 0;
    while (clock64() - t0 < cycles) acc += sm[threadIdx.x & 31];
    if (acc == 12345) out[0] = acc;
}
__global__ void small(int* out) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (threadIdx.x == 0 && blockIdx.x == 0) out[1] += 1;
}

static void launch(cudaStream_t s, bool pdl, void (*k)(long long, int*), int grid, int block, size_t smem,
                   long long cyc, int* out) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid; cfg.blockDim = block; cfg.dynamicSmemBytes = smem; cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at; cfg.numAttrs = pdl ? 1 : 0;
    cudaLaunchKernelEx(&cfg, k, cyc, out);
}
static void launch_small(cudaStream_t s, bool pdl, int grid, int* out) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid; cfg.blockDim = 256; cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at; cfg.numAttrs = pdl ? 1 : 0;
    cudaLaunchKernelEx(&cfg, small, out);
}

int main() {
    int* out; cudaMalloc(&out, 64);
    const size_t smem = 200 * 1024;
    cudaFuncSetAttribute(spin, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaStream_t a, b; cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking); cudaStreamCreateWithFlags(&b, cudaStreamNonBlocking);
    cudaEvent_t e0, e1, fork, join; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventCreateWithFlags(&fork, cudaEventDisableTiming); cudaEventCreateWithFlags(&join, cudaEventDisableTiming);
    const long long cyc = 100000;  // ~50 us
    for (int variant = 0; variant < 8; ++variant) {
        const bool pdl = variant & 1, smalls = variant & 2, big_small = variant & 4;
        float best = 1e9;
        for (int rep = 0; rep < 5; ++rep) {
            cudaDeviceSynchronize();
            cudaEventRecord(e0, a);
            cudaEventRecord(fork, a);
            cudaStreamWaitEvent(b, fork, 0);
            launch_small(b, pdl, 1, out);
            launch(b, pdl, spin, 1, 256, smem, cyc, out);         // side: one long single-CTA kernel
            for (int k = 0; k < 4; ++k) {                           // main: four single-CTA kernels
                if (smalls) launch_small(a, pdl, big_small ? 2000 : 100, out);
                launch(a, pdl, spin, 1, 256, smem, cyc / 4, out);
            }
            cudaEventRecord(join, b);
            cudaStreamWaitEvent(a, join, 0);
            cudaEventRecord(e1, a);
            cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            if (ms < best) best = ms;
        }
        printf("pdl=%d smalls=%d(big=%d): %.1f us (serial would be ~2x the side kernel)\n", pdl, smalls ? 1 : 0,
               big_small ? 1 : 0, best * 1e3);
    }
    // reference: side kernel alone
    cudaEventRecord(e0, b); launch(b, false, spin, 1, 256, smem, cyc, out); cudaEventRecord(e1, b); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); printf("side kernel alone: %.1f us\n", ms * 1e3);
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
