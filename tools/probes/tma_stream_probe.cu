// Per-SM DRAM streaming probe (tuning aid): how fast can ONE CTA pull data from HBM with bulk TMA
// copies into an R-stage ring of 32 KB stages when nothing consumes the data (no MMA, no SMEM reads)?
// One elected thread issues cp.async.bulk (global -> shared, complete_tx on the stage's mbarrier),
// waits for each stage in order and re-issues it.  Every CTA streams its own 64 MB slice of a buffer
// far larger than L2, so every byte comes from DRAM.  Prints GB/s per CTA and in total for
// R in {1, 2, 3, 4, 6} and {1, 16, 74, 148, 296} CTAs (two per SM at 296, R <= 3).
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tma_stream_probe tools/probes/tma_stream_probe.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

constexpr int kStage = 32768;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

__global__ void stream(const unsigned char* __restrict__ src, size_t per_cta, int R, unsigned long long* sink) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ __align__(8) unsigned long long bar[8];
    if (threadIdx.x != 0) return;
    for (int i = 0; i < R; ++i)
        asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(smem_u32(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const unsigned char* base = src + (size_t)blockIdx.x * per_cta;
    const int n = (int)(per_cta / kStage);
    auto issue = [&](int t) {
        const int st = t % R;
        const uint32_t b = smem_u32(&bar[st]);
        asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(b), "r"(kStage) : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                smem_u32(sm + st * kStage)),
            "l"(base + (size_t)t * kStage), "r"(kStage), "r"(b)
            : "memory");
    };
    for (int t = 0; t < R && t < n; ++t) issue(t);
    unsigned long long acc = 0;
    for (int t = 0; t < n; ++t) {
        const int st = t % R;
        const uint32_t b = smem_u32(&bar[st]);
        const uint32_t par = (uint32_t)(t / R) & 1u;
        asm volatile(
            "{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n\t@!p bra W;\n\t}" ::"r"(b),
            "r"(par)
            : "memory");
        acc += sm[st * kStage + (t & 1023)];
        if (t + R < n) issue(t + R);
    }
    sink[blockIdx.x] = acc;
}

int main() {
    const size_t per_cta = 64ull << 20;
    const int max_ctas = 296;
    unsigned char* buf;
    unsigned long long* sink;
    if (cudaMalloc(&buf, per_cta * max_ctas) != cudaSuccess) {   // 18.5 GB
        printf("alloc failed\n");
        return 1;
    }
    cudaMemset(buf, 1, per_cta * max_ctas);
    cudaMalloc(&sink, max_ctas * sizeof(unsigned long long));
    cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 6 * kStage);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int Rs[] = {1, 2, 3, 4, 6};
    const int Cs[] = {1, 16, 74, 148, 296};
    for (int C : Cs) {
        for (int R : Rs) {
            if (C > 148 && R > 3) continue;   // two CTAs per SM: <= 3 stages each
            // per-CTA bytes: enough for >= ~2 ms of streaming, bounded by the slice
            const size_t bytes = C <= 16 ? per_cta : (C <= 148 ? 32ull << 20 : 16ull << 20);
            stream<<<C, 32, R * kStage>>>(buf, bytes, R, sink);
            cudaEventRecord(e0);
            stream<<<C, 32, R * kStage>>>(buf, bytes, R, sink);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            const double per = bytes / (ms * 1e-3) / 1e9;
            printf("ctas %3d stages %d (%3d KB in flight): %7.1f GB/s per CTA, %7.0f GB/s total (%s)\n", C, R,
                   R * 32, per, per * C, cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
