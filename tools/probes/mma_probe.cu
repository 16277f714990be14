// tcgen05.mma issue-rate probe (tuning aid): cycles per kind::f16 MMA (K=16, SW128 K-major A and B from
// SMEM, fp32 accumulate in TMEM) for the decode kernel's shapes and their transposes.  NACC > 1: the MMAs
// rotate over NACC accumulators (independent chains) instead of all accumulating into one.
#include <cuda_runtime.h>
#include <cstdio>
#include "lf_tc_ptx.cuh"
using namespace lf;

template <int M, int N, int kAMN, int NACC>
__global__ void __launch_bounds__(128, 1) mma_rate(int reps, long long* out) {
    extern __shared__ unsigned char smem_raw[];
    unsigned char* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
    const uint32_t a = ptx::smem_u32(smem), b = a + 65536, bar = b + 65536, tslot = bar + 8;
    for (int i = threadIdx.x; i < 131072 / 4; i += 128) ((uint32_t*)smem)[i] = 0x3f803f80u;
    ptx::fence_proxy_async_smem();
    if (threadIdx.x == 0) {
        ptx::mbar_init(bar, 1);
        ptx::fence_mbar_init();
    }
    if (threadIdx.x < 32) ptx::tmem_alloc(tslot, 512);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *(volatile uint32_t*)(smem + (tslot - a));
    if (threadIdx.x == 0) {
        constexpr uint32_t idesc = ptx::idesc_bf16_f32(M, N, kAMN, 0);
        const long long t0 = clock64();
        for (int r = 0; r < reps; ++r) {
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
                const uint64_t da = kAMN ? ptx::smem_desc_sw128(a + kk * 2048, 16384, 1024)
                                         : ptx::smem_desc_sw128(a + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024);
                const uint64_t db = ptx::smem_desc_sw128(b + (kk >> 2) * 32768 + (kk & 3) * 32, 16, 1024);
                ptx::mma_bf16(tmem + (uint32_t)((kk % NACC) * (N < 16 ? 16 : N)), da, db, idesc, (r | (kk / NACC)) > 0);
            }
        }
        ptx::mma_commit(bar);
        ptx::mbar_wait(bar, 0);
        out[0] = clock64() - t0;
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem, 512);
    }
}

template <int M, int N, int kAMN, int NACC = 1>
void run(long long* d) {
    cudaFuncSetAttribute(mma_rate<M, N, kAMN, NACC>, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
    const int reps = 64;
    for (int i = 0; i < 2; ++i) mma_rate<M, N, kAMN, NACC><<<1, 128, 140 * 1024>>>(reps, d);
    cudaDeviceSynchronize();
    long long h;
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    const double per = (double)h / (reps * 8);
    printf("NACC %d M%3d N%3d A %s: %6.1f cycles per MMA  (%.0f FMA/cycle, A+B %d B per MMA)  err=%s\n", NACC, M, N,
           kAMN ? "MN-major" : "K-major ", per, (double)M * N * 16 / per, (M + N) * 32,
           cudaGetErrorString(cudaGetLastError()));
}

int main() {
    long long* d;
    cudaMalloc(&d, 8);
    run<128, 8, 0>(d);
    run<128, 16, 0>(d);
    run<128, 16, 1>(d);
    run<128, 32, 0>(d);
    run<128, 64, 0>(d);
    run<128, 128, 0>(d);
    run<128, 256, 0>(d);
    run<64, 8, 0>(d);
    run<64, 16, 0>(d);
    run<64, 64, 0>(d);
    run<64, 128, 0>(d);
    run<64, 256, 0>(d);
    run<128, 8, 0, 2>(d);
    run<128, 8, 0, 4>(d);
    run<128, 8, 0, 8>(d);
    run<128, 16, 1, 2>(d);
    run<128, 16, 1, 4>(d);
    run<128, 16, 1, 8>(d);
    return 0;
}
