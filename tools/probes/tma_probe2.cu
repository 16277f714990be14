// TMA overlap probe (tuning aid): is a K-stage ring really overlapping loads?  One CTA, L2-resident
// data, 32 KB stages (1D bulk copies).  Variants: (A) issue all S stages at t=0, then wait each and
// spin `delay` cycles; (B) producer/consumer threads as in the kernel ring.  Prints us per stage.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include "lf_tc_ptx.cuh"
using namespace lf;

__device__ __forceinline__ void bulk_load_1d(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}

__global__ void probe_a(const unsigned char* g, int S, int stage_bytes, int delay, long long* out) {
    extern __shared__ unsigned char smem_raw[];
    unsigned char* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
    const uint32_t ring = ptx::smem_u32(smem), bars = ring + S * stage_bytes;
    if (threadIdx.x != 0) return;
    for (int i = 0; i < S; ++i) ptx::mbar_init(bars + 8 * i, 1);
    ptx::fence_mbar_init();
    const long long t0 = clock64();
    for (int i = 0; i < S; ++i) {
        ptx::mbar_arrive_expect_tx(bars + 8 * i, stage_bytes);
        bulk_load_1d(ring + i * stage_bytes, g + (size_t)i * stage_bytes, stage_bytes, bars + 8 * i);
    }
    long long land[16];
    for (int i = 0; i < S; ++i) {
        ptx::mbar_wait(bars + 8 * i, 0);
        land[i] = clock64() - t0;
        const long long t1 = clock64();
        while (clock64() - t1 < delay) {
        }
    }
    for (int i = 0; i < S; ++i) out[i] = land[i];
}

template <int kW>
__device__ __forceinline__ void wait_v(uint32_t bar, uint32_t parity) {
    if (kW == 0) {
        ptx::mbar_wait(bar, parity);
    } else if (kW == 1) {   // poll with nanosleep backoff
        while (!ptx::mbar_try_wait(bar, parity)) __nanosleep(32);
    } else if (kW == 2) {   // try_wait with a suspend-time hint (hardware sleeps until the phase completes)
        uint32_t ok = 0;
        while (!ok) {
            asm volatile(
                "{\n\t.reg .pred p;\n\t"
                "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
                "selp.u32 %0, 1, 0, p;\n\t}"
                : "=r"(ok)
                : "r"(bar), "r"(parity), "r"(1000000u)
                : "memory");
        }
    } else {                // test_wait spin (never suspends)
        uint32_t ok = 0;
        while (!ok) {
            asm volatile(
                "{\n\t.reg .pred p;\n\t"
                "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                "selp.u32 %0, 1, 0, p;\n\t}"
                : "=r"(ok)
                : "r"(bar), "r"(parity)
                : "memory");
        }
    }
}

// (B) ring: thread 0 produces, thread 32 consumes; `iters` stages over a region of `region` bytes
template <int kW>
__global__ void probe_b(const unsigned char* g, int S, int stage_bytes, int iters, int region, long long* out) {
    extern __shared__ unsigned char smem_raw[];
    unsigned char* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
    const uint32_t ring = ptx::smem_u32(smem), full = ring + S * stage_bytes, empty = full + 8 * S;
    if (threadIdx.x == 0) {
        for (int i = 0; i < S; ++i) {
            ptx::mbar_init(full + 8 * i, 1);
            ptx::mbar_init(empty + 8 * i, 1);
        }
        ptx::fence_mbar_init();
    }
    __syncthreads();
    const long long t0 = clock64();
    if (threadIdx.x == 0) {
        for (int it = 0; it < iters; ++it) {
            const int st = it % S;
            wait_v<kW>(empty + 8 * st, ((it / S) & 1) ^ 1);
            ptx::mbar_arrive_expect_tx(full + 8 * st, stage_bytes);
            bulk_load_1d(ring + st * stage_bytes, g + (size_t)(it * stage_bytes % region), stage_bytes, full + 8 * st);
        }
    } else if (threadIdx.x == 32) {
        for (int it = 0; it < iters; ++it) {
            const int st = it % S;
            wait_v<kW>(full + 8 * st, (it / S) & 1);
            if (it < 64) out[it] = clock64() - t0;
            ptx::mbar_arrive(empty + 8 * st);
        }
    }
}

int main() {
    unsigned char* g;
    cudaMalloc(&g, 64 << 20);
    cudaMemset(g, 1, 64 << 20);
    long long* d;
    cudaMalloc(&d, 16 * 8);
    cudaFuncSetAttribute(probe_a, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    for (int sb : {16384, 32768}) {
        for (int delay : {0, 2000}) {
            const int S = 6;
            for (int rep = 0; rep < 2; ++rep) {   // rep 0 warms L2
                probe_a<<<1, 32, S * sb + 2048>>>(g, S, sb, delay, d);
                cudaDeviceSynchronize();
            }
            long long h[16];
            cudaMemcpy(h, d, S * 8, cudaMemcpyDeviceToHost);
            printf("stage %5d B delay %4d: landed at cycles", sb, delay);
            for (int i = 0; i < S; ++i) printf(" %lld", h[i]);
            printf("\n");
        }
    }
    // cold (HBM): fresh region each time
    for (int sb : {16384, 32768}) {
        const int S = 6;
        probe_a<<<1, 32, S * sb + 2048>>>(g + (32 << 20) + (sb == 32768 ? (8 << 20) : 0), S, sb, 0, d);
        cudaDeviceSynchronize();
        long long h[16];
        cudaMemcpy(h, d, S * 8, cudaMemcpyDeviceToHost);
        printf("cold stage %5d B: landed at cycles", sb);
        for (int i = 0; i < S; ++i) printf(" %lld", h[i]);
        printf("\n");
    }
    cudaMalloc(&d, 64 * 8);
    for (int w = 0; w < 4; ++w) {
        auto k = w == 0 ? probe_b<0> : w == 1 ? probe_b<1> : w == 2 ? probe_b<2> : probe_b<3>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        for (int S : {2, 4, 6}) {
            const int sb = 32768, region = 8 << 20;
            for (int rep = 0; rep < 2; ++rep) {
                k<<<1, 64, S * sb + 2048>>>(g, S, sb, 64, region, d);
                cudaDeviceSynchronize();
            }
            long long h[64];
            cudaMemcpy(h, d, 64 * 8, cudaMemcpyDeviceToHost);
            printf("ring wait=%s S=%d: cycles per stage over 8..63: %.0f; first 6:",
                   w == 0 ? "try_wait" : w == 1 ? "nanosleep" : w == 2 ? "try_wait+hint" : "test_wait", S,
                   (h[63] - h[7]) / 56.0);
            for (int i = 0; i < 6; ++i) printf(" %lld", h[i]);
            printf("\n");
        }
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
