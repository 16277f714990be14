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
    } else if (kW == 4) {   // hinted try_wait loop bounded by an iteration count (no clock reads)
        uint32_t n = 0;
        for (;;) {
            uint32_t ok;
            asm volatile(
                "{\n\t.reg .pred p;\n\t"
                "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
                "selp.u32 %0, 1, 0, p;\n\t}"
                : "=r"(ok)
                : "r"(bar), "r"(parity), "r"(1000000u)
                : "memory");
            if (ok) break;
            if (++n > (1u << 24)) __trap();
        }
    } else if (kW == 6) {   // loop inside one asm block, bounded by an iteration count
        asm volatile(
            "{\n\t.reg .pred p;\n\t.reg .u32 n;\n\tmov.u32 n, 0;\n"
            "LF_WAIT:\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
            "@p bra.uni LF_DONE;\n\t"
            "add.u32 n, n, 1;\n\t"
            "setp.lt.u32 p, n, 0x10000000;\n\t"
            "@p bra.uni LF_WAIT;\n\t"
            "trap;\n"
            "LF_DONE:\n\t}" ::"r"(bar), "r"(parity)
            : "memory");
    } else if (kW == 7) {   // loop inside one asm block, unbounded
        asm volatile(
            "{\n\t.reg .pred p;\n"
            "LF_WAIT:\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
            "@!p bra.uni LF_WAIT;\n\t}" ::"r"(bar), "r"(parity)
            : "memory");
    } else if (kW == 5) {   // plain try_wait loop (no hint, no bound)
        while (!ptx::mbar_try_wait(bar, parity)) {
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

// (C) ring whose consumer is the QK MMA of the decode kernel: 8 x tcgen05.mma M128 N8 K16 per 32 KB
// stage (A = the landed tile, SW128 K-major), tcgen05.commit -> EMPTY.  kMma = 0: consumer arrives
// without MMA (control).
template <int kMma>
__global__ void __launch_bounds__(128, 1) probe_c(const unsigned char* g, int S, int iters, int region, long long* out) {
    extern __shared__ unsigned char smem_raw[];
    unsigned char* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
    const int sb = 32768;
    const uint32_t ring = ptx::smem_u32(smem), qb = ring + S * sb, full = qb + 4096, empty = full + 8 * S,
                   tslot = empty + 8 * S;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < S; ++i) {
            ptx::mbar_init(full + 8 * i, 1);
            ptx::mbar_init(empty + 8 * i, 1);
        }
        ptx::fence_mbar_init();
    }
    if (warp == 1) ptx::tmem_alloc(tslot, 32);
    for (int i = threadIdx.x; i < 1024; i += 128) ((uint32_t*)(smem + S * sb))[i] = 0;
    ptx::fence_proxy_async_smem();
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *(volatile uint32_t*)(smem + (tslot - ring));
    const long long t0 = clock64();
    if (threadIdx.x == 0) {
        for (int it = 0; it < iters; ++it) {
            const int st = it % S;
            ptx::mbar_wait(empty + 8 * st, ((it / S) & 1) ^ 1);
            ptx::mbar_arrive_expect_tx(full + 8 * st, sb);
            bulk_load_1d(ring + st * sb, g + (size_t)(it * sb % region), sb, full + 8 * st);
        }
    } else if (kMma == 3 && warp == 1) {   // the whole warp walks the loop, one elected lane issues
        constexpr uint32_t idesc = ptx::idesc_bf16_f32(128, 8, 0, 0);
        for (int it = 0; it < iters; ++it) {
            const int st = it % S;
            ptx::mbar_wait(full + 8 * st, (it / S) & 1);
            if (it < 64 && lane == 0) out[it] = clock64() - t0;
            ptx::tc_fence_after();
            const uint32_t base = ring + st * sb;
            const uint64_t da0 = ptx::smem_desc_sw128(base, 16, 1024), db0 = ptx::smem_desc_sw128(qb, 16, 1024);
            if (ptx::elect_one()) {
#pragma unroll
                for (int kk = 0; kk < 8; ++kk)
                    ptx::mma_bf16(tmem + 8u * (it & 3), da0 + (uint64_t)((kk >> 2) * 1024 + (kk & 3) * 2),
                                  db0 + (uint64_t)((kk >> 2) * 64 + (kk & 3) * 2), idesc, kk > 0);
                ptx::mma_commit(empty + 8 * st);
            }
            __syncwarp();
        }
    } else if (kMma != 3 && threadIdx.x == 32) {
        constexpr uint32_t idesc = ptx::idesc_bf16_f32(128, 8, 0, 0);
        for (int it = 0; it < iters; ++it) {
            const int st = it % S;
            ptx::mbar_wait(full + 8 * st, (it / S) & 1);
            if (it < 64) out[it] = clock64() - t0;
            if (kMma) {
                ptx::tc_fence_after();
                const uint32_t base = ring + st * sb;
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const uint64_t da = ptx::smem_desc_sw128(base + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024);
                    const uint64_t db = ptx::smem_desc_sw128(qb + (kk >> 2) * 1024 + (kk & 3) * 32, 16, 1024);
                    ptx::mma_bf16(tmem + 8u * (it & 3), da, db, idesc, kk > 0);
                }
                if (kMma == 1) ptx::mma_commit(empty + 8 * st);
                else ptx::mbar_arrive(empty + 8 * st);   // kMma 2: stage released at issue (timing only)
            } else {
                ptx::mbar_arrive(empty + 8 * st);
            }
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem, 32);
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
    for (int w = 0; w < 8; ++w) {
        auto k = w == 0 ? probe_b<0> : w == 1 ? probe_b<1> : w == 2 ? probe_b<2> : w == 3 ? probe_b<3> : w == 4 ? probe_b<4> : w == 5 ? probe_b<5> : w == 6 ? probe_b<6> : probe_b<7>;
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
                   w == 0 ? "mbar_wait" : w == 1 ? "nanosleep" : w == 2 ? "try_wait+hint" : w == 3 ? "test_wait" : w == 4 ? "hint+count" : w == 5 ? "try_wait" : w == 6 ? "asm-loop+bound" : "asm-loop", S,
                   (h[63] - h[7]) / 56.0);
            for (int i = 0; i < 6; ++i) printf(" %lld", h[i]);
            printf("\n");
        }
    }
    for (int m = 0; m < 4; ++m) {
        auto k = m == 3 ? probe_c<3> : m == 2 ? probe_c<2> : m ? probe_c<1> : probe_c<0>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        for (int S : {2, 4, 6}) {
            for (int rep = 0; rep < 2; ++rep) {
                k<<<1, 128, S * 32768 + 4096 + 2048>>>(g, S, 64, 8 << 20, d);
                cudaDeviceSynchronize();
            }
            long long h[64];
            cudaMemcpy(h, d, 64 * 8, cudaMemcpyDeviceToHost);
            printf("ring+%s S=%d: cycles per stage over 8..63: %.0f\n", m == 3 ? "QK-MMA(warp + elect)" : m == 2 ? "QK-MMA(release at issue)" : m ? "QK-MMA" : "no-MMA", S, (h[63] - h[7]) / 56.0);
        }
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
