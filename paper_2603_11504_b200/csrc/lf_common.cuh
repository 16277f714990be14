// Device code shared by the two split-KV decode kernels: bf16 helpers and the cluster-wide
// combine / LongFlowScore finalisation / argmin / eviction write.
#pragma once
#include <cooperative_groups.h>
#include <stdint.h>

#include "lf_internal.h"

namespace lf {

namespace cg = cooperative_groups;

__device__ __forceinline__ float bf16_to_f32(uint16_t b) { return __uint_as_float(((uint32_t)b) << 16); }

__device__ __forceinline__ uint16_t f32_to_bf16_rne(float f) {
    uint32_t u = __float_as_uint(f);
    if ((u & 0x7fffffffu) > 0x7f800000u) return (uint16_t)((u >> 16) | 0x40);  // quiet NaN
    u += 0x7fffu + ((u >> 16) & 1u);
    return (uint16_t)(u >> 16);
}

// fp32 -> uint32 whose unsigned order is the float order (argmin key, -inf smallest)
__device__ __forceinline__ uint32_t ordered_bits(float f) {
    uint32_t u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// explicit shared-state-space accesses for pointers the compiler only sees as generic
__device__ __forceinline__ float lds_f32(const float* p) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"((uint32_t)__cvta_generic_to_shared(p)));
    return v;
}

// Programmatic dependent launch: let the next kernel in the stream start its prologue now, and wait
// until the previous kernel's memory is visible before the first dependent global access.
// 16-byte global -> SMEM copies that bypass registers (LDGSTS), many in flight per thread
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gmem_src) {
    uint32_t d = (uint32_t)__cvta_generic_to_shared(smem_dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ unsigned long long umin64(unsigned long long a, unsigned long long b) {
    return a < b ? a : b;
}

// Per-CTA scratch the finalisation works on (all in this CTA's shared memory).
struct Partials {
    float* ex_m;                 // [16]     this CTA's max m_g over its chunk (log2 units), -inf if empty
    float* ex_z;                 // [16]     sum_j 2^(x_gj - m_g)
    float* ex_o;                 // [GP][D]  sum_j 2^(x_gj - m_g) v_j   (un-normalised)
    float* X;                    // [G][chunk] x_gj = q_g.k_j * scale * log2(e)
    float* L;                    // [chunk]  lambda_j = ||v_j||_1
    float* misc;                 // [128]
    unsigned long long* keys;    // [16]
};

// Cluster combine + scores + argmin + write-back.  Must be called by every thread of every CTA
// of the unit's cluster after the CTA's partials are complete (no barrier needed before).
//   M_g  = max(max_s m_g,s, x_g*)                    (x_g* = current token)
//   Z_g  = sum_s Z_g,s 2^(m_g,s - M_g) + 2^(x_g* - M_g)      (Eq. 4's Z over t tokens)
//   I_j  = lambda_j / G * sum_g 2^(x_gj - M_g) / Z_g  (Eq. 6, normalised once as Alg. 1)
//   slot = lowest-index argmin over log2 I_j (R7); append at n while n < N (R11)
//   out  = (sum_s o_s 2^(m_s - M) + 2^(x* - M) v*) / Z   (Alg. 1)
template <int D, int GP, int NT>
__device__ __forceinline__ void cluster_finalize(const StepParams& p, const Partials& t, int u, int n, int c0,
                                                 int c1, int nv) {
    cg::cluster_group cluster = cg::this_cluster();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int NW = NT / 32;
    const int G = p.G, N = p.N, chunk = p.chunk, S = p.splits;
    const int s = (int)cluster.block_rank();
    const int b = u / p.Hkv, h = u % p.Hkv;
    float* xnew = t.misc;       // [16]
    float* gM = t.misc + 16;    // [16]
    float* glz = t.misc + 32;   // [16]
    float* gZ = t.misc + 48;    // [16]

    // current token's logit x_g*, computed identically (same order) by every CTA of the cluster
    {
        const uint16_t* kn = p.k_new + (size_t)u * D;
        for (int g = warp; g < G; g += NW) {
            const uint16_t* qg = p.q + ((size_t)b * p.Hq + (size_t)h * G + g) * D;
            float acc = 0.f;
            for (int l = lane; l < D; l += 32) acc = fmaf(bf16_to_f32(qg[l]), bf16_to_f32(kn[l]), acc);
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
            if (lane == 0) xnew[g] = p.deferred ? -INFINITY : acc * p.scale_log2;
        }
    }
    cluster.sync();   // #1: every CTA's (m, Z, o) partials visible cluster-wide
    if (tid < G) {
        const int g = tid;
        float M = xnew[g];
        for (int r = 0; r < S; ++r) M = fmaxf(M, cluster.map_shared_rank(t.ex_m, r)[g]);
        float Z = 0.f;
        for (int r = 0; r < S; ++r) {
            const float mr = cluster.map_shared_rank(t.ex_m, r)[g];
            const float zr = cluster.map_shared_rank(t.ex_z, r)[g];
            Z += zr * exp2f(mr - M);
        }
        Z += exp2f(xnew[g] - M);
        gM[g] = M;
        gZ[g] = Z;
        glz[g] = log2f(Z);
    }
    __syncthreads();
    // scores and local argmin over this CTA's valid slots
    unsigned long long best = ~0ull;
    const float log2G = log2f((float)G);
    const float invG = 1.0f / (float)G;
    const int excl = (p.deferred && p.exclude_newest) ? p.written[u] : -1;
    for (int j = tid; j < nv; j += NT) {
        const float lam = lds_f32(t.L + j);
        float a[GP];
        float amax = -INFINITY;
#pragma unroll
        for (int g = 0; g < GP; ++g) {
            a[g] = g < G ? lds_f32(t.X + g * chunk + j) - gM[g] - glz[g] : -INFINITY;
            amax = fmaxf(amax, a[g]);
        }
        float ssum = 0.f, sc = 0.f;
#pragma unroll
        for (int g = 0; g < GP; ++g) {
            ssum += exp2f(a[g] - amax);
            sc += exp2f(a[g]);
        }
        const float ls = log2f(lam) + amax + log2f(ssum) - log2G;   // log2 I_j (no underflow)
        if (p.scores) p.scores[(size_t)u * N + c0 + j] = lam * sc * invG;
        if (c0 + j != excl) best = umin64(best, ((unsigned long long)ordered_bits(ls) << 32) | (unsigned)(c0 + j));
    }
    if (p.scores)
        for (int j = nv + tid; j < c1 - c0; j += NT) p.scores[(size_t)u * N + c0 + j] = INFINITY;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) best = umin64(best, __shfl_xor_sync(0xffffffffu, best, off));
    if (lane == 0) t.keys[1 + warp] = best;
    __syncthreads();
    if (tid == 0) {
        unsigned long long m = t.keys[1];
        for (int w = 1; w < NW; ++w) m = umin64(m, t.keys[1 + w]);
        t.keys[0] = m;
    }
    cluster.sync();   // #2: per-CTA argmin keys visible
    if (s == 0) {
        int* s_slot = (int*)(t.misc + 64);
        if (tid == 0) {
            unsigned long long m = ~0ull;
            for (int r = 0; r < S; ++r) m = umin64(m, cluster.map_shared_rank(t.keys, r)[0]);
            if (p.deferred) {            // next step's victim; the current token is already in place
                p.pend[u] = (int)(m & 0xffffffffull);
                *s_slot = -1;
            } else {
                const int sl = n < N ? n : (int)(m & 0xffffffffull);
                *s_slot = sl;
                p.slot[u] = sl;
                if (n < N) p.n_valid[u] = n + 1;
            }
        }
        __syncthreads();
        const int sl = *s_slot;
        const uint16_t* vn = p.v_new + (size_t)u * D;
        for (int i = tid; i < G * D; i += NT) {
            const int g = i / D, l = i % D;
            float acc = 0.f;
            for (int r = 0; r < S; ++r) {
                const float mr = cluster.map_shared_rank(t.ex_m, r)[g];
                acc += cluster.map_shared_rank(t.ex_o, r)[g * D + l] * exp2f(mr - gM[g]);
            }
            acc += exp2f(xnew[g] - gM[g]) * bf16_to_f32(vn[l]);
            const float ov = acc / gZ[g];
            const size_t oi = ((size_t)b * p.Hq + (size_t)h * G + g) * D + l;
            if (p.out_f32) ((float*)p.out)[oi] = ov;
            else ((uint16_t*)p.out)[oi] = f32_to_bf16_rne(ov);
        }
        // in-place eviction write (or append): every CTA finished reading K/V before sync #1
        if (sl >= 0 && tid < D / 8) {
            const size_t unit_off = (size_t)u * N * D;
            const uint4* ks = (const uint4*)(p.k_new + (size_t)u * D);
            const uint4* vs = (const uint4*)(p.v_new + (size_t)u * D);
            ((uint4*)(p.K + unit_off + (size_t)sl * D))[tid] = ks[tid];
            ((uint4*)(p.V + unit_off + (size_t)sl * D))[tid] = vs[tid];
        }
    }
    cluster.sync();   // #3: rank 0 is done reading remote shared memory
}

}  // namespace lf
