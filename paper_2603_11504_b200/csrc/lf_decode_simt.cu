// CUDA-core split-KV LongFlow decode step (the G <= 2 path, and the reference CUDA path the
// tcgen05 kernel is checked against).  One thread-block CLUSTER per unit u = (sequence, kv head);
// CTA s of the cluster owns cache slots [s*chunk, (s+1)*chunk).
//
// Per CTA (Alg. 1 P:500-547 restructured for sm_100a):
//   K pass  stream K tiles (64 tokens) HBM -> SMEM with 16-byte cp.async (coalesced, XOR-swizzled
//           16 B chunks so the per-token reads are bank-conflict free); GQA logits
//           x_gj = (q_g . k_j) * scale * log2(e)  (Eq. 1, Alg. 1) kept in SMEM for the chunk;
//           invalid slots j >= n are masked (R6).
//   max     exact per-CTA max m_g over the chunk (R5: replaces the paper's dropped running max).
//   V pass  stream V tiles; p_gj = 2^(x_gj - m_g), Z_g += p, o_g += p v_j
//           (P:530-531), lambda_j = ||v_j||_1 from the same tile (Eq. 6; the contribution
//           vector C_j = p v_j is never materialised: ||p v||_1 = p ||v||_1 since p >= 0, R9).
//   combine cluster-wide over DSMEM: M_g = max(m_g,s, x_g*), Z_g = sum_s Z_g,s 2^(m_g,s - M_g)
//           + 2^(x_g* - M_g) (the current token), in rank order (deterministic).
//   scores  I_j = lambda_j / G * sum_g 2^(x_gj - M_g) / Z_g  (Eq. 6 with Alg. 1 P:540's single
//           normalisation, mean over the group R2); the argmin key uses the log2 of the same
//           quantity so fp32 underflow never merges distinct scores.
//   argmin  thread -> warp shuffle -> CTA -> cluster on the 64-bit key (ordered log-score, slot):
//           lowest index on exact ties (R7).
//   write   rank 0: out = (sum_s o_s 2^(m_s - M) + 2^(x* - M) v*) / Z, slot, in-place eviction
//           write of (k*, v*) into the victim (Fig. 2) or append at n (R11).
#include <mutex>

#include "lf_common.cuh"

namespace lf {
namespace {

constexpr int kTT = 64;    // tokens per tile
constexpr int kNT = 256;   // threads per CTA (8 warps)
constexpr int kMaxSmem = 112 * 1024;

__host__ __device__ constexpr int gpad(int G) { return G <= 1 ? 1 : G <= 2 ? 2 : G <= 4 ? 4 : 8; }

// Shared-memory carve-up (bytes), identical on host and device.
struct SimtSmem {
    int tile, qs, red, P, exch_m, exch_z, exch_o, misc, key, X, L, total;
};
__host__ __device__ inline SimtSmem simt_smem(int D, int GP, int G, int chunk) {
    SimtSmem s;
    int off = 0;
    s.tile = off;   off += 2 * kTT * D * 2;            // K or V tiles, double buffered (also O reduction)
    s.qs = off;     off += GP * D * 4;                 // q_g as fp32
    s.red = off;    off += 4 * GP * kTT * 4;           // partial dots of the 4 d-quarters
    s.P = off;      off += GP * kTT * 4;               // p_gj of the current tile
    s.exch_m = off; off += 16 * 4;                     // cluster exchange: m_g
    s.exch_z = off; off += 16 * 4;                     //                   Z_g
    s.exch_o = off; off += GP * D * 4;                 //                   o_g (un-normalised)
    s.misc = off;   off += 128 * 4;                    // x_g*, M_g, log2 Z_g, Z_g, reduction slots
    s.key = off;    off += 16 * 8;                     // argmin keys
    s.X = off;      off += G * chunk * 4;              // x_gj for the chunk (log2 units)
    s.L = off;      off += chunk * 4;                  // lambda_j for the chunk
    s.total = off;
    return s;
}

__device__ __forceinline__ void bf16x8_to_f32(const uint4& w, float* f) {
    f[0] = __uint_as_float(w.x << 16); f[1] = __uint_as_float(w.x & 0xffff0000u);
    f[2] = __uint_as_float(w.y << 16); f[3] = __uint_as_float(w.y & 0xffff0000u);
    f[4] = __uint_as_float(w.z << 16); f[5] = __uint_as_float(w.z & 0xffff0000u);
    f[6] = __uint_as_float(w.w << 16); f[7] = __uint_as_float(w.w & 0xffff0000u);
}

// Stage one tile (vt valid rows starting at slot j0) of a unit's K or V into swizzled SMEM:
// 16-byte chunk c of row r lives at chunk position c ^ (r & 7) of that row.
template <int D>
__device__ __forceinline__ void load_tile(uint16_t* dst, const uint16_t* src_unit, int j0, int vt) {
    constexpr int CPR = D / 8;
    for (int i = threadIdx.x; i < kTT * CPR; i += kNT) {
        int r = i / CPR, c = i % CPR;
        if (r < vt) cp_async16(dst + (r * CPR + (c ^ (r & 7))) * 8, src_unit + (size_t)(j0 + r) * D + c * 8);
    }
    cp_async_commit();
}

template <int D, int GP>
__global__ void __launch_bounds__(kNT) simt_decode_kernel(StepParams p) {
    extern __shared__ __align__(128) unsigned char smem[];
    constexpr int CPR = D / 8;
    const int G = p.G, N = p.N, chunk = p.chunk;
    const SimtSmem so = simt_smem(D, GP, G, chunk);
    uint16_t* tile = (uint16_t*)(smem + so.tile);
    float* qs = (float*)(smem + so.qs);
    float* red = (float*)(smem + so.red);
    float* Ps = (float*)(smem + so.P);
    float* ex_m = (float*)(smem + so.exch_m);
    float* ex_z = (float*)(smem + so.exch_z);
    float* ex_o = (float*)(smem + so.exch_o);
    float* misc = (float*)(smem + so.misc);
    float* wred = misc + 64;       // [64] per-warp reduction slots (misc[0,64) is the finaliser's)
    unsigned long long* keys = (unsigned long long*)(smem + so.key);
    float* X = (float*)(smem + so.X);
    float* Ls = (float*)(smem + so.L);

    cg::cluster_group cluster = cg::this_cluster();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int S = p.splits;
    const int s = (int)cluster.block_rank();
    const int u = blockIdx.x / S;
    const int b = u / p.Hkv, h = u % p.Hkv;
    pdl_trigger();   // the next step's prologue may overlap this step
    pdl_wait();      // the previous step's cache writes are visible from here on
    const int n = p.n_valid[u];
    const int c0 = s * chunk;
    const int c1 = min(c0 + chunk, N);
    const int hi = min(c1, n);
    const int nv = max(0, hi - c0);            // valid tokens of this CTA's chunk
    const int ntiles = (nv + kTT - 1) / kTT;
    const size_t unit_off = (size_t)u * N * D;

    // query group as fp32 (rows g >= G are zero so padded heads contribute nothing)
    for (int i = tid; i < GP * D; i += kNT) {
        int g = i / D, l = i % D;
        qs[i] = g < G ? bf16_to_f32(p.q[((size_t)b * p.Hq + (size_t)h * G + g) * D + l]) : 0.f;
    }
    // ---------------- K pass: logits -------------------------------------------------------
    const uint16_t* Ku = p.K + unit_off;
    if (ntiles > 0) load_tile<D>(tile, Ku, c0, min(kTT, nv));
    __syncthreads();
    {
        const int r = tid % kTT, part = tid / kTT;   // token row and d-quarter of this thread
        for (int t = 0; t < ntiles; ++t) {
            if (t + 1 < ntiles) load_tile<D>(tile + ((t + 1) & 1) * kTT * D, Ku, c0 + (t + 1) * kTT,
                                             min(kTT, nv - (t + 1) * kTT));
            else cp_async_commit();
            cp_async_wait<1>();
            __syncthreads();
            const uint16_t* buf = tile + (t & 1) * kTT * D;
            float acc[GP];
#pragma unroll
            for (int g = 0; g < GP; ++g) acc[g] = 0.f;
#pragma unroll
            for (int i = 0; i < CPR / 4; ++i) {
                const int c = part + 4 * i;
                uint4 w = *(const uint4*)(buf + (r * CPR + (c ^ (r & 7))) * 8);
                float kf[8];
                bf16x8_to_f32(w, kf);
#pragma unroll
                for (int g = 0; g < GP; ++g) {
                    const float4 qa = *(const float4*)(qs + g * D + c * 8);
                    const float4 qb = *(const float4*)(qs + g * D + c * 8 + 4);
                    acc[g] = fmaf(kf[0], qa.x, acc[g]); acc[g] = fmaf(kf[1], qa.y, acc[g]);
                    acc[g] = fmaf(kf[2], qa.z, acc[g]); acc[g] = fmaf(kf[3], qa.w, acc[g]);
                    acc[g] = fmaf(kf[4], qb.x, acc[g]); acc[g] = fmaf(kf[5], qb.y, acc[g]);
                    acc[g] = fmaf(kf[6], qb.z, acc[g]); acc[g] = fmaf(kf[7], qb.w, acc[g]);
                }
            }
#pragma unroll
            for (int g = 0; g < GP; ++g) red[(part * GP + g) * kTT + r] = acc[g];
            __syncthreads();
            const int vt = min(kTT, nv - t * kTT);
            for (int e = tid; e < G * kTT; e += kNT) {
                const int g = e / kTT, rr = e % kTT;
                if (rr < vt) {
                    float dot = ((red[(0 * GP + g) * kTT + rr] + red[(1 * GP + g) * kTT + rr]) +
                                 red[(2 * GP + g) * kTT + rr]) + red[(3 * GP + g) * kTT + rr];
                    X[g * chunk + t * kTT + rr] = dot * p.scale_log2;
                }
            }
        }
    }
    __syncthreads();
    // ---------------- exact per-CTA max ----------------------------------------------------
    for (int g = 0; g < G; ++g) {
        float m = -INFINITY;
        for (int j = tid; j < nv; j += kNT) m = fmaxf(m, X[g * chunk + j]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        if (lane == 0) wred[warp * 8 + (g & 7)] = m;
        if ((g & 7) == 7 || g == G - 1) {
            __syncthreads();
            if (tid <= (g & 7)) {
                float mm = -INFINITY;
                for (int w = 0; w < 8; ++w) mm = fmaxf(mm, wred[w * 8 + tid]);
                ex_m[(g & ~7) + tid] = mm;
            }
            __syncthreads();
        }
    }
    // ---------------- V pass: p, Z, PV, lambda ---------------------------------------------
    const uint16_t* Vu = p.V + unit_off;
    if (ntiles > 0) load_tile<D>(tile, Vu, c0, min(kTT, nv));
    constexpr int KSTEP = kNT / CPR;      // rows handled per pass by one d-chunk column
    const int pc = tid % CPR, pk = tid / CPR;
    float o[GP][8];
#pragma unroll
    for (int g = 0; g < GP; ++g)
#pragma unroll
        for (int e = 0; e < 8; ++e) o[g][e] = 0.f;
    float zacc[(GP + 3) / 4];
#pragma unroll
    for (int k = 0; k < (GP + 3) / 4; ++k) zacc[k] = 0.f;
    for (int t = 0; t < ntiles; ++t) {
        if (t + 1 < ntiles) load_tile<D>(tile + ((t + 1) & 1) * kTT * D, Vu, c0 + (t + 1) * kTT,
                                         min(kTT, nv - (t + 1) * kTT));
        else cp_async_commit();
        const int vt = min(kTT, nv - t * kTT);
        // p_gj = 2^(x_gj - m_g) for the tile (thread (tid/64 + 4k) owns head g)
#pragma unroll
        for (int k = 0; k < (GP + 3) / 4; ++k) {
            const int e = tid + k * kNT;
            if (e < GP * kTT) {
                const int g = e / kTT, rr = e % kTT;
                float pv = 0.f;
                if (g < G && rr < vt) pv = exp2f(X[g * chunk + t * kTT + rr] - ex_m[g]);
                Ps[e] = pv;
                zacc[k] += pv;
            }
        }
        cp_async_wait<1>();
        __syncthreads();
        const uint16_t* buf = tile + (t & 1) * kTT * D;
#pragma unroll
        for (int i = 0; i < kTT / KSTEP; ++i) {
            const int r = pk + KSTEP * i;
            float lam = 0.f;
            if (r < vt) {
                uint4 w = *(const uint4*)(buf + (r * CPR + (pc ^ (r & 7))) * 8);
                float vf[8];
                bf16x8_to_f32(w, vf);
#pragma unroll
                for (int e = 0; e < 8; ++e) lam += fabsf(vf[e]);
#pragma unroll
                for (int g = 0; g < GP; ++g) {
                    const float pg = Ps[g * kTT + r];
#pragma unroll
                    for (int e = 0; e < 8; ++e) o[g][e] = fmaf(pg, vf[e], o[g][e]);
                }
            }
#pragma unroll
            for (int off = CPR / 2; off > 0; off >>= 1) lam += __shfl_xor_sync(0xffffffffu, lam, off);
            if (pc == 0 && r < vt) Ls[t * kTT + r] = lam;
        }
        __syncthreads();
    }
    // ---------------- reduce o over the rows, Z over the tokens ----------------------------
    {
        // lanes sharing a d-chunk inside the warp: pc = lane % CPR
#pragma unroll
        for (int g = 0; g < GP; ++g)
#pragma unroll
            for (int e = 0; e < 8; ++e)
#pragma unroll
                for (int off = CPR; off < 32; off <<= 1) o[g][e] += __shfl_xor_sync(0xffffffffu, o[g][e], off);
        float* obuf = (float*)tile;   // [8 warps][GP][D]
        if (lane < CPR) {
#pragma unroll
            for (int g = 0; g < GP; ++g)
#pragma unroll
                for (int e = 0; e < 8; ++e) obuf[(warp * GP + g) * D + pc * 8 + e] = o[g][e];
        }
#pragma unroll
        for (int k = 0; k < (GP + 3) / 4; ++k) {
            float z = zacc[k];
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) z += __shfl_xor_sync(0xffffffffu, z, off);
            if (lane == 0) wred[warp * 4 + k] = z;   // warp w holds head g = w/2 + 4k
        }
        __syncthreads();
        for (int i = tid; i < GP * D; i += kNT) {
            float acc = 0.f;
#pragma unroll
            for (int w = 0; w < 8; ++w) acc += obuf[w * GP * D + i];
            ex_o[i] = acc;
        }
        if (tid < G) {
            const int g = tid, k = g / 4, w = 2 * (g % 4);
            ex_z[g] = wred[w * 4 + k] + wred[(w + 1) * 4 + k];
        }
    }
    Partials pt{ex_m, ex_z, ex_o, X, Ls, misc, keys};
    cluster_finalize<D, GP, kNT>(p, pt, u, n, c0, c1, nv);
}

template <int D, int GP>
cudaError_t launch_t(const StepParams& p, const Plan& plan, cudaStream_t stream) {
    auto kern = simt_decode_kernel<D, GP>;
    // kernel attributes are per device: set once to the largest values any plan uses, under a lock
    // (host-side, outside any stream capture; concurrent cache creation is race-free)
    static std::mutex mu;
    static bool done[64] = {false};
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev >= 64) return cudaErrorInvalidDevice;
    {
        std::lock_guard<std::mutex> lock(mu);
        if (!done[dev]) {
            e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem);
            if (e == cudaSuccess) e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
            if (e != cudaSuccess) return e;
            done[dev] = true;
        }
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(plan.splits * p.B * p.Hkv, 1, 1);   // cluster (splits,1,1) = one unit
    cfg.blockDim = dim3(kNT, 1, 1);
    cfg.dynamicSmemBytes = plan.smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    cfg.numAttrs = fill_launch_attrs(attr, plan.splits);
    cfg.attrs = attr;
    return cudaLaunchKernelEx(&cfg, kern, p);
}

}  // namespace

bool simt_supported(int G, int d) { return G >= 1 && G <= 8 && (d == 64 || d == 128); }

Plan simt_plan(int units, int G, int d, int N, int split_tokens, int num_sms) {
    Plan pl;
    pl.kernel = LF_KERNEL_SIMT;
    pl.clusters = 0;
    pl.stages = 2;
    pl.tmem_cols = 0;
    pl.solo_rounds = 0;
    pl.lat = 0;
    const int GP = gpad(G);
    const int fixed = simt_smem(d, GP, G, 0).total;
    int chunk_max = (kMaxSmem - fixed) / ((G + 1) * 4) / 128 * 128;
    if (chunk_max > 4096) chunk_max = 4096;
    const int Nr = (N + 127) / 128 * 128;
    int chunk;
    if (split_tokens > 0) {
        chunk = split_tokens;
    } else {
        // ~4 CTAs per SM in flight over the step; at most 8 CTAs per cluster unless N forces more
        int want = (4 * num_sms + units - 1) / units;
        int smin = (Nr + chunk_max - 1) / chunk_max;
        int S = want > smin ? want : smin;
        int cap = smin > 8 ? 16 : 8;
        if (S > cap) S = cap;
        chunk = ((Nr + S - 1) / S + 127) / 128 * 128;
        if (chunk < 128) chunk = 128;
    }
    pl.chunk = chunk;
    pl.splits = (N + chunk - 1) / chunk;
    if (chunk > chunk_max) pl.splits = -1;   // does not fit shared memory
    pl.smem = simt_smem(d, GP, G, chunk).total;
    return pl;
}

cudaError_t simt_launch(const StepParams& p, const Plan& plan, cudaStream_t stream) {
    const int GP = gpad(p.G);
    if (p.d == 128) {
        switch (GP) {
            case 1: return launch_t<128, 1>(p, plan, stream);
            case 2: return launch_t<128, 2>(p, plan, stream);
            case 4: return launch_t<128, 4>(p, plan, stream);
            default: return launch_t<128, 8>(p, plan, stream);
        }
    }
    switch (GP) {
        case 1: return launch_t<64, 1>(p, plan, stream);
        case 2: return launch_t<64, 2>(p, plan, stream);
        case 4: return launch_t<64, 4>(p, plan, stream);
        default: return launch_t<64, 8>(p, plan, stream);
    }
}

}  // namespace lf
