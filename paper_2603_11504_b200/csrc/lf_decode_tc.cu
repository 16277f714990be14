// TMA + tcgen05 split-KV LongFlow decode step for head_dim 128 and 2 <= G <= 8 (B200, sm_100a).
//
// One thread-block cluster per unit u = (sequence, kv head); CTA s owns slots [s*chunk, (s+1)*chunk)
// and streams them in 128-token tiles (K tiles first, then V tiles) through a 2-stage TMA ring
// (SWIZZLE_128B, two 64-column boxes per tile).  Warp roles (192 threads):
//   warp 0     TMA producer (one elected lane)
//   warp 1     TMEM allocator + tcgen05.mma issuer (one lane)
//   warps 2-5  softmax / score / epilogue warps; warp w owns TMEM lanes [32(w%4), 32(w%4)+32)
//
// K pass   S^T[128 tok x 16] = K_tile[128 x 128] . Q^T[128 x 16]  (M=128, N=16, K=128; K-major A/B),
//          fp32 in TMEM (double buffered); the softmax warps move x_gj = S*scale*log2e to SMEM
//          (Alg. 1) and track the exact per-CTA max (R5).
// V pass   P_g = 2^(x_g - m_g) split into bf16 hi + lo (N = 16 = 8 hi rows + 8 lo rows: bf16 P alone
//          misses the 2e-3 output bar), O^T[128 d x 16] += V^T[d x 128 tok] . P^T
//          (M=128, N=16, K=16 per MMA, A MN-major straight from the TMA tile); lambda_j = ||v_j||_1
//          from the same tile on the CUDA cores (Eq. 6, R9).  Invalid rows of the last tile are
//          zeroed in SMEM before the MMA reads them.
// Then the shared cluster finalisation (lf_common.cuh): DSMEM combine, scores, argmin, eviction.
#include <cuda.h>
#include <cudaTypedefs.h>

#include "lf_common.cuh"
#include "lf_tc_ptx.cuh"

namespace lf {
namespace {

constexpr int kStages = 2;
constexpr int kNT = 192;
constexpr int kStageBytes = 32768;   // 128 tokens x 128 d x bf16 (two 16 KB boxes)
constexpr int kBoxBytes = 16384;
constexpr int kMaxSmem = 110 * 1024; // two CTAs per SM
constexpr uint32_t kTmemCols = 64;   // S double buffer (2 x 16) + O (16), power of two

struct TcArgs {
    CUtensorMap tmK;
    CUtensorMap tmV;
    StepParams p;
};

struct TcSmem {
    int ring, q, pbuf, X, L, exo, exm, exz, misc, keys, red, bars, tmem, total;
};
__host__ __device__ inline TcSmem tc_smem(int G, int GP, int chunk) {
    TcSmem s;
    int off = 0;
    s.ring = off; off += kStages * kStageBytes;   // 1024-aligned (swizzle atoms)
    s.q = off;    off += 4096;                    // Q^T operand: 16 rows x 128 d, 2 boxes of 2 KB
    s.pbuf = off; off += 2 * 4096;                // P^T operand, double buffered: 16 rows x 128 tok
    s.X = off;    off += G * chunk * 4;
    s.L = off;    off += chunk * 4;
    s.exo = off;  off += GP * 128 * 4;
    s.exm = off;  off += 64;
    s.exz = off;  off += 64;
    s.misc = off; off += 128 * 4;
    s.keys = off; off += 16 * 8;
    s.red = off;  off += 2 * 4 * 16 * 4;
    s.bars = off; off += 16 * 8;
    s.tmem = off; off += 16;
    s.total = off + 1024;                         // slack for 1024-byte alignment of the base
    return s;
}

// barrier slots
constexpr int FULL = 0, EMPTY = 2, SFULL = 4, SFREE = 6, PREADY = 8, PFREE = 10, OFULL = 12;

__device__ __forceinline__ float habs_sum8(const uint4& w) {
    return (fabsf(__uint_as_float(w.x << 16)) + fabsf(__uint_as_float(w.x & 0xffff0000u))) +
           (fabsf(__uint_as_float(w.y << 16)) + fabsf(__uint_as_float(w.y & 0xffff0000u))) +
           (fabsf(__uint_as_float(w.z << 16)) + fabsf(__uint_as_float(w.z & 0xffff0000u))) +
           (fabsf(__uint_as_float(w.w << 16)) + fabsf(__uint_as_float(w.w & 0xffff0000u)));
}

template <int GP>
__global__ void __launch_bounds__(kNT, 2) tc_decode_kernel(const __grid_constant__ TcArgs a) {
    extern __shared__ unsigned char smem_raw[];
    const StepParams& p = a.p;
    // 1024-byte aligned base for the swizzle-128B atoms; offset arithmetic on the __shared__
    // pointer keeps the accesses in the shared state space (STS/LDS, not generic ST/LD)
    unsigned char* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
    const int G = p.G, N = p.N, chunk = p.chunk;
    const TcSmem so = tc_smem(G, GP, chunk);
    float* X = (float*)(smem + so.X);
    float* Ls = (float*)(smem + so.L);
    float* ex_o = (float*)(smem + so.exo);
    float* ex_m = (float*)(smem + so.exm);
    float* ex_z = (float*)(smem + so.exz);
    float* misc = (float*)(smem + so.misc);
    float* red = (float*)(smem + so.red);
    unsigned long long* keys = (unsigned long long*)(smem + so.keys);
    const uint32_t ring = ptx::smem_u32(smem + so.ring);
    const uint32_t qs = ptx::smem_u32(smem + so.q);
    const uint32_t pbuf = ptx::smem_u32(smem + so.pbuf);
    const uint32_t bars = ptx::smem_u32(smem + so.bars);
    auto BAR = [&](int i) { return bars + 8u * (uint32_t)i; };

    cg::cluster_group cluster = cg::this_cluster();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int S = p.splits;
    const int u = blockIdx.x / S;
    const int s = (int)cluster.block_rank();
    const int b = u / p.Hkv, h = u % p.Hkv;
    const int n = p.n_valid[u];
    const int c0 = s * chunk;
    const int c1 = min(c0 + chunk, N);
    const int nv = max(0, min(c1, n) - c0);
    const int ntiles = (nv + 127) / 128;

    if (tid == 0) {
        for (int i = 0; i < kStages; ++i) {
            ptx::mbar_init(BAR(FULL + i), 1);      // producer's expect_tx arrival
            ptx::mbar_init(BAR(EMPTY + i), 5);     // MMA commit + 4 softmax warps
        }
        for (int i = 0; i < 2; ++i) {
            ptx::mbar_init(BAR(SFULL + i), 1);
            ptx::mbar_init(BAR(SFREE + i), 4);
            ptx::mbar_init(BAR(PREADY + i), 4);
            ptx::mbar_init(BAR(PFREE + i), 1);
        }
        ptx::mbar_init(BAR(OFULL), 1);
        ptx::fence_mbar_init();
        ptx::tma_prefetch_desc(&a.tmK);
        ptx::tma_prefetch_desc(&a.tmV);
    }
    if (warp == 1) ptx::tmem_alloc<kTmemCols>(ptx::smem_u32(smem + so.tmem));
    if (warp >= 2) {
        // Q^T as the K-major SW128 B operand: row n (query head, zero for n >= G), column k (d);
        // 16-byte chunk (k%64)/8 of row n sits at chunk position ((k%64)/8) ^ (n%8)
        const int sidx = tid - 64;
        uint16_t* qsm = (uint16_t*)(smem + so.q);
        for (int e = sidx; e < 16 * 128; e += 128) {
            const int row = e >> 7, col = e & 127, cc = col & 63;
            const uint16_t v = row < G ? p.q[((size_t)b * p.Hq + (size_t)h * G + row) * 128 + col] : (uint16_t)0;
            qsm[((col >> 6) * 2048 + row * 128 + ((((cc >> 3) ^ (row & 7)) << 4)) + (cc & 7) * 2) >> 1] = v;
        }
        uint4* pz = (uint4*)(smem + so.pbuf);
        for (int e = sidx; e < 2 * 4096 / 16; e += 128) pz[e] = make_uint4(0, 0, 0, 0);
        ptx::fence_proxy_async_smem();
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *(volatile uint32_t*)(smem + so.tmem);

    if (warp == 0) {
        // ------------------------------ TMA producer ------------------------------------------
        if (lane == 0) {
            for (int i = 0; i < 2 * ntiles; ++i) {
                const int st = i % kStages;
                const uint32_t ph = (uint32_t)(i / kStages) & 1u;
                ptx::mbar_wait(BAR(EMPTY + st), ph ^ 1u);
                ptx::mbar_arrive_expect_tx(BAR(FULL + st), kStageBytes);
                const int tile = i < ntiles ? i : i - ntiles;
                const int row = u * N + c0 + tile * 128;
                const void* tm = i < ntiles ? (const void*)&a.tmK : (const void*)&a.tmV;
                const uint32_t dst = ring + (uint32_t)st * kStageBytes;
                ptx::tma_load_2d(dst, tm, BAR(FULL + st), 0, row);
                ptx::tma_load_2d(dst + kBoxBytes, tm, BAR(FULL + st), 64, row);
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        // ------------------------------ MMA issuer --------------------------------------------
        if (lane == 0) {
            constexpr uint32_t idesc_qk = ptx::idesc_bf16_f32(128, 16, 0, 0);
            constexpr uint32_t idesc_pv = ptx::idesc_bf16_f32(128, 16, 1, 0);
            for (int i = 0; i < ntiles; ++i) {          // S^T = K_tile . Q^T
                const int st = i % kStages;
                ptx::mbar_wait(BAR(FULL + st), (uint32_t)(i / kStages) & 1u);
                const int sb = i & 1;
                ptx::mbar_wait(BAR(SFREE + sb), ((uint32_t)(i >> 1) & 1u) ^ 1u);
                ptx::tc_fence_after();
                const uint32_t base = ring + (uint32_t)st * kStageBytes;
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const uint64_t da = ptx::smem_desc_sw128(base + (kk >> 2) * kBoxBytes + (kk & 3) * 32, 16, 1024);
                    const uint64_t db = ptx::smem_desc_sw128(qs + (kk >> 2) * 2048 + (kk & 3) * 32, 16, 1024);
                    ptx::mma_bf16(tmem + (uint32_t)sb * 16, da, db, idesc_qk, kk > 0);
                }
                ptx::mma_commit(BAR(SFULL + sb));
                ptx::mma_commit(BAR(EMPTY + st));
            }
            for (int i = 0; i < ntiles; ++i) {          // O^T += V^T . P^T
                const int j = ntiles + i, st = j % kStages;
                ptx::mbar_wait(BAR(FULL + st), (uint32_t)(j / kStages) & 1u);
                const int pb = i & 1;
                ptx::mbar_wait(BAR(PREADY + pb), (uint32_t)(i >> 1) & 1u);
                ptx::tc_fence_after();
                const uint32_t base = ring + (uint32_t)st * kStageBytes;
                const uint32_t pbase = pbuf + (uint32_t)pb * 4096;
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const uint64_t da = ptx::smem_desc_sw128(base + kk * 2048, kBoxBytes, 1024);
                    const uint64_t db = ptx::smem_desc_sw128(pbase + (kk >> 2) * 2048 + (kk & 3) * 32, 16, 1024);
                    ptx::mma_bf16(tmem + 32, da, db, idesc_pv, (i | kk) > 0);
                }
                ptx::mma_commit(BAR(EMPTY + st));
                ptx::mma_commit(BAR(PFREE + pb));
            }
            ptx::mma_commit(BAR(OFULL));
        }
        __syncwarp();
    } else {
        // ------------------------------ softmax / score warps ----------------------------------
        const int q4 = warp & 3;
        const int row = 32 * q4 + lane;                 // TMEM lane = token row of the tile / d index
        const uint32_t tl = tmem + ((uint32_t)(32 * q4) << 16);
        float mloc[GP];
#pragma unroll
        for (int g = 0; g < GP; ++g) mloc[g] = -INFINITY;
        for (int i = 0; i < ntiles; ++i) {
            const int st = i % kStages, sb = i & 1;
            ptx::mbar_wait(BAR(SFULL + sb), (uint32_t)(i >> 1) & 1u);
            ptx::tc_fence_after();
            uint32_t r[8];
            ptx::tmem_ld_x8(tl + (uint32_t)sb * 16, r);
            ptx::tmem_ld_wait();
            const int tok = i * 128 + row;
            const bool valid = tok < nv;
#pragma unroll
            for (int g = 0; g < GP; ++g) {
                if (g < G) {
                    const float x = valid ? __uint_as_float(r[g]) * p.scale_log2 : -INFINITY;
                    X[g * chunk + tok] = x;
                    mloc[g] = fmaxf(mloc[g], x);
                }
            }
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                ptx::mbar_arrive(BAR(SFREE + sb));
                ptx::mbar_arrive(BAR(EMPTY + st));
            }
        }
        // exact per-CTA max over the 128 softmax threads
#pragma unroll
        for (int g = 0; g < GP; ++g) {
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) mloc[g] = fmaxf(mloc[g], __shfl_xor_sync(0xffffffffu, mloc[g], off));
        }
        if (lane == 0) {
#pragma unroll
            for (int g = 0; g < GP; ++g) red[q4 * 16 + g] = mloc[g];
        }
        ptx::named_bar_sync(1, 128);
        float m[GP];
#pragma unroll
        for (int g = 0; g < GP; ++g)
            m[g] = fmaxf(fmaxf(red[0 * 16 + g], red[1 * 16 + g]), fmaxf(red[2 * 16 + g], red[3 * 16 + g]));
        if (tid == 64) {
#pragma unroll
            for (int g = 0; g < GP; ++g)
                if (g < G) ex_m[g] = m[g];
        }
        float z[GP];
#pragma unroll
        for (int g = 0; g < GP; ++g) z[g] = 0.f;
        const int box = row >> 6, cc = row & 63;
        for (int i = 0; i < ntiles; ++i) {
            const int pb = i & 1;
            ptx::mbar_wait(BAR(PFREE + pb), ((uint32_t)(i >> 1) & 1u) ^ 1u);
            const int tok = i * 128 + row;
            const bool valid = tok < nv;
            unsigned char* P = smem + so.pbuf + pb * 4096 + box * 2048;
#pragma unroll
            for (int g = 0; g < GP; ++g) {
                if (g < G) {
                    const float pv = valid ? exp2f(X[g * chunk + tok] - m[g]) : 0.f;
                    z[g] += pv;
                    const uint16_t hi = f32_to_bf16_rne(pv);
                    const uint16_t lo = f32_to_bf16_rne(pv - bf16_to_f32(hi));
                    *(uint16_t*)(P + g * 128 + ((((cc >> 3) ^ g) & 7) << 4) + (cc & 7) * 2) = hi;
                    *(uint16_t*)(P + (8 + g) * 128 + ((((cc >> 3) ^ (8 + g)) & 7) << 4) + (cc & 7) * 2) = lo;
                }
            }
            const int j = ntiles + i, st = j % kStages;
            ptx::mbar_wait(BAR(FULL + st), (uint32_t)(j / kStages) & 1u);   // V tile landed
            unsigned char* Vt = smem + so.ring + st * kStageBytes;
            if (!valid) {   // rows past n may hold stale data: P = 0 must not meet Inf/NaN
#pragma unroll
                for (int bb = 0; bb < 2; ++bb)
#pragma unroll
                    for (int c = 0; c < 8; ++c)
                        *(uint4*)(Vt + bb * kBoxBytes + row * 128 + c * 16) = make_uint4(0, 0, 0, 0);
            }
            ptx::fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(BAR(PREADY + pb));
            float lam = 0.f;
            if (valid) {
#pragma unroll
                for (int bb = 0; bb < 2; ++bb)
#pragma unroll
                    for (int c = 0; c < 8; ++c)
                        lam += habs_sum8(*(const uint4*)(Vt + bb * kBoxBytes + row * 128 + ((c ^ (row & 7)) << 4)));
            }
            Ls[tok] = lam;
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(BAR(EMPTY + st));
        }
        // Z over the 128 softmax threads (fixed order)
#pragma unroll
        for (int g = 0; g < GP; ++g) {
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) z[g] += __shfl_xor_sync(0xffffffffu, z[g], off);
        }
        if (lane == 0) {
#pragma unroll
            for (int g = 0; g < GP; ++g) red[64 + q4 * 16 + g] = z[g];
        }
        ptx::named_bar_sync(1, 128);
        if (tid == 64) {
            for (int g = 0; g < G; ++g)
                ex_z[g] = ((red[64 + 0 * 16 + g] + red[64 + 1 * 16 + g]) + red[64 + 2 * 16 + g]) + red[64 + 3 * 16 + g];
        }
        // un-normalised O^T from TMEM: this thread's lane is d = row
        ptx::mbar_wait(BAR(OFULL), 0);
        ptx::tc_fence_after();
        if (ntiles > 0) {
            uint32_t o[16];
            ptx::tmem_ld_x16(tl + 32, o);
            ptx::tmem_ld_wait();
#pragma unroll
            for (int g = 0; g < GP; ++g)
                if (g < G) ex_o[g * 128 + row] = __uint_as_float(o[g]) + __uint_as_float(o[8 + g]);
        } else {
            for (int g = 0; g < G; ++g) ex_o[g * 128 + row] = 0.f;
        }
        ptx::tc_fence_before();
    }
    __syncthreads();
    Partials pt{ex_m, ex_z, ex_o, X, Ls, misc, keys};
    cluster_finalize<128, GP, kNT>(p, pt, u, n, c0, c1, nv);
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<kTmemCols>(tmem);
    }
}

template <int GP>
cudaError_t launch_t(const TcArgs& args, const Plan& plan, cudaStream_t stream) {
    auto kern = tc_decode_kernel<GP>;
    static int smem_set[64] = {0};
    static bool np_set[64] = {false};
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 64 && plan.smem > smem_set[dev]) {
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, plan.smem);
        if (e != cudaSuccess) return e;
        smem_set[dev] = plan.smem;
    }
    if (plan.splits > 8 && dev < 64 && !np_set[dev]) {
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return e;
        np_set[dev] = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(plan.splits * args.p.B * args.p.Hkv, 1, 1);
    cfg.blockDim = dim3(kNT, 1, 1);
    cfg.dynamicSmemBytes = plan.smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = plan.splits;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, args);
}

__host__ __device__ constexpr int gpad_tc(int G) { return G <= 4 ? 4 : 8; }

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (PFN_cuTensorMapEncodeTiled_v12000)f;
    }
    return fn;
}

bool encode_2d(CUtensorMap* m, void* base, uint64_t rows, int d) {
    auto fn = get_encode();
    if (!fn) return false;
    cuuint64_t dims[2] = {(cuuint64_t)d, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)d * 2};
    cuuint32_t box[2] = {64, 128};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

}  // namespace

bool tc_supported(int G, int d) { return d == 128 && G >= 2 && G <= 8; }

Plan tc_plan(int units, int G, int d, int N, int split_tokens, int num_sms) {
    Plan pl;
    pl.kernel = LF_KERNEL_TCGEN05;
    const int GP = gpad_tc(G);
    const int fixed = tc_smem(G, GP, 0).total;
    int chunk_max = (kMaxSmem - fixed) / ((G + 1) * 4) / 128 * 128;
    if (chunk_max < 128) chunk_max = 128;
    const int Nr = (N + 127) / 128 * 128;
    int chunk;
    if (split_tokens > 0) {
        chunk = split_tokens;
    } else {
        int want = (2 * num_sms + units - 1) / units;        // >= one wave of 2 CTAs per SM
        int smin = (Nr + chunk_max - 1) / chunk_max;
        int S = want > smin ? want : smin;
        int cap = smin > 8 ? 16 : 8;
        if (S > cap) S = cap;
        chunk = ((Nr + S - 1) / S + 127) / 128 * 128;
    }
    pl.chunk = chunk;
    pl.splits = (N + chunk - 1) / chunk;
    pl.smem = tc_smem(G, GP, chunk).total;
    if (pl.smem > 227 * 1024) pl.splits = -1;
    (void)d;
    return pl;
}

bool tc_make_maps(TcMaps* maps, void* K, void* V, long long units, int N, int d) {
    static_assert(sizeof(CUtensorMap) <= sizeof(maps->k), "tensor map size");
    return encode_2d((CUtensorMap*)maps->k, K, (uint64_t)units * (uint64_t)N, d) &&
           encode_2d((CUtensorMap*)maps->v, V, (uint64_t)units * (uint64_t)N, d);
}

cudaError_t tc_launch(const StepParams& p, const Plan& plan, const TcMaps& maps, cudaStream_t stream) {
    TcArgs args;
    memcpy(&args.tmK, maps.k, sizeof(CUtensorMap));
    memcpy(&args.tmV, maps.v, sizeof(CUtensorMap));
    args.p = p;
    if (gpad_tc(p.G) == 4) return launch_t<4>(args, plan, stream);
    return launch_t<8>(args, plan, stream);
}

}  // namespace lf
