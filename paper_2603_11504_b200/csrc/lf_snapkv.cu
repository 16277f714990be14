// SnapKV prefill compression (NEXT-f3; "if the number of tokens in the prefill stage exceeds
// the budget, we first use SnapKV to compress the tokens to the budget size").  Readings R22-R24
// (DESIGN.md): rows r = (g, k) are the G query heads x the last w prompt positions p_k = n-w+k;
// row r attends causally (tokens <= p_k); score_i = mean_r alpha_{r,i} over prefix tokens i < n-w;
// pooled = 1-D max pool (odd kernel, 'same'); keep the (budget - w) largest pooled (ties: lower
// index) plus the w window tokens, ascending, into slots [0, budget).
//
// Kernels (per sequence, one launch each):
//   snapkv_logits_tc grid (Hkv, tiles of 128 tokens), 128 threads: K tile and the observation rows
//                   -> SW128 SMEM, one tcgen05 MMA chain into TMEM; pass 0 writes per-tile per-row
//                   (max, sum exp); pass 1 (after snapkv_rowstats) writes score_i
//   snapkv_rowstats grid (Hkv, R/32): combine the per-tile (max, sum) of every row
//   snapkv_pool     grid (np/256, Hkv): 1-D max pool of the scores
//   snapkv_select   grid Hkv, 1024 threads: radix select of the (budget-w)-th largest pooled value,
//                   ascending compaction of the kept indices
//   snapkv_gather   grid (N*d/8/256, Hkv): kept K/V rows -> cache slots [0, N), n_valid = N
#include <float.h>

#include "lf_common.cuh"
#include "lf_tc_ptx.cuh"

namespace lf {
namespace {

constexpr int kTile = 128;
constexpr int kRowsMax = 128;   // G * w (observation rows per kv head)

struct SnapParams {
    const uint16_t* k;      // bf16 [Hkv][n][d]
    const uint16_t* v;
    const uint16_t* q_obs;  // bf16 [Hq][w][d]
    uint16_t* K;            // cache [B][Hkv][N][d]
    uint16_t* V;
    int32_t* n_valid;       // [B][Hkv]
    int32_t* kept;          // [Hkv][N] or nullptr
    float* part;            // [Hkv][tiles][R][2] per-tile (max, sum 2^(t - max)) in log2 units
    float* rows;            // [Hkv][R] log2 of the row softmax denominators (M + log2 Z, log2 units)
    float* score;           // [Hkv][np]
    float* pooled;          // [Hkv][np]
    int32_t* kidx;          // [Hkv][N] scratch
    int seq, Hkv, G, d, n, w, ks, N, tiles;
    float scale;
};

// Both logits passes run on the tensor core (tcgen05, kind::f16, fp32 accumulate in TMEM): the
// window-query rows x prompt keys product is a dense [R x d] . [d x 128] contraction per tile.
// SMEM operands are K-major SWIZZLE_128B panels of 64 columns (128 rows x 128 B = 16 KB per panel):
// the K tile (128 tokens) and the R <= 128 observation rows (zero padded to 128).
//   pass 0: D[128 rows r][128 tokens] = Qo . K^T  (A = Qo, B = K tile): thread = row r, its max and
//           sum of exp over the tile's causally visible tokens are thread-local
//   pass 1: D[128 tokens][R] = K . Qo^T  (A = K tile, B = Qo): thread = token i < n-w, its score
//           sum_r exp(s_ri - M_r) / Z_r is thread-local (prefix tokens are visible to every row)
constexpr int kPanelBytes = kTile * 128;

// rows [0, rows_valid) of a [rows][D] bf16 matrix -> SW128 K-major panels by cp.async (all copies in
// flight at once); rows past rows_valid are zero-filled
__device__ __forceinline__ void stage_rows_sw128(unsigned char* dst, const uint16_t* src, int rows_valid, int D,
                                                 int tid, int nthreads) {
    const int cpr = D / 8;   // 16-byte chunks per row
    for (int e = tid; e < kTile * cpr; e += nthreads) {
        const int r = e / cpr, c = e % cpr;
        unsigned char* d = dst + (c >> 3) * kPanelBytes + r * 128 + (((c & 7) ^ (r & 7)) << 4);
        if (r < rows_valid) cp_async16(d, src + (size_t)r * D + c * 8);
        else *(uint4*)d = make_uint4(0, 0, 0, 0);
    }
}

template <int D>
__global__ void __launch_bounds__(128) snapkv_logits_tc(SnapParams p, int pass) {
    extern __shared__ unsigned char smem_raw[];
    unsigned char* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
    constexpr int KP = D / 64;
    unsigned char* kt = smem;                          // K tile, KP panels
    unsigned char* qo = smem + KP * kPanelBytes;       // observation rows, KP panels
    float* rs = (float*)(qo + KP * kPanelBytes);       // [kRowsMax][2] (M_r, 1/Z_r) for pass 1
    uint32_t* tslot = (uint32_t*)(rs + 2 * kRowsMax);
    const uint32_t bar = ptx::smem_u32(tslot + 2);
    const int h = blockIdx.x, t = blockIdx.y;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int R = p.G * p.w, n = p.n, np = n - p.w;
    const int i0 = t * kTile;
    if (tid == 0) {
        ptx::mbar_init(bar, 1);
        ptx::fence_mbar_init();
    }
    if (warp == 0) ptx::tmem_alloc(ptx::smem_u32(tslot), 128);
    stage_rows_sw128(kt, p.k + ((size_t)h * n + i0) * D, min(kTile, n - i0), D, tid, 128);
    stage_rows_sw128(qo, p.q_obs + (size_t)h * R * D, R, D, tid, 128);
    if (pass == 1)   // per-row offset M_r + log2 Z_r (log2 units)
        for (int r = tid; r < R; r += 128) rs[r] = p.rows[(size_t)h * R + r];
    cp_async_commit();
    cp_async_wait<0>();
    ptx::fence_proxy_async_smem();   // generic-proxy SMEM writes -> visible to the tensor core
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *(volatile uint32_t*)tslot;
    if (tid == 0) {
        const uint32_t a = ptx::smem_u32(pass == 0 ? qo : kt), b = ptx::smem_u32(pass == 0 ? kt : qo);
        const int NR = pass == 0 ? kTile : (R + 15) / 16 * 16;
        const uint32_t idesc = ptx::idesc_bf16_f32(128, NR, 0, 0);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t off = (uint32_t)((kk >> 2) * kPanelBytes + (kk & 3) * 32);
            ptx::mma_bf16(tmem, ptx::smem_desc_sw128(a + off, 16, 1024), ptx::smem_desc_sw128(b + off, 16, 1024),
                          idesc, kk > 0);
        }
        ptx::mma_commit(bar);
    }
    ptx::mbar_wait(bar, 0);
    ptx::tc_fence_after();
    const uint32_t tl = tmem + ((uint32_t)(32 * warp) << 16);   // this warp's 32 TMEM lanes
    const int lrow = 32 * warp + lane;                           // TMEM lane of this thread
    const float sl2 = p.scale * 1.4426950408889634f;            // logits in log2 units
    if (pass == 0) {
        // thread = observation row r; columns = the tile's tokens
        const int r = lrow;
        const int pos = np + (r % p.w);
        const int jmax = min(kTile, min(n, pos + 1) - i0);       // visible tokens j < jmax
        float m = -INFINITY;
        for (int c0 = 0; c0 < kTile; c0 += 16) {
            uint32_t v[16];
            ptx::tmem_ld_x16(tl + (uint32_t)c0, v);
            ptx::tmem_ld_wait();
            if (c0 + 16 <= jmax) {
#pragma unroll
                for (int j = 0; j < 16; ++j) m = fmaxf(m, __uint_as_float(v[j]));
            } else {
#pragma unroll
                for (int j = 0; j < 16; ++j)
                    if (c0 + j < jmax) m = fmaxf(m, __uint_as_float(v[j]));
            }
        }
        m *= sl2;   // scale > 0: the max commutes with the scaling
        float z = 0.f;
        for (int c0 = 0; c0 < kTile; c0 += 16) {
            uint32_t v[16];
            ptx::tmem_ld_x16(tl + (uint32_t)c0, v);
            ptx::tmem_ld_wait();
            if (c0 + 16 <= jmax) {
#pragma unroll
                for (int j = 0; j < 16; ++j) z += ptx::ex2_approx(fmaf(__uint_as_float(v[j]), sl2, -m));
            } else {
#pragma unroll
                for (int j = 0; j < 16; ++j)
                    if (c0 + j < jmax) z += ptx::ex2_approx(fmaf(__uint_as_float(v[j]), sl2, -m));
            }
        }
        if (r < R) {
            float* pr = p.part + (((size_t)h * p.tiles + t) * R + r) * 2;
            pr[0] = m;
            pr[1] = z;
        }
    } else {
        // thread = token i; columns = observation rows; alpha_ri = 2^(t_ri - (M_r + log2 Z_r))
        const int i = i0 + lrow;
        float acc = 0.f;
        for (int c0 = 0; c0 < R; c0 += 16) {
            uint32_t v[16];
            ptx::tmem_ld_x16(tl + (uint32_t)c0, v);
            ptx::tmem_ld_wait();
            if (c0 + 16 <= R) {
#pragma unroll
                for (int j = 0; j < 16; ++j) acc += ptx::ex2_approx(fmaf(__uint_as_float(v[j]), sl2, -rs[c0 + j]));
            } else {
#pragma unroll
                for (int j = 0; j < 16; ++j)
                    if (c0 + j < R) acc += ptx::ex2_approx(fmaf(__uint_as_float(v[j]), sl2, -rs[c0 + j]));
            }
        }
        if (i < np) p.score[(size_t)h * np + i] = acc / (float)R;
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem, 128);
    }
}

// (>= 57 KB keeps <= 4 CTAs per SM, so their 128-column TMEM allocations always fit in 512 columns)
constexpr int snapkv_tc_smem(int D) {
    return 2 * (D / 64) * kPanelBytes + 2 * kRowsMax * 4 + 16 + 1024 > 57 * 1024
               ? 2 * (D / 64) * kPanelBytes + 2 * kRowsMax * 4 + 16 + 1024
               : 57 * 1024;
}

// per-row softmax statistics over all tiles: block (h, 32 rows), thread = (row, tile group of 8);
// online (max, sum) merge over its tiles, then an 8-way merge in SMEM
__global__ void __launch_bounds__(256) snapkv_rowstats(SnapParams p) {
    __shared__ float sm[8][32], sz[8][32];
    const int h = blockIdx.x, R = p.G * p.w;
    const int rl = threadIdx.x & 31, tg = threadIdx.x >> 5, r = blockIdx.y * 32 + rl;
    float M = -INFINITY, Z = 0.f;
    if (r < R) {
        for (int t = tg; t < p.tiles; t += 8) {
            const float2 pr = *(const float2*)(p.part + (((size_t)h * p.tiles + t) * R + r) * 2);
            if (pr.x == -INFINITY) continue;
            const float nm = fmaxf(M, pr.x);
            Z = Z * exp2f(M - nm) + pr.y * exp2f(pr.x - nm);
            M = nm;
        }
    }
    sm[tg][rl] = M;
    sz[tg][rl] = Z;
    __syncthreads();
    if (tg == 0 && r < R) {
        float MM = -INFINITY;
        for (int q = 0; q < 8; ++q) MM = fmaxf(MM, sm[q][rl]);
        float ZZ = 0.f;
        for (int q = 0; q < 8; ++q)
            if (sm[q][rl] != -INFINITY) ZZ += sz[q][rl] * exp2f(sm[q][rl] - MM);
        p.rows[(size_t)h * R + r] = MM + log2f(ZZ);   // log2 of the row's softmax denominator
    }
}

// 1-D max pool ('same', odd kernel) of the scores: block (256 tokens, h)
__global__ void __launch_bounds__(256) snapkv_pool(SnapParams p) {
    const int h = blockIdx.y, np = p.n - p.w, rad = (p.ks - 1) / 2;
    const int i = blockIdx.x * 256 + threadIdx.x;
    if (i >= np) return;
    const float* sc = p.score + (size_t)h * np;
    float m = sc[i];
    for (int j = max(0, i - rad); j <= min(np - 1, i + rad); ++j) m = fmaxf(m, sc[j]);
    p.pooled[(size_t)h * np + i] = m;
}

// gather the kept rows (kidx) into slots [0, N) of (seq, h): block (chunk of 16-byte copies, h)
__global__ void __launch_bounds__(256) snapkv_gather(SnapParams p) {
    const int h = blockIdx.y, CPR = p.d / 8;
    const int e = blockIdx.x * 256 + threadIdx.x;
    const int32_t* idx = p.kidx + (size_t)h * p.N;
    if (e < p.N * CPR) {
        const int j = e / CPR, c = e % CPR;
        const int src = idx[j];
        const size_t unit = ((size_t)p.seq * p.Hkv + h) * p.N * p.d;
        ((uint4*)(p.K + unit))[e] = __ldg((const uint4*)(p.k + ((size_t)h * p.n + src) * p.d) + c);
        ((uint4*)(p.V + unit))[e] = __ldg((const uint4*)(p.v + ((size_t)h * p.n + src) * p.d) + c);
    }
    if (blockIdx.x == 0) {
        if (p.kept)
            for (int j = threadIdx.x; j < p.N; j += 256) p.kept[(size_t)h * p.N + j] = idx[j];
        if (threadIdx.x == 0) p.n_valid[(size_t)p.seq * p.Hkv + h] = p.N;
    }
}

// inclusive prefix sum over a 1024-thread block; *total = the block sum (both barriers inside)
__device__ __forceinline__ unsigned block_incl_scan1024(unsigned v, int tid, unsigned* wsum, unsigned* total) {
    const int lane = tid & 31, warp = tid >> 5;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const unsigned a = __shfl_up_sync(0xffffffffu, v, off);
        if (lane >= off) v += a;
    }
    if (lane == 31) wsum[warp] = v;
    __syncthreads();
    if (warp == 0) {
        unsigned w = wsum[lane];
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const unsigned a = __shfl_up_sync(0xffffffffu, w, off);
            if (lane >= off) w += a;
        }
        wsum[lane] = w;   // inclusive over warps
    }
    __syncthreads();
    const unsigned r = v + (warp > 0 ? wsum[warp - 1] : 0u);
    *total = wsum[31];
    __syncthreads();   // wsum reusable
    return r;
}
// suffix sum S(b) = sum_{b' >= b} h[b'] over threads 0..255 (called by those 256 threads only;
// named barrier 1 synchronises them)
__device__ __forceinline__ unsigned block_suffix_sum256(unsigned h, int tid, unsigned* wsum) {
    const int lane = tid & 31, warp = tid >> 5;
    unsigned v = h;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {   // suffix within the warp
        const unsigned a = __shfl_down_sync(0xffffffffu, v, off);
        if (lane + off < 32) v += a;
    }
    if (lane == 0) wsum[warp] = v;             // warp totals
    asm volatile("bar.sync 1, 256;" ::: "memory");
    unsigned above = 0;
    for (int w = warp + 1; w < 8; ++w) above += wsum[w];
    asm volatile("bar.sync 1, 256;" ::: "memory");
    return v + above;
}

__global__ void __launch_bounds__(1024) snapkv_select(SnapParams p) {
    __shared__ unsigned hist[256];
    __shared__ unsigned wsum[33];
    __shared__ unsigned s_base[2];
    const int h = blockIdx.x, tid = threadIdx.x;
    const int np = p.n - p.w, k = p.N - p.w;
    const float* pl = p.pooled + (size_t)h * np;
    // radix select on the float bits (pooled >= 0: unsigned order == float order), MSB first:
    // find T = the k-th largest value
    unsigned prefix = 0, mask = 0, remaining = (unsigned)k;
    for (int shift = 24; shift >= 0; shift -= 8) {
        for (int b = tid; b < 256; b += 1024) hist[b] = 0;
        __syncthreads();
        for (int i = tid; i < np; i += 1024) {
            const unsigned u = __float_as_uint(pl[i]);
            if ((u & mask) == prefix) atomicAdd(&hist[(u >> shift) & 255u], 1u);
        }
        __syncthreads();
        // digit of the k-th largest: the bin b with S(b+1) < remaining <= S(b), S = suffix sums of
        // the histogram (bin 0 if none: S(0) = all candidates >= remaining)
        if (tid < 256) {
            const unsigned sb = block_suffix_sum256(hist[tid], tid, wsum);
            const unsigned above = sb - hist[tid];
            if (above < remaining && (remaining <= sb || tid == 0)) {
                s_base[0] = (unsigned)tid;
                s_base[1] = remaining - above;
            }
        }
        __syncthreads();
        prefix |= s_base[0] << shift;
        mask |= 255u << shift;
        remaining = s_base[1];
        __syncthreads();
    }
    const unsigned T = prefix;           // bits of the k-th largest pooled value
    const unsigned need_eq = remaining;  // how many == T to keep (the lowest indices)
    // ascending compaction: keep u > T, and the first need_eq with u == T
    unsigned base = 0, eq_base = 0;
    int32_t* out = p.kidx + (size_t)h * p.N;
    for (int c0 = 0; c0 < np; c0 += 1024) {
        const int i = c0 + tid;
        const unsigned u = i < np ? __float_as_uint(pl[i]) : 0u;
        const unsigned is_eq = (i < np && u == T) ? 1u : 0u;
        // inclusive scans over the chunk (warp shuffles + one warp over the 32 warp totals)
        unsigned eq_tot;
        const unsigned eq_incl = block_incl_scan1024(is_eq, tid, wsum, &eq_tot);
        const unsigned eq_rank = eq_base + eq_incl - is_eq;
        const unsigned keep = (i < np && (u > T || (is_eq && eq_rank < need_eq))) ? 1u : 0u;
        unsigned keep_tot;
        const unsigned keep_incl = block_incl_scan1024(keep, tid, wsum, &keep_tot);
        if (keep) out[base + keep_incl - 1] = i;
        base += keep_tot;
        eq_base += eq_tot;
    }
    for (int j = tid; j < p.w; j += 1024) out[k + j] = np + j;
}

size_t align256(size_t x) { return (x + 255) / 256 * 256; }

}  // namespace

size_t snapkv_workspace_bytes(int Hkv, int G, int n, int w, int N) {
    const int tiles = (n + kTile - 1) / kTile, R = G * w, np = n - w;
    return align256((size_t)Hkv * tiles * R * 2 * 4) + align256((size_t)Hkv * R * 2 * 4) +
           2 * align256((size_t)Hkv * np * 4) + align256((size_t)Hkv * N * 4);
}

cudaError_t snapkv_launch(uint16_t* K, uint16_t* V, int32_t* n_valid, int seq, int Hkv, int G, int d, int N,
                          const void* k, const void* v, const void* q_obs, int n, int w, int ks, float scale,
                          int32_t* kept, void* workspace, cudaStream_t stream) {
    SnapParams p;
    p.k = (const uint16_t*)k;
    p.v = (const uint16_t*)v;
    p.q_obs = (const uint16_t*)q_obs;
    p.K = K;
    p.V = V;
    p.n_valid = n_valid;
    p.kept = kept;
    p.seq = seq;
    p.Hkv = Hkv;
    p.G = G;
    p.d = d;
    p.n = n;
    p.w = w;
    p.ks = ks;
    p.N = N;
    p.tiles = (n + kTile - 1) / kTile;
    p.scale = scale;
    const int R = G * w, np = n - w;
    char* ws = (char*)workspace;
    p.part = (float*)ws;
    ws += align256((size_t)Hkv * p.tiles * R * 2 * 4);
    p.rows = (float*)ws;
    ws += align256((size_t)Hkv * R * 2 * 4);
    p.score = (float*)ws;
    ws += align256((size_t)Hkv * np * 4);
    p.pooled = (float*)ws;
    ws += align256((size_t)Hkv * np * 4);
    p.kidx = (int32_t*)ws;
    dim3 grid(Hkv, p.tiles);
    auto run = [&](auto kern, int smem) -> cudaError_t {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        kern<<<grid, 128, smem, stream>>>(p, 0);
        snapkv_rowstats<<<dim3(Hkv, (G * w + 31) / 32), 256, 0, stream>>>(p);
        kern<<<grid, 128, smem, stream>>>(p, 1);
        return cudaGetLastError();
    };
    cudaError_t e = d == 128 ? run(snapkv_logits_tc<128>, snapkv_tc_smem(128)) : run(snapkv_logits_tc<64>, snapkv_tc_smem(64));
    if (e != cudaSuccess) return e;
    snapkv_pool<<<dim3((n - w + 255) / 256, Hkv), 256, 0, stream>>>(p);
    snapkv_select<<<Hkv, 1024, 0, stream>>>(p);
    snapkv_gather<<<dim3((N * (d / 8) + 255) / 256, Hkv), 256, 0, stream>>>(p);
    return cudaGetLastError();
}

}  // namespace lf
