// SnapKV prefill compression (NEXT-f3; "if the number of tokens in the prefill stage exceeds
// the budget, we first use SnapKV to compress the tokens to the budget size").  Readings R22-R24
// (DESIGN.md): rows r = (g, k) are the G query heads x the last w prompt positions p_k = n-w+k;
// row r attends causally (tokens <= p_k); score_i = mean_r alpha_{r,i} over prefix tokens i < n-w;
// pooled = 1-D max pool (odd kernel, 'same'); keep the (budget - w) largest pooled (ties: lower
// index) plus the w window tokens, ascending, into slots [0, budget).
//
// Kernels (per sequence, one launch each):
//   snapkv_logits   grid (Hkv, tiles of 128 tokens), 256 threads: K tile -> SMEM (XOR-swizzled
//                   16-byte chunks), thread = (token, row group); pass 0 writes per-tile per-row
//                   (max, sum exp); pass 1 (after snapkv_rowstats) writes score_i
//   snapkv_rowstats grid Hkv: combine the per-tile (max, sum) of every row
//   snapkv_select   grid Hkv, 1024 threads: max pool, radix select of the (budget-w)-th largest
//                   pooled value, ascending compaction, gather of the kept K/V rows into the cache
#include <float.h>

#include "lf_common.cuh"

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
    float* part;            // [Hkv][tiles][R][2]
    float* rows;            // [Hkv][R][2]  (M, 1/Z)
    float* score;           // [Hkv][np]
    float* pooled;          // [Hkv][np]
    int32_t* kidx;          // [Hkv][N] scratch
    int seq, Hkv, G, d, n, w, ks, N, tiles;
    float scale;
};

__device__ __forceinline__ void ld_row(const uint16_t* tile, int r, int D, float* f, int c) {
    const int cpr = D / 8;
    const uint4 wv = *(const uint4*)(tile + (r * cpr + (c ^ (r & 7))) * 8);
    f[0] = __uint_as_float(wv.x << 16); f[1] = __uint_as_float(wv.x & 0xffff0000u);
    f[2] = __uint_as_float(wv.y << 16); f[3] = __uint_as_float(wv.y & 0xffff0000u);
    f[4] = __uint_as_float(wv.z << 16); f[5] = __uint_as_float(wv.z & 0xffff0000u);
    f[6] = __uint_as_float(wv.w << 16); f[7] = __uint_as_float(wv.w & 0xffff0000u);
}

template <int D>
__global__ void __launch_bounds__(256) snapkv_logits(SnapParams p, int pass) {
    __shared__ __align__(16) uint16_t tile[kTile * D];
    __shared__ float qs[8 * D];   // 8 query rows staged as fp32
    __shared__ float wm[8][kRowsMax];
    __shared__ float wz[8][kRowsMax];
    __shared__ float sc2[2][kTile];
    const int h = blockIdx.x, t = blockIdx.y;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int R = p.G * p.w, n = p.n, np = n - p.w;
    const int i0 = t * kTile;
    const int tok = tid & (kTile - 1), rg = tid >> 7;   // thread = (token, row group)
    const int i = i0 + tok;
    constexpr int CPR = D / 8;
    // K tile -> SMEM, 16-byte chunk c of row r at chunk c ^ (r & 7)
    for (int e = tid; e < kTile * CPR; e += 256) {
        const int r = e / CPR, c = e % CPR;
        uint4 val = make_uint4(0, 0, 0, 0);
        if (i0 + r < n) val = *(const uint4*)(p.k + ((size_t)h * n + i0 + r) * D + c * 8);
        *(uint4*)(tile + (r * CPR + (c ^ (r & 7))) * 8) = val;
    }
    __syncthreads();
    float kf[D];
#pragma unroll
    for (int c = 0; c < CPR; ++c) ld_row(tile, tok, D, kf + 8 * c, c);
    float acc_score = 0.f;
    for (int r0 = 0; r0 < R; r0 += 8) {
        // stage 8 query rows as fp32
        __syncthreads();
        for (int e = tid; e < 8 * D; e += 256) {
            const int rr = r0 + e / D, l = e % D;
            float val = 0.f;
            if (rr < R) {
                const int g = rr / p.w, kq = rr % p.w;
                val = bf16_to_f32(p.q_obs[(((size_t)h * p.G + g) * p.w + kq) * D + l]);
            }
            qs[e] = val;
        }
        __syncthreads();
        for (int j = rg; j < 8; j += 2) {
            const int r = r0 + j;
            if (r >= R) break;                                   // warp-uniform
            const int pos = np + (r % p.w);                      // causal position of the row
            float s = 0.f;
#pragma unroll
            for (int l = 0; l < D; ++l) s = fmaf(kf[l], qs[j * D + l], s);
            s *= p.scale;
            const bool valid = i < n && i <= pos;
            if (pass == 0) {
                float m = valid ? s : -INFINITY;
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
                float z = valid ? expf(s - m) : 0.f;
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) z += __shfl_xor_sync(0xffffffffu, z, off);
                if (lane == 0) {
                    wm[warp][r] = m;
                    wz[warp][r] = z;
                }
            } else if (i < np) {
                acc_score += expf(s - p.rows[((size_t)h * R + r) * 2]) * p.rows[((size_t)h * R + r) * 2 + 1];
            }
        }
    }
    __syncthreads();
    if (pass == 0) {
        // combine the 4 token-warps of each row group: warps 4*rg .. 4*rg+3 hold rows of parity rg
        for (int r = tid; r < R; r += 256) {
            const int g0 = (r & 1) * 4;
            float M = -INFINITY;
            for (int q = 0; q < 4; ++q) M = fmaxf(M, wm[g0 + q][r]);
            float Z = 0.f;
            for (int q = 0; q < 4; ++q) Z += (wm[g0 + q][r] == -INFINITY) ? 0.f : wz[g0 + q][r] * expf(wm[g0 + q][r] - M);
            float* pr = p.part + (((size_t)h * p.tiles + t) * R + r) * 2;
            pr[0] = M;
            pr[1] = Z;
        }
    } else {
        sc2[rg][tok] = acc_score;
        __syncthreads();
        if (tid < kTile && i < np) p.score[(size_t)h * np + i] = (sc2[0][tok] + sc2[1][tok]) / (float)R;
    }
}

__global__ void __launch_bounds__(256) snapkv_rowstats(SnapParams p) {
    const int h = blockIdx.x, R = p.G * p.w;
    for (int r = threadIdx.x; r < R; r += 256) {
        float M = -INFINITY;
        for (int t = 0; t < p.tiles; ++t) M = fmaxf(M, p.part[(((size_t)h * p.tiles + t) * R + r) * 2]);
        float Z = 0.f;
        for (int t = 0; t < p.tiles; ++t) {
            const float* pr = p.part + (((size_t)h * p.tiles + t) * R + r) * 2;
            if (pr[0] != -INFINITY) Z += pr[1] * expf(pr[0] - M);
        }
        p.rows[((size_t)h * R + r) * 2] = M;
        p.rows[((size_t)h * R + r) * 2 + 1] = 1.0f / Z;
    }
}

__global__ void __launch_bounds__(1024) snapkv_select(SnapParams p) {
    __shared__ unsigned hist[256];
    __shared__ unsigned scan[1024];
    __shared__ unsigned s_base[2];
    const int h = blockIdx.x, tid = threadIdx.x;
    const int np = p.n - p.w, k = p.N - p.w, rad = (p.ks - 1) / 2;
    const float* sc = p.score + (size_t)h * np;
    float* pl = p.pooled + (size_t)h * np;
    // 1-D max pool ('same')
    for (int i = tid; i < np; i += 1024) {
        float m = sc[i];
        for (int j = max(0, i - rad); j <= min(np - 1, i + rad); ++j) m = fmaxf(m, sc[j]);
        pl[i] = m;
    }
    __syncthreads();
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
        if (tid == 0) {   // walk digits from the top until `remaining` is covered
            unsigned acc = 0;
            int dgt = 255;
            for (; dgt > 0; --dgt) {
                if (acc + hist[dgt] >= remaining) break;
                acc += hist[dgt];
            }
            s_base[0] = (unsigned)dgt;
            s_base[1] = remaining - acc;
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
        // exclusive scan of is_eq within the chunk
        scan[tid] = is_eq;
        __syncthreads();
        for (int off = 1; off < 1024; off <<= 1) {
            const unsigned a = tid >= off ? scan[tid - off] : 0u;
            __syncthreads();
            scan[tid] += a;
            __syncthreads();
        }
        const unsigned eq_rank = eq_base + scan[tid] - is_eq;
        const unsigned keep = (i < np && (u > T || (is_eq && eq_rank < need_eq))) ? 1u : 0u;
        const unsigned eq_tot = scan[1023];
        __syncthreads();
        scan[tid] = keep;
        __syncthreads();
        for (int off = 1; off < 1024; off <<= 1) {
            const unsigned a = tid >= off ? scan[tid - off] : 0u;
            __syncthreads();
            scan[tid] += a;
            __syncthreads();
        }
        if (keep) out[base + scan[tid] - 1] = i;
        base += scan[1023];
        eq_base += eq_tot;
        __syncthreads();
    }
    for (int j = tid; j < p.w; j += 1024) out[k + j] = np + j;
    __syncthreads();
    // gather the kept rows into slots [0, N) of (seq, h)
    const int CPR = p.d / 8;
    const size_t unit = ((size_t)p.seq * p.Hkv + h) * p.N * p.d;
    for (int e = tid; e < p.N * CPR; e += 1024) {
        const int j = e / CPR, c = e % CPR;
        const int src = out[j];
        ((uint4*)(p.K + unit))[e] = ((const uint4*)(p.k + ((size_t)h * p.n + src) * p.d))[c];
        ((uint4*)(p.V + unit))[e] = ((const uint4*)(p.v + ((size_t)h * p.n + src) * p.d))[c];
    }
    if (p.kept)
        for (int j = tid; j < p.N; j += 1024) p.kept[(size_t)h * p.N + j] = out[j];
    if (tid == 0) p.n_valid[(size_t)p.seq * p.Hkv + h] = p.N;
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
    if (d == 128) {
        snapkv_logits<128><<<grid, 256, 0, stream>>>(p, 0);
        snapkv_rowstats<<<Hkv, 256, 0, stream>>>(p);
        snapkv_logits<128><<<grid, 256, 0, stream>>>(p, 1);
    } else {
        snapkv_logits<64><<<grid, 256, 0, stream>>>(p, 0);
        snapkv_rowstats<<<Hkv, 256, 0, stream>>>(p);
        snapkv_logits<64><<<grid, 256, 0, stream>>>(p, 1);
    }
    snapkv_select<<<Hkv, 1024, 0, stream>>>(p);
    return cudaGetLastError();
}

}  // namespace lf
