// Approximation diagnostics at scale (NEXT-f4; §3.3, App. A).
// Not on the hot path: a plain CUDA-core kernel, one CTA per unit (sequence, kv head), reading the
// pre-step cache.  For the current query (the same attended set as the decode step: the n cached
// tokens plus the current token) it computes, per cached token i and query head g:
//   alpha_gi, o_g (Eq. 1), LongFlowScore I_i = mean_g alpha_gi ||v_i||_1 (Eq. 6, R2),
//   the exact eviction objective with the current query (Eq. 3's right-hand side, via the exact
//   remainder of App. A):  Delta o_gi = alpha_gi / (1 - alpha_gi) (v_i - o_g),
//   E_i = mean_g ||Delta o_gi||_2^2                                          (reading R25),
//   and the remainder bound ratio ||R_gi|| / (2 V alpha_gi / (1 - alpha_gi)) with
//   R_gi = -alpha/(1-alpha) (o_g - alpha v_i), V = max ||v||_2 over the attended tokens.
// Per unit it reports the LongFlow victim, the exact-objective victim (lowest index on ties), the
// rank of the LongFlow victim under E, E at both victims, and the largest remainder ratio (<= 1).
#include "lf_common.cuh"

namespace lf {
namespace {

constexpr int kNT = 256;

struct DiagParams {
    const uint16_t* q;      // [B][Hq][d]
    const uint16_t* k_new;  // [B][Hkv][d]
    const uint16_t* v_new;
    const uint16_t* K;      // [B][Hkv][N][d]
    const uint16_t* V;
    const int32_t* n_valid; // [B][Hkv]
    float* ws;              // [units][G][N + 1] attention weights
    int32_t* islot;         // [units][3]: LongFlow victim, exact victim, rank of the LongFlow victim
    float* fstat;           // [units][3]: E(LongFlow victim), E(exact victim), max remainder ratio
    int Hq, Hkv, G, d, N;
    float scale;
};

__device__ __forceinline__ float block_max(float v, float* red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    float r = red[0];
    for (int w = 1; w < kNT / 32; ++w) r = fmaxf(r, red[w]);
    return r;
}
__device__ __forceinline__ float block_sum(float v, float* red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    float r = 0.f;
    for (int w = 0; w < kNT / 32; ++w) r += red[w];
    return r;
}
__device__ __forceinline__ unsigned long long block_min64(unsigned long long v, unsigned long long* red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = umin64(v, __shfl_xor_sync(0xffffffffu, v, o));
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    unsigned long long r = red[0];
    for (int w = 1; w < kNT / 32; ++w) r = umin64(r, red[w]);
    return r;
}

__global__ void __launch_bounds__(kNT) diag_kernel(DiagParams p) {
    __shared__ float redf[32];
    __shared__ unsigned long long redk[32];
    __shared__ float o_s[8 * 128];   // o_g, G <= 8, d <= 128
    const int u = blockIdx.x, tid = threadIdx.x;
    const int b = u / p.Hkv, h = u % p.Hkv;
    const int G = p.G, d = p.d, N = p.N;
    const int n = p.n_valid[u];
    const int T = n + 1;                       // + the current token (index n)
    const uint16_t* Ku = p.K + (size_t)u * N * d;
    const uint16_t* Vu = p.V + (size_t)u * N * d;
    const uint16_t* kn = p.k_new + (size_t)u * d;
    const uint16_t* vn = p.v_new + (size_t)u * d;
    float* A = p.ws + (size_t)u * G * (N + 1);
    auto krow = [&](int j) { return j < n ? Ku + (size_t)j * d : kn; };
    auto vrow = [&](int j) { return j < n ? Vu + (size_t)j * d : vn; };
    // alpha_gj (Eq. 1 with the exact max)
    for (int g = 0; g < G; ++g) {
        const uint16_t* qg = p.q + ((size_t)b * p.Hq + (size_t)h * G + g) * d;
        float mloc = -INFINITY;
        for (int j = tid; j < T; j += kNT) {
            const uint16_t* kr = krow(j);
            float s = 0.f;
            for (int l = 0; l < d; ++l) s = fmaf(bf16_to_f32(qg[l]), bf16_to_f32(kr[l]), s);
            s *= p.scale;
            A[g * (N + 1) + j] = s;
            mloc = fmaxf(mloc, s);
        }
        const float m = block_max(mloc, redf);
        float zloc = 0.f;
        for (int j = tid; j < T; j += kNT) {
            const float e = expf(A[g * (N + 1) + j] - m);
            A[g * (N + 1) + j] = e;
            zloc += e;
        }
        const float Z = block_sum(zloc, redf);
        for (int j = tid; j < T; j += kNT) A[g * (N + 1) + j] /= Z;
    }
    __syncthreads();
    // o_g = sum_j alpha_gj v_j (thread = (g, l))
    for (int e = tid; e < G * d; e += kNT) {
        const int g = e / d, l = e % d;
        float acc = 0.f;
        for (int j = 0; j < T; ++j) acc = fmaf(A[g * (N + 1) + j], bf16_to_f32(vrow(j)[l]), acc);
        o_s[g * d + l] = acc;
    }
    __syncthreads();
    // V = max ||v||_2 over the attended tokens
    float vloc = 0.f;
    for (int j = tid; j < T; j += kNT) {
        const uint16_t* vr = vrow(j);
        float s = 0.f;
        for (int l = 0; l < d; ++l) s = fmaf(bf16_to_f32(vr[l]), bf16_to_f32(vr[l]), s);
        vloc = fmaxf(vloc, sqrtf(s));
    }
    const float Vmax = block_max(vloc, redf);
    // E_i = mean_g (alpha/(1-alpha))^2 ||v_i - o_g||^2
    auto E_of = [&](int i) {
        const uint16_t* vr = Vu + (size_t)i * d;
        float E = 0.f;
        for (int g = 0; g < G; ++g) {
            const float a = A[g * (N + 1) + i];
            float dist2 = 0.f;
            for (int l = 0; l < d; ++l) {
                const float vl = bf16_to_f32(vr[l]), ol = o_s[g * d + l];
                dist2 = fmaf(vl - ol, vl - ol, dist2);
            }
            const float f = a / (1.f - a);
            E += f * f * dist2;
        }
        return E / (float)G;
    };
    // per cached token: I_i, E_i, remainder ratio
    unsigned long long kI = ~0ull, kE = ~0ull;
    float rmax = 0.f;
    for (int i = tid; i < n; i += kNT) {
        const uint16_t* vr = Vu + (size_t)i * d;
        float l1 = 0.f;
        for (int l = 0; l < d; ++l) l1 += fabsf(bf16_to_f32(vr[l]));
        float I = 0.f;
        for (int g = 0; g < G; ++g) {
            const float a = A[g * (N + 1) + i];
            float rem2 = 0.f;
            for (int l = 0; l < d; ++l) {
                const float vl = bf16_to_f32(vr[l]), ol = o_s[g * d + l];
                rem2 = fmaf(ol - a * vl, ol - a * vl, rem2);
            }
            I += a * l1;
            if (a > 0.f) rmax = fmaxf(rmax, sqrtf(rem2) / (2.f * Vmax));   // ||R|| / bound
        }
        I /= (float)G;
        const float E = E_of(i);
        kI = umin64(kI, ((unsigned long long)ordered_bits(I) << 32) | (unsigned)i);
        kE = umin64(kE, ((unsigned long long)ordered_bits(E) << 32) | (unsigned)i);
    }
    const unsigned long long bI = block_min64(kI, redk);
    const unsigned long long bE = block_min64(kE, redk);
    const float rm = block_max(rmax, redf);
    const int lf = n > 0 ? (int)(bI & 0xffffffffu) : -1;
    const int ex = n > 0 ? (int)(bE & 0xffffffffu) : -1;
    // E at both victims, recomputed exactly as in the loop below (same order: rank is consistent)
    __shared__ float e_vic[2];
    if (tid == 0) {
        e_vic[0] = n > 0 ? E_of(lf) : 0.f;
        e_vic[1] = n > 0 ? E_of(ex) : 0.f;
    }
    __syncthreads();
    const float e_lf = e_vic[0], e_ex = e_vic[1];
    unsigned cnt = 0;
    for (int i = tid; i < n; i += kNT) cnt += (E_of(i) < e_lf) ? 1u : 0u;
    const float rank = block_sum((float)cnt, redf);
    if (tid == 0) {
        p.islot[u * 3 + 0] = lf;
        p.islot[u * 3 + 1] = ex;
        p.islot[u * 3 + 2] = (int)rank;
        p.fstat[u * 3 + 0] = e_lf;
        p.fstat[u * 3 + 1] = e_ex;
        p.fstat[u * 3 + 2] = rm;
    }
}

}  // namespace

size_t diag_workspace_bytes(int units, int G, int N) { return (size_t)units * G * (N + 1) * 4; }

cudaError_t diag_launch(const StepParams& p, const int32_t* n_valid, void* workspace, int32_t* islot, float* fstat,
                        cudaStream_t stream) {
    DiagParams d;
    d.q = p.q;
    d.k_new = p.k_new;
    d.v_new = p.v_new;
    d.K = p.K;
    d.V = p.V;
    d.n_valid = n_valid;
    d.ws = (float*)workspace;
    d.islot = islot;
    d.fstat = fstat;
    d.Hq = p.Hq;
    d.Hkv = p.Hkv;
    d.G = p.G;
    d.d = p.d;
    d.N = p.N;
    d.scale = p.scale_log2 / 1.4426950408889634f;
    diag_kernel<<<p.B * p.Hkv, kNT, 0, stream>>>(d);
    return cudaGetLastError();
}

}  // namespace lf
