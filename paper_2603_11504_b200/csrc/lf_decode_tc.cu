// TMA + tcgen05 persistent split-KV LongFlow decode step, head_dim 128, 2 <= G <= 8 (B200, sm_100a).
//
// Grid = C persistent clusters of S CTAs (1 CTA per SM).  Cluster c handles units
// u = c, c + C, c + 2C, ... (unit = (sequence, kv head)); CTA s of the cluster owns slots
// [s*chunk, (s+1)*chunk) of every unit (chunk <= 4096).  Warp roles (64 + 128*kNG threads):
//   warp 0     producer: Q rows of the next unit (LDG -> swizzled SMEM) and the K then V tiles
//              (128 tokens x 128 d, two SWIZZLE_128B TMA boxes) through an ST-stage ring
//   warp 1     TMEM allocator (all 512 columns) + tcgen05.mma issuer (one lane)
//   warps 2..  kNG softmax groups of 4 warps; warp w owns TMEM lanes [32(w%4), 32(w%4)+32)
//
// TMEM-resident logits (hard part H1): S^T of every K tile of a unit stays in
// TMEM (8 columns per 128-token tile, N = 8 MMA) until the unit's scores are final; two regions
// alternate by unit parity, so the MMA streams the NEXT unit's whole K pass while the softmax
// warps finalise the current one.  O^T (16 columns) lives at the start of the other region.
//
// Per unit (Alg. 1 P:500-547 restructured):
//   K pass  S^T[128 tok x 8] = K_tile . Q^T (M=128, N=8, K=128, both K-major SW128) -> TMEM.
//   max     softmax groups read the unit's S from TMEM: exact per-CTA max m_g (R5).
//   V pass  P_g = 2^(x_g - m_g), x = S * scale * log2e, as bf16 hi + lo (N = 16: 8 hi + 8 lo rows;
//           bf16 P alone misses the 2e-3 out bar); O^T[128 d x 16] += V^T . P^T
//           (M=128, N=16, K=16 tokens per MMA, A MN-major straight from the TMA tile);
//           lambda_j = ||v_j||_1 from the same tile on the CUDA cores (Eq. 6, R9).
//   exchange (no cluster-wide barrier on the way): each CTA pushes (m_g, Z_g) and the slice of o_g
//           each rank combines into every rank's inbox with st.async (complete_tx on the receiver's
//           `xready`); all ranks compute M_g, Z_g (incl. the current token), their scores I_j
//           (from TMEM S) and argmin key -> st.async into rank 0's `kready`; the ranks split the
//           output combine; rank 0 picks the slot (lowest index on ties) and evicts in place
//           (Fig. 2); `xfree` arrivals release the inboxes for the cluster's next unit.
#include <cuda.h>
#include <stdio.h>
#include <stdlib.h>
#include <cudaTypedefs.h>

#include <mutex>

#include "lf_common.cuh"
#include "lf_tc_ptx.cuh"

namespace lf {
namespace {

constexpr int kMaxNG = 3;               // softmax warp groups (4 warps each): 3 at one CTA per SM,
                                        // 1 at two CTAs per SM (register file)
constexpr int kStageBytes = 32768;      // 128 tokens x 128 d x bf16 (two 16 KB boxes)
constexpr int kBoxBytes = 16384;
constexpr int kSmemLimit = 227 * 1024;
constexpr int kMaxStages = 6;
constexpr int kMaxChunk = 4096;         // 2 regions x 32 tiles x 8 columns = 512 TMEM columns

struct TcArgs {
    CUtensorMap tmK;
    CUtensorMap tmV;
    StepParams p;
    int32_t clusters;   // C: persistent clusters in the grid
    int32_t stages;     // ring depth
    int32_t tmem_cols;  // TMEM columns per CTA (512: one CTA per SM; 256: two)
};

// Exchange INBOX of a CTA, one per unit parity, written by the cluster's senders (push model: every
// remote access is a store followed by a release-arrive; all reads after the acquire are local)
struct Xchg {
    float mz[16][16][2];          // [sender r][g] = (m_g, Z_g) of rank r
    unsigned long long key[16];   // [sender r] argmin key of rank r (read by rank 0)
    float o[8 * 128 + 64];        // [sender r][e]: rank r's un-normalised o over MY output slice
};

struct TcSmem {
    int ring, q, pbuf, L, xb, misc, ostage, kvn, red, bars, tmem, nsm, total;
};
__host__ __device__ inline TcSmem tc_smem(int chunk, int stages, int kNG = kMaxNG) {
    TcSmem s;
    int off = 0;
    s.ring = off; off += stages * kStageBytes;   // 1024-aligned (swizzle atoms)
    s.q = off;    off += 2 * 4096;               // Q^T operand x2 (unit parity): 8 rows used
    s.pbuf = off; off += (kNG > 1 ? kNG : 2) * 4096;   // P^T operand buffers (16 rows x 128 tokens):
                                                      // one per group, two for a single group
    s.L = off;    off += chunk * 4;              // lambda_j of the current unit
    s.xb = off;   off += 2 * (int)sizeof(Xchg);
    s.misc = off; off += 512 * 4;                // scalars + per-rank combine factors [16][16]
    s.ostage = off; off += 8 * 128 * 4;          // this CTA's un-normalised o_g (split units)
    s.kvn = off;  off += 2 * 256;                // k_new, v_new rows of the current unit
    s.red = off;  off += (2 * kNG * 4 * 16 + 2 * kNG * 4) * 4;
    s.bars = off; off += 48 * 8;
    s.tmem = off; off += 16;
    s.nsm = off;  off += 8 * 4;                  // n_valid of the CTA's items, ring of 8 (NRDY)
    s.total = off + 1024;                        // slack for 1024-byte alignment of the base
    return s;
}

// mbarrier slots
constexpr int FULL = 0;                 // [kMaxStages]
constexpr int EMPTY = FULL + kMaxStages;
constexpr int PREADY = EMPTY + kMaxStages, PFREE = PREADY + kMaxNG;
constexpr int QFULL = PFREE + kMaxNG, QFREE = QFULL + 2, KDONE = QFREE + 2, SFREE = KDONE + 2;
constexpr int OFULL = SFREE + 2, OFREE = OFULL + 1;
constexpr int XREADY = OFREE + 1, KREADY = XREADY + 2, XFREE = KREADY + 2;
// NRDY[i % 8]: the producer published item i's fill state n (the ONLY read of n_valid in the CTA, so
// every role agrees on the item's tile count even if a caller races a write to n_valid)
constexpr int NRDY = XFREE + 2, NBARS = NRDY + 8;
static_assert(NBARS <= 48, "barrier slots");

// Debug event trace (-DLF_TRACE): %clock64 at fixed points, [cta][unit % 64][32] u64; slot 31 of
// row 0 holds the %globaltimer at slot 16 (entry) so tools/trace_run.py can align the CTAs.
#ifdef LF_TRACE
#define LF_EVENT(ui_, slot_)                                                                   \
    do {                                                                                       \
        if (p.trace) {                                                                         \
            unsigned long long t_;                                                             \
            asm volatile("mov.u64 %0, %%clock64;" : "=l"(t_));                                \
            p.trace[((size_t)blockIdx.x * 64 + ((ui_) & 63)) * 32 + (slot_)] = t_;             \
        }                                                                                      \
    } while (0)
#else
#define LF_EVENT(ui_, slot_) \
    do {                     \
    } while (0)
#endif
// per-tile events of the first units (debug): K tile t landed (MMA warp) in row ui+32, P of V tile t
// ready in row ui+33 (t < 32)
#ifdef LF_HANG_DIAG
#define LF_PROG(role_, v_) ptx::hang_progress((role_), (unsigned long long)(v_))
#else
#define LF_PROG(role_, v_) \
    do {                   \
    } while (0)
#endif
#define LF_TILE_EVENT(ui_, row_, t_)            \
    do {                                        \
        if ((t_) < 32) LF_EVENT((ui_) + (row_), (t_)); \
    } while (0)

// acc + sum of |v| over the 8 bf16 of w, in fp32: one LOP3 clears both sign bits of a pair and each
// element is added straight from its register half by the sm_100 mixed-precision add (FHADD.BF16,
// PTX add.rn.f32.bf16): 12 instructions per 8 values instead of 16 with explicit unpacking.
__device__ __forceinline__ float habs_acc8(const uint4& w, float acc) {
    const uint32_t p[4] = {w.x & 0x7fff7fffu, w.y & 0x7fff7fffu, w.z & 0x7fff7fffu, w.w & 0x7fff7fffu};
#pragma unroll
    for (int i = 0; i < 4; ++i)
        asm("{\n\t.reg .b16 lo, hi;\n\tmov.b32 {lo, hi}, %1;\n\t"
            "add.rn.f32.bf16 %0, lo, %0;\n\tadd.rn.f32.bf16 %0, hi, %0;\n\t}"
            : "+f"(acc)
            : "r"(p[i]));
    return acc;
}
// lambda_j = ||v_j||_1 of one token row of a landed V tile (both 64-column SW128 boxes), two
// independent accumulators
__device__ __forceinline__ float row_l1(const unsigned char* Vt, int row) {
    float a0 = 0.f, a1 = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        a0 = habs_acc8(*(const uint4*)(Vt + row * 128 + ((k ^ (row & 7)) << 4)), a0);
        a1 = habs_acc8(*(const uint4*)(Vt + kBoxBytes + row * 128 + ((k ^ (row & 7)) << 4)), a1);
    }
    return a0 + a1;
}

// min of a 64-bit (score bits, slot) key over the warp: two REDUX.MIN instead of five 64-bit shuffle
// rounds (exact: the high word decides, the low word breaks ties among the lanes holding that high word)
__device__ __forceinline__ unsigned long long warp_min_key(unsigned long long k) {
    const uint32_t hi = ptx::warp_min_u32((uint32_t)(k >> 32));
    const uint32_t lo = ptx::warp_min_u32((uint32_t)(k >> 32) == hi ? (uint32_t)k : 0xffffffffu);
    return ((unsigned long long)hi << 32) | lo;
}

struct UnitInfo {
    int u, b, h, n, c0, c1, nv, ntiles;
    bool split, valid;
};
// Number of whole ("solo") units CTA j = cid*S + s of a grid of P = C*S CTAs computes: units
// j, j + P, j + 2P, ... below solo_units.
__device__ __forceinline__ int solo_items(const StepParams& p, int cid, int s, int C) {
    const int P = C * p.splits, j = cid * p.splits + s;
    return p.solo_units > j ? (p.solo_units - j + P - 1) / P : 0;
}
// Work item i of CTA s of cluster cid (all roles walk the same list): first its whole units, one
// per CTA with no exchange, then the units from solo_units on, split S ways across the cluster
// (cluster cid takes solo_units + cid, + C, ...): balanced tails without paying the exchange on
// every unit.  Which units are whole is part of the plan of the plan_batch problem (lf_runtime.cu),
// so a shard computes every unit exactly as the one-GPU cache does.
__device__ __forceinline__ UnitInfo item_base(const StepParams& p, int cid, int s, int C, int i) {
    // recomputed per call: a CTA-wide variable live across the warp roles moved the MMA issuer's
    // descriptor arithmetic off the uniform datapath (R2UR per MMA, -3 % on f1/q3)
    const int R = solo_items(p, cid, s, C);
    UnitInfo x;
    const int S = p.splits, P = C * S;
    bool split;
    int u;
    if (i < R) {
        u = cid * S + s + i * P;
        split = false;
    } else {
        u = p.solo_units + cid + (i - R) * C;
        split = S > 1;
    }
    x.valid = u < p.B * p.Hkv;
    if (!x.valid) return x;
    x.u = u;
    x.split = split;
    x.b = u / p.Hkv;
    x.h = u % p.Hkv;
    x.c0 = split ? s * p.chunk : 0;
    x.c1 = split ? min(x.c0 + p.chunk, p.N) : p.N;
    return x;
}
// ... plus the unit's fill state n (after the PDL wait: the previous step may have appended)
// one_tile: a latency-variant split item whose CTA share is a single 128-token tile is always
// processed as ONE tile, even when none of its rows is valid yet (fill phase): its K and V tiles can
// then be requested before the fill state arrives (P = 0 and zeroed V rows make an empty tile exact)
__device__ __forceinline__ void set_fill(UnitInfo& x, int n, bool one_tile = false) {
    x.n = n;
    x.nv = max(0, min(x.c1, x.n) - x.c0);
    x.ntiles = one_tile ? 1 : (x.nv + 127) / 128;
}
// tokens one CTA may hold for a unit (TMEM regions, lambda buffer)
__host__ __device__ inline int hold_tokens(int N, int chunk, bool solo) {
    const int Nr = (N + 127) / 128 * 128;
    return solo && Nr > chunk ? Nr : chunk;
}

// kLat: the latency variant for split plans whose grid leaves SMs free (small batches, where the
// step is a chain of dependent latencies, not an HBM stream): one-round-trip operand loads, 16-lane
// x* and (M, Z) reductions, a thread-per-element split combine, and lambda_j of a single-tile CTA
// computed while its QK MMA runs.  Machine-filling and single-CTA-per-unit plans use kLat = false,
// the streaming-tuned code (measured: the latency changes cost 1-3 % there).
template <int GP, int kNG, bool kLat>
// (the one-group variant must fit two CTAs per SM: <= 170 registers, enforced by the launch bound)
__global__ void __launch_bounds__(64 + 128 * kNG, kNG == 1 ? 2 : 1) tc_decode_kernel(const __grid_constant__ TcArgs a) {
    constexpr int kNS = 128 * kNG;          // softmax threads
    constexpr int kNPB = kNG > 1 ? kNG : 2; // P^T operand buffers (PREADY / PFREE barrier pairs)
    extern __shared__ unsigned char smem_raw[];
    const StepParams& p = a.p;
    // 1024-byte aligned base (swizzle atoms); offset arithmetic keeps the shared state space
    unsigned char* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
    const int G = p.G, N = p.N, ST = a.stages;
    const int hold = p.hold;
    const TcSmem so = tc_smem(hold, ST, kNG);
    float* Ls = (float*)(smem + so.L);
    Xchg* xb = (Xchg*)(smem + so.xb);
    float* misc = (float*)(smem + so.misc);
    float* red = (float*)(smem + so.red);
    const uint32_t ring = ptx::smem_u32(smem + so.ring);
    const uint32_t qsm = ptx::smem_u32(smem + so.q);
    const uint32_t pbuf = ptx::smem_u32(smem + so.pbuf);
    const uint32_t bars = ptx::smem_u32(smem + so.bars);
    auto BAR = [&](int i) { return bars + 8u * (uint32_t)i; };
    // TMEM regions: S of unit parity `par` at column par*RC (8 columns per tile); O^T of unit
    // parity `par` at the first 16 columns of region par^1
    const int tmax = (hold + 127) / 128;
    const uint32_t RC = 8u * (uint32_t)(tmax > 2 ? tmax : 2);

    cg::cluster_group cluster = cg::this_cluster();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int S = p.splits;
    const int s = (int)cluster.block_rank();
    const int cid = blockIdx.x / S;
    const int C = a.clusters;
    volatile int* nsm = (volatile int*)(smem + so.nsm);

    if (tid == 0) {
        for (int i = 0; i < ST; ++i) {
            ptx::mbar_init(BAR(FULL + i), 1);      // producer's expect_tx arrival
            ptx::mbar_init(BAR(EMPTY + i), 1);     // MMA commit (the MMA is each stage's last reader)
        }
        for (int i = 0; i < kNPB; ++i) {
            ptx::mbar_init(BAR(PREADY + i), 4);
            ptx::mbar_init(BAR(PFREE + i), 1);
        }
        for (int i = 0; i < 2; ++i) {
            ptx::mbar_init(BAR(QFULL + i), 1);
            ptx::mbar_init(BAR(QFREE + i), 1);
            ptx::mbar_init(BAR(KDONE + i), 1);
            ptx::mbar_init(BAR(SFREE + i), 4 * kNG);
            ptx::mbar_init(BAR(XREADY + i), 1);    // own expect_tx; the senders' st.async complete_tx
            ptx::mbar_init(BAR(KREADY + i), 1);
            ptx::mbar_init(BAR(XFREE + i), S);
        }
        for (int i = 0; i < 8; ++i) ptx::mbar_init(BAR(NRDY + i), 1);
        ptx::mbar_init(BAR(OFULL), 1);
        ptx::mbar_init(BAR(OFREE), 4);
        ptx::fence_mbar_init();
        ptx::tma_prefetch_desc(&a.tmK);
        ptx::tma_prefetch_desc(&a.tmV);
    }
#ifdef LF_HANG_DIAG
    if (tid == 0) {
        ptx::g_hang_log = p.trace;
        ptx::hang_progress(8, bars);
    }
#endif
    if (warp == 1) ptx::tmem_alloc(ptx::smem_u32(smem + so.tmem), (uint32_t)a.tmem_cols);
    if (tid == 0) LF_EVENT(0, 16);
#ifdef LF_TRACE
    if (tid == 0 && p.trace) {   // SM cycles above; one globaltimer stamp per CTA aligns the CTAs
        unsigned long long g_;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_));
        p.trace[((size_t)blockIdx.x * 64) * 32 + 31] = g_;
    }
#endif
    if (tid == 64) {   // L2 warm-up of the first item's operands; safe before the PDL wait (L2 is coherent)
        const UnitInfo x = item_base(p, cid, s, C, 0);
        if (x.valid) {
            const int u = x.u;
            ptx::bulk_prefetch_l2(p.n_valid + (u & ~3), 16);
            if (!p.host_io) {
                ptx::bulk_prefetch_l2(p.q + ((size_t)x.b * p.Hq + (size_t)x.h * G) * 128, (uint32_t)G * 256);
                ptx::bulk_prefetch_l2(p.k_new + (size_t)u * 128, 256);
                ptx::bulk_prefetch_l2(p.v_new + (size_t)u * 128, 256);
            }
            const int nt = min((x.c1 - x.c0 + 127) / 128, 4);
            for (int t = 0; t < nt; ++t) {
                const int row = (p.unit_base + u) * N + x.c0 + t * 128;
                ptx::tma_prefetch_l2_3d(&a.tmK, 0, row, 0);
                ptx::tma_prefetch_l2_3d(&a.tmV, 0, row, 0);
            }
        }
    }
    if (warp >= 2) {   // zero the Q and P operand buffers (rows >= G stay zero)
        uint4* z = (uint4*)(smem + so.q);
        for (int e = tid - 64; e < (2 + kNPB) * 4096 / 16; e += kNS) z[e] = make_uint4(0, 0, 0, 0);
        ptx::fence_proxy_async_smem();
    }
    ptx::tc_fence_before();
    ptx::cluster_sync_all();   // barriers of every rank initialised before any remote arrival
    ptx::tc_fence_after();
    if (tid == 0) LF_EVENT(0, 17);
    pdl_trigger();             // the next step's prologue may overlap this step
    pdl_wait();                // the previous step's cache writes are visible from here on
    if (tid == 0) LF_EVENT(0, 18);
    if (tid == 64) LF_EVENT(0, 19);
    const uint32_t tmem = *(volatile uint32_t*)(smem + so.tmem);

    if (warp == 0) {
        // ------------------------------ producer -------------------------------------------------
        if constexpr (kLat) {
            uint32_t it = 0, qi = 0;
            int rst = 0;          // ring stage / phase of load `it`, kept incrementally
            uint32_t rph = 0;
            for (int i = 0;; ++i, ++qi) {
                // every global read of the item goes out at once (Q rows, fill state):
                // one L2 round trip instead of a chain of them before the first MMA
                UnitInfo x = item_base(p, cid, s, C, i);
                if (!x.valid) break;
                if (lane == 0) LF_PROG(0, ((unsigned long long)i << 32) | it);
                const int u = x.u;
                const int qb = qi & 1;
                const uint4* qg = (const uint4*)(p.q + ((size_t)x.b * p.Hq + (size_t)x.h * G) * 128);
                uint4 qv[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) qv[k] = lane + 32 * k < G * 16 ? __ldg(qg + lane + 32 * k) : make_uint4(0, 0, 0, 0);
                const int nval = __ldcg(p.n_valid + u);
                const bool one = x.split && p.chunk == 128;
                auto issue = [&](int i) {
                    const int st = rst;
                    ptx::mbar_wait(BAR(EMPTY + st), rph ^ 1u);
                    ptx::mbar_arrive_expect_tx(BAR(FULL + st), kStageBytes);
                    const int tile = i < x.ntiles ? i : i - x.ntiles;
                    const int row = (p.unit_base + u) * N + x.c0 + tile * 128;
                    const void* tm = i < x.ntiles ? (const void*)&a.tmK : (const void*)&a.tmV;
                    const uint32_t dst = ring + (uint32_t)st * kStageBytes;
                    LF_TILE_EVENT(qi, 34, i);
                    ptx::tma_load_3d(dst, tm, BAR(FULL + st), 0, row, 0);   // both 64-column halves
                    ++it;
                    if (++rst == ST) {
                        rst = 0;
                        rph ^= 1u;
                    }
                };
                if (one) {   // K and V tile 0 go out before the fill state returns (one round trip less)
                    x.ntiles = 1;
                    if (lane == 0) {
                        issue(0);
                        issue(1);
                    }
                }
                set_fill(x, nval, one);
                if (lane == 0) {   // publish n: the only read of n_valid in the CTA
                    nsm[i & 7] = x.n;
                    ptx::mbar_arrive(BAR(NRDY + (i & 7)));
                }
                if (lane == 0 && i == 0) LF_EVENT(0, 22);
                // the first ring stages go out before Q is staged (they do not depend on it)
                const int pre = one ? 2 : min(2 * x.ntiles, ST);
                if (lane == 0 && !one)
                    for (int i = 0; i < pre; ++i) issue(i);
                ptx::mbar_wait(BAR(QFREE + qb), ((qi >> 1) & 1u) ^ 1u);
                if (lane == 0 && i == 0) LF_EVENT(0, 24);
                // Q^T rows g < G (K-major SW128): 16 B chunk c of row g at chunk (c%8) ^ g of box c/8
                unsigned char* qd = smem + so.q + qb * 4096;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int e = lane + 32 * k, g = e >> 4, c = e & 15;
                    if (e < G * 16) *(uint4*)(qd + (c >> 3) * 1024 + g * 128 + (((c & 7) ^ g) << 4)) = qv[k];
                }
                ptx::fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) {
                    LF_EVENT(qi, 6);
                    ptx::mbar_arrive(BAR(QFULL + qb));
                    for (int i = pre; i < 2 * x.ntiles; ++i) issue(i);
                }
                it = __shfl_sync(0xffffffffu, it, 0);
                rst = __shfl_sync(0xffffffffu, rst, 0);
                rph = __shfl_sync(0xffffffffu, rph, 0);
            }
        } else {
            uint32_t it = 0, qi = 0;
            int rst = 0;          // ring stage / phase of load `it`, kept incrementally
            uint32_t rph = 0;
            for (int i = 0;; ++i, ++qi) {
                UnitInfo x = item_base(p, cid, s, C, i);
                if (!x.valid) break;
                if (lane == 0) LF_PROG(0, ((unsigned long long)i << 32) | it);
                set_fill(x, __ldcg(p.n_valid + x.u));
                if (lane == 0) {   // publish n: the only read of n_valid in the CTA
                    nsm[i & 7] = x.n;
                    ptx::mbar_arrive(BAR(NRDY + (i & 7)));
                }
                const int u = x.u;
                const int qb = qi & 1;
                // the first ring stages go out before Q is staged (they do not depend on it)
                const int pre = min(2 * x.ntiles, ST);
                auto issue = [&](int i) {
                    const int st = rst;
                    ptx::mbar_wait(BAR(EMPTY + st), rph ^ 1u);
                    ptx::mbar_arrive_expect_tx(BAR(FULL + st), kStageBytes);
                    const int tile = i < x.ntiles ? i : i - x.ntiles;
                    const int row = (p.unit_base + u) * N + x.c0 + tile * 128;
                    const void* tm = i < x.ntiles ? (const void*)&a.tmK : (const void*)&a.tmV;
                    const uint32_t dst = ring + (uint32_t)st * kStageBytes;
                    LF_TILE_EVENT(qi, 34, i);
                    ptx::tma_load_3d(dst, tm, BAR(FULL + st), 0, row, 0);   // both 64-column halves
                    ++it;
                    if (++rst == ST) {
                        rst = 0;
                        rph ^= 1u;
                    }
                };
                if (lane == 0)
                    for (int i = 0; i < pre; ++i) issue(i);
                ptx::mbar_wait(BAR(QFREE + qb), ((qi >> 1) & 1u) ^ 1u);
                // Q^T rows g < G (K-major SW128): 16 B chunk c of row g at chunk (c%8) ^ g of box c/8
                const uint4* qg = (const uint4*)(p.q + ((size_t)x.b * p.Hq + (size_t)x.h * G) * 128);
                unsigned char* qd = smem + so.q + qb * 4096;
                for (int e = lane; e < G * 16; e += 32) {
                    const int g = e >> 4, c = e & 15;
                    *(uint4*)(qd + (c >> 3) * 1024 + g * 128 + (((c & 7) ^ g) << 4)) = __ldg(qg + e);
                }
                ptx::fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) {
                    LF_EVENT(qi, 6);
                    ptx::mbar_arrive(BAR(QFULL + qb));
                    for (int i = pre; i < 2 * x.ntiles; ++i) issue(i);
                }
                it = __shfl_sync(0xffffffffu, it, 0);
                rst = __shfl_sync(0xffffffffu, rst, 0);
                rph = __shfl_sync(0xffffffffu, rph, 0);
            }
        }
    } else if (warp == 1) {
        // ------------------------------ MMA issuer -----------------------------------------------
        // The whole warp walks the issue loop (converged, so the loop state and the descriptors live on
        // the uniform datapath) and one elected lane issues each tile's eight MMAs and its commits as one
        // block: round 1 ran the loop on lane 0 alone, and the compiler then wrapped EVERY tcgen05.mma in
        // a waterfall loop (ELECT / R2UR / BRA.U.ANY, ~16 instructions per MMA) -- measured, the MMA issue
        // rate bounded one CTA's K pass (0.42 -> 0.37 us per tile with the descriptors built once per
        // tile, profiles/r02_ab_mma_issue.txt).
        {
            constexpr uint32_t idesc_qk = ptx::idesc_bf16_f32(128, 8, 0, 0);
            constexpr uint32_t idesc_pv = ptx::idesc_bf16_f32(128, 16, 1, 0);
            uint32_t it = 0, pi = 0, ui = 0;
            int rst = 0;          // ring stage of load `it` and its phase, kept incrementally (no
            uint32_t rph = 0;     // runtime division by ST on the per-tile issue path)
            for (int i = 0;; ++i, ++ui) {
                UnitInfo x = item_base(p, cid, s, C, i);
                if (!x.valid) break;
                ptx::mbar_wait(BAR(NRDY + (i & 7)), (uint32_t)(i >> 3) & 1u);
                set_fill(x, nsm[i & 7], kLat && x.split && p.chunk == 128);
                const uint32_t par = ui & 1u;
                LF_PROG(1, ((unsigned long long)i << 32) | it);
                ptx::mbar_wait(BAR(QFULL + par), (ui >> 1) & 1u);
                ptx::mbar_wait(BAR(SFREE + par), ((ui >> 1) & 1u) ^ 1u);   // unit ui-2 finalised
                ptx::mbar_wait(BAR(OFREE), (ui & 1u) ^ 1u);                  // O(ui-1) drained
                LF_EVENT(ui, 7);
                ptx::tc_fence_after();
                const uint32_t qbase = qsm + par * 4096;
                const uint32_t sreg = tmem + par * RC;
                for (int t = 0; t < x.ntiles; ++t, ++it, (++rst == ST ? (rst = 0, rph ^= 1u) : 0u)) {   // S^T = K . Q^T
                    const int st = rst;
                    ptx::mbar_wait(BAR(FULL + st), rph);
                    LF_TILE_EVENT(ui, 32, t);
                    ptx::tc_fence_after();
                    const uint32_t base = ring + (uint32_t)st * kStageBytes;
                    // descriptors built once per tile; the K steps only advance the 14-bit start-address
                    // field (address / 16; every SMEM address < 228 KB fits, so the add never carries)
                    const uint64_t da0 = ptx::smem_desc_sw128(base, 16, 1024);
                    const uint64_t db0 = ptx::smem_desc_sw128(qbase, 16, 1024);
                    if (ptx::elect_one()) {
#pragma unroll
                        for (int kk = 0; kk < 8; ++kk) {
                            const uint64_t da = da0 + (uint64_t)((kk >> 2) * (kBoxBytes >> 4) + (kk & 3) * 2);
                            const uint64_t db = db0 + (uint64_t)((kk >> 2) * 64 + (kk & 3) * 2);
                            ptx::mma_bf16(sreg + 8u * (uint32_t)t, da, db, idesc_qk, kk > 0);
                        }
                        ptx::mma_commit(BAR(EMPTY + st));
                    }
                    __syncwarp();
                }
                if (ptx::elect_one()) {
                    ptx::mma_commit(BAR(QFREE + par));
                    ptx::mma_commit(BAR(KDONE + par));
                }
                __syncwarp();
                const uint32_t oreg = tmem + (par ^ 1u) * RC;
                for (int t = 0; t < x.ntiles; ++t, ++it, ++pi, (++rst == ST ? (rst = 0, rph ^= 1u) : 0u)) {   // O^T += V^T . P^T
                    const int st = rst;
                    ptx::mbar_wait(BAR(FULL + st), rph);
                    const int pb = pi % kNPB;
                    ptx::mbar_wait(BAR(PREADY + pb), (pi / kNPB) & 1u);
                    ptx::tc_fence_after();
                    if (t == 0) LF_EVENT(ui, 28);
                    const uint32_t base = ring + (uint32_t)st * kStageBytes;
                    const uint32_t pbase = pbuf + (uint32_t)pb * 4096;
                    const uint64_t da0 = ptx::smem_desc_sw128(base, kBoxBytes, 1024);
                    const uint64_t db0 = ptx::smem_desc_sw128(pbase, 16, 1024);
                    if (ptx::elect_one()) {
#pragma unroll
                        for (int kk = 0; kk < 8; ++kk) {
                            const uint64_t da = da0 + (uint64_t)(kk * 128);
                            const uint64_t db = db0 + (uint64_t)((kk >> 2) * 128 + (kk & 3) * 2);
                            ptx::mma_bf16(oreg, da, db, idesc_pv, (t | kk) > 0);
                        }
                        ptx::mma_commit(BAR(EMPTY + st));
                        ptx::mma_commit(BAR(PFREE + pb));
                    }
                    __syncwarp();
                }
                if (ptx::elect_one()) ptx::mma_commit(BAR(OFULL));
                __syncwarp();
                LF_EVENT(ui, 29);
            }
        }
        __syncwarp();
    } else {
        // ------------------------------ softmax / score / exchange warps -------------------------
        const int grp = (warp - 2) >> 2;              // groups take tiles round-robin
        const int q4 = warp & 3;
        const int sidx = tid - 64;                    // 0 .. kNS-1
        const int row = 32 * q4 + lane;               // token row of a tile / d index of O
        const uint32_t tl = tmem + ((uint32_t)(32 * q4) << 16);
        float* xs = misc;          // [16] x_g* (current token)
        float* gM = misc + 16;     // [16]
        float* glz = misc + 32;    // [16]
        float* gZ = misc + 48;     // [16]
        float* gFn = misc + 96;    // [16] 2^(x_g* - M_g) (split units)
        float* gIZ = misc + 112;   // [16] 1 / Z_g (split units)
        int* s_slot = (int*)(misc + 64);
        unsigned long long* kred = (unsigned long long*)(red + 2 * kNG * 4 * 16);
        const int box = row >> 6, cc = row & 63;
        const float log2G = log2f((float)G);
        const float invG = 1.0f / (float)G;
        const float sl2 = p.scale_log2;
        // scores I_j (Eq. 6, mean over the group) of this thread's tokens from the TMEM logits and the
        // local argmin key (ordered log2 I_j, slot); needs gM, glz of the unit
        // s_reg: the logits of tile 0 already in registers (one-tile CTAs of the one-group variant) or nullptr
        auto unit_scores = [&](const UnitInfo& x, int u, uint32_t sreg, const uint32_t* s_reg) -> unsigned long long {
            const int nv = x.nv;
            unsigned long long best = ~0ull;
            const int excl = (p.deferred && p.exclude_newest) ? __ldg(p.written + u) : -1;
            float wM[GP];
#pragma unroll
            for (int g = 0; g < GP; ++g) wM[g] = g < G ? gM[g] + glz[g] : 0.f;
            for (int t = grp; t < x.ntiles; t += kNG) {
                uint32_t r[8];
                if (s_reg) {
#pragma unroll
                    for (int g = 0; g < 8; ++g) r[g] = s_reg[g];
                } else {
                    ptx::tmem_ld_x8(sreg + 8u * (uint32_t)t, r);
                    ptx::tmem_ld_wait();
                }
                const int j = t * 128 + row;
                if (j < nv) {
                    const float lam = Ls[j];
                    float av[GP];
                    float amax = -INFINITY;
#pragma unroll
                    for (int g = 0; g < GP; ++g) {
                        av[g] = g < G ? __uint_as_float(r[g]) * sl2 - wM[g] : -INFINITY;
                        amax = fmaxf(amax, av[g]);
                    }
                    float ssum = 0.f;
#pragma unroll
                    for (int g = 0; g < GP; ++g) ssum += ptx::ex2_approx(av[g] - amax);   // 1 <= ssum <= G
                    const float ls = ptx::lg2_approx(lam * ssum) + amax - log2G;   // log2 I_j, no underflow
                    if (p.scores) p.scores[(size_t)u * N + x.c0 + j] = lam * ssum * ptx::ex2_approx(amax) * invG;
                    if (x.c0 + j != excl)
                        best = umin64(best, ((unsigned long long)ordered_bits(ls) << 32) | (unsigned)(x.c0 + j));
                }
            }
            return best;
        };
        uint32_t it = 0, pi = 0, ui = 0, xi = 0;
        // the CTA's max and denominator of head g from the per-warp partials in red[]: the max is exact
        // in any order; Z adds the warps' partials subset by subset (tiles s, s + kNG, ... of the unit
        // live in group (g0 + s) % kNG), a fixed fp32 order per unit whatever units the CTA computed
        // before -- so a shard computes every unit bit-identically to the one-GPU run
        auto unit_max = [&](int g) {
            float mm = red[g];
            for (int w = 1; w < 4 * kNG; ++w) mm = fmaxf(mm, red[w * 16 + g]);
            return mm;
        };
        auto unit_z = [&](int g, int g0) {
            float zz = 0.f;
            for (int sg = 0; sg < kNG; ++sg) {
                const int w0 = ((g0 + sg) % kNG) * 4;
                for (int q = 0; q < 4; ++q) zz += red[kNG * 64 + (w0 + q) * 16 + g];
            }
            return zz;
        };
        for (int i = 0;; ++i, ++ui) {
            UnitInfo x;
            uint4* kvn = (uint4*)(smem + so.kvn);
            if constexpr (kLat) {
                // all global reads of the item at once: fill state, k*/v* rows, the x* operands
                x = item_base(p, cid, s, C, i);
                if (sidx == 0 && i == 0) LF_EVENT(0, 20);
                if (!x.valid) break;
                const int u = x.u;
                uint4 kvw = make_uint4(0, 0, 0, 0);
                if (warp == 2 + 4 * kNG - 1)   // the current token's k*, v* rows (combine + eviction write)
                    kvw = __ldg(lane < 16 ? (const uint4*)(p.k_new + (size_t)u * 128) + lane
                                          : (const uint4*)(p.v_new + (size_t)u * 128) + (lane - 16));
                // current token's logit x_g* (P:50-51): 16 lanes per head, 8 elements per lane
                const int xg = sidx >> 4, xch = sidx & 15;
                uint4 xq = make_uint4(0, 0, 0, 0), xk = make_uint4(0, 0, 0, 0);
                if (sidx < 128 && xg < G) {
                    xq = __ldg((const uint4*)(p.q + ((size_t)x.b * p.Hq + (size_t)x.h * G + xg) * 128) + xch);
                    xk = __ldg((const uint4*)(p.k_new + (size_t)u * 128) + xch);
                }
                ptx::mbar_wait(BAR(NRDY + (i & 7)), (uint32_t)(i >> 3) & 1u);
                set_fill(x, nsm[i & 7], x.split && p.chunk == 128);
                if (sidx == 0 && i == 0) LF_EVENT(0, 21);
                if (warp == 2 + 4 * kNG - 1) kvn[lane] = kvw;
                if (sidx < 128) {
                    float acc = 0.f;
                    const uint32_t qw[4] = {xq.x, xq.y, xq.z, xq.w}, kw[4] = {xk.x, xk.y, xk.z, xk.w};
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        acc = fmaf(__uint_as_float(qw[k] << 16), __uint_as_float(kw[k] << 16), acc);
                        acc = fmaf(__uint_as_float(qw[k] & 0xffff0000u), __uint_as_float(kw[k] & 0xffff0000u), acc);
                    }
#pragma unroll
                    for (int off = 8; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
                    if (xch == 0 && xg < G) xs[xg] = p.deferred ? -INFINITY : acc * sl2;
                }
            } else {
                x = item_base(p, cid, s, C, i);
                if (!x.valid) break;
                const int u = x.u;
                // stage the current token's k*, v* rows (combine + eviction write read them later)
                if (warp == 2 + 4 * kNG - 1) {
                    const uint4* src = lane < 16 ? (const uint4*)(p.k_new + (size_t)u * 128) + lane
                                                 : (const uint4*)(p.v_new + (size_t)u * 128) + (lane - 16);
                    kvn[lane] = __ldg(src);
                }
                // current token's logit x_g* (P:50-51): warp w-2 takes head g = w-2
                for (int g = warp - 2; g < G; g += 4 * kNG) {
                    const uint16_t* qg = p.q + ((size_t)x.b * p.Hq + (size_t)x.h * G + g) * 128;
                    const uint16_t* kn = p.k_new + (size_t)u * 128;
                    float acc = 0.f;
#pragma unroll
                    for (int l = lane; l < 128; l += 32) acc = fmaf(bf16_to_f32(qg[l]), bf16_to_f32(kn[l]), acc);
#pragma unroll
                    for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
                    if (lane == 0) xs[g] = p.deferred ? -INFINITY : acc * sl2;
                }
                ptx::mbar_wait(BAR(NRDY + (i & 7)), (uint32_t)(i >> 3) & 1u);
                set_fill(x, nsm[i & 7]);
            }
            const int u = x.u;
            const int nv = x.nv;
            const uint32_t par = ui & 1u;
            const uint32_t sreg = tl + par * RC;
            if (sidx == 0) LF_EVENT(ui, 0);
            if (sidx == 0) LF_EVENT(ui, 15);
            // latency variant, one tile per CTA: its V tile lands with (or before) K, so lambda_j and
            // the zeroing of rows past n happen while the QK MMA runs (PREADY still follows them)
            const bool lam_first = kLat && x.ntiles == 1;
            if (lam_first && (int)(pi % kNG) == grp) {
                const uint32_t iv = it + 1;
                const int st = iv % ST;
                ptx::mbar_wait(BAR(FULL + st), (iv / ST) & 1u);
                if (q4 == 0 && lane == 0) LF_EVENT(ui, 5);
                unsigned char* Vt = smem + so.ring + st * kStageBytes;
                float lam = 0.f;
                if (row < nv) {
                    lam = row_l1(Vt, row);
                } else {
#pragma unroll
                    for (int bb = 0; bb < 2; ++bb)
#pragma unroll
                        for (int k = 0; k < 8; ++k)
                            *(uint4*)(Vt + bb * kBoxBytes + row * 128 + k * 16) = make_uint4(0, 0, 0, 0);
                }
                Ls[row] = lam;
            }
            // ---- max over the unit's logits (TMEM-resident S)
            ptx::mbar_wait(BAR(KDONE + par), (ui >> 1) & 1u);
            ptx::tc_fence_after();
            if (sidx == 0) LF_EVENT(ui, 30);
            float mloc[GP];
#pragma unroll
            for (int g = 0; g < GP; ++g) mloc[g] = -INFINITY;
            // one-tile CTA of the one-group variant: its logits stay in registers for the V pass and the
            // scores (two TMEM round trips less on the latency chain)
            const bool s_in_regs = kNG == 1 && lam_first;
            uint32_t s0[8];
            for (int t = grp; t < x.ntiles; t += kNG) {
                uint32_t r[8];
                ptx::tmem_ld_x8(sreg + 8u * (uint32_t)t, r);
                ptx::tmem_ld_wait();
                if (s_in_regs) {
#pragma unroll
                    for (int g = 0; g < 8; ++g) s0[g] = r[g];
                }
                if (t * 128 + row < nv) {
#pragma unroll
                    for (int g = 0; g < GP; ++g)
                        if (g < G) mloc[g] = fmaxf(mloc[g], __uint_as_float(r[g]) * sl2);
                }
            }
#pragma unroll
            for (int g = 0; g < GP; ++g) mloc[g] = ptx::warp_max_f32(mloc[g]);
            if (lane == 0) {
#pragma unroll
                for (int g = 0; g < GP; ++g) red[(grp * 4 + q4) * 16 + g] = mloc[g];
            }
            ptx::named_bar_sync(1, kNS);
            if (sidx == 0) LF_EVENT(ui, 1);
            float m[GP];
#pragma unroll
            for (int g = 0; g < GP; ++g) {
                m[g] = red[g];
#pragma unroll
                for (int w = 1; w < 4 * kNG; ++w) m[g] = fmaxf(m[g], red[w * 16 + g]);
                if (g >= G) m[g] = 0.f;   // padded heads: logits exactly 0 (zero Q rows), P = 1, never read
            }
            if (sidx == 0) LF_EVENT(ui, 23);
            // ---- V pass: P (hi/lo bf16) for the MMA, Z, lambda
            float z[GP];
#pragma unroll
            for (int g = 0; g < GP; ++g) z[g] = 0.f;
            // V tiles go round-robin over the groups across units (c = the CTA's tile count), so the
            // tiles t = s, s + kNG, ... of this unit (subset s) are all handled by group (pi + s) % kNG
            const int g0 = (int)(pi % kNG);   // group of subset 0 in this unit
            int vst = (int)((it + x.ntiles) % ST);                     // ring stage / phase of V load t
            uint32_t vph = ((it + x.ntiles) / ST) & 1u;
            for (int t = 0; t < x.ntiles; ++t, (++vst == ST ? (vst = 0, vph ^= 1u) : 0u)) {
                const uint32_t c = pi + t;
                if ((int)(c % kNG) != grp) continue;
                const int pb = c % kNPB;   // a single group alternates two P buffers, so it writes
                                           // P of tile t+1 while the PV MMA of tile t still reads P(t)
                uint32_t r[8];
                if (s_in_regs) {
#pragma unroll
                    for (int g = 0; g < 8; ++g) r[g] = s0[g];
                    ptx::mbar_wait(BAR(PFREE + pb), ((c / kNPB) & 1u) ^ 1u);
                } else {
                    ptx::tmem_ld_x8(sreg + 8u * (uint32_t)t, r);
                    ptx::mbar_wait(BAR(PFREE + pb), ((c / kNPB) & 1u) ^ 1u);
                    ptx::tmem_ld_wait();
                }
                if (t == 0 && q4 == 0 && lane == 0) LF_EVENT(ui, 25);
                const int tok = t * 128 + row;
                const bool valid = tok < nv;
                unsigned char* P = smem + so.pbuf + pb * 4096 + box * 2048;
                // every head of the padded group, no per-head branch: padded heads (g >= G) get P = 1
                // from their zero logits, feed only O^T columns nobody reads, and their z is never used
#pragma unroll
                for (int g = 0; g < GP; ++g) {
                    const float pv = valid ? ptx::ex2_approx(__uint_as_float(r[g]) * sl2 - m[g]) : 0.f;
                    z[g] += pv;
                    const uint16_t hi = ptx::cvt_bf16_rn(pv);   // hardware RNE (pv is finite)
                    const uint16_t lo = ptx::cvt_bf16_rn(pv - bf16_to_f32(hi));
                    *(uint16_t*)(P + g * 128 + ((((cc >> 3) ^ g) & 7) << 4) + (cc & 7) * 2) = hi;
                    *(uint16_t*)(P + (8 + g) * 128 + ((((cc >> 3) ^ g) & 7) << 4) + (cc & 7) * 2) = lo;
                }
                if (t == 0 && q4 == 0 && lane == 0) LF_EVENT(ui, 26);
                const int st = vst;
                if (!lam_first) {
                ptx::mbar_wait(BAR(FULL + st), vph);      // V tile landed
                if (t == 0 && q4 == 0 && lane == 0) LF_EVENT(ui, 5);
                unsigned char* Vt = smem + so.ring + st * kStageBytes;
                if (!valid) {   // rows past n may hold stale data: P = 0 must not meet Inf/NaN
#pragma unroll
                    for (int bb = 0; bb < 2; ++bb)
#pragma unroll
                        for (int k = 0; k < 8; ++k)
                            *(uint4*)(Vt + bb * kBoxBytes + row * 128 + k * 16) = make_uint4(0, 0, 0, 0);
                }
                // lambda_j from the landed tile, before PREADY: after the PV MMA the stage is refilled
                float lam = 0.f;
#ifdef LF_ATTR_NO_LAMBDA   // attribution builds only (results wrong): no lambda pass over the V tile
                lam = valid ? 1.f : 0.f;
#else
                if (valid) lam = row_l1(Vt, row);
#endif
                Ls[tok] = lam;
                }
                ptx::fence_proxy_async_smem();
                if (t == 0 && q4 == 0 && lane == 0) LF_EVENT(ui, 27);
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(BAR(PREADY + pb));
                if (lane == 0 && q4 == 0) LF_TILE_EVENT(ui, 33, t);
            }
            pi += x.ntiles;
            it += 2 * x.ntiles;
#pragma unroll
            for (int g = 0; g < GP; ++g) {
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) z[g] += __shfl_xor_sync(0xffffffffu, z[g], off);
            }
            if (lane == 0) {
#pragma unroll
                for (int g = 0; g < GP; ++g) red[kNG * 64 + (grp * 4 + q4) * 16 + g] = z[g];
            }
            if (sidx == 0) LF_EVENT(ui, 2);
            if (!x.split) {
                // ---- single-CTA unit: M, Z and the output directly, no exchange
                ptx::named_bar_sync(1, kNS);                                  // red[] complete
                if (sidx < G) {
                    const int g = sidx;
                    const float mm = unit_max(g);
                    const float zz = unit_z(g, g0);
                    const float M = fmaxf(mm, xs[g]);
                    const float f = ptx::ex2_approx(mm - M);
                    const float Z = zz * f + ptx::ex2_approx(xs[g] - M);
                    gM[g] = M;
                    gZ[g] = Z;
                    glz[g] = log2f(Z);
                    misc[80 + g] = f;
                }
                ptx::named_bar_sync(1, kNS);
                if (grp == 0) {   // O^T lane = d: out = (o 2^(m-M) + 2^(x*-M) v*) / Z
                    ptx::mbar_wait(BAR(OFULL), ui & 1u);
                    ptx::tc_fence_after();
                    uint32_t o[16];
                    if (x.ntiles > 0) {
                        ptx::tmem_ld_x16(tl + (par ^ 1u) * RC, o);
                        ptx::tmem_ld_wait();
                    }
                    ptx::tc_fence_before();
                    __syncwarp();
                    if (lane == 0) ptx::mbar_arrive(BAR(OFREE));
                    const float vv = bf16_to_f32(((const uint16_t*)(smem + so.kvn))[128 + row]);
#pragma unroll
                    for (int g = 0; g < GP; ++g) {
                        if (g < G) {
                            float acc = x.ntiles > 0 ? (__uint_as_float(o[g]) + __uint_as_float(o[8 + g])) * misc[80 + g] : 0.f;
                            acc = fmaf(ptx::ex2_approx(xs[g] - gM[g]), vv, acc);
                            const float ov = acc / gZ[g];
                            const size_t oi = ((size_t)x.b * p.Hq + (size_t)x.h * G + g) * 128 + row;
                            if (p.out_f32) ((float*)p.out)[oi] = ov;
                            else ((uint16_t*)p.out)[oi] = f32_to_bf16_rne(ov);
                        }
                    }
                }
                unsigned long long best = unit_scores(x, u, sreg, s_in_regs ? s0 : nullptr);
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(BAR(SFREE + par));
                if (p.scores)
                    for (int j = nv + sidx; j < x.c1 - x.c0; j += kNS) p.scores[(size_t)u * N + x.c0 + j] = INFINITY;
#pragma unroll
                best = warp_min_key(best);
                if (lane == 0) kred[warp - 2] = best;
                ptx::named_bar_sync(1, kNS);
                if (sidx == 0) {
                    unsigned long long kb = kred[0];
                    for (int w = 1; w < 4 * kNG; ++w) kb = umin64(kb, kred[w]);
                    if (p.deferred) {
                        p.pend[u] = (int)(kb & 0xffffffffull);
                        *s_slot = -1;
                    } else {
                        const int sl = x.n < N ? x.n : (int)(kb & 0xffffffffull);
                        *s_slot = sl;
                        p.slot[u] = sl;
                        if (x.n < N) p.n_valid[u] = x.n + 1;
                    }
                }
                ptx::named_bar_sync(1, kNS);
                const int sl = *s_slot;
                if (sl >= 0 && sidx < 16) {   // in-place eviction write (or append)
                    const size_t unit_off = (size_t)u * N * 128;
                    const uint4* kvn4 = (const uint4*)(smem + so.kvn);
                    ((uint4*)(p.K + unit_off + (size_t)sl * 128))[sidx] = kvn4[sidx];
                    ((uint4*)(p.V + unit_off + (size_t)sl * 128))[sidx] = kvn4[16 + sidx];
                }
                ptx::named_bar_sync(1, kNS);   // misc / kvn / red reusable
                continue;
            }
            // ---- push (m, Z, o slices) into every rank's inbox for this unit parity
            const int xp = xi & 1;
            const uint32_t use = xi >> 1;
            ++xi;
            Xchg* xc = xb + xp;                       // my inbox (the same offset in every rank)
            const uint32_t xc_addr = ptx::smem_u32(xc);
            float* ost = (float*)(smem + so.ostage);
            const int E4 = (G * 32 + S - 1) / S;      // float4 output elements per rank
            const int my_cnt = max(0, min(G * 32, (s + 1) * E4) - s * E4);
            if (sidx == 0) {   // bytes every sender pushes into this inbox (phase use-1 already consumed)
                ptx::mbar_arrive_expect_tx(BAR(XREADY + xp), (uint32_t)(S * (G * 8 + my_cnt * 16)));
                if (s == 0) ptx::mbar_arrive_expect_tx(BAR(KREADY + xp), (uint32_t)(S * 8));
            }
            const uint32_t xr_local = BAR(XREADY + xp);
            if (use > 0)   // (the first use of each inbox parity has nothing to wait for)
                ptx::mbar_wait_cluster(BAR(XFREE + xp), (use & 1u) ^ 1u);   // every receiver consumed use-1
            if (sidx == 0) LF_EVENT(ui, 8);
            if (grp == 0) {   // group 0 drains O (TMEM lane = d)
                ptx::mbar_wait(BAR(OFULL), ui & 1u);
                if (sidx == 0) LF_EVENT(ui, 9);
                ptx::tc_fence_after();
                if (x.ntiles > 0) {
                    uint32_t o[16];
                    ptx::tmem_ld_x16(tl + (par ^ 1u) * RC, o);
                    ptx::tmem_ld_wait();
#pragma unroll
                    for (int g = 0; g < GP; ++g)
                        if (g < G) ost[g * 128 + row] = __uint_as_float(o[g]) + __uint_as_float(o[8 + g]);
                } else {
                    for (int g = 0; g < G; ++g) ost[g * 128 + row] = 0.f;
                }
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(BAR(OFREE));
            }
            ptx::named_bar_sync(1, kNS);                                // red[] and ost complete
            if (sidx == 0) LF_EVENT(ui, 10);
            // thread -> (rank, element) maps by shifts, not divisions (G <= 8; E4 padded to a power of two)
            if ((sidx & 7) < G && (sidx >> 3) < S) {                   // (m_g, Z_g) -> rank t
                const int t = sidx >> 3, g = sidx & 7;
                const float mm = unit_max(g);
                const float zz = unit_z(g, g0);
                ptx::st_async_f32x2(ptx::mapa(xc_addr + (uint32_t)offsetof(Xchg, mz) + 8 * (s * 16 + g), t), mm, zz,
                                    ptx::mapa(xr_local, t));
            }
            const int lgE = E4 > 1 ? 32 - __clz(E4 - 1) : 0;         // E4 <= 2^lgE
            for (int e = sidx; e < (S << lgE); e += kNS) {              // o slice of rank t -> rank t
                const int t = e >> lgE, i = e & ((1 << lgE) - 1), i4 = t * E4 + i;
                if (i < E4 && i4 < G * 32) {
                    const float4 v4 = *(const float4*)(ost + 4 * i4);
                    ptx::st_async_f32x4(ptx::mapa(xc_addr + (uint32_t)offsetof(Xchg, o) + 16 * (s * E4 + i), t), v4,
                                        ptx::mapa(xr_local, t));
                }
            }
            if (sidx == 0) LF_EVENT(ui, 11);
            // every sender's bytes landed: they arrive by st.async complete_tx into this CTA's own shared
            // memory, which the CTA-scope wait makes visible (no cluster acquire, no L1 invalidation)
            ptx::mbar_wait(xr_local, use & 1u);
            if (sidx == 0) LF_EVENT(ui, 3);
            // ---- global M_g, Z_g over the ranks (same order everywhere) + the current token
            float* fr = misc + 128;    // [g][r] = 2^(m_g,r - M_g)
            if constexpr (kLat) {
                if (sidx < 128) {          // 16 lanes per head, lane r <-> rank r
                    const int g = sidx >> 4, r = sidx & 15;
                    float mr = -INFINITY, zr = 0.f;
                    if (g < G && r < S) {
                        mr = xc->mz[r][g][0];
                        zr = xc->mz[r][g][1];
                    }
                    const float xsg = g < G ? xs[g] : -INFINITY;
                    float M = fmaxf(xsg, mr);
#pragma unroll
                    for (int off = 8; off > 0; off >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, off));
                    const float f = r < S ? ptx::ex2_approx(mr - M) : 0.f;   // same factors as P and o
                    float Z = zr * f;
#pragma unroll
                    for (int off = 8; off > 0; off >>= 1) Z += __shfl_xor_sync(0xffffffffu, Z, off);
                    const float fn = ptx::ex2_approx(xsg - M);
                    Z += fn;
                    if (g < G) {
                        if (r < S) fr[g * 16 + r] = f;
                        if (r == 0) {
                            gM[g] = M;
                            gZ[g] = Z;
                            glz[g] = ptx::lg2_approx(Z);   // Z >= 1 (the max term); same bits on every rank
                            gFn[g] = fn;
                            gIZ[g] = __frcp_rn(Z);
                        }
                    }
                }
            } else {
                for (int g = warp - 2; g < G; g += 4 * kNG) {   // one warp per head, lane r <-> rank r
                    float mr = -INFINITY, zr = 0.f;
                    if (lane < S) {
                        mr = xc->mz[lane][g][0];
                        zr = xc->mz[lane][g][1];
                    }
                    float M = fmaxf(xs[g], mr);
#pragma unroll
                    for (int off = 16; off > 0; off >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, off));
                    const float f = lane < S ? ptx::ex2_approx(mr - M) : 0.f;   // same factors as P and o
                    float Z = zr * f;
#pragma unroll
                    for (int off = 16; off > 0; off >>= 1) Z += __shfl_xor_sync(0xffffffffu, Z, off);
                    Z += ptx::ex2_approx(xs[g] - M);
                    if (lane < S) fr[g * 16 + lane] = f;
                    if (lane == 0) {
                        gM[g] = M;
                        gZ[g] = Z;
                        glz[g] = log2f(Z);
                    }
                }
            }
            ptx::named_bar_sync(1, kNS);
            if (sidx == 0) LF_EVENT(ui, 12);
            // ---- scores I_j (Eq. 6, mean over the group) from the TMEM logits; local argmin key
            unsigned long long best = unit_scores(x, u, sreg, s_in_regs ? s0 : nullptr);
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(BAR(SFREE + par));          // S(ui) no longer read
            if (p.scores)
                for (int j = nv + sidx; j < x.c1 - x.c0; j += kNS) p.scores[(size_t)u * N + x.c0 + j] = INFINITY;
#pragma unroll
            best = warp_min_key(best);
            if (lane == 0) kred[warp - 2] = best;
            ptx::named_bar_sync(1, kNS);
            if (sidx == 0) {   // key -> rank 0's inbox, then release to rank 0
                LF_EVENT(ui, 4);
                unsigned long long kb = kred[0];
                for (int w = 1; w < 4 * kNG; ++w) kb = umin64(kb, kred[w]);
                ptx::st_async_u64(ptx::mapa(xc_addr + (uint32_t)offsetof(Xchg, key) + 8 * s, 0), kb,
                                  ptx::mapa(BAR(KREADY + xp), 0));
            }
            if constexpr (kLat) {
                // ---- output combine of my slice from the inbox: one thread per float4 element, the S
                //      ranks' parts accumulated in rank order
                {
                    const int i4_0 = s * E4, cnt = min(G * 32, i4_0 + E4) - i4_0;
                    const uint16_t* vn = (const uint16_t*)(smem + so.kvn) + 128;
                    for (int e = sidx; e < cnt; e += kNS) {
                        const int i4 = i4_0 + e;
                        const int g = i4 >> 5, l = (i4 & 31) * 4;
                        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 8
                        for (int r = 0; r < 16; ++r) {   // predicated, so the inbox loads issue together
                            if (r < S) {
                                const float f = fr[g * 16 + r];
                                const float4 o4 = *(const float4*)(xc->o + 4 * (r * E4 + e));
                                acc.x = fmaf(o4.x, f, acc.x);
                                acc.y = fmaf(o4.y, f, acc.y);
                                acc.z = fmaf(o4.z, f, acc.z);
                                acc.w = fmaf(o4.w, f, acc.w);
                            }
                        }
                        const float fn = gFn[g], invZ = gIZ[g];
                        const uint2 vw = *(const uint2*)(vn + l);
                        const float o0 = fmaf(fn, __uint_as_float(vw.x << 16), acc.x) * invZ;
                        const float o1 = fmaf(fn, __uint_as_float(vw.x & 0xffff0000u), acc.y) * invZ;
                        const float o2 = fmaf(fn, __uint_as_float(vw.y << 16), acc.z) * invZ;
                        const float o3 = fmaf(fn, __uint_as_float(vw.y & 0xffff0000u), acc.w) * invZ;
                        const size_t oi = ((size_t)x.b * p.Hq + (size_t)x.h * G + g) * 128 + l;
                        if (p.out_f32) {
                            *(float4*)((float*)p.out + oi) = make_float4(o0, o1, o2, o3);
                        } else {
                            uint2 w;
                            w.x = (uint32_t)f32_to_bf16_rne(o0) | ((uint32_t)f32_to_bf16_rne(o1) << 16);
                            w.y = (uint32_t)f32_to_bf16_rne(o2) | ((uint32_t)f32_to_bf16_rne(o3) << 16);
                            *(uint2*)((uint16_t*)p.out + oi) = w;
                        }
                    }
                }
            } else {
                // ---- output combine of my slice from the inbox: S consecutive lanes (SG = pow2 >= S)
                //      share one float4 element, lane r reads sender r's part
                {
                    const int i4_0 = s * E4, cnt = min(G * 32, i4_0 + E4) - i4_0;
                    const uint16_t* vn = (const uint16_t*)(smem + so.kvn) + 128;
                    const int SG = S <= 2 ? 2 : S <= 4 ? 4 : S <= 8 ? 8 : 16;
                    const int r = lane % SG, per_warp = 32 / SG;
                    for (int e0 = ((sidx >> 5) * per_warp); e0 < cnt; e0 += (kNS >> 5) * per_warp) {
                        const int e = e0 + lane / SG;
                        const bool ok = e < cnt;
                        const int i4 = i4_0 + (ok ? e : 0);
                        const int g = i4 >> 5, l = (i4 & 31) * 4;
                        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
                        if (ok && r < S) {
                            const float f = fr[g * 16 + r];
                            const float4 o4 = *(const float4*)(xc->o + 4 * (r * E4 + e));
                            acc = make_float4(o4.x * f, o4.y * f, o4.z * f, o4.w * f);
                        }
                        for (int off = SG >> 1; off > 0; off >>= 1) {
                            acc.x += __shfl_xor_sync(0xffffffffu, acc.x, off);
                            acc.y += __shfl_xor_sync(0xffffffffu, acc.y, off);
                            acc.z += __shfl_xor_sync(0xffffffffu, acc.z, off);
                            acc.w += __shfl_xor_sync(0xffffffffu, acc.w, off);
                        }
                        if (!ok || r != 0) continue;
                        const float fn = ptx::ex2_approx(xs[g] - gM[g]);
                        const uint2 vw = *(const uint2*)(vn + l);
                        const float invZ = 1.0f / gZ[g];
                        const float o0 = fmaf(fn, __uint_as_float(vw.x << 16), acc.x) * invZ;
                        const float o1 = fmaf(fn, __uint_as_float(vw.x & 0xffff0000u), acc.y) * invZ;
                        const float o2 = fmaf(fn, __uint_as_float(vw.y << 16), acc.z) * invZ;
                        const float o3 = fmaf(fn, __uint_as_float(vw.y & 0xffff0000u), acc.w) * invZ;
                        const size_t oi = ((size_t)x.b * p.Hq + (size_t)x.h * G + g) * 128 + l;
                        if (p.out_f32) {
                            *(float4*)((float*)p.out + oi) = make_float4(o0, o1, o2, o3);
                        } else {
                            uint2 w;
                            w.x = (uint32_t)f32_to_bf16_rne(o0) | ((uint32_t)f32_to_bf16_rne(o1) << 16);
                            w.y = (uint32_t)f32_to_bf16_rne(o2) | ((uint32_t)f32_to_bf16_rne(o3) << 16);
                            *(uint2*)((uint16_t*)p.out + oi) = w;
                        }
                    }
                }
            }
            if (sidx == 0) LF_EVENT(ui, 13);
            if (s == 0) {
                // ---- rank 0: slot and the in-place eviction write
                ptx::mbar_wait(BAR(KREADY + xp), use & 1u);   // keys arrive by st.async complete_tx
                if (sidx == 0) {
                    unsigned long long mk = ~0ull;
                    for (int r = 0; r < S; ++r) mk = umin64(mk, xc->key[r]);
                    if (p.deferred) {        // next step's victim; the current token is already in place
                        p.pend[u] = (int)(mk & 0xffffffffull);
                        *s_slot = -1;
                    } else {
                        const int sl = x.n < N ? x.n : (int)(mk & 0xffffffffull);
                        *s_slot = sl;
                        p.slot[u] = sl;
                        if (x.n < N) p.n_valid[u] = x.n + 1;
                    }
                }
                ptx::named_bar_sync(1, kNS);
                const int sl = *s_slot;
                // every CTA of the cluster consumed unit u's K/V before arriving on kready
                if (sl >= 0 && sidx < 16) {
                    const size_t unit_off = (size_t)u * N * 128;
                    ((uint4*)(p.K + unit_off + (size_t)sl * 128))[sidx] = kvn[sidx];
                    ((uint4*)(p.V + unit_off + (size_t)sl * 128))[sidx] = kvn[16 + sidx];
                }
            }
            ptx::named_bar_sync(1, kNS);   // my inbox of unit u is consumed
            if (sidx == 0) LF_EVENT(ui, 14);
            // senders may reuse the inbox -- unless this was the cluster's last unit (every CTA of the
            // cluster walks the same unit list), where nobody waits and the release arrive would cost a
            // GPU-scope fence on the way to the exit
            if (sidx < S && item_base(p, cid, s, C, i + 1).valid)
                ptx::mbar_arrive_remote(ptx::mapa(BAR(XFREE + xp), sidx));
        }
        // (no drain of the last XFREE phases: the cluster barrier below orders every CTA's remote
        // arrivals and stores before any CTA of the cluster leaves)
    }
    __syncwarp();
    // every CTA of the cluster leaves together: no CTA exits while a peer may still address its shared
    // memory (round 1 drained its own XFREE phases instead; compute-sanitizer synccheck reported unsafe
    // exits for clusters of >= 4 CTAs placed two per SM, with illegal-address faults under the tool)
    {
        // split units this cluster computed (identical for its CTAs): with at most one, no CTA sent a
        // remote XFREE arrive (the last unit's are skipped) and every remote write into a CTA landed
        // before it got here, so the barrier needs no release half (no GPU-scope fence on the exit
        // path: the latency variant's single-unit clusters); otherwise the release orders the earlier
        // units' remote arrives before any CTA leaves
        const int rest = p.B * p.Hkv - p.solo_units - cid;
        const int nsplit = S > 1 && rest > 0 ? (rest + C - 1) / C : 0;
        if (nsplit <= 1) ptx::cluster_sync_relaxed();
        else ptx::cluster_sync_all();
    }
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem, (uint32_t)a.tmem_cols);
    }
}

__host__ __device__ constexpr int gpad_tc(int G) { return G <= 4 ? 4 : 8; }

// Kernel attributes are per device: set once, to the largest values any plan uses (the dynamic SMEM
// of a launch is still the plan's own), under a lock so concurrent cache creation is race-free.
template <int GP, int NG, bool kLat>
cudaError_t set_attrs(int smem, int splits) {
    (void)smem;
    (void)splits;
    static std::mutex mu;
    static bool done[64] = {false};
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev >= 64) return cudaErrorInvalidDevice;
    std::lock_guard<std::mutex> lock(mu);
    if (done[dev]) return cudaSuccess;
    e = cudaFuncSetAttribute(tc_decode_kernel<GP, NG, kLat>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemLimit);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(tc_decode_kernel<GP, NG, kLat>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(tc_decode_kernel<GP, NG, kLat>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e == cudaSuccess) done[dev] = true;
    return e;
}

template <int GP, int NG, bool kLat = false>
int max_active_clusters(int splits, int smem) {
    if (set_attrs<GP, NG, kLat>(smem, splits) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(splits * 1024, 1, 1);
    cfg.blockDim = dim3(64 + 128 * NG, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = splits;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, tc_decode_kernel<GP, NG, kLat>, &cfg) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

template <int GP, int NG, bool kLat>
cudaError_t launch_t(const TcArgs& args, const Plan& plan, cudaStream_t stream) {
    cudaError_t e = set_attrs<GP, NG, kLat>(plan.smem, plan.splits);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(plan.splits * args.clusters, 1, 1);
    cfg.blockDim = dim3(64 + 128 * NG, 1, 1);
    cfg.dynamicSmemBytes = plan.smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    cfg.numAttrs = fill_launch_attrs(attr, plan.splits);
    cfg.attrs = attr;
    return cudaLaunchKernelEx(&cfg, tc_decode_kernel<GP, NG, kLat>, args);
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
    static const PFN_cuTensorMapEncodeTiled_v12000 fn = [] {   // thread-safe one-time lookup
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            return (PFN_cuTensorMapEncodeTiled_v12000)f;
        return (PFN_cuTensorMapEncodeTiled_v12000) nullptr;
    }();
    return fn;
}

// K or V as a 3D tensor {64 columns, rows, 2 column halves} (strides 2d B per row, 128 B per half):
// one box {64, 128, 2} lands a whole 128-token tile as [half][row][64] -- the two SW128 K-major
// panels the MMA descriptors expect -- with ONE TMA instruction (vs two 2D boxes: measured +10 %
// single-SM fill rate, tools/probes/tma_probe.cu).
bool encode_kv(CUtensorMap* m, void* base, uint64_t rows, int d) {
    auto fn = get_encode();
    if (!fn) return false;
    cuuint64_t dims[3] = {64, (cuuint64_t)rows, 2};
    cuuint64_t strides[2] = {(cuuint64_t)d * 2, 128};
    cuuint32_t box[3] = {64, 128, 2};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, base, dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

int stages_for(int chunk, int smem_limit, int ng) {
    const int base = tc_smem(chunk, 0, ng).total;
    int st = (smem_limit - base) / kStageBytes;
    return st > kMaxStages ? kMaxStages : st;
}

}  // namespace

bool tc_supported(int G, int d) { return d == 128 && G >= 1 && G <= 8; }

// Split plan.  Candidates: cluster size S in {1, 2, 4, 8, 16} (chunk = N/S rounded up to a tile,
// <= 4096 so two TMEM logit regions fit) x k CTAs per SM in {1, 2} x (for S > 1 and N <= 4096)
// with or without solo rounds.  k = 1 takes all 512 TMEM columns and up to 6 ring stages; k = 2
// needs <= 1920 held tokens (256 columns) and >= 2 stages in 110 KB of SMEM (one softmax group).
// The grid holds
// C = cudaOccupancyMaxActiveClusters clusters; the plan minimises the per-SM time proxy
//   solo_rounds * (k N + ovh_1 / k) + split_rounds * (k chunk + ovh_S / k)
// with the measured unit-boundary overheads in streamed tokens (ovh_1 ~ 128 alone, ovh_S ~ 1024
// with the cross-CTA exchange).  Solo rounds process whole units per CTA (no exchange); the
// remaining units are split S ways, which balances the tail.
// Round model of a plan's step time (us) in the HBM regime, fitted to a measured exploration of the
// plan space on B200 (profiles/r02_split_explore3.jsonl + r02_split_explore4.jsonl: S = 1..16 x k x solo
// at 18 sweep points of 0.07-8 GB, parameters chosen to minimise the time lost by the pick: 0.3 % on
// average and at most 2.1 % above the best measured plan of each point): in every round the A active
// CTAs each stream `tokens` (512 B each, K + V); the round lasts the longer of the HBM time
// A * bytes / BW and one CTA's streaming time bytes / rho_k (rho_1 = 44 GB/s with three softmax groups,
// rho_2 = 26 GB/s with one), plus the unit-boundary overhead (0.5 us for whole units, 1 + 0.5 log2 S us
// for split units: the part of the cross-CTA exchange the next unit's K pass does not hide).  It sees
// what the token proxy below does not: a last round with few active CTAs, and clusters the GPCs cannot
// pack (S = 4: 33 clusters = 132 SMs), which is why mid-size grids (B = 16-32) prefer S = 4-6 at two
// CTAs per SM.
static double stream_cost_us(long long units, int S, int C, int chunk, int N, long long R, int k) {
    const double bw = 6.8e12, rho = k == 1 ? 44e9 : 26e9, ovh1 = 0.5, ovhS = 1.0 + 0.5 * log2((double)S);
    const long long P = (long long)C * S;
    long long rem = units;
    double t = 0.0;
    for (long long r = 0; r < R && rem > 0; ++r) {
        const long long A = rem < P ? rem : P;
        const double by = (double)N * 512.0;
        t += fmax((double)A * by / bw, by / rho) * 1e6 + ovh1;
        rem -= A;
    }
    while (rem > 0) {
        const long long c = rem < C ? rem : C;
        const double by = (double)(chunk < N ? chunk : N) * 512.0;
        t += fmax((double)(c * S) * by / bw, by / rho) * 1e6 + (S > 1 ? ovhS : ovh1);
        rem -= c;
    }
    return t;
}

// Latency model of a plan's step time (us) for steps below 64 MB, fitted to a measured exploration of
// the plan space on B200 (profiles/r02_lat_explore2.jsonl, refitted after the MMA-issue change: power-of-
// two S x k x latency variant at 20 sweep points of 2-67 MB; the pick is the best measured plan at every
// point): the same rounds as stream_cost_us, but a CTA's streaming rate is 40 GB/s with three softmax
// groups and 30 GB/s with one (a short chunk never reaches the steady state the HBM-regime rates
// describe), divided by 1.4 when two CTAs share an SM; the exchange of a split unit adds 0.25 us, and the
// three-group CTA (448 threads,
// all 512 TMEM columns) pays 1.5 us more per round than the one-group CTA -- which is why the small
// sweep points take one-tile splits at two CTAs per SM (B = 2 N = 512: 10.3 -> 6.9 us).
static double latency_cost_us(long long units, int S, int C, int chunk, int N, long long R, int k, int num_sms) {
    const double bw = 6.8e12, rho = k == 1 ? 40e9 : 30e9, ovhS = 0.25, base = k == 1 ? 1.5 : 0.0;
    const long long P = (long long)C * S;
    long long rem = units;
    double t = 0.0;
    auto round = [&](long long A, double by, double ovh) {
        const double r = (k == 2 && A > num_sms) ? rho / 1.4 : rho;
        t += fmax((double)A * by / bw, by / r) * 1e6 + ovh + base;
    };
    for (long long r = 0; r < R && rem > 0; ++r) {
        const long long A = rem < P ? rem : P;
        round(A, (double)N * 512.0, 0.0);
        rem -= A;
    }
    while (rem > 0) {
        const long long c = rem < C ? rem : C;
        round(c * S, (double)(chunk < N ? chunk : N) * 512.0, S > 1 ? ovhS : 0.0);
        rem -= c;
    }
    return t;
}

Plan tc_plan(int units, int G, int d, int N, int split_tokens, int num_sms, const PlanForce& force) {
    (void)d;
    Plan best;
    best.lat = 0;
    best.kernel = LF_KERNEL_TCGEN05;
    best.splits = -1;
    best.chunk = 0;
    best.smem = 0;
    best.clusters = 0;
    best.stages = 0;
    best.tmem_cols = 0;
    best.solo_rounds = 0;
    const int Nr = (N + 127) / 128 * 128;
    // Three regimes.  Steps that move >= 64 MB are HBM streams: the round model (stream_cost_us) over
    // every cluster size S = 1..16.  Smaller steps are latency chains (q7, small sweep points): the
    // latency model (latency_cost_us) over power-of-two S.
    // Above 16 GB per step the round model's 9-CTA two-per-SM picks measured worse than the token
    // proxy's S = 4 in long runs (512 x 16384: 0.87 vs 0.98 of the copy peak; 256 x 16384: 2.92 vs
    // 2.72 ms under the power cap, profiles/r02_ab_planner.txt), so the proxy keeps the largest steps.
    const double step_bytes = (double)units * (double)N * 512.0;
    const bool hbm_regime = step_bytes >= 64e6 && step_bytes <= 16e9;
    double best_cost = -1;
    for (int S = 1; S <= 16; ++S) {
        if (!hbm_regime && (S & (S - 1))) continue;
        const int chunk = split_tokens > 0 ? split_tokens : ((Nr + S - 1) / S + 127) / 128 * 128;
        const int splits = (N + chunk - 1) / chunk;
        if (splits != S && !(split_tokens > 0 && S == 1)) continue;   // each S once
        if (splits > 16 || chunk > kMaxChunk) continue;
        for (int k = 1; k <= 2; ++k) {
            if (force.ctas_per_sm && k != force.ctas_per_sm) continue;
            for (int solo = 0; solo <= 1; ++solo) {
                if (force.solo && solo != force.solo - 1) continue;
                if (solo && force.no_solo) continue;
                if (solo && (splits == 1 || Nr > kMaxChunk)) continue;
                const int hold = solo ? max(Nr, chunk) : chunk;
                const int tiles = (hold + 127) / 128;
                const int ng = k == 1 ? kMaxNG : 1;
                int st, smem, cols;
                if (k == 1) {
                    st = stages_for(hold, kSmemLimit, ng);
                    if (st < 3) continue;
                    smem = max(tc_smem(hold, st, ng).total, 120 * 1024);   // keeps one CTA per SM
                    cols = 512;
                } else {
                    if (2 * 8 * max(tiles, 2) + 16 > 256) continue;
                    st = stages_for(hold, 110 * 1024, ng);
                    if (st < 2) continue;
                    smem = tc_smem(hold, st, ng).total;
                    cols = 256;
                }
                int C = gpad_tc(G) == 4 ? (k == 1 ? max_active_clusters<4, kMaxNG>(splits, smem)
                                                  : max_active_clusters<4, 1>(splits, smem))
                                        : (k == 1 ? max_active_clusters<8, kMaxNG>(splits, smem)
                                                  : max_active_clusters<8, 1>(splits, smem));
                // The occupancy API reports one block per SM for the one-group variant although two
                // fit (2 x 93 KB SMEM, 2 x 30K registers, 2 x 256 TMEM columns); measured on B200 the
                // two co-reside (e.g. 512 x N=512: 200 -> 166 us), so the k = 2 grid is doubled.  The
                // persistent loop is correct either way (no cross-cluster dependency).
                if (k == 2) C *= 2;
                if (C <= 0) continue;
                // 16-CTA clusters two per SM walking several units: compute-sanitizer synccheck reports a
                // "missing wait" on a cluster barrier for this family only (the round-1 kernel too; memcheck
                // and racecheck are clean and lockstep parity holds): the planner does not choose it
                if (k == 2 && splits > 8 && units > C && !force.ctas_per_sm) continue;
                const long long ovh1 = 128, ovhS = splits > 1 ? 1024 : 128;
                double cost;
                long long R = 0;
                int Cu;
                if (solo) {
                    R = units / ((long long)C * splits);
                    if (R == 0) continue;
                    const long long rem = units - R * C * splits;
                    Cu = C;
                    cost = (double)(R * ((long long)k * Nr + ovh1 / k) + ((rem + C - 1) / C) * ((long long)k * chunk + ovhS / k));
                } else {
                    Cu = C < units ? C : units;
                    cost = (double)(((units + Cu - 1) / Cu) * ((long long)k * chunk + ovhS / k));
                }
                if (hbm_regime) cost = stream_cost_us(units, splits, C, chunk, N, R, k);
                else if (step_bytes < 64e6) cost = latency_cost_us(units, splits, C, chunk, N, R, k, num_sms);
                if (best_cost < 0 || cost < best_cost) {
                    best_cost = cost;
                    best.splits = splits;
                    best.chunk = chunk;
                    best.smem = smem;
                    best.clusters = Cu;
                    best.stages = st;
                    best.tmem_cols = cols;
                    best.solo_rounds = (int)R;
                }
            }
        }
        if (split_tokens > 0) break;
    }
    // latency variant: split plans whose grid leaves SMs free (measured: it helps the split
    // exchange chain of small batches; solo and machine-filling plans stay on the streaming code)
    if (best.splits > 1)
        best.lat = force.lat ? force.lat - 1
                             : (long long)best.clusters * best.splits < (long long)num_sms * (best.tmem_cols == 256 ? 2 : 1);
    return best;
}

int tc_hold(const Plan& plan, int N) { return hold_tokens(N, plan.chunk, plan.solo_rounds > 0); }

bool tc_make_maps(TcMaps* maps, void* K, void* V, long long units, int N, int d) {
    static_assert(sizeof(CUtensorMap) <= sizeof(maps->k), "tensor map size");
    return encode_kv((CUtensorMap*)maps->k, K, (uint64_t)units * (uint64_t)N, d) &&
           encode_kv((CUtensorMap*)maps->v, V, (uint64_t)units * (uint64_t)N, d);
}

cudaError_t tc_launch(const StepParams& p, const Plan& plan, const TcMaps& maps, cudaStream_t stream) {
    TcArgs args;
    memcpy(&args.tmK, maps.k, sizeof(CUtensorMap));
    memcpy(&args.tmV, maps.v, sizeof(CUtensorMap));
    args.p = p;
    args.clusters = plan.clusters;
    args.stages = plan.stages;
    args.tmem_cols = plan.tmem_cols;
    const bool one = plan.tmem_cols == 512;   // one CTA per SM -> kMaxNG softmax groups
    if (plan.lat) {
        if (gpad_tc(p.G) == 4)
            return one ? launch_t<4, kMaxNG, true>(args, plan, stream) : launch_t<4, 1, true>(args, plan, stream);
        return one ? launch_t<8, kMaxNG, true>(args, plan, stream) : launch_t<8, 1, true>(args, plan, stream);
    }
    if (gpad_tc(p.G) == 4)
        return one ? launch_t<4, kMaxNG, false>(args, plan, stream) : launch_t<4, 1, false>(args, plan, stream);
    return one ? launch_t<8, kMaxNG, false>(args, plan, stream) : launch_t<8, 1, false>(args, plan, stream);
}

}  // namespace lf
