/*
 * longflow.h -- C ABI of the B200-native LongFlow fused decode-step operator.
 *
 * Citation key: P:n = PAPER.md line n (arXiv 2603.11504), S:n = SPEC.md line n; readings
 * R1..R17 are listed in DESIGN.md ("Readings of the paper").
 *
 * The operation (Alg. 1; Eq. 1, Eq. 5, Eq. 6): for every unit
 * u = (sequence b, kv head h) of a static, pre-allocated KV cache one decode step
 *   - attends the G = Hq/Hkv query heads hq = h*G + g of the current token over the n valid
 *     cached tokens plus the current token (R1),
 *   - scores every cached token with LongFlowScore I_j = (1/G) sum_g alpha_gj ||v_j||_1
 *     (Eq. 6, mean over the query group R2) from the same pass,
 *   - selects slot = lowest-index argmin_j I_j (R7) and overwrites it in place
 *     with the current token's K/V (Fig. 2) -- or, while n < budget, appends
 *     the token at slot n (R11).
 *
 * Conventions (all entry points):
 *   - Tensor arguments are DEVICE pointers unless the name ends in _host.  bf16 means IEEE
 *     bfloat16 bit patterns (uint16).  Row-major layouts are given per argument.
 *   - The caller owns every tensor it passes.  The cache slab is library-owned (one
 *     cudaMalloc in lf_cache_create) or caller-owned (device_buf != NULL); lf_cache_destroy
 *     frees only library-owned memory.  A handle must outlive all work enqueued with it.
 *   - Errors are status codes; no exception or abort crosses the ABI.  Arguments are
 *     validated on the host before any launch; launch failures map to LF_ERR_CUDA with the
 *     CUDA error text in lf_last_error().  Asynchronous device faults surface at the
 *     caller's next synchronisation.
 *   - Device entry points only enqueue work on `stream` (a cudaStream_t; NULL = legacy
 *     default stream) and never synchronise the host, so they are CUDA-graph capturable.
 *   - A handle is not thread-safe; distinct handles (e.g. one per GPU rank) are independent
 *     (S:169).  RoPE, if any, is applied by the caller before q/k reach the ABI.
 */
#ifndef LONGFLOW_H
#define LONGFLOW_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct lf_cache lf_cache; /* opaque: host struct + device slab */

typedef enum {
    LF_OK = 0,
    LF_ERR_INVALID_ARGUMENT = 1,        /* bad shape / pointer / index */
    LF_ERR_UNSUPPORTED = 2,             /* valid but not built for (e.g. head_dim not in {64,128}) */
    LF_ERR_OUT_OF_MEMORY = 3,
    LF_ERR_PREFILL_EXCEEDS_BUDGET = 4,  /* "prefill exceeds budget; compress first" */
    LF_ERR_CUDA = 5
} lf_status;

typedef enum { LF_DTYPE_BF16 = 0, LF_DTYPE_F32 = 1 } lf_dtype;

typedef enum {
    LF_EVICT_SAME_STEP = 0,                /* R1: the current token is attended, then covers the
                                              victim chosen in this step (default)               */
    LF_EVICT_DEFERRED = 1,                 /* Fig. 2 literal: the current token first covers
                                              the slot chosen at the previous step (or is appended),
                                              attention runs over the cache, every valid slot is a
                                              candidate, the argmin is covered at the next step   */
    LF_EVICT_DEFERRED_EXCLUDE_NEWEST = 2   /* as DEFERRED, the slot just written is not a candidate */
} lf_evict_mode;

typedef enum {
    LF_KERNEL_AUTO = 0,     /* tcgen05 path when built for (G in [1, 8], d = 128), else the CUDA-core path */
    LF_KERNEL_SIMT = 1,     /* CUDA-core split-KV kernel (G <= 8, d in {64, 128}) */
    LF_KERNEL_TCGEN05 = 2   /* TMA + tcgen05 (TMEM) split-KV kernel, 2 <= G <= 8 */
} lf_kernel;

typedef struct {
    int32_t batch;         /* sequences held by this cache (a GPU rank's shard), >= 1          */
    int32_t num_q_heads;   /* Hq, multiple of num_kv_heads                                      */
    int32_t num_kv_heads;  /* Hkv; query head hq reads kv head hq / (Hq/Hkv) (R2)               */
    int32_t head_dim;      /* d in {64, 128}; other values -> LF_ERR_UNSUPPORTED                */
    int32_t budget;        /* N >= 2 static slots per (sequence, kv head)               */
    int32_t out_dtype;     /* lf_dtype of `out`: BF16 (production) or F32 (parity, R12)         */
    float softmax_scale;   /* <= 0 -> 1/sqrt(head_dim) (Eq. 1, Alg. 1, R4)          */
    int32_t mode;          /* lf_evict_mode                                                     */
    int32_t kernel;        /* lf_kernel                                                         */
    int32_t split_tokens;  /* tokens per split-KV CTA (multiple of 128), 0 = automatic plan     */
    /* Sharding by sequence ("beneficial in distributed systems").  The
     * split plan fixes each unit's reduction order (how its tokens are divided among CTAs and in
     * which order the partial (m, Z, o) are merged), so it is computed for the GLOBAL problem: a
     * rank holding sequences [seq_offset, seq_offset + batch) of a global batch passes
     * plan_batch = the global batch, and every unit is computed exactly as the one-GPU cache of
     * plan_batch sequences computes it (bit-identical out, scores and slot).  0 = this cache is
     * the whole problem (plan_batch = batch, seq_offset = 0). */
    int32_t plan_batch;    /* 0, or >= seq_offset + batch                                        */
    int32_t seq_offset;    /* first sequence of this cache in the global batch (0 if plan_batch == 0) */
    int32_t plan_shards;   /* 0/1, or P: the plan is chosen for ONE of P equal shards of plan_batch
                              (the per-GPU work of a P-GPU deployment) and then fixed for every cache of
                              that problem; it uses no whole-unit rounds, so every unit is split the same
                              way whichever cache holds it.  A one-GPU cache of the whole batch with the
                              same plan_shards reproduces the P-GPU run bit for bit.                   */
    /* Plan overrides (tests and measurements; 0 = automatic).  They change which CTAs compute a
     * unit, never what is computed. */
    int32_t ctas_per_sm;      /* tcgen05: 1 (three softmax groups, 512 TMEM columns) or 2 (one group, 256) */
    int32_t solo;             /* tcgen05: 1 = every unit split across its cluster, 2 = rounds of whole units
                                 per CTA before the split tail (needs splits > 1 and budget <= 4096)      */
    int32_t latency_variant;  /* tcgen05 split plans: 1 = streaming code, 2 = latency variant           */
} lf_cache_config;

/* Bytes of the device slab for `cfg` (K, V, per-unit valid counts, staging for the host
 * entry point), for callers that provide their own memory. */
lf_status lf_cache_bytes(const lf_cache_config* cfg, size_t* bytes);

/* Creates a cache on CUDA device `device`: every slot invalid (n_valid = 0).  device_buf ==
 * NULL -> the library performs exactly one cudaMalloc; else device_buf (>= 256-byte
 * aligned, buf_bytes >= lf_cache_bytes) is used and stays caller-owned.  Synchronous. */
lf_status lf_cache_create(const lf_cache_config* cfg, int device, void* device_buf,
                          size_t buf_bytes, lf_cache** out);

/* Frees library-owned memory and the handle (after synchronising its device). */
lf_status lf_cache_destroy(lf_cache* c);

/* Prefill: slots [0, n) of every kv head of sequence `seq` <- rows of
 * k, v (bf16 [Hkv][n][d], device), n_valid[seq][*] = n; slots >= n become invalid.
 * n > budget -> LF_ERR_PREFILL_EXCEEDS_BUDGET (SnapKV compression happens upstream).
 * n == 0 resets the sequence.  Enqueued on `stream`. */
lf_status lf_prefill_fill(lf_cache* c, int32_t seq, const void* k, const void* v, int32_t n,
                          void* stream);

/* SnapKV prefill compression (NEXT-f3; "if the number of tokens in the prefill stage exceeds
 * the budget, we first use SnapKV to compress the tokens to the budget size"; readings R22-R24):
 * per kv head, rows (g, k) = the G query heads x the last w prompt positions attend causally;
 * score_i = mean attention of prefix token i < n-w; pooled = odd-kernel 1-D max pool ('same');
 * the (budget - w) largest pooled prefix tokens (ties: lower index) plus the w window tokens, in
 * ascending order, fill slots [0, budget) of sequence `seq` (n_valid = budget).  n <= budget is a
 * plain lf_prefill_fill.
 *   k, v       bf16 [Hkv][n][d] (post-RoPE)      q_obs bf16 [Hq][w][d]: queries of positions n-w..n-1
 *   kept       int32 [Hkv][budget] or NULL: the kept prompt positions
 *   workspace  device memory of lf_snapkv_workspace_bytes(c, n, w) bytes (caller-owned)
 * Limits: n <= 65536, 1 <= w <= min(budget, n), G * w <= 128, pool_kernel odd.  Enqueued on
 * `stream`. */
lf_status lf_snapkv_workspace_bytes(const lf_cache* c, int32_t n, int32_t w, size_t* bytes);
lf_status lf_prefill_snapkv(lf_cache* c, int32_t seq, const void* k, const void* v, const void* q_obs,
                            int32_t n, int32_t w, int32_t pool_kernel, int32_t* kept, void* workspace,
                            void* stream);

/* One fused decode step over the whole cache (Alg. 1 + Fig. 2 left, same-step mode R1):
 *   q      bf16 [B][Hq][d]       current token's queries (post-RoPE)
 *   k_new  bf16 [B][Hkv][d]      current token's key   (post-RoPE)
 *   v_new  bf16 [B][Hkv][d]      current token's value
 *   out    out_dtype [B][Hq][d]  attention output o_t (Eq. 1 over n cached + current token)
 *   slot   int32 [B][Hkv]        slot now holding the current token: the evicted victim when
 *                                the unit was full, else the append slot n
 *   scores fp32 [B][Hkv][budget] or NULL: I_j of the pre-write cache, +INF for j >= n
 * The victim's K/V rows are overwritten in place; n_valid grows by one for appending units.
 * Enqueued on `stream`; no host synchronisation. */
lf_status lf_decode_step(lf_cache* c, const void* q, const void* k_new, const void* v_new,
                         void* out, int32_t* slot, float* scores, void* stream);

/* Approximation diagnostics (NEXT-f4; PAPER §3.3, App. A): call BEFORE lf_decode_step with the same
 * inputs; reads the pre-step cache.  Per unit, the exact eviction objective with the current query
 * E_i = mean_g ||o_g - o_g^(\i)||^2 (Eq. 3's right-hand side, via the exact remainder P:424-426) is
 * compared with LongFlowScore (Eq. 6):
 *   islot int32 [B][Hkv][3]: {LongFlow victim, argmin_i E_i (lowest index on ties), rank of the
 *                             LongFlow victim under E (0 = the same quality)}  (-1 if n == 0)
 *   fstat fp32 [B][Hkv][3]:  {E(LongFlow victim), E(exact victim), max_i ||R_i|| / bound (<= 1)}
 *   workspace: lf_diag_workspace_bytes bytes of device memory.  Plain CUDA-core kernel (not the hot path). */
lf_status lf_diag_workspace_bytes(const lf_cache* c, size_t* bytes);
lf_status lf_diagnose_step(lf_cache* c, const void* q, const void* k_new, const void* v_new, int32_t* islot,
                           float* fstat, void* workspace, void* stream);

/* Same step with HOST buffers (the end-to-end entry point), synchronous: small steps (<= 256 KB of
 * I/O) are packed into the cache's mapped pinned staging buffer and the kernel reads the inputs and
 * writes out/slot there directly (zero-copy); larger steps copy q/k_new/v_new host -> device (pinned
 * host memory recommended), run lf_decode_step on `stream` and copy out and slot device -> host.
 * `stream` is synchronised before returning. Layouts as above. */
lf_status lf_decode_step_host(lf_cache* c, const void* q_host, const void* k_new_host,
                              const void* v_new_host, void* out_host, int32_t* slot_host,
                              void* stream);

/* Device views for snapshots and tests: K, V bf16 [B][Hkv][budget][d]; n_valid int32
 * [B][Hkv] (one count per unit; all heads of a sequence carry the same value). */
lf_status lf_cache_views(const lf_cache* c, void** k, void** v, int32_t** n_valid);

/* The split plan the next lf_decode_step will launch: kernel id (lf_kernel), splits per
 * unit (CTAs per cluster) and tokens per split. */
lf_status lf_cache_plan(const lf_cache* c, int32_t* kernel, int32_t* splits,
                        int32_t* split_tokens);

/* More of the plan: persistent clusters in the grid (0 = one cluster per unit), TMA ring stages,
 * TMEM columns per CTA (512 = one CTA per SM, 256 = two, 0 = CUDA-core kernel), SMEM bytes per CTA,
 * rounds of whole units per CTA before the units split across the cluster (of the plan_batch
 * problem), and whether split units use the latency variant (1) or the streaming code (0).  NULL
 * outputs are skipped. */
lf_status lf_cache_plan_detail(const lf_cache* c, int32_t* clusters, int32_t* stages, int32_t* tmem_cols,
                               int32_t* smem_bytes, int32_t* solo_rounds, int32_t* latency_variant);

/* Deferred modes: device view of int32 [B][Hkv], the slot the next step's token will cover
 * (-1 = none yet).  In deferred modes lf_decode_step's `slot` returns where the current token
 * was written, and `scores` covers every valid slot including it. */
lf_status lf_cache_pending(const lf_cache* c, int32_t** pend);

/* Number of CUDA kernels lf_decode_step launches per call (for launch accounting). */
int32_t lf_kernels_per_step(const lf_cache* c);

/* Debug only: buffer receiving per-CTA %globaltimer events from builds compiled with -DLF_TRACE, or
 * (mapped pinned host memory) the stuck-wait log and progress counters of -DLF_HANG_DIAG builds
 * (tools/hang_diag.py); ignored by the product build; NULL disables.  Layout: DESIGN.md "Tracing". */
lf_status lf_debug_set_trace(lf_cache* c, void* device_buf);

const char* lf_status_string(lf_status s);
const char* lf_last_error(void); /* thread-local detail text of the last failure */

#ifdef __cplusplus
}
#endif
#endif /* LONGFLOW_H */
