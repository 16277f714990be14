// Host runtime of the LongFlow C ABI (include/longflow.h): validation, the static cache slab,
// prefill, split planning and decode-step dispatch.  No torch types anywhere.
//
// Static memory ("allocations == 1"): one slab per cache holding
//   K, V       bf16 [B][Hkv][N][d]
//   n_valid    int32 [B][Hkv]
//   staging    q/k_new/v_new/out/slot device copies for lf_decode_step_host
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <mutex>
#include <new>
#include <utility>
#include <vector>

#include "lf_internal.h"

namespace {

thread_local char g_err[512] = "";

lf_status fail(lf_status s, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
lf_status fail(lf_status s, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return s;
}

lf_status cuda_fail(cudaError_t e, const char* what) {
    return fail(LF_ERR_CUDA, "%s: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
}

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

struct Layout {
    size_t k_off, v_off, nv_off, pd_off, sq_off, sk_off, sv_off, so_off, ss_off, total;
};

Layout layout_of(const lf_cache_config& c) {
    Layout L;
    size_t kv = (size_t)c.batch * c.num_kv_heads * c.budget * c.head_dim * 2;
    size_t off = 0;
    L.k_off = off; off = align_up(off + kv, 256);
    L.v_off = off; off = align_up(off + kv, 256);
    L.nv_off = off; off = align_up(off + (size_t)c.batch * c.num_kv_heads * 4, 256);
    L.pd_off = off; off = align_up(off + (size_t)c.batch * c.num_kv_heads * 4, 256);
    L.sq_off = off; off = align_up(off + (size_t)c.batch * c.num_q_heads * c.head_dim * 2, 256);
    L.sk_off = off; off = align_up(off + (size_t)c.batch * c.num_kv_heads * c.head_dim * 2, 256);
    L.sv_off = off; off = align_up(off + (size_t)c.batch * c.num_kv_heads * c.head_dim * 2, 256);
    L.so_off = off; off = align_up(off + (size_t)c.batch * c.num_q_heads * c.head_dim * 4, 256);
    L.ss_off = off; off = align_up(off + (size_t)c.batch * c.num_kv_heads * 4, 256);
    L.total = off;
    return L;
}

lf_status validate(const lf_cache_config* c) {
    if (!c) return fail(LF_ERR_INVALID_ARGUMENT, "cfg is NULL");
    if (c->batch < 1) return fail(LF_ERR_INVALID_ARGUMENT, "batch must be >= 1 (got %d)", c->batch);
    if (c->num_kv_heads < 1 || c->num_q_heads < 1)
        return fail(LF_ERR_INVALID_ARGUMENT, "head counts must be >= 1");
    if (c->num_q_heads % c->num_kv_heads)
        return fail(LF_ERR_INVALID_ARGUMENT, "num_q_heads %% num_kv_heads != 0 (%d, %d)",
                    c->num_q_heads, c->num_kv_heads);
    if (c->head_dim < 1) return fail(LF_ERR_INVALID_ARGUMENT, "head_dim must be >= 1");
    if (c->budget < 2) return fail(LF_ERR_INVALID_ARGUMENT, "budget must be >= 2 (S:123)");
    if (c->out_dtype != LF_DTYPE_BF16 && c->out_dtype != LF_DTYPE_F32)
        return fail(LF_ERR_INVALID_ARGUMENT, "unknown out_dtype %d", c->out_dtype);
    if (c->mode != LF_EVICT_SAME_STEP && c->mode != LF_EVICT_DEFERRED && c->mode != LF_EVICT_DEFERRED_EXCLUDE_NEWEST)
        return fail(LF_ERR_INVALID_ARGUMENT, "unknown mode %d", c->mode);
    if (c->kernel < LF_KERNEL_AUTO || c->kernel > LF_KERNEL_TCGEN05)
        return fail(LF_ERR_INVALID_ARGUMENT, "unknown kernel %d", c->kernel);
    if (c->split_tokens < 0 || c->split_tokens % 128)
        return fail(LF_ERR_INVALID_ARGUMENT, "split_tokens must be a multiple of 128 (got %d)",
                    c->split_tokens);
    if (c->head_dim != 64 && c->head_dim != 128)
        return fail(LF_ERR_UNSUPPORTED, "head_dim %d not built (64, 128)", c->head_dim);
    int G = c->num_q_heads / c->num_kv_heads;
    if (G > 16) return fail(LF_ERR_UNSUPPORTED, "group size %d > 16 not built", G);
    if (c->plan_batch < 0 || c->seq_offset < 0)
        return fail(LF_ERR_INVALID_ARGUMENT, "plan_batch and seq_offset must be >= 0");
    if (c->plan_batch == 0 && c->seq_offset != 0)
        return fail(LF_ERR_INVALID_ARGUMENT, "seq_offset %d needs plan_batch (the global batch)", c->seq_offset);
    if (c->plan_batch > 0 && (long long)c->seq_offset + c->batch > c->plan_batch)
        return fail(LF_ERR_INVALID_ARGUMENT, "sequences [%d, %d) exceed plan_batch %d", c->seq_offset,
                    c->seq_offset + c->batch, c->plan_batch);
    if (c->plan_shards < 0 || c->plan_shards > 4096)
        return fail(LF_ERR_INVALID_ARGUMENT, "plan_shards %d out of [0, 4096]", c->plan_shards);
    if (c->plan_shards > 1 && c->solo == 2)
        return fail(LF_ERR_INVALID_ARGUMENT, "plan_shards > 1 plans have no whole-unit rounds (solo = 2)");
    if (c->ctas_per_sm < 0 || c->ctas_per_sm > 2 || c->solo < 0 || c->solo > 2 || c->latency_variant < 0 ||
        c->latency_variant > 2)
        return fail(LF_ERR_INVALID_ARGUMENT, "plan overrides must be 0 (automatic), 1 or 2");
    if ((long long)(c->plan_batch > c->batch ? c->plan_batch : c->batch) * c->num_kv_heads > 0x7fffffff / 2)
        return fail(LF_ERR_INVALID_ARGUMENT, "too many units");
    if (c->budget > 65536) return fail(LF_ERR_UNSUPPORTED, "budget %d > 65536 not built", c->budget);
    return LF_OK;
}

__global__ void fill_i32(int32_t* p, int32_t v, int n) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = v;
}

// Deferred mode pre-pass (Fig. 2 left): one warp per unit.  The current token covers the
// slot chosen at the previous step when the unit is full, else it is appended at n (R11);
// slot[u] returns where it went.  A full unit always has a pending slot here: every step sets one
// and lf_decode_step refuses a sequence whose prefill filled the whole budget (R26); the
// fallback to slot 0 only guards against a caller overwriting pend through the views.
__global__ void deferred_write_kernel(lf::StepParams p) {
    const int u = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (u >= p.B * p.Hkv) return;
    const int n = p.n_valid[u];
    int s;
    if (n < p.N) s = n;
    else s = p.pend[u] >= 0 && p.pend[u] < p.N ? p.pend[u] : 0;
    const int rows = p.d / 8;   // uint4 per row
    const size_t dst = ((size_t)u * p.N + s) * p.d;
    if (lane < rows) ((uint4*)(p.K + dst))[lane] = ((const uint4*)(p.k_new + (size_t)u * p.d))[lane];
    else if (lane < 2 * rows) ((uint4*)(p.V + dst))[lane - rows] = ((const uint4*)(p.v_new + (size_t)u * p.d))[lane - rows];
    if (lane == 0) {
        p.slot[u] = s;
        if (n < p.N) p.n_valid[u] = n + 1;
    }
}

}  // namespace

struct lf_cache {
    lf_cache_config cfg;
    int device;
    int num_sms;
    void* slab;
    size_t slab_bytes;
    bool owns;
    Layout L;
    lf::Plan plan;       // the plan of the plan_batch problem (fixes every unit's reduction order)
    int32_t launch_clusters;   // clusters launched for THIS cache's units
    int32_t solo_units;        // this cache's units [0, solo_units) are computed whole by one CTA
    std::vector<unsigned char> needs_pend;   // deferred modes: sequence full after prefill, no victim yet
    lf::TcMaps maps;
    unsigned long long* trace;
    char* host_stage;      // mapped pinned staging for small lf_decode_step_host calls (zero-copy)
    char* host_stage_dev;  // its device-side address

};

namespace {
// lf_decode_step_host packs the inputs (and the outputs) into one transfer each when they are small:
// a copy costs microseconds of fixed latency, a host memcpy of a few KB almost nothing
constexpr size_t kPackLimit = 256 * 1024;
size_t stage_in_bytes(const Layout& L, const lf_cache_config& g) {
    return L.sv_off + (size_t)g.batch * g.num_kv_heads * g.head_dim * 2 - L.sq_off;
}
size_t stage_out_bytes(const Layout& L, const lf_cache_config& g) {
    return L.ss_off + (size_t)g.batch * g.num_kv_heads * 4 - L.so_off;
}
}  // namespace

namespace lf {
int fill_launch_attrs(cudaLaunchAttribute* attr, int cluster_x) {
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cluster_x;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    return 2;
}

cudaError_t deferred_write_launch(const StepParams& p, cudaStream_t stream) {
    const int units = p.B * p.Hkv;
    deferred_write_kernel<<<(units + 7) / 8, 256, 0, stream>>>(p);
    return cudaGetLastError();
}
}  // namespace lf

namespace {

lf_status make_plan(lf_cache* c) {
    const lf_cache_config& g = c->cfg;
    int G = g.num_q_heads / g.num_kv_heads;
    const int units = g.batch * g.num_kv_heads;
    const int plan_units = (g.plan_batch > 0 ? g.plan_batch : g.batch) * g.num_kv_heads;
    const int shards = g.plan_shards > 1 ? g.plan_shards : 1;
    const int shard_units = (plan_units + shards - 1) / shards;   // the plan is chosen for one shard
    bool want_tc = g.kernel == LF_KERNEL_TCGEN05 ||
                   (g.kernel == LF_KERNEL_AUTO && lf::tc_supported(G, g.head_dim));
    c->solo_units = 0;
    if (want_tc) {
        if (!lf::tc_supported(G, g.head_dim))
            return fail(LF_ERR_UNSUPPORTED, "tcgen05 kernel not built for G=%d d=%d", G, g.head_dim);
        // The plan depends only on the problem shape, the overrides and the device (occupancy queries:
        // ~1 ms per plan), and a model creates one cache per layer with the same shape: memoise it.
        struct Key {
            int dev, units, G, d, N, split, sms, k, solo, lat, shards;
            bool operator==(const Key& o) const {
                return dev == o.dev && units == o.units && G == o.G && d == o.d && N == o.N && split == o.split &&
                       sms == o.sms && k == o.k && solo == o.solo && lat == o.lat && shards == o.shards;
            }
        };
        static std::mutex mu;
        static std::vector<std::pair<Key, lf::Plan>> memo;
        const Key k{c->device, shard_units, G, g.head_dim, g.budget, g.split_tokens, c->num_sms,
                    g.ctas_per_sm, g.solo, g.latency_variant, shards > 1};
        bool hit = false;
        {
            std::lock_guard<std::mutex> lock(mu);
            for (const auto& e : memo)
                if (e.first == k) {
                    c->plan = e.second;
                    hit = true;
                    break;
                }
        }
        if (!hit) {
            const lf::PlanForce force{g.ctas_per_sm, g.solo, g.latency_variant, shards > 1};
            c->plan = lf::tc_plan(shard_units, G, g.head_dim, g.budget, g.split_tokens, c->num_sms, force);
            if (c->plan.splits > 0) {
                std::lock_guard<std::mutex> lock(mu);
                memo.push_back({k, c->plan});
            }
        }
        if (c->plan.splits < 1)
            return fail(LF_ERR_UNSUPPORTED, "no tcgen05 plan for budget %d, split_tokens %d and the overrides "
                        "(ctas_per_sm %d, solo %d, latency_variant %d)", g.budget, g.split_tokens,
                        g.ctas_per_sm, g.solo, g.latency_variant);
        // this cache's share of the plan_batch problem: the same units are whole or split as there
        const long long P = (long long)c->plan.clusters * c->plan.splits;
        long long gsolo = (long long)c->plan.solo_rounds * P;
        if (gsolo > plan_units) gsolo = plan_units;
        long long ls = gsolo - (long long)g.seq_offset * g.num_kv_heads;
        c->solo_units = (int32_t)(ls < 0 ? 0 : ls > units ? units : ls);
        c->launch_clusters = c->plan.clusters;
        if (c->solo_units == 0 && c->launch_clusters > units) c->launch_clusters = units;
    } else {
        if (!lf::simt_supported(G, g.head_dim))
            return fail(LF_ERR_UNSUPPORTED, "CUDA-core kernel not built for G=%d d=%d", G, g.head_dim);
        c->plan = lf::simt_plan(shard_units, G, g.head_dim, g.budget, g.split_tokens, c->num_sms);
        c->launch_clusters = 0;
    }
    if (c->plan.splits < 1 || c->plan.splits > 16)
        return fail(LF_ERR_UNSUPPORTED, "split plan out of range (%d splits)", c->plan.splits);
    return LF_OK;
}

}  // namespace

extern "C" {

const char* lf_status_string(lf_status s) {
    switch (s) {
        case LF_OK: return "LF_OK";
        case LF_ERR_INVALID_ARGUMENT: return "LF_ERR_INVALID_ARGUMENT";
        case LF_ERR_UNSUPPORTED: return "LF_ERR_UNSUPPORTED";
        case LF_ERR_OUT_OF_MEMORY: return "LF_ERR_OUT_OF_MEMORY";
        case LF_ERR_PREFILL_EXCEEDS_BUDGET: return "LF_ERR_PREFILL_EXCEEDS_BUDGET";
        case LF_ERR_CUDA: return "LF_ERR_CUDA";
    }
    return "LF_ERR_UNKNOWN";
}

const char* lf_last_error(void) { return g_err; }

lf_status lf_cache_bytes(const lf_cache_config* cfg, size_t* bytes) {
    lf_status s = validate(cfg);
    if (s) return s;
    if (!bytes) return fail(LF_ERR_INVALID_ARGUMENT, "bytes is NULL");
    *bytes = layout_of(*cfg).total;
    return LF_OK;
}

lf_status lf_cache_create(const lf_cache_config* cfg, int device, void* device_buf, size_t buf_bytes,
                          lf_cache** out) {
    lf_status s = validate(cfg);
    if (s) return s;
    if (!out) return fail(LF_ERR_INVALID_ARGUMENT, "out is NULL");
    *out = nullptr;
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDeviceCount");
    if (device < 0 || device >= ndev) return fail(LF_ERR_INVALID_ARGUMENT, "device %d of %d", device, ndev);
    int prev = 0;
    cudaGetDevice(&prev);
    if ((e = cudaSetDevice(device)) != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
    cudaDeviceProp prop;
    if ((e = cudaGetDeviceProperties(&prop, device)) != cudaSuccess) return cuda_fail(e, "props");
    if (prop.major != 10) {
        cudaSetDevice(prev);
        return fail(LF_ERR_UNSUPPORTED, "device %d is sm_%d%d; this library is built for sm_100a",
                    device, prop.major, prop.minor);
    }
    lf_cache* c = new (std::nothrow) lf_cache();
    if (!c) return fail(LF_ERR_OUT_OF_MEMORY, "host allocation");
    c->cfg = *cfg;
    if (!(c->cfg.softmax_scale > 0.f)) c->cfg.softmax_scale = 1.0f / sqrtf((float)cfg->head_dim);
    c->device = device;
    c->num_sms = prop.multiProcessorCount;
    c->L = layout_of(c->cfg);
    c->needs_pend.assign((size_t)cfg->batch, 0);
    if ((s = make_plan(c)) != LF_OK) { delete c; cudaSetDevice(prev); return s; }
    if (device_buf) {
        if (buf_bytes < c->L.total || ((uintptr_t)device_buf & 255)) {
            delete c;
            cudaSetDevice(prev);
            return fail(LF_ERR_INVALID_ARGUMENT, "device_buf too small (%zu < %zu) or not 256-aligned",
                        buf_bytes, c->L.total);
        }
        c->slab = device_buf;
        c->owns = false;
    } else {
        e = cudaMalloc(&c->slab, c->L.total);
        if (e != cudaSuccess) {
            delete c;
            cudaSetDevice(prev);
            cudaGetLastError();
            return fail(LF_ERR_OUT_OF_MEMORY, "cudaMalloc(%zu): %s", c->L.total, cudaGetErrorString(e));
        }
        c->owns = true;
    }
    c->slab_bytes = c->L.total;
    c->host_stage = nullptr;
    c->host_stage_dev = nullptr;
    if (stage_in_bytes(c->L, c->cfg) + stage_out_bytes(c->L, c->cfg) <= kPackLimit) {
        if (cudaHostAlloc((void**)&c->host_stage, stage_in_bytes(c->L, c->cfg) + stage_out_bytes(c->L, c->cfg),
                          cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess ||
            cudaHostGetDevicePointer((void**)&c->host_stage_dev, c->host_stage, 0) != cudaSuccess) {
            if (c->host_stage) cudaFreeHost(c->host_stage);
            c->host_stage = nullptr;   // optional: fall back to one copy per tensor
            c->host_stage_dev = nullptr;
            cudaGetLastError();
        }
    }
    if (c->plan.kernel == LF_KERNEL_TCGEN05 &&
        !lf::tc_make_maps(&c->maps, (char*)c->slab + c->L.k_off, (char*)c->slab + c->L.v_off,
                          (long long)cfg->batch * cfg->num_kv_heads, cfg->budget, cfg->head_dim)) {
        if (c->owns) cudaFree(c->slab);
        delete c;
        cudaSetDevice(prev);
        return fail(LF_ERR_CUDA, "cuTensorMapEncodeTiled failed for the K/V tensor maps");
    }
    // all slots invalid; zero-filled storage; no pending victim (-1)
    e = cudaMemset(c->slab, 0, c->L.total);
    if (e == cudaSuccess) e = cudaMemset((char*)c->slab + c->L.pd_off, 0xff, (size_t)cfg->batch * cfg->num_kv_heads * 4);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    cudaSetDevice(prev);
    if (e != cudaSuccess) {
        if (c->owns) cudaFree(c->slab);
        delete c;
        return cuda_fail(e, "cache init");
    }
    *out = c;
    return LF_OK;
}

lf_status lf_cache_destroy(lf_cache* c) {
    if (!c) return fail(LF_ERR_INVALID_ARGUMENT, "cache is NULL");
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(c->device);
    cudaError_t e = cudaDeviceSynchronize();
    if (c->owns) cudaFree(c->slab);
    if (c->host_stage) cudaFreeHost(c->host_stage);
    cudaSetDevice(prev);
    delete c;
    if (e != cudaSuccess) return cuda_fail(e, "destroy");
    return LF_OK;
}

lf_status lf_cache_views(const lf_cache* c, void** k, void** v, int32_t** n_valid) {
    if (!c) return fail(LF_ERR_INVALID_ARGUMENT, "cache is NULL");
    char* base = (char*)c->slab;
    if (k) *k = base + c->L.k_off;
    if (v) *v = base + c->L.v_off;
    if (n_valid) *n_valid = (int32_t*)(base + c->L.nv_off);
    return LF_OK;
}

lf_status lf_cache_plan(const lf_cache* c, int32_t* kernel, int32_t* splits, int32_t* split_tokens) {
    if (!c) return fail(LF_ERR_INVALID_ARGUMENT, "cache is NULL");
    if (kernel) *kernel = c->plan.kernel;
    if (splits) *splits = c->plan.splits;
    if (split_tokens) *split_tokens = c->plan.chunk;
    return LF_OK;
}

lf_status lf_cache_plan_detail(const lf_cache* c, int32_t* clusters, int32_t* stages, int32_t* tmem_cols,
                                int32_t* smem_bytes, int32_t* solo_rounds, int32_t* latency_variant) {
    if (!c) return fail(LF_ERR_INVALID_ARGUMENT, "cache is NULL");
    if (solo_rounds) *solo_rounds = c->plan.solo_rounds;
    if (latency_variant) *latency_variant = c->plan.lat;
    if (clusters) *clusters = c->launch_clusters;
    if (stages) *stages = c->plan.stages;
    if (tmem_cols) *tmem_cols = c->plan.tmem_cols;
    if (smem_bytes) *smem_bytes = c->plan.smem;
    return LF_OK;
}

int32_t lf_kernels_per_step(const lf_cache* c) { return c ? (c->cfg.mode == LF_EVICT_SAME_STEP ? 1 : 2) : 0; }

lf_status lf_cache_pending(const lf_cache* c, int32_t** pend) {
    if (!c || !pend) return fail(LF_ERR_INVALID_ARGUMENT, "cache or pend is NULL");
    *pend = (int32_t*)((char*)c->slab + c->L.pd_off);
    return LF_OK;
}

lf_status lf_debug_set_trace(lf_cache* c, void* device_buf) {
    if (!c) return fail(LF_ERR_INVALID_ARGUMENT, "cache is NULL");
    c->trace = (unsigned long long*)device_buf;
    return LF_OK;
}

// After a prefill of n tokens: n_valid = n for every kv head of `seq`, no pending victim (deferred
// modes), and a sequence whose prefill filled the whole budget is marked: its first deferred step
// would have no slot to cover (R26)
static cudaError_t reset_seq(lf_cache* c, int32_t seq, int32_t n, cudaStream_t st) {
    const lf_cache_config& g = c->cfg;
    char* base = (char*)c->slab;
    const int blocks = (g.num_kv_heads + 255) / 256;
    int32_t* nv = (int32_t*)(base + c->L.nv_off) + (size_t)seq * g.num_kv_heads;
    int32_t* pd = (int32_t*)(base + c->L.pd_off) + (size_t)seq * g.num_kv_heads;
    fill_i32<<<blocks, 256, 0, st>>>(nv, n, g.num_kv_heads);
    fill_i32<<<blocks, 256, 0, st>>>(pd, -1, g.num_kv_heads);
    if (g.mode != LF_EVICT_SAME_STEP) c->needs_pend[seq] = n >= g.budget;
    return cudaGetLastError();
}

lf_status lf_prefill_fill(lf_cache* c, int32_t seq, const void* k, const void* v, int32_t n,
                          void* stream) {
    if (!c) return fail(LF_ERR_INVALID_ARGUMENT, "cache is NULL");
    const lf_cache_config& g = c->cfg;
    if (seq < 0 || seq >= g.batch) return fail(LF_ERR_INVALID_ARGUMENT, "seq %d of %d", seq, g.batch);
    if (n < 0) return fail(LF_ERR_INVALID_ARGUMENT, "n < 0");
    if (n > g.budget)
        return fail(LF_ERR_PREFILL_EXCEEDS_BUDGET, "prefill exceeds budget; compress first (%d > %d)", n,
                    g.budget);
    if (n > 0 && (!k || !v)) return fail(LF_ERR_INVALID_ARGUMENT, "k or v is NULL");
    cudaStream_t st = (cudaStream_t)stream;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(c->device);
    char* base = (char*)c->slab;
    size_t row = (size_t)g.head_dim * 2;
    size_t unit = (size_t)g.budget * row;
    cudaError_t e = cudaSuccess;
    if (n > 0) {
        char* K = base + c->L.k_off + (size_t)seq * g.num_kv_heads * unit;
        char* V = base + c->L.v_off + (size_t)seq * g.num_kv_heads * unit;
        e = cudaMemcpy2DAsync(K, unit, k, n * row, n * row, g.num_kv_heads, cudaMemcpyDeviceToDevice, st);
        if (e == cudaSuccess)
            e = cudaMemcpy2DAsync(V, unit, v, n * row, n * row, g.num_kv_heads, cudaMemcpyDeviceToDevice, st);
    }
    if (e == cudaSuccess) e = reset_seq(c, seq, n, st);
    cudaSetDevice(prev);
    if (e != cudaSuccess) return cuda_fail(e, "prefill");
    return LF_OK;
}

static lf_status snapkv_check(const lf_cache* c, int32_t n, int32_t w, int32_t pool_kernel) {
    const lf_cache_config& g = c->cfg;
    const int G = g.num_q_heads / g.num_kv_heads;
    if (n < 1 || n > 65536) return fail(LF_ERR_INVALID_ARGUMENT, "prompt length %d out of [1, 65536]", n);
    if (w < 1 || w > g.budget || w > n) return fail(LF_ERR_INVALID_ARGUMENT, "window %d must be in [1, min(budget, n)]", w);
    if ((long long)G * w > lf::kSnapRowsMax)
        return fail(LF_ERR_UNSUPPORTED, "G * window = %d > %d observation rows", G * w, lf::kSnapRowsMax);
    if (pool_kernel < 1 || pool_kernel % 2 == 0) return fail(LF_ERR_INVALID_ARGUMENT, "pool kernel must be odd");
    return LF_OK;
}

lf_status lf_snapkv_workspace_bytes(const lf_cache* c, int32_t n, int32_t w, size_t* bytes) {
    if (!c || !bytes) return fail(LF_ERR_INVALID_ARGUMENT, "cache or bytes is NULL");
    lf_status s = snapkv_check(c, n, w, 1);
    if (s) return s;
    const lf_cache_config& g = c->cfg;
    *bytes = n > g.budget ? lf::snapkv_workspace_bytes(g.num_kv_heads, g.num_q_heads / g.num_kv_heads, n, w, g.budget)
                          : 0;
    return LF_OK;
}

lf_status lf_prefill_snapkv(lf_cache* c, int32_t seq, const void* k, const void* v, const void* q_obs, int32_t n,
                            int32_t w, int32_t pool_kernel, int32_t* kept, void* workspace, void* stream) {
    if (!c) return fail(LF_ERR_INVALID_ARGUMENT, "cache is NULL");
    const lf_cache_config& g = c->cfg;
    if (seq < 0 || seq >= g.batch) return fail(LF_ERR_INVALID_ARGUMENT, "seq %d of %d", seq, g.batch);
    lf_status s = snapkv_check(c, n, w, pool_kernel);
    if (s) return s;
    if (!k || !v) return fail(LF_ERR_INVALID_ARGUMENT, "k or v is NULL");
    if (n <= g.budget) return lf_prefill_fill(c, seq, k, v, n, stream);   // nothing to compress
    if (!q_obs || !workspace) return fail(LF_ERR_INVALID_ARGUMENT, "q_obs and workspace are required when n > budget");
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(c->device);
    char* base = (char*)c->slab;
    cudaError_t e = reset_seq(c, seq, 0, (cudaStream_t)stream);
    if (e == cudaSuccess)
        e = lf::snapkv_launch((uint16_t*)(base + c->L.k_off), (uint16_t*)(base + c->L.v_off),
                              (int32_t*)(base + c->L.nv_off), seq, g.num_kv_heads, g.num_q_heads / g.num_kv_heads,
                              g.head_dim, g.budget, k, v, q_obs, n, w, pool_kernel, g.softmax_scale, kept,
                              workspace, (cudaStream_t)stream);
    if (g.mode != LF_EVICT_SAME_STEP) c->needs_pend[seq] = 1;   // SnapKV fills the whole budget
    cudaSetDevice(prev);
    if (e != cudaSuccess) return cuda_fail(e, "snapkv");
    return LF_OK;
}

lf_status lf_diag_workspace_bytes(const lf_cache* c, size_t* bytes) {
    if (!c || !bytes) return fail(LF_ERR_INVALID_ARGUMENT, "cache or bytes is NULL");
    const lf_cache_config& g = c->cfg;
    *bytes = lf::diag_workspace_bytes(g.batch * g.num_kv_heads, g.num_q_heads / g.num_kv_heads, g.budget);
    return LF_OK;
}

lf_status lf_diagnose_step(lf_cache* c, const void* q, const void* k_new, const void* v_new, int32_t* islot,
                           float* fstat, void* workspace, void* stream) {
    if (!c) return fail(LF_ERR_INVALID_ARGUMENT, "cache is NULL");
    if (!q || !k_new || !v_new || !islot || !fstat || !workspace)
        return fail(LF_ERR_INVALID_ARGUMENT, "q, k_new, v_new, islot, fstat and workspace must be non-NULL");
    const lf_cache_config& g = c->cfg;
    if (g.num_q_heads / g.num_kv_heads > 8) return fail(LF_ERR_UNSUPPORTED, "diagnostics built for G <= 8");
    char* base = (char*)c->slab;
    lf::StepParams p = {};
    p.q = (const uint16_t*)q;
    p.k_new = (const uint16_t*)k_new;
    p.v_new = (const uint16_t*)v_new;
    p.K = (uint16_t*)(base + c->L.k_off);
    p.V = (uint16_t*)(base + c->L.v_off);
    p.B = g.batch;
    p.Hq = g.num_q_heads;
    p.Hkv = g.num_kv_heads;
    p.G = g.num_q_heads / g.num_kv_heads;
    p.d = g.head_dim;
    p.N = g.budget;
    p.scale_log2 = (float)((double)g.softmax_scale * 1.4426950408889634);
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(c->device);
    cudaError_t e = lf::diag_launch(p, (const int32_t*)(base + c->L.nv_off), workspace, islot, fstat,
                                    (cudaStream_t)stream);
    cudaSetDevice(prev);
    if (e != cudaSuccess) return cuda_fail(e, "diagnose");
    return LF_OK;
}

// One decode-step launch over sequences [b0, b0 + nb) of the cache (the whole cache for the public
// entry point; the host entry point pipelines chunks).  q, k_new, v_new, out, slot and scores point at
// the rows of sequence b0.  A chunk computes every unit exactly as the whole-cache launch does: same
// plan, whole-vs-split decided by cache unit index, TMA rows from unit_base.
static lf_status decode_impl(lf_cache* c, const void* q, const void* k_new, const void* v_new, void* out,
                             int32_t* slot, float* scores, void* stream, int host_io, int b0, int nb);

lf_status lf_decode_step(lf_cache* c, const void* q, const void* k_new, const void* v_new, void* out,
                         int32_t* slot, float* scores, void* stream) {
    return decode_impl(c, q, k_new, v_new, out, slot, scores, stream, 0, 0, c ? c->cfg.batch : 0);
}

static lf_status decode_impl(lf_cache* c, const void* q, const void* k_new, const void* v_new, void* out,
                             int32_t* slot, float* scores, void* stream, int host_io, int b0, int nb) {
    if (!c) return fail(LF_ERR_INVALID_ARGUMENT, "cache is NULL");
    if (!q || !k_new || !v_new || !out || !slot)
        return fail(LF_ERR_INVALID_ARGUMENT, "q, k_new, v_new, out and slot must be non-NULL");
    // the kernels move q, k_new, v_new and out in 16-byte vectors
    if (((uintptr_t)q | (uintptr_t)k_new | (uintptr_t)v_new | (uintptr_t)out) & 15)
        return fail(LF_ERR_INVALID_ARGUMENT, "q, k_new, v_new and out must be 16-byte aligned");
    if (((uintptr_t)slot | (uintptr_t)scores) & 3)
        return fail(LF_ERR_INVALID_ARGUMENT, "slot and scores must be 4-byte aligned");
    const lf_cache_config& g = c->cfg;
    if (g.mode != LF_EVICT_SAME_STEP)
        for (int b = 0; b < g.batch; ++b)
            if (c->needs_pend[b])
                return fail(LF_ERR_INVALID_ARGUMENT,
                            "deferred mode: sequence %d was prefilled to the whole budget, so there is no slot "
                            "chosen at a previous step for its current token to cover (Fig. 2, P:152; R26); "
                            "prefill fewer than budget tokens or use LF_EVICT_SAME_STEP", b);
    char* base = (char*)c->slab;
    const size_t u0 = (size_t)b0 * g.num_kv_heads;   // first cache unit of this launch
    lf::StepParams p;
    p.q = (const uint16_t*)q;
    p.k_new = (const uint16_t*)k_new;
    p.v_new = (const uint16_t*)v_new;
    p.K = (uint16_t*)(base + c->L.k_off) + u0 * g.budget * g.head_dim;
    p.V = (uint16_t*)(base + c->L.v_off) + u0 * g.budget * g.head_dim;
    p.n_valid = (int32_t*)(base + c->L.nv_off) + u0;
    p.out = out;
    p.slot = slot;
    p.scores = scores;
    p.trace = c->trace;
    p.deferred = g.mode != LF_EVICT_SAME_STEP;
    p.exclude_newest = g.mode == LF_EVICT_DEFERRED_EXCLUDE_NEWEST;
    p.pend = (int32_t*)(base + c->L.pd_off) + u0;
    p.written = slot;
    p.B = nb;
    p.Hq = g.num_q_heads;
    p.Hkv = g.num_kv_heads;
    p.G = g.num_q_heads / g.num_kv_heads;
    p.d = g.head_dim;
    p.N = g.budget;
    p.out_f32 = g.out_dtype == LF_DTYPE_F32;
    p.scale_log2 = (float)((double)g.softmax_scale * 1.4426950408889634);
    p.splits = c->plan.splits;
    p.chunk = c->plan.chunk;
    const long long units = (long long)nb * g.num_kv_heads;
    long long ls = (long long)c->solo_units - (long long)u0;
    p.solo_units = (int32_t)(ls < 0 ? 0 : ls > units ? units : ls);
    p.unit_base = (int32_t)u0;
    p.host_io = host_io;
    p.hold = c->plan.kernel == LF_KERNEL_TCGEN05 ? lf::tc_hold(c->plan, g.budget) : 0;
    lf::Plan lp = c->plan;
    lp.clusters = c->launch_clusters;
    if (p.solo_units == 0 && lp.clusters > units) lp.clusters = (int32_t)units;
    int prev = 0;
    cudaGetDevice(&prev);
    if (prev != c->device) cudaSetDevice(c->device);
    cudaError_t e = cudaSuccess;
    if (p.deferred) e = lf::deferred_write_launch(p, (cudaStream_t)stream);
    if (e == cudaSuccess)
        e = c->plan.kernel == LF_KERNEL_TCGEN05 ? lf::tc_launch(p, lp, c->maps, (cudaStream_t)stream)
                                                 : lf::simt_launch(p, lp, (cudaStream_t)stream);
    if (prev != c->device) cudaSetDevice(prev);
    if (e != cudaSuccess) return cuda_fail(e, "decode launch");
    return LF_OK;
}

lf_status lf_decode_step_host(lf_cache* c, const void* q_host, const void* k_new_host,
                              const void* v_new_host, void* out_host, int32_t* slot_host, void* stream) {
    if (!c) return fail(LF_ERR_INVALID_ARGUMENT, "cache is NULL");
    if (!q_host || !k_new_host || !v_new_host || !out_host || !slot_host)
        return fail(LF_ERR_INVALID_ARGUMENT, "host buffers must be non-NULL");
    const lf_cache_config& g = c->cfg;
    cudaStream_t st = (cudaStream_t)stream;
    char* base = (char*)c->slab;
    size_t qb = (size_t)g.batch * g.num_q_heads * g.head_dim * 2;
    size_t kb = (size_t)g.batch * g.num_kv_heads * g.head_dim * 2;
    size_t ob = (size_t)g.batch * g.num_q_heads * g.head_dim * (g.out_dtype == LF_DTYPE_F32 ? 4 : 2);
    size_t sb = (size_t)g.batch * g.num_kv_heads * 4;
    // Caller buffers in pinned, device-mapped host memory (e.g. torch pin_memory): the kernel reads the
    // inputs and writes out/slot there directly over the host link, overlapped with its own K/V
    // streaming -- no copy at all, one stream sync.
    {
        auto mapped = [](const void* h) -> void* {
            cudaPointerAttributes a;
            if (cudaPointerGetAttributes(&a, h) != cudaSuccess) {
                cudaGetLastError();
                return nullptr;
            }
            return a.type == cudaMemoryTypeHost ? a.devicePointer : nullptr;
        };
        void* dq = mapped(q_host);
        void* dk = dq ? mapped(k_new_host) : nullptr;
        void* dv = dk ? mapped(v_new_host) : nullptr;
        void* dout = dv ? mapped(out_host) : nullptr;
        void* dslot = dout ? mapped(slot_host) : nullptr;
        if (dslot) {
            lf_status s = decode_impl(c, dq, dk, dv, dout, (int32_t*)dslot, nullptr, stream, 1, 0, g.batch);
            if (s) return s;
            int prev = 0;
            cudaGetDevice(&prev);
            cudaSetDevice(c->device);
            const cudaError_t e = cudaStreamSynchronize(st);
            cudaSetDevice(prev);
            if (e != cudaSuccess) return cuda_fail(e, "host step");
            return LF_OK;
        }
    }
    char* hs = c->host_stage;
    if (hs) {
        // small step, zero-copy: the inputs are packed into the mapped pinned staging buffer, the kernel
        // reads them and writes out + slot there directly over the host link, one stream sync
        memcpy(hs, q_host, qb);
        memcpy(hs + (c->L.sk_off - c->L.sq_off), k_new_host, kb);
        memcpy(hs + (c->L.sv_off - c->L.sq_off), v_new_host, kb);
        char* hd = c->host_stage_dev;
        const size_t in_b = stage_in_bytes(c->L, g);
        const size_t so = in_b, ss = in_b + (c->L.ss_off - c->L.so_off);
        lf_status s = decode_impl(c, hd, hd + (c->L.sk_off - c->L.sq_off), hd + (c->L.sv_off - c->L.sq_off),
                                  hd + so, (int32_t*)(hd + ss), nullptr, stream, 1, 0, g.batch);
        if (s) return s;
        int prev = 0;
        cudaGetDevice(&prev);
        cudaSetDevice(c->device);
        const cudaError_t e = cudaStreamSynchronize(st);
        cudaSetDevice(prev);
        if (e != cudaSuccess) return cuda_fail(e, "host step");
        memcpy(out_host, hs + so, ob);
        memcpy(slot_host, hs + ss, sb);
        return LF_OK;
    }
    // larger steps: three H2D copies from the caller's (pinned) buffers, the kernel, two D2H copies, one
    // stream sync.  (Chunking the batch so the copies of one chunk overlap the kernel of another was
    // measured slower on r / q3 / f1: profiles/r02_ab_chunked_host_rejected.txt.)
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(c->device);
    cudaError_t e = cudaMemcpyAsync(base + c->L.sq_off, q_host, qb, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(base + c->L.sk_off, k_new_host, kb, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(base + c->L.sv_off, v_new_host, kb, cudaMemcpyHostToDevice, st);
    cudaSetDevice(prev);
    if (e != cudaSuccess) return cuda_fail(e, "h2d");
    lf_status s = lf_decode_step(c, base + c->L.sq_off, base + c->L.sk_off, base + c->L.sv_off,
                                 base + c->L.so_off, (int32_t*)(base + c->L.ss_off), nullptr, stream);
    if (s) return s;
    cudaSetDevice(c->device);
    e = cudaMemcpyAsync(out_host, base + c->L.so_off, ob, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(slot_host, base + c->L.ss_off, sb, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    cudaSetDevice(prev);
    if (e != cudaSuccess) return cuda_fail(e, "d2h");
    return LF_OK;
}

}  // extern "C"
