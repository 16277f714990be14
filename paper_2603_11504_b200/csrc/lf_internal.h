// Internal declarations shared by the host runtime and the decode kernels (not part of the ABI).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/longflow.h"

namespace lf {

// Everything one decode-step launch needs (passed by value as a kernel parameter).
struct StepParams {
    const uint16_t* q;      // bf16 [B][Hq][d]
    const uint16_t* k_new;  // bf16 [B][Hkv][d]
    const uint16_t* v_new;  // bf16 [B][Hkv][d]
    uint16_t* K;            // bf16 [B][Hkv][N][d]   (cache, updated in place)
    uint16_t* V;            // bf16 [B][Hkv][N][d]
    int32_t* n_valid;       // int32 [B][Hkv]
    void* out;              // bf16 or fp32 [B][Hq][d]
    int32_t* slot;          // int32 [B][Hkv]
    float* scores;          // fp32 [B][Hkv][N] or nullptr
    unsigned long long* trace;  // debug event trace (LF_TRACE builds only), or nullptr
    int32_t deferred;       // 1: Fig. 2-literal deferred mode (k*, v* already written; no current-token term)
    int32_t exclude_newest; // deferred mode: the slot just written is not a candidate
    int32_t* pend;          // deferred mode: int32 [B][Hkv] slot covered at the next step
    const int32_t* written; // deferred mode: int32 [B][Hkv] slot the current token was written to
    int32_t B, Hq, Hkv, G, d, N;
    int32_t out_f32;        // 1: fp32 out, 0: bf16 out
    float scale_log2;       // softmax_scale * log2(e): logits live in log2 units on chip
    int32_t splits;         // CTAs per unit (= cluster size)
    int32_t chunk;          // tokens per CTA (multiple of 128)
    int32_t solo_units;     // tcgen05 kernel: units [0, solo_units) are computed whole by one CTA each
                            // (round-robin over the grid's CTAs); the rest split across their cluster
    int32_t hold;           // tcgen05 kernel: tokens one CTA holds for a unit (TMEM regions, lambda buffer)
    int32_t unit_base;      // tcgen05 kernel: cache unit of this launch's unit 0 (TMA rows); the unit-indexed
                            // pointers (K, V, n_valid, pend, slot, scores, q, out, ...) are already offset
    int32_t host_io;        // 1: q, k_new, v_new, out, slot live in mapped pinned HOST memory (the host entry
                            // point's zero-copy path): read/written by the kernels directly, never prefetched
};

// launch attributes shared by the decode kernels: cluster dims + programmatic dependent launch
// (the kernels call griddepcontrol.wait before their first dependent global access); LF_NO_PDL=1
// disables the latter
int fill_launch_attrs(cudaLaunchAttribute* attr, int cluster_x);

// Plan overrides (lf_cache_config ctas_per_sm / solo / latency_variant; 0 = automatic)
struct PlanForce {
    int32_t ctas_per_sm;
    int32_t solo;
    int32_t lat;
    int32_t no_solo;   // plan_shards > 1: every unit split the same way in every shard (no solo rounds)
};

struct Plan {
    int32_t kernel;   // lf_kernel (resolved: SIMT or TCGEN05)
    int32_t splits;
    int32_t chunk;
    int32_t smem;     // dynamic shared memory bytes per CTA
    int32_t clusters; // persistent clusters in the grid (tcgen05 kernel), 0 = one cluster per unit
    int32_t stages;   // TMA ring depth (tcgen05 kernel)
    int32_t tmem_cols;  // TMEM columns per CTA (tcgen05 kernel)
    int32_t solo_rounds;  // tcgen05: rounds of whole units per CTA before the split tail
    int32_t lat;          // tcgen05: 1 = latency variant (split plan, grid leaves SMs free), 0 = streaming
};

// deferred mode pre-pass: the current token covers pend[u] (or is appended) before attention
cudaError_t deferred_write_launch(const StepParams& p, cudaStream_t stream);

// SnapKV prefill compression (lf_snapkv.cu, NEXT-f3)
constexpr int kSnapRowsMax = 128;
size_t snapkv_workspace_bytes(int Hkv, int G, int n, int w, int N);
cudaError_t snapkv_launch(uint16_t* K, uint16_t* V, int32_t* n_valid, int seq, int Hkv, int G, int d, int N,
                          const void* k, const void* v, const void* q_obs, int n, int w, int ks, float scale,
                          int32_t* kept, void* workspace, cudaStream_t stream);

// approximation diagnostics (lf_diag.cu, NEXT-f4)
size_t diag_workspace_bytes(int units, int G, int N);
cudaError_t diag_launch(const StepParams& p, const int32_t* n_valid, void* workspace, int32_t* islot, float* fstat,
                        cudaStream_t stream);

// CUDA-core split-KV kernel (lf_decode_simt.cu)
bool simt_supported(int G, int d);
Plan simt_plan(int units, int G, int d, int N, int split_tokens, int num_sms);
cudaError_t simt_launch(const StepParams& p, const Plan& plan, cudaStream_t stream);

// TMA + tcgen05 split-KV kernel (lf_decode_tc.cu)
struct TcMaps {               // two CUtensorMap (K, V) encoded once per cache (the slab is static)
    alignas(64) unsigned char k[128];
    alignas(64) unsigned char v[128];
};
bool tc_supported(int G, int d);
Plan tc_plan(int units, int G, int d, int N, int split_tokens, int num_sms, const PlanForce& force);
int tc_hold(const Plan& plan, int N);
bool tc_make_maps(TcMaps* maps, void* K, void* V, long long units, int N, int d);
cudaError_t tc_launch(const StepParams& p, const Plan& plan, const TcMaps& maps, cudaStream_t stream);

}  // namespace lf
