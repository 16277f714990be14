// Kernel-parameter (constant bank) latency probe (tuning aid): cycles for a chain of 8 DEPENDENT reads
// of a __grid_constant__ parameter array (each index comes from the previous read, so every read is an
// LDC with a register index), measured right after griddepcontrol.wait and again (warm) after it.
// Variants: (0) plain launch, no pre-read; (1) the same chain is read once BEFORE griddepcontrol.wait
// (does the warm-up survive the wait?); (2) launched with programmatic stream serialization behind a
// short kernel, pre-read before the wait (the decode kernel's situation under PDL).
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o param_probe tools/probes/param_probe.cu
#include <cuda_runtime.h>
#include <cstdio>

struct Args {
    int idx[64];   // 256 B: idx[i] = next index (a permutation cycle with a 64-B stride)
    long long* out;
};

__global__ void prev_kernel(int* sink) {
    if (threadIdx.x == 0 && blockIdx.x == 0) sink[0] += 1;
}

// clock read that the hardware can only issue once `dep` has arrived (predicated on a compare of it)
__device__ __forceinline__ long long clock_after(int dep) {
    long long t;
    asm volatile("{\n\t.reg .pred p;\n\tsetp.lt.s32 p, %1, -1000;\n\t@p mov.u64 %0, 0;\n\t@!p mov.u64 %0, %%clock64;\n\t}"
                 : "=l"(t) : "r"(dep) : "memory");
    return t;
}
__device__ __forceinline__ int chase(const Args& a, int i, long long* t) {
    const long long t0 = clock_after(i);
#pragma unroll 1
    for (int k = 0; k < 8; ++k) i = a.idx[i];
    *t = clock_after(i) - t0;
    return i;
}

__global__ void probe(const __grid_constant__ Args a, int pre) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    long long t_pre = 0, t_cold = 0, t_warm = 0;
    int i = 0;
    if (pre) i = chase(a, i, &t_pre);
    asm volatile("griddepcontrol.wait;" ::: "memory");
    i = chase(a, i, &t_cold);
    i = chase(a, i, &t_warm);
    a.out[0] = t_pre;
    a.out[1] = t_cold;
    a.out[2] = t_warm;
    a.out[3] = i;
}

int main() {
    Args a;
    for (int k = 0; k < 64; ++k) a.idx[k] = (k + 16) % 64;   // 16 ints = 64 B stride
    long long* out;
    int* sink;
    cudaMalloc(&out, 64);
    cudaMalloc(&sink, 4);
    a.out = out;
    cudaStream_t s;
    cudaStreamCreate(&s);
    for (int variant = 0; variant < 3; ++variant) {
        for (int rep = 0; rep < 4; ++rep) {
            a.idx[63] = rep;   // a fresh parameter block every launch
            a.idx[63] = 15;
            if (variant == 2) {
                prev_kernel<<<1, 32, 0, s>>>(sink);
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = dim3(1);
                cfg.blockDim = dim3(32);
                cfg.stream = s;
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
                at[0].val.programmaticStreamSerializationAllowed = 1;
                cfg.attrs = at;
                cfg.numAttrs = 1;
                cudaLaunchKernelEx(&cfg, probe, a, 1);
            } else {
                probe<<<1, 32, 0, s>>>(a, variant);
            }
            long long h[4];
            cudaMemcpyAsync(h, out, 32, cudaMemcpyDeviceToHost, s);
            cudaStreamSynchronize(s);
            printf("variant %d rep %d: 8 dependent param reads: pre-wait %lld, first after wait %lld, again %lld cycles\n",
                   variant, rep, h[0], h[1], h[2]);
        }
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
