// Global-load latency probe (tuning aid): how long does ONE dependent L2-resident load take at the
// start of a kernel, right after griddepcontrol.wait, and in steady state?  One thread chases a
// pointer chain of 12 loads (ld.global.cg) and records the cycles of each.
// Variants: (0) plain launch, data L2-resident; (1) launched with programmatic stream serialization
// behind a short "previous" kernel, loads after griddepcontrol.wait; (2) as (1) but 64 CTAs (one
// timed), mirroring the q7 grid.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/probes/lat_probe tools/probes/lat_probe.cu
#include <cuda_runtime.h>
#include <cstdio>

__global__ void prev_kernel(int* sink) {
    if (threadIdx.x == 0 && blockIdx.x == 0) sink[0] += 1;
}

__global__ void chase(const int* __restrict__ chain, long long* out, int pdl) {
    if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
    if (blockIdx.x != 0 || threadIdx.x != 0) return;
    int idx = 0;
    long long t = clock64();
    for (int i = 0; i < 12; ++i) {
        idx = __ldcg(chain + idx);
        const long long t1 = clock64() + (idx & 0);   // dependent on the load
        out[i] = t1 - t;
        t = t1;
    }
    out[12] = idx;
}

int main() {
    const int n = 1 << 20;   // 4 MB chain: one line per 4 KB stride
    int* h = new int[n];
    for (int i = 0; i < n; ++i) h[i] = (i + 1024 + 17) % n;
    int *d, *sink;
    long long* out;
    cudaMalloc(&d, n * 4);
    cudaMalloc(&sink, 4);
    cudaMalloc(&out, 16 * 8);
    cudaMemcpy(d, h, n * 4, cudaMemcpyHostToDevice);
    cudaStream_t st;
    cudaStreamCreate(&st);
    long long r[16];
    for (int variant = 0; variant < 3; ++variant) {
        for (int rep = 0; rep < 3; ++rep) {
            prev_kernel<<<1, 32, 0, st>>>(sink);
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(variant == 2 ? 64 : 1);
            cfg.blockDim = dim3(32);
            cfg.stream = st;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            attr[0].val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = attr;
            cfg.numAttrs = variant >= 1 ? 1 : 0;
            cudaLaunchKernelEx(&cfg, chase, (const int*)d, out, variant >= 1 ? 1 : 0);
            cudaStreamSynchronize(st);
            cudaMemcpy(r, out, 13 * 8, cudaMemcpyDeviceToHost);
            printf("variant %d rep %d cycles per dependent load:", variant, rep);
            for (int i = 0; i < 12; ++i) printf(" %lld", r[i]);
            printf("\n");
        }
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
