// Instruction-fetch probe (tuning aid): cycles for ~6k straight-line SASS instructions executed
// once per launch, launch after launch (is the instruction cache warm across kernel launches?),
// and the same code executed twice within one launch (second pass = warm).
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/probes/icache_probe tools/probes/icache_probe.cu
#include <cuda_runtime.h>
#include <cstdio>

__global__ void straight(float* out, long long* t, float a) {
    float x0 = a, x1 = a + 1, x2 = a + 2, x3 = a + 3, x4 = a + 4, x5 = a + 5, x6 = a + 6, x7 = a + 7;
    long long c[3];
    c[0] = clock64();
    for (int pass = 0; pass < 2; ++pass) {
#pragma unroll
        for (int i = 0; i < 768; ++i) {
            x0 = fmaf(x0, 1.0001f, (float)i); x1 = fmaf(x1, 0.9999f, (float)i); x2 = fmaf(x2, 1.0002f, x0);
            x3 = fmaf(x3, 0.9998f, x1); x4 = fmaf(x4, 1.0003f, x2); x5 = fmaf(x5, 0.9997f, x3);
            x6 = fmaf(x6, 1.0004f, x4); x7 = fmaf(x7, 0.9996f, x5);
        }
        c[pass + 1] = clock64() + (long long)(x7 * 0.f);
    }
    if (threadIdx.x == 0) {
        out[blockIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
        t[blockIdx.x * 2] = c[1] - c[0];
        t[blockIdx.x * 2 + 1] = c[2] - c[1];
    }
}

int main() {
    float* out;
    long long* t;
    cudaMalloc(&out, 4096);
    cudaMalloc(&t, 148 * 16);
    long long h[4];
    for (int rep = 0; rep < 5; ++rep) {
        straight<<<1, 32>>>(out, t, 1.0f + rep);
        cudaDeviceSynchronize();
        cudaMemcpy(h, t, 16, cudaMemcpyDeviceToHost);
        printf("launch %d: first pass %lld cycles, second pass %lld cycles\n", rep, h[0], h[1]);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
