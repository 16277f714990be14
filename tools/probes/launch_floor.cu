// Launch-floor probe (tuning aid for the latency-bound q7 shape): the per-launch period of a kernel
// with the q7 decode plan's launch configuration -- 64 CTAs in clusters of 16, 192 threads, 100 KB
// dynamic SMEM, programmatic dependent launch, a prologue of mbarrier inits + TMEM alloc + cluster sync
// before griddepcontrol.wait -- doing no work, in a CUDA graph of 252 back-to-back launches (as bench.py
// times q7).  Variants: 0 = no prologue, no PDL; 1 = prologue + PDL (the decode kernel's shape);
// 2 = variant 1 plus one dependent L2 round trip and a global store after the wait.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/launch_floor tools/probes/launch_floor.cu
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <cstdio>

namespace cg = cooperative_groups;

__global__ void floor_kernel(int variant, int* buf) {
    extern __shared__ __align__(1024) unsigned char smem[];
    __shared__ uint32_t tmem_slot;
    const int tid = threadIdx.x;
    if (variant >= 1) {
        if (tid == 0) {
            for (int i = 0; i < 42; ++i) {
                const uint32_t bar = (uint32_t)__cvta_generic_to_shared(smem + 8 * i);
                asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(1) : "memory");
            }
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        if (tid / 32 == 1) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                             (uint32_t)__cvta_generic_to_shared(&tmem_slot)),
                         "r"(256)
                         : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
        }
        asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
        asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
        asm volatile("griddepcontrol.wait;" ::: "memory");
        if (variant == 2 && tid == 0) {
            const int v = __ldcg(buf + blockIdx.x);
            buf[1024 + blockIdx.x] = v + 1;
        }
        __syncthreads();
        if (tid / 32 == 1) {
            const uint32_t t = tmem_slot;
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(t), "r"(256) : "memory");
        }
    }
}

int main() {
    int* buf;
    cudaMalloc(&buf, 8192 * 4);
    cudaMemset(buf, 0, 8192 * 4);
    cudaFuncSetAttribute(floor_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    cudaFuncSetAttribute(floor_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaStream_t st;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    for (int variant = 0; variant < 3; ++variant) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(64);
        cfg.blockDim = dim3(192);
        cfg.dynamicSmemBytes = 100 * 1024;
        cfg.stream = st;
        cudaLaunchAttribute attr[2];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 16;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[1].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = variant == 0 ? 1 : 2;
        cudaGraph_t g;
        cudaGraphExec_t ge;
        cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
        for (int i = 0; i < 252; ++i) cudaLaunchKernelEx(&cfg, floor_kernel, variant, buf);
        cudaStreamEndCapture(st, &g);
        cudaGraphInstantiate(&ge, g, 0);
        cudaGraphLaunch(ge, st);
        cudaStreamSynchronize(st);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        float best = 1e30f;
        for (int rep = 0; rep < 5; ++rep) {
            cudaEventRecord(e0, st);
            cudaGraphLaunch(ge, st);
            cudaEventRecord(e1, st);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (ms < best) best = ms;
        }
        printf("variant %d: %.2f us per launch (%s)\n", variant, best * 1e3f / 252,
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
