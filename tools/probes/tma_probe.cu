// TMA streaming microbenchmark (tuning aid, not product code): every CTA streams its own contiguous
// row range of a [rows][128] bf16 tensor through an ST-stage SMEM ring with SW128 2D TMA boxes
// {64 cols, BR rows}; a consumer thread releases each stage as soon as it lands (no compute).
// Reports GB/s per CTA and in total for CTA counts x stage counts x box rows.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2603_11504_b200/csrc \
//        -o tools/probes/tma_probe tools/probes/tma_probe.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "lf_tc_ptx.cuh"

using namespace lf;

__device__ __forceinline__ void tma_load_3d(uint32_t dst, const void* tmap, uint32_t bar, int c0, int c1, int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(dst),
        "l"(tmap), "r"(bar), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}

__device__ __forceinline__ void bulk_load_1d(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}

// kMode 0: 2D tensor map, two 64-column boxes per stage; 1: 3D map, one box per stage;
//       2: 1D bulk copy of the stage's contiguous bytes (no swizzle)
template <int kMode>
__global__ void __launch_bounds__(64, 1) stream_kernel(const __grid_constant__ CUtensorMap tm, int rows_per_cta,
                                                        int box_rows, int stages, int passes, const unsigned char* gbase,
                                                        int delay) {
    extern __shared__ unsigned char smem_raw[];
    unsigned char* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
    const uint32_t stage_bytes = (uint32_t)box_rows * 256;   // two 64-col boxes of box_rows x 128 B
    const uint32_t ring = ptx::smem_u32(smem);
    const uint32_t bars = ring + stages * stage_bytes;
    auto FULL = [&](int i) { return bars + 8u * i; };
    auto EMPTY = [&](int i) { return bars + 8u * (stages + i); };
    if (threadIdx.x == 0) {
        for (int i = 0; i < stages; ++i) {
            ptx::mbar_init(FULL(i), 1);
            ptx::mbar_init(EMPTY(i), 1);
        }
        ptx::fence_mbar_init();
        ptx::tma_prefetch_desc(&tm);
    }
    __syncthreads();
    const int tiles = rows_per_cta / box_rows;
    const int row0 = blockIdx.x * rows_per_cta;
    const int total = tiles * passes;
    if (threadIdx.x == 0) {
        for (int it = 0; it < total; ++it) {
            const int st = it % stages;
            ptx::mbar_wait(EMPTY(st), ((it / stages) & 1u) ^ 1u);
            ptx::mbar_arrive_expect_tx(FULL(st), stage_bytes);
            const int row = row0 + (it % tiles) * box_rows;
            const uint32_t dst = ring + st * stage_bytes;
            if (kMode == 2) {
                bulk_load_1d(dst, gbase + (size_t)row * 256, stage_bytes, FULL(st));
            } else if (kMode == 1) {
                tma_load_3d(dst, &tm, FULL(st), 0, row, 0);   // both 64-column halves, one instruction
            } else {
                ptx::tma_load_2d(dst, &tm, FULL(st), 0, row);
                ptx::tma_load_2d(dst + stage_bytes / 2, &tm, FULL(st), 64, row);
            }
        }
    } else if (threadIdx.x == 32) {
        for (int it = 0; it < total; ++it) {
            const int st = it % stages;
            ptx::mbar_wait(FULL(st), (it / stages) & 1u);
            if (delay) {
                const long long t0 = clock64();
                while (clock64() - t0 < delay) {
                }
            }
            ptx::mbar_arrive(EMPTY(st));
        }
    }
    __syncthreads();
}

int main(int argc, char** argv) {
    const int rows_per_cta = argc > 1 ? atoi(argv[1]) : 8192;   // 2 MB per CTA
    const int max_ctas = 148;
    const size_t rows = (size_t)rows_per_cta * max_ctas;
    void* buf;
    cudaMalloc(&buf, rows * 256);
    cudaMemset(buf, 1, rows * 256);
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
    auto enc = (PFN_cuTensorMapEncodeTiled_v12000)f;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaFuncSetAttribute(stream_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(stream_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(stream_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    const int only_ctas = argc > 2 ? atoi(argv[2]) : 0;
    for (int mode = 0; mode < 3; ++mode)
    for (int box_rows : {64, 128, 256}) {
        CUtensorMap tm;
        CUresult r = CUDA_SUCCESS;
        if (mode == 0) {
            cuuint64_t dims[2] = {128, (cuuint64_t)rows};
            cuuint64_t strides[1] = {256};
            cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
            cuuint32_t estr[2] = {1, 1};
            r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        } else if (mode == 1) {   // {64 cols, rows, 2 halves}: SMEM [half][row][64] = the 2-box layout in one box
            cuuint64_t dims[3] = {64, (cuuint64_t)rows, 2};
            cuuint64_t strides[2] = {256, 128};
            cuuint32_t box[3] = {64, (cuuint32_t)box_rows, 2};
            cuuint32_t estr[3] = {1, 1, 1};
            r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, buf, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        }
        if (r != CUDA_SUCCESS) {
            printf("encode failed (mode=%d box_rows=%d): %d\n", mode, box_rows, (int)r);
            continue;
        }
        for (int ctas : {1, 16, 148}) {
            if (only_ctas && ctas != only_ctas) continue;
            for (int stages : {2, 4}) {
              for (int delay : {0, 1000}) {
                const size_t smem = (size_t)stages * box_rows * 256 + 16 * stages * 2 + 1024;
                if (smem > 227 * 1024) continue;
                const int passes = 2;
                auto kern = mode == 0 ? stream_kernel<0> : mode == 1 ? stream_kernel<1> : stream_kernel<2>;
                kern<<<ctas, 64, smem>>>(tm, rows_per_cta, box_rows, stages, 1, (const unsigned char*)buf, 0);
                cudaEventRecord(e0);
                kern<<<ctas, 64, smem>>>(tm, rows_per_cta, box_rows, stages, passes, (const unsigned char*)buf, delay);
                cudaEventRecord(e1);
                cudaError_t err = cudaEventSynchronize(e1);
                if (err != cudaSuccess) {
                    printf("error %s\n", cudaGetErrorString(err));
                    return 1;
                }
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                const double bytes = (double)rows_per_cta * 256 * passes;
                printf("%s stage %3d KB stages %2d delay %4d ctas %3d: %7.1f GB/s per CTA  %7.0f GB/s total (%.3f us/stage)\n",
                       mode == 0 ? "2d" : mode == 1 ? "3d" : "1d", box_rows * 256 / 1024, stages, delay, ctas,
                       bytes / (ms * 1e-3) / 1e9, bytes * ctas / (ms * 1e-3) / 1e9,
                       ms * 1e3 / ((double)rows_per_cta / box_rows * passes));
              }
            }
        }
    }
    return 0;
}
