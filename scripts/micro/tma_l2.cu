// Microbenchmark: L2 -> SM bandwidth of TMA 2-D box loads (the prefill kernels' operand
// traffic is L2-resident): a 24 MB buffer (inside the 126 MB L2) re-read by every CTA in
// 16 KB boxes (128 rows x 64 bf16, 128-byte swizzle) through a ring of `stages` slots per CTA;
// a consumer lane releases each slot as soon as it lands. Reports aggregate GB/s and the
// implied per-slot latency (in flight / per-SM rate).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include "../../paper_2511_04805_b200/csrc/tc_ptx.cuh"
using namespace pz;

__global__ void k_l2(const __grid_constant__ CUtensorMap tm, int n_row_blocks, int n_col_blocks, int stages,
                     int iters, int* sink, int box_rows, int nprod, int shared_mode) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem0 = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~uintptr_t(1023));
  const int kStage = box_rows * 128;
  const int pr = threadIdx.x >> 6;  // producer pair index: warps 2pr (producer), 2pr+1 (consumer)
  if (pr >= nprod) return;
  uint8_t* smem = smem0 + (size_t)pr * stages * kStage;
  uint64_t* full = (uint64_t*)(smem0 + (size_t)nprod * stages * kStage) + pr * 2 * stages;
  uint64_t* empty = full + stages;
  if ((threadIdx.x & 63) == 0) {
    for (int s = 0; s < stages; ++s) { ptx::mbar_init(&full[s], 1); ptx::mbar_init(&empty[s], 1); }
    ptx::fence_mbar_init();
  }
  __syncthreads();
  const int n_tiles = n_row_blocks * n_col_blocks;
  if ((threadIdx.x & 63) == 0) {
    int st = 0; uint32_t ph = 0;
    for (int i = 0; i < iters; ++i) {
      // shared_mode 0: every CTA its own tile sequence; k > 0: groups of k CTAs read the same
      // tiles at the same time (the prefill pattern: one token tile, many weight row blocks)
      const int t = shared_mode ? ((blockIdx.x / shared_mode) * 977 + pr * 131 + i) % n_tiles
                                : (blockIdx.x * 7 + pr * 131 + i) % n_tiles;
      ptx::mbar_wait(&empty[st], ph ^ 1);
      ptx::mbar_arrive_expect_tx(&full[st], kStage);
      ptx::tma_load_2d(smem + st * kStage, &tm, &full[st], (t % n_col_blocks) * 64, (t / n_col_blocks) * box_rows);
      if (++st == stages) { st = 0; ph ^= 1; }
    }
  } else if ((threadIdx.x & 63) == 32) {
    int st = 0; uint32_t ph = 0; int acc = 0;
    for (int i = 0; i < iters; ++i) {
      ptx::mbar_wait(&full[st], ph);
      acc += smem[st * kStage + (i & 63)];
      ptx::mbar_arrive(&empty[st]);
      if (++st == stages) { st = 0; ph ^= 1; }
    }
    if (acc == 12345) *sink = acc;
  }
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  void* fnp; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
  EncFn enc = (EncFn)fnp;
  const long rows = 3072, cols = 4096;  // 24 MB
  uint16_t* buf; cudaMalloc(&buf, rows * cols * 2); cudaMemset(buf, 1, rows * cols * 2);
  int* sink; cudaMalloc(&sink, 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 2048;
  const int box_rows = 128;
  CUtensorMap tm;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE)) {
    printf("encode failed\n");
    return 1;
  }
  const int kStage = box_rows * 128;
  for (int shared_mode : {0, 2, 8, 22, 148}) {
    for (int nprod : {1, 3}) {
      for (int stages : {3, 4}) {
        size_t smem = 1024 + (size_t)nprod * stages * kStage + 1024;
        if (smem > 227 * 1024) continue;
        cudaFuncSetAttribute(k_l2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        const int grid = sms;
        k_l2<<<grid, 64 * nprod, smem>>>(tm, rows / box_rows, cols / 64, stages, iters, sink, box_rows, nprod, shared_mode);
        cudaEventRecord(e0);
        for (int i = 0; i < 3; ++i)
          k_l2<<<grid, 64 * nprod, smem>>>(tm, rows / box_rows, cols / 64, stages, iters, sink, box_rows, nprod, shared_mode);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        const double bytes = 3.0 * grid * nprod * iters * (double)kStage;
        const double gbs = bytes / (ms / 1e3) / 1e9;
        const double per_sm = gbs / sms;
        printf("same-tile group %3d producers %d stages %d in flight/SM %3d KB: %6.0f GB/s (%5.1f KB/us per SM, latency %.2f us) err=%s\n",
               shared_mode, nprod, stages, nprod * stages * kStage / 1024, gbs, per_sm,
               nprod * stages * kStage / 1024.0 / per_sm, cudaGetErrorString(cudaGetLastError()));
      }
    }
  }
  return 0;
}
