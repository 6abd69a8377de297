// Microbenchmark: HBM streaming bandwidth of TMA 2-D box loads into a multi-stage smem ring
// (consumer warp just releases stages), for different box shapes / stages / CTAs per SM.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <string>
#include "../../paper_2511_04805_b200/csrc/tc_ptx.cuh"
using namespace pz;

__global__ void k_stream(const __grid_constant__ CUtensorMap tm, int rows_total, int cols, int box_rows, int box_cols,
                         int stages, int stage_bytes, int n_tiles, int* sink) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~uintptr_t(1023));
  uint64_t* full = (uint64_t*)(smem + stages * stage_bytes);
  uint64_t* empty = full + stages;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) { ptx::mbar_init(&full[s], 1); ptx::mbar_init(&empty[s], 1); }
    ptx::fence_mbar_init();
  }
  __syncthreads();
  const int tiles_per_row = cols / box_cols;
  if (threadIdx.x == 0) {
    int st = 0; uint32_t ph = 0;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
      // tile t: row block (t / tiles_per_row), column block (t % tiles_per_row)  -> walk K first
      int rb = t / tiles_per_row, cb = t % tiles_per_row;
      ptx::mbar_wait(&empty[st], ph ^ 1);
      ptx::mbar_arrive_expect_tx(&full[st], box_rows * box_cols * 2);
      ptx::tma_load_2d(smem + st * stage_bytes, &tm, &full[st], cb * box_cols, rb * box_rows);
      if (++st == stages) { st = 0; ph ^= 1; }
    }
  } else if (threadIdx.x == 32) {
    int st = 0; uint32_t ph = 0; int acc = 0;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
      ptx::mbar_wait(&full[st], ph);
      acc += smem[st * stage_bytes + (t & 63)];
      ptx::mbar_arrive(&empty[st]);
      if (++st == stages) { st = 0; ph ^= 1; }
    }
    if (acc == 12345) *sink = acc;
  }
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main(int argc, char** argv) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  void* fnp; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
  EncFn enc = (EncFn)fnp;
  // Mixtral w13 packed [4 x 2 x 14336, 4096] (940 MB) or, with argv[1] = "w2", w2 [4 x 4096, 14336]
  const bool w2 = argc > 1 && std::string(argv[1]) == "w2";
  const long rows = w2 ? 4 * 4096 : 4 * 2 * 14336, cols = w2 ? 14336 : 4096;
  uint16_t* buf; cudaMalloc(&buf, rows * cols * 2); cudaMemset(buf, 1, rows * cols * 2);
  int* sink; cudaMalloc(&sink, 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  struct Cfg { int box_rows, box_cols, swz, stages, ctas_per_sm; };
  std::vector<Cfg> cfgs = {{64, 64, 1, 4, 2}, {128, 64, 1, 4, 2}, {128, 64, 1, 6, 1}, {64, 64, 1, 8, 2},
                           {32, 256, 0, 4, 2}, {16, 256, 0, 8, 2}, {64, 256, 0, 4, 2}, {128, 64, 1, 3, 2},
                           {256, 64, 1, 3, 1}, {64, 64, 1, 2, 4}};
  for (auto c : cfgs) {
    CUtensorMap tm;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
    cuuint32_t box[2] = {(cuuint32_t)c.box_cols, (cuuint32_t)c.box_rows};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     c.swz ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r) { printf("encode failed %d\n", r); continue; }
    int stage_bytes = c.box_rows * c.box_cols * 2;
    size_t smem = 1024 + c.stages * stage_bytes + 256;
    cudaFuncSetAttribute(k_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int n_tiles = (rows / c.box_rows) * (cols / c.box_cols);
    int grid = sms * c.ctas_per_sm;
    k_stream<<<grid, 64, smem>>>(tm, rows, cols, c.box_rows, c.box_cols, c.stages, stage_bytes, n_tiles, sink);
    cudaEventRecord(e0);
    for (int i = 0; i < 5; ++i)
      k_stream<<<grid, 64, smem>>>(tm, rows, cols, c.box_rows, c.box_cols, c.stages, stage_bytes, n_tiles, sink);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("box %3dx%3d swz%d stages %d ctas/SM %d (in flight/SM %3d KB): %.0f GB/s  err=%s\n", c.box_rows, c.box_cols, c.swz,
           c.stages, c.ctas_per_sm, c.stages * stage_bytes * c.ctas_per_sm / 1024, 5.0 * rows * cols * 2 / (ms / 1e3) / 1e9,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
