// Microbenchmark: the decode kernel's TMEM pipeline without HBM traffic. 8 "decoder" warps
// write a 128-row x 64-k bf16 A stage per position into a 3-deep TMEM ring (tcgen05.st,
// optional), MMA warp(s) issue M=128 x N x K=16 tcgen05.mma with A from TMEM and B from smem
// (4 per position per stage) and commit to release the A buffer. Reports ns per stage per CTA.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "../../paper_2511_04805_b200/csrc/tc_ptx.cuh"
using namespace pz;

__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ void named_bar_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// cfg bits: 1 = decoders store A with tcgen05.st, 2 = two MMA warps (one per position),
//           4 = extra commit per stage (second barrier), 8 = decoders skip waiting for A free
__global__ void __launch_bounds__(352, 1) k_pipe(int stages, int N, int cfg, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t a_full[3], a_empty[3], x_empty[3];
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  const bool st_on = cfg & 1, two = cfg & 2, extra = cfg & 4;
  for (int i = threadIdx.x; i < 16 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) {
    for (int j = 0; j < 3; ++j) {
      ptx::mbar_init(&a_full[j], 8);
      ptx::mbar_init(&a_empty[j], two ? 2 : 1);
      ptx::mbar_init(&x_empty[j], two ? 2 : 1);
    }
    ptx::fence_mbar_init();
  }
  if (warp == 0) ptx::tmem_alloc<256>(&tbase);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tm = tbase;
  const unsigned long long t0 = gt();
  if (warp >= 2 && warp < 10) {
    const int q = warp & 3, kh = (warp - 2) >> 2;
    const uint32_t lt = tm + ((uint32_t)(32 * q) << 16);
    uint32_t d[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) d[i] = 0x3c003c00u + i;
    int j = 0;
    uint32_t ph = 0;
    for (int s = 0; s < stages; ++s) {
      if (!(cfg & 8)) ptx::mbar_wait(&a_empty[j], ph ^ 1);
      ptx::tc_fence_after();
      if (st_on) {
        ptx::tmem_st_32x32b_x16(lt + 64u * j + 16u * kh, d);
        ptx::tmem_st_32x32b_x16(lt + 64u * j + 32u + 16u * kh, d);
        ptx::tmem_st_wait();
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&a_full[j]);
      if (++j == 3) { j = 0; ph ^= 1; }
    }
  } else if (warp == 1 || (two && warp == 10)) {
    const int mypos = warp == 1 ? 0 : 1;
    const uint32_t idesc = ptx::idesc_bf16_f32(128, N);
    const uint32_t xs = ptx::smem_u32(smem);
    int j = 0;
    uint32_t ph = 0;
    for (int s = 0; s < stages; ++s) {
      ptx::mbar_wait(&a_full[j], ph);
      ptx::tc_fence_after();
      for (int p = 0; p < 2; ++p) {
        if (two && p != mypos) continue;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          ptx::mma_bf16_ts_elect(tm + 192 + 32 * p, tm + 64u * j + 32u * p + 8 * kk,
                                 ptx::smem_desc_sw128(xs + 4096 * p + 32 * kk), idesc, (s | kk) != 0);
      }
      ptx::mma_commit_elect(&a_empty[j]);
      if (extra) ptx::mma_commit_elect(&x_empty[j]);
      if (++j == 3) { j = 0; ph ^= 1; }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  const unsigned long long t1 = gt();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = t1 - t0;
  if (warp == 0) ptx::tmem_dealloc<256>(tm);
}

int main() {
  unsigned long long* d_out;
  cudaMalloc(&d_out, 16);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(k_pipe, cudaFuncAttributeMaxDynamicSharedMemorySize, 20 * 1024);
  setvbuf(stdout, nullptr, _IONBF, 0);
  const int stages = 2000;
  printf("N  st  mma_warps  extra_commit  nowait  CTAs/SM  ns_per_stage_per_CTA\n");
  for (int N : {16, 32})
    for (int cfg : {0, 1, 2, 3, 5, 7})
      for (int cps : {1, 2}) {
        k_pipe<<<cps * sms, 352, 20 * 1024>>>(stages, N, cfg, d_out);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        k_pipe<<<cps * sms, 352, 20 * 1024>>>(stages, N, cfg, d_out);
        cudaEventRecord(e1);
        cudaError_t e = cudaGetLastError();
        if (e == cudaSuccess) e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
          printf("error %s\n", cudaGetErrorString(e));
          return 1;
        }
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("%d  %d  %d  %d  %d  %d  %8.1f\n", N, cfg & 1, cfg & 2 ? 2 : 1, (cfg >> 2) & 1, (cfg >> 3) & 1, cps,
               ms * 1e6 / stages);
      }
  return 0;
}
