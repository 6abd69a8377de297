// Microbenchmark: sustained tcgen05.mma throughput of the prefill TS shape (A = 128 x 16 bf16
// from TMEM, B = N tokens x 16 from shared memory, D fp32 in TMEM): 1 CTA per SM, `iss` issuer
// warps each accumulating into its own N-column range, 4 MMAs (one 64-wide K stage) between
// commits, `commits` tcgen05.commit per stage per issuer (the kernel commits 2-3 per stage).
// Also the SS form (A and B from shared memory) at M = 128, N = 256 for reference.
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

__global__ void k_rate(int stages, int N, int ts, int iss, int commits, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar[4][4];
  __shared__ uint32_t tbase;
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i)
      for (int j = 0; j < 4; ++j) ptx::mbar_init(&bar[i][j], 1);
    ptx::fence_mbar_init();
  }
  if (threadIdx.x < 32) ptx::tmem_alloc<512>(&tbase);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tm = tbase;
  const uint32_t sa = ptx::smem_u32(smem), sb = sa + 32 * 1024;
  const int w = threadIdx.x >> 5;
  unsigned long long t0 = gt();
  if (w < iss) {
    const uint32_t idesc = ptx::idesc_bf16_f32(128, N);
    const uint32_t d = ts ? tm + 128 + (uint32_t)w * 192 : tm + (uint32_t)w * 256;
    for (int s = 0; s < stages; ++s) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (ts == 2) {
          if (k == 0) ptx::mma_bf16_ts_stage4_elect(d, tm + 32u * (s & 3), ptx::smem_desc_sw128(sb), idesc, s != 0);
        } else if (ts)
          ptx::mma_bf16_ts_elect(d, tm + 32u * (s & 3) + 8u * k, ptx::smem_desc_sw128(sb + 32 * k), idesc, (s | k) != 0);
        else {
          if ((threadIdx.x & 31) == 0)
            ptx::mma_bf16_ss(d, ptx::smem_desc_sw128(sa + (uint32_t)w * 16384 + 32 * k), ptx::smem_desc_sw128(sb + 32 * k),
                             idesc, (s | k) != 0);
        }
      }
      for (int c = 0; c < commits; ++c) ptx::mma_commit_elect(&bar[w][c]);
    }
    ptx::mma_commit_elect(&bar[w][3]);
    ptx::mbar_wait(&bar[w][3], 0);
  }
  __syncthreads();
  unsigned long long t2 = gt();
  if (threadIdx.x == 0) out[blockIdx.x] = t2 - t0;
  ptx::tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) ptx::tmem_dealloc<512>(tm);
}

int main() {
  unsigned long long* d_out;
  cudaMalloc(&d_out, 8 * 1024);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(k_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  const int stages = 512;
  printf("form N_per_issuer issuers commits/stage  ns_per_stage  TFLOP/s(148 SMs)  frac_of_1658\n");
  for (int ts = 2; ts >= 0; --ts)
    for (int N : {64, 96, 128, 144, 176, 192, 256})
      for (int iss : {1, 2})
        for (int commits : {0, 2}) {
          if (ts && N > 192) continue;
          if (!ts && N != 256) continue;
          k_rate<<<sms, 128, 100 * 1024>>>(stages, N, ts, iss, commits, d_out);
          k_rate<<<sms, 128, 100 * 1024>>>(stages, N, ts, iss, commits, d_out);
          cudaError_t e = cudaDeviceSynchronize();
          if (e != cudaSuccess) {
            printf("error %s\n", cudaGetErrorString(e));
            return 1;
          }
          unsigned long long h[1024];
          cudaMemcpy(h, d_out, 8 * sms, cudaMemcpyDeviceToHost);
          unsigned long long mx = 0;
          for (int i = 0; i < sms; ++i) mx = h[i] > mx ? h[i] : mx;
          const double per_stage = (double)mx / stages;
          const double flops = 2.0 * 128 * N * 64 * iss;  // per stage per SM
          const double tf = flops / per_stage * 1e-3 * sms;
          printf("%s %4d %d %d %8.1f %8.1f %.3f\n", ts == 2 ? "ts4" : ts ? "ts" : "ss", N, iss, commits, per_stage, tf, tf / 1658.6);
        }
  return 0;
}
