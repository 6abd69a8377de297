// Microbenchmark: tcgen05.mma (kind::f16, K = 16) cost for small N. A from TMEM (".ts", the
// decode GEMV's form) or shared memory (".ss"); 1 or 2 issuing threads (separate warps, separate
// accumulators); M = 64 or 128; 1 or 2 CTAs per SM. Reports ns per MMA per SM (aggregate over
// the issuers of an SM) from issue start to the final commit landing.
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

template <uint32_t kCols>
__global__ void k_umma(int n_mma, int M, int N, int ts, int issuers, unsigned long long* out, int lanes_mode) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar[4];
  __shared__ uint32_t tbase;
  for (int i = threadIdx.x; i < 32 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar[0], 1);
    ptx::mbar_init(&bar[1], 1);
    ptx::mbar_init(&bar[2], 1);
    ptx::mbar_init(&bar[3], 1);
    ptx::fence_mbar_init();
  }
  if (threadIdx.x < 32) ptx::tmem_alloc<kCols>(&tbase);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tm = tbase;
  const uint32_t sa = ptx::smem_u32(smem), sb = sa + 16 * 1024;
  const uint32_t idesc = ptx::idesc_bf16_f32(M, N);
  // lanes_mode 0: issuer w = lane 0 of warp w; 1: issuer w = lane w of warp 0
  const int who = lanes_mode ? (threadIdx.x < 32 ? threadIdx.x : 99) : ((threadIdx.x & 31) == 0 ? threadIdx.x / 32 : 99);
  unsigned long long t0 = gt();
  if (who < issuers) {
    // A operand columns [0, 32); issuer w accumulates into columns [32 + w * (kCols - 32) / 2, ...)
    const uint32_t d = tm + 32 + (uint32_t)who * ((kCols - 32) / 4);
    for (int i = 0; i < n_mma; ++i) {
      if (ts)
        ptx::mma_bf16_ts(d, tm + (uint32_t)(8 * (i & 3)), ptx::smem_desc_sw128(sb + 32 * (i & 3)), idesc, i > 0);
      else
        ptx::mma_bf16_ss(d, ptx::smem_desc_sw128(sa + 32 * (i & 3)), ptx::smem_desc_sw128(sb + 32 * (i & 3)), idesc,
                         i > 0);
    }
    ptx::mma_commit(&bar[who]);
    ptx::mbar_wait(&bar[who], 0);
  }
  __syncthreads();
  unsigned long long t2 = gt();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = t2 - t0;
  ptx::tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) ptx::tmem_dealloc<kCols>(tm);
}

int main() {
  unsigned long long* d_out;
  cudaMalloc(&d_out, 16);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(k_umma<512>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  cudaFuncSetAttribute(k_umma<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  const int n = 2048;
  printf("form  M  N  issuers/CTA  lanes?  CTAs/SM  ns_per_MMA_per_SM  TFLOP/s(all SMs)\n");
  for (int ts = 1; ts >= 0; --ts)
    for (int N : {16, 32, 64})
      for (int iss : {1, 2, 4})
        for (int lm : {0, 1})
          for (int cps : {1, 2}) {
            if (iss == 1 && lm == 1) continue;
            const int M = 128;
            for (int rep = 0; rep < 2; ++rep) {
              if (cps == 1) k_umma<512><<<sms, 128, 64 * 1024>>>(n, M, N, ts, iss, d_out, lm);
              else k_umma<256><<<2 * sms, 128, 64 * 1024>>>(n, M, N, ts, iss, d_out, lm);
            }
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) {
              printf("error %s\n", cudaGetErrorString(e));
              return 1;
            }
            unsigned long long h;
            cudaMemcpy(&h, d_out, 8, cudaMemcpyDeviceToHost);
            const double per = (double)h / (n * iss * cps);
            const double tf = 2.0 * M * N * 16 / per * 1e-3 * sms;
            printf("%s %4d %4d  %d  %s  %d  %8.1f  %8.1f\n", ts ? "ts" : "ss", M, N, iss, lm ? "lanes" : "warps", cps, per, tf);
          }
  return 0;
}
