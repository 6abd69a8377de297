// Does griddepcontrol.wait (cudaGridDependencySynchronize) in a PDL-launched kernel wait for the
// primary grid to COMPLETE, or only for every primary CTA to have executed
// griddepcontrol.launch_dependents? The primary triggers first, then spins ~50 us, then writes
// a flag; the secondary waits, then reads the flag.
#include <cuda_runtime.h>

#include <cstdio>

__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__global__ void primary(int* flag, unsigned long long* t, int trigger_first) {
  if (trigger_first) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const unsigned long long t0 = gt();
  while (gt() - t0 < 50000) {
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    *(volatile int*)flag = 1;
    t[0] = gt();
  }
}

__global__ void secondary(int* flag, unsigned long long* t, int* seen) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    t[1] = gt();
    *seen = *(volatile int*)flag;
  }
}

int main() {
  int *flag, *seen;
  unsigned long long* t;
  cudaMalloc(&flag, 4);
  cudaMalloc(&seen, 4);
  cudaMalloc(&t, 16);
  for (int trig = 0; trig < 2; ++trig) {
    cudaMemset(flag, 0, 4);
    cudaMemset(seen, 0, 4);
    primary<<<8, 32>>>(flag, t, trig);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(8);
    cfg.blockDim = dim3(32);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, secondary, flag, t, seen);
    cudaError_t e = cudaDeviceSynchronize();
    int h_seen = -1;
    unsigned long long ht[2];
    cudaMemcpy(&h_seen, seen, 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(ht, t, 16, cudaMemcpyDeviceToHost);
    printf("trigger_first=%d err=%s secondary saw flag=%d, secondary wait returned %lld ns after the primary's write\n",
           trig, cudaGetErrorString(e), h_seen, (long long)(ht[1] - ht[0]));
  }
  return 0;
}
