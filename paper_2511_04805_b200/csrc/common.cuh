// Shared device helpers for libpuzzlemoe (sm_100a only). Nothing here is shared with
// oracle/ (the CPU oracle is an independent statement of the same paper passages).
#pragma once

#include <cuda_runtime.h>
#include <cstdio>
#include <stdint.h>

#include <atomic>
#include <string>
#include <utility>

#include "../../include/puzzlemoe.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ != 1000)
#error "libpuzzlemoe targets sm_100a (B200) only"
#endif

namespace pz {

// ---- host-side error plumbing (thread-local detail string) ----
void set_error(const std::string& msg);
int fail(int status, const std::string& msg);
int cuda_check(cudaError_t e, const char* what);
int num_sms();

constexpr int kMaxExperts = 512;

// Checked builds (-DPZ_CHECKED, scripts/build_variant.py): device-side invariant checks at the
// index computations of every kernel (a violated check prints and traps). The substitute for
// compute-sanitizer, which the GPU pool refuses (profiles/r02/sanitizer_refused.log).
#ifdef PZ_CHECKED
#define PZ_DCHECK(cond)                                                                        \
  do {                                                                                         \
    if (!(cond)) {                                                                             \
      printf("PZ_DCHECK failed %s:%d block %d thread %d: %s\n", __FILE__, __LINE__, (int)blockIdx.x, \
             (int)threadIdx.x, #cond);                                                         \
      __trap();                                                                                \
    }                                                                                          \
  } while (0)
#else
#define PZ_DCHECK(cond) \
  do {                  \
  } while (0)
#endif

// The current device (attributes and SM counts below are per device: a process may drive
// several GPUs, one per thread or one after the other).
int current_device();

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device): `mask` is the
// kernel's own set of devices already configured (bit = device ordinal, < 64).
template <typename K>
cudaError_t ensure_smem_attr(K* kern, size_t bytes, std::atomic<uint64_t>& mask) {
  const uint64_t bit = 1ull << (current_device() & 63);
  if (mask.load(std::memory_order_acquire) & bit) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) mask.fetch_or(bit, std::memory_order_acq_rel);
  return e;
}

// Per-kernel event bracketing while a puzzle_profile window is open (abi.cu).
void prof_mark_begin(const char* name, cudaStream_t s);
void prof_mark_end(cudaStream_t s);
struct ProfScope {
  cudaStream_t s;
  ProfScope(const char* name, cudaStream_t st) : s(st) { prof_mark_begin(name, st); }
  ~ProfScope() { prof_mark_end(s); }
};

// ---- Programmatic Dependent Launch (the forward's kernel chain) ----
// A kernel launched with launch_pdl may start (prologue: barrier init, descriptor prefetch)
// while its predecessor on the stream is still finishing; pdl_wait() blocks until every
// prerequisite grid has completed and its writes are visible (a no-op for a normal launch).
// pdl_trigger() lets the NEXT kernel's CTAs start launching early.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Same, launched as clusters of 2 CTAs (grid.x even)
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl_cluster2(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                                Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = 2;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                       Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// Copy one row of n16 16-byte words with a warp: 8 loads in flight per lane before the stores
// (a row is latency-bound: one load->store round trip per 512 B otherwise).
__device__ __forceinline__ void warp_copy_row(const uint4* __restrict__ sp, uint4* __restrict__ dp, int64_t n16,
                                              int lane) {
  constexpr int U = 8;
  for (int64_t c0 = lane; c0 < n16; c0 += 32 * U) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (c0 + u * 32 < n16) v[u] = sp[c0 + u * 32];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (c0 + u * 32 < n16) dp[c0 + u * 32] = v[u];
  }
}

// ---- packed word layout (Algorithm 1) ----
// bit15 S_i | bit14 S_j | bit13 M_i | bit12 M_j | bits 11..7 e' = e-112 | bits 6..0 mantissa

// f32 -> bf16 round-to-nearest-even in integer arithmetic (reading R3). Integer-only so
// that FTZ / fast-math settings can never change the result. NaN stays NaN (quiet, sign and
// top payload bits kept: IEEE / torch's cast), so an overflow inside an expert propagates.
__device__ __forceinline__ uint32_t f32_to_bf16_rne_bits(float x) {
  uint32_t u = __float_as_uint(x);
  if ((u & 0x7FFFFFFFu) > 0x7F800000u) return (u >> 16) | 0x40u;
  return (u + 0x7FFFu + ((u >> 16) & 1u)) >> 16;
}

// Encode one word from a magnitude already rounded to bf16 bits + 4 header bits.
// Returns the word; sets *lo / *hi when the exponent was clamped (R1).
__device__ __forceinline__ uint32_t encode_word(uint32_t h, uint32_t s0, uint32_t s1, uint32_t m0,
                                                uint32_t m1, uint32_t* lo, uint32_t* hi) {
  uint32_t e = (h >> 7) & 0xFFu;
  *lo = e < 112u;
  *hi = e > 143u;
  e = e < 112u ? 112u : (e > 143u ? 143u : e);
  return (s0 << 15) | (s1 << 14) | (m0 << 13) | (m1 << 12) | ((e - 112u) << 7) | (h & 0x7Fu);
}

// prmt with msb-replicate: for each 16-bit lane, 0xFFFF if bit 15 of the lane is set.
__device__ __forceinline__ uint32_t lane_msb_mask(uint32_t v) {
  uint32_t r;
  asm("prmt.b32 %0, %1, 0, 0xBB99;" : "=r"(r) : "r"(v));
  return r;
}

// Two-lane SWAR Algorithm 1: decode both packed words held in `w` for expert `POS`.
// Per 16-bit lane: mask ? (sign << 15) | ((w & 0x0F80) + (112 << 7)) | (w & 0x7F) : 0.
// (w & 0x0FFF) + 0x3800 == (w & 0x0F80) + (112 << 7) | (w & 0x7F) since the 0x3800 add
// never carries out of bits 11..7 (max 0x0FFF + 0x3800 = 0x47FF < 0x8000): no cross-lane carry.
template <int POS>
__device__ __forceinline__ uint32_t decode2(uint32_t w, uint32_t base) {
  const uint32_t sign_src = POS == 0 ? w : (w << 1);         // sign bit 15 (pos 0) / 14 (pos 1)
  const uint32_t val = (sign_src & 0x80008000u) | base;      // one LOP3
  const uint32_t mask = lane_msb_mask(w << (2 + POS));       // mask bit 13 / 12 -> bit 15
  return val & mask;
}
__device__ __forceinline__ uint32_t decode_base(uint32_t w) {
  return (w & 0x0FFF0FFFu) + 0x38003800u;
}
template <int POS>
__device__ __forceinline__ uint32_t decode2(uint32_t w) {
  return decode2<POS>(w, decode_base(w));
}

// Integer multiply / multiply-add through inline PTX with a register operand (a value ptxas
// cannot see), so shifts and adds of the SWAR decode issue as IMAD on the FMA pipe.
__device__ __forceinline__ uint32_t imul(uint32_t a, uint32_t b) {
  uint32_t r;
  asm("mul.lo.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}
__device__ __forceinline__ uint32_t imad(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t r;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
  return r;
}

// ---- memory helpers ----
__device__ __forceinline__ uint4 ldg_nc_v4(const void* p) {
  uint4 r;
  asm("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// silu(g) * u with the SFU exponential and an approximate division (both ~2 ulp of fp32, far
// below the bf16 rounding of h that follows): the IEEE expf + division cost ~30 instructions
// and dominated the prefill epilogue. g -> -inf: exp -> inf, the quotient -> 0 (silu's limit).
__device__ __forceinline__ float silu_mul(float g, float u) { return __fdividef(g, 1.0f + __expf(-g)) * u; }

__device__ __forceinline__ uint16_t f32_to_bf16_bits_rn(float x) {
  return (uint16_t)f32_to_bf16_rne_bits(x);
}
__device__ __forceinline__ float bf16_bits_to_f32(uint32_t h) { return __uint_as_float(h << 16); }

}  // namespace pz
