// (a1) pack, (a2) unpack and the fused Eq. 1-7 merge+pack (NEXT-1) kernels.
// All three are elementwise and HBM-bound: 128-bit vector loads/stores, grid-stride
// loops sized to a multiple of the SM count, integer-only bf16 rounding.
#include "common.cuh"

namespace pz {

namespace {

constexpr int kThreads = 256;

struct StatAcc {
  uint32_t lo = 0, hi = 0, nf = 0, neg = 0;
};

__device__ __forceinline__ void flush_stats(const StatAcc& s, puzzle_pack_stats* stats) {
  if (stats == nullptr) return;
  // warp-aggregate, then one 64-bit atomic per warp per non-zero counter
  uint32_t lo = __reduce_add_sync(0xffffffffu, s.lo);
  uint32_t hi = __reduce_add_sync(0xffffffffu, s.hi);
  uint32_t nf = __reduce_add_sync(0xffffffffu, s.nf);
  uint32_t ng = __reduce_add_sync(0xffffffffu, s.neg);
  if ((threadIdx.x & 31) == 0) {
    if (lo) atomicAdd(&stats->rounded_up, (unsigned long long)lo);
    if (hi) atomicAdd(&stats->saturated, (unsigned long long)hi);
    if (nf) atomicAdd(&stats->nonfinite, (unsigned long long)nf);
    if (ng) atomicAdd(&stats->negative, (unsigned long long)ng);
  }
}

__device__ __forceinline__ uint32_t pack_one(float w, uint32_t m0, uint32_t m1, uint32_t s0,
                                             uint32_t s1, StatAcc& acc) {
  acc.nf += !isfinite(w);
  acc.neg += (w < 0.0f);
  uint32_t lo, hi;
  uint32_t word = encode_word(f32_to_bf16_rne_bits(w), s0 != 0, s1 != 0, m0 != 0, m1 != 0, &lo, &hi);
  acc.lo += lo;
  acc.hi += hi;
  return word;
}

// 4 elements per thread per iteration when every array is 16/4-byte aligned.
__global__ void __launch_bounds__(kThreads) k_pack_vec4(const float4* __restrict__ w,
                                                        const uchar4* __restrict__ m0,
                                                        const uchar4* __restrict__ m1,
                                                        const uchar4* __restrict__ s0,
                                                        const uchar4* __restrict__ s1, int64_t n4,
                                                        uint2* __restrict__ out,
                                                        puzzle_pack_stats* stats) {
  StatAcc acc;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4;
       i += (int64_t)gridDim.x * blockDim.x) {
    float4 v = w[i];
    uchar4 a = m0[i], b = m1[i], c = s0[i], d = s1[i];
    uint32_t p0 = pack_one(v.x, a.x, b.x, c.x, d.x, acc);
    uint32_t p1 = pack_one(v.y, a.y, b.y, c.y, d.y, acc);
    uint32_t p2 = pack_one(v.z, a.z, b.z, c.z, d.z, acc);
    uint32_t p3 = pack_one(v.w, a.w, b.w, c.w, d.w, acc);
    out[i] = make_uint2(p0 | (p1 << 16), p2 | (p3 << 16));
  }
  flush_stats(acc, stats);
}

__global__ void __launch_bounds__(kThreads) k_pack_scalar(const float* __restrict__ w,
                                                          const uint8_t* __restrict__ m0,
                                                          const uint8_t* __restrict__ m1,
                                                          const uint8_t* __restrict__ s0,
                                                          const uint8_t* __restrict__ s1,
                                                          int64_t begin, int64_t n,
                                                          uint16_t* __restrict__ out,
                                                          puzzle_pack_stats* stats) {
  StatAcc acc;
  for (int64_t i = begin + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (uint16_t)pack_one(w[i], m0[i], m1[i], s0[i], s1[i], acc);
  flush_stats(acc, stats);
}

template <int POS>
__global__ void __launch_bounds__(kThreads) k_unpack_vec8(const uint4* __restrict__ in, int64_t n8,
                                                          uint4* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n8;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint4 v = ldg_nc_v4(in + i);
    out[i] = make_uint4(decode2<POS>(v.x), decode2<POS>(v.y), decode2<POS>(v.z), decode2<POS>(v.w));
  }
}

template <int POS>
__global__ void __launch_bounds__(kThreads) k_unpack_scalar(const uint16_t* __restrict__ in,
                                                            int64_t begin, int64_t n,
                                                            uint16_t* __restrict__ out) {
  for (int64_t i = begin + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (uint16_t)decode2<POS>((uint32_t)in[i]);
}

// Eq. 1-7 in IEEE f32 with explicit _rn intrinsics (no contraction), identical operation
// order to the expressions as written in the paper / oracle O2.
__device__ __forceinline__ uint32_t merge_pack_one(uint32_t wi_bits, uint32_t wj_bits, float ni,
                                                   float nj, float tau, StatAcc& acc) {
  const float wi = bf16_bits_to_f32(wi_bits);
  const float wj = bf16_bits_to_f32(wj_bits);
  const float a = fabsf(wi);
  const float b = fabsf(wj);
  // Eq. 1 (0/0 := 0, R4)
  const float delta = (a == 0.0f && b == 0.0f) ? 0.0f : __fdiv_rn(fabsf(__fsub_rn(a, b)), __fadd_rn(a, b));
  const uint32_t sim = delta <= tau;                       // Eq. 2
  const uint32_t si = wi < 0.0f, sj = wj < 0.0f;           // Eq. 3
  const float Ai = __fmul_rn(a, ni), Aj = __fmul_rn(b, nj);  // Eq. 4
  const uint32_t sal_i = Ai >= Aj;                         // Eq. 5 (tie -> i)
  const uint32_t mi = sal_i | sim, mj = (1u - sal_i) | sim;  // Eq. 6
  const float wm = sim ? __fmul_rn(__fadd_rn(a, b), 0.5f) : (sal_i ? a : b);  // Eq. 7
  return pack_one(wm, mi, mj, si, sj, acc);
}

// 8 columns per thread per iteration; requires cols % 8 == 0 (checked on the host).
__global__ void __launch_bounds__(kThreads) k_merge_experts_pack(
    const uint4* __restrict__ wi, const uint4* __restrict__ wj, const float* __restrict__ ni,
    const float* __restrict__ nj, int64_t rows, int64_t cols, int64_t total8, float tau,
    uint4* __restrict__ out, puzzle_pack_stats* stats) {
  StatAcc acc;
  const int64_t cols8 = cols / 8;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total8;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c8 = i % cols8;
    const int64_t mat = i / (cols8 * rows);
    const float* nip = ni + mat * cols + c8 * 8;
    const float* njp = nj + mat * cols + c8 * 8;
    const float4 ni0 = *reinterpret_cast<const float4*>(nip);
    const float4 ni1 = *reinterpret_cast<const float4*>(nip + 4);
    const float4 nj0 = *reinterpret_cast<const float4*>(njp);
    const float4 nj1 = *reinterpret_cast<const float4*>(njp + 4);
    const float nis[8] = {ni0.x, ni0.y, ni0.z, ni0.w, ni1.x, ni1.y, ni1.z, ni1.w};
    const float njs[8] = {nj0.x, nj0.y, nj0.z, nj0.w, nj1.x, nj1.y, nj1.z, nj1.w};
    const uint4 a = ldg_nc_v4(wi + i);
    const uint4 b = ldg_nc_v4(wj + i);
    const uint32_t av[4] = {a.x, a.y, a.z, a.w};
    const uint32_t bv[4] = {b.x, b.y, b.z, b.w};
    uint32_t o[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint32_t lo = merge_pack_one(av[q] & 0xFFFFu, bv[q] & 0xFFFFu, nis[2 * q], njs[2 * q], tau, acc);
      uint32_t hi = merge_pack_one(av[q] >> 16, bv[q] >> 16, nis[2 * q + 1], njs[2 * q + 1], tau, acc);
      o[q] = lo | (hi << 16);
    }
    out[i] = make_uint4(o[0], o[1], o[2], o[3]);
  }
  flush_stats(acc, stats);
}

int grid_for(int64_t work_items, int threads) {
  int64_t blocks = (work_items + threads - 1) / threads;
  int64_t cap = (int64_t)num_sms() * 8;  // 8 resident 256-thread CTAs per SM
  if (blocks > cap) blocks = cap;
  return (int)(blocks < 1 ? 1 : blocks);
}

bool aligned(const void* p, uintptr_t a) { return (reinterpret_cast<uintptr_t>(p) & (a - 1)) == 0; }

}  // namespace

int launch_merge_pack(const float* w, const uint8_t* m0, const uint8_t* m1, const uint8_t* s0,
                      const uint8_t* s1, int64_t n, uint16_t* out, puzzle_pack_stats* stats,
                      cudaStream_t stream) {
  int64_t done = 0;
  if (aligned(w, 16) && aligned(m0, 4) && aligned(m1, 4) && aligned(s0, 4) && aligned(s1, 4) &&
      aligned(out, 8) && n >= 4) {
    int64_t n4 = n / 4;
    { ProfScope _ps("pack", stream); k_pack_vec4<<<grid_for(n4, kThreads), kThreads, 0, stream>>>(
        reinterpret_cast<const float4*>(w), reinterpret_cast<const uchar4*>(m0),
        reinterpret_cast<const uchar4*>(m1), reinterpret_cast<const uchar4*>(s0),
        reinterpret_cast<const uchar4*>(s1), n4, reinterpret_cast<uint2*>(out), stats); }
    done = n4 * 4;
  }
  if (done < n)
    { ProfScope _ps("pack_tail", stream); k_pack_scalar<<<grid_for(n - done, kThreads), kThreads, 0, stream>>>(w, m0, m1, s0, s1, done, n,
                                                                        out, stats); }
  return cuda_check(cudaGetLastError(), "puzzle_merge_pack launch");
}

int launch_unpack(const uint16_t* in, int pos, int64_t n, uint16_t* out, cudaStream_t stream) {
  int64_t done = 0;
  if (aligned(in, 16) && aligned(out, 16) && n >= 8) {
    int64_t n8 = n / 8;
    if (pos == 0)
      { ProfScope _ps("unpack", stream); k_unpack_vec8<0><<<grid_for(n8, kThreads), kThreads, 0, stream>>>(
          reinterpret_cast<const uint4*>(in), n8, reinterpret_cast<uint4*>(out)); }
    else
      { ProfScope _ps("unpack", stream); k_unpack_vec8<1><<<grid_for(n8, kThreads), kThreads, 0, stream>>>(
          reinterpret_cast<const uint4*>(in), n8, reinterpret_cast<uint4*>(out)); }
    done = n8 * 8;
  }
  if (done < n) {
    if (pos == 0)
      { ProfScope _ps("unpack_tail", stream); k_unpack_scalar<0><<<grid_for(n - done, kThreads), kThreads, 0, stream>>>(in, done, n, out); }
    else
      { ProfScope _ps("unpack_tail", stream); k_unpack_scalar<1><<<grid_for(n - done, kThreads), kThreads, 0, stream>>>(in, done, n, out); }
  }
  return cuda_check(cudaGetLastError(), "puzzle_unpack launch");
}

int launch_merge_experts_pack(const uint16_t* wi, const uint16_t* wj, const float* ni,
                              const float* nj, int64_t n_mats, int64_t rows, int64_t cols,
                              float tau, uint16_t* out, puzzle_pack_stats* stats,
                              cudaStream_t stream) {
  const int64_t total8 = n_mats * rows * cols / 8;
  if (total8 == 0) return PUZZLE_OK;
  { ProfScope _ps("merge_experts_pack", stream); k_merge_experts_pack<<<grid_for(total8, kThreads), kThreads, 0, stream>>>(
      reinterpret_cast<const uint4*>(wi), reinterpret_cast<const uint4*>(wj), ni, nj, rows, cols,
      total8, tau, reinterpret_cast<uint4*>(out), stats); }
  return cuda_check(cudaGetLastError(), "puzzle_merge_experts_pack launch");
}

}  // namespace pz
