// Decode-shape expert kernels (a4)+(a5), memory-bound: each touched pair's packed words are
// streamed from HBM ONCE and decoded for expert pos 0 and/or pos 1 (Algorithm 1)
// in registers, right before mma.sync m16n8k16 bf16 tensor-core MMAs ("swap-AB": weight
// rows are the M = 16 side, the 1..64 routed tokens the N = 8 side).
//
// Warp-specialised, persistent CTAs (one producer warp + 4 consumer warps):
//   producer  one lane issues TMA (cp.async.bulk.tensor) loads of 64-wide K stages of the
//             packed weight tile (128 rows: w13 = 64 gate + the same 64 up rows, w2 = 128
//             d_model rows) and of the tokens' activation rows of both positions into a
//             4-deep ring of 128-byte-swizzled shared-memory stages (mbarrier full/empty);
//             bytes in flight cost no registers, so every SM keeps >100 KB of HBM reads
//             outstanding.
//   consumers each owns 32 weight rows (two 16-row m-tiles) of the CTA tile; per stage it
//             reads its fragments from shared memory, SWAR-decodes two words per 32-bit
//             register, and issues the MMAs for each position that has tokens.
// K-permutation: in sub-step s (of 2 per 64-wide stage), lane (g, tig) takes the 8 physical
// k of 16-byte chunk 2*tig+s of rows g and g+8; its first 4 k feed MMA#0 fragments (a0,a2),
// the last 4 feed MMA#1. The activation fragments use the identical permutation, so each dot
// product sums exactly the same products (bank-conflict-free under the 128-byte swizzle).
// Work item = (active pair, 64/128-row block, K split); split-K partials are reduced in
// fixed split order by the last CTA to finish a row block (deterministic).
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "common.cuh"
#include "tc_ptx.cuh"
#include "tmap.cuh"

namespace pz {

namespace {

constexpr int kConsumerWarps = 8;
constexpr int kThreads = 32 * (1 + kConsumerWarps);
constexpr int kBK = 64;                         // K per stage (128-byte rows)
constexpr int kRowsPerCta = 128;                // weight rows per CTA tile
constexpr int kWBytes = kRowsPerCta * kBK * 2;  // 16 KB packed weights per stage
constexpr int kStages = 4;

template <int NT>
struct Cfg {
  static constexpr int kXRows = 8 * NT;             // tokens per position per pass
  static constexpr int kXBytes = kXRows * kBK * 2;  // per position
  static constexpr int kStageBytes = kWBytes + 2 * kXBytes;
  static constexpr size_t kSmem = 1024 + (size_t)kStages * kStageBytes + 256 + 4 * (2 * kMaxExperts + 8);
  static_assert(kSmem * 2 <= 227 * 1024, "two CTAs per SM");
};

struct PairTokens {
  int off0, cnt0, off1, cnt1;
};

__device__ __forceinline__ uint4 lds128(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}

// byte offset of (row, 16-byte chunk) inside a 128-byte-swizzled TMA box with 128-byte rows
__device__ __forceinline__ uint32_t swz(int row, int chunk) {
  return (uint32_t)(row * 128 + ((chunk ^ (row & 7)) << 4));
}

__device__ __forceinline__ void named_bar_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

__device__ __forceinline__ PairTokens load_pair(const int32_t* bucket_off, int p) {
  PairTokens pt;
  pt.off0 = bucket_off[2 * p];
  pt.off1 = bucket_off[2 * p + 1];
  pt.cnt0 = pt.off1 - pt.off0;
  pt.cnt1 = bucket_off[2 * p + 2] - pt.off1;
  return pt;
}

// Multipliers kept in registers (values unknown to ptxas) so the SWAR shifts / adds of the
// decode are emitted as IMAD on the FMA pipe instead of SHF / IADD3 on the ALU pipe.
struct Muls {
  uint32_t one, two, four, eight;
};

// One 32-wide K sub-step of one warp: decode the 8 packed registers of its m16 tile for the
// active position(s) and issue D[16 x 8N] += A[16 x 32] X for the first N n-tiles.
// MODE bit 0 = position 0 has tokens, bit 1 = position 1. Unpredicated, fully unrolled MMAs;
// both positions' MMAs are interleaved so consecutive HMMAs are independent.
// A fragment: a[2i] = (row g, k-pair i), a[2i+1] = (row g+8, k-pair i); registers 0..3 feed
// k16-half 0, registers 4..7 half 1 (see the K-permutation note at the top).
template <int NT, int N, int MODE>
__device__ __forceinline__ void sub_step(float (&acc0)[NT][4], float (&acc1)[NT][4], const uint4& wl,
                                         const uint4& wh, uint32_t xs0, uint32_t xs1, const Muls& mu) {
  const uint32_t W[8] = {wl.x, wh.x, wl.y, wh.y, wl.z, wh.z, wl.w, wh.w};
  uint32_t a0[8], a1[8];
  uint4 x0[N], x1[N];
  if (MODE & 1) {
#pragma unroll
    for (int t = 0; t < N; ++t) x0[t] = lds128(xs0 + t * 1024);
  }
  if (MODE & 2) {
#pragma unroll
    for (int t = 0; t < N; ++t) x1[t] = lds128(xs1 + t * 1024);
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    // b0 = (w & 0x8FFF8FFF) + 0x38003800: exponent rebuilt, sign S_i riding in bit 15
    const uint32_t b0 = imad(W[i] & 0x8FFF8FFFu, mu.one, 0x38003800u);
    if (MODE & 1) a0[i] = b0 & lane_msb_mask(imul(W[i], mu.four));                    // mask M_i
    if (MODE & 2)
      a1[i] = lop3_select_sign(imul(W[i], mu.two), b0) & lane_msb_mask(imul(W[i], mu.eight));  // S_j, M_j
  }
#pragma unroll
  for (int h = 0; h < 2; ++h) {
#pragma unroll
    for (int t = 0; t < N; ++t) {
      if (MODE & 1)
        mma_bf16_16816(acc0[t], a0[4 * h], a0[4 * h + 1], a0[4 * h + 2], a0[4 * h + 3], h ? x0[t].z : x0[t].x,
                       h ? x0[t].w : x0[t].y);
      if (MODE & 2)
        mma_bf16_16816(acc1[t], a1[4 * h], a1[4 * h + 1], a1[4 * h + 2], a1[4 * h + 3], h ? x1[t].z : x1[t].x,
                       h ? x1[t].w : x1[t].y);
    }
  }
}

template <int NT>
__device__ __forceinline__ void sub_dispatch(float (&acc0)[NT][4], float (&acc1)[NT][4], const uint4& wl,
                                             const uint4& wh, uint32_t xs0, uint32_t xs1, int nta0, int nta1,
                                             const Muls& mu) {
  const int mode = (nta0 > 0) | ((nta1 > 0) << 1);
  const int n = max(nta0, nta1);  // both active: empty tiles of the shorter position are harmless
#define PZ_CASE(NN)                                                                          \
  if (n == NN) {                                                                             \
    if (mode == 3) sub_step<NT, NN, 3>(acc0, acc1, wl, wh, xs0, xs1, mu);                    \
    else if (mode == 1) sub_step<NT, NN, 1>(acc0, acc1, wl, wh, xs0, xs1, mu);               \
    else sub_step<NT, NN, 2>(acc0, acc1, wl, wh, xs0, xs1, mu);                              \
    return;                                                                                  \
  }
  if (NT >= 4) PZ_CASE((NT >= 4 ? 4 : 1))
  if (NT >= 3) PZ_CASE((NT >= 3 ? 3 : 1))
  if (NT >= 2) PZ_CASE((NT >= 2 ? 2 : 1))
  PZ_CASE(1)
#undef PZ_CASE
}

// kW13: weights = packed w13 ([P*2f][d]); CTA rows = 64 gate rows + the same 64 up rows.
// !kW13: weights = packed w2 ([P*d][f]); CTA rows = 128 d_model rows.
template <int NT, bool kW13>
__global__ void __launch_bounds__(kThreads, 2) k_gemv_tma(
    const __grid_constant__ CUtensorMap tm_w, const __grid_constant__ CUtensorMap tm_x,
    const int32_t* __restrict__ bucket_off, const int32_t* __restrict__ active_pairs,
    const int32_t* __restrict__ n_active_ptr, int K, int f, int d, int n_rb, int ks,
    int64_t n_assign_cap, float* __restrict__ part, int32_t* __restrict__ counters,
    int32_t* __restrict__ work_ctr, uint16_t* __restrict__ h_out, float* __restrict__ y_out,
    uint32_t mul_one, int n_bucket_pairs) {
  using C = Cfg<NT>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)kStages * C::kStageBytes);
  uint64_t* empty = full + kStages;
  int4* hdr = reinterpret_cast<int4*>(empty + kStages);  // per-stage {item, pass base, kb, 0}
  int* s_last = reinterpret_cast<int*>(hdr + kStages);
  int32_t* s_off = s_last + 4;                   // bucket_off[0 .. 2P], cached once
  int32_t* s_active = s_off + kMaxExperts + 1;   // active_pairs[0 .. n_active)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], kConsumerWarps);
    }
    ptx::fence_mbar_init();
    ptx::tma_prefetch_desc(&tm_w);
    ptx::tma_prefetch_desc(&tm_x);
  }
  pdl_wait();     // route / gather / previous projection complete and visible
  pdl_trigger();  // the next kernel may begin its prologue as CTAs of this one retire
  // routing metadata in shared memory: per-item lookups stay on-chip (no dependent global
  // loads between one item's last TMA and the next item's first)
  const int n_active = *n_active_ptr;
  for (int i = threadIdx.x; i < n_active; i += blockDim.x) s_active[i] = active_pairs[i];
  for (int i = threadIdx.x; i <= 2 * n_bucket_pairs; i += blockDim.x) s_off[i] = bucket_off[i];
  __syncthreads();
  const int per_pair = n_rb * ks;
  const int kchunk = K / ks;
  const int nk = kchunk / kBK;

  if (warp == 0) {
    // ============================== producer ==============================
    // Dynamic scheduler: items are claimed with one atomicAdd each, so SMs that run ahead
    // take more work; every stage carries a header telling the consumers what it holds.
    if (lane != 0) return;
    const int n_items = n_active * per_pair;
    int stage = 0;
    uint32_t phase = 0;
    // the claim of the NEXT item is issued before the current one streams, so the atomic's
    // round trip overlaps the TMA traffic instead of draining the ring
    int next = atomicAdd(work_ctr, 1);
    for (;;) {
      const int item = next;
      if (item < n_items) next = atomicAdd(work_ctr, 1);
      if (item >= n_items) {
        ptx::mbar_wait(&empty[stage], phase ^ 1);
        hdr[stage] = make_int4(-1, 0, 0, 0);
        ptx::mbar_arrive(&full[stage]);  // completes the phase without data: "no more work"
        break;
      }
      const int z = item / per_pair;
      const int rb = (item / ks) % n_rb, kss = item % ks;
      const int p = s_active[z];
      const PairTokens pt = load_pair(s_off, p);
      const int maxcnt = max(pt.cnt0, pt.cnt1);
      const int wrow = kW13 ? p * 2 * f + rb * (kRowsPerCta / 2) : p * d + rb * kRowsPerCta;
      for (int base = 0; base < maxcnt; base += C::kXRows) {
        const bool a0 = pt.cnt0 > base, a1 = pt.cnt1 > base;
        const uint32_t bytes = kWBytes + (a0 ? C::kXBytes : 0) + (a1 ? C::kXBytes : 0);
        for (int kb = 0; kb < nk; ++kb) {
          const int kc = kss * kchunk + kb * kBK;
          ptx::mbar_wait_sleep(&empty[stage], phase ^ 1, 2000);
          uint8_t* st = smem + (size_t)stage * C::kStageBytes;
          hdr[stage] = make_int4(item, base, kb, 0);
          ptx::mbar_arrive_expect_tx(&full[stage], bytes);
          if (kW13) {
            ptx::tma_load_2d(st, &tm_w, &full[stage], kc, wrow);
            ptx::tma_load_2d(st + kWBytes / 2, &tm_w, &full[stage], kc, wrow + f);
          } else {
            ptx::tma_load_2d(st, &tm_w, &full[stage], kc, wrow);
          }
          if (a0) ptx::tma_load_2d(st + kWBytes, &tm_x, &full[stage], kc, pt.off0 + base);
          if (a1) ptx::tma_load_2d(st + kWBytes + C::kXBytes, &tm_x, &full[stage], kc, pt.off1 + base);
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
      }
    }
    return;
  }

  // ============================== consumers ==============================
  // Warp cw owns ONE m16 tile. w13: tile rows 0..7 = gate rows f0+8cw..+7, rows 8..15 = the
  // SAME d_ff indices' up rows, so each thread's C fragment holds g (c0,c1) and u (c2,c3)
  // of one (d_ff index, token) pair and SwiGLU happens in registers. w2: 16 d_model rows.
  const int cw = warp - 1;
  const int g = lane >> 2, tig = lane & 3;
  const uint32_t smem_base = (ptx::smem_u32(smem_raw) + 1023u) & ~1023u;  // == smem, shared window
  const Muls mu{mul_one, mul_one * 2u, mul_one * 4u, mul_one * 8u};
  const int trow_lo = kW13 ? cw * 8 + g : cw * 16 + g;            // tile row of fragment row g
  const int trow_hi = kW13 ? (kRowsPerCta / 2) + cw * 8 + g : cw * 16 + 8 + g;  // fragment row g+8
  // per-thread smem offsets (relative to the stage base) of its weight and activation fragments
  uint32_t off_lo[2], off_hi[2], off_x[2][NT];
#pragma unroll
  for (int sub = 0; sub < 2; ++sub) {
    // sub-step `sub` of lane tig reads 16-byte chunk 2*tig + sub of its rows: within every
    // 8-lane LDS phase (rows g, g+1) the chunks {2t+s} ^ g and {2t+s} ^ (g+1) are 8 distinct
    // bank groups under the 128-byte swizzle -> conflict-free (4*sub + tig would be 2-way)
    off_lo[sub] = swz(trow_lo, 2 * tig + sub);
    off_hi[sub] = swz(trow_hi, 2 * tig + sub);
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) off_x[sub][nt] = kWBytes + swz(nt * 8 + g, 2 * tig + sub);
  }
  int stage = 0;
  uint32_t phase = 0;
  for (;;) {
    // the first stage of each item names it (or says "no more work")
    ptx::mbar_wait(&full[stage], phase);
    const int4 h0 = hdr[stage];
    if (h0.x < 0) break;
    const int item = h0.x;
    const int z = item / per_pair;
    const int rb = (item / ks) % n_rb, kss = item % ks;
    const int p = s_active[z];
    const PairTokens pt = load_pair(s_off, p);
    const int maxcnt = max(pt.cnt0, pt.cnt1);
    // output features of fragment rows g and g+8
    const int ofeat_lo = kW13 ? rb * (kRowsPerCta / 2) + cw * 8 + g : rb * kRowsPerCta + cw * 16 + g;
    const int ofeat_hi = kW13 ? ofeat_lo : ofeat_lo + 8;
    for (int base = 0; base < maxcnt; base += C::kXRows) {
      const int n0 = min(max(pt.cnt0 - base, 0), C::kXRows);
      const int n1 = min(max(pt.cnt1 - base, 0), C::kXRows);
      const int nta0 = (n0 + 7) >> 3, nta1 = (n1 + 7) >> 3;  // n-tiles with tokens (warp-uniform)
      float acc0[NT][4], acc1[NT][4];
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc0[nt][q] = acc1[nt][q] = 0.f;

      for (int kb = 0; kb < nk; ++kb) {
        ptx::mbar_wait(&full[stage], phase);
        const uint32_t st = smem_base + (uint32_t)stage * C::kStageBytes;
        // both sub-steps' weight fragments are requested up front (LDS latency overlap)
        const uint4 wl0 = lds128(st + off_lo[0]), wh0 = lds128(st + off_hi[0]);
        const uint4 wl1 = lds128(st + off_lo[1]), wh1 = lds128(st + off_hi[1]);
        sub_dispatch<NT>(acc0, acc1, wl0, wh0, st + off_x[0][0], st + off_x[0][0] + C::kXBytes, nta0, nta1, mu);
        sub_dispatch<NT>(acc0, acc1, wl1, wh1, st + off_x[1][0], st + off_x[1][0] + C::kXBytes, nta0, nta1, mu);
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&empty[stage]);
        if (++stage == kStages) { stage = 0; phase ^= 1; }
      }
      // ---- epilogue of this pass: c0,c1 = (row g, tokens 2tig, 2tig+1); c2,c3 = row g+8 ----
      const bool lo_ok = kW13 || ofeat_lo < d, hi_ok = kW13 || ofeat_hi < d;  // w2 box overhang
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int tok = nt * 8 + 2 * tig + j;
#pragma unroll
          for (int ps = 0; ps < 2; ++ps) {
            const int nn = ps ? n1 : n0;
            if (tok >= nn) continue;
            const float lo = ps ? acc1[nt][j] : acc0[nt][j];
            const float hi = ps ? acc1[nt][2 + j] : acc0[nt][2 + j];
            const size_t a = (size_t)((ps ? pt.off1 : pt.off0) + base + tok);
            if (ks == 1) {
              if (kW13) {
                h_out[a * f + ofeat_lo] = f32_to_bf16_bits_rn(silu_mul(lo, hi));
              } else {
                if (lo_ok) y_out[a * d + ofeat_lo] = lo;
                if (hi_ok) y_out[a * d + ofeat_hi] = hi;
              }
            } else {
              // partials: w13 -> part[kss][a][0:f] = g, [f:2f] = u ; w2 -> part[kss][a][0:d]
              const int width = kW13 ? 2 * f : d;
              float* dst = part + ((size_t)kss * n_assign_cap + a) * width;
              if (kW13) {
                dst[ofeat_lo] = lo;
                dst[f + ofeat_lo] = hi;
              } else {
                if (lo_ok) dst[ofeat_lo] = lo;
                if (hi_ok) dst[ofeat_hi] = hi;
              }
            }
          }
        }
    }
    if (ks > 1) {
      // ---- the last of the ks CTAs of this (pair, row block) reduces in split order ----
      // (the barrier orders every consumer's partial stores before thread 32's gpu-scope
      //  fence, which is cumulative, so one fence publishes them all)
      named_bar_sync(1, kConsumerWarps * 32);
      const int ctr = p * n_rb + rb;
      if (threadIdx.x == 32) {
        __threadfence();
        const int prev = atomicAdd(&counters[ctr], 1);
        *s_last = (prev == ks - 1);
        if (*s_last) counters[ctr] = 0;  // ready for the next call on this stream
      }
      if (threadIdx.x == 32 && *s_last) __threadfence();  // acquire side of the counter
      named_bar_sync(1, kConsumerWarps * 32);
      if (*s_last) {
        const int row_base = kW13 ? rb * (kRowsPerCta / 2) : rb * kRowsPerCta;
        const int rows = kW13 ? kRowsPerCta / 2 : min(kRowsPerCta, d - row_base);  // multiple of 4
        const int q4 = rows / 4;
        const int n_tot = pt.cnt0 + pt.cnt1;  // buckets 2p and 2p+1 are adjacent
        const int width = kW13 ? 2 * f : d;
        for (int i = threadIdx.x - 32; i < n_tot * q4; i += kConsumerWarps * 32) {
          const size_t a = (size_t)(pt.off0 + i / q4);
          const int r = row_base + 4 * (i % q4);
          float4 s0 = make_float4(0.f, 0.f, 0.f, 0.f), s1 = s0;
          const float* src = part + a * width + r;
          const size_t split_stride = (size_t)n_assign_cap * width;
#pragma unroll 4
          for (int s = 0; s < ks; ++s) {
            const float4 v = __ldcg(reinterpret_cast<const float4*>(src + s * split_stride));
            s0.x += v.x; s0.y += v.y; s0.z += v.z; s0.w += v.w;
            if (kW13) {
              const float4 u = __ldcg(reinterpret_cast<const float4*>(src + s * split_stride + f));
              s1.x += u.x; s1.y += u.y; s1.z += u.z; s1.w += u.w;
            }
          }
          if (kW13) {
            uint2 o;
            o.x = f32_to_bf16_rne_bits(silu_mul(s0.x, s1.x)) | (f32_to_bf16_rne_bits(silu_mul(s0.y, s1.y)) << 16);
            o.y = f32_to_bf16_rne_bits(silu_mul(s0.z, s1.z)) | (f32_to_bf16_rne_bits(silu_mul(s0.w, s1.w)) << 16);
            *reinterpret_cast<uint2*>(h_out + a * f + r) = o;
          } else {
            *reinterpret_cast<float4*>(y_out + a * d + r) = s0;
          }
        }
      }
      named_bar_sync(1, kConsumerWarps * 32);
    }
  }
}

// Largest split count s <= want with (K / s) % kBK == 0.
int pick_split(int K, int want) {
  int best = 1;
  for (int s = 1; s <= want; ++s)
    if (K % (s * kBK) == 0) best = s;
  return best;
}

template <int NT, bool kW13>
int launch_one(const CUtensorMap& tw, const CUtensorMap& tx, const int32_t* bucket_off, const int32_t* active,
               const int32_t* n_active, int K, int f, int d, int n_rb, int ks, int max_active, int64_t n_assign_cap,
               float* part, int32_t* counters, int32_t* work_ctr, uint16_t* h, float* y, int n_pairs,
               cudaStream_t stream) {
  using C = Cfg<NT>;
  auto kern = k_gemv_tma<NT, kW13>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::kSmem);
    attr = true;
  }
  const int n_items = max_active * n_rb * ks;  // upper bound; the device knows the active count
  const int grid = std::min(n_items, 2 * num_sms());
  {
    ProfScope _ps(kW13 ? "w13_gemv" : "w2_gemv", stream);
    cudaError_t e = launch_pdl(kern, dim3(grid), dim3(kThreads), C::kSmem, stream, tw, tx, bucket_off, active, n_active,
                               K, f, d, n_rb, ks, n_assign_cap, part, counters, work_ctr, h, y, 1u, n_pairs);
    if (e != cudaSuccess) return cuda_check(e, kW13 ? "w13_gemv launch" : "w2_gemv launch");
  }
  return cuda_check(cudaGetLastError(), kW13 ? "w13_gemv launch" : "w2_gemv launch");
}

}  // namespace

namespace {
int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return (v && *v) ? atoi(v) : dflt;
}
}  // namespace

// PUZZLE_GEMV_NT / PUZZLE_GEMV_KS13 / PUZZLE_GEMV_KS2 / PUZZLE_GEMV_ITEMS_PER_CTA override the
// heuristics below (tuning experiments only; results are identical up to fp32 summation order).
// n-tiles (8 tokens each) per position per pass: sized for a typical bucket of a uniform
// router, mean mu = T*k/E tokens, so that a second pass (re-reading the item's weights from L2)
// is rare: ceil((mu + 1.5 sqrt(mu) + 1) / 8), capped by the batch itself.
int gemv_nt_for(int64_t T, int k, int E) {
  const int forced = env_int("PUZZLE_GEMV_NT", 0);
  if (forced >= 1 && forced <= 4) return forced;
  const double mu = (double)T * k / E;
  int nt = (int)ceil((mu + 1.5 * sqrt(mu) + 1.0) / 8.0);
  nt = std::min(nt, (int)((T + 7) / 8));
  return std::max(1, std::min(nt, 4));
}

// Split-K so that each resident CTA (2 per SM) gets several work items: the dynamic scheduler's
// tail is at most one item. Partials cost n_assign * ks * width floats, so small batches (where
// they are negligible) split finer than large ones.
void gemv_splits(int d, int f, int max_active, int64_t n_assign, int* ks13, int* ks2) {
  (void)n_assign;  // (finer splits for small batches measured slower: per-item overheads dominate)
  const int per_cta = env_int("PUZZLE_GEMV_ITEMS_PER_CTA", 2);
  const int target = num_sms() * 2 * per_cta;
  const int items13 = (f / 64) * max_active, items2 = ((d + kRowsPerCta - 1) / kRowsPerCta) * max_active;
  int want13 = (target + items13 - 1) / items13, want2 = (target + items2 - 1) / items2;
  want13 = std::min(std::max(want13, 1), 16);
  want2 = std::min(std::max(want2, 1), 32);
  while (want13 > 1 && d / want13 < 128) --want13;
  while (want2 > 1 && f / want2 < 128) --want2;
  *ks13 = pick_split(d, env_int("PUZZLE_GEMV_KS13", want13));
  *ks2 = pick_split(f, env_int("PUZZLE_GEMV_KS2", want2));
}

bool gemv_supported(int d, int f) { return d % 64 == 0 && f % 64 == 0; }

// x_rows: [n_assign_cap][d] bf16 in bucket order (TMA source); h: [n_assign_cap][f]; y: [n_assign_cap][d]
int launch_gemv_experts(const uint16_t* w13, const uint16_t* w2, int n_pairs, int d, int f, const uint16_t* x_rows,
                        const int32_t* bucket_off, const int32_t* active_pairs, const int32_t* n_active,
                        int max_active, int64_t n_assign_cap, int nt, int ks13, int ks2, float* part13,
                        float* part2, int32_t* counters13, int32_t* counters2, int32_t* work_ctrs,
                        uint16_t* h, float* y, cudaStream_t stream) {
  if (max_active == 0 || n_assign_cap == 0) return PUZZLE_OK;
  const int xrows = 8 * nt;
  CUtensorMap tw13, tx13, tw2, tx2;
  int rc;
  if ((rc = make_tmap_2d(&tw13, w13, (int64_t)n_pairs * 2 * f, d, 64, kBK))) return rc;
  if ((rc = make_tmap_2d(&tx13, x_rows, n_assign_cap, d, xrows, kBK))) return rc;
  if ((rc = make_tmap_2d(&tw2, w2, (int64_t)n_pairs * d, f, kRowsPerCta, kBK))) return rc;
  if ((rc = make_tmap_2d(&tx2, h, n_assign_cap, f, xrows, kBK))) return rc;
  const int rb13 = f / 64, rb2 = (d + kRowsPerCta - 1) / kRowsPerCta;
#define PZ_GO(NT)                                                                                             \
  do {                                                                                                        \
    if ((rc = launch_one<NT, true>(tw13, tx13, bucket_off, active_pairs, n_active, d, f, d, rb13, ks13,        \
                                   max_active, n_assign_cap, part13, counters13, work_ctrs, h, y, n_pairs,     \
                                   stream)))                                                                  \
      return rc;                                                                                              \
    return launch_one<NT, false>(tw2, tx2, bucket_off, active_pairs, n_active, f, f, d, rb2, ks2, max_active, \
                                 n_assign_cap, part2, counters2, work_ctrs + 1, h, y, n_pairs, stream);      \
  } while (0)
  if (nt == 1) PZ_GO(1);
  if (nt == 2) PZ_GO(2);
  if (nt == 3) PZ_GO(3);
  PZ_GO(4);
#undef PZ_GO
}

}  // namespace pz
