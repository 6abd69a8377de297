// Prefill-shape expert kernels (a4)+(a5) on the 5th-generation tensor cores.
//
// Grouped GEMM over the 2P (pair, pos) buckets: D[tokens, n] = X_b[tokens, K] . W^_b[n, K]^T
// with W^_b = Algorithm-1 decode of the pair's packed words for position pos.
// One persistent CTA per SM walks a static tile list (n-block major, so the CTAs running at
// the same time share the packed weight tiles in L2; both positions of a pair follow each
// other so one packed tile serves both experts).
//
// Per CTA tile: 256 tokens (two M=128 UMMAs into two TMEM accumulators of 256 fp32
// columns each = all 512 TMEM columns) x 256 output rows, K in 64-wide stages:
//   warp 0      TMA producer: X tile [256 x 64] bf16 and the PACKED weight tile [256 x 64]
//               u16, both 128-byte swizzled, completing on full[s]
//   warps 2..5  decode warpgroup: Alg. 1 in place on the packed tile (elementwise, so the
//               swizzled layout is preserved), fence.proxy.async, arrive on dec[s];
//               after the last k-block of a tile they are the epilogue (TMEM -> registers
//               -> SwiGLU / fp32 -> global)
//   warp 1      MMA issuer: one elected lane issues tcgen05.mma (A, B from SMEM
//               descriptors, D in TMEM), tcgen05.commit frees the stage (empty[s]) and,
//               after the last k-block, signals tmem_full.
// w13 variant: the B tile is 128 gate rows + the same 128 up rows (N = 256) so the
// epilogue sees g and u of one d_ff index in one thread: h = silu(g) * u -> bf16.
// w2 variant: B = 256 rows of W2 (N = 256 d_model rows), epilogue writes fp32 y.
#include <cuda.h>

#include <mutex>

#include "common.cuh"
#include "tc_ptx.cuh"
#include "tmap.cuh"

namespace pz {

#ifdef PZ_TRACE  // pipeline timeline of one CTA (tuning builds only; scripts/trace_tc.py)
__device__ unsigned long long g_tct[6][4096];  // 0 TMA issue, 1 decode done, 2 MMA issued, 3 epi start, 4 epi end
__device__ unsigned long long g_tcc[2][1024][2];  // [kernel][cta] {start after wait, end}
__device__ __forceinline__ unsigned long long tc_gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define PZ_TT(ev, idx) \
  if (kW13 && blockIdx.x == PZ_TRACE && (idx) < 4096) g_tct[ev][idx] = tc_gtimer()
extern "C" __attribute__((visibility("default"))) int puzzle_debug_tc(void* dst, size_t bytes, void* dst2,
                                                                    size_t bytes2) {
  int rc = (int)cudaMemcpyFromSymbol(dst, g_tct, bytes);
  if (rc) return rc;
  return (int)cudaMemcpyFromSymbol(dst2, g_tcc, bytes2);
}
#else
#define PZ_TT(ev, idx)
#endif

namespace {

#ifndef PZ_TC_DEFER_EPI  // 0: epilogue right after a tile's last stage (A/B experiments)
#define PZ_TC_DEFER_EPI 1
#endif
constexpr int BM = 256;  // tokens per tile (2 x UMMA M=128)
constexpr int BN = 256;  // output rows per tile (UMMA N=256)
constexpr int BK = 64;   // K per stage (= one 128-byte swizzle row of bf16)
constexpr int kStages = 3;
constexpr int kABytes = BM * BK * 2;  // 32 KB
constexpr int kBBytes = BN * BK * 2;  // 32 KB
constexpr int kStageBytes = kABytes + kBBytes;
constexpr int kDecodeWarps = 8;       // also the epilogue warps (2 per TMEM lane quarter)
constexpr int kThreads = 96 + 32 * kDecodeWarps;  // + warp 10: second MMA issuer
constexpr uint32_t kTmemCols = 512;
constexpr int kMaxBuckets = 2 * 256;

struct alignas(8) SmemCtl {
  int32_t hdr[kStages];  // tile of each stage (-1 = no more work), written by the producer
  int32_t pad_;
  uint64_t full[kStages];
  uint64_t dec[kStages];
  uint64_t empty[kStages];
  uint64_t tmem_full;
  uint64_t tmem_empty[2];  // accumulator of M-block 0 / 1 drained (released one after the other)
  uint32_t tmem_base;
  int32_t n_buckets;
  int32_t bucket_off[kMaxBuckets + 1];
  int32_t mtiles[kMaxBuckets];          // M tiles of each bucket
  int32_t pair_off[kMaxBuckets / 2 + 1];  // first tile of each pair (pair-major tile order)
  uint8_t dense[kMaxBuckets / 2];         // slot holds plain bf16 weights: no decode (R20)
};

constexpr size_t kSmemBytes = 1024 /*align slack*/ + (size_t)kStages * kStageBytes + sizeof(SmemCtl);

struct TileInfo {
  int bucket, m_tile, n_block, row0, valid;
};

// Tile order: pair-major, then n-block, then (pos, m-tile). The CTAs of one wave therefore
// work on a band of n-blocks of ONE pair: the pair's activation rows and that band of its
// packed weight tiles are re-read from L2, not HBM.
__device__ __forceinline__ TileInfo tile_info(const SmemCtl& c, int tile, int n_blocks) {
  TileInfo t;
  int lo = 0, hi = c.n_buckets / 2 - 1;  // last pair with pair_off[p] <= tile
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (c.pair_off[mid] <= tile) lo = mid; else hi = mid - 1;
  }
  const int p = lo;
  const int m0 = c.mtiles[2 * p], m01 = m0 + c.mtiles[2 * p + 1];
  const int rem = tile - c.pair_off[p];
  t.n_block = rem / m01;
  const int r2 = rem - t.n_block * m01;
  t.bucket = 2 * p + (r2 >= m0);
  t.m_tile = r2 >= m0 ? r2 - m0 : r2;
  t.row0 = c.bucket_off[t.bucket] + t.m_tile * BM;
  t.valid = min(BM, c.bucket_off[t.bucket + 1] - t.row0);
  return t;
}

__device__ __forceinline__ uint4 lds128(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}
__device__ __forceinline__ void sts128(uint32_t addr, const uint4& v) {
  asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

// Algorithm 1 in place on one packed B stage (shared-space address `b_tile`): elementwise, so
// the TMA's swizzled layout is preserved. Per 32-bit register (2 words):
//   mag = (w & 0x0FFF0FFF) + 0x57805780   |W^| x 2^63 (exponent e' + 112 + 63, no lane carry)
//   W^  = bf16x2(mag) x bf16x2(w' & 0xA000A000), w' = w (pos 0) or w << 1 (pos 1)
// the sign and mask bits of the position form +-2^-63 or +-0, so one exact bf16x2 multiply
// applies sign, mask and rescale on the FMA pipe (gemv_tc.cu uses the same form).
__device__ __forceinline__ uint32_t bf16x2_mul_tc(uint32_t a, uint32_t b) {
  uint32_t r;
  asm("mul.rn.bf16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}
#ifndef PZ_TC_ORMAG  // 1: |W^| x 2^48 by ORing the exponent offset (one LOP3), tiles hold W^ x 2^-15,
#define PZ_TC_ORMAG 1  //    the epilogue scales packed tiles' accumulators by 2^15 (exact)
#endif
template <int POS>
__device__ __forceinline__ uint32_t dec_word(uint32_t w, uint32_t one, uint32_t two, uint32_t orc) {
#if PZ_TC_ORMAG
  const uint32_t mag = (w & 0x0FFF0FFFu) | orc;  // exponent e' + 160 = e' | 0xA0 (e' < 32)
#else
  (void)orc;
  const uint32_t mag = imad(w & 0x0FFF0FFFu, one, 0x57805780u);
#endif
  return bf16x2_mul_tc(mag, (POS == 0 ? w : imul(w, two)) & 0xA000A000u);
}
template <int POS>
__device__ __forceinline__ void decode_tile(uint32_t b_tile, int tid, uint32_t one) {
  const uint32_t two = one * 2u, orc = one * 0x50005000u;  // orc: a register operand for the LOP3
  constexpr int kPer = kBBytes / 16 / (kDecodeWarps * 32);  // uint4 per thread per stage
  uint4 v[kPer];
#pragma unroll
  for (int j = 0; j < kPer; ++j) v[j] = lds128(b_tile + (uint32_t)(tid + j * kDecodeWarps * 32) * 16u);
#pragma unroll
  for (int j = 0; j < kPer; ++j) {
    v[j].x = dec_word<POS>(v[j].x, one, two, orc);
    v[j].y = dec_word<POS>(v[j].y, one, two, orc);
    v[j].z = dec_word<POS>(v[j].z, one, two, orc);
    v[j].w = dec_word<POS>(v[j].w, one, two, orc);
  }
#pragma unroll
  for (int j = 0; j < kPer; ++j) sts128(b_tile + (uint32_t)(tid + j * kDecodeWarps * 32) * 16u, v[j]);
}

template <bool kW13>
__global__ void __launch_bounds__(kThreads, 1) k_tc_experts(
    const __grid_constant__ CUtensorMap tmap_a,  // X rows (w13) or h rows (w2): [n_rows][K] bf16
    const __grid_constant__ CUtensorMap tmap_b,  // packed w13 [P*2*f][d] or w2 [P*d][f] u16
    const int32_t* __restrict__ bucket_off, int n_buckets, int K, int f, int d, int n_blocks,
    uint16_t* __restrict__ h_out,  // w13: [n_assign][f] bf16
    float* __restrict__ y_out,     // w2:  [n_assign][d] f32
    int32_t* __restrict__ work_ctr,  // zero on entry: tiles are claimed with an atomic
    uint32_t mul_one,              // = 1, opaque to ptxas (keeps decode shifts on the FMA pipe)
    const uint8_t* __restrict__ pair_dense) {  // NULL or [n_buckets / 2]
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  SmemCtl& c = *reinterpret_cast<SmemCtl*>(smem + (size_t)kStages * kStageBytes);
  const uint32_t smem_base = (ptx::smem_u32(smem_raw) + 1023u) & ~1023u;  // shared-window address of smem
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // ---- setup: bucket / tile offsets, barriers, TMEM ----
  pdl_wait();
#ifdef PZ_TRACE
  if (threadIdx.x == 0) g_tcc[kW13][blockIdx.x][0] = tc_gtimer();
#endif
  pdl_trigger();
  for (int i = threadIdx.x; i <= n_buckets; i += blockDim.x) c.bucket_off[i] = bucket_off[i];
  for (int i = threadIdx.x; i < n_buckets / 2; i += blockDim.x) c.dense[i] = pair_dense ? pair_dense[i] : 0;
  __syncthreads();
  if (threadIdx.x == 0) {
    c.n_buckets = n_buckets;
    int run = 0;
    for (int b = 0; b < n_buckets; ++b) c.mtiles[b] = (c.bucket_off[b + 1] - c.bucket_off[b] + BM - 1) / BM;
    for (int p = 0; p < n_buckets / 2; ++p) {
      c.pair_off[p] = run;
      run += n_blocks * (c.mtiles[2 * p] + c.mtiles[2 * p + 1]);
    }
    c.pair_off[n_buckets / 2] = run;
    for (int s = 0; s < kStages; ++s) {
      ptx::mbar_init(&c.full[s], 1);
      ptx::mbar_init(&c.dec[s], kDecodeWarps);
      ptx::mbar_init(&c.empty[s], 2);  // a commit from each MMA issuer
    }
    ptx::mbar_init(&c.tmem_full, 2);
    ptx::mbar_init(&c.tmem_empty[0], kDecodeWarps);
    ptx::mbar_init(&c.tmem_empty[1], kDecodeWarps);
    ptx::fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch_desc(&tmap_a);
    ptx::tma_prefetch_desc(&tmap_b);
  }
  if (warp == 1) ptx::tmem_alloc<kTmemCols>(&c.tmem_base);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = c.tmem_base;
  const int n_tiles = c.pair_off[n_buckets / 2];
  const int nk = K / BK;

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int tcount = 0;
      (void)tcount;
      // tiles are claimed dynamically (their costs differ: ragged M tiles, pairs with one
      // position); the next claim overlaps the current tile's stream
#ifndef PZ_TC_STATIC  // 1: static round-robin tile assignment (A/B experiments)
#define PZ_TC_STATIC 0
#endif
      int next = PZ_TC_STATIC ? (int)blockIdx.x : atomicAdd(work_ctr, 1);
      for (;;) {
        const int tile = next;
        if (tile >= n_tiles) break;
        next = PZ_TC_STATIC ? next + (int)gridDim.x : atomicAdd(work_ctr, 1);
        const TileInfo t = tile_info(c, tile, n_blocks);
        const int pair = t.bucket >> 1;
        for (int kb = 0; kb < nk; ++kb) {
          ptx::mbar_wait(&c.empty[stage], phase ^ 1);
          PZ_TT(0, tcount);
          ++tcount;
          c.hdr[stage] = tile;
          uint8_t* sa = smem + (size_t)stage * kStageBytes;
          uint8_t* sb = sa + kABytes;
          ptx::mbar_arrive_expect_tx(&c.full[stage], kStageBytes);
          ptx::tma_load_2d(sa, &tmap_a, &c.full[stage], kb * BK, t.row0);
          if (kW13) {
            const int gate_row = pair * 2 * f + t.n_block * (BN / 2);
            ptx::tma_load_2d(sb, &tmap_b, &c.full[stage], kb * BK, gate_row);
            ptx::tma_load_2d(sb + kBBytes / 2, &tmap_b, &c.full[stage], kb * BK, gate_row + f);
          } else {
            ptx::tma_load_2d(sb, &tmap_b, &c.full[stage], kb * BK, pair * d + t.n_block * BN);
          }
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
      }
      ptx::mbar_wait(&c.empty[stage], phase ^ 1);  // "no more work": a phase without data
      c.hdr[stage] = -1;
      ptx::mbar_arrive(&c.full[stage]);
    }
  } else if (warp == 1 || warp == 2 + kDecodeWarps) {
    // ===================== MMA issuers =====================
    // warp 1 issues M-block 0's MMAs, the last warp M-block 1's: two instruction streams
    // (one thread's tcgen05.mma retire one after the other; scripts/micro/umma_rate.cu)
    const int mblk = warp == 1 ? 0 : 1;
    constexpr uint32_t idesc = ptx::idesc_bf16_f32(128, BN);
    int stage = 0;
    uint32_t phase = 0, acc_phase = 0;
    int tcount = 0;
    (void)tcount;
    for (;;) {
      ptx::mbar_wait(&c.dec[stage], phase);  // the tile's first stage (or "no more work")
      const int tile = c.hdr[stage];
      if (tile < 0) break;
      const TileInfo t = tile_info(c, tile, n_blocks);
      const bool active = mblk == 0 || t.valid > 128;
      ptx::mbar_wait(&c.tmem_empty[mblk], acc_phase ^ 1);  // this M-block's accumulator drained
      ptx::tc_fence_after();
      for (int kb = 0; kb < nk; ++kb) {
        if (kb) ptx::mbar_wait(&c.dec[stage], phase);
        ptx::tc_fence_after();
        if (lane == 0) {
          const uint32_t sa = ptx::smem_u32(smem + (size_t)stage * kStageBytes) + (uint32_t)(mblk * (kABytes / 2));
          const uint32_t sb = ptx::smem_u32(smem + (size_t)stage * kStageBytes) + kABytes;
          if (active) {
#pragma unroll
            for (int k = 0; k < BK / 16; ++k)
              ptx::mma_bf16_ss(tmem + 256u * mblk, ptx::smem_desc_sw128(sa + k * 32), ptx::smem_desc_sw128(sb + k * 32),
                               idesc, (kb | k) != 0);
          }
          ptx::mma_commit(&c.empty[stage]);  // (an issuer with nothing pending arrives at once)
          if (kb == nk - 1) ptx::mma_commit(&c.tmem_full);
          if (mblk == 0) PZ_TT(2, tcount);
        }
        ++tcount;
        __syncwarp();
        if (++stage == kStages) { stage = 0; phase ^= 1; }
      }
      acc_phase ^= 1;
    }
  } else {
    // ===================== decode warpgroup + epilogue =====================
    const int tid = threadIdx.x - 64;      // 0 .. 32*kDecodeWarps-1
    const int q = warp & 3;                // TMEM lane quarter this warp may access
    const int ch = (warp - 2) >> 2;        // which half of the columns (2 warps per quarter)
    int stage = 0;
    uint32_t phase = 0, acc_phase = 0;
    int tcount = 0, tiles_done = 0;
    (void)tcount;
    (void)tiles_done;
    // ---- epilogue of tile e: drains M-block 0 then 1, releasing each as soon as it is read ----
    auto epilogue = [&](const TileInfo& e) {
      if (threadIdx.x == 64) PZ_TT(3, tiles_done);
      ptx::mbar_wait(&c.tmem_full, acc_phase);
      ptx::tc_fence_after();
      // packed tiles were decoded as W^ x 2^-15 (PZ_TC_ORMAG): exact rescale; dense slots as stored
      const float sc = (PZ_TC_ORMAG && !c.dense[e.bucket >> 1]) ? 32768.0f : 1.0f;
      for (int half = 0; half < 2; ++half) {
        const int m = half * 128 + q * 32 + lane;  // token row within the tile
        const uint32_t tbase = tmem + ((uint32_t)(q * 32) << 16) + half * 256;
        const bool ok = m < e.valid;
        const int64_t a = e.row0 + m;
        if (half == 0 || e.valid > 128) {
          if (kW13) {
            for (int j = ch * 64; j < ch * 64 + 64; j += 32) {
              uint32_t g[32], u[32];
              ptx::tmem_ld_32x32b_x32(tbase + j, g);
              ptx::tmem_ld_32x32b_x32(tbase + 128 + j, u);
              ptx::tmem_ld_wait();
              if (ok) {
                uint32_t pk[16];
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                  const float h0 = silu_mul(__uint_as_float(g[2 * i]) * sc, __uint_as_float(u[2 * i]) * sc);
                  const float h1 = silu_mul(__uint_as_float(g[2 * i + 1]) * sc, __uint_as_float(u[2 * i + 1]) * sc);
                  pk[i] = f32_to_bf16_rne_bits(h0) | (f32_to_bf16_rne_bits(h1) << 16);
                }
                uint4* dst = reinterpret_cast<uint4*>(h_out + a * f + e.n_block * (BN / 2) + j);
#pragma unroll
                for (int i = 0; i < 4; ++i) dst[i] = make_uint4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]);
              }
            }
          } else {
            for (int j = ch * 128; j < ch * 128 + 128; j += 32) {
              uint32_t v[32];
              ptx::tmem_ld_32x32b_x32(tbase + j, v);
              ptx::tmem_ld_wait();
              if (ok) {
                uint4* dst = reinterpret_cast<uint4*>(y_out + a * d + e.n_block * BN + j);
#pragma unroll
                for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) * sc);
#pragma unroll
                for (int i = 0; i < 8; ++i) dst[i] = make_uint4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
              }
            }
          }
        }
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&c.tmem_empty[half]);
      }
      if (threadIdx.x == 64) PZ_TT(4, tiles_done);
      ++tiles_done;
      acc_phase ^= 1;
    };
    TileInfo pend{};
    bool have_pend = false;
    for (;;) {
      ptx::mbar_wait(&c.full[stage], phase);  // the tile's first stage (or "no more work")
      const int tile = c.hdr[stage];
      if (tile < 0) {
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&c.dec[stage]);  // pass the end on to the MMA warp
        break;
      }
      const TileInfo t = tile_info(c, tile, n_blocks);
      const int pos = t.bucket & 1;
      const bool dense = c.dense[t.bucket >> 1] != 0;  // the TMA-loaded words are the bf16 weights
      for (int kb = 0; kb < nk; ++kb) {
        ptx::mbar_wait(&c.full[stage], phase);
        const uint32_t sb = smem_base + (uint32_t)stage * kStageBytes + kABytes;
        if (dense) {
        } else if (pos == 0) {
          decode_tile<0>(sb, tid, mul_one);
        } else {
          decode_tile<1>(sb, tid, mul_one);
        }
        ptx::fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&c.dec[stage]);
        if (threadIdx.x == 64) PZ_TT(1, tcount);
        ++tcount;
        if (++stage == kStages) { stage = 0; phase ^= 1; }
        // the previous tile's epilogue once this tile's first stage is decoded: its last MMAs
        // have completed by then, and this tile's first MMAs (M-block 0) can start as soon as
        // M-block 0 is drained
        if (kb == 0 && have_pend) {
          epilogue(pend);
          have_pend = false;
        }
      }
      pend = t;
      have_pend = true;
      if (!PZ_TC_DEFER_EPI) {
        epilogue(pend);
        have_pend = false;
      }
    }
    if (have_pend) epilogue(pend);
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) ptx::tmem_dealloc<kTmemCols>(tmem);
#ifdef PZ_TRACE
  if (threadIdx.x == 0) g_tcc[kW13][blockIdx.x][1] = tc_gtimer();
#endif
}

}  // namespace

bool tc_supported(int d, int f) { return d % BN == 0 && f % (BN / 2) == 0 && d % BK == 0 && f % BK == 0; }

// x_rows: [n_rows_cap][d] bf16 grouped by bucket; h: [n_rows_cap][f]; y: [n_rows_cap][d]
// work_ctrs: 2 ints, zero on entry (tile claim counters of the w13 and the w2 launch).
// pair_dense: NULL or [n_pairs] device flags (slot holds one unmerged expert's bf16 weights).
int launch_tc_experts(const uint16_t* w13, const uint16_t* w2, const uint8_t* pair_dense, int n_pairs, int d,
                      int f, const uint16_t* x_rows, const int32_t* bucket_off, int64_t n_rows_cap, uint16_t* h,
                      float* y, int32_t* work_ctrs, cudaStream_t stream) {
  if (!tc_supported(d, f)) return fail(PUZZLE_ERR_UNSUPPORTED, "tcgen05 path needs d % 256 == 0 and d_ff % 128 == 0");
  if (n_rows_cap == 0) return PUZZLE_OK;
  static std::atomic<uint64_t> attr13{0}, attr2{0};
  if (int rc = cuda_check(ensure_smem_attr(k_tc_experts<true>, kSmemBytes, attr13), "w13_tc smem attribute")) return rc;
  if (int rc = cuda_check(ensure_smem_attr(k_tc_experts<false>, kSmemBytes, attr2), "w2_tc smem attribute")) return rc;
  CUtensorMap ta13, tb13, ta2, tb2;
  int rc;
  if ((rc = make_tmap_2d(&ta13, x_rows, n_rows_cap, d, BM, BK))) return rc;
  if ((rc = make_tmap_2d(&tb13, w13, (int64_t)n_pairs * 2 * f, d, BN / 2, BK))) return rc;
  if ((rc = make_tmap_2d(&ta2, h, n_rows_cap, f, BM, BK))) return rc;
  if ((rc = make_tmap_2d(&tb2, w2, (int64_t)n_pairs * d, f, BN, BK))) return rc;
  const int grid = num_sms();
  {
    ProfScope _ps("w13_tc", stream);
    cudaError_t e = launch_pdl(k_tc_experts<true>, dim3(grid), dim3(kThreads), kSmemBytes, stream, ta13, tb13,
                               bucket_off, 2 * n_pairs, d, f, d, f / (BN / 2), h, (float*)nullptr, work_ctrs, 1u,
                               pair_dense);
    if (e != cudaSuccess) return cuda_check(e, "w13_tc launch");
  }
  if ((rc = cuda_check(cudaGetLastError(), "w13_tc launch"))) return rc;
  {
    ProfScope _ps("w2_tc", stream);
    cudaError_t e = launch_pdl(k_tc_experts<false>, dim3(grid), dim3(kThreads), kSmemBytes, stream, ta2, tb2,
                               bucket_off, 2 * n_pairs, f, f, d, d / BN, (uint16_t*)nullptr, y, work_ctrs + 1, 1u,
                               pair_dense);
    if (e != cudaSuccess) return cuda_check(e, "w2_tc launch");
  }
  return cuda_check(cudaGetLastError(), "w2_tc launch");
}

}  // namespace pz
