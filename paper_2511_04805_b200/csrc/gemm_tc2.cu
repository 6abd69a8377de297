// Prefill-shape expert kernels (a4)+(a5) on CTA PAIRS (tcgen05 cta_group::2).
//
// Same grouped GEMM as gemm_tc.cu -- D[tokens, n] = X_b[tokens, K] . W^_b[n, K]^T with W^_b the
// Algorithm-1 decode of a pair's packed words -- but each 256-token x 256-output tile
// is computed by a cluster of two CTAs on two SMs: CTA r holds the tile's token rows
// r*128..r*128+127 (A) and output rows r*128..r*128+127 of the weight tile (B; for w13 rank 0
// holds the 128 gate rows, rank 1 the same features' 128 up rows), and one thread of the even
// CTA issues tcgen05.mma.cta_group::2 (M = 256, N = 256) that reads both CTAs' shared memory.
// Each CTA therefore stages and decodes HALF of the tile per K step (32 KB), so 6 stages fit in
// shared memory (vs 3 for the one-CTA kernel). Measured (scripts/trace_tc2.py): 0.51 us per
// stage = 8.2 TFLOP/s per SM, below the one-CTA kernel's 9.7: per SM and stage the shared
// memory moves 112 KB (TMA 32, in-place decode 32, MMA reads 48 -- each CTA's B half is read by
// both tensor cores), ~112 B/clk, at the shared-memory bandwidth like the one-CTA kernel (same
// 26.7 KB per MFLOP). Kept as the PUZZLE_PREFILL_IMPL=pair option (parity-green).
//
// Per CTA: warp 0 = TMA producer (its A and B halves), warp 1 = MMA issuer (even CTA) / TMEM
// allocation, warps 2-9 = decoders (Algorithm 1 in place on the B half, then arrive on the even
// CTA's dec barrier), warps 10-13 = epilogue (one per TMEM lane quarter: tcgen05.ld of this CTA's
// 128 rows x 256 columns -> SwiGLU / fp32 -> global), so epilogues overlap the next tile's MMAs
// (two 256-column accumulator buffers, all 512 TMEM columns). Commits are multicast to both
// CTAs' barriers.
#include <cuda.h>

#include <mutex>

#include "common.cuh"
#include "tc_ptx.cuh"
#include "tmap.cuh"

namespace pz {

#ifdef PZ_TRACE  // per-stage timeline of cluster 0 (tuning builds only)
__device__ unsigned long long g_t2[2][4][2048];  // [cta rank][event][stage]: 0 TMA issue, 1 decoded, 2 MMA issued, 3 full seen
__device__ __forceinline__ unsigned long long t2_gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define PZ_T2(ev, idx) \
  if (kW13 && (blockIdx.x >> 1) == 0 && (idx) < 2048) g_t2[rank][ev][idx] = t2_gtimer()
extern "C" __attribute__((visibility("default"))) int puzzle_debug_tc2(void* dst, size_t bytes) {
  return (int)cudaMemcpyFromSymbol(dst, g_t2, bytes);
}
#else
#define PZ_T2(ev, idx)
#endif

namespace {

constexpr int BM = 256;  // tokens per tile (128 per CTA)
constexpr int BN = 256;  // output rows per tile (128 per CTA)
constexpr int BK = 64;   // K per stage (one 128-byte swizzle row)
constexpr int kStages = 6;
constexpr int kAB = 128 * BK * 2;  // 16 KB: this CTA's token rows
constexpr int kBB = 128 * BK * 2;  // 16 KB: this CTA's weight rows
constexpr int kStageBytes = kAB + kBB;
constexpr int kDecodeWarps = 8;
constexpr int kEpiWarps = 4;
constexpr int kRelays = 3;  // odd CTA: warps forwarding "stage decoded" to the even CTA, round robin
constexpr int kThreads = 64 + 32 * (kDecodeWarps + kEpiWarps + kRelays - 1);  // relay 0 = warp 1
constexpr uint32_t kTmemCols = 512;  // 2 accumulator buffers x 256 columns
constexpr int kMaxBuckets = 2 * 256;

struct alignas(8) SmemCtl {
  uint64_t full[kStages];     // this CTA's TMA (tx bytes)
  uint64_t dec[kStages];      // even CTA: its decoders + the odd CTA's relay
  uint64_t dloc[kStages];     // odd CTA: its decoders (CTA scope), relayed to the even CTA's dec
  uint64_t empty[kStages];    // every CTA: the MMA's multicast commit
  uint64_t tmem_full[2];      // every CTA: multicast commit after a tile's last MMAs
  uint64_t tmem_empty[2];     // even CTA: the epilogue warps of both CTAs
  alignas(16) uint32_t sig[kStages][4];  // 16-byte scratch: the odd CTA's "decoded" bulk signal
  uint32_t tmem_base;
  int32_t n_buckets;
  int32_t bucket_off[kMaxBuckets + 1];
  int32_t mtiles[kMaxBuckets];
  int32_t pair_off[kMaxBuckets / 2 + 1];
};

constexpr size_t kSmemBytes = 1024 + (size_t)kStages * kStageBytes + sizeof(SmemCtl);
static_assert(kSmemBytes + 1024 <= 228 * 1024, "one CTA per SM");

struct TileInfo {
  int bucket, m_tile, n_block, row0, valid;
};

// pair-major tile list (see gemm_tc.cu): a pair's n-blocks, both positions' M-tiles adjacent
__device__ __forceinline__ TileInfo tile_info(const SmemCtl& c, int tile, int n_blocks) {
  TileInfo t;
  int lo = 0, hi = c.n_buckets / 2 - 1;
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
__device__ __forceinline__ uint32_t bf16x2_mul2(uint32_t a, uint32_t b) {
  uint32_t r;
  asm("mul.rn.bf16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}
// Algorithm 1 for position POS on one 32-bit register (see gemm_tc.cu / gemv_tc.cu)
template <int POS>
__device__ __forceinline__ uint32_t dec_word2(uint32_t w, uint32_t one, uint32_t two) {
  const uint32_t mag = imad(w & 0x0FFF0FFFu, one, 0x57805780u);
  return bf16x2_mul2(mag, (POS == 0 ? w : imul(w, two)) & 0xA000A000u);
}
// in place on this CTA's packed B half (16 KB): 4 uint4 per decoder thread
template <int POS>
__device__ __forceinline__ void decode_half(uint32_t b_tile, int tid, uint32_t one) {
  const uint32_t two = one * 2u;
  constexpr int kPer = kBB / 16 / (kDecodeWarps * 32);
  uint4 v[kPer];
#pragma unroll
  for (int j = 0; j < kPer; ++j) v[j] = lds128(b_tile + (uint32_t)(tid + j * kDecodeWarps * 32) * 16u);
#pragma unroll
  for (int j = 0; j < kPer; ++j) {
    v[j].x = dec_word2<POS>(v[j].x, one, two);
    v[j].y = dec_word2<POS>(v[j].y, one, two);
    v[j].z = dec_word2<POS>(v[j].z, one, two);
    v[j].w = dec_word2<POS>(v[j].w, one, two);
  }
#pragma unroll
  for (int j = 0; j < kPer; ++j) sts128(b_tile + (uint32_t)(tid + j * kDecodeWarps * 32) * 16u, v[j]);
}

template <bool kW13>
__global__ void __launch_bounds__(kThreads, 1) k_tc2_experts(
    const __grid_constant__ CUtensorMap tmap_a,  // X rows (w13) or h rows (w2): [n_rows][K] bf16, box 128 rows
    const __grid_constant__ CUtensorMap tmap_b,  // packed w13 [P*2*f][d] or w2 [P*d][f] u16, box 128 rows
    const int32_t* __restrict__ bucket_off, int n_buckets, int K, int f, int d, int n_blocks,
    uint16_t* __restrict__ h_out,  // w13: [n_assign][f] bf16
    float* __restrict__ y_out,     // w2:  [n_assign][d] f32
    uint32_t mul_one) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  SmemCtl& c = *reinterpret_cast<SmemCtl*>(smem + (size_t)kStages * kStageBytes);
  const uint32_t smem_base = (ptx::smem_u32(smem_raw) + 1023u) & ~1023u;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = ptx::cluster_ctarank();  // 0: issues the MMAs of the pair
  const int cluster = blockIdx.x >> 1, n_clusters = gridDim.x >> 1;

  pdl_wait();
  pdl_trigger();
  for (int i = threadIdx.x; i <= n_buckets; i += blockDim.x) c.bucket_off[i] = bucket_off[i];
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
      ptx::mbar_init(&c.dec[s], kDecodeWarps + 1);  // + the producer's expect_tx (the odd CTA's bulk signal)
      ptx::mbar_init(&c.dloc[s], kDecodeWarps);
      ptx::mbar_init(&c.empty[s], 2);  // a multicast commit from each MMA issuer
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&c.tmem_full[b], 2);
      ptx::mbar_init(&c.tmem_empty[b], 2 * kEpiWarps);
    }
    ptx::fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch_desc(&tmap_a);
    ptx::tma_prefetch_desc(&tmap_b);
  }
  if (warp == 1) ptx::tmem_alloc2<kTmemCols>(&c.tmem_base);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  ptx::cluster_sync();  // both CTAs' barriers exist before any remote arrive / multicast commit
  const uint32_t tmem = c.tmem_base;
  const int n_tiles = c.pair_off[n_buckets / 2];
  const int nk = K / BK;

  if (warp == 0) {
    // ===================== TMA producer (each CTA: its halves) =====================
    if (lane == 0) {
      int stage = 0, tc = 0;
      uint32_t phase = 0;
      for (int tile = cluster; tile < n_tiles; tile += n_clusters) {
        const TileInfo t = tile_info(c, tile, n_blocks);
        const int pair = t.bucket >> 1;
        const int brow = kW13 ? pair * 2 * f + (int)rank * f + t.n_block * (BN / 2)   // gate (0) / up (1) rows
                              : pair * d + t.n_block * BN + (int)rank * (BN / 2);
        for (int kb = 0; kb < nk; ++kb) {
          ptx::mbar_wait(&c.empty[stage], phase ^ 1);
          PZ_T2(0, tc);
          ++tc;
          uint8_t* sa = smem + (size_t)stage * kStageBytes;
          ptx::mbar_arrive_expect_tx(&c.full[stage], kStageBytes);
          if (rank == 0) ptx::mbar_arrive_expect_tx(&c.dec[stage], 16);  // the odd CTA's signal
          ptx::tma_load_2d(sa, &tmap_a, &c.full[stage], kb * BK, t.row0 + (int)rank * 128);
          ptx::tma_load_2d(sa + kAB, &tmap_b, &c.full[stage], kb * BK, brow);
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1 || warp >= 2 + kDecodeWarps + kEpiWarps) {
    // ===================== MMA issuer (even CTA) / relays (odd CTA) =====================
    // The odd CTA forwards "half decoded" to the even CTA's dec barrier as a 16-byte bulk copy
    // completing tx there (non-blocking; a cluster-scope release arrive stalls its thread ~0.8 us),
    // from kRelays threads, stage i by relay i % kRelays.
    const int relay = warp == 1 ? 0 : warp - (2 + kDecodeWarps + kEpiWarps) + 1;
    if (rank == 1 && lane == 0) {
      const int total = max(((n_tiles - cluster + n_clusters - 1) / n_clusters) * nk, 0);
      for (int i = relay; i < total; i += kRelays) {
        ptx::mbar_wait(&c.dloc[i % kStages], (uint32_t)((i / kStages) & 1));  // this CTA's half decoded
        ptx::fence_proxy_async_smem();  // the decoders' writes (acquired via dloc) -> async proxy
        ptx::bulk_signal_cluster(ptx::mapa(&c.sig[i % kStages][0], 0), &c.sig[i % kStages][0], 16,
                                 ptx::mapa(&c.dec[i % kStages], 0));
      }
    }
    // even CTA: two MMA issuers, each N = 128 of the 256-wide tile (B rows 64h..64h+63 of each
    // CTA's half), two instruction streams (one thread's MMAs retire one after another)
    const int issuer = warp == 1 ? 0 : (warp == 2 + kDecodeWarps + kEpiWarps ? 1 : -1);
    if (rank == 0 && issuer >= 0) {
      constexpr uint32_t idesc = ptx::idesc_bf16_f32(2 * 128, BN / 2);
      int stage = 0, buf = 0, tc = 0;
      uint32_t phase = 0, acc_phase = 0;
      (void)tc;
      for (int tile = cluster; tile < n_tiles; tile += n_clusters) {
        ptx::mbar_wait(&c.tmem_empty[buf], acc_phase ^ 1);  // both CTAs drained this buffer
        ptx::tc_fence_after();
        for (int kb = 0; kb < nk; ++kb) {
          ptx::mbar_wait(&c.dec[stage], phase);  // both CTAs' halves loaded and decoded
          ptx::tc_fence_after();
          if (lane == 0) {
            const uint32_t sa = smem_base + (uint32_t)stage * kStageBytes;
            const uint32_t sb = sa + kAB + (uint32_t)issuer * (64 * 128);
#pragma unroll
            for (int k = 0; k < BK / 16; ++k)
              ptx::mma2_bf16_ss(tmem + 256u * buf + 128u * issuer, ptx::smem_desc_sw128(sa + k * 32),
                                ptx::smem_desc_sw128(sb + k * 32), idesc, (kb | k) != 0);
            ptx::mma2_commit_multicast(&c.empty[stage], 0x3);
            if (kb == nk - 1) ptx::mma2_commit_multicast(&c.tmem_full[buf], 0x3);
            if (issuer == 0) PZ_T2(2, tc);
          }
          ++tc;
          __syncwarp();
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
        if (++buf == 2) { buf = 0; acc_phase ^= 1; }
      }
    }
  } else if (warp < 2 + kDecodeWarps) {
    // ===================== decoders (each CTA: its B half) =====================
    const int tid = threadIdx.x - 64;
    const uint32_t one = mul_one;
    int stage = 0, tc = 0;
    uint32_t phase = 0;
    for (int tile = cluster; tile < n_tiles; tile += n_clusters) {
      const int pos = tile_info(c, tile, n_blocks).bucket & 1;
      for (int kb = 0; kb < nk; ++kb) {
        ptx::mbar_wait(&c.full[stage], phase);
        if (threadIdx.x == 64) PZ_T2(3, tc);
        const uint32_t sb = smem_base + (uint32_t)stage * kStageBytes + kAB;
        if (pos == 0) decode_half<0>(sb, tid, one); else decode_half<1>(sb, tid, one);
        ptx::fence_proxy_async_smem();  // generic writes -> the tensor core's (async proxy) reads
        __syncwarp();
        // CTA-scope arrives only: the even CTA's decoders on its dec barrier, the odd CTA's on
        // its local dloc barrier, which its relay thread forwards with one cluster-scope release
        // (a cluster-scope release right after the decode stalls a warp ~0.6 us)
        if (lane == 0) ptx::mbar_arrive(rank == 0 ? &c.dec[stage] : &c.dloc[stage]);
        if (threadIdx.x == 64) PZ_T2(1, tc);
        ++tc;
        if (++stage == kStages) { stage = 0; phase ^= 1; }
      }
    }
  } else {
    // ===================== epilogue (each CTA: its 128 token rows) =====================
    const int q = warp & 3;  // TMEM lane quarter (warps 10..13 cover all four)
    int buf = 0;
    uint32_t acc_phase = 0;
    for (int tile = cluster; tile < n_tiles; tile += n_clusters) {
      const TileInfo t = tile_info(c, tile, n_blocks);
      ptx::mbar_wait(&c.tmem_full[buf], acc_phase);
      ptx::tc_fence_after();
      const int m = (int)rank * 128 + q * 32 + lane;  // token row within the tile
      const bool ok = m < t.valid;
      const int64_t a = t.row0 + m;
      const uint32_t tbase = tmem + ((uint32_t)(q * 32) << 16) + 256u * buf;
      // accumulator columns: issuer h wrote [128h, 128h + 64) = the even CTA's weight rows
      // 64h.. (w13: gate features 64h..) and [128h + 64, 128h + 128) = the odd CTA's rows 64h..
      // (w13: up features 64h..)
      if (kW13) {
        for (int j = 0; j < 128; j += 32) {
          uint32_t g[32], u[32];
          const uint32_t gc = 128u * (j / 64) + (j % 64);
          ptx::tmem_ld_32x32b_x32(tbase + gc, g);
          ptx::tmem_ld_32x32b_x32(tbase + gc + 64, u);
          ptx::tmem_ld_wait();
          if (ok) {
            uint32_t pk[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const float h0 = silu_mul(__uint_as_float(g[2 * i]), __uint_as_float(u[2 * i]));
              const float h1 = silu_mul(__uint_as_float(g[2 * i + 1]), __uint_as_float(u[2 * i + 1]));
              pk[i] = f32_to_bf16_rne_bits(h0) | (f32_to_bf16_rne_bits(h1) << 16);
            }
            uint4* dst = reinterpret_cast<uint4*>(h_out + a * f + t.n_block * (BN / 2) + j);
#pragma unroll
            for (int i = 0; i < 4; ++i) dst[i] = make_uint4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]);
          }
        }
      } else {
        for (int j = 0; j < 256; j += 32) {
          uint32_t v[32];
          ptx::tmem_ld_32x32b_x32(tbase + j, v);
          ptx::tmem_ld_wait();
          if (ok) {
            const int orow = ((j % 128) / 64) * 128 + (j / 128) * 64 + (j % 64);  // output row of column j
            uint4* dst = reinterpret_cast<uint4*>(y_out + a * d + t.n_block * BN + orow);
#pragma unroll
            for (int i = 0; i < 8; ++i) dst[i] = make_uint4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
          }
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive_cluster(ptx::mapa(&c.tmem_empty[buf], 0));
      if (++buf == 2) { buf = 0; acc_phase ^= 1; }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::cluster_sync();  // the even CTA's MMAs read this CTA's shared memory until the last tile
  ptx::tc_fence_after();
  if (warp == 1) ptx::tmem_dealloc2<kTmemCols>(tmem);
}

template <bool kW13>
cudaError_t launch_tc2(int grid, cudaStream_t stream, const CUtensorMap& ta, const CUtensorMap& tb,
                       const int32_t* bucket_off, int n_buckets, int K, int f, int d, int n_blocks, uint16_t* h,
                       float* y) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kSmemBytes;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, k_tc2_experts<kW13>, ta, tb, bucket_off, n_buckets, K, f, d, n_blocks, h, y, 1u);
}

}  // namespace

// Same contract as launch_tc_experts (gemm_tc.cu).
int launch_tc2_experts(const uint16_t* w13, const uint16_t* w2, int n_pairs, int d, int f, const uint16_t* x_rows,
                       const int32_t* bucket_off, int64_t n_rows_cap, uint16_t* h, float* y, cudaStream_t stream) {
  if (d % BN != 0 || f % (BN / 2) != 0 || d % BK != 0 || f % BK != 0)
    return fail(PUZZLE_ERR_UNSUPPORTED, "tcgen05 path needs d % 256 == 0 and d_ff % 128 == 0");
  if (n_rows_cap == 0) return PUZZLE_OK;
  static std::once_flag attr_once;
  std::call_once(attr_once, [] {
    cudaFuncSetAttribute(k_tc2_experts<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes);
    cudaFuncSetAttribute(k_tc2_experts<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes);
    cudaFuncSetAttribute(k_tc2_experts<true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 0);
    cudaFuncSetAttribute(k_tc2_experts<false>, cudaFuncAttributeNonPortableClusterSizeAllowed, 0);
  });
  CUtensorMap ta13, tb13, ta2, tb2;
  int rc;
  if ((rc = make_tmap_2d(&ta13, x_rows, n_rows_cap, d, 128, BK))) return rc;
  if ((rc = make_tmap_2d(&tb13, w13, (int64_t)n_pairs * 2 * f, d, 128, BK))) return rc;
  if ((rc = make_tmap_2d(&ta2, h, n_rows_cap, f, 128, BK))) return rc;
  if ((rc = make_tmap_2d(&tb2, w2, (int64_t)n_pairs * d, f, 128, BK))) return rc;
  const int grid = 2 * (num_sms() / 2);
  {
    ProfScope _ps("w13_tc", stream);
    if ((rc = cuda_check(launch_tc2<true>(grid, stream, ta13, tb13, bucket_off, 2 * n_pairs, d, f, d, f / (BN / 2), h,
                                          nullptr),
                         "w13_tc2 launch")))
      return rc;
  }
  {
    ProfScope _ps("w2_tc", stream);
    if ((rc = cuda_check(launch_tc2<false>(grid, stream, ta2, tb2, bucket_off, 2 * n_pairs, f, f, d, d / BN, nullptr,
                                           y),
                         "w2_tc2 launch")))
      return rc;
  }
  return PUZZLE_OK;
}

}  // namespace pz
