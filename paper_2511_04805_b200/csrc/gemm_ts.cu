// Prefill-shape expert kernels (a4)+(a5), second form: decoded weights as the TMEM A operand,
// tokens on the N side (D[weight rows x tokens] = W^_b[rows, K] . X_b[tokens, K]^T, the
// "swap-AB" orientation of the decode kernels in gemv_tc.cu), W^_b the Algorithm-1 decode
// of the pair's packed words for the bucket's position.
//
// Why (profiles/r02): the shared-memory-operand grouped GEMM (gemm_tc.cu) decodes a 256-row
// weight tile per 256-token M tile, so a bucket of 273 tokens (Qwen1.5 at T = 4096) costs two
// full weight-tile decodes and MMA M-blocks for 17 live rows. Here one work item covers up to
// kNmax tokens of a bucket (N in steps of 32), so a fine-grained bucket is ONE pass over its
// weights, the decoded 128-row stage never goes back through shared memory (tcgen05.st into
// TMEM, the MMA reads it from there), and the packed slot is released as soon as the decoders
// hold the words in registers.
//
// Persistent, one CTA per SM (512 TMEM columns) in clusters of two, 25 warps (72 registers per
// thread). A TMA instruction costs its issuing thread ~165 ns whatever the box size
// (scripts/micro/tma_l2.cu, profiles/r02), so every producer thread issues ONE box per stage:
//   warp 0      W producer: walks the cluster's items (static round robin over clusters; the
//               two CTAs take adjacent row blocks of one token chunk), TMA of each 64-wide K stage of
//               the PACKED 128-row weight tile (w13: one 3-D box = 64 gate + the same features'
//               64 up rows) into a kWStages ring (released by the decoders once read); queues
//               every stage for the X producers and every item for the epilogue
//   warps 1, 2  X producers, one per token half h: the half's token rows (one box of 16..kNH
//               rows, loaded by CTA h of the cluster and multicast into both) into its own
//               kXStages ring (released by both CTAs' half-h MMA commits)
//   warps 3, 4  MMA issuers, one per token half (N = N0 + N1, fixed TMEM column ranges):
//               tcgen05.mma.kind::f16, A = decoded stage in TMEM, B = token rows from smem
//   warps 5-8   decoders: warp q = warp % 4 decodes tile rows 32q..32q+31 of a stage (Algorithm
//               1 as one LOP3 + one exact bf16x2 multiply per 2 words, as in gemv_tc.cu) and
//               stores them with tcgen05.st into A buffer j (of kAStages)
//   warps 9-24  epilogue: drain the accumulators (tcgen05.ld), SwiGLU (w13) or fp32 rows (w2)
//               -> global; two warps per (half, TMEM lane quarter) take alternate 16-column
//               chunks (a half drains in 4.6 us instead of 5.3 with one warp each,
//               profiles/r02/ts_epilogue.txt); each half is released as soon as it is read
// TMEM columns: A buffers [0, 32 kAStages); accumulator half h at kAccCol + kNH h.
// w13 tiles: TMEM lane quarter q = 16 gate rows (features f0 + 16q ..) then the same 16
// features' up rows, so g and u of one d_ff index meet in lanes i, i + 16 of one warp.
#include <cuda.h>

#include <algorithm>
#include <type_traits>

#include "common.cuh"
#include "tc_ptx.cuh"
#include "tmap.cuh"

namespace pz {

#ifdef PZ_TRACE  // per-stage pipeline timeline of CTA PZ_TRACE of the w13 launch (scripts/trace_ts.py)
__device__ unsigned long long g_tst[18][4096];  // 14-17: epilogue internals (see the epilogue)  // 13: decoder reaches stage (before the W wait)
__device__ unsigned long long g_tsc[2][1024][2];  // [kernel][cta] {start after wait, end}
__device__ __forceinline__ unsigned long long ts_gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// 0 W TMA issued, 1 X0 TMA issued, 2 decoder (warp 5) words loaded, 3 decoder A free,
// 4 decoder afull arrived, 5 MMA0 xfull seen, 6 MMA0 afull seen, 7 MMA0 commits issued,
// 8 epilogue accfull[0] seen (per item), 9 epilogue item end (per item), 10 half 0 drained,
// 11 accfull[1] seen, 12 first TMEM load of half 0 landed, 13 half 0 loads done (stores pending)
#define PZ_TS(ev, idx) \
  if (kW13 && blockIdx.x == PZ_TRACE && (idx) < 4096) g_tst[ev][idx] = ts_gtimer()
extern "C" __attribute__((visibility("default"))) int puzzle_debug_ts(void* dst, size_t bytes, void* dst2,
                                                                    size_t bytes2) {
  int rc = (int)cudaMemcpyFromSymbol(dst, g_tst, bytes);
  if (rc) return rc;
  return (int)cudaMemcpyFromSymbol(dst2, g_tsc, bytes2);
}
#else
#define PZ_TS(ev, idx)
#endif

namespace {

constexpr int kBK = 64;                   // K per stage (one 128-byte swizzle row of bf16)
constexpr int kRows = 128;                // weight rows per item (UMMA M)
constexpr int kWBytes = kRows * kBK * 2;  // 16 KB of packed words per stage
#ifndef PZ_TS_NH
#define PZ_TS_NH 192  // max tokens per half (UMMA N <= 256, multiple of 16)
#endif
#ifndef PZ_TS_XST
#define PZ_TS_XST 3
#endif
#ifndef PZ_TS_WST
#define PZ_TS_WST 4
#endif
constexpr int kNH = PZ_TS_NH;
constexpr int kNmax = 2 * kNH;             // tokens per work item (multiple of 32)
constexpr int kXStages = PZ_TS_XST;
constexpr int kWStages = PZ_TS_WST;
constexpr int kXBytes = kNH * kBK * 2;     // token rows of one half-stage
constexpr int kAStages = (512 - 2 * kNH) / 32 > 8 ? 8 : (512 - 2 * kNH) / 32;  // TMEM A buffers (32 columns = 64 k)
constexpr uint32_t kAccCol = 32 * kAStages;
constexpr int kSq = 8;                     // stage queue W producer -> X producer
constexpr int kIq = 4;                     // item queue W producer -> epilogue
#ifndef PZ_TS_DECW
#define PZ_TS_DECW 4  // decoder warps: 4 (each a full 64-wide stage of its 32 rows) or 8 (a K half)
#endif
constexpr int kDecWarps = PZ_TS_DECW;
constexpr int kKH = 8 / kDecWarps;          // K halves per decoder warp
#ifndef PZ_TS_PAIR  // a pair whose two buckets each fit a half (<= kNH tokens) is ONE item: half h
#define PZ_TS_PAIR 1  // = bucket 2p + h, each weight stage streamed and decoded once for both experts
#endif
#ifndef PZ_TS_EPIW
#define PZ_TS_EPIW 16
#endif
// 4 or 8 per accumulator half: one or two per TMEM lane quarter (two split a half's 16-column
// chunks between them, alternately)
constexpr int kEpiWarps = PZ_TS_EPIW;
constexpr int kEpiSplit = kEpiWarps / 8;
constexpr int kThreads = 32 * (5 + kDecWarps + kEpiWarps);
constexpr int kXMaps = kNH / 16;           // X box heights 16, 32, .., kNH rows
constexpr int kW_DEC0 = 5, kW_EPI0 = 5 + kDecWarps;
constexpr int kMaxBuckets = kMaxExperts;
static_assert(kNH % 16 == 0 && kNH <= 256 && kAccCol + 2 * kNH <= 512, "TMEM: A ring + two token halves");

// X tensor maps of every box height, passed by value (kernel parameter space)
struct XMaps {
  CUtensorMap m[kXMaps];
};

struct alignas(16) Ctl {
  int2 whdr[kWStages];  // {item, kb}; item -1 = no more work
  int2 xhdr[2][kXStages];
  int2 sq[kSq];
  int32_t iq[kIq];
  uint64_t wfull[kWStages], wempty[kWStages], xfull[2][kXStages], xempty[2][kXStages];
  uint64_t afull[kAStages], aempty[kAStages], sqfull[kSq], sqempty[kSq], iqfull[kIq], iqempty[kIq];
  uint64_t accfull[2], accempty[2];
  uint32_t tmem_base;
  int32_t n_items;
  int32_t off[kMaxBuckets + 1];          // bucket offsets (bucket-major assignment rows)
  int16_t nch[kMaxBuckets];              // work items (token chunks) of each bucket per row block
  int16_t ncw[kMaxBuckets];              // chunk width (multiple of 32, <= kNmax)
  int32_t pair_off[kMaxBuckets / 2 + 1]; // first item of each pair (pair-major order)
  uint8_t dense[kMaxBuckets / 2];        // slot holds plain bf16 weights: no decode (R20)
  uint8_t paired[kMaxBuckets / 2];       // PZ_TS_PAIR: the pair's two buckets form one item per row block
};

constexpr size_t kSmemBytes = 1024 + (size_t)kWStages * kWBytes + 2 * (size_t)kXStages * kXBytes + sizeof(Ctl);
static_assert(kSmemBytes <= 227 * 1024, "shared memory");

// A work item: row block rb (128 weight rows) of the pair b / 2 and either a token chunk of bucket
// b (its tokens split over the two halves) or, `paired`, both buckets of the pair (half h = bucket
// 2 (b / 2) + h, decoded for its own position). Half h: rows [base_h, base_h + nv_h) of the
// bucket-ordered token rows, MMA width n_h (a multiple of 16 >= nv_h).
struct Item {
  int b, rb, row0, nvalid, n0, n1;
  int base1, nv0, nv1;  // half 1's first row; valid tokens of half 0 / 1 (half 0 starts at row0)
  bool ghost;   // rb >= n_rb: the odd row-block count's spare CTA of a cluster (no outputs)
  bool paired;
};

// Item order: pair-major, then row-block pair, then (position, chunk): the clusters of one wave
// work on a band of row blocks of ONE pair, whose packed tiles and token rows are re-read from
// L2. A cluster item is two adjacent row blocks of one token chunk: CTA `rank` takes 2 rbp + rank.
template <bool kPair>
__device__ __forceinline__ Item item_info(const Ctl& c, int item, int n_pairs, int rank, int n_rb) {
  PZ_DCHECK(item >= 0 && item < c.n_items);
  int lo = 0, hi = n_pairs - 1;  // last pair with pair_off[p] <= item
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (c.pair_off[mid] <= item) lo = mid; else hi = mid - 1;
  }
  const int p = lo;
  const bool paired = kPair && c.paired[p];
  const int c0 = c.nch[2 * p], c01 = paired ? 1 : c0 + c.nch[2 * p + 1];
  const int rem = item - c.pair_off[p];
  Item it;
  const int rbp = rem / c01;
  it.rb = 2 * rbp + rank;
  it.ghost = it.rb >= n_rb;
  it.paired = paired;
  if (paired) {
    it.b = 2 * p;
    it.row0 = c.off[2 * p];
    it.base1 = c.off[2 * p + 1];
    it.nv0 = c.off[2 * p + 1] - c.off[2 * p];
    it.nv1 = c.off[2 * p + 2] - c.off[2 * p + 1];
    it.nvalid = it.nv0 + it.nv1;
    it.n0 = (it.nv0 + 15) & ~15;
    it.n1 = (it.nv1 + 15) & ~15;
    PZ_DCHECK(it.nv0 >= 1 && it.nv1 >= 1 && it.n0 <= kNH && it.n1 <= kNH && it.rb < n_rb + 1);
    return it;
  }
  const int r2 = rem - rbp * c01;
  it.b = 2 * p + (r2 >= c0);
  const int ch = r2 >= c0 ? r2 - c0 : r2;
  const int w = c.ncw[it.b];
  it.row0 = c.off[it.b] + ch * w;
  it.nvalid = min(w, c.off[it.b + 1] - it.row0);
  const int n = (it.nvalid + 31) & ~31;  // MMA width: the live tokens rounded up to 32
  it.n0 = n >> 1;
  it.n1 = n >> 1;
  it.base1 = it.row0 + it.n0;
  it.nv0 = min(it.n0, it.nvalid);
  it.nv1 = it.nvalid - it.nv0;
  PZ_DCHECK(p >= 0 && p < n_pairs && it.b < 2 * n_pairs && it.nvalid >= 1 && it.row0 >= c.off[it.b] &&
            it.row0 + it.nvalid <= c.off[it.b + 1] && n <= kNmax && it.rb < n_rb + 1);
  return it;
}

__device__ __forceinline__ uint4 lds128(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}
__device__ __forceinline__ uint32_t bf16x2_mul(uint32_t a, uint32_t b) {
  uint32_t r;
  asm("mul.rn.bf16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}
// byte offset of (row, 16-byte chunk) inside a 128-byte-swizzled tile with 128-byte rows
__device__ __forceinline__ uint32_t swz(int row, int chunk) {
  return (uint32_t)(row * 128 + ((chunk ^ (row & 7)) << 4));
}

// Every pipeline wait suspends the waiting thread in the mbarrier unit (try_wait with a
// suspend-time hint) instead of spinning: spinning waiters' SYNCS/MIO traffic slowed the
// epilogue's shuffles ~10x (profiles/r02).
#ifndef PZ_TS_SUSPEND_NS
#define PZ_TS_SUSPEND_NS 20000
#endif
__device__ __forceinline__ void mbar_wait_ts(uint64_t* bar, uint32_t parity) {
  if (PZ_TS_SUSPEND_NS > 0) ptx::mbar_wait_sleep(bar, parity, PZ_TS_SUSPEND_NS);
  else ptx::mbar_wait(bar, parity);
}

__device__ __forceinline__ void mbar_arrive_ts(uint64_t* bar) { ptx::mbar_arrive(bar); }

// silu(g) * u = g u / (1 + 2^(-g log2 e)) with the SFU's approximate exp2 and reciprocal (flush
// to zero; ~2 ulp of fp32, far below the bf16 rounding of h that follows)
__device__ __forceinline__ float silu_mul_fast(float g, float u) {
  float e, r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(g * -1.4426950408889634f));
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(1.0f + e));
  return g * r * u;
}
// two fp32 -> bf16x2, round to nearest even (NaN stays NaN), lo in the low half
__device__ __forceinline__ uint32_t f32x2_to_bf16x2_rn(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}

struct Ring {
  int i;
  uint32_t ph;
  template <int N>
  __device__ __forceinline__ void next() {
    if (++i == N) { i = 0; ph ^= 1; }
  }
};

// kPair: paired items (PZ_TS_PAIR) compiled in, with 8 epilogue warps (the pair decode needs the
// registers); without, the kernel is the unpaired form with kEpiWarps epilogue warps
template <bool kPair>
constexpr int ts_epi_warps() { return kPair ? 8 : kEpiWarps; }
template <bool kPair>
constexpr int ts_threads() { return 32 * (5 + kDecWarps + ts_epi_warps<kPair>()); }

template <bool kW13, bool kPair>
__global__ void __launch_bounds__(ts_threads<kPair>(), 1) k_ts_experts(
    const __grid_constant__ CUtensorMap tm_w,  // packed w13 [2P][f][d] (3-D, {64, 64, 2} boxes) / w2 [P*d][f] (128-row boxes)
    const __grid_constant__ XMaps tm_x,        // token rows [n_rows][K] bf16, boxes of 16 (i + 1) rows
    const int32_t* __restrict__ bucket_off, int n_pairs, int K, int f, int d, int n_rb,
    uint16_t* __restrict__ h_out,  // w13: [n_assign][f] bf16
    float* __restrict__ y_out,     // w2:  [n_assign][d] f32
    uint32_t mul_one,                // = 1, opaque to ptxas
    const uint8_t* __restrict__ pair_dense) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t smem_w = (ptx::smem_u32(smem_raw) + 1023u) & ~1023u;
  const uint32_t smem_x = smem_w + kWStages * kWBytes;  // half h, slot j at smem_x + (h kXStages + j) kXBytes
  Ctl& c = *reinterpret_cast<Ctl*>(smem + (size_t)kWStages * kWBytes + 2 * (size_t)kXStages * kXBytes);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_buckets = 2 * n_pairs;
  constexpr int kEW = ts_epi_warps<kPair>(), kES = kEW / 8;  // epilogue warps, chunk streams per quarter

  if (threadIdx.x == 0) {
    for (int s = 0; s < kWStages; ++s) {
      ptx::mbar_init(&c.wfull[s], 1);
      ptx::mbar_init(&c.wempty[s], kDecWarps);
    }
    for (int h = 0; h < 2; ++h)
      for (int s = 0; s < kXStages; ++s) {
        ptx::mbar_init(&c.xfull[h][s], 1);
        ptx::mbar_init(&c.xempty[h][s], 2);  // the (multicast) commits of both CTAs' half-h MMA issuers
      }
    for (int s = 0; s < kAStages; ++s) {
      ptx::mbar_init(&c.afull[s], kDecWarps);
      ptx::mbar_init(&c.aempty[s], 2);
    }
    for (int s = 0; s < kSq; ++s) {
      ptx::mbar_init(&c.sqfull[s], 1);
      ptx::mbar_init(&c.sqempty[s], 2);  // both X producers
    }
    for (int s = 0; s < kIq; ++s) {
      ptx::mbar_init(&c.iqfull[s], 1);
      ptx::mbar_init(&c.iqempty[s], kEW);
    }
    for (int h = 0; h < 2; ++h) {
      ptx::mbar_init(&c.accfull[h], 1);
      ptx::mbar_init(&c.accempty[h], kEW / 2);
    }
    ptx::fence_mbar_init();
    ptx::tma_prefetch_desc(&tm_w);
    for (int i = 0; i < kXMaps; ++i) ptx::tma_prefetch_desc(&tm_x.m[i]);
  }
  if (warp == 3) ptx::tmem_alloc<512>(&c.tmem_base);
  pdl_wait();     // routing / the previous projection complete and visible
  pdl_trigger();
#ifdef PZ_TRACE
  if (threadIdx.x == 0) g_tsc[kW13][blockIdx.x][0] = ts_gtimer();
#endif
  for (int i = threadIdx.x; i <= n_buckets; i += blockDim.x) c.off[i] = bucket_off[i];
  for (int i = threadIdx.x; i < n_pairs; i += blockDim.x) c.dense[i] = pair_dense ? pair_dense[i] : 0;
  __syncthreads();
  for (int i = threadIdx.x; i < n_pairs; i += blockDim.x) {
    const int c0 = c.off[2 * i + 1] - c.off[2 * i], c1 = c.off[2 * i + 2] - c.off[2 * i + 1];
    c.paired[i] = kPair && !c.dense[i] && c0 > 0 && c1 > 0 && c0 <= kNH && c1 <= kNH;
  }
  for (int b = threadIdx.x; b < n_buckets; b += blockDim.x) {  // token chunks of each bucket
    const int cnt = c.off[b + 1] - c.off[b];
    const int nch = (cnt + kNmax - 1) / kNmax;
    c.nch[b] = (int16_t)nch;
    c.ncw[b] = (int16_t)(nch ? ((cnt + nch - 1) / nch + 31) & ~31 : 0);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int run = 0;
    for (int p = 0; p < n_pairs; ++p) {
      c.pair_off[p] = run;
      run += ((n_rb + 1) >> 1) * (c.paired[p] ? 1 : c.nch[2 * p] + c.nch[2 * p + 1]);
    }
    c.pair_off[n_pairs] = run;
    c.n_items = run;
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  ptx::cluster_sync();  // both CTAs' barriers exist before any multicast load / commit reaches them
  const uint32_t tmem = c.tmem_base;
  const int nk = K / kBK;
  const int n_items = c.n_items;
  const int rank = (int)ptx::cluster_ctarank(), cluster = blockIdx.x >> 1, n_clusters = gridDim.x >> 1;

  if (warp == 0) {
    // ============================== W producer ==============================
    if (lane == 0) {
      Ring w{0, 0}, sq{0, 0}, iq{0, 0};
      int tw = 0;
      (void)tw;
      // static round robin over the clusters (both CTAs of a cluster walk the same items)
      for (int item = cluster; item < n_items; item += n_clusters) {
        mbar_wait_ts(&c.iqempty[iq.i], iq.ph ^ 1);
        c.iq[iq.i] = item;
        ptx::mbar_arrive(&c.iqfull[iq.i]);
        iq.next<kIq>();
        const Item it = item_info<kPair>(c, item, n_pairs, rank, n_rb);
        const int pair = it.b >> 1;
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait_ts(&c.wempty[w.i], w.ph ^ 1);
          PZ_TS(0, tw);
          ++tw;
          c.whdr[w.i] = make_int2(item, kb);
          uint8_t* sw = smem + (size_t)w.i * kWBytes;
          ptx::mbar_arrive_expect_tx(&c.wfull[w.i], kWBytes);
          if (kW13)  // 64 gate rows, then the same features' 64 up rows: one 3-D box
            ptx::tma_load_3d(sw, &tm_w, &c.wfull[w.i], kb * kBK, it.rb * (kRows / 2), 2 * pair);
          else
            ptx::tma_load_2d(sw, &tm_w, &c.wfull[w.i], kb * kBK, pair * d + it.rb * kRows);
          w.next<kWStages>();
          mbar_wait_ts(&c.sqempty[sq.i], sq.ph ^ 1);
          c.sq[sq.i] = make_int2(item, kb);
          ptx::mbar_arrive(&c.sqfull[sq.i]);
          sq.next<kSq>();
        }
      }
      // "no more work" on every queue
      mbar_wait_ts(&c.wempty[w.i], w.ph ^ 1);
      c.whdr[w.i] = make_int2(-1, 0);
      ptx::mbar_arrive(&c.wfull[w.i]);
      mbar_wait_ts(&c.sqempty[sq.i], sq.ph ^ 1);
      c.sq[sq.i] = make_int2(-1, 0);
      ptx::mbar_arrive(&c.sqfull[sq.i]);
      mbar_wait_ts(&c.iqempty[iq.i], iq.ph ^ 1);
      c.iq[iq.i] = -1;
      ptx::mbar_arrive(&c.iqfull[iq.i]);
    }
  } else if (warp == 1 || warp == 2) {
    // ============================== X producers ==============================
    if (lane == 0) {
      const int half = warp - 1;
      int tx = 0;
      (void)tx;
      Ring sq{0, 0}, x{0, 0};
      int cur = -1;
      Item it{};
      for (;;) {
        mbar_wait_ts(&c.sqfull[sq.i], sq.ph);
        const int2 h = c.sq[sq.i];
        ptx::mbar_arrive(&c.sqempty[sq.i]);
        sq.next<kSq>();
        mbar_wait_ts(&c.xempty[half][x.i], x.ph ^ 1);
        c.xhdr[half][x.i] = h;
        if (h.x < 0) {
          ptx::mbar_arrive(&c.xfull[half][x.i]);
          break;
        }
        if (h.x != cur) {
          cur = h.x;
          it = item_info<kPair>(c, cur, n_pairs, rank, n_rb);
        }
        const int nh = half ? it.n1 : it.n0;
        const int box = nh >> 4;  // one box of exactly nh rows (nh % 16 == 0)
        if (half == 0) PZ_TS(1, tx);
        ++tx;
        uint8_t* sx = smem + (size_t)kWStages * kWBytes + (size_t)(half * kXStages + x.i) * kXBytes;
        // both CTAs of the cluster need this half's token rows: CTA `half` loads them once,
        // multicast into the same slot of both (each CTA expects the bytes on its own barrier)
        ptx::mbar_arrive_expect_tx(&c.xfull[half][x.i], (uint32_t)box * 16 * (kBK * 2));
        if (rank == half)
          ptx::tma_load_2d_multicast(sx, &tm_x.m[box - 1], &c.xfull[half][x.i], h.y * kBK,
                                     kPair ? (half ? it.base1 : it.row0) : it.row0 + half * it.n0, 0x3);
        x.next<kXStages>();
      }
    }
  } else if (warp == 3 || warp == 4) {
    // ============================== MMA issuers ==============================
    const int half = warp - 3;
    int tm_ = 0;
    (void)tm_;
    Ring x{0, 0}, a{0, 0};
    uint32_t accph = 0;
    int cur = -1;
    Item it{};
    const uint32_t acc = tmem + kAccCol + (uint32_t)(kNH * half);
    for (;;) {
      mbar_wait_ts(&c.xfull[half][x.i], x.ph);
      const int2 h = c.xhdr[half][x.i];
      if (h.x < 0) break;
      if (lane == 0) PZ_TS(half ? 10 : 5, tm_);
      if (h.x != cur) {
        cur = h.x;
        it = item_info<kPair>(c, cur, n_pairs, rank, n_rb);
      }
      const int nh = half ? it.n1 : it.n0;
      if (h.y == 0) {
        mbar_wait_ts(&c.accempty[half], accph ^ 1);  // the previous item's half drained
        ptx::tc_fence_after();
      }
      // a paired item's stage fills two A buffers (position 0, position 1): half h reads buffer h
      Ring a1 = a;
      if (kPair && it.paired) a1.next<kAStages>();
      const Ring am = (kPair && it.paired && half) ? a1 : a;
      mbar_wait_ts(&c.afull[am.i], am.ph);
      if (lane == 0) PZ_TS(half ? 11 : 6, tm_);
      ptx::tc_fence_after();
      if (nh > 0) {
        const uint32_t xs = smem_x + (uint32_t)(half * kXStages + x.i) * kXBytes;
        const uint32_t ta = tmem + 32u * am.i;
        const uint32_t idesc = ptx::idesc_bf16_f32(128, (uint32_t)nh);
#pragma unroll
        for (int kk = 0; kk < kBK / 16; ++kk)
          ptx::mma_bf16_ts_elect(acc, ta + 8 * kk, ptx::smem_desc_sw128(xs + 32 * kk), idesc, (h.y | kk) != 0);
      }
      ptx::mma_commit_elect(&c.aempty[a.i]);  // A buffer free once these MMAs complete
      if (kPair && it.paired) ptx::mma_commit_elect(&c.aempty[a1.i]);  // both buffers: two commits each
      ptx::mma_commit_multicast_elect(&c.xempty[half][x.i], 0x3);  // token slot: in both CTAs (multicast reload)
      if (h.y == nk - 1) {
        ptx::mma_commit_elect(&c.accfull[half]);
        accph ^= 1;
      }
      if (lane == 0) PZ_TS(half ? 12 : 7, tm_);
      ++tm_;
      x.next<kXStages>();
      a.next<kAStages>();
      if (kPair && it.paired) a.next<kAStages>();
    }
  } else if (warp < kW_EPI0) {
    // ============================== decoders ==============================
    const int q = warp & 3;          // TMEM lane quarter
    const int kh0 = ((warp - kW_DEC0) >> 2) * kKH;  // first K half of a stage this warp decodes
    // smem row of this thread's tile row: w13 stages hold 64 gate rows then the same features'
    // 64 up rows; lanes 0-15 of quarter q take gate rows 16q.., lanes 16-31 the up rows
    const int srow = kW13 ? (lane < 16 ? 16 * q + lane : 64 + 16 * q + lane - 16) : 32 * q + lane;
    uint32_t w_off[4 * kKH];
#pragma unroll
    for (int i = 0; i < 4 * kKH; ++i) w_off[i] = swz(srow, 4 * kh0 + i);
    const uint32_t lane_tmem = tmem + ((uint32_t)(32 * q) << 16);
    const uint32_t orc = mul_one * 0x50005000u, two = mul_one * 2u;
    Ring w{0, 0}, a{0, 0};
    int cur = -1, mode = 0;
    int td = 0;
    (void)td;
    for (;;) {
      if (warp == kW_DEC0 && lane == 0) PZ_TS(13, td);  // decoder reaches the stage
      mbar_wait_ts(&c.wfull[w.i], w.ph);
      const int2 h = c.whdr[w.i];
      if (h.x < 0) break;
      if (h.x != cur) {
        cur = h.x;
        const Item it = item_info<kPair>(c, cur, n_pairs, rank, n_rb);
        // 0 / 1: packed position, 2: dense slot (pos 0), 3: paired item (both positions)
        mode = (kPair && it.paired) ? 3 : c.dense[it.b >> 1] ? 2 : (it.b & 1);
      }
      const uint32_t st = smem_w + (uint32_t)w.i * kWBytes;
      uint4 v[4 * kKH];
#pragma unroll
      for (int i = 0; i < 4 * kKH; ++i) v[i] = lds128(st + w_off[i]);
      __syncwarp();
      if (warp == kW_DEC0 && lane == 0) PZ_TS(2, td);
      if (lane == 0) mbar_arrive_ts(&c.wempty[w.i]);  // words in registers: the slot may refill
      w.next<kWStages>();
      // decode the stage for one position (MD: 0 / 1 packed position, 2 dense slot) into the next
      // A buffer. The unpaired kernel keeps one copy with the position chosen at run time; the
      // paired one (kPair) instantiates a copy per position -- a paired stage decodes position 0,
      // then position 1 (the words stay in v) -- since a run-time choice costs the selects of all
      // three forms per word (measured: paired Mixtral T 256 0.44 ms specialised, 0.66 not)
      if constexpr (kPair) {
        auto emit = [&](auto mdc) {
          constexpr int MD = decltype(mdc)::value;
          uint32_t dv[kKH][16];  // decoded while the A buffer may still be in use
#pragma unroll
          for (int i = 0; i < 4 * kKH; ++i) {
            const uint32_t xs[4] = {v[i].x, v[i].y, v[i].z, v[i].w};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const uint32_t xw = xs[j];
              // |W^| * 2^48 (exponent field e' + 160 = e' | 0xA0, one LOP3); sign S and mask M of the
              // position form +-2^-63 or +-0: one exact product leaves W^ * 2^-15 (rescaled in the
              // epilogue); dense slots: the bf16 weight * 2^-15 to match
              const uint32_t mag = (xw & 0x0FFF0FFFu) | orc;
              dv[i >> 2][4 * (i & 3) + j] = MD == 2   ? bf16x2_mul(xw, 0x38003800u)
                                            : MD == 0 ? bf16x2_mul(mag, xw & 0xA000A000u)
                                                      : bf16x2_mul(mag, (xw * two) & 0xA000A000u);
            }
          }
          mbar_wait_ts(&c.aempty[a.i], a.ph ^ 1);  // the MMAs that read this A buffer completed
          if (warp == kW_DEC0 && lane == 0) PZ_TS(3, td);
          ptx::tc_fence_after();
#pragma unroll
          for (int k = 0; k < kKH; ++k) ptx::tmem_st_32x32b_x16(lane_tmem + 32u * a.i + 16u * (kh0 + k), dv[k]);
          ptx::tmem_st_wait();
          ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_ts(&c.afull[a.i]);
          a.next<kAStages>();
        };
        using P0 = std::integral_constant<int, 0>;
        using P1 = std::integral_constant<int, 1>;
        if (mode == 3) {
          emit(P0{});
          emit(P1{});
        } else if (mode == 0) {
          emit(P0{});
        } else if (mode == 1) {
          emit(P1{});
        } else {
          emit(std::integral_constant<int, 2>{});
        }
      } else {
        const int MD = mode;
        uint32_t dv[kKH][16];  // decoded while the A buffer may still be in use
#pragma unroll
        for (int i = 0; i < 4 * kKH; ++i) {
          const uint32_t xs[4] = {v[i].x, v[i].y, v[i].z, v[i].w};
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint32_t xw = xs[j];
            // |W^| * 2^48 (exponent field e' + 160 = e' | 0xA0, one LOP3); sign S and mask M of the
            // position form +-2^-63 or +-0: one exact product leaves W^ * 2^-15 (rescaled in the
            // epilogue); dense slots: the bf16 weight * 2^-15 to match
            const uint32_t mag = (xw & 0x0FFF0FFFu) | orc;
            dv[i >> 2][4 * (i & 3) + j] = MD == 2   ? bf16x2_mul(xw, 0x38003800u)
                                          : MD == 0 ? bf16x2_mul(mag, xw & 0xA000A000u)
                                                    : bf16x2_mul(mag, (xw * two) & 0xA000A000u);
          }
        }
        mbar_wait_ts(&c.aempty[a.i], a.ph ^ 1);  // the MMAs that read this A buffer completed
        if (warp == kW_DEC0 && lane == 0) PZ_TS(3, td);
        ptx::tc_fence_after();
#pragma unroll
        for (int k = 0; k < kKH; ++k) ptx::tmem_st_32x32b_x16(lane_tmem + 32u * a.i + 16u * (kh0 + k), dv[k]);
        ptx::tmem_st_wait();
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_ts(&c.afull[a.i]);
        a.next<kAStages>();
      }
      if (warp == kW_DEC0 && lane == 0) PZ_TS(4, td);
      ++td;
    }
  } else {
    // ============================== epilogue ==============================
    // warp (q, half): TMEM lane quarter q of accumulator half `half`; the two halves drain in
    // parallel and are released independently
    const int q = warp & 3;
    const int half = ((warp - kW_EPI0) >> 2) & 1;
    const int part = (warp - kW_EPI0) >> 3;  // which of the quarter's kEpiSplit chunk streams
    const int row = 32 * q + lane;  // tile row == TMEM lane
    const uint32_t acc_t = tmem + ((uint32_t)(32 * q) << 16) + kAccCol + (uint32_t)(kNH * half);
    const bool up = lane >= 16;  // w13: lanes 16-31 hold the up rows of lanes 0-15's features
    Ring iq{0, 0};
    uint32_t accph = 0;
    float sink_ = 0.f;
    (void)sink_;
    int te = 0;
    (void)te;
    for (;;) {
      mbar_wait_ts(&c.iqfull[iq.i], iq.ph);
      const int item = c.iq[iq.i];
      __syncwarp();
      if (lane == 0) mbar_arrive_ts(&c.iqempty[iq.i]);
      iq.next<kIq>();
      if (item < 0) break;
      const Item it = item_info<kPair>(c, item, n_pairs, rank, n_rb);
      const int nh = it.ghost ? 0 : (half ? it.n1 : it.n0);  // a ghost drains nothing
      // this half's first row and valid tokens
      const int hb = kPair ? (half ? it.base1 : it.row0) : it.row0 + half * it.n0;
      const int hv = kPair ? (half ? it.nv1 : it.nv0) : it.nvalid - half * it.n0;
      mbar_wait_ts(&c.accfull[half], accph);
      accph ^= 1;
      if (warp == kW_EPI0 && lane == 0) PZ_TS(8, te);
      if (warp == kW_EPI0 + 4 && lane == 0) PZ_TS(17, te);  // half 1's accumulator seen
      ptx::tc_fence_after();
      auto process = [&](const uint32_t(&v)[16], int c0) {
        if (kW13) {
          // lanes 0-15 hold g, lanes 16-31 u of the same 16 features: each lane sends its partner
          // the half of the 16 tokens it does not finish (gate lanes finish c0..c0+7, up lanes
          // c0+8..c0+15); independent chains per token (shuffles, then SFU math, then stores)
          const int tok0 = c0 + (up ? 8 : 0);  // first token (of this half) this lane finishes
          float gv[8], uv[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float mine = __uint_as_float(up ? v[8 + i] : v[i]);
            const float other = __shfl_xor_sync(0xffffffffu, __uint_as_float(up ? v[i] : v[8 + i]), 16);
            gv[i] = (up ? other : mine) * 32768.0f;  // A = W^ * 2^-15
            uv[i] = (up ? mine : other) * 32768.0f;
          }
          float hf[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) hf[i] = silu_mul_fast(gv[i], uv[i]);
          const int lim = min(min(8, hv - tok0), nh - tok0);
          uint16_t* dst = h_out + (size_t)(hb + tok0) * f + it.rb * (kRows / 2) + 16 * q + (lane & 15);
#pragma unroll
          for (int i = 0; i < 8; i += 2) {
            const uint32_t pk = f32x2_to_bf16x2_rn(hf[i], hf[i + 1]);
#ifdef PZ_TS_NOSTORE  // diagnostic builds only: results discarded
            if (i < lim) sink_ += __uint_as_float(pk);
#else
            if (i < lim) dst[(size_t)i * f] = (uint16_t)(pk & 0xFFFFu);
            if (i + 1 < lim) dst[(size_t)(i + 1) * f] = (uint16_t)(pk >> 16);
#endif
          }
        } else {
          float* dst = y_out + (size_t)(hb + c0) * d + it.rb * kRows + row;  // d_model row
          const int lim = min(min(16, hv - c0), nh - c0);
#pragma unroll
          for (int i = 0; i < 16; ++i) {
#ifdef PZ_TS_NOSTORE
            if (i < lim) sink_ += __uint_as_float(v[i]);
#else
            if (i < lim) dst[(size_t)i * d] = __uint_as_float(v[i]) * 32768.0f;
#endif
          }
        }
      };
      {
      // 16 token columns per step, the next step's TMEM load in flight while this one is
      // processed (nh is a multiple of 16)
      // this warp's chunks: 16 part, 16 part + cs, ... (cs = 16 kEpiSplit)
      uint32_t ra[16], rb[16];
      constexpr int cs = 16 * kES;
      if (16 * part < nh) ptx::tmem_ld_32x32b_x16(acc_t + 16 * part, ra);
      for (int c0 = 16 * part; c0 < nh; c0 += 2 * cs) {
        ptx::tmem_ld_wait();
        if (c0 == 0 && warp == kW_EPI0 && lane == 0) PZ_TS(14, te);  // first TMEM load landed
        if (c0 + cs < nh) ptx::tmem_ld_32x32b_x16(acc_t + c0 + cs, rb);
        process(ra, c0);
        if (c0 + cs >= nh) break;
        ptx::tmem_ld_wait();
        if (c0 + 2 * cs < nh) ptx::tmem_ld_32x32b_x16(acc_t + c0 + 2 * cs, ra);
        process(rb, c0 + cs);
      }
      }
      if (warp == kW_EPI0 && lane == 0) PZ_TS(15, te);      // half 0 (quarter 0) processed
      if (warp == kW_EPI0 + 4 && lane == 0) PZ_TS(16, te);  // half 1 (quarter 0) processed
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_ts(&c.accempty[half]);
#ifdef PZ_TS_NOSTORE
      if (sink_ == 1.2345f) h_out[0] = 0;
#endif
      if (warp == kW_EPI0 && lane == 0) PZ_TS(9, te);
      ++te;
    }
  }
  // every MMA completed (the epilogue waited for the last item) and every tcgen05.ld waited on;
  // no CTA leaves while its peer may still multicast into it or commit to its barriers
  ptx::tc_fence_before();
  __syncthreads();
  ptx::cluster_sync();
  if (warp == 3) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tmem);
  }
#ifdef PZ_TRACE
  if (threadIdx.x == 0) g_tsc[kW13][blockIdx.x][1] = ts_gtimer();
#endif
}

template <bool kPair>
int launch_ts(const uint16_t* w13, const uint16_t* w2, const uint8_t* pair_dense, int n_pairs, int d, int f,
              const uint16_t* x_rows, const int32_t* bucket_off, int64_t n_rows_cap, uint16_t* h, float* y,
              cudaStream_t stream) {
  static std::atomic<uint64_t> attr13{0}, attr2{0};  // per instantiation
  if (int rc = cuda_check(ensure_smem_attr(k_ts_experts<true, kPair>, kSmemBytes, attr13), "w13_ts smem attribute")) return rc;
  if (int rc = cuda_check(ensure_smem_attr(k_ts_experts<false, kPair>, kSmemBytes, attr2), "w2_ts smem attribute")) return rc;
  CUtensorMap tw13, tw2;
  XMaps x13, x2;
  int rc;
  if ((rc = make_tmap_3d(&tw13, w13, (int64_t)n_pairs * 2, f, d, f, kRows / 2, kBK, 2))) return rc;
  if ((rc = make_tmap_2d(&tw2, w2, (int64_t)n_pairs * d, f, kRows, kBK))) return rc;
  for (int i = 0; i < kXMaps; ++i) {
    if ((rc = make_tmap_2d(&x13.m[i], x_rows, n_rows_cap, d, 16 * (i + 1), kBK))) return rc;
    if ((rc = make_tmap_2d(&x2.m[i], h, n_rows_cap, f, 16 * (i + 1), kBK))) return rc;
  }
  const int grid = num_sms() & ~1;  // clusters of 2 CTAs, one CTA per SM
  {
    ProfScope _ps("w13_ts", stream);
    cudaError_t e = launch_pdl_cluster2(k_ts_experts<true, kPair>, dim3(grid), dim3(ts_threads<kPair>()), kSmemBytes, stream, tw13, x13, bucket_off, n_pairs, d, f, d, f / (kRows / 2), h, (float*)nullptr, 1u,
                               pair_dense);
    if (e != cudaSuccess) return cuda_check(e, "w13_ts launch");
  }
  if ((rc = cuda_check(cudaGetLastError(), "w13_ts launch"))) return rc;
  {
    ProfScope _ps("w2_ts", stream);
    cudaError_t e = launch_pdl_cluster2(k_ts_experts<false, kPair>, dim3(grid), dim3(ts_threads<kPair>()), kSmemBytes, stream, tw2, x2, bucket_off, n_pairs, f, f, d, d / kRows, (uint16_t*)nullptr, y, 1u,
                               pair_dense);
    if (e != cudaSuccess) return cuda_check(e, "w2_ts launch");
  }
  return cuda_check(cudaGetLastError(), "w2_ts launch");
}

}  // namespace

bool ts_supported(int d, int f) { return d % kRows == 0 && f % kBK == 0 && d % kBK == 0; }

// x_rows: [n_rows_cap][d] bf16 grouped by bucket; h: [n_rows_cap][f]; y: [n_rows_cap][d];
int launch_ts_experts(const uint16_t* w13, const uint16_t* w2, const uint8_t* pair_dense, int n_pairs, int d, int f,
                      const uint16_t* x_rows, const int32_t* bucket_off, int64_t n_rows_cap, uint16_t* h, float* y,
                      cudaStream_t stream) {
  if (!ts_supported(d, f)) return fail(PUZZLE_ERR_UNSUPPORTED, "prefill TS path needs d_model % 128 == 0 and d_ff % 64 == 0");
  if (n_pairs > kMaxBuckets / 2) return fail(PUZZLE_ERR_UNSUPPORTED, "n_pairs > 256");
  if (n_rows_cap == 0) return PUZZLE_OK;
  // paired items while the buckets average <= 160 tokens (most pairs then have both buckets
  // within a half); profiles/r02/ts_pair_ab.txt
  const bool pair = PZ_TS_PAIR && n_rows_cap <= (int64_t)160 * 2 * n_pairs;
  return pair ? launch_ts<true>(w13, w2, pair_dense, n_pairs, d, f, x_rows, bucket_off, n_rows_cap, h, y, stream)
              : launch_ts<false>(w13, w2, pair_dense, n_pairs, d, f, x_rows, bucket_off, n_rows_cap, h, y, stream);
}


}  // namespace pz
