// Decode-shape expert kernels (a4)+(a5) on the 5th-generation tensor cores, weights on the
// M side ("swap-AB"): D[weight rows x tokens] = W^_pos[rows, K] . X_pos[tokens, K]^T, where
// W^_pos is the Algorithm-1 decode of the pair's packed words. Each touched pair's
// packed words are streamed from HBM ONCE and decoded for position 0 and/or 1.
//
// Warp-specialised, persistent CTAs (2 per SM, 256 TMEM columns each):
//   warp 0     W producer: one lane walks the CTA's stream-K range of stages (see StreamK)
//              and issues the TMA loads of each 64-wide K stage of the PACKED 128-row weight
//              tile (2 boxes) into a 4-deep W ring, released by the decoders as soon as they
//              hold the words in registers; every stage is queued for
//   warp 11    X producer: one lane loads the tokens' activation rows of both positions (one
//              32-row box each per pass) into a 5-deep X ring, released by the MMAs' commit.
//              (Two producer threads: each TMA instruction costs its issuing thread tens of
//              ns, and weight loads must never wait behind activation slots.)
//   warps 2-9  decoders: warp (q = warp % 4, kh) owns tile rows 32q..32q+31 (= the TMEM lanes
//              it may access) and K half kh of a stage: 4 x LDS.128 (conflict-free under the
//              swizzle), SWAR Algorithm 1 for the active position(s), tcgen05.st of the bf16
//              rows into TMEM A buffer j (lane = row, column = k pair). After the last stage of
//              a pass they are the epilogue (tcgen05.ld of the fp32 accumulators).
//   warps 1,10 MMA issuers, one per position: tcgen05.mma.kind::f16 (A from TMEM, B = the
//              tokens, N = 16 or 32, from a shared-memory descriptor, accumulators in TMEM);
//              two instruction streams, since one thread's MMAs retire ~57 ns apart at these
//              N (scripts/micro/umma_rate.cu). Commits release the A buffer and the X slot.
// w13: TMEM lane quarter q holds 16 gate rows (features f0+16q ..+15) then the same 16
// features' up rows (the decoders pick the rows from the gate / up halves of the stage), so g
// and u of one d_ff index sit in lanes i and i+16 of ONE warp and SwiGLU needs only a shuffle.
// w2 tile rows: 128 consecutive d_model rows.
// TMEM columns: A buffer j (of 3), position p at 64 j + 32 p (64 bf16 k = 32 columns);
// accumulators of position p at 192 + 32 p (32 fp32 token columns).
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "tc_ptx.cuh"
#include "tmap.cuh"

namespace pz {

namespace {

constexpr int kDecWarps = 8;
// warp 0 W producer, warp 1 MMA (position 0), warps 2..9 decoders, warp 10 MMA (position 1),
// warp 11 X producer
constexpr int kThreads = 128 + 32 * kDecWarps;
constexpr int kBK = 64;                          // K per stage (one 128-byte swizzle row)
constexpr int kRows = 128;                       // weight rows per tile (UMMA M)
constexpr int kWBytes = kRows * kBK * 2;         // 16 KB packed words per stage
#ifndef PZ_TC_DEFER  // decoders drain a pass's accumulators after two stages of the next pass
#define PZ_TC_DEFER 0
#endif
#ifndef PZ_TC_ORMAG  // 1: |W^| * 2^48 with one LOP3 (exponent offset ORed in), accumulators x 2^15
#define PZ_TC_ORMAG 1
#endif
#ifndef PZ_TC_WST  // W ring depth of the decode configuration (tuning knob)
#define PZ_TC_WST 4
#endif
#ifndef PZ_W2_EARLY  // w2: only the X producer waits for w13 (weights stream during w13's tail)
#define PZ_W2_EARLY 1
#endif
#ifndef PZ_TC_XST  // X ring depth of the decode configuration (tuning knob)
#define PZ_TC_XST 5
#endif
constexpr int kSq = 8;       // stage queue W producer -> X producer
constexpr int kMinStages = 8;  // stream-K: minimum stages per CTA

// Configurations (2 CTAs per SM, 256 TMEM columns each): NX = 32 tokens per position per pass
// with 3 TMEM A buffers (decode batches: <= 24 tokens per expert on average), or NX = 64 with 2
// A buffers and shallower rings (intermediate batches: one pass of up to 64 tokens per position
// instead of two passes of 32, each of which streams the pair's weights again).
#ifndef PZ_TC_WST1  // W / X ring depths of the one-CTA-per-SM (NX 128) configuration: 32 KB X slots
// (profiles/r02/nx128_rings_ab.txt: 5 / 4 ahead of 6 / 3, 3 / 5, 4 / 4 by 1-5 %)
#define PZ_TC_WST1 5
#endif
#ifndef PZ_TC_XST1
#define PZ_TC_XST1 4
#endif
#ifndef PZ_TC_WST_Q  // W ring depth of the quantised class (half-size slots)
#define PZ_TC_WST_Q PZ_TC_WST
#endif
template <int NX, int CTAS, int FMT = 0>
struct Cfg {
  static constexpr int kNX = NX;                          // tokens per position per pass (UMMA N <= NX)
  static constexpr int kXPos = NX * kBK * 2;              // one position's activation rows per stage
  static constexpr int kXBytes = 2 * kXPos;               // X stage: both positions
  // W slots: a stage of 128 rows x 64 k -- 16 KB of packed words, or 8 KB of quantised code bytes
  // (a deeper ring of half-size slots, 6 / 8, measured neutral: the quantised class is bound by
  // its decode on the ALU pipe, profiles/r02/quant_forward.txt)
  static constexpr int kWSlot = FMT ? kRows * kBK : kWBytes;
  // decoder warps: 8 per CTA at 2 CTAs per SM; 16 in the one-CTA-per-SM configuration (each
  // decodes a K quarter of a stage instead of a K half: the same 16 decoder warps per SM)
  static constexpr int kDec = CTAS == 1 ? 16 : 8;
  static constexpr int kThreads = 128 + 32 * kDec;
  static constexpr int kKC = 32 / kDec;  // 16-byte chunks (8 packed words) per decoder thread per stage
  static constexpr int kWStages = FMT ? PZ_TC_WST_Q : (NX == 32 ? PZ_TC_WST : CTAS == 1 ? PZ_TC_WST1 : 3);
  static constexpr int kXStages = NX == 32 ? PZ_TC_XST : CTAS == 1 ? PZ_TC_XST1 : 3;
  static_assert(FMT == 0 || CTAS == 2, "the quantised class runs the two-CTA configuration");
  static constexpr int kAStages = NX == 32 ? 3 : 2;  // TMEM A buffers (64 columns: 64 k of both positions)
  static constexpr uint32_t kAccCol = 64 * kAStages;  // accumulators of position p at kAccCol + NX p
  static constexpr uint32_t kTmemCols = CTAS == 2 ? 256 : 512;
  static_assert(kAccCol + 2 * NX <= kTmemCols, "TMEM: A ring + accumulators");
};

#ifdef PZ_TRACE  // pipeline timeline of one CTA (tuning builds only; scripts/trace_gemv.py)
__device__ unsigned long long g_trace[8][4096];
__device__ unsigned long long g_cta[2][1024][4];  // [kernel][cta] {start, first W issue, producer done, end}
__device__ unsigned long long g_after_wait[2][1024];  // [kernel][cta] pdl_wait returned
__device__ unsigned int g_smid[2][1024];
__device__ unsigned long long g_red[2][1024][8];  // [kernel][cta] reducer: {epilogue start, wait start, counter seen, end}
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define PZ_TR(ev, idx) \
  if (kW13 && blockIdx.x == PZ_TRACE && (idx) < 4096) g_trace[ev][idx] = gtimer()
#define PZ_TRD(ev, idx) \
  if (kW13 && blockIdx.x == PZ_TRACE && (idx) < 4096 && threadIdx.x == 64) g_trace[ev][idx] = gtimer()
#else
#define PZ_TR(ev, idx)
#define PZ_TRD(ev, idx)
#endif

// mbarrier waits: a spinning waiter re-issues try_wait (and the loop around it) on the SM's
// issue slots; with a suspend-time hint the hardware parks the thread until the phase
// completes (or the hint expires). Producers / MMA issuers (PZ_TC_SLEEP_ROLES) and decoders
// (PZ_TC_SLEEP_DEC) separately selectable; measured, no gain (profiles/r02/wait_sleep_ab.txt): off.
#ifndef PZ_TC_SLEEP_ROLES
#define PZ_TC_SLEEP_ROLES 0
#endif
#ifndef PZ_TC_SLEEP_DEC
#define PZ_TC_SLEEP_DEC 0
#endif
__device__ __forceinline__ void wait_role(uint64_t* bar, uint32_t parity) {
  if (PZ_TC_SLEEP_ROLES) ptx::mbar_wait_sleep(bar, parity, 20000);
  else ptx::mbar_wait(bar, parity);
}
__device__ __forceinline__ void wait_dec(uint64_t* bar, uint32_t parity) {
  if (PZ_TC_SLEEP_DEC) ptx::mbar_wait_sleep(bar, parity, 20000);
  else ptx::mbar_wait(bar, parity);
}

template <int WST, int XST, int AST>
struct alignas(16) Ctl {
  int4 whdr[WST];  // stage headers (see Pass); item -1 = no more work
  int4 xhdr[XST];
  int4 sq[kSq];         // W producer -> X producer: {k column, row0 | active0 << 28, row1 | ...}
  int4 sqh[kSq];        //   ... and the stage headers
  uint64_t wfull[WST], wempty[WST], xfull[XST], xempty[XST], a_full[AST], a_empty[AST];
  uint64_t sqfull[kSq], sqempty[kSq];
  uint64_t pdone;  // decoders -> X producer: partials of this CTA's first (signalling) piece stored
  uint64_t acc_full, acc_empty;
  uint64_t red_bar;  // reducer: staged partials landed (bulk copies)
  uint32_t tmem_base;
  int s_last;
  int32_t s_off[kMaxExperts + 1];       // bucket_off[0 .. 2P]
  int32_t s_active[kMaxExperts / 2];    // active_pairs[0 .. n_active)
  int32_t s_item[kMaxExperts / 2 + 1];  // first work item of each active pair (prefix sum)
};

template <class C>
constexpr size_t smem_bytes() {
  return 1024 + (size_t)C::kWStages * C::kWSlot + (size_t)C::kXStages * C::kXBytes +
         sizeof(Ctl<C::kWStages, C::kXStages, C::kAStages>);
}
static_assert(2 * (smem_bytes<Cfg<32, 2>>() + 1024) <= 228 * 1024, "decode: two CTAs per SM");
static_assert(2 * (smem_bytes<Cfg<32, 2, 1>>() + 1024) <= 228 * 1024, "decode (quantised): two CTAs per SM");
static_assert(2 * (smem_bytes<Cfg<64, 2>>() + 1024) <= 228 * 1024, "NX 64: two CTAs per SM");
static_assert(smem_bytes<Cfg<128, 1>>() <= 227 * 1024, "NX 128: one CTA per SM");

struct PairTokens {
  int off0, cnt0, off1, cnt1;
};

__device__ __forceinline__ PairTokens load_pair(const int32_t* off, int p) {
  PairTokens pt;
  pt.off0 = off[2 * p];
  pt.off1 = off[2 * p + 1];
  pt.cnt0 = pt.off1 - pt.off0;
  pt.cnt1 = off[2 * p + 2] - pt.off1;
  return pt;
}

__device__ __forceinline__ uint4 lds128(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// 1-D bulk copy global -> this CTA's shared memory, completion on an mbarrier (tx bytes)
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(ptx::smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void st_f32_hint(float* a, float v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(a), "f"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void ptx_sts_f32(uint32_t addr, float v) {
  asm volatile("st.shared.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}
__device__ __forceinline__ float4 ptx_lds_f4(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
  return v;
}
__device__ __forceinline__ void ptx_sts_f4(uint32_t addr, float4 v) {
  asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
}
__device__ __forceinline__ int4 lds_int4(uint32_t addr) {
  int4 v;
  asm volatile("ld.shared.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}

// byte offset of (row, 16-byte chunk) inside a 128-byte-swizzled tile with 128-byte rows
__device__ __forceinline__ uint32_t swz(int row, int chunk) {
  return (uint32_t)(row * 128 + ((chunk ^ (row & 7)) << 4));
}

__device__ __forceinline__ void named_bar_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

struct Muls {
  uint32_t one, two, four, eight;
  uint32_t orc;  // 0x50005000 in a register: LOP3 takes one immediate, the mask is the other
};

__device__ __forceinline__ uint32_t comp(const uint4& v, int j) { return j == 0 ? v.x : j == 1 ? v.y : j == 2 ? v.z : v.w; }

// Exact bf16x2 product (one operand is +-2^k or +-0, no overflow / subnormal): the decode's
// sign and mask application on the FMA pipe instead of the integer ALU.
__device__ __forceinline__ uint32_t bf16x2_mul(uint32_t a, uint32_t b) {
  uint32_t r;
  asm("mul.rn.bf16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}

// Ring cursor: slot index + mbarrier phase parity.
struct Ring {
  int i;
  uint32_t ph;
  template <int N>
  __device__ __forceinline__ void next() {
    if (++i == N) { i = 0; ph ^= 1; }
  }
};

// Stream-K partition: the S = (active pairs x row blocks) x nk stages are cut into G
// contiguous ranges, CTA g taking stages [b_g, b_{g+1}), b_g = ceil(g S / G). A work item
// (pair, row block) that straddles a cut is computed in pieces (one per CTA it spans) whose
// fp32 partials are summed in CTA order by the CTA owning the item's first stage: there the
// piece is the LAST of that CTA's range, while every other piece is the FIRST of its CTA's
// range, finished long before. Those signal with a counter (their X producer thread does the
// fence + atomic, off the decoders' path); the reducer waits for the count at its range end.
struct StreamK {
  int S, G;
  __device__ __forceinline__ int begin(int g) const { return (int)(((int64_t)g * S + G - 1) / G); }
  __device__ __forceinline__ int owner(int s) const { return (int)(((int64_t)s * G) / S); }
};

__device__ __forceinline__ int ld_acquire_gpu(const int32_t* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Work items: for every active pair z, its row blocks x its token passes (npass(z) = passes of
// NX tokens over the larger of its two buckets), pass-minor so that consecutive items share
// their packed weight rows (L2). Stage header {item, base, kb, kb0 << 16 | kb1}: k-block kb of
// the piece [kb0, kb1) of `item`, which covers tokens [base, base + NX) of each position.
struct Pass {
  int item, base, kb0, kb1, rb, p;
  PairTokens pt;
  int n0, n1;  // tokens of position 0 / 1 in this pass (0 .. NX)
};

__device__ __forceinline__ int npass_of(const PairTokens& pt, int nx) {
  return max(1, (max(pt.cnt0, pt.cnt1) + nx - 1) / nx);
}

// item -> (active pair z, row block, pass): binary search over the per-pair item prefix
template <int WST, int XST, int AST>
__device__ __forceinline__ void locate(const Ctl<WST, XST, AST>& c, int n_active, int item, int nx, int& p,
                                      PairTokens& pt, int& rb, int& base) {
  int lo = 0, hi = n_active - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (c.s_item[mid] <= item) lo = mid; else hi = mid - 1;
  }
  p = c.s_active[lo];
  PZ_DCHECK(lo >= 0 && lo < n_active && p >= 0 && item >= c.s_item[lo]);
  pt = load_pair(c.s_off, p);
  const int np = npass_of(pt, nx), rem = item - c.s_item[lo];
  rb = rem / np;
  base = (rem % np) * nx;
}

template <int WST, int XST, int AST>
__device__ __forceinline__ Pass make_pass(const Ctl<WST, XST, AST>& c, int4 h, int n_active, int nx) {
  Pass s;
  s.item = h.x;
  s.kb0 = h.w >> 16;
  s.kb1 = h.w & 0xFFFF;
  locate(c, n_active, h.x, nx, s.p, s.pt, s.rb, s.base);
  s.n0 = min(max(s.pt.cnt0 - s.base, 0), nx);
  s.n1 = min(max(s.pt.cnt1 - s.base, 0), nx);
  return s;
}

// One pass of the decoders over the piece's stages for the active position(s) (MODE bit 0 =
// pos 0, bit 1 = pos 1, bit 2 = pos 0 of a dense slot: the words are the bf16 weights): decode this thread's 32 packed words per stage (16 registers, k =
// 32 kh .. 32 kh + 31 of its row) and store the bf16 rows into the TMEM A buffer: register r
// of chunk i -> column 16 kh + 4 i + r (k pair 32 kh + 8 i + 2 r).
template <int MODE, int KC, int WST, int XST, int AST, class Epi>
__device__ __forceinline__ void decode_pass(Ctl<WST, XST, AST>& c, uint32_t smem_w, uint32_t lane_tmem,
                                            const uint32_t (&w_off)[KC],
                                            int kh, int n_stages, Ring& w, Ring& a, const Muls& mu, int& tcount,
                                            bool kW13, int ep_at, Epi&& epi) {
  const int lane = threadIdx.x & 31;
  (void)tcount;
  (void)kW13;
  for (int kb = 0; kb < n_stages; ++kb) {
    if (kb) wait_dec(&c.wfull[w.i], w.ph);
    PZ_TRD(2, tcount);
    const uint32_t st = smem_w + (uint32_t)w.i * kWBytes;
    uint4 v[KC];
#pragma unroll
    for (int i = 0; i < KC; ++i) v[i] = lds128(st + w_off[i]);
    uint32_t d0[4 * KC], d1[4 * KC];
#pragma unroll
    for (int i = 0; i < KC; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t x = comp(v[i], j);
#if PZ_TC_ORMAG
        // |W^| * 2^48: exponent field e' + 160 = e' | 0xA0 (e' < 32: no carry), ONE LOP3; the
        // 2^-63 of the sign/mask factor leaves W^ * 2^-15, undone (exactly) in the epilogue
        const uint32_t mag = (x & 0x0FFF0FFFu) | mu.orc;
#else
        // |W^| * 2^63: exponent field e' + 112 + 63 (never carries out of a lane)
        const uint32_t mag = imad(x & 0x0FFF0FFFu, mu.one, 0x57805780u);
#endif
        // sign S_i (bit 15) + mask M_i (bit 13) = +-2^-63 or +-0 as bf16: one exact product
        if (MODE & 1) d0[4 * i + j] = bf16x2_mul(mag, x & 0xA000A000u);
        if (MODE & 4) d0[4 * i + j] = PZ_TC_ORMAG ? bf16x2_mul(x, 0x38003800u) : x;  // x 2^-15 (exact)
        // S_j (bit 14) and M_j (bit 12) shifted to bits 15 / 13
        if (MODE & 2) d1[4 * i + j] = bf16x2_mul(mag, imul(x, mu.two) & 0xA000A000u);
      }
    __syncwarp();
    if (lane == 0) ptx::mbar_arrive(&c.wempty[w.i]);  // packed words consumed: the slot may refill
    w.next<WST>();
    wait_dec(&c.a_empty[a.i], a.ph ^ 1);  // the MMAs that read A buffer a.i have completed
    PZ_TRD(3, tcount);
    ptx::tc_fence_after();
    const uint32_t t0 = lane_tmem + 64u * a.i + 4u * KC * kh;
    if constexpr (KC == 4) {
      if (MODE & 5) ptx::tmem_st_32x32b_x16(t0, d0);
      if (MODE & 2) ptx::tmem_st_32x32b_x16(t0 + 32u, d1);
    } else {
      if (MODE & 5) ptx::tmem_st_32x32b_x8(t0, d0);
      if (MODE & 2) ptx::tmem_st_32x32b_x8(t0 + 32u, d1);
    }
    ptx::tmem_st_wait();
    ptx::tc_fence_before();
    __syncwarp();
    if (lane == 0) ptx::mbar_arrive(&c.a_full[a.i]);
    PZ_TRD(4, tcount);
    ++tcount;
    a.next<AST>();
    if (kb == ep_at) epi();  // the previous pass's epilogue, once the tensor pipe has work queued
  }
}

// NEXT-3, the quantised weight class (R21-R23): one byte per merged element, S_i S_j M_i M_j 0 c2
// c1 c0, and an f32 scale per group of 128 columns. Decoded element of position p:
// (-1)^S_p * M_p * bf16_rne(f32(c * scale)) (R23), bit-exact: the 8 magnitudes of the thread's
// group (its 32 k of a stage lie in one group) are formed once per stage with the same f32
// product and RNE, then selected per byte pair with byte permutes (prmt); sign and mask are
// integer ops (no scaling trick: exact for every finite scale).
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
  return r;
}
__device__ __forceinline__ uint32_t bf16x2_of(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
// two code bytes (bits 0-15 of y) -> bf16x2 of position 0 / 1 (MODE bits 0 / 1)
template <int MODE>
__device__ __forceinline__ void qdecode2(uint32_t y, const uint32_t (&L)[4], uint32_t& o0, uint32_t& o1) {
  const uint32_t sel = (y & 0x0303u) * 0x22u + 0x1010u;        // bytes 2(c & 3), 2(c & 3) + 1
  const uint32_t lo = prmt(L[0], L[1], sel), hi = prmt(L[2], L[3], sel);
  const uint32_t m3 = prmt(y << 5, 0u, 0x9988u);                // code bit 2 -> 16-bit lane mask
  const uint32_t mag = (lo & ~m3) | (hi & m3);                   // |W^| as bf16x2
  const uint32_t p = prmt(y, 0u, 0x1404u);                       // byte k -> bits 16k + 8 .. 16k + 15
  if (MODE & 1) o0 = (mag | (p & 0x80008000u)) & prmt(y << 2, 0u, 0x9988u);         // S_i bit 7, M_i bit 5
  if (MODE & 2) o1 = (mag | ((p << 1) & 0x80008000u)) & prmt(y << 3, 0u, 0x9988u);  // S_j bit 6, M_j bit 4
}

// The same two bytes through byte tables and the exact-product sign / mask of the packed words
// (about 2.4x fewer integer-pipe instructions): Tl / Th hold the low / high bytes of the 8
// magnitudes x 2^63, indexed by the code nibble of each byte (bit 3 of the format is 0), and
// (-1)^S * M * 2^-63 is formed from the flag bits as a bf16 factor (S_p -> bit 15, M_p -> bit
// 13: +-2^-63 or +-0), one exact bf16x2 product per position. Exact while every magnitude
// times 2^63 is finite and every non-zero product normal: 2^-126 <= scale <= 2^61 (the
// caller keeps qdecode2 for other groups).
template <int MODE>
__device__ __forceinline__ void qdecode2_tab(uint32_t y, const uint32_t (&Tl)[2], const uint32_t (&Th)[2], uint32_t& o0,
                                            uint32_t& o1) {
  const uint32_t lo = prmt(Tl[0], Tl[1], y), hi = prmt(Th[0], Th[1], y);  // selector nibbles 0 / 2: the codes
  const uint32_t mag = prmt(lo, hi, 0x6240u);                              // bf16x2 |W^| * 2^63
  const uint32_t p = prmt(y, 0u, 0x1404u);  // byte k -> bits 16k + 8 .. 16k + 15: S_i S_j M_i M_j at 15 .. 12
  if (MODE & 1) o0 = bf16x2_mul(mag, p & 0xA000A000u);
  if (MODE & 2) o1 = bf16x2_mul(mag, (p << 1) & 0xA000A000u);
}

template <int MODE, int WST, int XST, int AST, class Epi>
__device__ __forceinline__ void decode_pass_q(Ctl<WST, XST, AST>& c, uint32_t smem_w, uint32_t lane_tmem,
                                              const uint32_t (&w_off)[2], int kh, int n_stages, Ring& w, Ring& a,
                                              const float* __restrict__ row_scales, int kb0, int& tcount, int ep_at,
                                              Epi&& epi) {
  const int lane = threadIdx.x & 31;
  (void)tcount;
  float sc_next = __ldg(row_scales + (kb0 >> 1));  // a group = 2 stages of 64
  for (int kb = 0; kb < n_stages; ++kb) {
    if (kb) wait_dec(&c.wfull[w.i], w.ph);
    const uint32_t st = smem_w + (uint32_t)w.i * (kRows * kBK);  // quantised W slots: 8 KB
    const uint4 v0 = lds128(st + w_off[0]), v1 = lds128(st + w_off[1]);
    const float sc = sc_next;
    if (kb + 1 < n_stages) sc_next = __ldg(row_scales + ((kb0 + kb + 1) >> 1));  // in flight meanwhile
    __syncwarp();
    if (lane == 0) ptx::mbar_arrive(&c.wempty[w.i]);  // bytes in registers: the slot may refill
    w.next<WST>();
    uint32_t d0[16], d1[16];
    const uint32_t words[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
    if (sc >= 0x1p-126f && sc <= 0x1p61f) {  // byte-table decode (exact in this scale range)
      uint32_t L[4];
#pragma unroll
      for (int j = 0; j < 4; ++j)
        L[j] = bf16x2_of(__fmul_rn(__fmul_rn((float)(2 * j), sc), 0x1p63f), __fmul_rn(__fmul_rn((float)(2 * j + 1), sc), 0x1p63f));
      const uint32_t Tl[2] = {prmt(L[0], L[1], 0x6420u), prmt(L[2], L[3], 0x6420u)};
      const uint32_t Th[2] = {prmt(L[0], L[1], 0x7531u), prmt(L[2], L[3], 0x7531u)};
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        qdecode2_tab<MODE>(words[i], Tl, Th, d0[2 * i], d1[2 * i]);
        qdecode2_tab<MODE>(words[i] >> 16, Tl, Th, d0[2 * i + 1], d1[2 * i + 1]);
      }
    } else {  // any other finite scale: integer sign / mask (exact for every scale)
      uint32_t L[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) L[j] = bf16x2_of(__fmul_rn((float)(2 * j), sc), __fmul_rn((float)(2 * j + 1), sc));
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        qdecode2<MODE>(words[i], L, d0[2 * i], d1[2 * i]);
        qdecode2<MODE>(words[i] >> 16, L, d0[2 * i + 1], d1[2 * i + 1]);
      }
    }
    wait_dec(&c.a_empty[a.i], a.ph ^ 1);  // the MMAs that read A buffer a.i have completed
    ptx::tc_fence_after();
    const uint32_t t0 = lane_tmem + 64u * a.i + 16u * kh;
    if (MODE & 1) ptx::tmem_st_32x32b_x16(t0, d0);
    if (MODE & 2) ptx::tmem_st_32x32b_x16(t0 + 32u, d1);
    ptx::tmem_st_wait();
    ptx::tc_fence_before();
    __syncwarp();
    if (lane == 0) ptx::mbar_arrive(&c.a_full[a.i]);
    ++tcount;
    a.next<AST>();
    if (kb == ep_at) epi();
  }
}

// part: 2 slots per CTA ([g][0] = its first piece, [g][1] = its last piece), each
// [2 positions][NX tokens of the pass][128 tile rows] fp32 (w13 rows 0-63 = g, 64-127 = u);
// counters: one per work item, zero on entry.
// FMT 0: packed 16-bit words (Algorithm 1); FMT 1: the quantised byte format (NEXT-3) with
// qscales f32 [weight rows][K / 128].
template <bool kW13, int NX, int CTAS, int FMT = 0>
__global__ void __maxnreg__(80) k_gemv_tc(  // 2 CTAs x 12 warps: 6 warps per SM sub-partition
    const __grid_constant__ CUtensorMap tm_w, const __grid_constant__ CUtensorMap tm_x,
    const int32_t* __restrict__ bucket_off, const int32_t* __restrict__ active_pairs,
    const int32_t* __restrict__ n_active_ptr, int K, int f, int d, int n_rb,
    float* __restrict__ part, int32_t* __restrict__ counters, uint16_t* __restrict__ h_out,
    float* __restrict__ y_out, uint32_t mul_one, int n_bucket_pairs, const uint8_t* __restrict__ pair_dense,
    const float* __restrict__ qscales = nullptr) {
  using C = Cfg<NX, CTAS, FMT>;
  constexpr int kDecWarps = C::kDec;  // (shadows the two-CTA default)
  constexpr int kKC = C::kKC;
  constexpr uint32_t kWStageBytes = C::kWSlot;  // bytes of one W stage (codes: 1 B each)
  constexpr int kWStages = C::kWStages, kXStages = C::kXStages, kXBytes = C::kXBytes, kXPos = C::kXPos;
  constexpr int kSlot = 2 * NX * kRows;  // floats per partial slot
  constexpr uint32_t kRowB = kRows * 4;   // one slot row (a (position, token) of 128 outputs): 512 bytes
  // the reducer stages the partial slots in the idle W / X rings when two slots of the item's
  // active (position, token) rows fit (always at NX = 32); otherwise (wide configurations with
  // many rows) it sums them from L2 directly
  constexpr uint32_t kRing = kWStages * kWStageBytes + kXStages * kXBytes;
  constexpr bool kStagedRed = kRing >= 2u * (2 * NX) * kRowB;
  auto staged_red = [&](int n_rows) { return kStagedRed || 2u * (uint32_t)n_rows * kRowB <= kRing; };
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t smem_w = (ptx::smem_u32(smem_raw) + 1023u) & ~1023u;  // == smem, shared window
  const uint32_t smem_x = smem_w + kWStages * kWStageBytes;
  auto& c = *reinterpret_cast<Ctl<kWStages, kXStages, C::kAStages>*>(smem + (size_t)kWStages * kWStageBytes +
                                                         (size_t)kXStages * kXBytes);
  const uint32_t whdr_s = ptx::smem_u32(&c.whdr[0]), xhdr_s = ptx::smem_u32(&c.xhdr[0]);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kWStages; ++s) {
      ptx::mbar_init(&c.wfull[s], 1);
      ptx::mbar_init(&c.wempty[s], kDecWarps);
    }
    for (int j = 0; j < kXStages; ++j) {
      ptx::mbar_init(&c.xfull[j], 1);
      ptx::mbar_init(&c.xempty[j], 2);  // commits of both MMA warps
    }
    for (int j = 0; j < C::kAStages; ++j) {
      ptx::mbar_init(&c.a_full[j], kDecWarps);
      ptx::mbar_init(&c.a_empty[j], 2);
    }
    for (int j = 0; j < kSq; ++j) {
      ptx::mbar_init(&c.sqfull[j], 1);
      ptx::mbar_init(&c.sqempty[j], 1);
    }
    ptx::mbar_init(&c.pdone, kDecWarps);
    ptx::mbar_init(&c.acc_full, 2);
    ptx::mbar_init(&c.acc_empty, kDecWarps);
    ptx::mbar_init(&c.red_bar, 1);
    ptx::fence_mbar_init();
    ptx::tma_prefetch_desc(&tm_w);
    ptx::tma_prefetch_desc(&tm_x);
  }
#ifdef PZ_TRACE
  if (threadIdx.x == 0) g_cta[kW13][blockIdx.x][0] = gtimer();
#endif
  if (warp == 1) ptx::tmem_alloc<C::kTmemCols>(&c.tmem_base);
  // w13 reads the routing tables below: wait for the route kernel. w2 (PZ_W2_EARLY) only waits
  // in its X producer, before the first load of h (the one input w13 writes): its weight stream,
  // decode and TMEM A buffers fill during w13's tail. The routing tables are complete by then:
  // this grid launches only once every w13 CTA has passed its own wait (route complete) and
  // triggered; they are read through L2 (__ldcg). Partial slots (shared with w13) are written
  // only after an MMA, i.e. after that wait.
  if (kW13 || !PZ_W2_EARLY) pdl_wait();
#ifdef PZ_TRACE
  if (threadIdx.x == 0) {
    g_after_wait[kW13][blockIdx.x] = gtimer();
    unsigned int smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    g_smid[kW13][blockIdx.x] = smid;
  }
#endif
  pdl_trigger();  // the next kernel may begin its prologue as CTAs of this one retire
  // routing tables in one round trip (all P slots of active_pairs, whatever n_active is; this
  // setup is on w13's critical path: ~4 us from the wait to the first weight load before)
  for (int i = threadIdx.x; i <= 2 * n_bucket_pairs; i += blockDim.x) c.s_off[i] = __ldcg(bucket_off + i);
  for (int i = threadIdx.x; i < n_bucket_pairs; i += blockDim.x) c.s_active[i] = __ldcg(active_pairs + i);
  const int n_active = __ldcg(n_active_ptr);
  __syncthreads();
  if (warp == 0) {  // work items per active pair (row blocks x token passes): warp prefix sum
    int run = 0;
    for (int z0 = 0; z0 < n_active; z0 += 32) {
      const int z = z0 + lane;
      const int own = z < n_active ? n_rb * npass_of(load_pair(c.s_off, c.s_active[z]), NX) : 0;
      int v = own;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += t;
      }
      if (z < n_active) c.s_item[z] = run + v - own;
      run += __shfl_sync(0xffffffffu, v, 31);
    }
    if (lane == 0) c.s_item[n_active] = run;
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = c.tmem_base;
  const int nk = K / kBK;
  StreamK sk;
  sk.S = c.s_item[n_active] * nk;
  sk.G = max(1, min((int)gridDim.x, sk.S / kMinStages));  // >= kMinStages stages per CTA
  const int g = blockIdx.x;
  const int s_begin = g < sk.G ? sk.begin(g) : 0, s_end = g < sk.G ? sk.begin(g + 1) : 0;

  if (warp == 0) {
    // ============================== W producer ==============================
    // walks this CTA's stage range piece by piece (a piece = the part of one work item in the
    // range), pass by pass: one TMA stage of packed words per free W slot; each stage is also
    // queued (sq) for the X producer
    if (lane != 0) return;
    Ring w{0, 0}, sq{0, 0};
    int tw = 0;
    (void)tw;
    for (int s0 = s_begin; s0 < s_end;) {
      const int item = s0 / nk, kb0 = s0 % nk, kb1 = min(nk, kb0 + (s_end - s0));
      s0 += kb1 - kb0;
      int p, rb, base;
      PairTokens pt;
      locate(c, n_active, item, NX, p, pt, rb, base);
      const int wrow = kW13 ? p * 2 * f + rb * (kRows / 2) : p * d + rb * kRows;
      {
        // X-side parameters: one activation box per active position (flag in bit 28)
        const int r0 = (pt.off0 + base) | ((pt.cnt0 > base) << 28);
        const int r1 = (pt.off1 + base) | ((pt.cnt1 > base) << 28);
        for (int kb = kb0; kb < kb1; ++kb) {
          const int kc = kb * kBK;
          const int4 hv = make_int4(item, base, kb, (kb0 << 16) | kb1);
          wait_role(&c.wempty[w.i], w.ph ^ 1);
          PZ_TR(0, tw);
#ifdef PZ_TRACE
          if (tw == 0) g_cta[kW13][blockIdx.x][1] = gtimer();
#endif
          c.whdr[w.i] = hv;
          uint8_t* sw = smem + (size_t)w.i * kWStageBytes;
          ptx::mbar_arrive_expect_tx(&c.wfull[w.i], kWStageBytes);
          if (kW13) {  // 64 gate rows, then the same features' 64 up rows
            ptx::tma_load_2d(sw, &tm_w, &c.wfull[w.i], kc, wrow);
            ptx::tma_load_2d(sw + kWStageBytes / 2, &tm_w, &c.wfull[w.i], kc, wrow + f);
          } else {
            ptx::tma_load_2d(sw, &tm_w, &c.wfull[w.i], kc, wrow);
          }
          w.next<kWStages>();
          ++tw;
          wait_role(&c.sqempty[sq.i], sq.ph ^ 1);
          c.sqh[sq.i] = hv;
          c.sq[sq.i] = make_int4(kc, r0, r1, 0);
          ptx::mbar_arrive(&c.sqfull[sq.i]);
          sq.next<kSq>();
        }
      }
    }
#ifdef PZ_TRACE
    g_cta[kW13][blockIdx.x][2] = gtimer();
#endif
    // "no more work": complete one more phase of the W ring and the queue without data
    wait_role(&c.wempty[w.i], w.ph ^ 1);
    c.whdr[w.i] = make_int4(-1, 0, 0, 0);
    ptx::mbar_arrive(&c.wfull[w.i]);
    wait_role(&c.sqempty[sq.i], sq.ph ^ 1);
    c.sqh[sq.i] = make_int4(-1, 0, 0, 0);
    ptx::mbar_arrive(&c.sqfull[sq.i]);
    return;
  }

  if (warp == 3 + kDecWarps) {
    // ============================== X producer ==============================
    // the activation rows of each queued stage into the next free X slot
    if (lane != 0) return;
    Ring sq{0, 0}, x{0, 0};
    int tx = 0;
    (void)tx;
    if (!kW13 && PZ_W2_EARLY) {
      pdl_wait();  // h (w13's output) complete and visible
#ifdef PZ_TRACE
      g_after_wait[kW13][blockIdx.x] = gtimer();
#endif
    }
    // this CTA's first piece signals its item's reducer when the item is split and started
    // in an earlier CTA's range
    int sig_item = s_begin < s_end && s_begin % nk != 0 ? s_begin / nk : -1;
    if (sig_item >= 0) {  // (an active pair always has rows; an empty one would never signal)
      int p, rb, base;
      PairTokens pt;
      locate(c, n_active, sig_item, NX, p, pt, rb, base);
      if (max(pt.cnt0, pt.cnt1) <= base) sig_item = -1;
    }
    bool signalled = sig_item < 0;
    auto signal = [&]() {
      // release at gpu scope, cumulative over the decoders' partial stores (acquired via
      // pdone); a reduction, not an atomic with a return value: the thread does not wait for
      // the round trip (it must keep the X ring fed)
      asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(&counters[sig_item]), "r"(1) : "memory");
      signalled = true;
    };
    for (;;) {
      if (!signalled && ptx::mbar_test(&c.pdone, 0)) signal();
      wait_role(&c.sqfull[sq.i], sq.ph);
      const int4 h = c.sqh[sq.i];
      const int4 q = c.sq[sq.i];
      ptx::mbar_arrive(&c.sqempty[sq.i]);
      sq.next<kSq>();
      wait_role(&c.xempty[x.i], x.ph ^ 1);
      c.xhdr[x.i] = h;
      if (h.x < 0) {
        ptx::mbar_arrive(&c.xfull[x.i]);  // "no more work"
        break;
      }
      if (!signalled && ptx::mbar_test(&c.pdone, 0)) signal();
      PZ_TR(1, tx);
      ++tx;
      const bool a0 = (q.y >> 28) & 1, a1 = (q.z >> 28) & 1;
      uint8_t* sx = smem + (size_t)kWStages * kWStageBytes + (size_t)x.i * kXBytes;
      ptx::mbar_arrive_expect_tx(&c.xfull[x.i], (uint32_t)(a0 + a1) * kXPos);
      if (a0) ptx::tma_load_2d(sx, &tm_x, &c.xfull[x.i], q.x, q.y & 0x0FFFFFFF);
      if (a1) ptx::tma_load_2d(sx + kXPos, &tm_x, &c.xfull[x.i], q.x, q.z & 0x0FFFFFFF);
      x.next<kXStages>();
    }
    if (!signalled) {
      ptx::mbar_wait(&c.pdone, 0);
      signal();
    }
    return;
  }

  if (warp == 1 || warp == 2 + kDecWarps) {
    // ============================== MMA issuers ==============================
    // warp 1 issues position 0's MMAs, warp 10 position 1's: two instruction streams, since
    // one thread's tcgen05.mma retire ~57 ns apart at these N (scripts/micro/umma_rate.cu)
    const int mypos = warp == 1 ? 0 : 1;
    Ring x{0, 0}, a{0, 0};
    uint32_t accph = 0;
    int tcount = 0;
    (void)tcount;
    for (;;) {
      wait_role(&c.xfull[x.i], x.ph);
      const int4 h = lds_int4(xhdr_s + 16u * x.i);
      if (h.x < 0) break;
      const Pass s = make_pass(c, h, n_active, NX);
      const int np = mypos ? s.n1 : s.n0;
      const uint32_t idp = ptx::idesc_bf16_f32(128, (uint32_t)((np + 15) & ~15));
      const uint32_t acc_col = tmem + C::kAccCol + (uint32_t)NX * mypos;
      wait_role(&c.acc_empty, accph ^ 1);  // the previous pass's epilogue drained TMEM
      ptx::tc_fence_after();
      for (int kb = s.kb0; kb < s.kb1; ++kb) {
        if (kb != s.kb0) wait_role(&c.xfull[x.i], x.ph);
        if (mypos == 0) PZ_TR(6, tcount);
        wait_role(&c.a_full[a.i], a.ph);
        if (mypos == 0) PZ_TR(5, tcount);
        ptx::tc_fence_after();
        const uint32_t xs = smem_x + (uint32_t)x.i * kXBytes + (uint32_t)(kXPos * mypos);
        const uint32_t ta = tmem + 64u * a.i + 32u * mypos;
        if (np > 0) {
#pragma unroll
          for (int kk = 0; kk < kBK / 16; ++kk)
            ptx::mma_bf16_ts_elect(acc_col, ta + 8 * kk, ptx::smem_desc_sw128(xs + 32 * kk), idp,
                                   (kb != s.kb0) | (kk != 0));
        }
        ptx::mma_commit_elect(&c.a_empty[a.i]);  // A buffer free once these MMAs complete
        ptx::mma_commit_elect(&c.xempty[x.i]);   // X slot likewise
        if (kb == s.kb1 - 1) ptx::mma_commit_elect(&c.acc_full);
        if (mypos == 0) PZ_TR(7, tcount);
        ++tcount;
        x.next<kXStages>();
        a.next<C::kAStages>();
      }
      accph ^= 1;
    }
  } else {
    // ============================== decoders + epilogue ==============================
    const int dtid = threadIdx.x - 64;
    const int q = warp & 3;          // TMEM lane quarter this warp may access
    const int kh = (warp - 2) >> 2;  // K half (quarter: 16 decoders) of a stage
    const int row = 32 * q + lane;   // tile row == TMEM lane
    // shared-memory row this thread decodes. w13: the stage holds 64 gate rows then the same
    // features' 64 up rows; lanes 0-15 of quarter q take gate rows 16q.., lanes 16-31 the up
    // rows of the same features, so g and u of one d_ff index land in lanes i, i+16 of one warp
    const int srow = kW13 ? (lane < 16 ? 16 * q + lane : 64 + 16 * q + lane - 16) : row;
    // partial-slot row of this thread: w13 g rows 0-63 / u rows 64-127 by feature, w2 the tile row
    const int prow = kW13 ? (lane < 16 ? 16 * q + lane : 64 + 16 * q + lane - 16) : row;
    const uint32_t lane_tmem = tmem + ((uint32_t)(32 * q) << 16);
    const Muls mu{mul_one, mul_one * 2u, mul_one * 4u, mul_one * 8u, mul_one * 0x50005000u};
    uint32_t w_off[kKC];
#pragma unroll
    for (int i = 0; i < kKC; ++i) w_off[i] = swz(srow, kKC * kh + i);
    // quant stages: 64-byte rows under the 64-byte swizzle (16-byte chunk c of row r at chunk
    // c ^ ((r >> 1) & 3)); this thread reads chunks 2 kh, 2 kh + 1 (its 32 k)
    uint32_t wq_off[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) wq_off[i] = (uint32_t)(srow * 64 + (((2 * kh + i) ^ ((srow >> 1) & 3)) << 4));
    (void)wq_off;
    Ring w{0, 0}, a{0, 0};
    uint32_t accph = 0;
    int tcount = 0;
    const int first_item = s_begin / nk;  // pieces of this CTA: [g][0] = first, [g][1] = last
    // ---- epilogue of pass s: warp (q, pos = kh) reads its rows' accumulators ----
    auto finish = [&](const Pass& s) {
#ifdef PZ_TRACE
      if (dtid == 0 && !(s.kb0 == 0 && s.kb1 == nk) && g == sk.owner(s.item * nk)) g_red[kW13][blockIdx.x][0] = gtimer();
#endif
      wait_dec(&c.acc_full, accph);
      accph ^= 1;
      ptx::tc_fence_after();
      const bool whole = s.kb0 == 0 && s.kb1 == nk;  // the item is not split: final outputs
      const bool reducer = !whole && g == sk.owner(s.item * nk);  // the item's first piece: this CTA sums
      // warp (q, kh): position kh & 1; with 16 decoders, token chunks of 16 alternate between
      // the warps kh and kh + 2
      const int pos = kh & 1;
      const int np = pos ? s.n1 : s.n0;
      const int offp = (pos ? s.pt.off1 : s.pt.off0) + s.base;  // first assignment of this warp
      float* slot = part + (size_t)(2 * g + (s.item == first_item ? 0 : 1)) * kSlot;
      const uint32_t acc_t = lane_tmem + C::kAccCol + (uint32_t)NX * pos;
      PZ_DCHECK(np >= 0 && np <= NX && offp >= 0 && (np == 0 || offp + np <= c.s_off[2 * n_bucket_pairs]));
      PZ_DCHECK(s.item < n_rb * (n_bucket_pairs + c.s_off[2 * n_bucket_pairs] / 32 + 1));
      // the A operand is W^ * 2^-15 (PZ_TC_ORMAG; dense slots scaled to match): scale back, exact
      constexpr float acc_scale = (PZ_TC_ORMAG && FMT == 0) ? 32768.0f : 1.0f;  // quant bytes decode exactly
      for (int c0 = 16 * (kh >> 1); c0 < np; c0 += 16 * (kDecWarps / 8)) {
        uint32_t r[16];
        ptx::tmem_ld_32x32b_x16(acc_t + c0, r);
        ptx::tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 16; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * acc_scale);
        if (!whole && reducer && staged_red(s.n0 + s.n1)) {
          // the reducer's own piece (the sum's first term): straight into staged slot 0 of the
          // W ring -- idle now: every stage was decoded before the MMAs completed
          const uint32_t a0 = smem_w + (uint32_t)((pos ? s.n0 : 0) + c0) * kRowB + (uint32_t)prow * 4u;
#pragma unroll
          for (int i = 0; i < 16; ++i)
            if (c0 + i < np) ptx_sts_f32(a0 + (uint32_t)i * kRowB, __uint_as_float(r[i]));
        } else if (!whole) {
          // evict_last: the reducer reads these back up to a whole range later, after hundreds
          // of MB of weights have streamed through L2; from HBM, behind the weight stream's
          // queues, that read took ~5 us (scripts/red_stats.py)
          const uint64_t keep = l2_policy_evict_last();
          const int t0 = pos * NX + c0;  // (position, token of the pass)
#pragma unroll
          for (int i = 0; i < 16; ++i)
            if (c0 + i < np) st_f32_hint(slot + (size_t)(t0 + i) * kRows + prow, __uint_as_float(r[i]), keep);
        } else if (kW13) {
          // exchange g <-> u with the partner lane; gate lanes finish tokens c0..c0+7,
          // up lanes tokens c0+8..c0+15
          const bool up = lane >= 16;
          const int feat = s.rb * (kRows / 2) + 16 * q + (lane & 15);  // d_ff index of this row
          PZ_DCHECK(feat < f);
          float o[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) o[i] = __shfl_xor_sync(0xffffffffu, __uint_as_float(r[i]), 16);
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const float gv = up ? o[8 + j] : __uint_as_float(r[j]);
            const float uv = up ? __uint_as_float(r[8 + j]) : o[j];
            const int tok = c0 + (up ? 8 : 0) + j;
            if (tok < np) h_out[(size_t)(offp + tok) * f + feat] = f32_to_bf16_bits_rn(silu_mul(gv, uv));
          }
        } else {
          const int r_out = s.rb * kRows + row;  // d_model row (the last block may overhang d)
          if (r_out < d) {
#pragma unroll
            for (int i = 0; i < 16; ++i)
              if (c0 + i < np) y_out[(size_t)(offp + c0 + i) * d + r_out] = __uint_as_float(r[i]);
          }
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&c.acc_empty);

      if (!whole) {  // a split piece
        const int g_first = sk.owner(s.item * nk), g_last = sk.owner(s.item * nk + nk - 1);
        if (g != g_first) {
          // a signalling piece: the X producer publishes it (fence + counter)
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(&c.pdone);
        } else {
          // the reducer (this CTA's last piece): wait for the other pieces' signals, then sum
          // the partials in CTA order (own slot included)
#ifdef PZ_TRACE
          if (dtid == 0) g_red[kW13][blockIdx.x][1] = gtimer();
#endif
          named_bar_sync(1, kDecWarps * 32);
          if (dtid == 0) {
            while (ld_acquire_gpu(&counters[s.item]) < g_last - g_first) __nanosleep(64);
            counters[s.item] = 0;  // ready for the next call on this stream
#ifdef PZ_TRACE
            g_red[kW13][blockIdx.x][2] = gtimer();
#endif
          }
          named_bar_sync(1, kDecWarps * 32);
          // Sum the slots of CTAs g_first .. g_last in CTA order (from 0). The active rows of
          // every slot are staged into the idle W / X rings by two TMA bulk copies per slot (one
          // per lane of the first decoder warp, all in flight at once), then summed from shared memory; slots beyond the
          // rings' capacity are staged in further rounds, the running sum carried in staged slot
          // 0. The rings are idle: this is the CTA's last piece and its MMAs have completed.
          // Mixtral w2 (3 slots x 35 rows): 8.6 us with per-thread float4 loads, 5.6 us staged
          // with 16-byte cp.async (LSU issue bound beside the co-resident CTA's decode), 2.0 us
          // with bulk copies (scripts/red_stats.py; profiles/r02/reduce_ab.txt).
          const int r0 = s.rb * (kW13 ? kRows / 2 : kRows);
          const int cols = kW13 ? kRows / 2 : min(kRows, d - r0);  // outputs of this tile, multiple of 4
          const int q4 = cols / 4;
          const int n_rows = s.n0 + s.n1;                           // active (position, token) rows
          if (!staged_red(n_rows)) {
            // every piece (own included) is in its global slot: sum them in CTA order from L2
            for (int u = dtid; u < n_rows * q4; u += kDecWarps * 32) {
              const int r = u / q4, cq = 4 * (u % q4);
              const int t = r < s.n0 ? r : NX + r - s.n0;  // (position, token) row of a slot
              float4 s0 = make_float4(0.f, 0.f, 0.f, 0.f), s1 = s0;
              for (int gg = g_first; gg <= g_last; ++gg) {
                const float* src = part + (size_t)(2 * gg + (s.item == sk.begin(gg) / nk ? 0 : 1)) * kSlot +
                                   (size_t)t * kRows + cq;
                const float4 v4 = __ldcg(reinterpret_cast<const float4*>(src));
                s0.x += v4.x; s0.y += v4.y; s0.z += v4.z; s0.w += v4.w;
                if (kW13) {
                  const float4 u4 = __ldcg(reinterpret_cast<const float4*>(src + kRows / 2));
                  s1.x += u4.x; s1.y += u4.y; s1.z += u4.z; s1.w += u4.w;
                }
              }
              const size_t aa = (size_t)((r < s.n0 ? s.pt.off0 + r : s.pt.off1 + r - s.n0) + s.base);
              if (kW13) {
                uint2 o;
                o.x = f32_to_bf16_rne_bits(silu_mul(s0.x, s1.x)) | (f32_to_bf16_rne_bits(silu_mul(s0.y, s1.y)) << 16);
                o.y = f32_to_bf16_rne_bits(silu_mul(s0.z, s1.z)) | (f32_to_bf16_rne_bits(silu_mul(s0.w, s1.w)) << 16);
                *reinterpret_cast<uint2*>(h_out + aa * f + r0 + cq) = o;
              } else {
                *reinterpret_cast<float4*>(y_out + aa * d + r0 + cq) = s0;
              }
            }
            named_bar_sync(1, kDecWarps * 32);
            return;
          }
          const int m = min(g_last - g_first + 1, (int)(kRing / (n_rows * kRowB)));  // >= 2 slots
          const int n_units = n_rows * q4;
          const uint64_t drop = l2_policy_evict_first();  // the partials are dead once read
          uint32_t red_ph = 0;  // one reduction per CTA (its last piece): red_bar phases from 0
          // staged position 0 of the first round already holds this CTA's own piece (stored from
          // TMEM above); every other slot comes in by bulk copies
          for (int gg = g_first, k0 = 0; gg <= g_last; k0 = 1) {
            const int cnt = min(m - k0, g_last - gg + 1);
            const int skip = gg == g_first ? 1 : 0;  // own piece: not copied
            if (dtid < 32 && cnt > skip) {  // two bulk copies per slot (its position-0 rows, its
                                            // position-1 rows), one per lane: a TMA instruction
                                            // costs its issuing thread ~165 ns
              if (dtid == 0) ptx::mbar_arrive_expect_tx(&c.red_bar, (uint32_t)((cnt - skip) * n_rows) * kRowB);
              __syncwarp();
              for (int l = dtid + 2 * skip; l < 2 * cnt; l += 32) {
                const int k = l >> 1, pos = l & 1, gk = gg + k;
                const int rows = pos ? s.n1 : s.n0;
                if (rows == 0) continue;
                // generic-proxy data (the acquired partials; staged rows read by the last round)
                // before async-proxy accesses
                asm volatile("fence.proxy.async;" ::: "memory");
                const float* src = part + (size_t)(2 * gk + (s.item == sk.begin(gk) / nk ? 0 : 1)) * kSlot +
                                   (size_t)pos * NX * kRows;
                const uint32_t dst = smem_w + (uint32_t)(k0 + k) * n_rows * kRowB + (uint32_t)(pos * s.n0) * kRowB;
                bulk_g2s(dst, src, (uint32_t)rows * kRowB, &c.red_bar, drop);
              }
            }
            if (cnt > skip) {
              ptx::mbar_wait(&c.red_bar, red_ph);
              red_ph ^= 1;
            }
#ifdef PZ_TRACE
            if (k0 == 0 && (dtid & 31) == 0) g_red[kW13][blockIdx.x][4 + (dtid >> 7)] = gtimer();  // warps 0 / 4 loads landed
#endif
            named_bar_sync(1, kDecWarps * 32);
#ifdef PZ_TRACE
            if (k0 == 0 && dtid == 0) g_red[kW13][blockIdx.x][6] = gtimer();
#endif
            const bool last = gg + cnt > g_last;
            for (int u = dtid; u < n_units; u += kDecWarps * 32) {
              const int r = u / q4, cq = 4 * (u % q4);
              const uint32_t a0 = smem_w + (uint32_t)r * kRowB + 16u * (cq / 4);
              float4 s0 = make_float4(0.f, 0.f, 0.f, 0.f), s1 = s0;
              if (k0) {  // the running sum of the earlier rounds
                s0 = ptx_lds_f4(a0);
                if (kW13) s1 = ptx_lds_f4(a0 + kRowB / 2);
              }
              for (int k = k0; k < k0 + cnt; ++k) {
                const uint32_t ak = a0 + (uint32_t)k * n_rows * kRowB;
                const float4 v4 = ptx_lds_f4(ak);
                s0.x += v4.x; s0.y += v4.y; s0.z += v4.z; s0.w += v4.w;
                if (kW13) {
                  const float4 u4 = ptx_lds_f4(ak + kRowB / 2);
                  s1.x += u4.x; s1.y += u4.y; s1.z += u4.z; s1.w += u4.w;
                }
              }
              if (!last) {
                ptx_sts_f4(a0, s0);
                if (kW13) ptx_sts_f4(a0 + kRowB / 2, s1);
                continue;
              }
              const size_t aa = (size_t)((r < s.n0 ? s.pt.off0 + r : s.pt.off1 + r - s.n0) + s.base);
              if (kW13) {
                uint2 o;
                o.x = f32_to_bf16_rne_bits(silu_mul(s0.x, s1.x)) | (f32_to_bf16_rne_bits(silu_mul(s0.y, s1.y)) << 16);
                o.y = f32_to_bf16_rne_bits(silu_mul(s0.z, s1.z)) | (f32_to_bf16_rne_bits(silu_mul(s0.w, s1.w)) << 16);
                *reinterpret_cast<uint2*>(h_out + aa * f + r0 + cq) = o;
              } else {
                *reinterpret_cast<float4*>(y_out + aa * d + r0 + cq) = s0;
              }
            }
            gg += cnt;
            named_bar_sync(1, kDecWarps * 32);  // staged slots read before the next round refills them
          }
          named_bar_sync(1, kDecWarps * 32);
#ifdef PZ_TRACE
          if (dtid == 0) g_red[kW13][blockIdx.x][3] = gtimer();
#endif
        }
      }
    };
    Pass pend;
    bool have_pend = false;
    auto flush = [&]() {
      if (have_pend) finish(pend);
      have_pend = false;
    };
    for (;;) {
      wait_dec(&c.wfull[w.i], w.ph);
      const int4 h = lds_int4(whdr_s + 16u * w.i);
      if (h.x < 0) break;
      const Pass s = make_pass(c, h, n_active, NX);
      const int n_st = s.kb1 - s.kb0;
      // PZ_TC_DEFER: drain the previous pass after two stages of this one (its last MMAs have
      // completed by then; the A ring lets the decoders run ahead meanwhile)
      const int ep_at = PZ_TC_DEFER ? min(1, n_st - 1) : -1;
      // a dense slot (R20) is only ever routed at position 0
      if constexpr (FMT == 1) {
        // this thread's weight row (global) and its group scales [K / 128]
        const int64_t grow = kW13 ? (int64_t)s.p * 2 * f + (srow < 64 ? 0 : f) + s.rb * (kRows / 2) + (srow & 63)
                                  : (int64_t)s.p * d + s.rb * kRows + row;
        const float* rs = qscales + grow * (K / 128);
        if (s.n0 > 0 && s.n1 > 0) decode_pass_q<3>(c, smem_w, lane_tmem, wq_off, kh, n_st, w, a, rs, s.kb0, tcount, ep_at, flush);
        else if (s.n0 > 0) decode_pass_q<1>(c, smem_w, lane_tmem, wq_off, kh, n_st, w, a, rs, s.kb0, tcount, ep_at, flush);
        else decode_pass_q<2>(c, smem_w, lane_tmem, wq_off, kh, n_st, w, a, rs, s.kb0, tcount, ep_at, flush);
      } else {
      if (pair_dense != nullptr && pair_dense[s.p]) decode_pass<4, kKC>(c, smem_w, lane_tmem, w_off, kh, n_st, w, a, mu, tcount, kW13, ep_at, flush);
      else if (s.n0 > 0 && s.n1 > 0) decode_pass<3, kKC>(c, smem_w, lane_tmem, w_off, kh, n_st, w, a, mu, tcount, kW13, ep_at, flush);
      else if (s.n0 > 0) decode_pass<1, kKC>(c, smem_w, lane_tmem, w_off, kh, n_st, w, a, mu, tcount, kW13, ep_at, flush);
      else decode_pass<2, kKC>(c, smem_w, lane_tmem, w_off, kh, n_st, w, a, mu, tcount, kW13, ep_at, flush);
      }
      if (PZ_TC_DEFER) {
        pend = s;
        have_pend = true;
      } else {
        finish(s);
      }
    }
    flush();
  }
  // MMA warps + decoders: every MMA has completed (the last epilogue waited on it) and every
  // tcgen05.ld has been waited on -> release TMEM
  ptx::tc_fence_before();
  named_bar_sync(3, 64 + kDecWarps * 32);
  ptx::tc_fence_after();
  if (warp == 1) ptx::tmem_dealloc<C::kTmemCols>(tmem);
#ifdef PZ_TRACE
  if (threadIdx.x == 32) g_cta[kW13][blockIdx.x][3] = gtimer();
#endif
}

template <bool kW13, int NX, int CTAS, int FMT = 0>
int launch_one(const CUtensorMap& tw, const CUtensorMap& tx, const int32_t* bucket_off, const int32_t* active,
               const int32_t* n_active, int K, int f, int d, int n_rb, int max_active, int64_t n_assign, float* part,
               int32_t* counters, uint16_t* h, float* y, int n_pairs, const uint8_t* pair_dense,
               cudaStream_t stream, const float* qscales = nullptr) {
  using C = Cfg<NX, CTAS, FMT>;
  auto kern = k_gemv_tc<kW13, NX, CTAS, FMT>;
  constexpr size_t kSmem = smem_bytes<C>();
  static std::atomic<uint64_t> attr{0};
  if (int rc = cuda_check(ensure_smem_attr(kern, kSmem, attr), "gemv smem attribute")) return rc;
  // stream-K grid: every resident CTA slot, but >= kMinStages stages each (the device
  // recomputes the partition from the actual active pairs and passes)
  const int64_t S = ((int64_t)max_active + n_assign / NX) * n_rb * (K / kBK);  // >= the real stage count
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)CTAS * num_sms(), S / kMinStages));
  const char* name = FMT ? (kW13 ? "w13_gemv_q" : "w2_gemv_q") : (kW13 ? "w13_gemv" : "w2_gemv");
  {
    ProfScope _ps(name, stream);
    cudaError_t e = launch_pdl(kern, dim3(grid), dim3(C::kThreads), kSmem, stream, tw, tx, bucket_off, active, n_active,
                               K, f, d, n_rb, part, counters, h, y, 1u, n_pairs, pair_dense, qscales);
    if (e != cudaSuccess) return cuda_check(e, name);
  }
  return cuda_check(cudaGetLastError(), name);
}

template <int NX, int CTAS>
int launch_both(const uint16_t* w13, const uint16_t* w2, const uint8_t* pair_dense, int n_pairs, int d, int f, const uint16_t* x_rows,
                const int32_t* bucket_off, const int32_t* active_pairs, const int32_t* n_active, int max_active,
                int64_t n_assign_cap, float* part, int32_t* counters13, int32_t* counters2, uint16_t* h, float* y,
                cudaStream_t stream) {
  if (max_active == 0 || n_assign_cap == 0) return PUZZLE_OK;
  CUtensorMap tw13, tx13, tw2, tx2;
  int rc;
  if ((rc = make_tmap_2d(&tw13, w13, (int64_t)n_pairs * 2 * f, d, kRows / 2, kBK))) return rc;
  if ((rc = make_tmap_2d(&tx13, x_rows, n_assign_cap, d, NX, kBK))) return rc;
  if ((rc = make_tmap_2d(&tw2, w2, (int64_t)n_pairs * d, f, kRows, kBK))) return rc;
  if ((rc = make_tmap_2d(&tx2, h, n_assign_cap, f, NX, kBK))) return rc;
  const int rb13 = f / (kRows / 2), rb2 = (d + kRows - 1) / kRows;
  if ((rc = launch_one<true, NX, CTAS>(tw13, tx13, bucket_off, active_pairs, n_active, d, f, d, rb13, max_active,
                                       n_assign_cap, part, counters13, h, y, n_pairs, pair_dense, stream)))
    return rc;
  return launch_one<false, NX, CTAS>(tw2, tx2, bucket_off, active_pairs, n_active, f, f, d, rb2, max_active,
                                     n_assign_cap, part, counters2, h, y, n_pairs, pair_dense, stream);
}

// NEXT-3: the same two launches over the quantised byte format (codes u8 [rows][K] + f32
// scales [rows][K / 128] per projection; no dense slots)
int launch_both_quant(const uint8_t* c13, const float* s13, const uint8_t* c2, const float* s2, int n_pairs, int d, int f,
                      const uint16_t* x_rows, const int32_t* bucket_off, const int32_t* active_pairs,
                      const int32_t* n_active, int max_active, int64_t n_assign_cap, float* part, int32_t* counters13,
                      int32_t* counters2, uint16_t* h, float* y, cudaStream_t stream) {
  constexpr int NX = 32, CTAS = 2;
  if (max_active == 0 || n_assign_cap == 0) return PUZZLE_OK;
  CUtensorMap tw13, tx13, tw2, tx2;
  int rc;
  if ((rc = make_tmap_2d_u8(&tw13, c13, (int64_t)n_pairs * 2 * f, d, kRows / 2, kBK))) return rc;
  if ((rc = make_tmap_2d(&tx13, x_rows, n_assign_cap, d, NX, kBK))) return rc;
  if ((rc = make_tmap_2d_u8(&tw2, c2, (int64_t)n_pairs * d, f, kRows, kBK))) return rc;
  if ((rc = make_tmap_2d(&tx2, h, n_assign_cap, f, NX, kBK))) return rc;
  const int rb13 = f / (kRows / 2), rb2 = (d + kRows - 1) / kRows;
  if ((rc = launch_one<true, NX, CTAS, 1>(tw13, tx13, bucket_off, active_pairs, n_active, d, f, d, rb13, max_active,
                                          n_assign_cap, part, counters13, h, y, n_pairs, nullptr, stream, s13)))
    return rc;
  return launch_one<false, NX, CTAS, 1>(tw2, tx2, bucket_off, active_pairs, n_active, f, f, d, rb2, max_active,
                                        n_assign_cap, part, counters2, h, y, n_pairs, nullptr, stream, s2);
}

}  // namespace

int launch_gemv_tc_experts_quant(const uint8_t* c13, const float* s13, const uint8_t* c2, const float* s2, int n_pairs,
                                 int d, int f, const uint16_t* x_rows, const int32_t* bucket_off,
                                 const int32_t* active_pairs, const int32_t* n_active, int max_active,
                                 int64_t n_assign_cap, float* part, int32_t* counters13, int32_t* counters2, uint16_t* h,
                                 float* y, cudaStream_t stream) {
  return launch_both_quant(c13, s13, c2, s2, n_pairs, d, f, x_rows, bucket_off, active_pairs, n_active, max_active,
                           n_assign_cap, part, counters13, counters2, h, y, stream);
}

// Partial-slot floats (2 slots per CTA x 2 CTAs per SM x 2 positions x NX x 128 with NX <= 64,
// or 2 slots x 1 CTA per SM x 2 positions x 128 x 128: the same size).
size_t gemv_tc_part_floats() { return (size_t)2 * 2 * num_sms() * 2 * 64 * kRows; }
// Work-item counters per projection: row blocks x (pairs + passes).
int64_t gemv_tc_counters(int n_rb, int n_pairs, int64_t n_assign) { return (int64_t)n_rb * (n_pairs + n_assign / 32 + 1); }
bool gemv_supported(int d, int f) { return d % 64 == 0 && f % 64 == 0 && d <= 65535 * 64 && f <= 65535 * 64; }

#ifndef PZ_NX64_TOKENS  // average tokens per expert above which the NX = 64 configuration runs
#define PZ_NX64_TOKENS 20
#endif
constexpr int kNx64Tokens = PZ_NX64_TOKENS;
#ifndef PZ_NX128_TOKENS  // ... and the NX = 128 configuration (one CTA per SM; NX 64 ahead at 48)
#define PZ_NX128_TOKENS 56
#endif
constexpr int kNx128Tokens = PZ_NX128_TOKENS;

// x_rows: [n_assign_cap][d] bf16 in bucket order (TMA source); h: [n_assign_cap][f];
// y: [n_assign_cap][d]; part: gemv_tc_part_floats(prefill) floats; counters13 / counters2:
// gemv_tc_counters(row blocks, ...) ints, zero. pair_dense: NULL or
// [n_pairs] device flags (slot holds one unmerged expert's bf16 weights, position 0 only).
int launch_gemv_tc_experts(const uint16_t* w13, const uint16_t* w2, const uint8_t* pair_dense, int n_pairs, int d, int f,
                           const uint16_t* x_rows, const int32_t* bucket_off, const int32_t* active_pairs,
                           const int32_t* n_active, int max_active, int64_t n_assign_cap, float* part,
                           int32_t* counters13, int32_t* counters2, uint16_t* h, float* y, cudaStream_t stream) {
  // one pass of 64 tokens per position instead of two of 32 once experts average more than
  // kNx64Tokens tokens, of 128 above kNx128Tokens (profiles/r02/nx64_crossover.log,
  // nx128_crossover.log)
  if (n_assign_cap > (int64_t)kNx128Tokens * 2 * n_pairs)  // one CTA per SM, 512 TMEM columns
    return launch_both<128, 1>(w13, w2, pair_dense, n_pairs, d, f, x_rows, bucket_off, active_pairs, n_active,
                               max_active, n_assign_cap, part, counters13, counters2, h, y, stream);
  if (n_assign_cap > (int64_t)kNx64Tokens * 2 * n_pairs)
    return launch_both<64, 2>(w13, w2, pair_dense, n_pairs, d, f, x_rows, bucket_off, active_pairs, n_active, max_active,
                              n_assign_cap, part, counters13, counters2, h, y, stream);
  return launch_both<32, 2>(w13, w2, pair_dense, n_pairs, d, f, x_rows, bucket_off, active_pairs, n_active, max_active,
                            n_assign_cap, part, counters13, counters2, h, y, stream);
}

#ifdef PZ_TRACE
extern "C" __attribute__((visibility("default"))) int puzzle_debug_trace(void* dst, size_t bytes) {
  return (int)cudaMemcpyFromSymbol(dst, g_trace, bytes);
}
extern "C" __attribute__((visibility("default"))) int puzzle_debug_red(void* dst, size_t bytes) {
  return (int)cudaMemcpyFromSymbol(dst, g_red, bytes);
}
extern "C" __attribute__((visibility("default"))) int puzzle_debug_cta(void* dst, size_t bytes) {
  return (int)cudaMemcpyFromSymbol(dst, g_cta, bytes);
}
extern "C" __attribute__((visibility("default"))) int puzzle_debug_wait(void* dst, size_t bytes) {
  return (int)cudaMemcpyFromSymbol(dst, g_after_wait, bytes);
}
extern "C" __attribute__((visibility("default"))) int puzzle_debug_smid(void* dst, size_t bytes) {
  return (int)cudaMemcpyFromSymbol(dst, g_smid, bytes);
}
#endif

}  // namespace pz
