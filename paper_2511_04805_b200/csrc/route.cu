// (a3) routing: top-k, gates, grouping of assignments by (pair, pos) bucket;
// (a6) combine; plus a bf16 row gather used for token permutation / EP packing.
//
// Top-k is warp-per-token: each lane holds E/32 logits in registers and ranks them against
// all E logits (ties -> lower expert id, R13); gates come from two shuffle reductions. Small batches (decode) run the whole routing in ONE CTA (histogram, warp scan,
// scatter in shared memory); large batches (prefill) use a grid of top-k CTAs, a one-CTA
// scan, and a grid of scatter CTAs that also copy each token row to its bucket slot (the
// TMA source of the expert kernels).
#include "common.cuh"

namespace pz {

#ifdef PZ_TRACE  // step timeline (tuning builds only): [kernel][min start, max end] in globaltimer ns
__device__ unsigned long long g_rt[4][2];  // route, gather, combine, route_topk
__device__ __forceinline__ void rt_stamp(int kid, bool end) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  if (end) atomicMax(&g_rt[kid][1], t);
  else atomicMin(&g_rt[kid][0], t);
}
#define PZ_RT(kid, end) \
  if (threadIdx.x == 0) rt_stamp(kid, end)
extern "C" __attribute__((visibility("default"))) int puzzle_debug_rt(void* dst, size_t bytes, int reset) {
  if (reset) {
    unsigned long long init[4][2];
    for (int i = 0; i < 4; ++i) { init[i][0] = ~0ull; init[i][1] = 0; }
    return (int)cudaMemcpyToSymbol(g_rt, init, sizeof(init));
  }
  return (int)cudaMemcpyFromSymbol(dst, g_rt, bytes);
}
#else
#define PZ_RT(kid, end)
#endif

namespace {

constexpr int kMaxTopK = 16;
constexpr int kSmallThreads = 1024;
// One CTA routes while T x k <= kSmallMaxAssign and T x E <= kSmallMaxScores (its top-k is T
// warp-serial selections over E logits); beyond, the three grids. Measured (profiles/r02/
// route_threshold.txt): the single CTA took 33 / 71 / 134 us at Mixtral T 512, Qwen1.5 T 512 /
// 1024 (the old bound T k <= 4096), the three grids ~30-35 us at every T <= 1024.
constexpr int kSmallMaxAssign = 512;
constexpr int kSmallMaxScores = 4096;
// Two-grid routing (top-k grid + scatter grid, deterministic slot order, row gather fused) up to
// kDecMaxTokens tokens while the scatter grid's per-CTA histogram prefix fits the default 48 KB
// of dynamic shared memory (route_dec_fits); the forward's larger batches take the three grids.
constexpr int64_t kDecMaxTokens = 512;

// One warp routes token t. Rank selection: lane l holds the logits of experts 32 i + l
// (i < PER); each counts how many of the E logits rank above each of its own (larger logit,
// or equal logit and lower expert id, R13) from 32 PER independent shuffles -- no serial
// k-round argmax. (Padding slots hold -inf and never rank above a real logit.)
// The j-th largest (rank j < k) is selected as slot j; emit(rank, expert, gate) is called by
// the lane holding it. Gates: softmax over the k selected (renormalize) or over all E.
template <int PER, class Emit>
__device__ __forceinline__ void warp_topk(const float* __restrict__ lg, int E, int k, int renorm, int lane,
                                          Emit&& emit) {
  float v[PER];
  int rank[PER];
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const int e = i * 32 + lane;
    v[i] = e < E ? lg[e] : -INFINITY;
    rank[i] = 0;
  }
#pragma unroll
  for (int i2 = 0; i2 < PER; ++i2)
#pragma unroll
    for (int src = 0; src < 32; ++src) {
      const float x = __shfl_sync(0xffffffffu, v[i2], src);  // logit of expert 32 i2 + src
      const int e2 = i2 * 32 + src;
#pragma unroll
      for (int i = 0; i < PER; ++i) rank[i] += (x > v[i]) | ((x == v[i]) & (e2 < i * 32 + lane));
    }
  float m = -INFINITY;  // the largest logit (rank 0)
#pragma unroll
  for (int i = 0; i < PER; ++i) m = fmaxf(m, v[i]);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const int e = i * 32 + lane;
    if (e < E && (renorm ? rank[i] < k : true)) s += expf(v[i] - m);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const int e = i * 32 + lane;
    if (e < E && rank[i] < k) emit(rank[i], e, expf(v[i] - m) / s);
  }
}

// Exclusive scan of s_count[0..n) by one warp into s_off[0..n].
__device__ __forceinline__ void warp_scan(const int32_t* s_count, int32_t* s_off, int n, int lane) {
  const int per = (n + 31) / 32;
  const int b0 = lane * per;
  int local = 0;
  for (int i = 0; i < per; ++i)
    if (b0 + i < n) local += s_count[b0 + i];
  int incl = local;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int o = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += o;
  }
  int run = incl - local;
  for (int i = 0; i < per; ++i)
    if (b0 + i < n) {
      s_off[b0 + i] = run;
      run += s_count[b0 + i];
    }
  if (lane == 31) s_off[n] = incl;
}

// Pairs with any tokens, ascending, into active_pairs (one warp).
__device__ __forceinline__ void warp_active(const int32_t* s_count, int n_pairs, int32_t* active_pairs,
                                            int32_t* n_active, int lane) {
  int na = 0;
  for (int p0 = 0; p0 < n_pairs; p0 += 32) {
    const int p = p0 + lane;
    const bool act = p < n_pairs && (s_count[2 * p] + s_count[2 * p + 1]) > 0;
    const uint32_t m = __ballot_sync(0xffffffffu, act);
    if (act) active_pairs[na + __popc(m & ((1u << lane) - 1u))] = p;
    na += __popc(m);
  }
  if (lane == 0) *n_active = na;
}

// ------------------------------------------------------------ small batches: one CTA
template <int PER>
__global__ void __launch_bounds__(kSmallThreads) k_route_small(
    const float* __restrict__ logits, int T, int E, int k, int renorm, const int32_t* __restrict__ expert_slot,
    int n_buckets, int32_t* __restrict__ topk_idx, float* __restrict__ topk_gate,
    int32_t* __restrict__ bucket_off, int32_t* __restrict__ assign_token, int32_t* __restrict__ assign_of,
    int32_t* __restrict__ active_pairs, int32_t* __restrict__ n_active, int32_t* __restrict__ zero_ptr,
    int n_zero) {
  __shared__ int32_t s_slot[kMaxExperts];
  __shared__ int32_t s_count[kMaxExperts];
  __shared__ int32_t s_off[kMaxExperts + 1];
  __shared__ int32_t s_bucket[kSmallMaxAssign];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  pdl_wait();  // the previous forward may still be using this workspace
  PZ_RT(0, false);
  pdl_trigger();
  // split-K arrival counters / scheduler counters of the expert kernels that follow
  for (int i = threadIdx.x; i < n_zero; i += blockDim.x) zero_ptr[i] = 0;
  for (int e = threadIdx.x; e < E; e += blockDim.x) s_slot[e] = expert_slot[e];
  for (int b = threadIdx.x; b < n_buckets; b += blockDim.x) s_count[b] = 0;
  __syncthreads();
  for (int t = warp; t < T; t += nwarps) {
    warp_topk<PER>(logits + (size_t)t * E, E, k, renorm, lane, [&](int j, int e, float gate) {
      topk_idx[t * k + j] = e;
      topk_gate[t * k + j] = gate;
      const int b = s_slot[e];
      s_bucket[t * k + j] = b;
      atomicAdd(&s_count[b], 1);
    });
  }
  __syncthreads();
  if (warp == 0) {
    warp_scan(s_count, s_off, n_buckets, lane);
    __syncwarp();
    for (int b = lane; b <= n_buckets; b += 32) bucket_off[b] = s_off[b];
  } else if (warp == 1 && active_pairs != nullptr) {
    warp_active(s_count, n_buckets / 2, active_pairs, n_active, lane);
  }
  __syncthreads();
  const int n_assign = T * k;
  for (int i = threadIdx.x; i < n_assign; i += blockDim.x) {
    PZ_DCHECK(s_bucket[i] >= 0 && s_bucket[i] < n_buckets);
    const int a = atomicAdd(&s_off[s_bucket[i]], 1);
    PZ_DCHECK(a >= 0 && a < n_assign);
    assign_token[a] = i / k;
    assign_of[i] = a;
  }
  PZ_RT(0, true);
}

// ------------------------------------------------------------ large batches: three grids
constexpr int kBigThreads = 256;
constexpr int kTokensPerWarp = 1;  // T = 4096: 512 CTAs (the rank selection is latency-bound per warp)

// top-k per token + per-CTA histogram folded into the global bucket counts
template <int PER>
__global__ void __launch_bounds__(kBigThreads) k_route_topk(const float* __restrict__ logits, int T, int E, int k,
                                                            int renorm, const int32_t* __restrict__ expert_slot,
                                                            int n_buckets, int32_t* __restrict__ topk_idx,
                                                            float* __restrict__ topk_gate,
                                                            int32_t* __restrict__ g_count) {
  __shared__ int32_t s_count[kMaxExperts];
  __shared__ int32_t s_slot[kMaxExperts];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  pdl_wait();
  pdl_trigger();
  for (int e = threadIdx.x; e < E; e += blockDim.x) s_slot[e] = expert_slot[e];
  for (int b = threadIdx.x; b < n_buckets; b += blockDim.x) s_count[b] = 0;
  __syncthreads();
  const int per_cta = kTokensPerWarp * (kBigThreads / 32);
  const int t_end = min(T, (int)(blockIdx.x + 1) * per_cta);
  for (int t = blockIdx.x * per_cta + warp; t < t_end; t += kBigThreads / 32) {
    warp_topk<PER>(logits + (size_t)t * E, E, k, renorm, lane, [&](int j, int e, float gate) {
      topk_idx[(size_t)t * k + j] = e;
      topk_gate[(size_t)t * k + j] = gate;
      atomicAdd(&s_count[s_slot[e]], 1);
    });
  }
  __syncthreads();
  for (int b = threadIdx.x; b < n_buckets; b += blockDim.x)
    if (s_count[b]) atomicAdd(&g_count[b], s_count[b]);
}

// one CTA: exclusive scan of the global counts -> bucket_off and the scatter cursors
__global__ void __launch_bounds__(64) k_route_scan(const int32_t* __restrict__ g_count, int n_buckets,
                                                   int32_t* __restrict__ bucket_off, int32_t* __restrict__ cursor,
                                                   int32_t* __restrict__ active_pairs,
                                                   int32_t* __restrict__ n_active) {
  __shared__ int32_t s_count[kMaxExperts];
  __shared__ int32_t s_off[kMaxExperts + 1];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  pdl_wait();
  pdl_trigger();
  for (int b = threadIdx.x; b < n_buckets; b += blockDim.x) s_count[b] = g_count[b];
  __syncthreads();
  if (warp == 0) {
    warp_scan(s_count, s_off, n_buckets, lane);
    __syncwarp();
    for (int b = lane; b <= n_buckets; b += 32) {
      bucket_off[b] = s_off[b];
      if (b < n_buckets) cursor[b] = s_off[b];
    }
  } else if (active_pairs != nullptr) {
    warp_active(s_count, n_buckets / 2, active_pairs, n_active, lane);
  }
}

// Each CTA reserves slot ranges for its chunk of assignments (one atomic per bucket), then its
// warps copy the assignments' token rows to their slots (fused gather into bucket order). 32
// assignments per CTA: the copy (the bulk of the bytes) is spread over >= 2 CTAs per SM at
// prefill sizes, 4 rows per warp with 4 x 16 B loads in flight per lane.
constexpr int kScatterChunk = 32;
__global__ void __launch_bounds__(kBigThreads) k_route_scatter(
    const int32_t* __restrict__ topk_idx, int64_t n_assign, int k, const int32_t* __restrict__ expert_slot,
    int n_buckets, int32_t* __restrict__ cursor, int32_t* __restrict__ assign_token,
    int32_t* __restrict__ assign_of, const uint16_t* __restrict__ hidden, int d, uint16_t* __restrict__ x_perm) {
  __shared__ int32_t s_count[kMaxExperts];
  __shared__ int32_t s_base[kMaxExperts];
  __shared__ int32_t s_slotof[kScatterChunk];
  pdl_wait();
  pdl_trigger();
  for (int b = threadIdx.x; b < n_buckets; b += blockDim.x) s_count[b] = 0;
  __syncthreads();
  const int64_t i0 = (int64_t)blockIdx.x * kScatterChunk;
  const int n = (int)(n_assign - i0 < kScatterChunk ? n_assign - i0 : kScatterChunk);
  int my_b = -1, my_local = 0;
  if ((int)threadIdx.x < n) {
    my_b = expert_slot[topk_idx[i0 + threadIdx.x]];
    my_local = atomicAdd(&s_count[my_b], 1);
  }
  __syncthreads();
  for (int b = threadIdx.x; b < n_buckets; b += blockDim.x)
    if (s_count[b]) s_base[b] = atomicAdd(&cursor[b], s_count[b]);
  __syncthreads();
  if ((int)threadIdx.x < n) {
    const int a = s_base[my_b] + my_local;
    PZ_DCHECK(my_b >= 0 && my_b < n_buckets && a >= 0);
    assign_token[a] = (int32_t)((i0 + threadIdx.x) / k);
    assign_of[i0 + threadIdx.x] = a;
    s_slotof[threadIdx.x] = a;
  }
  __syncthreads();
  if (x_perm == nullptr) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n16 = d / 8;  // 16-byte chunks per row
  for (int j = warp; j < n; j += kBigThreads / 32) {
    const int64_t t = (i0 + j) / k;
    const uint4* src = reinterpret_cast<const uint4*>(hidden + t * d);
    uint4* dst = reinterpret_cast<uint4*>(x_perm + (int64_t)s_slotof[j] * d);
    int c = lane;
    for (; c + 96 < n16; c += 128) {
      const uint4 v0 = ldg_nc_v4(src + c), v1 = ldg_nc_v4(src + c + 32), v2 = ldg_nc_v4(src + c + 64),
                  v3 = ldg_nc_v4(src + c + 96);
      dst[c] = v0;
      dst[c + 32] = v1;
      dst[c + 64] = v2;
      dst[c + 96] = v3;
    }
    for (; c < n16; c += 32) dst[c] = src[c];
  }
}

// ------------------------------------------------------------ decode batches: two grids
// (T <= kDecMaxTokens) Every step is spread over many SMs and no zero-initialised global state
// is needed (the workspace is caller memory): the top-k grid writes per-CTA bucket histograms and
// each assignment's bucket + its position inside its CTA's share; the scatter grid scans the
// histograms redundantly in every CTA (a few hundred ints), places each assignment and copies
// its token row to the slot (the TMA source of the expert kernels).
constexpr int kDecThreads = 256;  // one token per warp in the top-k grid, one assignment per warp in the scatter
constexpr int kDecTokensPerCta = kDecThreads / 32;

template <int PER>
__global__ void __launch_bounds__(kDecThreads) k_route_dec_topk(
    const float* __restrict__ logits, int T, int E, int k, int renorm, const int32_t* __restrict__ expert_slot,
    int n_buckets, int32_t* __restrict__ topk_idx, float* __restrict__ topk_gate, int32_t* __restrict__ hist,
    int32_t* __restrict__ bpos, int32_t* __restrict__ zero_ptr, int n_zero) {
  __shared__ int32_t s_count[kMaxExperts];
  __shared__ int32_t s_slot[kMaxExperts];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  pdl_wait();  // the previous forward may still be using this workspace
  PZ_RT(3, false);
  pdl_trigger();
  // split-piece counters of the expert kernels that follow
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_zero; i += gridDim.x * blockDim.x) zero_ptr[i] = 0;
  for (int e = threadIdx.x; e < E; e += blockDim.x) s_slot[e] = expert_slot[e];
  for (int b = threadIdx.x; b < n_buckets; b += blockDim.x) s_count[b] = 0;
  __syncthreads();
  const int t = blockIdx.x * kDecTokensPerCta + warp;
  if (t < T) {
    warp_topk<PER>(logits + (size_t)t * E, E, k, renorm, lane, [&](int j, int e, float gate) {
      topk_idx[t * k + j] = e;
      topk_gate[t * k + j] = gate;
      const int b = s_slot[e];
      bpos[t * k + j] = b | (atomicAdd(&s_count[b], 1) << 16);  // bucket | position in this CTA
    });
  }
  __syncthreads();
  for (int b = threadIdx.x; b < n_buckets; b += blockDim.x) hist[blockIdx.x * n_buckets + b] = s_count[b];
  PZ_RT(3, true);
}

__global__ void __launch_bounds__(kDecThreads) k_route_dec_scatter(
    const int32_t* __restrict__ hist, int n_hist, const int32_t* __restrict__ bpos, int n_assign, int k,
    int n_buckets, int32_t* __restrict__ bucket_off, int32_t* __restrict__ assign_token,
    int32_t* __restrict__ assign_of, int32_t* __restrict__ active_pairs, int32_t* __restrict__ n_active,
    const uint16_t* __restrict__ hidden, int d, uint16_t* __restrict__ x_perm) {
  extern __shared__ int32_t s_pre[];  // [n_hist][n_buckets] exclusive prefix over top-k CTAs
  __shared__ int32_t s_tot[kMaxExperts];
  __shared__ int32_t s_off[kMaxExperts + 1];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  pdl_wait();
  PZ_RT(0, false);
  pdl_trigger();
  for (int b = threadIdx.x; b < n_buckets; b += blockDim.x) {
    int run = 0;
    for (int c = 0; c < n_hist; ++c) {
      const int v = hist[c * n_buckets + b];
      s_pre[c * n_buckets + b] = run;
      run += v;
    }
    s_tot[b] = run;
  }
  __syncthreads();
  if (warp == 0) warp_scan(s_tot, s_off, n_buckets, lane);
  __syncthreads();
  if (blockIdx.x == 0) {
    if (warp == 0) {
      for (int b = lane; b <= n_buckets; b += 32) bucket_off[b] = s_off[b];
    } else if (warp == 1 && active_pairs != nullptr) {
      warp_active(s_tot, n_buckets / 2, active_pairs, n_active, lane);
    }
  }
  const int i = blockIdx.x * (kDecThreads / 32) + warp;  // assignment of this warp
  if (i < n_assign) {
    const int t = i / k, c = t / kDecTokensPerCta;
    const int bp = bpos[i], b = bp & 0xFFFF;
    const int a = s_off[b] + s_pre[c * n_buckets + b] + (bp >> 16);
    PZ_DCHECK(b < n_buckets && a >= 0 && a < n_assign);
    if (lane == 0) {
      assign_token[a] = t;
      assign_of[i] = a;
    }
    if (x_perm != nullptr) {  // the token row into its slot, 8 x 16 B in flight per lane
      const uint4* src = reinterpret_cast<const uint4*>(hidden + (size_t)t * d);
      uint4* dst = reinterpret_cast<uint4*>(x_perm + (size_t)a * d);
      const int n16 = d / 8;
      for (int c0 = 0; c0 < n16; c0 += 32 * 8) {
        uint4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (c0 + 32 * u + lane < n16) v[u] = src[c0 + 32 * u + lane];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (c0 + 32 * u + lane < n16) dst[c0 + 32 * u + lane] = v[u];
      }
    }
  }
  PZ_RT(0, true);
}

// out[t] = residual[t] + sum_j gate[t,j] * y[assign_of[t,j]], fp32 in slot order, one bf16 rounding.
// K > 0: top-k known at compile time (the common 1 / 2 / 4 / 6 / 8), so the k row loads are
// issued back to back; K = 0: any k.
template <int K>
__global__ void __launch_bounds__(256) k_combine(const float* __restrict__ y,
                                                 const int32_t* __restrict__ assign_of,
                                                 const float* __restrict__ gate, int k_rt, int d,
                                                 const uint16_t* __restrict__ residual,
                                                 uint16_t* __restrict__ out, int64_t T) {
  const int k = K > 0 ? K : k_rt;
  const int c4 = blockIdx.x * blockDim.x + threadIdx.x;  // index of a 4-column group
  pdl_wait();
  PZ_RT(2, false);
  pdl_trigger();
  if (c4 * 4 >= d) return;
  // tokens stride over gridDim.y (<= 65535 CTAs): any T
  for (int64_t t = blockIdx.y; t < T; t += gridDim.y) {
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  if (residual != nullptr) {
    const uint2 r = *reinterpret_cast<const uint2*>(residual + t * d + c4 * 4);
    acc = make_float4(bf16_bits_to_f32(r.x & 0xFFFFu), bf16_bits_to_f32(r.x >> 16),
                      bf16_bits_to_f32(r.y & 0xFFFFu), bf16_bits_to_f32(r.y >> 16));
  }
#pragma unroll
  for (int j = 0; j < k; ++j) {
    const float g = gate[t * k + j];
    const float4 v = *reinterpret_cast<const float4*>(y + (int64_t)assign_of[t * k + j] * d + c4 * 4);
    acc.x += g * v.x;
    acc.y += g * v.y;
    acc.z += g * v.z;
    acc.w += g * v.w;
  }
  uint2 o;
  o.x = f32_to_bf16_rne_bits(acc.x) | (f32_to_bf16_rne_bits(acc.y) << 16);
  o.y = f32_to_bf16_rne_bits(acc.z) | (f32_to_bf16_rne_bits(acc.w) << 16);
  *reinterpret_cast<uint2*>(out + t * d + c4 * 4) = o;
  }
  PZ_RT(2, true);
}

// dst[i] = src[index[i]] for bf16 rows; cols % 8 == 0 (16-byte chunks); one warp per row.
__global__ void __launch_bounds__(256) k_gather_rows(const uint16_t* __restrict__ src,
                                                     const int32_t* __restrict__ index, int64_t n_rows,
                                                     int64_t cols, uint16_t* __restrict__ dst) {
  const int64_t i = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  pdl_wait();
  PZ_RT(1, false);
  pdl_trigger();
  if (i >= n_rows) return;
  const int lane = threadIdx.x & 31;
  const int64_t s = index[i];
  const uint4* sp = reinterpret_cast<const uint4*>(src + s * cols);
  uint4* dp = reinterpret_cast<uint4*>(dst + i * cols);
  warp_copy_row(sp, dp, cols / 8, lane);
  __syncwarp();
  if (lane == 0) PZ_RT(1, true);
}

// Pairs with at least one routed row, ascending (the experts-only entry point, whose buckets
// come from the caller). One block of 256 threads, P <= 256.
__global__ void k_active_pairs(const int32_t* __restrict__ off, int n_pairs, int32_t* __restrict__ active,
                               int32_t* __restrict__ count) {
  __shared__ int warp_cnt[8];
  const int p = threadIdx.x, lane = p & 31, w = p >> 5;
  const bool has = p < n_pairs && off[2 * p + 2] > off[2 * p];
  const unsigned b = __ballot_sync(0xffffffffu, has);
  if (lane == 0) warp_cnt[w] = __popc(b);
  __syncthreads();
  int base = 0;
  for (int i = 0; i < w; ++i) base += warp_cnt[i];
  if (has) active[base + __popc(b & ((1u << lane) - 1u))] = p;
  if (p == 0) {
    int t = 0;
    for (int i = 0; i < 8; ++i) t += warp_cnt[i];
    *count = t;
  }
}

}  // namespace

int launch_active_pairs(const int32_t* bucket_off, int n_pairs, int32_t* active, int32_t* count, cudaStream_t stream) {
  {
    ProfScope _ps("active_pairs", stream);
    k_active_pairs<<<1, 256, 0, stream>>>(bucket_off, n_pairs, active, count);
  }
  return cuda_check(cudaGetLastError(), "active_pairs launch");
}

// logits per lane of the warp top-k, rounded up to a power of two
static int per_lane(int E) {
  int per = 1;
  while (per * 32 < E) per *= 2;
  return per;
}

bool route_is_small(int64_t T, int k, int E) { return T * k <= kSmallMaxAssign && T * E <= kSmallMaxScores; }

// Decode-batch routing scratch: per-CTA histograms + packed bucket positions (ints).
int64_t route_dec_scratch_ints(int64_t T, int k, int n_pairs) {
  return ((T + kDecTokensPerCta - 1) / kDecTokensPerCta) * 2 * n_pairs + T * k;
}

// Routing + fused row gather for T <= kDecMaxTokens: two multi-CTA kernels (see above).
bool route_dec_fits(int64_t T, int n_pairs) {
  const int64_t n_hist = (T + kDecTokensPerCta - 1) / kDecTokensPerCta;
  return T <= kDecMaxTokens && n_hist * 2 * n_pairs * (int64_t)sizeof(int32_t) <= 48 * 1024;
}

int launch_route_dec(const float* logits, int64_t T, int E, int k, int renorm, const int32_t* expert_slot,
                     int n_pairs, int32_t* topk_idx, float* topk_gate, int32_t* bucket_off, int32_t* assign_token,
                     int32_t* assign_of, int32_t* active_pairs, int32_t* n_active, int32_t* zero_ptr, int n_zero,
                     int32_t* scratch, const uint16_t* hidden, int d, uint16_t* x_perm, cudaStream_t stream) {
  if (k > kMaxTopK) return fail(PUZZLE_ERR_UNSUPPORTED, "top_k > 16 is not supported by the route kernel");
  if (E > kMaxExperts) return fail(PUZZLE_ERR_UNSUPPORTED, "n_experts > 512");
  if (!route_dec_fits(T, n_pairs)) return fail(PUZZLE_ERR_UNSUPPORTED, "two-grid routing: too many tokens");
  const int nb = 2 * n_pairs;
  const int n_hist = (int)((T + kDecTokensPerCta - 1) / kDecTokensPerCta);
  int32_t* hist = scratch;
  int32_t* bpos = scratch + (int64_t)n_hist * nb;
  const int per = per_lane(E);
  auto topk = per == 1 ? k_route_dec_topk<1> : per == 2 ? k_route_dec_topk<2> : per == 4 ? k_route_dec_topk<4>
            : per == 8 ? k_route_dec_topk<8> : k_route_dec_topk<16>;
  int rc;
  {
    ProfScope _ps("route_topk", stream);
    if ((rc = cuda_check(launch_pdl(topk, dim3(n_hist), dim3(kDecThreads), 0, stream, logits, (int)T, E, k, renorm,
                                    expert_slot, nb, topk_idx, topk_gate, hist, bpos, zero_ptr, n_zero),
                         "route_topk launch")))
      return rc;
  }
  const int n_assign = (int)(T * k);
  {
    ProfScope _ps("route_scatter", stream);
    if ((rc = cuda_check(launch_pdl(k_route_dec_scatter, dim3((n_assign + kDecThreads / 32 - 1) / (kDecThreads / 32)),
                                    dim3(kDecThreads), (size_t)n_hist * nb * sizeof(int32_t), stream,
                                    (const int32_t*)hist, n_hist, (const int32_t*)bpos, n_assign, k, nb, bucket_off,
                                    assign_token, assign_of, active_pairs, n_active, hidden, d, x_perm),
                         "route_scatter launch")))
      return rc;
  }
  return PUZZLE_OK;
}

// scratch: >= 2 * n_buckets int32 (global counts + cursors), used by the large-batch path only.
// hidden / x_perm (optional): the large-batch scatter also writes the bucket-ordered rows and
// then sets *rows_written.
int launch_route(const float* logits, int64_t T, int E, int k, int renorm, const int32_t* expert_slot,
                 int n_pairs, int32_t* topk_idx, float* topk_gate, int32_t* bucket_off,
                 int32_t* assign_token, int32_t* assign_of, int32_t* active_pairs, int32_t* n_active,
                 int32_t* zero_ptr, int n_zero, int32_t* scratch, const uint16_t* hidden, int d,
                 uint16_t* x_perm, bool* rows_written, cudaStream_t stream) {
  if (k > kMaxTopK) return fail(PUZZLE_ERR_UNSUPPORTED, "top_k > 16 is not supported by the route kernel");
  if (E > kMaxExperts) return fail(PUZZLE_ERR_UNSUPPORTED, "n_experts > 512");
  const int nb = 2 * n_pairs;
  if (rows_written) *rows_written = false;
  if (route_is_small(T, k, E)) {
    {
      ProfScope _ps("route", stream);
      const int per = per_lane(E);
      auto kern = per == 1 ? k_route_small<1> : per == 2 ? k_route_small<2> : per == 4 ? k_route_small<4>
                : per == 8 ? k_route_small<8> : k_route_small<16>;
      cudaError_t e = launch_pdl(kern, dim3(1), dim3(kSmallThreads), 0, stream, logits, (int)T, E, k, renorm,
                                 expert_slot, nb, topk_idx, topk_gate, bucket_off, assign_token, assign_of,
                                 active_pairs, n_active, zero_ptr, n_zero);
      if (e != cudaSuccess) return cuda_check(e, "route launch");
    }
    return cuda_check(cudaGetLastError(), "route launch");
  }
  if (scratch == nullptr) return fail(PUZZLE_ERR_WORKSPACE, "large-batch routing needs scratch space");
  int32_t* g_count = scratch;
  int32_t* cursor = scratch + nb;
  int rc;
  if ((rc = cuda_check(cudaMemsetAsync(g_count, 0, nb * sizeof(int32_t), stream), "route memset"))) return rc;
  if (n_zero > 0 && (rc = cuda_check(cudaMemsetAsync(zero_ptr, 0, n_zero * sizeof(int32_t), stream), "memset")))
    return rc;
  const int per_cta = kTokensPerWarp * (kBigThreads / 32);
  {
    ProfScope _ps("route_topk", stream);
    const int per = per_lane(E);
    auto kern = per == 1 ? k_route_topk<1> : per == 2 ? k_route_topk<2> : per == 4 ? k_route_topk<4>
              : per == 8 ? k_route_topk<8> : k_route_topk<16>;
    if ((rc = cuda_check(launch_pdl(kern, dim3((unsigned)((T + per_cta - 1) / per_cta)), dim3(kBigThreads), 0,
                                    stream, logits, (int)T, E, k, renorm, expert_slot, nb, topk_idx, topk_gate, g_count),
                         "route_topk launch")))
      return rc;
  }
  {
    ProfScope _ps("route_scan", stream);
    if ((rc = cuda_check(launch_pdl(k_route_scan, dim3(1), dim3(64), 0, stream, (const int32_t*)g_count, nb, bucket_off,
                                    cursor, active_pairs, n_active),
                         "route_scan launch")))
      return rc;
  }
  const int64_t n_assign = T * k;
  {
    ProfScope _ps("route_scatter", stream);
    if ((rc = cuda_check(launch_pdl(k_route_scatter, dim3((unsigned)((n_assign + kScatterChunk - 1) / kScatterChunk)),
                                    dim3(kBigThreads), 0, stream, (const int32_t*)topk_idx, n_assign, k, expert_slot, nb,
                                    cursor, assign_token, assign_of, hidden, d, x_perm),
                         "route_scatter launch")))
      return rc;
  }
  if (rows_written) *rows_written = x_perm != nullptr && hidden != nullptr;
  return cuda_check(cudaGetLastError(), "route launch");
}

int launch_combine(const float* y, const int32_t* assign_of, const float* gate, int64_t T, int k,
                   int d, const uint16_t* residual, uint16_t* out, cudaStream_t stream) {
  if (T == 0) return PUZZLE_OK;
  const int threads = 256;
  dim3 grid((unsigned)((d / 4 + threads - 1) / threads), (unsigned)std::min<int64_t>(T, 65535));
  {
    ProfScope _ps("combine", stream);
    auto kern = k == 1 ? k_combine<1> : k == 2 ? k_combine<2> : k == 4 ? k_combine<4> : k == 6 ? k_combine<6>
              : k == 8 ? k_combine<8> : k_combine<0>;
    cudaError_t e = launch_pdl(kern, grid, dim3(threads), 0, stream, y, assign_of, gate, k, d, residual, out, T);
    if (e != cudaSuccess) return cuda_check(e, "combine launch");
  }
  return cuda_check(cudaGetLastError(), "combine launch");
}

int launch_gather_rows(const uint16_t* src, const int32_t* index, int64_t n_rows, int64_t cols,
                       uint16_t* dst, cudaStream_t stream) {
  if (n_rows == 0) return PUZZLE_OK;
  {
    ProfScope _ps("gather_rows", stream);
    cudaError_t e = launch_pdl(k_gather_rows, dim3((unsigned)((n_rows + 7) / 8)), dim3(256), 0, stream, src, index, n_rows,
                               cols, dst);
    if (e != cudaSuccess) return cuda_check(e, "gather launch");
  }
  return cuda_check(cudaGetLastError(), "gather launch");
}

}  // namespace pz
