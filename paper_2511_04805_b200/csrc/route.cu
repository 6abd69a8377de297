// (a3) routing: top-k, gates, grouping of assignments by (pair, pos) bucket;
// (a6) combine; plus a bf16 row gather used for token permutation / EP packing.
//
// Top-k is warp-per-token: each lane holds E/32 logits in registers, k rounds of a shuffle
// argmax (ties -> lower expert id, R13) pick the experts, gates come from one more shuffle
// sum. Small batches (decode) run the whole routing in ONE CTA (histogram, warp scan,
// scatter in shared memory); large batches (prefill) use a grid of top-k CTAs, a one-CTA
// scan, and a grid of scatter CTAs that also copy each token row to its bucket slot (the
// TMA source of the expert kernels).
#include "common.cuh"

namespace pz {

namespace {

constexpr int kMaxTopK = 16;
constexpr int kMaxLogitsPerLane = kMaxExperts / 32;  // 16
constexpr int kSmallThreads = 1024;
constexpr int kSmallMaxAssign = 4096;  // single-CTA path keeps the assignment list in smem

// (v, e) ranks above (v2, e2): larger logit, or equal logit and lower expert id.
__device__ __forceinline__ bool ranks_above(float v, int e, float v2, int e2) {
  return v > v2 || (v == v2 && e < e2);
}

// One warp routes token t: lane j < k receives the j-th selected expert and its gate.
__device__ __forceinline__ void warp_topk(const float* __restrict__ lg, int E, int k, int renorm, int lane,
                                          int* sel_out, float* gate_out) {
  float v[kMaxLogitsPerLane];
  const int per = (E + 31) / 32;
#pragma unroll
  for (int i = 0; i < kMaxLogitsPerLane; ++i) {
    const int e = i * 32 + lane;
    v[i] = (i < per && e < E) ? lg[e] : -INFINITY;
  }
  float m_all = -INFINITY;  // the first selected logit = max over all experts
  float sel_v = 0.f;
  int sel_e = -1;
  uint32_t taken = 0;  // bit i: v[i] already selected
  for (int j = 0; j < k; ++j) {
    float bv = -INFINITY;
    int be = 0x7fffffff;
#pragma unroll
    for (int i = 0; i < kMaxLogitsPerLane; ++i) {
      const int e = i * 32 + lane;
      if (i < per && e < E && !((taken >> i) & 1u) && (be == 0x7fffffff || ranks_above(v[i], e, bv, be))) {
        bv = v[i];
        be = e;
      }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, bv, off);
      const int oe = __shfl_xor_sync(0xffffffffu, be, off);
      if (oe != 0x7fffffff && (be == 0x7fffffff || ranks_above(ov, oe, bv, be))) {
        bv = ov;
        be = oe;
      }
    }
    if ((be & 31) == lane) taken |= 1u << (be >> 5);
    if (j == 0) m_all = bv;
    if (lane == j) {
      sel_v = bv;
      sel_e = be;
    }
  }
  float s = 0.f;
  if (renorm) {
    s = lane < k ? expf(sel_v - m_all) : 0.f;
  } else {
#pragma unroll
    for (int i = 0; i < kMaxLogitsPerLane; ++i) {
      const int e = i * 32 + lane;
      if (i < per && e < E) s += expf(v[i] - m_all);
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  *sel_out = sel_e;
  *gate_out = lane < k ? expf(sel_v - m_all) / s : 0.f;
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
  pdl_trigger();
  // split-K arrival counters / scheduler counters of the expert kernels that follow
  for (int i = threadIdx.x; i < n_zero; i += blockDim.x) zero_ptr[i] = 0;
  for (int e = threadIdx.x; e < E; e += blockDim.x) s_slot[e] = expert_slot[e];
  for (int b = threadIdx.x; b < n_buckets; b += blockDim.x) s_count[b] = 0;
  __syncthreads();
  for (int t = warp; t < T; t += nwarps) {
    int sel;
    float gate;
    warp_topk(logits + (size_t)t * E, E, k, renorm, lane, &sel, &gate);
    if (lane < k) {
      topk_idx[t * k + lane] = sel;
      topk_gate[t * k + lane] = gate;
      const int b = s_slot[sel];
      s_bucket[t * k + lane] = b;
      atomicAdd(&s_count[b], 1);
    }
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
    const int a = atomicAdd(&s_off[s_bucket[i]], 1);
    assign_token[a] = i / k;
    assign_of[i] = a;
  }
}

// ------------------------------------------------------------ large batches: three grids
constexpr int kBigThreads = 256;
constexpr int kTokensPerWarp = 4;

// top-k per token + per-CTA histogram folded into the global bucket counts
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
    int sel;
    float gate;
    warp_topk(logits + (size_t)t * E, E, k, renorm, lane, &sel, &gate);
    if (lane < k) {
      topk_idx[(size_t)t * k + lane] = sel;
      topk_gate[(size_t)t * k + lane] = gate;
      atomicAdd(&s_count[s_slot[sel]], 1);
    }
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
// warps copy the assignments' token rows to their slots (fused gather into bucket order).
constexpr int kScatterChunk = kBigThreads;
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
    assign_token[a] = (int32_t)((i0 + threadIdx.x) / k);
    assign_of[i0 + threadIdx.x] = a;
    s_slotof[threadIdx.x] = a;
  }
  __syncthreads();
  if (x_perm == nullptr) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int j = warp; j < n; j += kBigThreads / 32) {
    const int64_t t = (i0 + j) / k;
    const uint4* src = reinterpret_cast<const uint4*>(hidden + t * d);
    uint4* dst = reinterpret_cast<uint4*>(x_perm + (int64_t)s_slotof[j] * d);
    for (int c = lane; c < d / 8; c += 32) dst[c] = src[c];
  }
}

// out[t] = residual[t] + sum_j gate[t,j] * y[assign_of[t,j]], fp32 in slot order, one bf16 rounding.
__global__ void __launch_bounds__(256) k_combine(const float* __restrict__ y,
                                                 const int32_t* __restrict__ assign_of,
                                                 const float* __restrict__ gate, int k, int d,
                                                 const uint16_t* __restrict__ residual,
                                                 uint16_t* __restrict__ out) {
  const int64_t t = blockIdx.y;
  const int c4 = blockIdx.x * blockDim.x + threadIdx.x;  // index of a 4-column group
  pdl_wait();
  pdl_trigger();
  if (c4 * 4 >= d) return;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  if (residual != nullptr) {
    const uint2 r = *reinterpret_cast<const uint2*>(residual + t * d + c4 * 4);
    acc = make_float4(bf16_bits_to_f32(r.x & 0xFFFFu), bf16_bits_to_f32(r.x >> 16),
                      bf16_bits_to_f32(r.y & 0xFFFFu), bf16_bits_to_f32(r.y >> 16));
  }
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

// dst[i] = src[index[i]] for bf16 rows; cols % 8 == 0 (16-byte chunks); one warp per row.
__global__ void __launch_bounds__(256) k_gather_rows(const uint16_t* __restrict__ src,
                                                     const int32_t* __restrict__ index, int64_t n_rows,
                                                     int64_t cols, uint16_t* __restrict__ dst) {
  const int64_t i = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  pdl_wait();
  pdl_trigger();
  if (i >= n_rows) return;
  const int lane = threadIdx.x & 31;
  const int64_t s = index[i];
  const uint4* sp = reinterpret_cast<const uint4*>(src + s * cols);
  uint4* dp = reinterpret_cast<uint4*>(dst + i * cols);
  for (int64_t c = lane; c < cols / 8; c += 32) dp[c] = sp[c];
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

bool route_is_small(int64_t T, int k) { return T * k <= kSmallMaxAssign; }

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
  if (route_is_small(T, k)) {
    {
      ProfScope _ps("route", stream);
      cudaError_t e = launch_pdl(k_route_small, dim3(1), dim3(kSmallThreads), 0, stream, logits, (int)T, E, k, renorm,
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
    if ((rc = cuda_check(launch_pdl(k_route_topk, dim3((unsigned)((T + per_cta - 1) / per_cta)), dim3(kBigThreads), 0,
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
  dim3 grid((unsigned)((d / 4 + threads - 1) / threads), (unsigned)T);
  {
    ProfScope _ps("combine", stream);
    cudaError_t e = launch_pdl(k_combine, grid, dim3(threads), 0, stream, y, assign_of, gate, k, d, residual, out);
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
