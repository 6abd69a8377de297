// (a3) routing: top-k, gates, grouping of assignments by (pair, pos) bucket;
// (a6) combine; plus a bf16 row gather used for token permutation / EP packing.
#include "common.cuh"

namespace pz {

namespace {

constexpr int kRouteThreads = 1024;
constexpr int kMaxTopK = 16;

// (v, e) ranks above (v2, e2) when v > v2, or v == v2 and e < e2 (ties -> lower id, R13).
__device__ __forceinline__ bool ranks_above(float v, int e, float v2, int e2) {
  return v > v2 || (v == v2 && e < e2);
}

// One CTA. Phase 1: per-token top-k + gates + bucket histogram (smem atomics).
// Phase 2: exclusive scan over the 2P buckets, active-pair list. Phase 3: scatter.
__global__ void __launch_bounds__(kRouteThreads) k_route(
    const float* __restrict__ logits, int64_t T, int E, int k, int renorm,
    const int32_t* __restrict__ expert_slot, int n_buckets, int32_t* __restrict__ topk_idx,
    float* __restrict__ topk_gate, int32_t* __restrict__ bucket_off,
    int32_t* __restrict__ assign_token, int32_t* __restrict__ assign_of,
    int32_t* __restrict__ active_pairs, int32_t* __restrict__ n_active,
    int32_t* __restrict__ zero_ptr, int n_zero) {
  // split-K arrival counters of the expert kernels that follow on this stream
  for (int i = threadIdx.x; i < n_zero; i += blockDim.x) zero_ptr[i] = 0;
  __shared__ int32_t s_slot[kMaxExperts];
  __shared__ int32_t s_count[kMaxExperts];
  __shared__ int32_t s_cursor[kMaxExperts];
  for (int e = threadIdx.x; e < E; e += blockDim.x) s_slot[e] = expert_slot[e];
  for (int b = threadIdx.x; b < n_buckets; b += blockDim.x) s_count[b] = 0;
  __syncthreads();

  for (int64_t t = threadIdx.x; t < T; t += blockDim.x) {
    const float* lg = logits + t * E;
    int sel[kMaxTopK];
    float val[kMaxTopK];
    float pv = INFINITY;
    int pe = -1;
    for (int j = 0; j < k; ++j) {
      int best = -1;
      float bv = -INFINITY;
      for (int e = 0; e < E; ++e) {
        float v = lg[e];
        bool below_prev = (pe < 0) || ranks_above(pv, pe, v, e);
        if (below_prev && (best < 0 || ranks_above(v, e, bv, best))) {
          best = e;
          bv = v;
        }
      }
      sel[j] = best;
      val[j] = bv;
      pv = bv;
      pe = best;
    }
    // gates (the top-1 logit is the max of the selected and of all experts)
    const float m = val[0];
    float denom = 0.0f;
    if (renorm) {
      for (int j = 0; j < k; ++j) denom += expf(val[j] - m);
    } else {
      for (int e = 0; e < E; ++e) denom += expf(lg[e] - m);
    }
    for (int j = 0; j < k; ++j) {
      topk_idx[t * k + j] = sel[j];
      topk_gate[t * k + j] = expf(val[j] - m) / denom;
      atomicAdd(&s_count[s_slot[sel[j]]], 1);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int run = 0;
    for (int b = 0; b < n_buckets; ++b) {
      bucket_off[b] = run;
      s_cursor[b] = run;
      run += s_count[b];
    }
    bucket_off[n_buckets] = run;
    if (active_pairs != nullptr) {
      int na = 0;
      for (int p = 0; p < n_buckets / 2; ++p)
        if (s_count[2 * p] + s_count[2 * p + 1] > 0) active_pairs[na++] = p;
      *n_active = na;
    }
  }
  __syncthreads();
  const int64_t n_assign = T * k;
  for (int64_t i = threadIdx.x; i < n_assign; i += blockDim.x) {
    const int b = s_slot[topk_idx[i]];
    const int a = atomicAdd(&s_cursor[b], 1);
    assign_token[a] = (int32_t)(i / k);
    assign_of[i] = a;
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

// dst[i] = src[index[i]] for bf16 rows; cols % 8 == 0 (16-byte chunks).
__global__ void __launch_bounds__(128) k_gather_rows(const uint16_t* __restrict__ src,
                                                     const int32_t* __restrict__ index,
                                                     int64_t cols, uint16_t* __restrict__ dst) {
  const int64_t i = blockIdx.x;
  const int64_t s = index[i];
  const uint4* sp = reinterpret_cast<const uint4*>(src + s * cols);
  uint4* dp = reinterpret_cast<uint4*>(dst + i * cols);
  for (int64_t c = threadIdx.x; c < cols / 8; c += blockDim.x) dp[c] = sp[c];
}

__global__ void k_iota(int32_t* v, int n, int32_t* count) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) v[i] = i;
  if (threadIdx.x == 0) *count = n;
}

}  // namespace

int launch_iota(int32_t* v, int n, int32_t* count, cudaStream_t stream) {
  { ProfScope _ps("iota", stream); k_iota<<<1, 256, 0, stream>>>(v, n, count); }
  return cuda_check(cudaGetLastError(), "iota launch");
}

int launch_route(const float* logits, int64_t T, int E, int k, int renorm, const int32_t* expert_slot,
                 int n_pairs, int32_t* topk_idx, float* topk_gate, int32_t* bucket_off,
                 int32_t* assign_token, int32_t* assign_of, int32_t* active_pairs, int32_t* n_active,
                 int32_t* zero_ptr, int n_zero, cudaStream_t stream) {
  if (k > kMaxTopK) return fail(PUZZLE_ERR_UNSUPPORTED, "top_k > 16 is not supported by the route kernel");
  { ProfScope _ps("route", stream); k_route<<<1, kRouteThreads, 0, stream>>>(logits, T, E, k, renorm, expert_slot, 2 * n_pairs,
                                           topk_idx, topk_gate, bucket_off, assign_token, assign_of,
                                           active_pairs, n_active, zero_ptr, n_zero); }
  return cuda_check(cudaGetLastError(), "route launch");
}

int launch_combine(const float* y, const int32_t* assign_of, const float* gate, int64_t T, int k,
                   int d, const uint16_t* residual, uint16_t* out, cudaStream_t stream) {
  if (T == 0) return PUZZLE_OK;
  const int threads = 256;
  dim3 grid((unsigned)((d / 4 + threads - 1) / threads), (unsigned)T);
  { ProfScope _ps("combine", stream); k_combine<<<grid, threads, 0, stream>>>(y, assign_of, gate, k, d, residual, out); }
  return cuda_check(cudaGetLastError(), "combine launch");
}

int launch_gather_rows(const uint16_t* src, const int32_t* index, int64_t n_rows, int64_t cols,
                       uint16_t* dst, cudaStream_t stream) {
  if (n_rows == 0) return PUZZLE_OK;
  { ProfScope _ps("gather_rows", stream); k_gather_rows<<<(unsigned)n_rows, 128, 0, stream>>>(src, index, cols, dst); }
  return cuda_check(cudaGetLastError(), "gather launch");
}

}  // namespace pz
