// NEXT-4: calibration statistics for the Wanda saliency of Eq. 4: ||X||_2 per input
// column over the activations routed to each expert, from a single forward pass.
// Computed as f64 column sums of squares per group of bucket-ordered bf16 rows (the forward's
// permuted x rows for W1/W3, its SwiGLU intermediate h for W2); norms = their square roots.
//
// HBM-bound column reduction: CTA (column chunk of 512, row split of ALL rows -- so empty groups
// cost nothing) streams its rows with 16-byte loads (64 threads x 8 columns per row, 4 row lanes
// x 8 loads in flight per thread), sums squares in f32 per 8 rows then in f64, reduces the 4
// row lanes in shared memory in a fixed order per group segment, and writes one partial per
// (split, group) it touches; a second kernel adds, per group, exactly the splits that intersect
// it, in split order. No atomics: results are bit-reproducible run to run.
#include "common.cuh"

namespace pz {

namespace {

constexpr int kColsPerCta = 512;  // 64 column threads x 8 bf16
constexpr int kRowLanes = 4;
#ifndef PZ_CALIB_UNROLL
#define PZ_CALIB_UNROLL 8
#endif
#ifndef PZ_CALIB_MINB  // resident CTAs per SM the register allocation must allow
#define PZ_CALIB_MINB 3
#endif
constexpr int kUnroll = PZ_CALIB_UNROLL;
constexpr int kCalibThreads = 64 * kRowLanes;
#ifndef PZ_CALIB_CTAS  // target CTAs per SM of the grid
#define PZ_CALIB_CTAS 3
#endif

// Row split s of the flattened rows [base, base + n): [base + n s / S, base + n (s + 1) / S).
__device__ __forceinline__ int64_t split_begin(int64_t base, int64_t n, int S, int s) { return base + n * s / S; }

__device__ __forceinline__ int split_of(int64_t base, int64_t n, int S, int64_t r) {
  int s = (int)(((r - base) * S) / n);
  while (s > 0 && split_begin(base, n, S, s) > r) --s;
  while (s + 1 < S && split_begin(base, n, S, s + 1) <= r) ++s;
  return s;
}

// CTA (column chunk, row split): its rows may span several groups; each group segment is
// reduced (4 row lanes, fixed order) and written to part[split][group]. Every thread sums its
// kUnroll rows in f32 (the square of a bf16 value is exact in f32; 8 terms lose <= 2^-21
// relative) and adds that to its f64 accumulators.
__global__ void __launch_bounds__(kCalibThreads, PZ_CALIB_MINB) k_group_colsumsq_part(const uint16_t* __restrict__ rows,
                                                                       const int32_t* __restrict__ group_off,
                                                                       int n_groups, int64_t cols, int splits,
                                                                       double* __restrict__ part) {
  __shared__ double s_acc[kRowLanes - 1][64][8];
  const int ct = threadIdx.x & 63, rl = threadIdx.x >> 6;
  const int64_t c0 = (int64_t)blockIdx.x * kColsPerCta + 8 * ct;
  const int sp = blockIdx.y;
  const int64_t base = group_off[0], n = group_off[n_groups] - base;
  const int64_t r0 = split_begin(base, n, splits, sp), r1 = split_begin(base, n, splits, sp + 1);
  int g = 0;
  while (g + 1 < n_groups && group_off[g + 1] <= r0) ++g;
  for (int64_t seg = r0; seg < r1; ++g) {
    const int64_t seg_end = r1 < (int64_t)group_off[g + 1] ? r1 : (int64_t)group_off[g + 1];
    if (seg_end <= seg) continue;  // empty group
    double acc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = 0.0;
    if (c0 < cols) {
      for (int64_t r = seg + rl; r < seg_end; r += kUnroll * kRowLanes) {
        uint4 v[kUnroll];  // kUnroll independent 16-B loads in flight per thread
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
          const int64_t rr = r + u * kRowLanes;
          v[u] = rr < seg_end ? ldg_nc_v4(rows + rr * cols + c0) : make_uint4(0u, 0u, 0u, 0u);
        }
        float fs[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) fs[i] = 0.0f;
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
          const uint32_t w[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
          for (int i = 0; i < 4; ++i) {  // low half = even column, high half = odd column
            const float a = __uint_as_float(w[i] << 16), b = __uint_as_float(w[i] & 0xFFFF0000u);
            fs[2 * i] = __fmaf_rn(a, a, fs[2 * i]);
            fs[2 * i + 1] = __fmaf_rn(b, b, fs[2 * i + 1]);
          }
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] += (double)fs[i];
      }
    }
    __syncthreads();  // s_acc of the previous segment consumed
    if (rl > 0)
#pragma unroll
      for (int i = 0; i < 8; ++i) s_acc[rl - 1][ct][i] = acc[i];
    __syncthreads();
    if (rl == 0 && c0 < cols) {
#pragma unroll
      for (int l = 0; l < kRowLanes - 1; ++l)
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] += s_acc[l][ct][i];
      double* dst = part + ((int64_t)sp * n_groups + g) * cols + c0;
#pragma unroll
      for (int i = 0; i < 8; i += 2) *reinterpret_cast<double2*>(dst + i) = make_double2(acc[i], acc[i + 1]);
    }
    seg = seg_end;
  }
}

// sumsq[g][c] += the partials of exactly the splits that intersect group g, in split order.
__global__ void k_group_colsumsq_reduce(const double* __restrict__ part, const int32_t* __restrict__ group_off,
                                        int n_groups, int64_t cols, int splits, double* __restrict__ sumsq) {
  const int64_t base = group_off[0], n = group_off[n_groups] - base;
  const int64_t total = (int64_t)n_groups * cols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int g = (int)(i / cols);
    const int64_t lo = group_off[g], hi = group_off[g + 1];
    if (hi <= lo) continue;
    const int s0 = split_of(base, n, splits, lo), s1 = split_of(base, n, splits, hi - 1);
    double s = 0.0;
    for (int sp = s0; sp <= s1; ++sp)  // empty splits (more splits than rows) wrote nothing
      if (split_begin(base, n, splits, sp) < split_begin(base, n, splits, sp + 1)) s += part[(int64_t)sp * total + i];
    sumsq[i] += s;
  }
}

}  // namespace

// Row splits: enough CTAs for ~PZ_CALIB_CTAS per SM over the whole grid.
int calib_splits(int n_groups, int64_t cols) {
  (void)n_groups;
  const int64_t chunks = (cols + kColsPerCta - 1) / kColsPerCta;
  const int64_t want = (PZ_CALIB_CTAS * (int64_t)num_sms() + chunks - 1) / chunks;
  return (int)std::max<int64_t>(1, std::min<int64_t>(want, 4096));
}

size_t calib_workspace_bytes(int n_groups, int64_t cols) {
  return (size_t)calib_splits(n_groups, cols) * n_groups * cols * sizeof(double);
}

// rows: [n][cols] bf16, groups [group_off[g], group_off[g+1]) (device offsets); sumsq: [n_groups][cols]
// f64, accumulated; part: calib_workspace_bytes(n_groups, cols) bytes (only the (split, group)
// blocks a split intersects are written and read). cols % 8 == 0, rows 16-B aligned.
int launch_group_colsumsq(const uint16_t* rows, const int32_t* group_off, int n_groups, int64_t cols, double* sumsq,
                          double* part, cudaStream_t stream) {
  if (n_groups == 0 || cols == 0) return PUZZLE_OK;
  const int splits = calib_splits(n_groups, cols);
  const dim3 grid((unsigned)((cols + kColsPerCta - 1) / kColsPerCta), (unsigned)splits);
  {
    ProfScope _ps("calib_colsumsq", stream);
    k_group_colsumsq_part<<<grid, kCalibThreads, 0, stream>>>(rows, group_off, n_groups, cols, splits, part);
  }
  int rc = cuda_check(cudaGetLastError(), "calib_colsumsq launch");
  if (rc) return rc;
  const int64_t n = (int64_t)n_groups * cols;
  const int blocks = (int)std::min<int64_t>((n + 255) / 256, 4 * (int64_t)num_sms());
  {
    ProfScope _ps("calib_reduce", stream);
    k_group_colsumsq_reduce<<<blocks, 256, 0, stream>>>(part, group_off, n_groups, cols, splits, sumsq);
  }
  return cuda_check(cudaGetLastError(), "calib_reduce launch");
}

}  // namespace pz
