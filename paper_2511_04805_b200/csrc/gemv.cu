// Decode-shape expert kernels (a4)+(a5): the packed weights of each touched pair are
// streamed from HBM ONCE (128-bit loads, no shared memory), decoded in registers for
// expert pos 0 and/or pos 1 with the two-lane SWAR form of Algorithm 1, and
// fed straight into mma.sync m16n8k16 bf16 tensor-core MMAs as the A operand
// (weights = rows, tokens = columns: "swap-AB" so that 1..64 tokens map onto N = 8 tiles).
//
// K-permutation trick: within each 32-wide K sub-chunk, lane (g, tig) loads the 16 bytes
// at physical k = 8*tig .. 8*tig+7 of rows g and g+8. Physical k 8tig+{0,1}/{2,3} feed
// MMA#0 fragments a0/a2 (logical k 2tig+{0,1} / 2tig+8+{0,1}); 8tig+{4..7} feed MMA#1. The
// B fragments (activations) are loaded with the identical permutation, so every dot
// product sums exactly the same products (in a different order).
#include "common.cuh"

namespace pz {

namespace {

constexpr int kWarps = 4;              // warps per CTA
constexpr int kThreads = kWarps * 32;
constexpr int kKStep = 64;             // K per main-loop iteration (two 32-wide sub-chunks)

struct PairTokens {
  int off0, cnt0, off1, cnt1;
};

__device__ __forceinline__ PairTokens pair_tokens(const int32_t* bucket_off, int p) {
  PairTokens r;
  r.off0 = bucket_off[2 * p];
  r.off1 = bucket_off[2 * p + 1];
  r.cnt0 = r.off1 - r.off0;
  r.cnt1 = bucket_off[2 * p + 2] - r.off1;
  return r;
}

// Two 16-row m-tiles (gate rows and up rows of the same 16 d_ff indices) per warp.
// NT = n-tiles (8 tokens each) per expert position per pass.
template <int NT>
__global__ void __launch_bounds__(kThreads) k_w13_gemv(
    const uint16_t* __restrict__ w13, const uint16_t* __restrict__ x,
    const int32_t* __restrict__ row_index, const int32_t* __restrict__ bucket_off,
    const int32_t* __restrict__ active_pairs, const int32_t* __restrict__ n_active, int d, int f,
    int ksplit, int64_t n_assign_cap, float* __restrict__ part, int32_t* __restrict__ counters,
    uint16_t* __restrict__ h) {
  const int zslot = blockIdx.z;
  if (zslot >= *n_active) return;
  const int p = active_pairs[zslot];
  const PairTokens pt = pair_tokens(bucket_off, p);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, tig = lane & 3;
  const int frow_cta = blockIdx.x * (kWarps * 16);
  const int frow0 = frow_cta + warp * 16;
  const int kchunk = d / ksplit;
  const int kbeg = blockIdx.y * kchunk, kend = kbeg + kchunk;
  const uint16_t* Wg = w13 + ((size_t)p * 2 + 0) * (size_t)f * d + (size_t)(frow0 + g) * d + 8 * tig;
  const uint16_t* Wu = w13 + ((size_t)p * 2 + 1) * (size_t)f * d + (size_t)(frow0 + g) * d + 8 * tig;
  const size_t row8 = (size_t)8 * d;

  const int maxcnt = max(pt.cnt0, pt.cnt1);
  for (int base = 0; base < maxcnt; base += 8 * NT) {
    const int n0 = min(max(pt.cnt0 - base, 0), 8 * NT);
    const int n1 = min(max(pt.cnt1 - base, 0), 8 * NT);
    // activation row pointers for this lane's token (column g of each n-tile)
    const uint16_t* xp0[NT];
    const uint16_t* xp1[NT];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      int i0 = min(base + nt * 8 + g, max(pt.cnt0 - 1, 0));
      int i1 = min(base + nt * 8 + g, max(pt.cnt1 - 1, 0));
      const int a0 = pt.off0 + i0, a1 = pt.off1 + i1;
      // rows of empty buckets are never dereferenced (the MMA loop is skipped)
      const int r0 = pt.cnt0 == 0 ? 0 : (row_index ? row_index[a0] : a0);
      const int r1 = pt.cnt1 == 0 ? 0 : (row_index ? row_index[a1] : a1);
      xp0[nt] = x + (size_t)r0 * d + 8 * tig;
      xp1[nt] = x + (size_t)r1 * d + 8 * tig;
    }
    float ag0[NT][4], au0[NT][4], ag1[NT][4], au1[NT][4];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int q = 0; q < 4; ++q) ag0[nt][q] = au0[nt][q] = ag1[nt][q] = au1[nt][q] = 0.f;

    // software pipeline: weights of iteration k+64 are in flight while k is consumed
    uint4 wg[2][2], wu[2][2];  // [sub-chunk][row g / row g+8]
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      wg[s][0] = ldg_nc_v4(Wg + kbeg + 32 * s);
      wg[s][1] = ldg_nc_v4(Wg + row8 + kbeg + 32 * s);
      wu[s][0] = ldg_nc_v4(Wu + kbeg + 32 * s);
      wu[s][1] = ldg_nc_v4(Wu + row8 + kbeg + 32 * s);
    }
    for (int k0 = kbeg; k0 < kend; k0 += kKStep) {
      uint4 cg[2][2], cu[2][2];
#pragma unroll
      for (int s = 0; s < 2; ++s)
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          cg[s][r] = wg[s][r];
          cu[s][r] = wu[s][r];
        }
      if (k0 + kKStep < kend) {
        const int kn = k0 + kKStep;
#pragma unroll
        for (int s = 0; s < 2; ++s) {
          wg[s][0] = ldg_nc_v4(Wg + kn + 32 * s);
          wg[s][1] = ldg_nc_v4(Wg + row8 + kn + 32 * s);
          wu[s][0] = ldg_nc_v4(Wu + kn + 32 * s);
          wu[s][1] = ldg_nc_v4(Wu + row8 + kn + 32 * s);
        }
      }
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        const int kk = k0 + 32 * s;
        const uint32_t gl[4] = {cg[s][0].x, cg[s][0].y, cg[s][0].z, cg[s][0].w};
        const uint32_t gh[4] = {cg[s][1].x, cg[s][1].y, cg[s][1].z, cg[s][1].w};
        const uint32_t ul[4] = {cu[s][0].x, cu[s][0].y, cu[s][0].z, cu[s][0].w};
        const uint32_t uh[4] = {cu[s][1].x, cu[s][1].y, cu[s][1].z, cu[s][1].w};
        uint32_t bgl[4], bgh[4], bul[4], buh[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          bgl[q] = decode_base(gl[q]);
          bgh[q] = decode_base(gh[q]);
          bul[q] = decode_base(ul[q]);
          buh[q] = decode_base(uh[q]);
        }
        if (n0 > 0) {
          // MMA#0 uses words {0,1}; MMA#1 uses words {2,3}
          const uint32_t g00 = decode2<0>(gl[0], bgl[0]), g01 = decode2<0>(gh[0], bgh[0]);
          const uint32_t g02 = decode2<0>(gl[1], bgl[1]), g03 = decode2<0>(gh[1], bgh[1]);
          const uint32_t g10 = decode2<0>(gl[2], bgl[2]), g11 = decode2<0>(gh[2], bgh[2]);
          const uint32_t g12 = decode2<0>(gl[3], bgl[3]), g13 = decode2<0>(gh[3], bgh[3]);
          const uint32_t u00 = decode2<0>(ul[0], bul[0]), u01 = decode2<0>(uh[0], buh[0]);
          const uint32_t u02 = decode2<0>(ul[1], bul[1]), u03 = decode2<0>(uh[1], buh[1]);
          const uint32_t u10 = decode2<0>(ul[2], bul[2]), u11 = decode2<0>(uh[2], buh[2]);
          const uint32_t u12 = decode2<0>(ul[3], bul[3]), u13 = decode2<0>(uh[3], buh[3]);
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            if (nt * 8 < n0) {
              const uint4 xv = ldg_v4(xp0[nt] + kk);
              mma_bf16_16816(ag0[nt], g00, g01, g02, g03, xv.x, xv.y);
              mma_bf16_16816(ag0[nt], g10, g11, g12, g13, xv.z, xv.w);
              mma_bf16_16816(au0[nt], u00, u01, u02, u03, xv.x, xv.y);
              mma_bf16_16816(au0[nt], u10, u11, u12, u13, xv.z, xv.w);
            }
          }
        }
        if (n1 > 0) {
          const uint32_t g00 = decode2<1>(gl[0], bgl[0]), g01 = decode2<1>(gh[0], bgh[0]);
          const uint32_t g02 = decode2<1>(gl[1], bgl[1]), g03 = decode2<1>(gh[1], bgh[1]);
          const uint32_t g10 = decode2<1>(gl[2], bgl[2]), g11 = decode2<1>(gh[2], bgh[2]);
          const uint32_t g12 = decode2<1>(gl[3], bgl[3]), g13 = decode2<1>(gh[3], bgh[3]);
          const uint32_t u00 = decode2<1>(ul[0], bul[0]), u01 = decode2<1>(uh[0], buh[0]);
          const uint32_t u02 = decode2<1>(ul[1], bul[1]), u03 = decode2<1>(uh[1], buh[1]);
          const uint32_t u10 = decode2<1>(ul[2], bul[2]), u11 = decode2<1>(uh[2], buh[2]);
          const uint32_t u12 = decode2<1>(ul[3], bul[3]), u13 = decode2<1>(uh[3], buh[3]);
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            if (nt * 8 < n1) {
              const uint4 xv = ldg_v4(xp1[nt] + kk);
              mma_bf16_16816(ag1[nt], g00, g01, g02, g03, xv.x, xv.y);
              mma_bf16_16816(ag1[nt], g10, g11, g12, g13, xv.z, xv.w);
              mma_bf16_16816(au1[nt], u00, u01, u02, u03, xv.x, xv.y);
              mma_bf16_16816(au1[nt], u10, u11, u12, u13, xv.z, xv.w);
            }
          }
        }
      }
    }
    // ---- epilogue: C fragment c0,c1 = (row g, tokens 2tig, 2tig+1); c2,c3 = row g+8 ----
    if (ksplit == 1) {
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int tok = nt * 8 + 2 * tig + (q & 1);
          const int row = frow0 + g + (q >> 1) * 8;
          if (tok < n0)
            h[(size_t)(pt.off0 + base + tok) * f + row] = f32_to_bf16_bits_rn(silu_mul(ag0[nt][q], au0[nt][q]));
          if (tok < n1)
            h[(size_t)(pt.off1 + base + tok) * f + row] = f32_to_bf16_bits_rn(silu_mul(ag1[nt][q], au1[nt][q]));
        }
    } else {
      float* pk = part + (size_t)blockIdx.y * n_assign_cap * 2 * f;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int tok = nt * 8 + 2 * tig + (q & 1);
          const int row = frow0 + g + (q >> 1) * 8;
          if (tok < n0) {
            float* dst = pk + (size_t)(pt.off0 + base + tok) * 2 * f;
            dst[row] = ag0[nt][q];
            dst[f + row] = au0[nt][q];
          }
          if (tok < n1) {
            float* dst = pk + (size_t)(pt.off1 + base + tok) * 2 * f;
            dst[row] = ag1[nt][q];
            dst[f + row] = au1[nt][q];
          }
        }
    }
  }
  if (ksplit == 1) return;
  // ---- split-K: the last CTA of this (pair, row block) reduces in fixed split order ----
  __shared__ int s_last;
  __threadfence();  // every thread publishes its partial stores before the arrival count
  __syncthreads();
  if (threadIdx.x == 0) {
    const int idx = p * gridDim.x + blockIdx.x;
    const int prev = atomicAdd(&counters[idx], 1);
    s_last = (prev == ksplit - 1);
    if (s_last) counters[idx] = 0;  // reset for the next call (stream-ordered)
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const int nrows = kWarps * 16;
  const int n_tot = pt.cnt0 + pt.cnt1;  // buckets 2p and 2p+1 are adjacent
  for (int i = threadIdx.x; i < n_tot * nrows; i += blockDim.x) {
    const int a = pt.off0 + i / nrows;
    const int row = frow_cta + i % nrows;
    float gs = 0.f, us = 0.f;
    for (int s = 0; s < ksplit; ++s) {
      const float* src = part + ((size_t)s * n_assign_cap + a) * 2 * f;
      gs += __ldcg(src + row);
      us += __ldcg(src + f + row);
    }
    h[(size_t)a * f + row] = f32_to_bf16_bits_rn(silu_mul(gs, us));
  }
}

// Down projection: one 16-row m-tile (d_model rows) per warp, K = d_ff, B = h rows.
template <int NT>
__global__ void __launch_bounds__(kThreads) k_w2_gemv(
    const uint16_t* __restrict__ w2, const uint16_t* __restrict__ h,
    const int32_t* __restrict__ bucket_off, const int32_t* __restrict__ active_pairs,
    const int32_t* __restrict__ n_active, int d, int f, int ksplit, int64_t n_assign_cap,
    float* __restrict__ part, int32_t* __restrict__ counters, float* __restrict__ y) {
  const int zslot = blockIdx.z;
  if (zslot >= *n_active) return;
  const int p = active_pairs[zslot];
  const PairTokens pt = pair_tokens(bucket_off, p);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, tig = lane & 3;
  const int row_cta = blockIdx.x * (kWarps * 16);
  const int row0 = row_cta + warp * 16;
  const int kchunk = f / ksplit;
  const int kbeg = blockIdx.y * kchunk, kend = kbeg + kchunk;
  const uint16_t* W = w2 + (size_t)p * d * f + (size_t)(row0 + g) * f + 8 * tig;
  const size_t row8 = (size_t)8 * f;

  const int maxcnt = max(pt.cnt0, pt.cnt1);
  for (int base = 0; base < maxcnt; base += 8 * NT) {
    const int n0 = min(max(pt.cnt0 - base, 0), 8 * NT);
    const int n1 = min(max(pt.cnt1 - base, 0), 8 * NT);
    const uint16_t* hp0[NT];
    const uint16_t* hp1[NT];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      const int i0 = min(base + nt * 8 + g, max(pt.cnt0 - 1, 0));
      const int i1 = min(base + nt * 8 + g, max(pt.cnt1 - 1, 0));
      hp0[nt] = h + (size_t)(pt.off0 + i0) * f + 8 * tig;
      hp1[nt] = h + (size_t)(pt.off1 + i1) * f + 8 * tig;
    }
    float a0[NT][4], a1[NT][4];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int q = 0; q < 4; ++q) a0[nt][q] = a1[nt][q] = 0.f;

    uint4 w[2][2];
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      w[s][0] = ldg_nc_v4(W + kbeg + 32 * s);
      w[s][1] = ldg_nc_v4(W + row8 + kbeg + 32 * s);
    }
    for (int k0 = kbeg; k0 < kend; k0 += kKStep) {
      uint4 c[2][2];
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        c[s][0] = w[s][0];
        c[s][1] = w[s][1];
      }
      if (k0 + kKStep < kend) {
#pragma unroll
        for (int s = 0; s < 2; ++s) {
          w[s][0] = ldg_nc_v4(W + k0 + kKStep + 32 * s);
          w[s][1] = ldg_nc_v4(W + row8 + k0 + kKStep + 32 * s);
        }
      }
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        const int kk = k0 + 32 * s;
        const uint32_t wl[4] = {c[s][0].x, c[s][0].y, c[s][0].z, c[s][0].w};
        const uint32_t wh[4] = {c[s][1].x, c[s][1].y, c[s][1].z, c[s][1].w};
        uint32_t bl[4], bh[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          bl[q] = decode_base(wl[q]);
          bh[q] = decode_base(wh[q]);
        }
        if (n0 > 0) {
          const uint32_t x00 = decode2<0>(wl[0], bl[0]), x01 = decode2<0>(wh[0], bh[0]);
          const uint32_t x02 = decode2<0>(wl[1], bl[1]), x03 = decode2<0>(wh[1], bh[1]);
          const uint32_t x10 = decode2<0>(wl[2], bl[2]), x11 = decode2<0>(wh[2], bh[2]);
          const uint32_t x12 = decode2<0>(wl[3], bl[3]), x13 = decode2<0>(wh[3], bh[3]);
#pragma unroll
          for (int nt = 0; nt < NT; ++nt)
            if (nt * 8 < n0) {
              const uint4 hv = ldg_v4(hp0[nt] + kk);
              mma_bf16_16816(a0[nt], x00, x01, x02, x03, hv.x, hv.y);
              mma_bf16_16816(a0[nt], x10, x11, x12, x13, hv.z, hv.w);
            }
        }
        if (n1 > 0) {
          const uint32_t x00 = decode2<1>(wl[0], bl[0]), x01 = decode2<1>(wh[0], bh[0]);
          const uint32_t x02 = decode2<1>(wl[1], bl[1]), x03 = decode2<1>(wh[1], bh[1]);
          const uint32_t x10 = decode2<1>(wl[2], bl[2]), x11 = decode2<1>(wh[2], bh[2]);
          const uint32_t x12 = decode2<1>(wl[3], bl[3]), x13 = decode2<1>(wh[3], bh[3]);
#pragma unroll
          for (int nt = 0; nt < NT; ++nt)
            if (nt * 8 < n1) {
              const uint4 hv = ldg_v4(hp1[nt] + kk);
              mma_bf16_16816(a1[nt], x00, x01, x02, x03, hv.x, hv.y);
              mma_bf16_16816(a1[nt], x10, x11, x12, x13, hv.z, hv.w);
            }
        }
      }
    }
    float* dstbase = ksplit == 1 ? y : part + (size_t)blockIdx.y * n_assign_cap * d;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int tok = nt * 8 + 2 * tig + (q & 1);
        const int row = row0 + g + (q >> 1) * 8;
        if (tok < n0) dstbase[(size_t)(pt.off0 + base + tok) * d + row] = a0[nt][q];
        if (tok < n1) dstbase[(size_t)(pt.off1 + base + tok) * d + row] = a1[nt][q];
      }
  }
  if (ksplit == 1) return;
  __shared__ int s_last;
  __threadfence();  // every thread publishes its partial stores before the arrival count
  __syncthreads();
  if (threadIdx.x == 0) {
    const int idx = p * gridDim.x + blockIdx.x;
    const int prev = atomicAdd(&counters[idx], 1);
    s_last = (prev == ksplit - 1);
    if (s_last) counters[idx] = 0;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const int nrows = kWarps * 16;
  const int n_tot = pt.cnt0 + pt.cnt1;
  for (int i = threadIdx.x; i < n_tot * nrows; i += blockDim.x) {
    const int a = pt.off0 + i / nrows;
    const int row = row_cta + i % nrows;
    float acc = 0.f;
    for (int s = 0; s < ksplit; ++s) acc += __ldcg(part + ((size_t)s * n_assign_cap + a) * d + row);
    y[(size_t)a * d + row] = acc;
  }
}

// Largest split count s <= want with (K / s) % kKStep == 0.
int pick_split(int K, int want) {
  int best = 1;
  for (int s = 1; s <= want; ++s)
    if (K % (s * kKStep) == 0) best = s;
  return best;
}

}  // namespace

int gemv_nt_for(int64_t T) { return T <= 8 ? 1 : (T <= 16 ? 2 : 4); }

// Split-K factor so that (row blocks x splits x active pairs) CTAs give >= ~4 waves.
void gemv_splits(int d, int f, int max_active, int* ks13, int* ks2) {
  const int target_ctas = num_sms() * 4 * 4;  // 4 CTAs of 4 warps per SM, 4 waves
  const int rb13 = f / (kWarps * 16), rb2 = d / (kWarps * 16);
  int want13 = (target_ctas + rb13 * max_active - 1) / (rb13 * max_active);
  int want2 = (target_ctas + rb2 * max_active - 1) / (rb2 * max_active);
  want13 = want13 < 1 ? 1 : (want13 > 8 ? 8 : want13);
  want2 = want2 < 1 ? 1 : (want2 > 16 ? 16 : want2);
  // keep at least 256 of K per split
  while (want13 > 1 && d / want13 < 256) --want13;
  while (want2 > 1 && f / want2 < 256) --want2;
  *ks13 = pick_split(d, want13);
  *ks2 = pick_split(f, want2);
}

int launch_gemv_experts(const uint16_t* w13, const uint16_t* w2, int n_pairs, int d, int f,
                        const uint16_t* x, const int32_t* row_index, const int32_t* bucket_off,
                        const int32_t* active_pairs, const int32_t* n_active, int max_active,
                        int64_t n_assign_cap, int nt, int ks13, int ks2, float* part13,
                        float* part2, int32_t* counters13, int32_t* counters2, uint16_t* h,
                        float* y, cudaStream_t stream) {
  (void)n_pairs;
  if (max_active == 0) return PUZZLE_OK;
  dim3 g13(f / (kWarps * 16), ks13, max_active);
  dim3 g2(d / (kWarps * 16), ks2, max_active);
#define PZ_LAUNCH13(NT)                                                                        \
  ProfScope _ps13("w13_gemv", stream);                                                         \
  k_w13_gemv<NT><<<g13, kThreads, 0, stream>>>(w13, x, row_index, bucket_off, active_pairs,    \
                                               n_active, d, f, ks13, n_assign_cap, part13,     \
                                               counters13, h)
#define PZ_LAUNCH2(NT)                                                                               \
  ProfScope _ps2("w2_gemv", stream);                                                                 \
  k_w2_gemv<NT><<<g2, kThreads, 0, stream>>>(w2, h, bucket_off, active_pairs, n_active, d, f, ks2, \
                                             n_assign_cap, part2, counters2, y)
  if (nt == 1) {
    { PZ_LAUNCH13(1); }
    { PZ_LAUNCH2(1); }
  } else if (nt == 2) {
    { PZ_LAUNCH13(2); }
    { PZ_LAUNCH2(2); }
  } else {
    { PZ_LAUNCH13(4); }
    { PZ_LAUNCH2(4); }
  }
#undef PZ_LAUNCH13
#undef PZ_LAUNCH2
  return cuda_check(cudaGetLastError(), "gemv launch");
}

}  // namespace pz
