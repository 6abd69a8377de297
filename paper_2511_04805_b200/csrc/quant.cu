// NEXT-3 packer pair: the quantised PuzzleMoE format (Appendix A.3; DESIGN.md
// readings R21-R23). Both kernels are elementwise / group-local and HBM-bound.
//   quant pack: one warp per group of 128 merged magnitudes (4 per lane, 16-byte loads):
//     warp max -> scale = max / 7 (f32, 1 for an all-zero group) -> code = round-half-even of
//     the exact 7 w / max (an f64 estimate plus one exact f64 boundary test, no division per
//     element; bit-identical to the oracle's f64 rint) -> one byte per element
//     S_i S_j M_i M_j 0 c2 c1 c0.
//   quant unpack: byte -> (-1)^S_pos M_pos bf16_rne(f32(code * scale)), 16 elements per thread.
#include "common.cuh"

namespace pz {

namespace {

constexpr int kQThreads = 256;

__global__ void __launch_bounds__(kQThreads) k_quant_pack(const float4* __restrict__ w, const uchar4* __restrict__ m0,
                                                          const uchar4* __restrict__ m1, const uchar4* __restrict__ s0,
                                                          const uchar4* __restrict__ s1, int64_t n_groups,
                                                          uchar4* __restrict__ codes, float* __restrict__ scales) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (kQThreads / 32);
  for (int64_t grp = blockIdx.x * (int64_t)(kQThreads / 32) + (threadIdx.x >> 5); grp < n_groups; grp += warps) {
    const int64_t i = grp * 32 + lane;  // this lane's 4 elements
    const float4 v = w[i];
    float mx = fmaxf(fmaxf(v.x, v.y), fmaxf(v.z, v.w));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    mx = fmaxf(mx, 0.0f);
    if (lane == 0) scales[grp] = mx == 0.0f ? 1.0f : __fdiv_rn(mx, 7.0f);
    const uchar4 a = m0[i], b = m1[i], c = s0[i], d = s1[i];
    const float vv[4] = {v.x, v.y, v.z, v.w};
    const uint8_t fa[4] = {a.x, a.y, a.z, a.w}, fb[4] = {b.x, b.y, b.z, b.w};
    const uint8_t fc[4] = {c.x, c.y, c.z, c.w}, fd[4] = {d.x, d.y, d.z, d.w};
    // code = round-half-even(7 w / max) without a division per element: the estimate
    // y = w * (7 / max) (f64, one division per group; finite even for a subnormal max) is within
    // a few ulps of the exact quotient x, so x lies in [j - 0.5, j + 1.5) for j = floor(y) and
    // only the boundary j + 1/2 needs an exact test -- 14 w against (2j + 1) max, both exact
    // in f64 (24-bit mantissas times 4-bit integers)
    const double mxd = (double)mx;
    const double r7 = mx == 0.0f ? 0.0 : __ddiv_rn(7.0, mxd);
    uint8_t out[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      int code = 0;
      if (mx != 0.0f) {
        const double y = (double)vv[k] * r7;
        const int j = (int)fmin(fmax(floor(y), -1.0), 7.0);  // codes clamp to [0, 7] anyway
        const double lhs = 14.0 * (double)vv[k], rhs = (double)(2 * j + 1) * mxd;
        code = j + (lhs > rhs ? 1 : 0) + ((lhs == rhs && (j & 1)) ? 1 : 0);
        code = min(max(code, 0), 7);
      }
      out[k] = (uint8_t)(((fc[k] != 0) << 7) | ((fd[k] != 0) << 6) | ((fa[k] != 0) << 5) | ((fb[k] != 0) << 4) |
                         code);
    }
    codes[i] = make_uchar4(out[0], out[1], out[2], out[3]);
  }
}

template <int POS>
__device__ __forceinline__ uint32_t dequant_one(uint32_t byte, float scale) {
  const uint32_t h = f32_to_bf16_rne_bits(__fmul_rn((float)(byte & 7u), scale));
  const uint32_t sign = (byte >> (7 - POS)) & 1u, mask = (byte >> (5 - POS)) & 1u;
  return mask ? (h | (sign << 15)) : 0u;
}

template <int POS>
__device__ __forceinline__ uint32_t dequant_word(uint32_t four, float sc, int half) {  // 2 of 4 bytes -> bf16x2
  const uint32_t b0 = (four >> (16 * half)) & 0xFFu, b1 = (four >> (16 * half + 8)) & 0xFFu;
  return dequant_one<POS>(b0, sc) | (dequant_one<POS>(b1, sc) << 16);
}

// 16 codes (one 16-byte load, inside one 128-group) -> 16 bf16 (two 16-byte stores) per thread
template <int POS>
__global__ void __launch_bounds__(kQThreads) k_quant_unpack(const uint4* __restrict__ codes,
                                                            const float* __restrict__ scales, int64_t n16,
                                                            uint4* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n16; i += (int64_t)gridDim.x * blockDim.x) {
    const uint4 b = ldg_nc_v4(codes + i);
    const float sc = __ldg(scales + (i >> 3));  // 8 threads per 128-group
    out[2 * i] = make_uint4(dequant_word<POS>(b.x, sc, 0), dequant_word<POS>(b.x, sc, 1),
                            dequant_word<POS>(b.y, sc, 0), dequant_word<POS>(b.y, sc, 1));
    out[2 * i + 1] = make_uint4(dequant_word<POS>(b.z, sc, 0), dequant_word<POS>(b.z, sc, 1),
                                dequant_word<POS>(b.w, sc, 0), dequant_word<POS>(b.w, sc, 1));
  }
}

// NEXT-3 expert GEMV over the quantised format (R23): the tokens routed to expert i of the pair
// see Ŵ_0, those routed to j see Ŵ_1, both from ONE decode of the code bytes (the magnitude
// bf16_rne(code * scale) is shared, only the sign / mask bits differ per position). Work item =
// (row pair, chunk of up to TB tokens of i and TB of j); one warp per item. Each lane takes 16
// codes of each of the 2 rows per step (one 16-byte load per row, inside one 128-group; the next
// step's loads are issued before this step's math), rounds the 32 magnitudes with 16
// cvt.rn.bf16x2.f32, then per position applies the sign / mask bits and FMAs against that
// position's tokens (f32, sequential per lane over its cols / 32 columns); the sums are
// warp-reduced (5 butterfly levels). CUDA cores, not tcgen05: at decode batch sizes the code
// bytes (1 per merged element) are the traffic and the per-byte decode is the ALU work.
// tokens per position per work item (TB): 1 or 2 for decode-sized inputs (fewer accumulator
// registers: TB = 1 fits 3 CTAs per SM), 4 otherwise (fewer re-decodes of the codes per token)

__device__ __forceinline__ uint32_t cvt_bf16x2(float hi, float lo) {
  uint32_t d;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(hi), "f"(lo));
  return d;
}

// 16 codes (4 words) x scale -> 16 f32 magnitudes (bf16-rounded), element e = byte e
__device__ __forceinline__ void decode_mag16(const uint32_t q[4], float s, uint32_t* mag) {
#pragma unroll
  for (int w = 0; w < 4; ++w) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const float lo = __fmul_rn((float)((q[w] >> (16 * h)) & 7u), s);
      const float hi = __fmul_rn((float)((q[w] >> (16 * h + 8)) & 7u), s);
      const uint32_t d = cvt_bf16x2(hi, lo);
      mag[4 * w + 2 * h] = d << 16;
      mag[4 * w + 2 * h + 1] = d & 0xFFFF0000u;
    }
  }
}

// signed, masked weight of element e (byte e of q) at position POS from its magnitude bits
template <int POS>
__device__ __forceinline__ float signed_w(const uint32_t q[4], const uint32_t* mag, int e) {
  const uint32_t byte = (q[e >> 2] >> (8 * (e & 3))) & 0xFFu;
  const uint32_t sign = (byte << (24 + POS)) & 0x80000000u;
  return ((byte >> (5 - POS)) & 1u) ? __uint_as_float(mag[e] | sign) : 0.0f;
}

__device__ __forceinline__ void bf16x8_to_f32(uint4 v, float* f) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    f[2 * k] = __uint_as_float(w[k] << 16);
    f[2 * k + 1] = __uint_as_float(w[k] & 0xFFFF0000u);
  }
}

template <int POS, int TB>
__device__ __forceinline__ void fma_tokens(const uint32_t q0[4], const uint32_t q1[4], const uint32_t* m0,
                                           const uint32_t* m1, const uint16_t* __restrict__ x, int64_t cols,
                                           int64_t c, int nt, float (*acc)[TB]) {
  float w0[16], w1[16];
#pragma unroll
  for (int e = 0; e < 16; ++e) {
    w0[e] = signed_w<POS>(q0, m0, e);
    w1[e] = signed_w<POS>(q1, m1, e);
  }
#pragma unroll
  for (int t = 0; t < TB; ++t) {
    if (t < nt) {
      const uint4* xp = reinterpret_cast<const uint4*>(x + t * cols + c);
      float xf[16];
      bf16x8_to_f32(__ldg(xp), xf);
      bf16x8_to_f32(__ldg(xp + 1), xf + 8);
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        acc[0][t] = __fmaf_rn(w0[e], xf[e], acc[0][t]);
        acc[1][t] = __fmaf_rn(w1[e], xf[e], acc[1][t]);
      }
    }
  }
}

template <int TB>
__device__ __forceinline__ void store_sums(float (*acc)[TB], int nt, int lane, float* y, int64_t rows,
                                           int64_t r0, bool has1) {
#pragma unroll
  for (int t = 0; t < TB; ++t) {
    if (t < nt) {  // nt is warp-uniform
      float a = acc[0][t], b = acc[1][t];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        b += __shfl_xor_sync(0xffffffffu, b, o);
      }
      if (lane == 0) {
        y[t * rows + r0] = a;
        if (has1) y[t * rows + r0 + 1] = b;
      }
    }
  }
}

template <int TB>
__global__ void __launch_bounds__(kQThreads, TB == 1 ? 3 : 2) k_quant_gemv(const uint8_t* __restrict__ codes,
                                                          const float* __restrict__ scales, int64_t rows,
                                                          int64_t cols, const uint16_t* __restrict__ x_i,
                                                          int64_t n_i, const uint16_t* __restrict__ x_j,
                                                          int64_t n_j, float* __restrict__ y_i,
                                                          float* __restrict__ y_j) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (kQThreads / 32);
  const int64_t nch = ((n_i > n_j ? n_i : n_j) + TB - 1) / TB;
  const int64_t n_rp = (rows + 1) / 2, gpr = cols / 128;
  for (int64_t item = blockIdx.x * (int64_t)(kQThreads / 32) + (threadIdx.x >> 5); item < n_rp * nch;
       item += warps) {
    const int64_t rp = item / nch, t0 = (item % nch) * TB;
    const int nti = (int)(n_i - t0 <= 0 ? 0 : (n_i - t0 < TB ? n_i - t0 : TB));
    const int ntj = (int)(n_j - t0 <= 0 ? 0 : (n_j - t0 < TB ? n_j - t0 : TB));
    const int64_t r0 = 2 * rp, r1 = r0 + 1 < rows ? r0 + 1 : r0;
    const uint8_t* c0 = codes + r0 * cols;
    const uint8_t* c1 = codes + r1 * cols;
    const uint16_t* xi = x_i + t0 * cols;
    const uint16_t* xj = x_j + t0 * cols;
    float ai[2][TB], aj[2][TB];
#pragma unroll
    for (int t = 0; t < TB; ++t) ai[0][t] = ai[1][t] = aj[0][t] = aj[1][t] = 0.0f;
    int64_t c = lane * 16;
    uint4 b0 = make_uint4(0, 0, 0, 0), b1 = b0;
    float s0 = 0.0f, s1 = 0.0f;
    if (c < cols) {
      b0 = ldg_nc_v4(c0 + c), b1 = ldg_nc_v4(c1 + c);
      s0 = __ldg(scales + r0 * gpr + (c >> 7)), s1 = __ldg(scales + r1 * gpr + (c >> 7));
    }
    for (; c < cols; c += 512) {
      const uint32_t q0[4] = {b0.x, b0.y, b0.z, b0.w}, q1[4] = {b1.x, b1.y, b1.z, b1.w};
      const float cs0 = s0, cs1 = s1;
      if (c + 512 < cols) {  // next step's codes in flight during this step's math
        b0 = ldg_nc_v4(c0 + c + 512), b1 = ldg_nc_v4(c1 + c + 512);
        s0 = __ldg(scales + r0 * gpr + ((c + 512) >> 7)), s1 = __ldg(scales + r1 * gpr + ((c + 512) >> 7));
      }
      uint32_t m0[16], m1[16];
      decode_mag16(q0, cs0, m0);
      decode_mag16(q1, cs1, m1);
      if (nti > 0) fma_tokens<0, TB>(q0, q1, m0, m1, xi, cols, c, nti, ai);
      if (ntj > 0) fma_tokens<1, TB>(q0, q1, m0, m1, xj, cols, c, ntj, aj);
    }
    store_sums(ai, nti, lane, y_i + t0 * rows, rows, r0, r0 + 1 < rows);
    store_sums(aj, ntj, lane, y_j + t0 * rows, rows, r0, r0 + 1 < rows);
  }
}

int qgrid(int64_t items, int per_cta) {
  int64_t blocks = (items + per_cta - 1) / per_cta;
  const int64_t cap = (int64_t)num_sms() * 8;
  return (int)std::max<int64_t>(1, std::min<int64_t>(blocks, cap));
}

}  // namespace

// w: f32 [rows][cols], planes u8 [rows][cols], cols % 128 == 0, 16-byte aligned (checked by the caller)
int launch_quant_pack(const float* w, const uint8_t* m0, const uint8_t* m1, const uint8_t* s0, const uint8_t* s1,
                      int64_t rows, int64_t cols, uint8_t* codes, float* scales, cudaStream_t stream) {
  const int64_t n_groups = rows * (cols / 128);
  if (n_groups == 0) return PUZZLE_OK;
  {
    ProfScope _ps("quant_pack", stream);
    k_quant_pack<<<qgrid(n_groups, kQThreads / 32), kQThreads, 0, stream>>>(
        reinterpret_cast<const float4*>(w), reinterpret_cast<const uchar4*>(m0), reinterpret_cast<const uchar4*>(m1),
        reinterpret_cast<const uchar4*>(s0), reinterpret_cast<const uchar4*>(s1), n_groups,
        reinterpret_cast<uchar4*>(codes), scales);
  }
  return cuda_check(cudaGetLastError(), "puzzle_quant_pack launch");
}

int launch_quant_unpack(const uint8_t* codes, const float* scales, int pos, int64_t rows, int64_t cols, uint16_t* out,
                        cudaStream_t stream) {
  const int64_t n16 = rows * cols / 16;
  if (n16 == 0) return PUZZLE_OK;
  {
    ProfScope _ps("quant_unpack", stream);
    auto kern = pos == 0 ? k_quant_unpack<0> : k_quant_unpack<1>;
    kern<<<qgrid(n16, kQThreads), kQThreads, 0, stream>>>(reinterpret_cast<const uint4*>(codes), scales, n16,
                                                          reinterpret_cast<uint4*>(out));
  }
  return cuda_check(cudaGetLastError(), "puzzle_quant_unpack launch");
}

// codes u8 [rows][cols] (cols % 128 == 0, 16-byte aligned), scales f32 [rows][cols/128],
// x_i / x_j bf16 [n][cols] (16-byte aligned), y_i / y_j f32 [n][rows]
int launch_quant_gemv(const uint8_t* codes, const float* scales, int64_t rows, int64_t cols, const uint16_t* x_i,
                      int64_t n_i, const uint16_t* x_j, int64_t n_j, float* y_i, float* y_j, cudaStream_t stream) {
  const int64_t nmax = std::max(n_i, n_j);
  const int tb = nmax <= 1 ? 1 : nmax <= 2 ? 2 : 4;
  const int64_t items = (rows + 1) / 2 * ((std::max(n_i, n_j) + tb - 1) / tb);
  if (items == 0) return PUZZLE_OK;
  {
    ProfScope _ps("quant_gemv", stream);
    auto kern = tb == 1 ? k_quant_gemv<1> : tb == 2 ? k_quant_gemv<2> : k_quant_gemv<4>;
    kern<<<qgrid(items, kQThreads / 32), kQThreads, 0, stream>>>(codes, scales, rows, cols, x_i, n_i, x_j, n_j, y_i,
                                                                 y_j);
  }
  return cuda_check(cudaGetLastError(), "puzzle_quant_gemv launch");
}

}  // namespace pz
