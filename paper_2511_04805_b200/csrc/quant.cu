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

}  // namespace pz
