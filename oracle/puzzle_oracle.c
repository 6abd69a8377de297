/*
 * PuzzleMoE CPU ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * This file is the plain, slow, obviously-correct CPU statement of what the
 * B200 hot path computes. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it. It shares no code, header,
 * table or constant generator with paper_2511_04805_b200/csrc (the CUDA path),
 * and neither side includes or links the other.
 *
 * Citations: "P:n" = PAPER.md line n (arXiv 2511.04805 LaTeX source);
 *            "S:n" = SPEC.md line n. Equation numbers follow SURVEY.md §0.
 *
 * Build: gcc -O2 -fno-fast-math -ffp-contract=off -fopenmp -shared -fPIC
 * (no contraction: every f32 expression below is evaluated as written).
 *
 * Parity status per function:
 *   oracle_bf16_round   pinned (torch CPU RNE sweep, halfway cases)
 *   oracle_merge        pinned (SPEC 2x2 worked example, identity merges,
 *                               App. B closed form, error bounds)
 *   oracle_pack         pinned (SPEC golden words, exhaustive bijection)
 *   oracle_unpack       pinned (exhaustive 2^16 x 2 vs byte-literal Alg. 1)
 *   oracle_route        pinned (torch.topk / torch.softmax library routines)
 *   oracle_moe_forward  pinned (self-merge == dense torch f64 FFN, top-1 gate
 *                               == 1, token-permutation equivariance; dense
 *                               slots == torch f64 FFN of the bf16 weights)
 *   oracle_quant_pack / oracle_quant_unpack  pinned (SPEC worked example
 *                               S:478, all-zero group, round-trip bound, masks
 *                               exactly zero, byte layout)
 *   oracle_calib_sumsq  pinned (numpy column norms of the routed rows, torch
 *                               f64 SwiGLU intermediate, duplicate-token scaling)
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------------ */
/* O1. bfloat16 bit helpers (1 sign, 8 exponent, 7 mantissa bits).    */
/* ------------------------------------------------------------------------ */

static uint32_t f32_bits(float x) {
  uint32_t u;
  memcpy(&u, &x, 4);
  return u;
}

static float bits_f32(uint32_t u) {
  float x;
  memcpy(&x, &u, 4);
  return x;
}

/* f32 -> bf16, round-to-nearest-even on the dropped 16 bits (the paper never
 * states a rounding mode; S:101 and DESIGN.md reading R3 fix RNE). */
static uint16_t bf16_rne(float x) {
  uint32_t u = f32_bits(x);
  uint32_t lsb = (u >> 16) & 1u;
  if ((u & 0x7FFFFFFFu) > 0x7F800000u) return (uint16_t)((u >> 16) | 0x40u); /* NaN stays a quiet NaN (IEEE) */
  return (uint16_t)((u + 0x7FFFu + lsb) >> 16);
}

static double bf16_to_double(uint16_t h) { return (double)bits_f32((uint32_t)h << 16); }

int oracle_bf16_round(const float* in, int64_t n, uint16_t* out) {
  for (int64_t i = 0; i < n; ++i) out[i] = bf16_rne(in[i]);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* O2. Pairwise dual-mask merge, Eq. 1-7, one linear slot.         */
/*     W_i, W_j are (rows x cols) = (out x in) row-major. norms_i/j    */
/*     have length cols: ||X||_2 per input column, broadcast over rows        */
/*     (Eq. 4). All arithmetic IEEE f32.            */
/* ------------------------------------------------------------------------ */
int oracle_merge(const float* w_i, const float* w_j, const float* norms_i, const float* norms_j,
                 int64_t rows, int64_t cols, float tau_sim,
                 float* w_merged, uint8_t* m_sim, uint8_t* m_sal_i, uint8_t* m_i, uint8_t* m_j,
                 uint8_t* s_i, uint8_t* s_j) {
  if (!(tau_sim >= 0.0f && tau_sim <= 1.0f)) return 1; /* tau in [0,1] */
  for (int64_t r = 0; r < rows; ++r) {
    for (int64_t c = 0; c < cols; ++c) {
      int64_t x = r * cols + c;
      float a = fabsf(w_i[x]);
      float b = fabsf(w_j[x]);
      /* Eq. 1: Delta = | |W_i| - |W_j| | / (|W_i| + |W_j|); 0/0 := 0 (reading R4) */
      float delta;
      if (a == 0.0f && b == 0.0f)
        delta = 0.0f;
      else
        delta = fabsf(a - b) / (a + b);
      /* Eq. 2: M^sim = 1{Delta <= tau_sim} */
      uint8_t sim = (delta <= tau_sim) ? 1 : 0;
      /* Eq. 3: S = 1{W < 0}  (-0.0 < 0 is false: reading R6) */
      uint8_t si = (w_i[x] < 0.0f) ? 1 : 0;
      uint8_t sj = (w_j[x] < 0.0f) ? 1 : 0;
      /* Eq. 4: A = |W| (.) ||X||_2 (per input column c) */
      float A_i = a * norms_i[c];
      float A_j = b * norms_j[c];
      /* Eq. 5: M^sal_i = 1{A_i >= A_j}; M^sal_j = 1 - M^sal_i (tie -> i) */
      uint8_t sal_i = (A_i >= A_j) ? 1 : 0;
      uint8_t sal_j = (uint8_t)(1 - sal_i);
      /* Eq. 6: M_i = M^sal_i OR M^sim; M_j = M^sal_j OR M^sim */
      uint8_t mi = (uint8_t)(sal_i | sim);
      uint8_t mj = (uint8_t)(sal_j | sim);
      /* Eq. 7: W_merged = M^sim (.) (|W_i|+|W_j|)/2
       *                 + (1-M^sim) (.) (M^sal_i (.) |W_i| + M^sal_j (.) |W_j|) */
      float wm;
      if (sim)
        wm = (a + b) * 0.5f;
      else
        wm = sal_i ? a : b;
      w_merged[x] = wm;
      if (m_sim) m_sim[x] = sim;
      if (m_sal_i) m_sal_i[x] = sal_i;
      m_i[x] = mi;
      m_j[x] = mj;
      s_i[x] = si;
      s_j[x] = sj;
    }
  }
  return 0;
}

/* ------------------------------------------------------------------------ */
/* O3. Pack (P:189-190 exponent shift; bit layout from Algorithm 1,           */
/*     P:196-209, confirmed by S:34):                                         */
/*   bit15 S_i | bit14 S_j | bit13 M_i | bit12 M_j | bits11-7 e' | bits6-0 m  */
/*   e' = clamp(e, 112, 143) - 112 ("any exponent smaller than 112 is rounded */
/*   up to 112, then all exponents are shifted down by 112").          */
/*   stats[0] = e < 112 (rounded up), stats[1] = e > 143 (saturated, R1),     */
/*   stats[2] = non-finite magnitude, stats[3] = negative magnitude.          */
/* ------------------------------------------------------------------------ */
int oracle_pack(const float* w_merged, const uint8_t* m0, const uint8_t* m1, const uint8_t* s0,
                const uint8_t* s1, int64_t n, uint16_t* out, uint64_t* stats) {
  uint64_t lo = 0, hi = 0, nonfinite = 0, negative = 0;
  for (int64_t x = 0; x < n; ++x) {
    float w = w_merged[x];
    if (!isfinite(w)) nonfinite++;
    if (w < 0.0f) negative++;
    uint16_t h = bf16_rne(w);           /* RNE before the clamp (R3) */
    uint32_t e = (h >> 7) & 0xFFu;      /* bf16 exponent field */
    uint32_t mant = h & 0x7Fu;          /* 7-bit mantissa, kept (R2) */
    if (e < 112u) { e = 112u; lo++; }
    if (e > 143u) { e = 143u; hi++; }
    uint32_t word = ((uint32_t)(s0[x] != 0) << 15) | ((uint32_t)(s1[x] != 0) << 14) |
                    ((uint32_t)(m0[x] != 0) << 13) | ((uint32_t)(m1[x] != 0) << 12) |
                    ((e - 112u) << 7) | mant;
    out[x] = (uint16_t)word;
  }
  if (stats) {
    stats[0] += lo;
    stats[1] += hi;
    stats[2] += nonfinite;
    stats[3] += negative;
  }
  return 0;
}

/* ------------------------------------------------------------------------ */
/* O4. Algorithm 1 "PuzzleMoE weight decoding", line by line.     */
/* ------------------------------------------------------------------------ */
static uint16_t decode_word(uint16_t W, int expert_pos) {
  /* line 1: mask_bit <- (W >> (13 - expert_pos)) & 1 */
  uint32_t mask_bit = ((uint32_t)W >> (13 - expert_pos)) & 1u;
  /* line 2-3: if mask_bit == 0: W_decoded <- 0 */
  if (mask_bit == 0) return 0;
  /* line 5: sign_bit <- (W >> (15 - expert_pos)) & 1 */
  uint32_t sign_bit = ((uint32_t)W >> (15 - expert_pos)) & 1u;
  /* line 6: exp <- (W & 0x0F80) + (112 << 7) */
  uint32_t exp = ((uint32_t)W & 0x0F80u) + (112u << 7);
  /* line 7: W_decoded <- (sign_bit << 15) | exp | (W & 0x007F) */
  return (uint16_t)((sign_bit << 15) | exp | ((uint32_t)W & 0x007Fu));
}

int oracle_unpack(const uint16_t* packed, int pos, int64_t n, uint16_t* out) {
  if (pos != 0 && pos != 1) return 1;
  for (int64_t x = 0; x < n; ++x) out[x] = decode_word(packed[x], pos);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* O4q. Quantised PuzzleMoE (NEXT-3; Appendix A.3): "the resultant */
/*      floating-point weights are subjected to uniform quantization with a   */
/*      group size of 128 ... symmetric group quantization ... no zero point;  */
/*      the final quantized values are stored alongside their corresponding   */
/*      sign and mask bits". Readings (R21-R23):                     */
/*   groups: 128 consecutive elements of a row (cols % 128 == 0);              */
/*   scale = max(group) / 7 in IEEE f32, or 1 if max == 0; code =     */
/*   rint(7 w / max) in f64 (= round(w / scale) in exact arithmetic, halves to  */
/*   even), clamped to [0, 7] (3-bit unsigned levels: W_merged >= 0);          */
/*   one byte per merged element: bit7 S_i | bit6 S_j | bit5 M_i | bit4 M_j |   */
/*   bit3 0 | bits2-0 code;                                                    */
/*   dequantised weight of position pos = (-1)^S_pos * M_pos * bf16_rne(f32(  */
/*   code * scale)) (the bf16 operand of the expert matmul).                   */
/* ------------------------------------------------------------------------ */
int oracle_quant_pack(const float* w_merged, const uint8_t* m0, const uint8_t* m1, const uint8_t* s0,
                      const uint8_t* s1, int64_t rows, int64_t cols, uint8_t* codes, float* scales) {
  if (cols % 128 != 0 || rows < 0) return 1;
  for (int64_t r = 0; r < rows; ++r) {
    for (int64_t g = 0; g < cols / 128; ++g) {
      const int64_t x0 = r * cols + g * 128;
      float mx = 0.0f;
      for (int i = 0; i < 128; ++i)
        if (w_merged[x0 + i] > mx) mx = w_merged[x0 + i];
      const float scale = mx == 0.0f ? 1.0f : mx / 7.0f;
      scales[r * (cols / 128) + g] = scale;
      for (int i = 0; i < 128; ++i) {
        const int64_t x = x0 + i;
        /* code = round(w / (max / 7)) evaluated as rint(7 w / max) in f64: 7 w is exact and the
         * one correctly rounded division keeps exact halves (2 / (4/7) = 3.5 -> 4) */
        double q = mx == 0.0f ? 0.0 : rint(7.0 * (double)w_merged[x] / (double)mx); /* half to even */
        if (q < 0.0) q = 0.0;
        if (q > 7.0) q = 7.0;
        codes[x] = (uint8_t)(((s0[x] != 0) << 7) | ((s1[x] != 0) << 6) | ((m0[x] != 0) << 5) |
                             ((m1[x] != 0) << 4) | (int)q);
      }
    }
  }
  return 0;
}

int oracle_quant_unpack(const uint8_t* codes, const float* scales, int pos, int64_t rows, int64_t cols,
                        uint16_t* out) {
  if (pos != 0 && pos != 1) return 1;
  if (cols % 128 != 0 || rows < 0) return 1;
  for (int64_t r = 0; r < rows; ++r)
    for (int64_t c = 0; c < cols; ++c) {
      const uint8_t b = codes[r * cols + c];
      const int sign = (b >> (7 - pos)) & 1;
      const int mask = (b >> (5 - pos)) & 1;
      const float v = (float)(b & 7) * scales[r * (cols / 128) + c / 128];
      const uint16_t h = bf16_rne(v);
      out[r * cols + c] = mask ? (uint16_t)(h | (sign << 15)) : 0;
    }
  return 0;
}

/* ------------------------------------------------------------------------ */
/* O5a. Router (the host model's, unchanged by the method: P:287). Per token, */
/*      top-k by logit, ties to the lower expert index (reading R13); gates:  */
/*      renormalize ? softmax over the k selected : softmax(all E)[selected]. */
/* ------------------------------------------------------------------------ */
static void route_token(const float* logits, int E, int k, int renormalize, int32_t* sel,
                        double* gate) {
  unsigned char taken[1024];
  memset(taken, 0, sizeof(taken));
  for (int j = 0; j < k; ++j) {
    int best = -1;
    for (int e = 0; e < E; ++e) {
      if (taken[e]) continue;
      if (best < 0 || logits[e] > logits[best]) best = e; /* strict >: ties keep lower index */
    }
    taken[best] = 1;
    sel[j] = best;
  }
  if (renormalize) {
    double m = (double)logits[sel[0]];
    for (int j = 1; j < k; ++j)
      if ((double)logits[sel[j]] > m) m = (double)logits[sel[j]];
    double s = 0.0;
    for (int j = 0; j < k; ++j) s += exp((double)logits[sel[j]] - m);
    for (int j = 0; j < k; ++j) gate[j] = exp((double)logits[sel[j]] - m) / s;
  } else {
    double m = (double)logits[0];
    for (int e = 1; e < E; ++e)
      if ((double)logits[e] > m) m = (double)logits[e];
    double s = 0.0;
    for (int e = 0; e < E; ++e) s += exp((double)logits[e] - m);
    for (int j = 0; j < k; ++j) gate[j] = exp((double)logits[sel[j]] - m) / s;
  }
}

int oracle_route(const float* logits, int64_t T, int E, int k, int renormalize, int32_t* topk_idx,
                 double* topk_gate) {
  if (E < 1 || E > 1024 || k < 1 || k > E) return 1;
  for (int64_t t = 0; t < T; ++t)
    route_token(logits + t * E, E, k, renormalize, topk_idx + t * k, topk_gate + t * k);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* O5b. MoE expert-FFN forward over packed pairs (SwiGLU expert;  */
/*      reconstruction Eq. 8 via Algorithm 1).          */
/*   w13: [P][2][f][d] packed (gate rows then up rows; HF gate_up_proj order) */
/*   w2 : [P][d][f]    packed                                                 */
/*   expert_slot[e] = 2*pair + pos (the pairing plan)              */
/*   hidden: bf16 bits [T][d]; logits: f32 [T][E]; residual: bf16 bits or 0   */
/*   out: f64 [T][d] = residual + sum_j gate_j * W2_e (silu(W1_e x) * W3_e x) */
/*   pair_dense: NULL, or u8 [P]: slot q holds ONE unmerged expert as plain   */
/*   bf16 bits in the same [2][f][d] / [d][f] shape, position 0 only (the 25% */
/*   compression ratio: experts cut to 75%, the rest kept unchanged;   */
/*   reading R20). E <= 2P; the slots of distinct experts must be distinct.   */
/* All products and sums in f64 on the exact bf16 operand values; h is NOT   */
/* rounded to bf16 (reading R16). One token per OpenMP iteration.            */
/* ------------------------------------------------------------------------ */
static double slot_weight(uint16_t w, int pos, int dense) {
  return bf16_to_double(dense ? w : decode_word(w, pos));
}

int oracle_moe_forward(const uint16_t* w13, const uint16_t* w2, const int32_t* expert_slot,
                       const uint8_t* pair_dense, int n_pairs, int d, int f, const uint16_t* hidden,
                       const float* logits, int64_t T, int E, int k, int renormalize,
                       const uint16_t* residual, double* out) {
  if (E < 1 || E > 1024 || E > 2 * n_pairs || k < 1 || k > E || d < 1 || f < 1) return 1;
  for (int e = 0; e < E; ++e) {
    if (expert_slot[e] < 0 || expert_slot[e] >= 2 * n_pairs) return 1;
    if (pair_dense && pair_dense[expert_slot[e] / 2] && expert_slot[e] % 2 != 0) return 1;
    for (int e2 = 0; e2 < e; ++e2)
      if (expert_slot[e2] == expert_slot[e]) return 1;
  }
  int err = 0;
#pragma omp parallel
  {
    double* x = (double*)malloc(sizeof(double) * (size_t)d);
    double* h = (double*)malloc(sizeof(double) * (size_t)f);
    double* y = (double*)malloc(sizeof(double) * (size_t)d);
    if (!x || !h || !y) {
#pragma omp atomic write
      err = 2;
    }
#pragma omp for schedule(dynamic, 1)
    for (int64_t t = 0; t < T; ++t) {
      if (!x || !h || !y) continue;
      int32_t sel[1024];
      double gate[1024];
      route_token(logits + t * E, E, k, renormalize, sel, gate);
      for (int c = 0; c < d; ++c) x[c] = bf16_to_double(hidden[t * d + c]);
      double* o = out + t * d;
      for (int c = 0; c < d; ++c) o[c] = residual ? bf16_to_double(residual[t * d + c]) : 0.0;
      for (int j = 0; j < k; ++j) {
        int slot = expert_slot[sel[j]];
        int pair = slot / 2, pos = slot % 2;
        int dense = pair_dense ? pair_dense[pair] != 0 : 0;
        const uint16_t* W1 = w13 + ((size_t)pair * 2 + 0) * (size_t)f * d; /* gate */
        const uint16_t* W3 = w13 + ((size_t)pair * 2 + 1) * (size_t)f * d; /* up   */
        const uint16_t* W2 = w2 + (size_t)pair * (size_t)d * f;
        for (int r = 0; r < f; ++r) {
          double g = 0.0, u = 0.0;
          for (int c = 0; c < d; ++c) {
            g += slot_weight(W1[(size_t)r * d + c], pos, dense) * x[c];
            u += slot_weight(W3[(size_t)r * d + c], pos, dense) * x[c];
          }
          h[r] = g / (1.0 + exp(-g)) * u; /* silu(g) * u */
        }
        for (int r = 0; r < d; ++r) {
          double acc = 0.0;
          for (int c = 0; c < f; ++c) acc += slot_weight(W2[(size_t)r * f + c], pos, dense) * h[c];
          y[r] = acc;
        }
        for (int r = 0; r < d; ++r) o[r] += gate[j] * y[r];
      }
    }
    free(x);
    free(h);
    free(y);
  }
  return err;
}

/* ------------------------------------------------------------------------ */
/* O6. Calibration statistics for Eq. 4 (NEXT-4): ||X||_2 per input column   */
/*     over "a sample of input activations to a certain expert",      */
/*     from "a single forward pass"; per column, unnormalised (R12).  */
/*     Returned as sums of squares per slot b = expert_slot[e] (the norms are */
/*     their square roots):                                                   */
/*       sumsq_x[b][c] = sum over (t, j) routed to b of x_t[c]^2  (W1/W3 in)  */
/*       sumsq_h[b][r] = sum over (t, j) routed to b of h_t[r]^2  (W2 input), */
/*       h = silu(W1 x) * (W3 x) of the slot's expert, f64, not rounded (R16).*/
/*     Serial, f64. Either output may be NULL.                                */
/* ------------------------------------------------------------------------ */
int oracle_calib_sumsq(const uint16_t* w13, const int32_t* expert_slot, const uint8_t* pair_dense,
                       int n_pairs, int d, int f, const uint16_t* hidden, const float* logits,
                       int64_t T, int E, int k, int renormalize, double* sumsq_x, double* sumsq_h) {
  if (E < 1 || E > 1024 || E > 2 * n_pairs || k < 1 || k > E || d < 1 || f < 1) return 1;
  for (int e = 0; e < E; ++e)
    if (expert_slot[e] < 0 || expert_slot[e] >= 2 * n_pairs) return 1;
  if (sumsq_x) memset(sumsq_x, 0, sizeof(double) * (size_t)2 * n_pairs * d);
  if (sumsq_h) memset(sumsq_h, 0, sizeof(double) * (size_t)2 * n_pairs * f);
  double* x = (double*)malloc(sizeof(double) * (size_t)d);
  if (!x) return 2;
  for (int64_t t = 0; t < T; ++t) {
    int32_t sel[1024];
    double gate[1024];
    route_token(logits + t * E, E, k, renormalize, sel, gate);
    for (int c = 0; c < d; ++c) x[c] = bf16_to_double(hidden[t * d + c]);
    for (int j = 0; j < k; ++j) {
      int slot = expert_slot[sel[j]];
      int pair = slot / 2, pos = slot % 2;
      int dense = pair_dense ? pair_dense[pair] != 0 : 0;
      if (sumsq_x)
        for (int c = 0; c < d; ++c) sumsq_x[(size_t)slot * d + c] += x[c] * x[c];
      if (!sumsq_h) continue;
      const uint16_t* W1 = w13 + ((size_t)pair * 2 + 0) * (size_t)f * d;
      const uint16_t* W3 = w13 + ((size_t)pair * 2 + 1) * (size_t)f * d;
      for (int r = 0; r < f; ++r) {
        double g = 0.0, u = 0.0;
        for (int c = 0; c < d; ++c) {
          g += slot_weight(W1[(size_t)r * d + c], pos, dense) * x[c];
          u += slot_weight(W3[(size_t)r * d + c], pos, dense) * x[c];
        }
        double h = g / (1.0 + exp(-g)) * u;
        sumsq_h[(size_t)slot * f + r] += h * h;
      }
    }
  }
  free(x);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* O5c. One expert of one pair on rows that are already routed to it:       */
/*      y[n] = W2_pos (silu(W1_pos x[n]) * (W3_pos x[n])), f64, no gate.     */
/*      (The EP tests' CPU stand-in for the expert kernels.)                  */
/* ------------------------------------------------------------------------ */
int oracle_expert_ffn(const uint16_t* w13, const uint16_t* w2, int pair, int pos, int dense, int d,
                      int f, const uint16_t* x_rows, int64_t n, double* y) {
  if (pos != 0 && pos != 1) return 1;
  if (dense && pos != 0) return 1;
  const uint16_t* W1 = w13 + ((size_t)pair * 2 + 0) * (size_t)f * d;
  const uint16_t* W3 = w13 + ((size_t)pair * 2 + 1) * (size_t)f * d;
  const uint16_t* W2 = w2 + (size_t)pair * (size_t)d * f;
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t t = 0; t < n; ++t) {
    double* h = (double*)malloc(sizeof(double) * (size_t)f);
    const uint16_t* x = x_rows + t * d;
    for (int r = 0; r < f; ++r) {
      double g = 0.0, u = 0.0;
      for (int c = 0; c < d; ++c) {
        double xc = bf16_to_double(x[c]);
        g += slot_weight(W1[(size_t)r * d + c], pos, dense) * xc;
        u += slot_weight(W3[(size_t)r * d + c], pos, dense) * xc;
      }
      h[r] = g / (1.0 + exp(-g)) * u;
    }
    for (int r = 0; r < d; ++r) {
      double acc = 0.0;
      for (int c = 0; c < f; ++c) acc += slot_weight(W2[(size_t)r * f + c], pos, dense) * h[c];
      y[t * d + r] = acc;
    }
    free(h);
  }
  return 0;
}

int oracle_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

void oracle_set_num_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}
