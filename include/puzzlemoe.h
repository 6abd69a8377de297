/*
 * puzzlemoe.h -- C ABI of the B200-native PuzzleMoE packed-expert MoE FFN library
 * (libpuzzlemoe.so, sm_100a).
 *
 * What it computes (arXiv 2511.04805, "PuzzleMoE"; P:n = PAPER.md line n, S:n = SPEC.md):
 *   Pairs of experts are merged offline (Eq. 1-7) into one magnitude tensor
 *   W_merged plus per-expert masks M_i, M_j and signs S_i, S_j. Those four bits are
 *   embedded into the exponent field of a bf16 word ("packed bf16"):
 *
 *       bit 15 S_i | bit 14 S_j | bit 13 M_i | bit 12 M_j | bits 11..7 e' | bits 6..0 mantissa
 *       e' = clamp(e, 112, 143) - 112,   e = bf16 exponent of W_merged
 *
 *   and decoded on the fly by Algorithm 1 to reconstruct expert `pos`
 *   (0 = expert i, 1 = expert j) as  W^ = (-1)^S (.) M (.) W_merged  (Eq. 8).
 *
 * Conventions for every call:
 *   - All tensor pointers are DEVICE pointers owned by the caller (the library never
 *     allocates, frees or retains caller memory). bf16 tensors are passed as uint16_t
 *     bit patterns. All layouts are dense row-major, little-endian.
 *   - Calls are asynchronous and stream-ordered on `stream` (a cudaStream_t; NULL is
 *     the legacy default stream). No call synchronises the host with the device.
 *   - Argument errors are detected on the host BEFORE any launch and returned
 *     synchronously; nothing is launched then. Launch failures return
 *     PUZZLE_ERR_CUDA. `puzzle_last_error()` gives a thread-local detail string.
 *   - Data-dependent conditions (exponent clamping, non-finite or negative magnitudes)
 *     are not errors: they are COUNTED into a caller-provided device
 *     `puzzle_pack_stats`, which may be NULL.
 *   - Thread safety: calls are stateless; distinct host threads may call concurrently
 *     on distinct streams. A workspace may be used by one in-flight call at a time.
 *   - There is no CPU fallback: without a CUDA device every compute call returns
 *     PUZZLE_ERR_CUDA.
 */
#ifndef PUZZLEMOE_H_
#define PUZZLEMOE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#pragma GCC visibility push(default) /* the library builds with -fvisibility=hidden */
#endif

/* cudaStream_t without including cuda_runtime.h */
typedef struct CUstream_st* puzzle_stream_t;

typedef enum {
  PUZZLE_OK = 0,
  PUZZLE_ERR_INVALID_ARGUMENT = 1, /* null pointer, pos not in {0,1}, k > E, E != 2P, tau outside [0,1] */
  PUZZLE_ERR_SHAPE_MISMATCH = 2,   /* SPEC ShapeMismatch / DimensionMismatch */
  PUZZLE_ERR_UNSUPPORTED = 3,      /* shape outside the kernels' tiling: d_model or d_ff not a multiple of 64,
                                      E > 512, misaligned pointer (16 B required for weights / activations) */
  PUZZLE_ERR_WORKSPACE = 4,        /* workspace NULL or smaller than puzzle_moe_workspace_size() */
  PUZZLE_ERR_CUDA = 5,             /* CUDA launch / device error (including: no device) */
  PUZZLE_ERR_NCCL = 6              /* NCCL not loadable or an NCCL call failed (the communicator is then
                                      aborted: every later call on that puzzle_ep returns this code) */
} puzzle_status;

/* Human-readable name of a status code (static storage). */
const char* puzzle_status_string(int status);
/* Thread-local detail of the last non-OK return on this thread ("" if none). */
const char* puzzle_last_error(void);
/* ABI version: (major << 16) | minor. */
int puzzle_abi_version(void);

/* Device-side counters, accumulated (never reset) by the pack calls. */
typedef struct {
  unsigned long long rounded_up; /* bf16 exponent e < 112, raised to 112 ("rounded up") */
  unsigned long long saturated;  /* e > 143, saturated to 143 (reading R1; never hit by trained weights) */
  unsigned long long nonfinite;  /* NaN / Inf magnitude (encoded per the same formula, but counted) */
  unsigned long long negative;   /* magnitude < 0 (its |.| bits are encoded; counted) */
} puzzle_pack_stats;

/* ---------------------------------------------------------------------------------------
 * puzzle_merge_pack -- (a1) merged magnitude + masks + signs -> packed bf16 words.
 *   P:186-190 (exponent shift), P:196-209 (bit layout read back by Algorithm 1).
 *   w_merged    f32 [n]  W_merged of Eq. 7 (>= 0, finite)
 *   m0, m1      u8  [n]  M_i, M_j of Eq. 6 (nonzero = 1)
 *   s0, s1      u8  [n]  S_i, S_j of Eq. 3 (nonzero = 1)
 *   packed_out  u16 [n]  output words
 *   stats       device puzzle_pack_stats*, accumulated; may be NULL
 *   Rounding: f32 -> bf16 round-to-nearest-even BEFORE the exponent clamp (R3).
 *   n == 0 is a no-op. Errors: INVALID_ARGUMENT (null pointer with n > 0, n < 0).
 * ------------------------------------------------------------------------------------- */
int puzzle_merge_pack(const float* w_merged, const uint8_t* m0, const uint8_t* m1,
                      const uint8_t* s0, const uint8_t* s1, int64_t n, uint16_t* packed_out,
                      puzzle_pack_stats* stats, puzzle_stream_t stream);

/* ---------------------------------------------------------------------------------------
 * puzzle_unpack -- (a2) Algorithm 1 over a whole tensor.
 *   packed    u16 [n]   packed words
 *   pos       0 (expert i: sign bit 15, mask bit 13) or 1 (expert j: bits 14, 12)
 *   bf16_out  u16 [n]   bf16 bits of W^_pos (Eq. 8); masked-out entries are +0.0 (0x0000)
 *   Errors: INVALID_ARGUMENT (pos not in {0,1}, null pointer with n > 0, n < 0).
 * ------------------------------------------------------------------------------------- */
int puzzle_unpack(const uint16_t* packed, int pos, int64_t n, uint16_t* bf16_out,
                  puzzle_stream_t stream);

/* ---------------------------------------------------------------------------------------
 * puzzle_merge_experts_pack -- fused Eq. 1-7 merge + pack, for a
 *   batch of `n_mats` independent matrices (one linear slot of one pair each).
 *   w_i, w_j        bf16 [n_mats][rows][cols]  the two experts' weights, (out x in)
 *   norms_i/_j      f32  [n_mats][cols]        ||X||_2 per input column (Eq. 4)
 *   tau_sim         similarity threshold in [0,1] (Eq. 2; the paper uses 0.4)
 *   packed_out      u16  [n_mats][rows][cols]  pos 0 = expert i, pos 1 = expert j
 *   Arithmetic: IEEE f32 exactly as the expressions of Eq. 1-7 are written, 0/0 in
 *   Eq. 1 := 0 (R4), saliency ties -> expert i (Eq. 5 ">="), then the same RNE + clamp as
 *   puzzle_merge_pack. Bit-identical to merging with the oracle and packing.
 *   Errors: INVALID_ARGUMENT (tau outside [0,1], null pointers, negative sizes).
 * ------------------------------------------------------------------------------------- */
int puzzle_merge_experts_pack(const uint16_t* w_i, const uint16_t* w_j, const float* norms_i,
                              const float* norms_j, int64_t n_mats, int64_t rows, int64_t cols,
                              float tau_sim, uint16_t* packed_out, puzzle_pack_stats* stats,
                              puzzle_stream_t stream);

/* ---------------------------------------------------------------------------------------
 * NEXT-3: the quantised PuzzleMoE format (Appendix A.3: "uniform quantization with
 * a group size of 128 ... symmetric group quantization ... stored alongside their
 * corresponding sign and mask bits"; readings R21-R23).
 *
 * puzzle_quant_pack -- merged magnitudes + bit-planes -> 3-bit codes with flags + scales.
 *   w_merged    f32 [rows][cols]  W_merged of Eq. 7 (>= 0, finite), cols % 128 == 0
 *   m0, m1, s0, s1  u8 [rows][cols]  M_i, M_j, S_i, S_j (nonzero = 1)
 *   codes_out   u8  [rows][cols]  bit7 S_i | bit6 S_j | bit5 M_i | bit4 M_j | 0 | 3-bit code
 *   scales_out  f32 [rows][cols/128]  max(group)/7 of each group of 128 consecutive elements of
 *                                     a row (1 for an all-zero group)
 *   code = round(w / scale) evaluated as rint(7 w / max) in f64 (halves to even), in [0, 7].
 *   Bit-identical to the oracle. Pointers 16-byte aligned (device). Errors: INVALID_ARGUMENT
 *   (NULL, negative sizes), UNSUPPORTED (cols % 128, alignment).
 *
 * puzzle_quant_unpack -- the dequantised bf16 weights of expert `pos` (0 = i, 1 = j):
 *   (-1)^S_pos * M_pos * bf16_rne(f32(code * scale)); masked entries are +0.
 * ------------------------------------------------------------------------------------- */
int puzzle_quant_pack(const float* w_merged, const uint8_t* m0, const uint8_t* m1, const uint8_t* s0,
                      const uint8_t* s1, int64_t rows, int64_t cols, uint8_t* codes_out,
                      float* scales_out, puzzle_stream_t stream);
int puzzle_quant_unpack(const uint8_t* codes, const float* scales, int pos, int64_t rows,
                        int64_t cols, uint16_t* bf16_out, puzzle_stream_t stream);

/* puzzle_quant_gemv -- the expert GEMV over the quantised format (NEXT-3; R23: Ŵ_pos is the bf16
 *   operand of the expert matmul, Algorithm 1 / Eq. 8's y = Ŵ x). One merged pair, both experts
 *   from one read of the code bytes:
 *   codes   u8  [rows][cols], scales f32 [rows][cols/128]  (puzzle_quant_pack's output)
 *   x_i     bf16 [n_i][cols]  tokens routed to expert i (position 0); x_j [n_j][cols] to j
 *   y_i     f32 [n_i][rows]   y_i[t][r] = sum_c Ŵ_0[r][c] x_i[t][c]; y_j likewise with Ŵ_1
 *   f32 FMA accumulation (each lane sums cols/32 products in order, then a 5-level warp tree).
 *   Device pointers; codes, x_i, x_j 16-byte aligned; the caller owns every buffer. n_i or n_j
 *   may be 0 (that side is not touched). Errors: INVALID_ARGUMENT (negative sizes, NULL),
 *   UNSUPPORTED (cols % 128, alignment).
 */
int puzzle_quant_gemv(const uint8_t* codes, const float* scales, int64_t rows, int64_t cols,
                      const uint16_t* x_i, int64_t n_i, const uint16_t* x_j, int64_t n_j,
                      float* y_i, float* y_j, puzzle_stream_t stream);

/* ---------------------------------------------------------------------------------------
 * One MoE layer whose experts are PuzzleMoE-merged pairs (50% compression), or --
 * the 25% ratio, experts cut to 75% of the original count -- some merged pairs plus
 * unmerged experts kept exactly (reading R20).
 * Weight orientation (out x in) row-major as in HF Mixtral/Qwen (reading R11):
 *   w13  u16 [n_pairs][2][d_ff][d_model]  packed gate (w1) rows, then up (w3) rows
 *   w2   u16 [n_pairs][d_model][d_ff]     packed down projection
 *   expert_slot  i32 [n_experts] (device) = 2*pair + pos  -- the pairing plan;
 *                distinct slots for distinct experts (not checked: device memory)
 *   pair_dense   u8 [n_pairs] (device) or NULL (= all slots merged pairs). pair_dense[q] != 0:
 *                slot q holds ONE unmerged expert as plain bf16 bits in the same w13/w2
 *                shape, read without Algorithm 1; only 2*q + 0 may appear in expert_slot
 *                (routing an expert to 2*q + 1 of such a slot gives undefined outputs).
 * Requirements: 1 <= n_experts <= 2*n_pairs <= 512; d_model and d_ff multiples of 64;
 * w13/w2 16-byte aligned.
 * ------------------------------------------------------------------------------------- */
typedef struct {
  int32_t n_experts;
  int32_t n_pairs;
  int32_t d_model;
  int32_t d_ff;
  const uint16_t* w13;
  const uint16_t* w2;
  const int32_t* expert_slot;
  const uint8_t* pair_dense;
} puzzle_moe_layer;

/* Kernel path for puzzle_moe_forward_ex. AUTO: GEMV while T <= 64 or the experts average
 * fewer than 96 tokens (T*top_k < 96*n_experts; 120 when d_ff >= 8192), else TS (else TC,
 * else GEMV). */
typedef enum {
  PUZZLE_PATH_AUTO = 0,
  PUZZLE_PATH_GEMV = 1,   /* decode shape: decode into TMEM + tcgen05.mma (weights on M), weights read once per pair */
  PUZZLE_PATH_TC = 2,     /* prefill shape: grouped tcgen05/TMEM GEMM, tiles decoded in shared memory */
  PUZZLE_PATH_TS = 3      /* prefill shape: decoded weights as the TMEM A operand, up to 384 tokens of a
                             bucket on N per pass (d_model % 128 == 0, d_ff % 64 == 0) */
} puzzle_path;

/* Bytes of device workspace puzzle_moe_forward needs for up to max_tokens tokens. */
size_t puzzle_moe_workspace_size(const puzzle_moe_layer* L, int64_t max_tokens, int top_k);

/* ---------------------------------------------------------------------------------------
 * puzzle_moe_forward -- the hot path: router top-k + gates (a3), gate/up projections over
 *   the on-the-fly decoded expert with SwiGLU (a4), down projection (a5), top-k combine
 *   (a6). Every step runs in this library's kernels; the packed weights are decoded in
 *   registers / shared memory and never materialised in HBM.
 *   hidden         bf16 [T][d_model]
 *   router_logits  f32  [T][n_experts]
 *   top_k          1 <= top_k <= n_experts; ties in the logits go to the lower expert id
 *   renormalize    1: gates = softmax over the k selected logits (Mixtral);
 *                  0: gates = softmax over all experts, taken at the selected (Qwen/DeepSeek)
 *   residual       bf16 [T][d_model] or NULL; out = residual + sum_j gate_j * FFN_{e_j}(x)
 *   out            bf16 [T][d_model] (may alias residual; must not alias hidden)
 *   workspace      device buffer of >= puzzle_moe_workspace_size(L, T, top_k) bytes
 *   T == 0 is a no-op. Accumulation is fp32; the SwiGLU intermediate is rounded to bf16.
 * ------------------------------------------------------------------------------------- */
int puzzle_moe_forward(const puzzle_moe_layer* L, const uint16_t* hidden,
                       const float* router_logits, int64_t T, int top_k, int renormalize,
                       const uint16_t* residual, uint16_t* out, void* workspace,
                       size_t workspace_bytes, puzzle_stream_t stream);

/* Same as puzzle_moe_forward with an explicit kernel path (tests / benchmarks). */
int puzzle_moe_forward_ex(const puzzle_moe_layer* L, const uint16_t* hidden,
                          const float* router_logits, int64_t T, int top_k, int renormalize,
                          const uint16_t* residual, uint16_t* out, void* workspace,
                          size_t workspace_bytes, int path, puzzle_stream_t stream);

/* ---------------------------------------------------------------------------------------
 * Building blocks of puzzle_moe_forward, exported for expert parallelism (the host splits
 * the layer between route and experts to exchange tokens with NCCL all-to-all).
 *
 * puzzle_moe_route -- (a3). For each token: top-k expert ids (ties -> lower id), gates,
 *   and the grouping of the T*top_k assignments by bucket b = expert_slot[e] (= 2*pair+pos).
 *   topk_idx     i32 [T][top_k]   selected expert ids
 *   topk_gate    f32 [T][top_k]   gates
 *   bucket_off   i32 [2*n_pairs+1] exclusive prefix of per-bucket counts (bucket-major)
 *   assign_token i32 [T*top_k]    token of assignment a (assignments grouped by bucket)
 *   assign_of    i32 [T*top_k]    assignment index of (t, j)
 *   The order of assignments inside one bucket is unspecified (results do not depend on it).
 *   T = 0 writes an all-zero bucket_off (every bucket empty) and nothing else.
 *   workspace: device scratch of >= puzzle_moe_route_workspace_size(L) bytes (decode batches,
 *   T <= 64, route with a top-k grid + a scatter grid and keep per-CTA histograms there; batches
 *   with T*top_k > 4096 keep global counts there; the sizes in between route inside one CTA).
 * ------------------------------------------------------------------------------------- */
size_t puzzle_moe_route_workspace_size(const puzzle_moe_layer* L);
int puzzle_moe_route(const puzzle_moe_layer* L, const float* router_logits, int64_t T,
                     int top_k, int renormalize, int32_t* topk_idx, float* topk_gate,
                     int32_t* bucket_off, int32_t* assign_token, int32_t* assign_of,
                     void* workspace, size_t workspace_bytes, puzzle_stream_t stream);

/* puzzle_moe_experts -- (a4)+(a5) over pre-grouped assignments:
 *   x_rows     bf16 [n_assign][d_model]  activations, already grouped by bucket
 *   bucket_off i32  [2*n_pairs+1] (device) bucket b owns rows [bucket_off[b], bucket_off[b+1])
 *   y_rows     f32  [n_assign][d_model]  unweighted expert outputs W2_pos(silu(W1 x)*(W3 x))
 *   n_assign   host-known upper bound of bucket_off[2P] (rows beyond it are untouched) */
size_t puzzle_moe_experts_workspace_size(const puzzle_moe_layer* L, int64_t n_assign);
int puzzle_moe_experts(const puzzle_moe_layer* L, const uint16_t* x_rows,
                       const int32_t* bucket_off, int64_t n_assign, float* y_rows,
                       void* workspace, size_t workspace_bytes, int path,
                       puzzle_stream_t stream);

/* puzzle_moe_combine -- (a6): out[t] = residual[t] + sum_{j<k} topk_gate[t,j] * y_rows[assign_of[t,j]]
 *   summed in fp32 in slot order j, rounded once to bf16. residual may be NULL.
 *   Errors: INVALID_ARGUMENT (T < 0, k < 1, d % 4, NULL). */
int puzzle_moe_combine(const float* y_rows, const int32_t* assign_of, const float* topk_gate,
                       int64_t T, int top_k, int d_model, const uint16_t* residual,
                       uint16_t* out, puzzle_stream_t stream);

/* puzzle_gather_rows -- dst[i] = src[index[i]] for bf16 rows of width `cols` (EP dispatch
 *   packing / token permutation). */
int puzzle_gather_rows(const uint16_t* src, const int32_t* index, int64_t n_rows, int64_t cols,
                       uint16_t* dst, puzzle_stream_t stream);

/* ---------------------------------------------------------------------------------------
 * Fixed-capacity expert-parallel dispatch (BASELINE.json config 5, "expert-
 * parallel with NCCL all-to-all"; the unit of placement is the merged PAIR, so
 * both experts of a pair stay on one GPU and each packed tile is still read once).
 * Every rank reserves R = cap + 1 rows per destination rank in its send buffer (cap >= T*top_k:
 * the worst case, all of its assignments on one owner; the extra HEADER row carries the
 * destination's bucket counts), so each all-to-all of a layer has EQUAL, host-known splits, rows
 * and counts travel together, and the index work runs on the device: the layer needs no
 * device->host copy and can be captured in a CUDA graph. All ranks must use the same cap.
 *
 * dest_pairs  HOST int32 [world][2]: rank q owns global pairs [dest_pairs[2q], dest_pairs[2q+1])
 *             (whole pairs; or, when pairs are split along d_ff, the one pair q holds a slice
 *             of). Every pair must have the same nonzero number S of owners.
 * Local bucket of rank q: 2*(pair - dest_pairs[2q]) + pos. lb_max >= every rank's local bucket
 * count, and 4*lb_max <= 2*d_model (the counts fit in one header row). Errors: INVALID_ARGUMENT
 * for bad sizes, NULL pointers or a malformed dest_pairs; UNSUPPORTED for world > 64,
 * world*(cap+1) >= 2^31, a header row too small for lb_max counts.
 *
 * puzzle_ep_dispatch -- sender side, after puzzle_moe_route on this rank's T tokens
 *   (n_assign = T*top_k, bucket_off / assign_token as route wrote them):
 *   send_rows  bf16 [world][cap+1][d_model], region q:
 *              row i < n_q = bucket_off[2 hi_q] - bucket_off[2 lo_q]: hidden[assign_token[
 *              bucket_off[2 lo_q] + i]] (q's rows, in bucket order); rows n_q..cap-1 are not
 *              written (never read downstream);
 *              row cap (header): int32 [lb_max] in its first 4*lb_max bytes = the counts of
 *              q's local buckets, 0-padded.
 */
int puzzle_ep_dispatch(const uint16_t* hidden, const int32_t* assign_token, const int32_t* bucket_off, int n_pairs,
                       const int32_t* dest_pairs, int world, int64_t n_assign, int64_t cap, int lb_max,
                       int d_model, uint16_t* send_rows, puzzle_stream_t stream);

/* puzzle_ep_recv_plan -- owner side, on recv_rows bf16 [world][cap+1][d_model] (region s = what
 *   source rank s sent: its rows for this rank, then the header with the counts of this rank's
 *   n_local_buckets buckets). Received row w of region s sits at s*(cap+1) + w. The local order
 *   is (bucket, source, arrival):
 *   local_off  i32 [n_local_buckets + 1]  bucket offsets of the regrouped rows (the bucket_off
 *              argument of puzzle_moe_experts on this rank's shard)
 *   gather_idx i32 [world*cap]      local row l <- received row gather_idx[l]; l >= local_off[last]
 *              -> 0 (padding: puzzle_gather_rows of all world*cap rows stays in bounds)
 *   return_idx i32 [world*(cap+1)]  received slot r <- local row return_idx[r] (0 for unused
 *              slots and header rows): gathering the experts' outputs with it gives the return
 *              buffer in the same region layout.
 *   Limits: n_local_buckets <= 1024, (3*world*n_local_buckets + world + n_local_buckets + 1)*4
 *   bytes <= 48 KB (UNSUPPORTED otherwise). */
int puzzle_ep_recv_plan(const uint16_t* recv_rows, int world, int n_local_buckets, int64_t cap, int d_model,
                        int32_t* local_off, int32_t* gather_idx, int32_t* return_idx, puzzle_stream_t stream);

/* puzzle_ep_home_index -- home side, after the return all-to-all (y rows [world][cap+1], region
 *   q = what owner q computed for this rank's rows, in the order puzzle_ep_dispatch sent them).
 *   For assignment (t, j) = a = assign_of[t*top_k + j] in global bucket g (pair p = g/2) and the
 *   s-th owner q_s of p (ascending rank, s < S):
 *   aof_s  i32 [T][top_k*S]: aof_s[t][j*S + s] = q_s*(cap+1) + (a - bucket_off[2 lo_{q_s}])
 *   gate_s f32 [T][top_k*S]: gate_s[t][j*S + s] = topk_gate[t][j]
 *   so puzzle_moe_combine(y, aof_s, gate_s, T, top_k*S, ...) sums the S d_ff-slice partials of
 *   every (t, j) with its gate (S = 1: the plain combine of (a6)). */
int puzzle_ep_home_index(const int32_t* assign_of, const float* topk_gate, const int32_t* bucket_off, int n_pairs,
                         const int32_t* dest_pairs, int world, int64_t cap, int64_t T, int top_k, int32_t* aof_s,
                         float* gate_s, puzzle_stream_t stream);

/* ---------------------------------------------------------------------------------------
 * The same fixed-capacity layer over NVLink PEER MEMORY: the dispatch kernel stores each
 * owner's rows (and header) straight into that owner's receive buffer, and the owner's return
 * kernel stores the expert outputs straight into each home rank's buffer -- the transfers are
 * fused into the gather / un-permute kernels (no NCCL on the data path, no staging copies).
 *
 * Every rank allocates ONE peer buffer of puzzle_ep_peer_buffer_size(world, cap, d_model) bytes
 * (symmetric: same size on all ranks, mapped into every peer's address space, e.g. CUDA IPC /
 * torch symmetric memory; 256-byte aligned; zero-initialised once). Layout:
 *   recv_x  bf16 [world][cap+1][d_model] at offset 0 (region s: rows + header from source s,
 *           exactly puzzle_ep_dispatch's region for this rank),
 *   recv_y  f32  [world][cap+1][d_model] at an offset aligned to 256 B after recv_x (region q:
 *           the outputs owner q returned for this rank's rows),
 *   flags   u32  [2][world] (dispatch / return epochs) after recv_y.
 * peer_bases  HOST u64 [world]: the device address of rank q's peer buffer as mapped on THIS
 *             rank (peer_bases[rank] = its own buffer).
 * state       device u32 [8], zero-initialised once, private to the rank and the layer: [0] the
 *             step counter (epochs), [1..3] the kernels' CTA completion counters, [4] the number
 *             of cross-rank waits that gave up after ~10 s (a peer never arrived: the outputs of
 *             that step are invalid; nonzero means the ranks' call sequences diverged).
 * Per layer call (stream-ordered on one stream; graph-capturable):
 *   puzzle_moe_route -> puzzle_ep_dispatch_peer -> puzzle_ep_recv_plan_peer (waits until every
 *   source's region of this step has landed, then plans on recv_x) -> gather ->
 *   puzzle_moe_experts -> puzzle_ep_return_peer -> puzzle_ep_combine_peer (waits for every
 *   owner's return, combines from recv_y, advances the step).
 * Every rank must make the same sequence of calls (the waits are cross-rank: a rank that stops
 * calling stalls its peers). Errors as for the NCCL form; peer_bases entries must be non-NULL and
 * 256-byte aligned.
 * ------------------------------------------------------------------------------------- */
size_t puzzle_ep_peer_buffer_size(int world, int64_t cap, int d_model);
int puzzle_ep_dispatch_peer(const uint16_t* hidden, const int32_t* assign_token, const int32_t* bucket_off,
                            int n_pairs, const int32_t* dest_pairs, int world, int rank, int64_t n_assign,
                            int64_t cap, int lb_max, int d_model, const unsigned long long* peer_bases,
                            uint32_t* state, puzzle_stream_t stream);
int puzzle_ep_wait_dispatch(const void* my_base, int world, int64_t cap, int d_model, uint32_t* state,
                            puzzle_stream_t stream);
/* puzzle_ep_wait_dispatch + puzzle_ep_recv_plan(recv_x of my_base) in one kernel (the form the
 * layer uses: one launch less). */
int puzzle_ep_recv_plan_peer(const void* my_base, int world, int n_local_buckets, int64_t cap, int d_model,
                             uint32_t* state, int32_t* local_off, int32_t* gather_idx, int32_t* return_idx,
                             puzzle_stream_t stream);
/* y_local f32 [world*cap][d_model] (the experts' outputs in local order), return_idx from
 * puzzle_ep_recv_plan: slot (s, w) of home rank s's recv_y region [rank] <- y_local[return_idx],
 * for the w < (rows source s sent, from the header of this rank's recv_x region s) only. */
int puzzle_ep_return_peer(const float* y_local, const int32_t* return_idx, int world, int rank, int n_local_buckets,
                          int64_t cap, int d_model, const unsigned long long* peer_bases, uint32_t* state,
                          puzzle_stream_t stream);
/* puzzle_ep_combine_peer -- the layer's last step: waits for every owner's return, then
 * out[t] = residual[t] + sum over slots (j, s) of topk_gate[t][j] * recv_y[row of (t, j, s)] with
 * the rows of puzzle_ep_home_index, fp32 in slot order, one bf16 rounding (the arithmetic of
 * puzzle_moe_combine on those tables, bit for bit); advances the step. residual may be NULL;
 * T <= 65535, top_k * S <= 256. */
int puzzle_ep_combine_peer(const int32_t* assign_of, const float* topk_gate, const int32_t* bucket_off, int n_pairs,
                           const int32_t* dest_pairs, int world, int64_t cap, int64_t T, int top_k, int d_model,
                           const void* my_base, const uint16_t* residual, uint16_t* out, uint32_t* state,
                           puzzle_stream_t stream);
/* As puzzle_ep_home_index (region stride cap+1), after waiting for every owner's return; advances
 * the step (use it with puzzle_moe_combine on recv_y INSTEAD of puzzle_ep_combine_peer). */
int puzzle_ep_home_index_peer(const int32_t* assign_of, const float* topk_gate, const int32_t* bucket_off,
                              int n_pairs, const int32_t* dest_pairs, int world, int64_t cap, int64_t T, int top_k,
                              int d_model, const void* my_base, int32_t* aof_s, float* gate_s, uint32_t* state,
                              puzzle_stream_t stream);

/* ---------------------------------------------------------------------------------------
 * NEXT-4: calibration statistics for Eq. 4 (reading R12). The Wanda saliency
 * A = |W| (.) ||X||_2 needs, per expert, the L2 norm of every input column over "a sample of
 * input activations to a certain expert", gathered in "a single forward pass"
 * (P:142). Both calls produce f64 SUMS OF SQUARES, ACCUMULATED into the caller's buffers
 * (zero them first; several calibration batches add up); the norms are their square roots.
 * Summation is deterministic (no atomics): the same inputs give the same bits every run.
 *
 * puzzle_group_colsumsq -- sumsq[g][c] += sum over rows r in [group_off[g], group_off[g+1])
 *   of rows[r][c]^2.
 *   rows       bf16 [group_off[n_groups]][cols] (device, 16-byte aligned), cols % 8 == 0
 *   group_off  i32  [n_groups + 1] (device) non-decreasing row offsets, group_off[0] >= 0
 *   sumsq      f64  [n_groups][cols] (device, 16-byte aligned), accumulated
 *   workspace  >= puzzle_group_colsumsq_workspace_size(n_groups, cols) bytes (device)
 *   Errors: INVALID_ARGUMENT (NULL, negative sizes), UNSUPPORTED (alignment, cols % 8),
 *   WORKSPACE. n_groups == 0 or cols == 0 is a no-op.
 *
 * puzzle_moe_forward_calib -- puzzle_moe_forward_ex (same arguments and output) that also
 *   accumulates, per bucket b = expert_slot[e] (= 2*pair + pos):
 *     sumsq_x  f64 [2*n_pairs][d_model]  squares of the x rows routed to b (W1 / W3 input)
 *     sumsq_h  f64 [2*n_pairs][d_ff]     squares of the bf16 SwiGLU rows silu(W1 x)*(W3 x)
 *                                        of b's assignments (W2 input; h is rounded to bf16
 *                                        as in the forward, reading R16)
 *   Either may be NULL (not both); 16-byte aligned. To calibrate an UNMERGED model, describe
 *   it as a layer of dense slots (pair_dense = 1, expert_slot[e] = 2e, n_pairs = n_experts):
 *   bucket 2e then holds expert e's statistics.
 *   workspace  >= puzzle_moe_calib_workspace_size(L, T, top_k) bytes.
 * ------------------------------------------------------------------------------------- */
size_t puzzle_group_colsumsq_workspace_size(int n_groups, int64_t cols);
int puzzle_group_colsumsq(const uint16_t* rows, const int32_t* group_off, int n_groups, int64_t cols,
                          double* sumsq, void* workspace, size_t workspace_bytes, puzzle_stream_t stream);
size_t puzzle_moe_calib_workspace_size(const puzzle_moe_layer* L, int64_t max_tokens, int top_k);
int puzzle_moe_forward_calib(const puzzle_moe_layer* L, const uint16_t* hidden,
                             const float* router_logits, int64_t T, int top_k, int renormalize,
                             const uint16_t* residual, uint16_t* out, double* sumsq_x,
                             double* sumsq_h, void* workspace, size_t workspace_bytes, int path,
                             puzzle_stream_t stream);

/* ---------------------------------------------------------------------------------------
 * Measurement plumbing (not part of the method). While a profiling window is open, every
 * kernel the library launches is bracketed by CUDA events recorded on the SAME stream the
 * kernel is launched on. puzzle_profile_end() synchronises those events and writes one
 * line per kernel name: "<name> <launches> <total_ms>\n" into buf (truncated to buflen).
 * Windows are process-global and not thread-safe; returns PUZZLE_ERR_CUDA on event errors.
 * ------------------------------------------------------------------------------------- */
int puzzle_profile_begin(void);
int puzzle_profile_end(char* buf, size_t buflen);

/* ---------------------------------------------------------------------------------------
 * NEXT-3: the quantised PuzzleMoE weight class (App. A.3; R21-R23) in the
 * forward. Each projection of each merged pair is puzzle_quant_pack's output: one byte per
 * merged element (S_i S_j M_i M_j 0 c2 c1 c0) and an f32 scale per group of 128 consecutive
 * columns of a row. The decode-shape kernels stream the code bytes of every touched pair ONCE
 * for both experts and decode them on the fly into the tcgen05 A operand:
 *   W^_pos = (-1)^S_pos * M_pos * bf16_rne(f32(code * scale))   (R23; masked entries +0)
 * -- then SwiGLU, the down projection and the combine exactly as puzzle_moe_forward. Every T is
 * accepted (passes of 32 tokens per position: the format is for decode-shape batches).
 * ------------------------------------------------------------------------------------- */
typedef struct {
  int32_t n_experts, n_pairs, d_model, d_ff;   /* d_model, d_ff multiples of 128 */
  const uint8_t* w13_codes;   /* [n_pairs][2][d_ff][d_model] (gate rows, then up rows), 16-byte aligned */
  const float* w13_scales;    /* [n_pairs][2][d_ff][d_model / 128] */
  const uint8_t* w2_codes;    /* [n_pairs][d_model][d_ff], 16-byte aligned */
  const float* w2_scales;     /* [n_pairs][d_model][d_ff / 128] */
  const int32_t* expert_slot; /* [n_experts] = 2*pair + pos (device) */
} puzzle_moe_quant_layer;

size_t puzzle_moe_quant_workspace_size(const puzzle_moe_quant_layer* Q, int64_t max_tokens, int top_k);
/* Arguments, errors and outputs as puzzle_moe_forward (UNSUPPORTED: d_model or d_ff not a
 * multiple of 128, scales not 4-byte aligned). */
int puzzle_moe_forward_quant(const puzzle_moe_quant_layer* Q, const uint16_t* hidden, const float* router_logits,
                             int64_t T, int top_k, int renormalize, const uint16_t* residual, uint16_t* out,
                             void* workspace, size_t workspace_bytes, puzzle_stream_t stream);

/* ---------------------------------------------------------------------------------------
 * Expert parallelism behind the boundary (BASELINE.json config 5: "expert-
 * parallel with NCCL all-to-all at 2/4/8 B200"; the deployment the paper reports is 2 GPUs -> 1,
 * P:375). One process per GPU. The library owns an NCCL communicator, bootstrapped from a
 * 128-byte ncclUniqueId that rank 0 creates (puzzle_ep_unique_id) and the caller broadcasts
 * (e.g. torch.distributed.broadcast_object_list); NCCL itself is loaded at run time
 * (libnccl.so.2, the copy PyTorch already loaded if any).
 *
 * Placement (puzzle_ep_partition): the unit is the merged PAIR, so both experts of a pair stay
 * on one GPU and each packed tile is still read once. world <= n_pairs: rank r owns
 * pairs [r*P/world, (r+1)*P/world). world > n_pairs (world % n_pairs == 0): every pair is split
 * along d_ff into S = world / n_pairs slices, rank r holding slice r % S of pair r / S (SwiGLU is
 * elementwise in d_ff, so each slice's down projection is an exact partial; the token's home
 * rank sums the S partials with the gate). A d_ff slice of a packed tensor is a valid packed
 * tensor (the decode is elementwise).
 * ------------------------------------------------------------------------------------- */
#define PUZZLE_EP_UNIQUE_ID_BYTES 128
typedef struct puzzle_ep puzzle_ep;

/* 128 bytes (ncclUniqueId) for puzzle_ep_create on every rank; call on rank 0 only. */
int puzzle_ep_unique_id(void* id_out);

/* Collective over the `world` ranks (every rank calls it with the same id): communicator of rank
 * `rank` on CUDA device `device`. *ep_out = NULL on failure. Errors: INVALID_ARGUMENT, CUDA (no
 * such device), NCCL. */
int puzzle_ep_create(puzzle_ep** ep_out, int world, int rank, const void* unique_id, int device);
/* Destroys the communicator (NULL is a no-op). */
int puzzle_ep_destroy(puzzle_ep* ep);

/* The placement: dest_pairs HOST int32 [world][2] (rank q owns global pairs [dest_pairs[2q],
 * dest_pairs[2q+1])) and *slices = S (1, or world / n_pairs). Either output may be NULL. */
int puzzle_ep_partition(int world, int n_pairs, int32_t* dest_pairs, int* slices);

/* Device workspace bytes of puzzle_moe_forward_ep (0: invalid arguments). */
size_t puzzle_moe_forward_ep_workspace_size(const puzzle_ep* ep, const puzzle_moe_layer* route_layer,
                                            const puzzle_moe_layer* local_shard, int64_t cap_tokens, int top_k);

/* puzzle_moe_forward_ep -- the MoE layer (a3)-(a6) expert-parallel over the communicator's ranks,
 *   with fixed-capacity dispatch: every rank reserves cap = cap_tokens*top_k rows (+1 header row
 *   carrying the bucket counts) per destination, so both all-to-alls have equal, host-known splits
 *   and the whole layer runs on the device without host synchronisation (CUDA-graph capturable).
 *   route_layer  GLOBAL routing metadata: n_experts, n_pairs, d_model, d_ff, expert_slot (device)
 *                of the whole layer (its weight pointers are not read; they must be non-NULL)
 *   local_shard  this rank's packed pairs per puzzle_ep_partition (n_pairs = its pair count,
 *                d_ff = route_layer->d_ff / S; pair_dense as in puzzle_moe_forward)
 *   hidden, router_logits, residual, out, top_k, renormalize: this rank's T tokens, as in
 *                puzzle_moe_forward; T <= cap_tokens; cap_tokens must be the same on all ranks;
 *                a rank with T = 0 (NULL activations allowed) still takes part in both all-to-alls
 *   path         kernel path of the local experts (AUTO picks by the capacity world*cap)
 * Steps: puzzle_moe_route -> puzzle_ep_dispatch -> NCCL all-to-all (grouped ncclSend/ncclRecv on
 * `stream`) -> puzzle_ep_recv_plan -> puzzle_gather_rows -> puzzle_moe_experts -> gather back
 * -> NCCL all-to-all -> puzzle_ep_home_index -> puzzle_moe_combine. Every rank must call it for
 * every layer (collective). Errors: as the building blocks; SHAPE_MISMATCH for a local shard
 * that does not match the partition; WORKSPACE; NCCL. */
int puzzle_moe_forward_ep(puzzle_ep* ep, const puzzle_moe_layer* route_layer, const puzzle_moe_layer* local_shard,
                          const uint16_t* hidden, const float* router_logits, int64_t T, int64_t cap_tokens,
                          int top_k, int renormalize, const uint16_t* residual, uint16_t* out, void* workspace,
                          size_t workspace_bytes, int path, puzzle_stream_t stream);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif

#ifdef __cplusplus
} /* extern "C" */
#endif

#endif /* PUZZLEMOE_H_ */
