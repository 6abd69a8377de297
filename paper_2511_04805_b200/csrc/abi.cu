// extern "C" boundary of libpuzzlemoe: host-side argument validation, workspace layout,
// kernel-path dispatch. Declared (with citations and contracts) in include/puzzlemoe.h.
#include <cstdio>
#include <cstring>
#include <mutex>
#include <map>
#include <string>
#include <vector>

#include "common.cuh"

namespace pz {

// kernel launchers (pack.cu, route.cu, gemv.cu, gemm_tc.cu)
int launch_merge_pack(const float*, const uint8_t*, const uint8_t*, const uint8_t*, const uint8_t*,
                      int64_t, uint16_t*, puzzle_pack_stats*, cudaStream_t);
int launch_unpack(const uint16_t*, int, int64_t, uint16_t*, cudaStream_t);
int launch_quant_pack(const float*, const uint8_t*, const uint8_t*, const uint8_t*, const uint8_t*, int64_t, int64_t,
                      uint8_t*, float*, cudaStream_t);
int launch_quant_unpack(const uint8_t*, const float*, int, int64_t, int64_t, uint16_t*, cudaStream_t);
int launch_quant_gemv(const uint8_t*, const float*, int64_t, int64_t, const uint16_t*, int64_t, const uint16_t*, int64_t,
                      float*, float*, cudaStream_t);
int launch_merge_experts_pack(const uint16_t*, const uint16_t*, const float*, const float*, int64_t,
                              int64_t, int64_t, float, uint16_t*, puzzle_pack_stats*, cudaStream_t);
int launch_route(const float*, int64_t, int, int, int, const int32_t*, int, int32_t*, float*, int32_t*,
                 int32_t*, int32_t*, int32_t*, int32_t*, int32_t*, int, int32_t*, const uint16_t*, int, uint16_t*,
                 bool*, cudaStream_t);
int launch_active_pairs(const int32_t*, int, int32_t*, int32_t*, cudaStream_t);
int64_t route_dec_scratch_ints(int64_t T, int k, int n_pairs);
bool route_dec_fits(int64_t T, int n_pairs);
int launch_route_dec(const float*, int64_t, int, int, int, const int32_t*, int, int32_t*, float*, int32_t*, int32_t*,
                     int32_t*, int32_t*, int32_t*, int32_t*, int, int32_t*, const uint16_t*, int, uint16_t*,
                     cudaStream_t);
const char* last_error_cstr();
int launch_combine(const float*, const int32_t*, const float*, int64_t, int, int, const uint16_t*,
                   uint16_t*, cudaStream_t);
int launch_gather_rows(const uint16_t*, const int32_t*, int64_t, int64_t, uint16_t*, cudaStream_t);
int launch_ep_dispatch(const uint16_t*, const int32_t*, const int32_t*, const int32_t*, int, int, int64_t, int, int,
                       uint16_t*, cudaStream_t);
size_t ep_recv_plan_smem(int world, int lb);
int launch_ep_recv_plan(const uint16_t*, int, int, int64_t, int, int32_t*, int32_t*, int32_t*, uint32_t*, cudaStream_t);
int launch_ep_home_index(const int32_t*, const float*, const int32_t*, int, const int32_t*, int, int64_t, int64_t,
                         int32_t*, float*, int*, cudaStream_t);
size_t ep_peer_buffer_bytes(int world, int64_t cap, int d);
int launch_ep_dispatch_peer(const uint16_t*, const int32_t*, const int32_t*, const int32_t*, int, int, int, int64_t, int,
                            int, const unsigned long long*, uint32_t*, cudaStream_t);
int launch_ep_wait_dispatch(const void*, int, int64_t, int, uint32_t*, cudaStream_t);
int launch_ep_return_peer(const float*, const int32_t*, int, int, int, int64_t, int, const unsigned long long*,
                          uint32_t*, cudaStream_t);
int launch_ep_home_index_peer(const int32_t*, const float*, const int32_t*, int, const int32_t*, int, int64_t, int,
                              int64_t, const void*, int32_t*, float*, uint32_t*, cudaStream_t);
int launch_ep_combine_peer(const int32_t*, const float*, const int32_t*, int, const int32_t*, int, int64_t, int64_t, int,
                           int, const void*, const uint16_t*, uint16_t*, uint32_t*, cudaStream_t);
bool tc_supported(int d, int f);
bool ts_supported(int d, int f);
int launch_gemv_tc_experts_quant(const uint8_t*, const float*, const uint8_t*, const float*, int, int, int,
                                 const uint16_t*, const int32_t*, const int32_t*, const int32_t*, int, int64_t, float*,
                                 int32_t*, int32_t*, uint16_t*, float*, cudaStream_t);
int launch_ts_experts(const uint16_t*, const uint16_t*, const uint8_t*, int, int, int, const uint16_t*, const int32_t*,
                      int64_t, uint16_t*, float*, cudaStream_t);
int launch_tc_experts(const uint16_t*, const uint16_t*, const uint8_t*, int, int, int, const uint16_t*,
                      const int32_t*, int64_t, uint16_t*, float*, int32_t*, cudaStream_t);
size_t gemv_tc_part_floats();
int64_t gemv_tc_counters(int n_rb, int n_pairs, int64_t n_assign);
bool gemv_supported(int d, int f);
size_t calib_workspace_bytes(int n_groups, int64_t cols);
int launch_group_colsumsq(const uint16_t*, const int32_t*, int, int64_t, double*, double*, cudaStream_t);
int launch_gemv_tc_experts(const uint16_t*, const uint16_t*, const uint8_t*, int, int, int, const uint16_t*,
                           const int32_t*,
                           const int32_t*, const int32_t*, int, int64_t, float*, int32_t*, int32_t*,
                           uint16_t*, float*, cudaStream_t);

namespace {
thread_local std::string g_last_error;

struct ProfRec {
  std::string name;
  cudaEvent_t beg, end;
};
bool g_prof_on = false;
std::vector<ProfRec> g_prof;
std::vector<cudaEvent_t> g_event_pool;

cudaEvent_t pool_event() {
  if (!g_event_pool.empty()) {
    cudaEvent_t e = g_event_pool.back();
    g_event_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}
}  // namespace

void prof_mark_begin(const char* name, cudaStream_t s) {
  if (!g_prof_on) return;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(s, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) return;  // graph capture
  ProfRec r{name, pool_event(), pool_event()};
  cudaEventRecord(r.beg, s);
  g_prof.push_back(r);
}

void prof_mark_end(cudaStream_t s) {
  if (!g_prof_on || g_prof.empty()) return;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(s, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) return;
  cudaEventRecord(g_prof.back().end, s);
}

void set_error(const std::string& msg) { g_last_error = msg; }
const char* last_error_cstr() { return g_last_error.c_str(); }

int fail(int status, const std::string& msg) {
  g_last_error = msg;
  return status;
}

int cuda_check(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return PUZZLE_OK;
  return fail(PUZZLE_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

int current_device() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) dev = 0;
  return dev;
}

// SM count of the current device, cached per device ordinal (thread-safe: a racing first
// query stores the same value twice).
int num_sms() {
  static std::atomic<int> cached[64];
  const int dev = current_device() & 63;
  int n = cached[dev].load(std::memory_order_relaxed);
  if (n > 0) return n;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, current_device()) != cudaSuccess || n <= 0)
    n = 148;  // B200
  cached[dev].store(n, std::memory_order_relaxed);
  return n;
}

namespace {

bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

int check_device() {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0)
    return fail(PUZZLE_ERR_CUDA, "no CUDA device: libpuzzlemoe has no CPU fallback");
  return PUZZLE_OK;
}

int check_layer(const puzzle_moe_layer* L) {
  if (!L) return fail(PUZZLE_ERR_INVALID_ARGUMENT, "layer descriptor is NULL");
  if (!L->w13 || !L->w2 || !L->expert_slot)
    return fail(PUZZLE_ERR_INVALID_ARGUMENT, "layer weights / expert_slot NULL");
  if (L->n_pairs < 1 || L->n_experts < 1 || L->n_experts > 2 * L->n_pairs)
    return fail(PUZZLE_ERR_INVALID_ARGUMENT, "need 1 <= n_experts <= 2*n_pairs");
  if (2 * L->n_pairs > kMaxExperts) return fail(PUZZLE_ERR_UNSUPPORTED, "2*n_pairs > 512");
  if (L->d_model < 64 || L->d_ff < 64 || L->d_model % 64 || L->d_ff % 64)
    return fail(PUZZLE_ERR_UNSUPPORTED, "d_model and d_ff must be positive multiples of 64");
  if (!al16(L->w13) || !al16(L->w2)) return fail(PUZZLE_ERR_UNSUPPORTED, "weights must be 16-byte aligned");
  return PUZZLE_OK;
}

// ---- workspace layout of puzzle_moe_forward / puzzle_moe_experts ----
struct Plan {
  int64_t T = 0, n_assign = 0;
  int k = 0, max_active = 0;
  int path = PUZZLE_PATH_GEMV;  // resolved (never AUTO)
};

// Decode shapes (<= 64 tokens) stream each touched pair once through the decode-shape kernels
// (gemv_tc.cu); larger token counts are tensor-bound and go to the tcgen05 grouped GEMM.
constexpr int64_t kGemvMaxTokens = 64;
constexpr int64_t kGemvMaxTokensPerExpert = 96;
constexpr int64_t kGemvMaxTokensPerExpertCoarse = 120;  // d_ff >= 8192 (Mixtral-like experts)

struct Layout {
  size_t topk_idx, topk_gate, bucket_off, assign_token, assign_of, active, n_active, cnt13, cnt2, h, y, part,
      x_perm, route_scratch, total;
};

Plan make_plan(const puzzle_moe_layer* L, int64_t T, int k, int path) {
  Plan p;
  p.T = T;
  p.k = k;
  p.n_assign = T * k;
  p.max_active = (int)std::min<int64_t>(L->n_pairs, p.n_assign);
  // The decode-shape kernels stream each touched pair once per pass of 32 / 64 / 128 tokens per
  // position (NX chosen from the average tokens per expert, gemv_tc.cu): they win while an
  // expert averages < 96 tokens (fine-grained layers: ahead at 72-85, level at 96-102), or
  // < 120 with coarse experts (Mixtral: ahead up to 96, level at 112, TS from 128) --
  // profiles/r02/retune_crossover.txt (with the staged wide reducer; nx128_crossover.log before).
  // Heavier batches: the decode-into-TMEM prefill kernel (gemm_ts.cu; ahead of or level with the
  // shared-memory-operand kernel on every config), else gemm_tc.cu.
  if (path == PUZZLE_PATH_AUTO)
    path = (T <= kGemvMaxTokens || T * k < (L->d_ff >= 8192 ? kGemvMaxTokensPerExpertCoarse : kGemvMaxTokensPerExpert) *
                                                   (int64_t)L->n_experts) ? PUZZLE_PATH_GEMV
           : ts_supported(L->d_model, L->d_ff)                                                ? PUZZLE_PATH_TS
           : tc_supported(L->d_model, L->d_ff)                                                ? PUZZLE_PATH_TC
                                                                                              : PUZZLE_PATH_GEMV;
  p.path = path;
  return p;
}

Layout make_layout(const puzzle_moe_layer* L, const Plan& p) {
  Layout o;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t at = off;
    off += align_up(bytes);
    return at;
  };
  const size_t na = (size_t)p.n_assign, P = (size_t)L->n_pairs, d = L->d_model, f = L->d_ff;
  o.topk_idx = take(na * 4);
  o.topk_gate = take(na * 4);
  o.bucket_off = take((2 * P + 1) * 4);
  o.assign_token = take(na * 4);
  o.assign_of = take(na * 4);
  o.active = take(P * 4);
  o.n_active = take(4);
  // work-item counters of the decode-into-TMEM kernels (also the tile claim counters of the
  // tcgen05 grouped GEMM); zeroed by the routing kernels every call
  o.cnt13 = take((size_t)gemv_tc_counters((int)(f / 64), (int)P, (int64_t)na) * 4);
  o.cnt2 = take((size_t)gemv_tc_counters((int)((d + 127) / 128), (int)P, (int64_t)na) * 4);
  o.h = take(na * f * 2);
  o.y = take(na * d * 4);
  // stream-K partial slots: 2 per CTA x 2 positions x tokens of a pass x 128 fp32
  o.part = take(p.path == PUZZLE_PATH_GEMV ? gemv_tc_part_floats() * 4 : 0);
  o.x_perm = take(na * d * 2);
  o.route_scratch = take((size_t)std::max<int64_t>(2 * 2 * (int64_t)P, route_dec_fits(p.T, (int)P)
                                                                          ? route_dec_scratch_ints(p.T, p.k, (int)P)
                                                                          : 0) * 4);
  o.total = off;
  return o;
}

size_t workspace_for(const puzzle_moe_layer* L, int64_t max_tokens, int k) {
  // The GEMV split factors depend on min(P, T*k); take the max over every distinct plan of
  // either path for any T <= max_tokens.
  size_t best = 0;
  int64_t knee = (L->n_pairs + k - 1) / k;
  for (int path : {(int)PUZZLE_PATH_GEMV, (int)PUZZLE_PATH_TC, (int)PUZZLE_PATH_TS}) {
    if (path == PUZZLE_PATH_TC && !tc_supported(L->d_model, L->d_ff)) continue;
    if (path == PUZZLE_PATH_TS && !ts_supported(L->d_model, L->d_ff)) continue;
    for (int64_t t = 1; t <= std::min<int64_t>(max_tokens, knee); ++t)
      best = std::max(best, make_layout(L, make_plan(L, t, k, path)).total);
    if (max_tokens > 0) best = std::max(best, make_layout(L, make_plan(L, max_tokens, k, path)).total);
  }
  return best;
}

template <typename T>
T* at(void* base, size_t off) {
  return reinterpret_cast<T*>(static_cast<char*>(base) + off);
}

}  // namespace
}  // namespace pz

using namespace pz;

extern "C" {

const char* puzzle_status_string(int status) {
  switch (status) {
    case PUZZLE_OK: return "PUZZLE_OK";
    case PUZZLE_ERR_INVALID_ARGUMENT: return "PUZZLE_ERR_INVALID_ARGUMENT";
    case PUZZLE_ERR_SHAPE_MISMATCH: return "PUZZLE_ERR_SHAPE_MISMATCH";
    case PUZZLE_ERR_UNSUPPORTED: return "PUZZLE_ERR_UNSUPPORTED";
    case PUZZLE_ERR_WORKSPACE: return "PUZZLE_ERR_WORKSPACE";
    case PUZZLE_ERR_CUDA: return "PUZZLE_ERR_CUDA";
    case PUZZLE_ERR_NCCL: return "PUZZLE_ERR_NCCL";
    default: return "PUZZLE_ERR_UNKNOWN";
  }
}

const char* puzzle_last_error(void) { return last_error_cstr(); }

int puzzle_abi_version(void) { return (1 << 16) | 0; }

int puzzle_profile_begin(void) {
  for (auto& r : g_prof) {
    g_event_pool.push_back(r.beg);
    g_event_pool.push_back(r.end);
  }
  g_prof.clear();
  g_prof_on = true;
  return PUZZLE_OK;
}

int puzzle_profile_end(char* buf, size_t buflen) {
  g_prof_on = false;
  std::map<std::string, std::pair<long, double>> agg;
  std::vector<std::string> order;
  for (auto& r : g_prof) {
    if (cudaEventSynchronize(r.end) != cudaSuccess) return fail(PUZZLE_ERR_CUDA, "profile event sync");
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, r.beg, r.end) != cudaSuccess) return fail(PUZZLE_ERR_CUDA, "profile elapsed");
    if (!agg.count(r.name)) order.push_back(r.name);
    agg[r.name].first += 1;
    agg[r.name].second += ms;
  }
  std::string out;
  for (auto& n : order) {
    char line[256];
    snprintf(line, sizeof(line), "%s %ld %.6f\n", n.c_str(), agg[n].first, agg[n].second);
    out += line;
  }
  if (buf && buflen) {
    size_t n = std::min(buflen - 1, out.size());
    memcpy(buf, out.data(), n);
    buf[n] = 0;
  }
  return PUZZLE_OK;
}

int puzzle_merge_pack(const float* w, const uint8_t* m0, const uint8_t* m1, const uint8_t* s0,
                      const uint8_t* s1, int64_t n, uint16_t* out, puzzle_pack_stats* stats,
                      puzzle_stream_t stream) {
  if (n < 0) return fail(PUZZLE_ERR_INVALID_ARGUMENT, "n < 0");
  if (n == 0) return PUZZLE_OK;
  if (!w || !m0 || !m1 || !s0 || !s1 || !out) return fail(PUZZLE_ERR_INVALID_ARGUMENT, "NULL pointer");
  if (int rc = check_device()) return rc;
  return launch_merge_pack(w, m0, m1, s0, s1, n, out, stats, (cudaStream_t)stream);
}

int puzzle_unpack(const uint16_t* packed, int pos, int64_t n, uint16_t* out, puzzle_stream_t stream) {
  if (pos != 0 && pos != 1) return fail(PUZZLE_ERR_INVALID_ARGUMENT, "pos must be 0 or 1");
  if (n < 0) return fail(PUZZLE_ERR_INVALID_ARGUMENT, "n < 0");
  if (n == 0) return PUZZLE_OK;
  if (!packed || !out) return fail(PUZZLE_ERR_INVALID_ARGUMENT, "NULL pointer");
  if (int rc = check_device()) return rc;
  return launch_unpack(packed, pos, n, out, (cudaStream_t)stream);
}

int puzzle_quant_pack(const float* w_merged, const uint8_t* m0, const uint8_t* m1, const uint8_t* s0,
                      const uint8_t* s1, int64_t rows, int64_t cols, uint8_t* codes_out, float* scales_out,
                      puzzle_stream_t stream) {
  if (rows < 0 || cols < 0) return fail(PUZZLE_ERR_INVALID_ARGUMENT, "negative sizes");
  if (cols % 128) return fail(PUZZLE_ERR_UNSUPPORTED, "cols must be a multiple of 128 (quantisation groups)");
  if (rows == 0 || cols == 0) return PUZZLE_OK;
  if (!w_merged || !m0 || !m1 || !s0 || !s1 || !codes_out || !scales_out)
    return fail(PUZZLE_ERR_INVALID_ARGUMENT, "NULL pointer");
  if (!al16(w_merged) || !al16(m0) || !al16(m1) || !al16(s0) || !al16(s1) || !al16(codes_out))
    return fail(PUZZLE_ERR_UNSUPPORTED, "arrays must be 16-byte aligned");
  if (int rc = check_device()) return rc;
  return launch_quant_pack(w_merged, m0, m1, s0, s1, rows, cols, codes_out, scales_out, (cudaStream_t)stream);
}

int puzzle_quant_unpack(const uint8_t* codes, const float* scales, int pos, int64_t rows, int64_t cols,
                        uint16_t* bf16_out, puzzle_stream_t stream) {
  if (pos != 0 && pos != 1) return fail(PUZZLE_ERR_INVALID_ARGUMENT, "pos must be 0 or 1");
  if (rows < 0 || cols < 0) return fail(PUZZLE_ERR_INVALID_ARGUMENT, "negative sizes");
  if (cols % 128) return fail(PUZZLE_ERR_UNSUPPORTED, "cols must be a multiple of 128 (quantisation groups)");
  if (rows == 0 || cols == 0) return PUZZLE_OK;
  if (!codes || !scales || !bf16_out) return fail(PUZZLE_ERR_INVALID_ARGUMENT, "NULL pointer");
  if (!al16(codes) || !al16(bf16_out)) return fail(PUZZLE_ERR_UNSUPPORTED, "arrays must be 16-byte aligned");
  if (int rc = check_device()) return rc;
  return launch_quant_unpack(codes, scales, pos, rows, cols, bf16_out, (cudaStream_t)stream);
}

int puzzle_quant_gemv(const uint8_t* codes, const float* scales, int64_t rows, int64_t cols, const uint16_t* x_i,
                      int64_t n_i, const uint16_t* x_j, int64_t n_j, float* y_i, float* y_j, puzzle_stream_t stream) {
  if (rows < 0 || cols < 0 || n_i < 0 || n_j < 0) return fail(PUZZLE_ERR_INVALID_ARGUMENT, "negative sizes");
  if (cols % 128) return fail(PUZZLE_ERR_UNSUPPORTED, "cols must be a multiple of 128 (quantisation groups)");
  if (rows == 0 || (n_i == 0 && n_j == 0)) return PUZZLE_OK;
  if (cols > 0 && (!codes || !scales)) return fail(PUZZLE_ERR_INVALID_ARGUMENT, "NULL pointer");
  if ((n_i > 0 && (!y_i || (cols > 0 && !x_i))) || (n_j > 0 && (!y_j || (cols > 0 && !x_j))))
    return fail(PUZZLE_ERR_INVALID_ARGUMENT, "NULL pointer");
  if (!al16(codes) || !al16(x_i) || !al16(x_j)) return fail(PUZZLE_ERR_UNSUPPORTED, "arrays must be 16-byte aligned");
  if (int rc = check_device()) return rc;
  return launch_quant_gemv(codes, scales, rows, cols, x_i, n_i, x_j, n_j, y_i, y_j, (cudaStream_t)stream);
}

int puzzle_merge_experts_pack(const uint16_t* wi, const uint16_t* wj, const float* ni, const float* nj,
                              int64_t n_mats, int64_t rows, int64_t cols, float tau, uint16_t* out,
                              puzzle_pack_stats* stats, puzzle_stream_t stream) {
  if (!(tau >= 0.0f && tau <= 1.0f)) return fail(PUZZLE_ERR_INVALID_ARGUMENT, "tau_sim outside [0,1]");
  if (n_mats < 0 || rows < 0 || cols < 0) return fail(PUZZLE_ERR_INVALID_ARGUMENT, "negative size");
  if (n_mats * rows * cols == 0) return PUZZLE_OK;
  if (!wi || !wj || !ni || !nj || !out) return fail(PUZZLE_ERR_INVALID_ARGUMENT, "NULL pointer");
  if (cols % 8) return fail(PUZZLE_ERR_UNSUPPORTED, "cols must be a multiple of 8");
  if (!al16(wi) || !al16(wj) || !al16(ni) || !al16(nj) || !al16(out))
    return fail(PUZZLE_ERR_UNSUPPORTED, "pointers must be 16-byte aligned");
  if (int rc = check_device()) return rc;
  return launch_merge_experts_pack(wi, wj, ni, nj, n_mats, rows, cols, tau, out, stats,
                                   (cudaStream_t)stream);
}

size_t puzzle_moe_workspace_size(const puzzle_moe_layer* L, int64_t max_tokens, int top_k) {
  if (check_layer(L) || max_tokens < 0 || top_k < 1 || top_k > L->n_experts) return 0;
  return workspace_for(L, max_tokens, top_k);
}

size_t puzzle_moe_experts_workspace_size(const puzzle_moe_layer* L, int64_t n_assign) {
  // the experts-only call is laid out like a forward with T = n_assign, k = 1
  if (check_layer(L) || n_assign < 0) return 0;
  return workspace_for(L, n_assign, 1);
}

static int run_experts(const puzzle_moe_layer* L, const Plan& plan, const Layout& lay, void* ws,
                       const uint16_t* x, const int32_t* row_index, const int32_t* bucket_off,
                       const int32_t* active, const int32_t* n_active, float* y, cudaStream_t s,
                       const puzzle_moe_quant_layer* Q = nullptr) {
  const uint16_t* rows = x;
  if (row_index) {  // token permutation into bucket order: both paths read rows by TMA
    int rc = launch_gather_rows(x, row_index, plan.n_assign, L->d_model, at<uint16_t>(ws, lay.x_perm), s);
    if (rc) return rc;
    rows = at<uint16_t>(ws, lay.x_perm);
  }
  if (Q)  // NEXT-3 quantised weight class: the decode-shape kernels over the byte format
    return launch_gemv_tc_experts_quant(Q->w13_codes, Q->w13_scales, Q->w2_codes, Q->w2_scales, L->n_pairs, L->d_model,
                                        L->d_ff, rows, bucket_off, active, n_active, plan.max_active, plan.n_assign,
                                        at<float>(ws, lay.part), at<int32_t>(ws, lay.cnt13), at<int32_t>(ws, lay.cnt2),
                                        at<uint16_t>(ws, lay.h), y, s);
  if (plan.path == PUZZLE_PATH_TS)
    return launch_ts_experts(L->w13, L->w2, L->pair_dense, L->n_pairs, L->d_model, L->d_ff, rows, bucket_off, plan.n_assign,
                             at<uint16_t>(ws, lay.h), y, s);
  if (plan.path == PUZZLE_PATH_TC)
    return launch_tc_experts(L->w13, L->w2, L->pair_dense, L->n_pairs, L->d_model, L->d_ff, rows, bucket_off, plan.n_assign,
                             at<uint16_t>(ws, lay.h), y, at<int32_t>(ws, lay.cnt13), s);  // cnt13: zeroed per call
  return launch_gemv_tc_experts(L->w13, L->w2, L->pair_dense, L->n_pairs, L->d_model, L->d_ff, rows, bucket_off, active,
                                n_active, plan.max_active, plan.n_assign, at<float>(ws, lay.part),
                                at<int32_t>(ws, lay.cnt13), at<int32_t>(ws, lay.cnt2), at<uint16_t>(ws, lay.h), y, s);
}

static size_t calib_bytes(const puzzle_moe_layer* L) {
  return align_up(std::max(calib_workspace_bytes(2 * L->n_pairs, L->d_model),
                           calib_workspace_bytes(2 * L->n_pairs, L->d_ff)));
}

// The forward; with sumsq_x / sumsq_h (NEXT-4) it also accumulates the per-bucket column sums of
// squares of the bucket-ordered x rows and SwiGLU rows, using `calib` bytes after the layout.
static int forward_impl(const puzzle_moe_layer* L, const uint16_t* hidden, const float* logits,
                        int64_t T, int k, int renorm, const uint16_t* residual, uint16_t* out,
                        void* ws, size_t ws_bytes, int path, puzzle_stream_t stream, double* sumsq_x,
                        double* sumsq_h, const puzzle_moe_quant_layer* Q = nullptr) {
  if (int rc = check_layer(L)) return rc;
  if (T < 0) return fail(PUZZLE_ERR_INVALID_ARGUMENT, "T < 0");
  if (k < 1 || k > L->n_experts) return fail(PUZZLE_ERR_INVALID_ARGUMENT, "top_k outside [1, n_experts]");
  if (path < PUZZLE_PATH_AUTO || path > PUZZLE_PATH_TS) return fail(PUZZLE_ERR_INVALID_ARGUMENT, "bad path");
  if (T == 0) return PUZZLE_OK;
  if (!hidden || !logits || !out) return fail(PUZZLE_ERR_INVALID_ARGUMENT, "NULL activation pointer");
  if (hidden == out) return fail(PUZZLE_ERR_INVALID_ARGUMENT, "out must not alias hidden");
  if (!al16(hidden) || !al16(out) || (residual && !al16(residual)))
    return fail(PUZZLE_ERR_UNSUPPORTED, "activations must be 16-byte aligned");
  if (int rc = check_device()) return rc;
  if (path == PUZZLE_PATH_TC && !tc_supported(L->d_model, L->d_ff))
    return fail(PUZZLE_ERR_UNSUPPORTED, "tcgen05 path needs d_model % 256 == 0 and d_ff % 128 == 0");
  if (path == PUZZLE_PATH_TS && !ts_supported(L->d_model, L->d_ff))
    return fail(PUZZLE_ERR_UNSUPPORTED, "TS prefill path needs d_model % 128 == 0 and d_ff % 64 == 0");
  const Plan plan = make_plan(L, T, k, path);
  const Layout lay = make_layout(L, plan);
  const bool calib = sumsq_x || sumsq_h;
  if (!ws || ws_bytes < lay.total + (calib ? calib_bytes(L) : 0))
    return fail(PUZZLE_ERR_WORKSPACE, calib ? "workspace smaller than puzzle_moe_calib_workspace_size(L, T, top_k)"
                                            : "workspace smaller than puzzle_moe_workspace_size(L, T, top_k)");
  cudaStream_t s = (cudaStream_t)stream;
  bool rows_written = false;
  int rc;
  // two-grid routing with the row gather fused (decode and intermediate batches: one top-k CTA per
  // 8 tokens, the slots from per-CTA histograms); larger batches: route.cu's single CTA / three grids
  if (route_dec_fits(T, L->n_pairs)) {
    rc = launch_route_dec(logits, T, L->n_experts, k, renorm, L->expert_slot, L->n_pairs,
                          at<int32_t>(ws, lay.topk_idx), at<float>(ws, lay.topk_gate), at<int32_t>(ws, lay.bucket_off),
                          at<int32_t>(ws, lay.assign_token), at<int32_t>(ws, lay.assign_of),
                          at<int32_t>(ws, lay.active), at<int32_t>(ws, lay.n_active), at<int32_t>(ws, lay.cnt13),
                          (int)((lay.h - lay.cnt13) / 4), at<int32_t>(ws, lay.route_scratch), hidden, L->d_model,
                          at<uint16_t>(ws, lay.x_perm), s);
    rows_written = true;
  } else {
  rc = launch_route(logits, T, L->n_experts, k, renorm, L->expert_slot, L->n_pairs,
                        at<int32_t>(ws, lay.topk_idx), at<float>(ws, lay.topk_gate),
                        at<int32_t>(ws, lay.bucket_off), at<int32_t>(ws, lay.assign_token),
                        at<int32_t>(ws, lay.assign_of), at<int32_t>(ws, lay.active),
                        at<int32_t>(ws, lay.n_active), at<int32_t>(ws, lay.cnt13),
                        (int)((lay.h - lay.cnt13) / 4), at<int32_t>(ws, lay.route_scratch), hidden, L->d_model,
                        at<uint16_t>(ws, lay.x_perm), &rows_written, s);
  }
  if (rc) return rc;
  // rows already in bucket order (fused into the large-batch scatter) or gathered now
  rc = run_experts(L, plan, lay, ws, rows_written ? at<uint16_t>(ws, lay.x_perm) : hidden,
                   rows_written ? nullptr : at<int32_t>(ws, lay.assign_token), at<int32_t>(ws, lay.bucket_off),
                   at<int32_t>(ws, lay.active), at<int32_t>(ws, lay.n_active), at<float>(ws, lay.y), s, Q);
  if (rc) return rc;
  // x_perm and h now hold the bucket-ordered x rows and SwiGLU rows of every assignment
  if (sumsq_x && (rc = launch_group_colsumsq(at<uint16_t>(ws, lay.x_perm), at<int32_t>(ws, lay.bucket_off),
                                             2 * L->n_pairs, L->d_model, sumsq_x, at<double>(ws, lay.total), s)))
    return rc;
  if (sumsq_h && (rc = launch_group_colsumsq(at<uint16_t>(ws, lay.h), at<int32_t>(ws, lay.bucket_off),
                                             2 * L->n_pairs, L->d_ff, sumsq_h, at<double>(ws, lay.total), s)))
    return rc;
  return launch_combine(at<float>(ws, lay.y), at<int32_t>(ws, lay.assign_of), at<float>(ws, lay.topk_gate),
                        T, k, L->d_model, residual, out, s);
}

int puzzle_moe_forward_ex(const puzzle_moe_layer* L, const uint16_t* hidden, const float* logits,
                          int64_t T, int k, int renorm, const uint16_t* residual, uint16_t* out,
                          void* ws, size_t ws_bytes, int path, puzzle_stream_t stream) {
  return forward_impl(L, hidden, logits, T, k, renorm, residual, out, ws, ws_bytes, path, stream, nullptr, nullptr);
}

size_t puzzle_moe_calib_workspace_size(const puzzle_moe_layer* L, int64_t max_tokens, int top_k) {
  const size_t base = puzzle_moe_workspace_size(L, max_tokens, top_k);
  return base ? base + calib_bytes(L) : 0;
}

int puzzle_moe_forward_calib(const puzzle_moe_layer* L, const uint16_t* hidden, const float* logits,
                             int64_t T, int k, int renorm, const uint16_t* residual, uint16_t* out,
                             double* sumsq_x, double* sumsq_h, void* ws, size_t ws_bytes, int path,
                             puzzle_stream_t stream) {
  if (!sumsq_x && !sumsq_h) return fail(PUZZLE_ERR_INVALID_ARGUMENT, "sumsq_x and sumsq_h both NULL");
  if ((sumsq_x && (reinterpret_cast<uintptr_t>(sumsq_x) & 15u)) || (sumsq_h && (reinterpret_cast<uintptr_t>(sumsq_h) & 15u)))
    return fail(PUZZLE_ERR_UNSUPPORTED, "sumsq outputs must be 16-byte aligned");
  return forward_impl(L, hidden, logits, T, k, renorm, residual, out, ws, ws_bytes, path, stream, sumsq_x, sumsq_h);
}

size_t puzzle_group_colsumsq_workspace_size(int n_groups, int64_t cols) {
  if (n_groups < 0 || cols < 0) return 0;
  return calib_workspace_bytes(n_groups, cols);
}

int puzzle_group_colsumsq(const uint16_t* rows, const int32_t* group_off, int n_groups, int64_t cols,
                          double* sumsq, void* ws, size_t ws_bytes, puzzle_stream_t stream) {
  if (n_groups < 0 || cols < 0) return fail(PUZZLE_ERR_INVALID_ARGUMENT, "negative sizes");
  if (n_groups == 0 || cols == 0) return PUZZLE_OK;
  if (!rows || !group_off || !sumsq) return fail(PUZZLE_ERR_INVALID_ARGUMENT, "NULL pointer");
  if (cols % 8 || !al16(rows) || (reinterpret_cast<uintptr_t>(sumsq) & 15u))
    return fail(PUZZLE_ERR_UNSUPPORTED, "cols % 8 == 0 and 16-byte aligned rows / sums required");
  if (int rc = check_device()) return rc;
  if (!ws || ws_bytes < calib_workspace_bytes(n_groups, cols) || (reinterpret_cast<uintptr_t>(ws) & 15u))
    return fail(PUZZLE_ERR_WORKSPACE, "workspace smaller than puzzle_group_colsumsq_workspace_size");
  return launch_group_colsumsq(rows, group_off, n_groups, cols, sumsq, static_cast<double*>(ws), (cudaStream_t)stream);
}

// NEXT-3: the quantised weight class through the forward (decode-shape kernels, any T)
static int quant_view(const puzzle_moe_quant_layer* Q, puzzle_moe_layer& L) {
  if (!Q) return fail(PUZZLE_ERR_INVALID_ARGUMENT, "quant layer descriptor is NULL");
  if (!Q->w13_scales || !Q->w2_scales) return fail(PUZZLE_ERR_INVALID_ARGUMENT, "quant scales NULL");
  if (Q->d_model % 128 || Q->d_ff % 128)
    return fail(PUZZLE_ERR_UNSUPPORTED, "quantised layers need d_model and d_ff multiples of 128 (groups of 128)");
  if ((reinterpret_cast<uintptr_t>(Q->w13_scales) | reinterpret_cast<uintptr_t>(Q->w2_scales)) & 3u)
    return fail(PUZZLE_ERR_UNSUPPORTED, "scales must be 4-byte aligned");
  L = puzzle_moe_layer{Q->n_experts, Q->n_pairs, Q->d_model, Q->d_ff, reinterpret_cast<const uint16_t*>(Q->w13_codes),
                       reinterpret_cast<const uint16_t*>(Q->w2_codes), Q->expert_slot, nullptr};
  return check_layer(&L);
}

size_t puzzle_moe_quant_workspace_size(const puzzle_moe_quant_layer* Q, int64_t max_tokens, int top_k) {
  puzzle_moe_layer L;
  if (quant_view(Q, L) || max_tokens < 0 || top_k < 1 || top_k > L.n_experts) return 0;
  size_t best = 0;  // the GEMV plan of every T <= max_tokens (split factors depend on min(P, T k))
  const int64_t knee = (L.n_pairs + top_k - 1) / top_k;
  for (int64_t t = 1; t <= std::min<int64_t>(max_tokens, knee); ++t)
    best = std::max(best, make_layout(&L, make_plan(&L, t, top_k, PUZZLE_PATH_GEMV)).total);
  if (max_tokens > 0) best = std::max(best, make_layout(&L, make_plan(&L, max_tokens, top_k, PUZZLE_PATH_GEMV)).total);
  return best;
}

int puzzle_moe_forward_quant(const puzzle_moe_quant_layer* Q, const uint16_t* hidden, const float* logits, int64_t T,
                             int k, int renorm, const uint16_t* residual, uint16_t* out, void* ws, size_t ws_bytes,
                             puzzle_stream_t stream) {
  puzzle_moe_layer L;
  if (int rc = quant_view(Q, L)) return rc;
  return forward_impl(&L, hidden, logits, T, k, renorm, residual, out, ws, ws_bytes, PUZZLE_PATH_GEMV, stream, nullptr,
                      nullptr, Q);
}

int puzzle_moe_forward(const puzzle_moe_layer* L, const uint16_t* hidden, const float* logits, int64_t T,
                       int k, int renorm, const uint16_t* residual, uint16_t* out, void* ws,
                       size_t ws_bytes, puzzle_stream_t stream) {
  return puzzle_moe_forward_ex(L, hidden, logits, T, k, renorm, residual, out, ws, ws_bytes,
                               PUZZLE_PATH_AUTO, stream);
}

size_t puzzle_moe_route_workspace_size(const puzzle_moe_layer* L) {
  if (check_layer(L)) return 0;
  // large batches: global counts + cursors; decode batches: the two-grid routing's histograms
  const int64_t ints = std::max<int64_t>(2 * 2 * (int64_t)L->n_pairs,
                                         route_dec_scratch_ints(kGemvMaxTokens, std::min(16, L->n_experts), L->n_pairs));
  return (size_t)ints * sizeof(int32_t);
}

int puzzle_moe_route(const puzzle_moe_layer* L, const float* logits, int64_t T, int k, int renorm,
                     int32_t* topk_idx, float* topk_gate, int32_t* bucket_off, int32_t* assign_token,
                     int32_t* assign_of, void* workspace, size_t workspace_bytes, puzzle_stream_t stream) {
  if (int rc = check_layer(L)) return rc;
  if (T < 0) return fail(PUZZLE_ERR_INVALID_ARGUMENT, "T < 0");
  if (k < 1 || k > L->n_experts) return fail(PUZZLE_ERR_INVALID_ARGUMENT, "top_k outside [1, n_experts]");
  if (!bucket_off || (T > 0 && (!logits || !topk_idx || !topk_gate || !assign_token || !assign_of)))
    return fail(PUZZLE_ERR_INVALID_ARGUMENT, "NULL pointer");
  if (int rc = check_device()) return rc;
  if (T == 0)  // no assignments: every bucket empty (consumers such as the EP dispatch read the offsets)
    return cuda_check(cudaMemsetAsync(bucket_off, 0, (size_t)(2 * L->n_pairs + 1) * sizeof(int32_t),
                                      (cudaStream_t)stream), "route memset");
  if (workspace_bytes < puzzle_moe_route_workspace_size(L) || (!workspace && workspace_bytes))
    return fail(PUZZLE_ERR_WORKSPACE, "workspace smaller than puzzle_moe_route_workspace_size(L)");
  if (T <= kGemvMaxTokens)  // decode batches: the forward's two-grid routing (top-k grid + scatter grid)
    return launch_route_dec(logits, T, L->n_experts, k, renorm, L->expert_slot, L->n_pairs, topk_idx, topk_gate,
                            bucket_off, assign_token, assign_of, nullptr, nullptr, nullptr, 0,
                            static_cast<int32_t*>(workspace), nullptr, L->d_model, nullptr, (cudaStream_t)stream);
  return launch_route(logits, T, L->n_experts, k, renorm, L->expert_slot, L->n_pairs, topk_idx, topk_gate,
                      bucket_off, assign_token, assign_of, nullptr, nullptr, nullptr, 0,
                      static_cast<int32_t*>(workspace), nullptr, L->d_model, nullptr, nullptr, (cudaStream_t)stream);
}

int puzzle_moe_experts(const puzzle_moe_layer* L, const uint16_t* x_rows, const int32_t* bucket_off,
                       int64_t n_assign, float* y_rows, void* ws, size_t ws_bytes, int path,
                       puzzle_stream_t stream) {
  if (int rc = check_layer(L)) return rc;
  if (n_assign < 0) return fail(PUZZLE_ERR_INVALID_ARGUMENT, "n_assign < 0");
  if (n_assign == 0) return PUZZLE_OK;
  if (!x_rows || !bucket_off || !y_rows) return fail(PUZZLE_ERR_INVALID_ARGUMENT, "NULL pointer");
  if (!al16(x_rows) || !al16(y_rows)) return fail(PUZZLE_ERR_UNSUPPORTED, "rows must be 16-byte aligned");
  if (int rc = check_device()) return rc;
  if (path < PUZZLE_PATH_AUTO || path > PUZZLE_PATH_TS) return fail(PUZZLE_ERR_INVALID_ARGUMENT, "bad path");
  if (path == PUZZLE_PATH_TC && !tc_supported(L->d_model, L->d_ff))
    return fail(PUZZLE_ERR_UNSUPPORTED, "tcgen05 path needs d_model % 256 == 0 and d_ff % 128 == 0");
  if (path == PUZZLE_PATH_TS && !ts_supported(L->d_model, L->d_ff))
    return fail(PUZZLE_ERR_UNSUPPORTED, "TS prefill path needs d_model % 128 == 0 and d_ff % 64 == 0");
  // Every pair may be touched: plan with T = n_assign, k = 1 (max_active = min(P, n_assign)).
  Plan plan = make_plan(L, n_assign, 1, path);
  const Layout lay = make_layout(L, plan);
  if (!ws || ws_bytes < lay.total) return fail(PUZZLE_ERR_WORKSPACE, "workspace too small");
  cudaStream_t s = (cudaStream_t)stream;
  // active list = the pairs with rows; counters zeroed
  int rc = cuda_check(cudaMemsetAsync(at<char>(ws, lay.cnt13), 0, lay.h - lay.cnt13, s), "memset");
  if (rc) return rc;
  rc = launch_active_pairs(bucket_off, L->n_pairs, at<int32_t>(ws, lay.active), at<int32_t>(ws, lay.n_active), s);
  if (rc) return rc;
  plan.max_active = L->n_pairs;
  return run_experts(L, plan, lay, ws, x_rows, nullptr, bucket_off, at<int32_t>(ws, lay.active),
                     at<int32_t>(ws, lay.n_active), y_rows, s);
}

int puzzle_moe_combine(const float* y, const int32_t* assign_of, const float* gate, int64_t T, int k,
                       int d, const uint16_t* residual, uint16_t* out, puzzle_stream_t stream) {
  if (T < 0 || k < 1 || d < 4 || d % 4) return fail(PUZZLE_ERR_INVALID_ARGUMENT, "bad sizes");
  if (T == 0) return PUZZLE_OK;
  if (!y || !assign_of || !gate || !out) return fail(PUZZLE_ERR_INVALID_ARGUMENT, "NULL pointer");
  if (int rc = check_device()) return rc;
  return launch_combine(y, assign_of, gate, T, k, d, residual, out, (cudaStream_t)stream);
}

int puzzle_gather_rows(const uint16_t* src, const int32_t* index, int64_t n_rows, int64_t cols,
                       uint16_t* dst, puzzle_stream_t stream) {
  if (n_rows < 0 || cols < 0) return fail(PUZZLE_ERR_INVALID_ARGUMENT, "negative size");
  if (n_rows == 0) return PUZZLE_OK;
  if (!src || !index || !dst) return fail(PUZZLE_ERR_INVALID_ARGUMENT, "NULL pointer");
  if (cols % 8 || !al16(src) || !al16(dst)) return fail(PUZZLE_ERR_UNSUPPORTED, "cols % 8 / alignment");
  if (int rc = check_device()) return rc;
  return launch_gather_rows(src, index, n_rows, cols, dst, (cudaStream_t)stream);
}

int puzzle_ep_dispatch(const uint16_t* hidden, const int32_t* assign_token, const int32_t* bucket_off, int n_pairs,
                       const int32_t* dest_pairs, int world, int64_t n_assign, int64_t cap, int lb_max,
                       int d_model, uint16_t* send_rows, puzzle_stream_t stream) {
  if (n_pairs < 1 || n_assign < 0 || cap < n_assign || lb_max < 0 || d_model < 8)
    return fail(PUZZLE_ERR_INVALID_ARGUMENT, "bad sizes (need n_pairs >= 1, 0 <= n_assign <= cap)");
  if (!dest_pairs || !bucket_off || !send_rows || (n_assign > 0 && (!hidden || !assign_token)))
    return fail(PUZZLE_ERR_INVALID_ARGUMENT, "NULL pointer");
  if (d_model % 8 || !al16(hidden) || !al16(send_rows)) return fail(PUZZLE_ERR_UNSUPPORTED, "d_model % 8 / alignment");
  if (int rc = check_device()) return rc;
  return launch_ep_dispatch(hidden, assign_token, bucket_off, dest_pairs, world, n_pairs, cap, lb_max, d_model,
                            send_rows, (cudaStream_t)stream);
}

static int check_recv_plan_sizes(int world, int n_local_buckets, int64_t cap, int d_model) {
  if (world < 1 || world > 64 || n_local_buckets < 0 || cap < 0 || d_model < 8 || d_model % 8)
    return fail(PUZZLE_ERR_INVALID_ARGUMENT, "bad sizes (1 <= world <= 64, n_local_buckets >= 0, cap >= 0, d_model % 8 == 0)");
  if (4 * (int64_t)n_local_buckets > 2 * (int64_t)d_model)
    return fail(PUZZLE_ERR_INVALID_ARGUMENT, "header row holds 2 * d_model / 4 counts: n_local_buckets too large");
  if (n_local_buckets > 1024 || pz::ep_recv_plan_smem(world, n_local_buckets) > 48 * 1024 ||
      (int64_t)world * (cap + 1) > INT32_MAX)
    return fail(PUZZLE_ERR_UNSUPPORTED, "n_local_buckets <= 1024, world * n_local_buckets <= ~4000, world * (cap + 1) < 2^31");
  return PUZZLE_OK;
}

int puzzle_ep_recv_plan(const uint16_t* recv_rows, int world, int n_local_buckets, int64_t cap, int d_model,
                        int32_t* local_off, int32_t* gather_idx, int32_t* return_idx, puzzle_stream_t stream) {
  if (int rc = check_recv_plan_sizes(world, n_local_buckets, cap, d_model)) return rc;
  if (!recv_rows || !local_off || !return_idx || (cap > 0 && !gather_idx))
    return fail(PUZZLE_ERR_INVALID_ARGUMENT, "NULL pointer");
  if (!al16(recv_rows)) return fail(PUZZLE_ERR_UNSUPPORTED, "recv_rows must be 16-byte aligned");
  if (int rc = check_device()) return rc;
  return launch_ep_recv_plan(recv_rows, world, n_local_buckets, cap, d_model, local_off, gather_idx, return_idx,
                             nullptr, (cudaStream_t)stream);
}

int puzzle_ep_recv_plan_peer(const void* my_base, int world, int n_local_buckets, int64_t cap, int d_model,
                             uint32_t* state, int32_t* local_off, int32_t* gather_idx, int32_t* return_idx,
                             puzzle_stream_t stream) {
  if (int rc = check_recv_plan_sizes(world, n_local_buckets, cap, d_model)) return rc;
  if (!my_base || !state || !local_off || !return_idx || (cap > 0 && !gather_idx))
    return fail(PUZZLE_ERR_INVALID_ARGUMENT, "NULL pointer");
  if (reinterpret_cast<uintptr_t>(my_base) & 255) return fail(PUZZLE_ERR_INVALID_ARGUMENT, "my_base must be 256-byte aligned");
  if (int rc = check_device()) return rc;
  return launch_ep_recv_plan(static_cast<const uint16_t*>(my_base), world, n_local_buckets, cap, d_model, local_off,
                             gather_idx, return_idx, state, (cudaStream_t)stream);
}

int puzzle_ep_home_index(const int32_t* assign_of, const float* topk_gate, const int32_t* bucket_off, int n_pairs,
                         const int32_t* dest_pairs, int world, int64_t cap, int64_t T, int top_k, int32_t* aof_s,
                         float* gate_s, puzzle_stream_t stream) {
  if (n_pairs < 1 || T < 0 || top_k < 1 || cap < T * top_k)
    return fail(PUZZLE_ERR_INVALID_ARGUMENT, "bad sizes (need n_pairs >= 1, T >= 0, top_k >= 1, cap >= T * top_k)");
  if (!dest_pairs || (T > 0 && (!assign_of || !topk_gate || !bucket_off || !aof_s || !gate_s)))
    return fail(PUZZLE_ERR_INVALID_ARGUMENT, "NULL pointer");
  if ((int64_t)world * (cap + 1) > INT32_MAX) return fail(PUZZLE_ERR_UNSUPPORTED, "world * (cap + 1) must fit in int32");
  if (T > 0)
    if (int rc = check_device()) return rc;
  return launch_ep_home_index(assign_of, topk_gate, bucket_off, n_pairs, dest_pairs, world, cap, T * top_k, aof_s,
                              gate_s, nullptr, (cudaStream_t)stream);
}

static int check_peer_common(int world, int rank, int64_t cap, int d_model) {
  if (world < 1 || world > 64 || rank < 0 || rank >= world || cap < 0 || d_model < 8 || d_model % 8)
    return fail(PUZZLE_ERR_INVALID_ARGUMENT, "bad sizes (1 <= world <= 64, 0 <= rank < world, cap >= 0, d_model % 8 == 0)");
  if ((int64_t)world * (cap + 1) > INT32_MAX) return fail(PUZZLE_ERR_UNSUPPORTED, "world * (cap + 1) must fit in int32");
  return PUZZLE_OK;
}

size_t puzzle_ep_peer_buffer_size(int world, int64_t cap, int d_model) {
  if (check_peer_common(world, 0, cap, d_model)) return 0;
  return pz::ep_peer_buffer_bytes(world, cap, d_model);
}

int puzzle_ep_dispatch_peer(const uint16_t* hidden, const int32_t* assign_token, const int32_t* bucket_off,
                            int n_pairs, const int32_t* dest_pairs, int world, int rank, int64_t n_assign,
                            int64_t cap, int lb_max, int d_model, const unsigned long long* peer_bases,
                            uint32_t* state, puzzle_stream_t stream) {
  if (int rc = check_peer_common(world, rank, cap, d_model)) return rc;
  if (n_pairs < 1 || n_assign < 0 || cap < n_assign || lb_max < 0)
    return fail(PUZZLE_ERR_INVALID_ARGUMENT, "bad sizes (need n_pairs >= 1, 0 <= n_assign <= cap)");
  if (!dest_pairs || !bucket_off || !peer_bases || !state || (n_assign > 0 && (!hidden || !assign_token)))
    return fail(PUZZLE_ERR_INVALID_ARGUMENT, "NULL pointer");
  for (int q = 0; q < world; ++q)
    if (!peer_bases[q] || (peer_bases[q] & 255)) return fail(PUZZLE_ERR_INVALID_ARGUMENT, "peer_bases: NULL or not 256-byte aligned");
  if (!al16(hidden)) return fail(PUZZLE_ERR_UNSUPPORTED, "hidden must be 16-byte aligned");
  if (int rc = check_device()) return rc;
  return launch_ep_dispatch_peer(hidden, assign_token, bucket_off, dest_pairs, world, rank, n_pairs, cap, lb_max,
                                 d_model, peer_bases, state, (cudaStream_t)stream);
}

int puzzle_ep_wait_dispatch(const void* my_base, int world, int64_t cap, int d_model, uint32_t* state,
                            puzzle_stream_t stream) {
  if (int rc = check_peer_common(world, 0, cap, d_model)) return rc;
  if (!my_base || !state) return fail(PUZZLE_ERR_INVALID_ARGUMENT, "NULL pointer");
  if (int rc = check_device()) return rc;
  return launch_ep_wait_dispatch(my_base, world, cap, d_model, state, (cudaStream_t)stream);
}

int puzzle_ep_return_peer(const float* y_local, const int32_t* return_idx, int world, int rank, int n_local_buckets,
                          int64_t cap, int d_model, const unsigned long long* peer_bases, uint32_t* state,
                          puzzle_stream_t stream) {
  if (int rc = check_peer_common(world, rank, cap, d_model)) return rc;
  if (n_local_buckets < 0 || 4 * (int64_t)n_local_buckets > 2 * (int64_t)d_model)
    return fail(PUZZLE_ERR_INVALID_ARGUMENT, "n_local_buckets outside [0, d_model / 2]");
  if (!y_local || !return_idx || !peer_bases || !state) return fail(PUZZLE_ERR_INVALID_ARGUMENT, "NULL pointer");
  for (int q = 0; q < world; ++q)
    if (!peer_bases[q] || (peer_bases[q] & 255)) return fail(PUZZLE_ERR_INVALID_ARGUMENT, "peer_bases: NULL or not 256-byte aligned");
  if (!al16(y_local)) return fail(PUZZLE_ERR_UNSUPPORTED, "y_local must be 16-byte aligned");
  if (int rc = check_device()) return rc;
  return launch_ep_return_peer(y_local, return_idx, world, rank, n_local_buckets, cap, d_model, peer_bases, state,
                               (cudaStream_t)stream);
}

int puzzle_ep_home_index_peer(const int32_t* assign_of, const float* topk_gate, const int32_t* bucket_off,
                              int n_pairs, const int32_t* dest_pairs, int world, int64_t cap, int64_t T, int top_k,
                              int d_model, const void* my_base, int32_t* aof_s, float* gate_s, uint32_t* state,
                              puzzle_stream_t stream) {
  if (int rc = check_peer_common(world, 0, cap, d_model)) return rc;
  if (n_pairs < 1 || T < 0 || top_k < 1 || cap < T * top_k)
    return fail(PUZZLE_ERR_INVALID_ARGUMENT, "bad sizes (need n_pairs >= 1, T >= 0, top_k >= 1, cap >= T * top_k)");
  if (!dest_pairs || !my_base || !state || !bucket_off || (T > 0 && (!assign_of || !topk_gate || !aof_s || !gate_s)))
    return fail(PUZZLE_ERR_INVALID_ARGUMENT, "NULL pointer");
  if (int rc = check_device()) return rc;
  return launch_ep_home_index_peer(assign_of, topk_gate, bucket_off, n_pairs, dest_pairs, world, cap, d_model,
                                   T * top_k, my_base, aof_s, gate_s, state, (cudaStream_t)stream);
}

int puzzle_ep_combine_peer(const int32_t* assign_of, const float* topk_gate, const int32_t* bucket_off, int n_pairs,
                           const int32_t* dest_pairs, int world, int64_t cap, int64_t T, int top_k, int d_model,
                           const void* my_base, const uint16_t* residual, uint16_t* out, uint32_t* state,
                           puzzle_stream_t stream) {
  if (int rc = check_peer_common(world, 0, cap, d_model)) return rc;
  if (n_pairs < 1 || T < 0 || T > 65535 || top_k < 1 || cap < T * top_k || d_model % 4)
    return fail(PUZZLE_ERR_INVALID_ARGUMENT, "bad sizes (need n_pairs >= 1, 0 <= T <= 65535, top_k >= 1, cap >= T * top_k)");
  if (!dest_pairs || !my_base || !state || !bucket_off || (T > 0 && (!assign_of || !topk_gate || !out)))
    return fail(PUZZLE_ERR_INVALID_ARGUMENT, "NULL pointer");
  if (reinterpret_cast<uintptr_t>(my_base) & 255) return fail(PUZZLE_ERR_INVALID_ARGUMENT, "my_base must be 256-byte aligned");
  if (int rc = check_device()) return rc;
  return launch_ep_combine_peer(assign_of, topk_gate, bucket_off, n_pairs, dest_pairs, world, cap, T, top_k, d_model,
                                my_base, residual, out, state, (cudaStream_t)stream);
}

}  // extern "C"
