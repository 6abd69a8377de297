// Expert parallelism behind the C ABI (BASELINE.json config 5): a C-owned
// NCCL communicator (bootstrapped from an ncclUniqueId the caller broadcasts, e.g. with
// torch.distributed) and the fixed-capacity expert-parallel layer puzzle_moe_forward_ep:
//   route -> puzzle_ep_dispatch -> all-to-all (NCCL, equal splits) -> puzzle_ep_recv_plan ->
//   gather -> local experts -> gather back -> all-to-all -> puzzle_ep_home_index -> combine,
// every step a kernel of this library on the caller's stream, no host synchronisation (the
// layer can be captured in a CUDA graph). The partition of the merged pairs over the ranks
// (the placement unit is the PAIR) is computed here (puzzle_ep_partition).
//
// NCCL is loaded at run time (dlopen of libnccl.so.2: the process may already hold the copy
// PyTorch loaded; the library keeps no link-time NCCL dependency) and compiled against the
// NCCL 2.x header; every NCCL failure returns PUZZLE_ERR_NCCL and aborts the communicator
// (later calls on the handle fail fast).
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <string>
#include <type_traits>
#include <vector>

#include "common.cuh"

namespace pz {

namespace {

struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*);
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*CommAbort)(ncclComm_t);
  const char* (*GetErrorString)(ncclResult_t);
  ncclResult_t (*GroupStart)();
  ncclResult_t (*GroupEnd)();
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  bool ok = false;
  std::string why;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // already in the process (torch)?
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      const char* e = dlerror();
      api.why = std::string("libnccl.so.2 not loadable: ") + (e ? e : "?");
      return;
    }
    bool all = true;
    auto sym = [&](auto& fn, const char* name) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
      if (!fn) all = false;
    };
    sym(api.GetUniqueId, "ncclGetUniqueId");
    sym(api.CommInitRank, "ncclCommInitRank");
    sym(api.CommDestroy, "ncclCommDestroy");
    sym(api.CommAbort, "ncclCommAbort");
    sym(api.GetErrorString, "ncclGetErrorString");
    sym(api.GroupStart, "ncclGroupStart");
    sym(api.GroupEnd, "ncclGroupEnd");
    sym(api.Send, "ncclSend");
    sym(api.Recv, "ncclRecv");
    api.ok = all;
    if (!all) api.why = "libnccl.so.2 lacks an expected symbol";
  });
  return api;
}

size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

// Pairs of every rank (host [world][2]) and the d_ff slices per pair: world <= n_pairs: rank r
// owns pairs [r P / G, (r + 1) P / G); world > n_pairs (world % n_pairs == 0): each pair is split
// along d_ff into S = G / P slices, rank r holds slice r % S of pair r / S (SwiGLU is
// elementwise in d_ff, so a slice's down projection is an exact partial sum).
int partition(int world, int n_pairs, std::vector<int32_t>& dest, int& slices) {
  if (world < 1 || world > 64 || n_pairs < 1) return fail(PUZZLE_ERR_INVALID_ARGUMENT, "partition: 1 <= world <= 64, n_pairs >= 1");
  dest.assign(2 * (size_t)world, 0);
  if (world <= n_pairs) {
    slices = 1;
    for (int r = 0; r < world; ++r) {
      dest[2 * r] = (int32_t)((int64_t)r * n_pairs / world);
      dest[2 * r + 1] = (int32_t)((int64_t)(r + 1) * n_pairs / world);
    }
  } else {
    if (world % n_pairs) return fail(PUZZLE_ERR_UNSUPPORTED, "expert parallelism with world > n_pairs needs world % n_pairs == 0");
    slices = world / n_pairs;
    for (int r = 0; r < world; ++r) {
      dest[2 * r] = r / slices;
      dest[2 * r + 1] = r / slices + 1;
    }
  }
  return PUZZLE_OK;
}

struct EpLayout {
  size_t topk_idx, topk_gate, bucket_off, assign_token, assign_of, route_ws, send, recv, local_off, gidx, ridx, x_local,
      y_local, y_recv, y_back, aof_s, gate_s, experts_ws, total;
  size_t route_ws_bytes, experts_ws_bytes;
};

int ep_layout(int world, const puzzle_moe_layer* route_layer, const puzzle_moe_layer* local, int64_t cap_tokens, int k,
              int slices, int n_local_buckets, EpLayout& o) {
  const size_t G = (size_t)world, d = (size_t)route_layer->d_model, cap = (size_t)cap_tokens * k, na = cap,
               P = (size_t)route_layer->n_pairs, S = (size_t)slices;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t at = off;
    off += align_up(bytes);
    return at;
  };
  o.route_ws_bytes = puzzle_moe_route_workspace_size(route_layer);
  o.experts_ws_bytes = puzzle_moe_experts_workspace_size(local, (int64_t)(G * cap));
  if (!o.route_ws_bytes || !o.experts_ws_bytes) return fail(PUZZLE_ERR_INVALID_ARGUMENT, "route / local layer descriptor rejected");
  o.topk_idx = take(na * 4);
  o.topk_gate = take(na * 4);
  o.bucket_off = take((2 * P + 1) * 4);
  o.assign_token = take(na * 4);
  o.assign_of = take(na * 4);
  o.route_ws = take(o.route_ws_bytes);
  o.send = take(G * (cap + 1) * d * 2);
  o.recv = take(G * (cap + 1) * d * 2);
  o.local_off = take(((size_t)n_local_buckets + 1) * 4);
  o.gidx = take(G * cap * 4);
  o.ridx = take(G * (cap + 1) * 4);
  o.x_local = take(G * cap * d * 2);
  o.y_local = take(G * cap * d * 4);
  o.y_recv = take(G * (cap + 1) * d * 4);
  o.y_back = take(G * (cap + 1) * d * 4);
  o.aof_s = take(na * S * 4);
  o.gate_s = take(na * S * 4);
  o.experts_ws = take(o.experts_ws_bytes);
  o.total = off;
  return PUZZLE_OK;
}

template <typename T>
T* at(void* base, size_t off) {
  return reinterpret_cast<T*>(static_cast<char*>(base) + off);
}

}  // namespace
}  // namespace pz

struct puzzle_ep {
  ncclComm_t comm = nullptr;
  int world = 0, rank = 0, device = 0;
  int broken = 0;  // sticky: a failed NCCL call aborted the communicator
  std::string why;
};

using namespace pz;

namespace {

int nccl_fail(puzzle_ep* ep, ncclResult_t r, const char* what) {
  const NcclApi& api = nccl();
  std::string msg = std::string(what) + ": " + (api.GetErrorString ? api.GetErrorString(r) : "NCCL error");
  if (ep && ep->comm && !ep->broken) {
    api.CommAbort(ep->comm);  // no half-finished collective may linger on the peers' side
    ep->broken = 1;
    ep->why = msg;
  }
  return fail(PUZZLE_ERR_NCCL, msg);
}

// Equal-split all-to-all of `bytes_per_peer` bytes: region q of send goes to rank q, region s
// of recv comes from rank s (grouped point-to-point, NCCL over NVLink / NVSwitch).
int all_to_all(puzzle_ep* ep, const void* send, void* recv, size_t bytes_per_peer, cudaStream_t s) {
  const NcclApi& api = nccl();
  ncclResult_t r = api.GroupStart();
  if (r != ncclSuccess) return nccl_fail(ep, r, "ncclGroupStart");
  for (int q = 0; q < ep->world; ++q) {
    r = api.Send(static_cast<const char*>(send) + q * bytes_per_peer, bytes_per_peer, ncclUint8, q, ep->comm, s);
    if (r != ncclSuccess) break;
    r = api.Recv(static_cast<char*>(recv) + q * bytes_per_peer, bytes_per_peer, ncclUint8, q, ep->comm, s);
    if (r != ncclSuccess) break;
  }
  const ncclResult_t r2 = api.GroupEnd();
  if (r != ncclSuccess) return nccl_fail(ep, r, "ncclSend/ncclRecv");
  if (r2 != ncclSuccess) return nccl_fail(ep, r2, "ncclGroupEnd");
  return PUZZLE_OK;
}

int check_ep(const puzzle_ep* ep) {
  if (!ep) return fail(PUZZLE_ERR_INVALID_ARGUMENT, "puzzle_ep handle is NULL");
  if (ep->broken) return fail(PUZZLE_ERR_NCCL, "communicator aborted after an earlier failure: " + ep->why);
  return PUZZLE_OK;
}

}  // namespace

extern "C" {

int puzzle_ep_unique_id(void* id_out) {
  if (!id_out) return fail(PUZZLE_ERR_INVALID_ARGUMENT, "id_out is NULL");
  const NcclApi& api = nccl();
  if (!api.ok) return fail(PUZZLE_ERR_NCCL, api.why);
  ncclUniqueId id;
  const ncclResult_t r = api.GetUniqueId(&id);
  if (r != ncclSuccess) return nccl_fail(nullptr, r, "ncclGetUniqueId");
  static_assert(sizeof(ncclUniqueId) == PUZZLE_EP_UNIQUE_ID_BYTES, "ncclUniqueId size");
  memcpy(id_out, &id, sizeof(id));
  return PUZZLE_OK;
}

int puzzle_ep_create(puzzle_ep** ep_out, int world, int rank, const void* unique_id, int device) {
  if (!ep_out || !unique_id) return fail(PUZZLE_ERR_INVALID_ARGUMENT, "NULL pointer");
  *ep_out = nullptr;
  if (world < 1 || world > 64 || rank < 0 || rank >= world || device < 0)
    return fail(PUZZLE_ERR_INVALID_ARGUMENT, "need 1 <= world <= 64, 0 <= rank < world, device >= 0");
  int n_dev = 0;
  if (cudaGetDeviceCount(&n_dev) != cudaSuccess || device >= n_dev)
    return fail(PUZZLE_ERR_CUDA, "no such CUDA device: libpuzzlemoe has no CPU fallback");
  const NcclApi& api = nccl();
  if (!api.ok) return fail(PUZZLE_ERR_NCCL, api.why);
  int prev = 0;
  cudaGetDevice(&prev);
  if (int rc = cuda_check(cudaSetDevice(device), "cudaSetDevice")) return rc;
  auto* ep = new puzzle_ep;
  ep->world = world;
  ep->rank = rank;
  ep->device = device;
  ncclUniqueId id;
  memcpy(&id, unique_id, sizeof(id));
  const ncclResult_t r = api.CommInitRank(&ep->comm, world, id, rank);  // collective over the group
  cudaSetDevice(prev);
  if (r != ncclSuccess) {
    delete ep;
    return nccl_fail(nullptr, r, "ncclCommInitRank");
  }
  *ep_out = ep;
  return PUZZLE_OK;
}

int puzzle_ep_destroy(puzzle_ep* ep) {
  if (!ep) return PUZZLE_OK;
  const NcclApi& api = nccl();
  ncclResult_t r = ncclSuccess;
  if (ep->comm && !ep->broken) r = api.CommDestroy(ep->comm);
  delete ep;
  if (r != ncclSuccess) return nccl_fail(nullptr, r, "ncclCommDestroy");
  return PUZZLE_OK;
}

int puzzle_ep_partition(int world, int n_pairs, int32_t* dest_pairs, int* slices) {
  std::vector<int32_t> dest;
  int S = 0;
  if (int rc = partition(world, n_pairs, dest, S)) return rc;
  if (dest_pairs) memcpy(dest_pairs, dest.data(), dest.size() * sizeof(int32_t));
  if (slices) *slices = S;
  return PUZZLE_OK;
}

size_t puzzle_moe_forward_ep_workspace_size(const puzzle_ep* ep, const puzzle_moe_layer* route_layer,
                                            const puzzle_moe_layer* local_shard, int64_t cap_tokens, int top_k) {
  if (!ep || !route_layer || !local_shard || cap_tokens < 1 || top_k < 1) return 0;
  std::vector<int32_t> dest;
  int S = 0;
  if (partition(ep->world, route_layer->n_pairs, dest, S)) return 0;
  EpLayout lay;
  const int lb = 2 * (dest[2 * ep->rank + 1] - dest[2 * ep->rank]);
  if (ep_layout(ep->world, route_layer, local_shard, cap_tokens, top_k, S, lb, lay)) return 0;
  return lay.total;
}

int puzzle_moe_forward_ep(puzzle_ep* ep, const puzzle_moe_layer* route_layer, const puzzle_moe_layer* local_shard,
                          const uint16_t* hidden, const float* router_logits, int64_t T, int64_t cap_tokens, int top_k,
                          int renormalize, const uint16_t* residual, uint16_t* out, void* workspace,
                          size_t workspace_bytes, int path, puzzle_stream_t stream) {
  if (int rc = check_ep(ep)) return rc;
  if (!route_layer || !local_shard) return fail(PUZZLE_ERR_INVALID_ARGUMENT, "layer descriptor is NULL");
  if (T < 0 || cap_tokens < T || cap_tokens < 1 || top_k < 1 || top_k > route_layer->n_experts)
    return fail(PUZZLE_ERR_INVALID_ARGUMENT, "need 0 <= T <= cap_tokens, cap_tokens >= 1, 1 <= top_k <= n_experts");
  if (path < PUZZLE_PATH_AUTO || path > PUZZLE_PATH_TS) return fail(PUZZLE_ERR_INVALID_ARGUMENT, "bad path");
  std::vector<int32_t> dest;
  int S = 0;
  if (int rc = partition(ep->world, route_layer->n_pairs, dest, S)) return rc;
  const int p0 = dest[2 * ep->rank], p1 = dest[2 * ep->rank + 1], lb = 2 * (p1 - p0);
  int lb_max = 0;
  for (int q = 0; q < ep->world; ++q) lb_max = std::max(lb_max, 2 * (dest[2 * q + 1] - dest[2 * q]));
  if (local_shard->n_pairs != p1 - p0 || local_shard->d_model != route_layer->d_model ||
      local_shard->d_ff * S != route_layer->d_ff)
    return fail(PUZZLE_ERR_SHAPE_MISMATCH, "local shard must hold this rank's pairs (puzzle_ep_partition) with d_ff / slices");
  if (!workspace || (T > 0 && (!hidden || !router_logits || !out)))  // T = 0: still joins the collectives
    return fail(PUZZLE_ERR_INVALID_ARGUMENT, "NULL pointer");
  EpLayout lay;
  if (int rc = ep_layout(ep->world, route_layer, local_shard, cap_tokens, top_k, S, lb, lay)) return rc;
  if (workspace_bytes < lay.total) return fail(PUZZLE_ERR_WORKSPACE, "workspace smaller than puzzle_moe_forward_ep_workspace_size");
  int prev = 0;
  cudaGetDevice(&prev);
  if (prev != ep->device)
    if (int rc = cuda_check(cudaSetDevice(ep->device), "cudaSetDevice")) return rc;
  struct Restore {
    int dev, prev;
    ~Restore() {
      if (dev != prev) cudaSetDevice(prev);
    }
  } restore{ep->device, prev};
  void* ws = workspace;
  const cudaStream_t s = (cudaStream_t)stream;
  const int64_t cap = cap_tokens * top_k, G = ep->world, d = route_layer->d_model;
  int rc;
  // 1. route this rank's tokens against the GLOBAL pairing (T = 0: empty buckets)
  if ((rc = puzzle_moe_route(route_layer, router_logits, T, top_k, renormalize, at<int32_t>(ws, lay.topk_idx),
                             at<float>(ws, lay.topk_gate), at<int32_t>(ws, lay.bucket_off), at<int32_t>(ws, lay.assign_token),
                             at<int32_t>(ws, lay.assign_of), at<char>(ws, lay.route_ws), lay.route_ws_bytes, stream)))
    return rc;
  // 2. every owner's rows + a header row of its bucket counts into its fixed region
  if ((rc = puzzle_ep_dispatch(hidden, at<int32_t>(ws, lay.assign_token), at<int32_t>(ws, lay.bucket_off),
                               route_layer->n_pairs, dest.data(), ep->world, T * top_k, cap, lb_max, (int)d,
                               at<uint16_t>(ws, lay.send), stream)))
    return rc;
  // 3. rows (and counts) to the owners
  if ((rc = all_to_all(ep, at<char>(ws, lay.send), at<char>(ws, lay.recv), (size_t)(cap + 1) * d * 2, s))) return rc;
  // 4. owner: regroup by (local bucket, source), local experts, outputs back into arrival slots
  if ((rc = puzzle_ep_recv_plan(at<uint16_t>(ws, lay.recv), ep->world, lb, cap, (int)d, at<int32_t>(ws, lay.local_off),
                                at<int32_t>(ws, lay.gidx), at<int32_t>(ws, lay.ridx), stream)))
    return rc;
  if ((rc = puzzle_gather_rows(at<uint16_t>(ws, lay.recv), at<int32_t>(ws, lay.gidx), G * cap, d,
                               at<uint16_t>(ws, lay.x_local), stream)))
    return rc;
  if ((rc = puzzle_moe_experts(local_shard, at<uint16_t>(ws, lay.x_local), at<int32_t>(ws, lay.local_off), G * cap,
                               at<float>(ws, lay.y_local), at<char>(ws, lay.experts_ws), lay.experts_ws_bytes, path, stream)))
    return rc;
  // (fp32 rows move as pairs of 16-bit columns)
  if ((rc = puzzle_gather_rows(at<uint16_t>(ws, lay.y_local), at<int32_t>(ws, lay.ridx), G * (cap + 1), 2 * d,
                               at<uint16_t>(ws, lay.y_recv), stream)))
    return rc;
  // 5. outputs home
  if ((rc = all_to_all(ep, at<char>(ws, lay.y_recv), at<char>(ws, lay.y_back), (size_t)(cap + 1) * d * 4, s))) return rc;
  if (T == 0) return PUZZLE_OK;
  // 6. home: every (t, j)'s S d_ff-slice partial rows with its gate, then the combine (a6)
  if ((rc = puzzle_ep_home_index(at<int32_t>(ws, lay.assign_of), at<float>(ws, lay.topk_gate),
                                 at<int32_t>(ws, lay.bucket_off), route_layer->n_pairs, dest.data(), ep->world, cap, T,
                                 top_k, at<int32_t>(ws, lay.aof_s), at<float>(ws, lay.gate_s), stream)))
    return rc;
  return puzzle_moe_combine(at<float>(ws, lay.y_back), at<int32_t>(ws, lay.aof_s), at<float>(ws, lay.gate_s), T,
                            top_k * S, (int)d, residual, out, stream);
}

}  // extern "C"
