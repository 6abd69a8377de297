// Host-side TMA tensor-map construction (driver entry point fetched through cudart, so the
// library links no libcuda symbol directly).
#include <cuda.h>

#include <mutex>
#include <string>

#include "common.cuh"
#include "tmap.cuh"

namespace pz {

namespace {

// ---------------------------------------------------------------- host: tensor maps
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

}  // namespace

// Encoded maps are cached per thread, keyed by everything the encoding depends on (base
// address, shape, strides, box): a forward re-uses its layer's and workspace's maps instead of
// re-encoding them on every call (the host cost of an un-captured puzzle_moe_forward). A key
// identifies the bytes of a map completely, so a stale entry can never be returned.
struct TmapKey {
  uintptr_t base;
  int64_t a, b, c, d;
  int e, f, g;
  bool operator==(const TmapKey& o) const {
    return base == o.base && a == o.a && b == o.b && c == o.c && d == o.d && e == o.e && f == o.f && g == o.g;
  }
};
struct TmapCache {
  static constexpr int kN = 64;  // small direct-mapped cache (a forward uses <= 26 maps)
  TmapKey key[kN];
  CUtensorMap map[kN];
  bool used[kN] = {};
  static int slot(const TmapKey& k) {
    uint64_t h = (uint64_t)k.base * 0x9E3779B97F4A7C15ull ^ (uint64_t)(k.a * 31 + k.b) * 0xC2B2AE3D27D4EB4Full ^
                 (uint64_t)(k.c * 131 + k.d * 7 + k.e * 13 + k.f * 17 + k.g);
    return (int)((h >> 32) % kN);
  }
};
thread_local TmapCache g_tmaps;

int make_tmap_2d_uncached(CUtensorMap* m, const void* base, int64_t rows, int64_t cols, int box_rows, int box_cols);

int make_tmap_2d(CUtensorMap* m, const void* base, int64_t rows, int64_t cols, int box_rows, int box_cols) {
  const TmapKey k{reinterpret_cast<uintptr_t>(base), rows, cols, 0, 0, box_rows, box_cols, 2};
  const int i = TmapCache::slot(k);
  if (g_tmaps.used[i] && g_tmaps.key[i] == k) {
    *m = g_tmaps.map[i];
    return PUZZLE_OK;
  }
  if (int rc = make_tmap_2d_uncached(m, base, rows, cols, box_rows, box_cols)) return rc;
  g_tmaps.key[i] = k;
  g_tmaps.map[i] = *m;
  g_tmaps.used[i] = true;
  return PUZZLE_OK;
}

int make_tmap_2d_uncached(CUtensorMap* m, const void* base, int64_t rows, int64_t cols, int box_rows, int box_cols) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return fail(PUZZLE_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(PUZZLE_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  return PUZZLE_OK;
}

// 2-D map over a u8 [rows][cols] tensor, box [box_rows][box_cols = 64 bytes], 64-byte swizzle
// (16-byte chunk c of smem row r at chunk c ^ ((r >> 1) & 3): conflict-free 16-byte row reads)
int make_tmap_2d_u8(CUtensorMap* m, const void* base, int64_t rows, int64_t cols, int box_rows, int box_cols) {
  const TmapKey k{reinterpret_cast<uintptr_t>(base), rows, cols, 0, 0, box_rows, box_cols, 100};
  const int i = TmapCache::slot(k);
  if (g_tmaps.used[i] && g_tmaps.key[i] == k) {
    *m = g_tmaps.map[i];
    return PUZZLE_OK;
  }
  EncodeTiledFn fn = encode_fn();
  if (!fn) return fail(PUZZLE_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(PUZZLE_ERR_CUDA, "cuTensorMapEncodeTiled (u8) failed: " + std::to_string((int)r));
  g_tmaps.key[i] = k;
  g_tmaps.map[i] = *m;
  g_tmaps.used[i] = true;
  return PUZZLE_OK;
}

// 3-D map over a [n2][rows][cols] bf16 / u16 tensor whose dim-2 stride is `stride2_rows` rows:
// a box {box_cols, box_rows, box_n2} lands in shared memory as box_n2 consecutive 2-D boxes
// (one TMA instruction for several row blocks that are far apart in memory, e.g. the gate and
// the up rows of the same features of a packed w13 pair).
int make_tmap_3d_uncached(CUtensorMap* m, const void* base, int64_t n2, int64_t rows, int64_t cols,
                          int64_t stride2_rows, int box_rows, int box_cols, int box_n2);

int make_tmap_3d(CUtensorMap* m, const void* base, int64_t n2, int64_t rows, int64_t cols, int64_t stride2_rows,
                 int box_rows, int box_cols, int box_n2) {
  const TmapKey k{reinterpret_cast<uintptr_t>(base), n2, rows, cols, stride2_rows, box_rows, box_cols, 300 + box_n2};
  const int i = TmapCache::slot(k);
  if (g_tmaps.used[i] && g_tmaps.key[i] == k) {
    *m = g_tmaps.map[i];
    return PUZZLE_OK;
  }
  if (int rc = make_tmap_3d_uncached(m, base, n2, rows, cols, stride2_rows, box_rows, box_cols, box_n2)) return rc;
  g_tmaps.key[i] = k;
  g_tmaps.map[i] = *m;
  g_tmaps.used[i] = true;
  return PUZZLE_OK;
}

int make_tmap_3d_uncached(CUtensorMap* m, const void* base, int64_t n2, int64_t rows, int64_t cols,
                          int64_t stride2_rows, int box_rows, int box_cols, int box_n2) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return fail(PUZZLE_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {(cuuint64_t)cols, (cuuint64_t)rows, (cuuint64_t)n2};
  cuuint64_t strides[2] = {(cuuint64_t)cols * 2, (cuuint64_t)stride2_rows * cols * 2};
  cuuint32_t box[3] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows, (cuuint32_t)box_n2};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(PUZZLE_ERR_CUDA, "cuTensorMapEncodeTiled (3-D) failed: " + std::to_string((int)r));
  return PUZZLE_OK;
}

}  // namespace pz
