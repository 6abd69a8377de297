#pragma once
#include <cuda.h>

#include <stdint.h>

namespace pz {
// 2-D row-major [rows][cols] 16-bit tensor; box [box_rows][box_cols] (box_cols * 2 B must be
// 128 B for the 128-byte swizzle used everywhere here); OOB rows read as zero.
int make_tmap_2d(CUtensorMap* m, const void* base, int64_t rows, int64_t cols, int box_rows, int box_cols);
int make_tmap_2d_u8(CUtensorMap* m, const void* base, int64_t rows, int64_t cols, int box_rows, int box_cols);
int make_tmap_3d(CUtensorMap* m, const void* base, int64_t n2, int64_t rows, int64_t cols, int64_t stride2_rows,
                 int box_rows, int box_cols, int box_n2);
}  // namespace pz
