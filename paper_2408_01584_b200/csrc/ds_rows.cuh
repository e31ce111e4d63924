// ds_rows.cuh -- cell-row ranges of a query disc over a world's uniform
// grid (device_layout.py), flattened into full 32-wide warp batches.
#pragma once

#include "ds_internal.cuh"

namespace ds {

constexpr unsigned kFullMask = 0xffffffffu;

// (int) of f clamped to [lo, hi]; f is an integral float (floorf) or a
// bound far outside the grid, never NaN: branch-free min / max
__device__ __forceinline__ int clampf(float f, int lo, int hi) {
  return (int)fminf(fmaxf(f, (float)lo), (float)hi);
}

// A lower bound of sqrt(x) for x >= 0 from the hardware reciprocal square
// root (relative error < 2^-21, covered by the 4e-6 factor): for culling
// distances that may only be underestimated
__device__ __forceinline__ float sqrt_dn(float x) {
  return x * rsqrtf(fmaxf(x, 1e-30f)) * (1.0f - 4e-6f);
}

// Cell rows of a query disc around (px, py) -- float coordinates relative to
// the grid origin: lane l owns row iy0 + l; the covered cells of a row are
// one contiguous range of the cell-sorted points.  The float arithmetic is
// widened by `marg` (>= 1 mm, far above its rounding error), so the cells
// returned are a superset of those the exact disc touches.
struct RowGeo {
  const int *cell_start;   // world's cell CSR (absolute point indices)
  float px, py, cs, inv_cs, marg;
  int nx, ny, iy0, nrows;
  __device__ __forceinline__ void init(float reach) {
    marg = 1e-3f + 3e-7f * (fabsf(px) + fabsf(py) + reach);
    const float r = reach + marg;
    const float fy0 = (py - r) * inv_cs, fy1 = (py + r) * inv_cs;
    iy0 = 0;
    nrows = 0;
    if (nx > 0 && ny > 0 && fy1 >= 0.0f && fy0 < (float)ny) {
      iy0 = clampf(floorf(fy0), 0, ny - 1);
      nrows = clampf(floorf(fy1), 0, ny - 1) - iy0 + 1;
      nrows = nrows < 32 ? nrows : 32;
    }
  }
  // range() split in two: the lane's two cell-table entries copied
  // asynchronously (cp.async, 4 B each) into shared dst[lane] /
  // dst[32 + lane] (zeros for a lane without cells), so nothing is held in
  // registers while they are in flight across unrelated work.  The caller
  // waits (cp.async.wait_all) and syncs the warp.
  __device__ __forceinline__ void range_issue_async(float reach, int lane, int *dst) const {
    const int *s0 = nullptr, *s1 = nullptr;
    if (lane < nrows) {
      const int iy = iy0 + lane;
      const float ylo = (float)iy * cs, yhi = ylo + cs;
      float dyb = 0.0f;
      if (py < ylo) dyb = ylo - py;
      else if (py > yhi) dyb = py - yhi;
      const float r = reach + marg;
      if (dyb <= r) {
        const float half = sqrtf(r * r - dyb * dyb) + marg;
        const float fx0 = (px - half) * inv_cs, fx1 = (px + half) * inv_cs;
        if (!(fx1 < 0.0f || fx0 >= (float)nx)) {
          const int ix0 = clampf(floorf(fx0), 0, nx - 1), ix1 = clampf(floorf(fx1), 0, nx - 1);
          const int *c = cell_start + (int64_t)iy * nx;
          s0 = c + ix0;
          s1 = c + ix1 + 1;
        }
      }
    }
    if (s0) {
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((uint32_t)__cvta_generic_to_shared(dst + lane)),
                   "l"(s0) : "memory");
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((uint32_t)__cvta_generic_to_shared(dst + 32 + lane)),
                   "l"(s1) : "memory");
    } else {
      dst[lane] = 0;
      dst[32 + lane] = 0;
    }
  }
  // range of lane's row for radius `reach` (a superset of the disc's points)
  __device__ __forceinline__ void range(float reach, int lane, int &sb, int &cnt) const {
    sb = 0;
    cnt = 0;
    if (lane >= nrows) return;
    const int iy = iy0 + lane;
    const float ylo = (float)iy * cs, yhi = ylo + cs;
    float dyb = 0.0f;
    if (py < ylo) dyb = ylo - py;
    else if (py > yhi) dyb = py - yhi;
    const float r = reach + marg;
    if (dyb > r) return;
    const float half = sqrtf(r * r - dyb * dyb) + marg;
    const float fx0 = (px - half) * inv_cs, fx1 = (px + half) * inv_cs;
    if (fx1 < 0.0f || fx0 >= (float)nx) return;
    const int ix0 = clampf(floorf(fx0), 0, nx - 1), ix1 = clampf(floorf(fx1), 0, nx - 1);
    const int *c = cell_start + (int64_t)iy * nx;
    sb = c[ix0];
    cnt = c[ix1 + 1] - sb;
  }
};

// Non-empty cell rows compacted to lanes 0..n-1 with inclusive prefix ends,
// so candidates are visited in full 32-wide batches across row boundaries.
// Lane o of the batch starting at f0 maps to row #(ends <= f0) plus the
// number of row ends inside (f0, f0 + o]: one OR-reduction of end offsets
// and a popcount (ends are distinct because empty rows were dropped).
struct FlatRows {
  int sb, cnt, pe, nr, total, src, base;
  __device__ __forceinline__ void build(int sb_in, int cnt_in, int lane) {
    const unsigned bal = __ballot_sync(kFullMask, cnt_in > 0);
    nr = __popc(bal);
    src = (int)__fns(bal, 0, lane + 1);
    src = (src >= 0 && src < 32) ? src : 0;
    sb = __shfl_sync(kFullMask, sb_in, src);
    cnt = __shfl_sync(kFullMask, cnt_in, src);
    if (lane >= nr) cnt = 0;
    pe = cnt;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int up = __shfl_up_sync(kFullMask, pe, off);
      if (lane >= off) pe += up;
    }
    total = __shfl_sync(kFullMask, pe, 31);
    base = sb - (pe - cnt);   // element index of flattened position f in this row: base + f
  }
  // point index of flattened candidate f0 + lane (valid when f0 + lane < total)
  __device__ __forceinline__ int map(int f0, int lane) const {
    const bool live = lane < nr;
    const int r0 = __popc(__ballot_sync(kFullMask, live && pe <= f0));
    const int off = pe - f0;
    const unsigned E = __reduce_or_sync(kFullMask, (live && off > 0 && off < 32) ? (1u << off) : 0u);
    const int r = (r0 + __popc(E & ((2u << lane) - 1u))) & 31;
    return __shfl_sync(kFullMask, base, r) + f0 + lane;
  }
  // build() with the compaction through 32 ints of per-warp shared scratch
  // (each non-empty lane stores its lane id at its compacted slot) instead
  // of a find-n-th-set-bit per lane
  __device__ __forceinline__ void build(int sb_in, int cnt_in, int lane, int *scratch) {
    const unsigned bal = __ballot_sync(kFullMask, cnt_in > 0);
    nr = __popc(bal);
    __syncwarp();
    if (cnt_in > 0) scratch[__popc(bal & ((1u << lane) - 1u))] = lane;
    __syncwarp();
    src = lane < nr ? scratch[lane] : 0;
    sb = __shfl_sync(kFullMask, sb_in, src);
    cnt = __shfl_sync(kFullMask, cnt_in, src);
    if (lane >= nr) cnt = 0;
    pe = cnt;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int up = __shfl_up_sync(kFullMask, pe, off);
      if (lane >= off) pe += up;
    }
    total = __shfl_sync(kFullMask, pe, 31);
    base = sb - (pe - cnt);
  }
  // as map(), also returning the original lane that owned the range
  __device__ __forceinline__ int map_owner(int f0, int lane, int &owner) const {
    const bool live = lane < nr;
    const int r0 = __popc(__ballot_sync(kFullMask, live && pe <= f0));
    const int off = pe - f0;
    const unsigned E = __reduce_or_sync(kFullMask, (live && off > 0 && off < 32) ? (1u << off) : 0u);
    const int r = (r0 + __popc(E & ((2u << lane) - 1u))) & 31;
    owner = __shfl_sync(kFullMask, src, r);
    return __shfl_sync(kFullMask, base, r) + f0 + lane;
  }
};


}  // namespace ds
