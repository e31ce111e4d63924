// ds_decimate.cu -- batched polyline decimation (scenario preprocessing,
// SURVEY §8f-4): decimate_polyline (pkg/src/drivesim/geometry.py:84-127) as
// applied by preprocess (pkg/src/drivesim/scenario.py:387-411).
//
// Iterative smallest-effective-area removal: while the minimum, over the
// alive interior points, of the triangle area (prev, i, next) is below the
// threshold, remove that point (ties: the smaller index) and recompute the
// areas of its two neighbours.  The reference pops a lazy-deletion heap keyed
// (area, index, version); a pop returns exactly the alive point with the
// smallest (current area, index), so any exact argmin gives the same removal
// sequence.  Areas use the reference's FP64 expression with no contraction.
//
// One warp per polyline (grid-stride over polylines): the alive interior
// points are lane-strided, each iteration is a warp argmin of (area, index)
// and a one-lane removal; prev / next links and areas live in caller-provided
// scratch (the library allocates nothing).
#include "ds_internal.cuh"

namespace ds {

namespace {

constexpr int kDecWarps = 8;

__device__ __forceinline__ double tri_area(const double *x, const double *y, int64_t a, int64_t b,
                                           int64_t c) {
  // geometry.triangle_area (geo:79-81), same operation order
  return 0.5 * fabs((x[b] - x[a]) * (y[c] - y[a]) - (x[c] - x[a]) * (y[b] - y[a]));
}

__global__ void __launch_bounds__(kDecWarps * 32) decimate_kernel(
    const double *__restrict__ x, const double *__restrict__ y, const int64_t *__restrict__ off,
    int64_t n_poly, const uint8_t *__restrict__ skip, double threshold, uint8_t *keep,
    int32_t *prev, int32_t *next, double *area) {
  const int lane = threadIdx.x & 31;
  const int64_t wstride = (int64_t)gridDim.x * kDecWarps;
  for (int64_t p = (int64_t)blockIdx.x * kDecWarps + (threadIdx.x >> 5); p < n_poly; p += wstride) {
    const int64_t b = off[p];
    const int n = (int)(off[p + 1] - b);
    for (int i = lane; i < n; i += 32) keep[b + i] = 1;
    if (n < 3 || !(threshold > 0.0) || (skip && skip[p])) continue;
    for (int i = lane; i < n; i += 32) {
      prev[b + i] = i - 1;
      next[b + i] = i + 1;
      area[b + i] = (i > 0 && i < n - 1) ? tri_area(x, y, b + i - 1, b + i, b + i + 1) : INFINITY;
    }
    __syncwarp();
    int alive = n - 2;
    while (alive > 0) {
      double best = INFINITY;
      int arg = 0x7fffffff;
      for (int i = 1 + lane; i < n - 1; i += 32) {
        if (!keep[b + i]) continue;
        const double a = area[b + i];
        if (a < best) {   // ascending i per lane: the first minimum is the smallest index
          best = a;
          arg = i;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oa = __shfl_xor_sync(0xffffffffu, arg, o);
        if (ob < best || (ob == best && oa < arg)) {
          best = ob;
          arg = oa;
        }
      }
      if (!(best < threshold)) break;   // also stops on NaN areas, like the heap's a >= t
      if (lane == 0) {
        const int i = arg;
        keep[b + i] = 0;
        const int pv = prev[b + i], nx = next[b + i];
        next[b + pv] = nx;
        prev[b + nx] = pv;
        if (pv > 0) area[b + pv] = tri_area(x, y, b + prev[b + pv], b + pv, b + nx);
        if (nx < n - 1) area[b + nx] = tri_area(x, y, b + pv, b + nx, b + next[b + nx]);
      }
      --alive;
      __syncwarp();
    }
  }
}

}  // namespace

cudaError_t launch_decimate(const double *x, const double *y, const int64_t *poly_off,
                            int64_t n_poly, const uint8_t *skip, double threshold, uint8_t *keep,
                            void *scratch, int64_t n_points, cudaStream_t s) {
  int32_t *prev = static_cast<int32_t *>(scratch);
  int32_t *next = prev + n_points;
  double *area = reinterpret_cast<double *>(next + n_points);
  const int64_t blocks64 = (n_poly + kDecWarps - 1) / kDecWarps;
  const unsigned blocks = (unsigned)(blocks64 < (1 << 20) ? blocks64 : (1 << 20));
  decimate_kernel<<<blocks, kDecWarps * 32, 0, s>>>(x, y, poly_off, n_poly, skip, threshold, keep,
                                                    prev, next, area);
  return cudaGetLastError();
}

}  // namespace ds
