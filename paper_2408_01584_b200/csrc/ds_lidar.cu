// ds_lidar.cu -- LiDAR / view-cone observation kernel (fill_lidar,
// observation.py:223-280; _ray_angles 213-220; raycast_obbs_arr
// geometry.py:399-424; raycast_segments_arr 380-396).
//
// One CTA per world, one warp per controlled agent (rows handed to warps
// dynamically), each lane owns rays lane, lane+32, ...  Per ray:
//  * boxes, box-major: the visible partners within max_range +
//    circumradius (the reference's candidate set, compacted first) are
//    tested with the exact FP64 slab test of raycast_obbs_arr only against
//    the rays inside a conservative angular interval around their bounding
//    circle; the minimum is the agent hit;
//  * road segments, segment-major: the warp visits the grid cells of the
//    max-range disc ring by ring around the origin's cell, skips cells whose
//    rays all hit something nearer already, and strides its lanes over the
//    segments binned in the surviving cells (flattened, full warp batches);
//    each segment is tested with the exact FP64 formula of
//    raycast_segments_arr only against the rays inside its angular span seen
//    from the origin, and merged per ray with one 64-bit atomicMin on
//    (distance bits << 1 | not_edge): nearest wins, an exact-distance tie
//    between a road edge and another road kind resolves to the edge (the
//    reference resolves such ties in its BVH traversal order, the oracle
//    uses the same edge-first rule);
//  * a road replaces the box hit only if strictly nearer; beyond max_range
//    the ray reports max_range with type none.
#include "ds_internal.cuh"
#include "ds_obs_out.cuh"
#include "ds_rows.cuh"

namespace ds {

// Dev-only work counters (a build with -DDS_LIDAR_STATS; tools/lidar_work.py):
// the executed exact tests behind the kernel's FP64 roofline.
#ifdef DS_LIDAR_STATS
__device__ unsigned long long g_lidar_stats[8];
#define LIDAR_STAT(i, v) \
  do { if (lane == 0) atomicAdd(&g_lidar_stats[i], (unsigned long long)(v)); } while (0)
#else
#define LIDAR_STAT(i, v) \
  do { } while (0)
#endif

namespace {

// warps per world CTA (2 CTAs per SM): 8 / 12 / 16 / 32 measured 4.94 /
// 5.28 / 4.82 / 5.12 ms at C4 (round 2).  DS_LIDAR_WARPS: A/B builds only
#ifndef DS_LIDAR_WARPS
#define DS_LIDAR_WARPS 16
#endif
constexpr int kLidarWarps = DS_LIDAR_WARPS;

__host__ __device__ inline size_t al16l(size_t v) { return (v + 15) & ~size_t(15); }

// per-agent shared arrays: x, y, c, s, hl, hw, circumradius (f64) + vis (u8),
// then the ego block of every agent (7 floats, padded to 8)
__host__ __device__ inline size_t lidar_agents_bytes(int amax) {
  return al16l((size_t)amax * (7 * sizeof(double) + 1)) + (size_t)amax * 8 * sizeof(float);
}

// per warp: ray dx, dy, box-min bits, segment-key min, limit (8 B each), the
// segment batch (4 f64 + edge flag per lane) + row (+16 B: the staged row is
// shifted by up to 3 floats to the output's phase)
constexpr size_t kSegCacheBytes = 32 * (4 * sizeof(double) + 1);
__host__ __device__ inline size_t lidar_warp_bytes(int obs_width, int n_rays) {
  return al16l((size_t)n_rays * 5 * sizeof(double) + al16l(kSegCacheBytes) + 32 * sizeof(int) +
               al16l((size_t)n_rays * sizeof(float)) + (size_t)obs_width * sizeof(float) + 16);
}

// Upper bound of asin(x) for 0 <= x (tan(asin x) = x / sqrt(1 - x^2) >=
// asin x), pi/2 and above for x >= 0.95: conservative angular half-spans
// without the cost of asinf
__device__ __forceinline__ float asin_upper(float x) {
  return x < 0.95f ? x * rsqrtf(1.0f - x * x) * (1.0f + 1e-6f) : 1.5708f;
}

constexpr double kInvTwoPi = 0.15915494309189535;

// atan2 for |(x, y)| > 0 with |error| < 3e-6 rad (octant reduction + odd
// minimax polynomial); only used for conservative angular ray ranges
__device__ __forceinline__ float fast_atan2(float y, float x) {
  const float ax = fabsf(x), ay = fabsf(y);
  const float a = __fdividef(fminf(ax, ay), fmaxf(ax, ay));
  const float s = a * a;
  // explicit FMAs: the library builds with --fmad=false (FP64 reference
  // arithmetic), which would split this float polynomial into mul + add
  float q = fmaf(s, -0.01172120f, 0.05265332f);
  q = fmaf(s, q, -0.11643287f);
  q = fmaf(s, q, 0.19354346f);
  q = fmaf(s, q, -0.33262347f);
  q = fmaf(s, q, 0.99997726f);
  float r = a * q;
  if (ay > ax) r = 1.57079637f - r;
  if (x < 0.0f) r = 3.14159274f - r;
  return y < 0.0f ? -r : r;
}

// Ray indices whose direction lies in the angular interval [rel, rel + span]
// (rel in [0, 2pi) relative to the sweep centre, widened by the callers far
// beyond the float error of rel, so the tight ceil / floor range is safe):
// full circle rays at 2 pi k / R (range may run past R - 1, callers wrap),
// cone rays at -fov/2 + fov k / (R - 1) (interval tried at rel and rel - 2pi).
__device__ __forceinline__ void ray_range(float rel, float span, bool full, int R, double fov,
                                          int &k_lo, int &k_hi) {
  if (full) {
    // only rays whose direction lies inside the (already widened) interval:
    // ceil / floor, possibly empty (k_hi < k_lo)
    const float scl = (float)R * (float)kInvTwoPi;
    k_lo = (int)ceilf(rel * scl);
    k_hi = (int)floorf((rel + span) * scl);
    if (k_hi - k_lo + 1 >= R) {
      k_lo = 0;
      k_hi = R - 1;
    }
    return;
  }
  if (R == 1) {
    k_lo = 0;
    k_hi = 0;
    return;
  }
  const float scl = (float)(R - 1) / (float)fov, hf = 0.5f * (float)fov;
  int lo = R, hi = -1;
  for (int sh = 0; sh < 2; ++sh) {
    const float rr = sh == 0 ? rel : rel - (float)kTwoPi;
    const int a2 = max((int)ceilf((rr + hf) * scl), 0);
    const int b2 = min((int)floorf((rr + span + hf) * scl), R - 1);
    if (a2 <= b2) {
      lo = min(lo, a2);
      hi = max(hi, b2);
    }
  }
  k_lo = lo;
  k_hi = hi;
}

// Chebyshev ring of cell q in ring-major order (ring r >= 1 holds
// q in [(2r - 1)^2, (2r + 1)^2))
__device__ __forceinline__ int ring_of(int q) {
  if (q <= 0) return 0;
  int s = (int)sqrtf((float)q);
  while (s * s > q) --s;
  while ((s + 1) * (s + 1) <= q) ++s;
  return (s + 1) >> 1;
}

// Cell offsets (dx, dy) from the origin's cell in ring-major order, for
// rings <= kRingTableR (the grid walk reads them instead of recomputing the
// ring / side / position of every cell)
constexpr int kRingTableR = 20;
constexpr int kRingTableN = (2 * kRingTableR + 1) * (2 * kRingTableR + 1);
struct RingTable {
  signed char d[kRingTableN][2];
};
constexpr RingTable make_ring_table() {
  RingTable t{};
  int q = 1;
  for (int r = 1; r <= kRingTableR; ++r) {
    for (int pos = 0; pos < 8 * r; ++pos, ++q) {
      const int side = pos / (2 * r), along = pos - side * 2 * r;
      int dx = 0, dy = 0;
      if (side == 0) { dx = -r + along; dy = -r; }
      else if (side == 1) { dx = r; dy = -r + along; }
      else if (side == 2) { dx = r - along; dy = r; }
      else { dx = -r; dy = r - along; }
      t.d[q][0] = (signed char)dx;
      t.d[q][1] = (signed char)dy;
    }
  }
  return t;
}
__device__ RingTable g_ring_cells = make_ring_table();

__device__ __forceinline__ void ring_cell(int q, bool table, int &dx, int &dy, int &ring) {
  if (table) {
    const char2 d = __ldg(reinterpret_cast<const char2 *>(g_ring_cells.d) + q);
    dx = d.x;
    dy = d.y;
    ring = max(abs(dx), abs(dy));
    return;
  }
  ring = ring_of(q);
  dx = dy = 0;
  if (ring > 0) {
    const int pos = q - (2 * ring - 1) * (2 * ring - 1);
    const int side = pos / (2 * ring), along = pos - side * 2 * ring;
    if (side == 0) { dx = -ring + along; dy = -ring; }
    else if (side == 1) { dx = ring; dy = -ring + along; }
    else if (side == 2) { dx = ring - along; dy = ring; }
    else { dx = -ring; dy = ring - along; }
  }
}

// current upper bound of ray k's road search: the box hit / max_range limit
// or the best segment so far (an unset key decodes to NaN, ignored by fmin)
__device__ __forceinline__ double ray_bound(double lim, unsigned long long seg_key) {
  return fmin(lim, __longlong_as_double((long long)(seg_key >> 1)));
}

// raycast_segments_arr (geo:380-396) for one ray and one segment, returning
// the reference's t (inf = miss) -- but only when it can be <= `beat`: the
// signs and magnitudes of the numerators decide most misses exactly without
// dividing (division preserves signs; |un| > |den| (1 + 2^-50) implies u > 1;
// |tn| > beat |den| (1 + 2^-50) implies t > beat); the reference's divisions
// run only for candidate hits.
__device__ __forceinline__ double ray_segment(double ox, double oy, double dx, double dy,
                                              double ax, double ay, double bx, double by,
                                              double beat) {
  const double ex = bx - ax, ey = by - ay;
  const double wx = ax - ox, wy = ay - oy;
  const double denom = dx * ey - dy * ex;
  if (denom == 0.0) return INFINITY;
  const double tn = wx * ey - wy * ex;
  const double un = wx * dy - wy * dx;
  const double ad = fabs(denom);
  const double ts = denom < 0.0 ? -tn : tn, us = denom < 0.0 ? -un : un;
  // negative quotients (a tiny one could underflow to -0, so keep a guard)
  if (ts < 0.0 && -ts > ad * 1e-280) return INFINITY;
  if (us < 0.0 && -us > ad * 1e-280) return INFINITY;
  if (us > ad * (1.0 + 1e-15)) return INFINITY;
  if (ts > beat * ad * (1.0 + 1e-15)) return INFINITY;
  const double t = tn / denom;
  // 0 <= us <= ad (1 - 1e-15) (the product rounded at most one ulp up, still
  // below ad) proves 0 <= u = us / ad < 1, so the rounded quotient lies in
  // [0, 1] without dividing; only u near 0- or 1 takes the reference's
  // division
  bool u_ok;
  if (us >= 0.0 && us <= ad * (1.0 - 1e-15)) {
    u_ok = true;
  } else {
    const double u = un / denom;
    u_ok = u >= 0.0 && u <= 1.0;
  }
  return t >= 0.0 && u_ok ? t : INFINITY;
}

// raycast_obbs_arr (geo:399-424) for one ray and one box; inf = miss.
__device__ __forceinline__ double ray_box(double ox, double oy, double dx, double dy, double cx,
                                          double cy, double c, double s, double hl, double hw) {
  const double px = (ox - cx) * c + (oy - cy) * s;
  const double py = -(ox - cx) * s + (oy - cy) * c;
  const double rx = dx * c + dy * s;
  const double ry = -dx * s + dy * c;
  double tmin = -INFINITY, tmax = INFINITY;
  bool ok = true;
#pragma unroll
  for (int axis = 0; axis < 2; ++axis) {
    const double p = axis == 0 ? px : py, r = axis == 0 ? rx : ry;
    const double h = axis == 0 ? hl : hw;
    if (r == 0.0) {
      ok = ok && (p >= -h) && (p <= h);
    } else {
      const double ta = (-h - p) / r, tb = (h - p) / r;
      const double lo = fmin(ta, tb), hi = fmax(ta, tb);
      tmin = fmax(tmin, lo);
      tmax = fmin(tmax, hi);
    }
  }
  ok = ok && (tmin <= tmax) && (tmax >= 0.0);
  return ok ? fmax(tmin, 0.0) : INFINITY;
}

// NR > 0: the ray count as a compile-time constant (the default 64: every
// per-warp array sits at a constant offset and the per-ray loops unroll);
// 0: taken from the config at run time.  FULL: a full-circle sweep known at
// compile time (LiDAR), else decided from the config (view cone).  AMAX > 0:
// the agent tables' stride as a compile-time constant (worlds of <= AMAX
// agents), 0: T.max_agents
template <int WARPS, int NR, bool FULL, int AMAX>
__global__ void __launch_bounds__(WARPS * 32, WARPS <= 8 ? 4 : (WARPS <= 16 ? 2 : 1)) obs_lidar_kernel(
    ds_tables T, ds_config C, ds_state St, const uint8_t *mask, const ObsOut O, const float *scale,
    int obs_width, const WorldStrides U) {
  const int R = NR > 0 ? NR : C.n_rays;
  const int w = blockIdx.x;
  if (mask && !mask[w]) return;
  const int64_t c0 = U.c0(T, w);
  const int nrow = (int)(U.c1(T, w) - c0);
  if (nrow == 0) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int next_row;
  if (threadIdx.x == 0) next_row = WARPS;
  const int amax = AMAX > 0 ? AMAX : T.max_agents;
  double *sx = reinterpret_cast<double *>(smem_raw);
  double *sy = sx + amax, *sc = sx + 2 * amax, *ss = sx + 3 * amax, *shl = sx + 4 * amax,
         *shw = sx + 5 * amax, *scr = sx + 6 * amax;
  uint8_t *svis = reinterpret_cast<uint8_t *>(sx + 7 * amax);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t per_warp = NR > 0 ? lidar_warp_bytes(7 + 5 * NR, NR) : lidar_warp_bytes(obs_width, R);
  unsigned char *wb = smem_raw + lidar_agents_bytes(amax) + (size_t)warp * per_warp;
  double *rdx = reinterpret_cast<double *>(wb);
  double *rdy = rdx + R;
  double *rlim = rdy + R;
  unsigned long long *rbest = reinterpret_cast<unsigned long long *>(rlim + R);
  unsigned long long *rseg = rbest + R;
  double *seg_ax = reinterpret_cast<double *>(rseg + R);
  double *seg_ay = seg_ax + 32, *seg_bx = seg_ax + 64, *seg_by = seg_ax + 96;
  uint8_t *seg_ne = reinterpret_cast<uint8_t *>(seg_ax + 128);
  // per-ray float upper bound of the road search bound (limit / best segment
  // hit), rounded up: the cell culling and the walk's stop test read it
  int *fscr = reinterpret_cast<int *>(reinterpret_cast<unsigned char *>(seg_ax) +
                                      al16l(kSegCacheBytes));   // FlatRows compaction
  float *rbf = reinterpret_cast<float *>(fscr + 32);
  float *const row0 = reinterpret_cast<float *>(reinterpret_cast<unsigned char *>(seg_ax) +
                                                al16l(kSegCacheBytes) + 32 * sizeof(int) +
                                                al16l((size_t)R * sizeof(float)));
  const int row0_phase = (int)((reinterpret_cast<uintptr_t>(row0) >> 2) & 3);

  const int64_t a0 = U.a0(T, w);
  const int A = (int)(U.a1(T, w) - a0);
  float *sego = reinterpret_cast<float *>(smem_raw + al16l((size_t)amax * (7 * sizeof(double) + 1)));
  for (int i = threadIdx.x; i < A; i += blockDim.x) {
    const int64_t g = a0 + i;
    const double x = St.x[g], y = St.y[g];
    double c, s;
    sincos(St.heading[g], &s, &c);
    sx[i] = x;
    sy[i] = y;
    sc[i] = c;
    ss[i] = s;
    shl[i] = T.half_l[g];
    shw[i] = T.half_w[g];
    scr[i] = T.circumradius[g];
    const uint16_t f = St.flags[g];
    svis[i] = (f & DS_F_PRESENT) && !(f & DS_F_REMOVED);
    // _fill_ego (obs:129-142), once per agent instead of per row on one lane
    const double gx = T.goal_x[g] - x, gy = T.goal_y[g] - y;
    float *e = sego + 8 * i;
    e[0] = (float)St.speed[g];
    e[1] = (float)T.length[g];
    e[2] = (float)T.width[g];
    e[3] = (float)(gx * c + gy * s);
    e[4] = (float)(-gx * s + gy * c);
    e[5] = (float)hypot(gx, gy);
    e[6] = (f & DS_F_COLLIDED) ? 1.0f : 0.0f;
  }
  // the grid origin in shared memory, read once per row where used (not
  // held in registers across the row loop)
  __shared__ double g_org[2];
  if (threadIdx.x == 0) {
    g_org[0] = T.grid_x0[w];
    g_org[1] = T.grid_y0[w];
  }
  __syncthreads();

  const int64_t cbase = T.grid_cell_off[w];
  const double cs = C.grid_cell;
  const int gnx = T.grid_nx[w], gny = T.grid_ny[w];
  const double max_range = C.max_range;
  const bool full_circle = FULL || C.obs_mode == DS_OBS_LIDAR || C.fov >= kTwoPi;

  // float32 rows without normalisation leave by bulk (TMA) stores
  const bool bulk_out = O.dtype == DS_OBS_F32 && scale == nullptr;
  // rows are handed out dynamically after a static first row per warp
  // (a row's cost varies with how far its rays reach)
  auto grab_row = [&]() {
    int v = 0;
    if (lane == 0) v = atomicAdd(&next_row, 1);
    return __shfl_sync(kFullMask, v, 0);
  };
  for (int r = warp; r < nrow; r = grab_row()) {
    const int64_t orow = c0 + r;
    const int64_t g = T.row_agent[orow];
    const int i = (int)(g - a0);
    const uint16_t f = St.flags[g];
    if (f & (DS_F_DONE | DS_F_REMOVED)) {
      zero_row(O, orow, lane);
      continue;
    }
    LIDAR_STAT(0, 1);
    float *const row = row0 + ((out_row_phase(O, orow) - row0_phase) & 3);
    const double ox = sx[i], oy = sy[i], h = St.heading[g];
    if (bulk_out) {
      // the previous row's bulk store must have read the staged row
      if (lane == 0) bulk_row_wait();
      __syncwarp();
    }
    if (lane < 7) row[lane] = sego[8 * i + lane];   // ego block, formed in the prologue
    double center = h;
    if (C.obs_mode == DS_OBS_VIEW_CONE) center += St.head_angle[g];
    const float fcenter = (float)center;
    // ray directions (_ray_angles, obs:213-220) and per-ray box minima
    #pragma unroll 1
    for (int k = lane; k < R; k += 32) {
      double ang;
      if (full_circle) ang = center + (2.0 * kPi * (double)k) / (double)R;
      else if (R == 1) ang = center;
      else ang = (center - 0.5 * C.fov) + (C.fov * (double)k) / (double)(R - 1);
      sincos(ang, &rdy[k], &rdx[k]);
      rbest[k] = 0x7ff0000000000000ull;   // +inf
    }
    __syncwarp();
    // boxes, box-major: the reference's candidates (visible, not ego, within
    // max_range + circumradius), each tested exactly only against the rays
    // of a conservative angular interval around its bounding circle.  The
    // candidates of up to 256 agents are first compacted (into the idle
    // segment cache), then their (box, ray) pairs are flattened into full
    // warp batches
    int *const clist = reinterpret_cast<int *>(seg_ax);
    for (int a0c = 0; a0c < A; a0c += 256) {
      int ncand = 0;
      for (int j0 = a0c; j0 < min(A, a0c + 256); j0 += 32) {
        const int j = j0 + lane;
        bool cand = false;
        if (j < A && j != i && svis[j]) {
          // float superset of the candidates: a box whose centre is farther
          // than max_range + circumradius cannot be hit within max_range
          const float cx = (float)(sx[j] - ox), cy = (float)(sy[j] - oy);
          const float cr = (float)scr[j] + 1e-3f;
          const float lim = (float)max_range + cr + 1e-3f;
          cand = cx * cx + cy * cy <= lim * lim;
        }
        const unsigned bal = __ballot_sync(kFullMask, cand);
        if (cand) clist[ncand + __popc(bal & ((1u << lane) - 1u))] = j;
        ncand += __popc(bal);
      }
      __syncwarp();
      for (int c0 = 0; c0 < ncand; c0 += 32) {
        int k_lo = 0, n_k = 0;
        if (c0 + lane < ncand) {
          const int j = clist[c0 + lane];
          const float cx = (float)(sx[j] - ox), cy = (float)(sy[j] - oy);
          const float cr = (float)scr[j] + 1e-3f;
          const float d2 = cx * cx + cy * cy;
          int k_hi = R - 1;
          const float dist = sqrt_dn(d2);   // underestimate: wider span
          if (dist > cr + 1e-3f) {
            const float half = asin_upper(cr / dist) + 1e-4f;
            float rel = fast_atan2(cy, cx) - half - fcenter;
            rel -= (float)kTwoPi * floorf(rel * (float)kInvTwoPi);   // [0, 2pi)
            ray_range(rel, 2.0f * half, full_circle, R, C.fov, k_lo, k_hi);
          }
          n_k = k_hi - k_lo + 1 > 0 ? k_hi - k_lo + 1 : 0;
        }
        FlatRows pairs;
        pairs.build(k_lo, n_k, lane, fscr);
        LIDAR_STAT(1, pairs.total);          // exact ray-box slab tests
        for (int p0 = 0; p0 < pairs.total; p0 += 32) {
          int owner;
          const int m = pairs.map_owner(p0, lane, owner);
          if (p0 + lane < pairs.total) {
            const int jj = clist[c0 + owner];
            const int k = m >= R ? m - R : m;
            const double d = ray_box(ox, oy, rdx[k], rdy[k], sx[jj], sy[jj], sc[jj], ss[jj], shl[jj],
                                     shw[jj]);
            if (d != INFINITY)   // d >= 0; + 0.0 maps -0 to +0 so the bit order is the value order
              atomicMin(&rbest[k], (unsigned long long)__double_as_longlong(d + 0.0));
          }
        }
      }
      __syncwarp();
    }
    __syncwarp();
    // per-ray limit for the segment phase: the box hit or max_range
    #pragma unroll 1
    for (int k = lane; k < R; k += 32) {
      rlim[k] = fmin(__longlong_as_double((long long)rbest[k]), max_range) * (1.0 + 1e-12) + 1e-9;
      rseg[k] = 0xffffffffffffffffull;
      rbf[k] = __double2float_ru(rlim[k]);
    }
    __syncwarp();
    // road segments, segment-major, grid cells in Chebyshev rings around the
    // origin's cell, nearest first, 32 cells per batch in ring-major order; a
    // cell of ring >= 2 is skipped when every ray of its angular span already
    // has a hit nearer than the cell, and the walk stops once no ray can
    // still be improved by the remaining cells.  The segments of the kept
    // cells are flattened into full warp batches, and their (segment, ray)
    // pairs again (the segment batch is staged per warp in shared memory)
    {
      asm volatile("" ::: "memory");
      const double gx0 = g_org[0], gy0 = g_org[1];
      const double inv_cs = 1.0 / cs;
      const int ocx = (int)fmin(fmax(floor((ox - gx0) * inv_cs), -1e6), 1e6);
      const int ocy = (int)fmin(fmax(floor((oy - gy0) * inv_cs), -1e6), 1e6);
      const double reach = max_range + 1e-6;
      // a cell of ring r lies >= (r - 1) cells from the origin's cell
      const int rmax = (int)floor(reach * inv_cs) + 1;
      const int n_cells = (2 * rmax + 1) * (2 * rmax + 1);
      const float cell_rad = (float)(cs * 0.7071067811865476) + 1e-3f;
      const bool table = rmax <= kRingTableR;
      // cell culling in float relative to the grid origin: |error| of the
      // cell distances < 1e-4 m here, absorbed by a 2e-3 m margin (culling
      // only ever keeps a superset of the cells that can hold a hit)
      const float fox = (float)(ox - gx0), foy = (float)(oy - gy0), fcs = (float)cs;
      const float freach = (float)reach;
      for (int q0 = 0; q0 < n_cells; q0 += 32) {
        const int q = q0 + lane;
        int sb = 0, cnt = 0;
        if (q < n_cells) {
          int dxc, dyc, ring;
          ring_cell(q, table, dxc, dyc, ring);
          const int ix = ocx + dxc, iy = ocy + dyc;
          if (ix >= 0 && ix < gnx && iy >= 0 && iy < gny) {
            const float xlo = (float)ix * fcs, ylo = (float)iy * fcs;
            const float ddx = fmaxf(fmaxf(xlo - fox, fox - (xlo + fcs)), 0.0f);
            const float ddy = fmaxf(fmaxf(ylo - foy, foy - (ylo + fcs)), 0.0f);
            const float dmin = sqrt_dn(ddx * ddx + ddy * ddy) - 2e-3f;
            bool keep = dmin <= freach;
            if (keep && ring >= 2) {
              // bounding-circle angular span of the cell (ring >= 2: the
              // origin is at least 1.5 cells from the cell centre)
              const float ccx = xlo + 0.5f * fcs - fox, ccy = ylo + 0.5f * fcs - foy;
              const float dc = sqrt_dn(ccx * ccx + ccy * ccy);
              const float half = asin_upper(cell_rad / dc) + 1e-4f;
              float rel = fast_atan2(ccy, ccx) - half - fcenter;
              rel -= (float)kTwoPi * floorf(rel * (float)kInvTwoPi);
              int k_lo, k_hi;
              ray_range(rel, 2.0f * half, full_circle, R, C.fov, k_lo, k_hi);
              keep = false;
              for (int m = k_lo; m <= k_hi && !keep; ++m) {
                const int k = m >= R ? m - R : m;
                keep = !(rbf[k] < dmin);
              }
            }
            if (keep) {
              const int *c = T.aseg_cell_start + cbase + (int64_t)iy * gnx + ix;
              sb = c[0];
              cnt = c[1] - sb;
            }
          }
        }
        FlatRows cells;
        cells.build(sb, cnt, lane, fscr);
        LIDAR_STAT(2, cells.total);        // segments fetched (kept cells)
        LIDAR_STAT(4, min(32, n_cells - q0));   // cells examined
        for (int f0 = 0; f0 < cells.total; f0 += 32) {
          const int e = cells.map(f0, lane);
          int k_lo = 0, n_k = 0;
          if (f0 + lane < cells.total) {
            // FP64 endpoints: one 32-B record (one sector)
            const double2 *sr = reinterpret_cast<const double2 *>(T.aseg_rec) + 2 * (int64_t)e;
            const double2 ra = sr[0], rb = sr[1];
            const double ax = ra.x, ay = ra.y, bx = rb.x, by = rb.y;
            seg_ax[lane] = ax;
            seg_ay[lane] = ay;
            seg_bx[lane] = bx;
            seg_by[lane] = by;
            seg_ne[lane] = T.aseg_edge[e] ? 0 : 1;
            // angular span of the segment seen from the origin (float, widened)
            const float fax = (float)(ax - ox), fay = (float)(ay - oy);
            const float fbx = (float)(bx - ox), fby = (float)(by - oy);
            int k_hi = R - 1;
            if (fminf(fax * fax + fay * fay, fbx * fbx + fby * fby) > 1.0f) {
              const float pa = fast_atan2(fay, fax), pb = fast_atan2(fby, fbx);
              float dlt = pb - pa;
              if (dlt > (float)kPi) dlt -= (float)kTwoPi;
              if (dlt < -(float)kPi) dlt += (float)kTwoPi;
              if (fabsf(dlt) < (float)kPi - 1e-3f) {
                float rel = (dlt >= 0.0f ? pa : pb) - 1e-4f - fcenter;
                rel -= (float)kTwoPi * floorf(rel * (float)kInvTwoPi);   // [0, 2pi)
                ray_range(rel, fabsf(dlt) + 2e-4f, full_circle, R, C.fov, k_lo, k_hi);
              }
            }
            n_k = k_hi - k_lo + 1 > 0 ? k_hi - k_lo + 1 : 0;
          }
          __syncwarp();
          FlatRows pairs;
          pairs.build(k_lo, n_k, lane, fscr);
          LIDAR_STAT(3, pairs.total);      // exact ray-segment tests
          for (int p0 = 0; p0 < pairs.total; p0 += 32) {
            int owner;
            const int m = pairs.map_owner(p0, lane, owner);
            if (p0 + lane < pairs.total) {
              const int k = m >= R ? m - R : m;
              const double lim = rlim[k];
              const double beat = ray_bound(lim, rseg[k]);
              const double t = ray_segment(ox, oy, rdx[k], rdy[k], seg_ax[owner], seg_ay[owner],
                                           seg_bx[owner], seg_by[owner], beat);
              if (t <= lim) {
                atomicMin(&rseg[k], ((unsigned long long)__double_as_longlong(t + 0.0) << 1) |
                                        (unsigned long long)seg_ne[owner]);
                // non-negative floats order like their bits
                atomicMin(reinterpret_cast<unsigned *>(rbf) + k,
                          __float_as_uint(__double2float_ru(t + 0.0)));
              }
            }
          }
          __syncwarp();
        }
        // the remaining cells lie in rings >= ring_of(q0 + 32), at least
        // (that ring - 1) cells from the origin's cell
        int rrem = 0;   // warp-uniform
        if (q0 + 32 < n_cells) {
          int ddx_, ddy_;
          ring_cell(q0 + 32, table, ddx_, ddy_, rrem);
        }
        if (rrem >= 2) {
          // float compare against far rounded down: only ever keeps walking
          // longer than the FP64 test would (extra cells cannot change hits)
          const float far = __double2float_rd((rrem - 1) * cs - 1e-6);
          bool open = false;
          #pragma unroll 1
          for (int k = lane; k < R; k += 32) open = open || !(rbf[k] < far);
          if (!__any_sync(kFullMask, open)) break;
        }
      }
    }
    __syncwarp();
    #pragma unroll 1
    for (int k = lane; k < R; k += 32) {
      double best = __longlong_as_double((long long)rbest[k]);
      int type = best != INFINITY ? 0 : 3;
      const unsigned long long sk = rseg[k];
      if (sk != 0xffffffffffffffffull) {
        const double smin = __longlong_as_double((long long)(sk >> 1));
        if (smin < best) {
          best = smin;
          type = (sk & 1ull) ? 2 : 1;
        }
      }
      if (best > max_range) {
        best = max_range;
        type = 3;
      }
      float *slot = row + 7 + 5 * k;
      slot[0] = (float)best;
      slot[1] = type == 0 ? 1.0f : 0.0f;
      slot[2] = type == 1 ? 1.0f : 0.0f;
      slot[3] = type == 2 ? 1.0f : 0.0f;
      slot[4] = type == 3 ? 1.0f : 0.0f;
    }
    __syncwarp();
    if (bulk_out) {
      write_row_bulk(O, orow, row, obs_width, lane);
    } else {
      write_row(O, orow, row, obs_width, scale, lane);
      __syncwarp();
    }
  }
  if (bulk_out && lane == 0) bulk_row_wait();   // the staging must outlive the copies
}

}  // namespace

// the fast variant: 64 rays over the full circle, worlds of <= 128 agents
// (agent tables at the compile-time stride 128)
constexpr int kLidarStride = 128;
static bool lidar_fast(const ds_config &c, int max_agents) {
  return c.n_rays == 64 && (c.obs_mode == DS_OBS_LIDAR || c.fov >= kTwoPi) && max_agents <= kLidarStride;
}

size_t lidar_smem_bytes(const ds_config &cfg, int max_agents, int obs_width) {
  const int n_rays = (obs_width - 7) / 5;
  const int am = lidar_fast(cfg, max_agents) ? kLidarStride : max_agents;
  return lidar_agents_bytes(am) + (size_t)kLidarWarps * lidar_warp_bytes(obs_width, n_rays);
}

int lidar_warps() { return kLidarWarps; }

cudaError_t configure_lidar_kernels(int max_dynamic_smem) {
  // the opt-in limit covers static + dynamic shared memory (the row counter)
  const void *ks[] = {(const void *)obs_lidar_kernel<kLidarWarps, 64, true, kLidarStride>,
                      (const void *)obs_lidar_kernel<kLidarWarps, 0, false, 0>};
  for (const void *k : ks) {
    cudaFuncAttributes fa;
    cudaError_t e = cudaFuncGetAttributes(&fa, k);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             max_dynamic_smem - (int)fa.sharedSizeBytes);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t launch_lidar(const ds_handle *h, const uint8_t *mask, void *obs, const float *scale,
                         cudaStream_t s) {
  const ObsOut O{obs, h->obs_dtype, h->obs_stride};
  if (lidar_fast(h->cfg, h->tab.max_agents))
    obs_lidar_kernel<kLidarWarps, 64, true, kLidarStride>
        <<<h->tab.n_worlds, kLidarWarps * 32, h->obs_smem, s>>>(h->tab, h->cfg, h->st, mask, O,
                                                                 scale, h->obs_width, world_strides(h));
  else
    obs_lidar_kernel<kLidarWarps, 0, false, 0><<<h->tab.n_worlds, kLidarWarps * 32, h->obs_smem, s>>>(
        h->tab, h->cfg, h->st, mask, O, scale, h->obs_width, world_strides(h));
  return cudaGetLastError();
}

}  // namespace ds

extern "C" int ds_lidar_supported(void) { return 1; }

#ifdef DS_LIDAR_STATS
extern "C" int ds_debug_lidar_stats(unsigned long long *out) {
  cudaMemcpyFromSymbol(out, ds::g_lidar_stats, sizeof(ds::g_lidar_stats));
  unsigned long long z[8] = {0};
  cudaMemcpyToSymbol(ds::g_lidar_stats, z, sizeof(z));
  return 0;
}
#endif
