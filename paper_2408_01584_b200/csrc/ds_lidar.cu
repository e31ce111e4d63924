// ds_lidar.cu -- LiDAR / view-cone observation kernel (fill_lidar,
// observation.py:223-280; _ray_angles 213-220; raycast_obbs_arr
// geometry.py:399-424; raycast_segments_arr 380-396).
//
// One CTA per world, one warp per controlled agent, each lane owns rays
// lane, lane+32, ...  Per ray:
//  * boxes: every visible partner within max_range + circumradius (the
//    reference's candidate set) is first rejected cheaply when the ray's line
//    passes farther than its circumradius (+1 mm) from its centre or it lies
//    behind the origin -- a superset test -- then the exact FP64 slab test
//    of raycast_obbs_arr gives the distance; the minimum is the agent hit;
//  * road segments: the ray walks the world's uniform grid row band by row
//    band in increasing distance, testing the segments binned in the covered
//    cells with the exact FP64 formula of raycast_segments_arr; the walk
//    stops once the next band starts beyond the best hit.  The first minimal
//    segment in index order wins (the reference takes the first in BVH
//    order; the two differ only for exact distance ties between segments of
//    different kinds);
//  * a road replaces the box hit only if strictly nearer; beyond max_range
//    the ray reports max_range with type none.
#include "ds_internal.cuh"

namespace ds {

namespace {

constexpr int kLidarWarps = 16;

__host__ __device__ inline size_t al16l(size_t v) { return (v + 15) & ~size_t(15); }

// per-agent shared arrays: x, y, c, s, hl, hw, circumradius (f64) + vis (u8)
__host__ __device__ inline size_t lidar_agents_bytes(int amax) {
  return al16l((size_t)amax * (7 * sizeof(double) + 1));
}

__host__ __device__ inline size_t lidar_warp_bytes(int obs_width, int n_rays) {
  return al16l((size_t)n_rays * 3 * sizeof(double) + (size_t)obs_width * sizeof(float));
}

__device__ __forceinline__ int clampl(double f, int lo, int hi) {
  if (f < (double)lo) return lo;
  if (f > (double)hi) return hi;
  return (int)f;
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
  const double u = un / denom;
  if (t >= 0.0 && u >= 0.0 && u <= 1.0) return t;
  return INFINITY;
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

struct SegGrid {
  const int *cell_start;   // world's all-segment cell CSR (absolute)
  const double *ax, *ay, *bx, *by;
  const int *sid;
  const uint8_t *edge;
  double gx0, gy0, cs, inv_cs;
  int nx, ny;
};

// Nearest segment hit along (ox, oy) + t (dx, dy), t <= limit; returns
// (t, edge) of the first minimal segment in index order.
__device__ double walk_segments(const SegGrid &G, double ox, double oy, double dx, double dy,
                                double limit, bool &edge_out) {
  double best = INFINITY;
  int best_id = 0x7fffffff;
  bool best_edge = false;
  if (G.nx <= 0 || G.ny <= 0) {
    edge_out = false;
    return best;
  }
  const double slack = 1e-6;
  const double y_end = oy + dy * limit;
  const int iya = clampl(floor((oy - G.gy0) * G.inv_cs), -1, G.ny);
  const int iyb = clampl(floor((y_end - G.gy0) * G.inv_cs), -1, G.ny);
  const int step = iyb >= iya ? 1 : -1;
  const double inv_dy = dy != 0.0 ? 1.0 / dy : 0.0;
  for (int iy = iya;; iy += step) {
    if (iy >= 0 && iy < G.ny) {
      const double ylo = G.gy0 + iy * G.cs - slack, yhi = G.gy0 + (iy + 1) * G.cs + slack;
      double t0, t1;
      if (dy == 0.0) {
        if (oy < ylo || oy > yhi) {
          t0 = 1.0;
          t1 = 0.0;
        } else {
          t0 = 0.0;
          t1 = limit;
        }
      } else {
        const double ta = (ylo - oy) * inv_dy, tb = (yhi - oy) * inv_dy;
        t0 = fmax(0.0, fmin(ta, tb) - 1e-9);
        t1 = fmin(limit, fmax(ta, tb) + 1e-9);
      }
      if (t0 > best) break;   // bands further out only hold larger distances
      if (t0 <= t1) {
        const double xa = ox + dx * t0, xb = ox + dx * t1;
        const double xl = fmin(xa, xb) - slack, xh = fmax(xa, xb) + slack;
        if (!(xh < G.gx0 || xl > G.gx0 + G.nx * G.cs)) {
          const int ix0 = clampl(floor((xl - G.gx0) * G.inv_cs), 0, G.nx - 1);
          const int ix1 = clampl(floor((xh - G.gx0) * G.inv_cs), 0, G.nx - 1);
          const int *c = G.cell_start + (int64_t)iy * G.nx;
          const int b = c[ix0], e = c[ix1 + 1];
          for (int k = b; k < e; ++k) {
            const double beat = best < limit ? best : limit;
            const double t =
                ray_segment(ox, oy, dx, dy, G.ax[k], G.ay[k], G.bx[k], G.by[k], beat);
            if (t < best || (t == best && G.sid[k] < best_id)) {
              if (t != INFINITY) {
                best = t;
                best_id = G.sid[k];
                best_edge = G.edge[k];
              }
            }
          }
        }
      }
    } else if ((step > 0 && iy >= G.ny) || (step < 0 && iy < 0)) {
      break;
    }
    if (iy == iyb) break;
  }
  edge_out = best_edge;
  return best;
}

template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32, 1) obs_lidar_kernel(
    ds_tables T, ds_config C, ds_state St, const uint8_t *mask, float *obs, const float *scale,
    int obs_width) {
  const int w = blockIdx.x;
  if (mask && !mask[w]) return;
  const int64_t c0 = T.c_off[w];
  const int nrow = (int)(T.c_off[w + 1] - c0);
  if (nrow == 0) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int amax = T.max_agents;
  double *sx = reinterpret_cast<double *>(smem_raw);
  double *sy = sx + amax, *sc = sx + 2 * amax, *ss = sx + 3 * amax, *shl = sx + 4 * amax,
         *shw = sx + 5 * amax, *scr = sx + 6 * amax;
  uint8_t *svis = reinterpret_cast<uint8_t *>(sx + 7 * amax);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t per_warp = lidar_warp_bytes(obs_width, C.n_rays);
  unsigned char *wb = smem_raw + lidar_agents_bytes(amax) + (size_t)warp * per_warp;
  double *rdx = reinterpret_cast<double *>(wb);
  double *rdy = rdx + C.n_rays;
  unsigned long long *rbest = reinterpret_cast<unsigned long long *>(rdy + C.n_rays);
  float *row = reinterpret_cast<float *>(rbest + C.n_rays);

  const int64_t a0 = T.a_off[w];
  const int A = (int)(T.a_off[w + 1] - a0);
  for (int i = threadIdx.x; i < A; i += blockDim.x) {
    const int64_t g = a0 + i;
    sx[i] = St.x[g];
    sy[i] = St.y[g];
    sc[i] = cos(St.heading[g]);
    ss[i] = sin(St.heading[g]);
    shl[i] = T.half_l[g];
    shw[i] = T.half_w[g];
    scr[i] = T.circumradius[g];
    const uint16_t f = St.flags[g];
    svis[i] = (f & DS_F_PRESENT) && !(f & DS_F_REMOVED);
  }
  __syncthreads();

  SegGrid G;
  const int64_t cbase = T.grid_cell_off[w];
  G.cell_start = T.aseg_cell_start + cbase;
  G.ax = T.aseg_ax; G.ay = T.aseg_ay; G.bx = T.aseg_bx; G.by = T.aseg_by;
  G.sid = T.aseg_id;
  G.edge = T.aseg_edge;
  G.gx0 = T.grid_x0[w];
  G.gy0 = T.grid_y0[w];
  G.cs = C.grid_cell;
  G.inv_cs = 1.0 / C.grid_cell;
  G.nx = T.grid_nx[w];
  G.ny = T.grid_ny[w];
  const double max_range = C.max_range;
  const int R = C.n_rays;
  const bool full_circle = C.obs_mode == DS_OBS_LIDAR || C.fov >= kTwoPi;

  for (int r = warp; r < nrow; r += WARPS) {
    const int64_t orow = c0 + r;
    float *out = obs + orow * (int64_t)obs_width;
    const int64_t g = T.row_agent[orow];
    const int i = (int)(g - a0);
    const uint16_t f = St.flags[g];
    if (f & (DS_F_DONE | DS_F_REMOVED)) {
      for (int c = lane; c < obs_width; c += 32) out[c] = 0.0f;
      continue;
    }
    const double ox = sx[i], oy = sy[i], h = St.heading[g];
    if (lane == 0) {
      // _fill_ego (obs:129-142)
      const double c = sc[i], s = ss[i];
      const double gx = T.goal_x[g] - ox, gy = T.goal_y[g] - oy;
      row[0] = (float)St.speed[g];
      row[1] = (float)T.length[g];
      row[2] = (float)T.width[g];
      row[3] = (float)(gx * c + gy * s);
      row[4] = (float)(-gx * s + gy * c);
      row[5] = (float)hypot(gx, gy);
      row[6] = (f & DS_F_COLLIDED) ? 1.0f : 0.0f;
    }
    double center = h;
    if (C.obs_mode == DS_OBS_VIEW_CONE) center += St.head_angle[g];
    // ray directions (_ray_angles, obs:213-220) and per-ray box minima
    for (int k = lane; k < R; k += 32) {
      double ang;
      if (full_circle) ang = center + (2.0 * kPi * (double)k) / (double)R;
      else if (R == 1) ang = center;
      else ang = (center - 0.5 * C.fov) + (C.fov * (double)k) / (double)(R - 1);
      rdx[k] = cos(ang);
      rdy[k] = sin(ang);
      rbest[k] = 0x7ff0000000000000ull;   // +inf
    }
    __syncwarp();
    // boxes, box-major: the reference's candidates (visible, not ego, within
    // max_range + circumradius), each tested exactly only against the rays
    // of a conservative angular interval around its bounding circle
    for (int j = lane; j < A; j += 32) {
      if (j == i || !svis[j]) continue;
      const double cx = sx[j] - ox, cy = sy[j] - oy;
      const double cr = scr[j];
      if (!(hypot(cx, cy) <= max_range + cr)) continue;
      const double dist = sqrt(cx * cx + cy * cy);
      int k_lo = 0, k_hi = R - 1;
      bool all = dist <= cr + 1e-3;
      double rel = 0.0, half = 0.0;
      if (!all) {
        half = asin(fmin(1.0, (cr + 1e-3) / dist)) + 1e-6;
        rel = atan2(cy, cx) - center;
        rel -= kTwoPi * floor(rel / kTwoPi);           // [0, 2pi)
      }
      if (full_circle && !all) {
        const double scl = (double)R / kTwoPi;
        k_lo = (int)floor((rel - half) * scl - 1e-6);
        k_hi = (int)ceil((rel + half) * scl + 1e-6);
        if (k_hi - k_lo + 1 >= R) {
          k_lo = 0;
          k_hi = R - 1;
        }
      }
      if (!full_circle && !all && R > 1) {
        // cone rays sit at rel angles -fov/2 + fov k/(R-1); try the interval
        // around rel and around rel - 2pi (cone centred on 0)
        const double scl = (double)(R - 1) / C.fov;
        int lo = R, hi = -1;
        for (int sh = 0; sh < 2; ++sh) {
          const double rr = sh == 0 ? rel : rel - kTwoPi;
          const int a = (int)floor((rr - half + 0.5 * C.fov) * scl - 1e-6);
          const int b = (int)ceil((rr + half + 0.5 * C.fov) * scl + 1e-6);
          const int a2 = a < 0 ? 0 : a, b2 = b > R - 1 ? R - 1 : b;
          if (a2 <= b2) {
            lo = min(lo, a2);
            hi = max(hi, b2);
          }
        }
        k_lo = lo;
        k_hi = hi;
      }
      for (int m = k_lo; m <= k_hi; ++m) {
        const int k = ((m % R) + R) % R;
        const double d = ray_box(ox, oy, rdx[k], rdy[k], sx[j], sy[j], sc[j], ss[j], shl[j], shw[j]);
        if (d != INFINITY)   // d >= 0; + 0.0 maps -0 to +0 so the bit order is the value order
          atomicMin(&rbest[k], (unsigned long long)__double_as_longlong(d + 0.0));
      }
    }
    __syncwarp();
    for (int k = lane; k < R; k += 32) {
      const double dx = rdx[k], dy = rdy[k];
      double best = __longlong_as_double((long long)rbest[k]);
      int type = best != INFINITY ? 0 : 3;
      bool edge = false;
      const double limit = fmin(best, max_range) * (1.0 + 1e-12) + 1e-9;
      const double smin = walk_segments(G, ox, oy, dx, dy, limit, edge);
      if (smin < best) {
        best = smin;
        type = edge ? 1 : 2;
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
    if (scale) {
      for (int c = lane; c < obs_width; c += 32) out[c] = row[c] / scale[c];
    } else {
      for (int c = lane; c < obs_width; c += 32) out[c] = row[c];
    }
    __syncwarp();
  }
}

}  // namespace

size_t lidar_smem_bytes(int max_agents, int obs_width) {
  const int n_rays = (obs_width - 7) / 5;
  return lidar_agents_bytes(max_agents) + (size_t)kLidarWarps * lidar_warp_bytes(obs_width, n_rays);
}

int lidar_warps() { return kLidarWarps; }

cudaError_t configure_lidar_kernels(int max_dynamic_smem) {
  return cudaFuncSetAttribute(obs_lidar_kernel<kLidarWarps>,
                              cudaFuncAttributeMaxDynamicSharedMemorySize, max_dynamic_smem);
}

cudaError_t launch_lidar(const ds_handle *h, const uint8_t *mask, float *obs, const float *scale,
                         cudaStream_t s) {
  obs_lidar_kernel<kLidarWarps><<<h->tab.n_worlds, kLidarWarps * 32, h->obs_smem, s>>>(
      h->tab, h->cfg, h->st, mask, obs, scale, h->obs_width);
  return cudaGetLastError();
}

}  // namespace ds

extern "C" int ds_lidar_supported(void) { return 1; }
