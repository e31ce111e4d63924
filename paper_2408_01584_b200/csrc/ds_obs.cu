// ds_obs.cu -- observation kernels (World._fill_obs, engine.py:500-512).
//
// Radial mode (fill_radial / radial_fill_core, observation.py:145-210,
// _fastpath.py:214-302): one warp per controlled agent, a CTA per world.  The
// world's agents sit in shared memory; road points are read from the world's
// uniform grid (device_layout.py): for every cell row that the radius disc
// touches, the points of the covered cells form ONE contiguous, cell-sorted
// range, read lane-strided (coalesced, L1/L2 resident across the world's
// agents).  Distances are FP64 with the glibc hypot port (ds_math.cuh), so
// radius membership and ordering are bit-identical to the reference.
//
// Exact top-k (the reference's insertion sort: nearest first, equal distances
// keep the smaller index): candidates (d, id) are pushed into a per-warp
// shared buffer with ballot compaction; selection is a monotone 256-bucket
// histogram of d (prefix scan -> threshold bucket b*), a counting-sort
// scatter of buckets <= b*, then an exact (d, id) rank inside each bucket.
// Small sets use a direct O(n^2/32) rank.  Buffers that fill up are compacted
// to their exact top-k on the fly (the union argument keeps this exact).
#include "ds_internal.cuh"

namespace ds {

constexpr unsigned kFull = 0xffffffffu;

struct WarpScratch {
  double *cd;      // [kCandCap] candidate distance
  int *cid;        // [kCandCap] tie-break id (original index in the world)
  int *caux;       // [kCandCap] payload (agent slot / grid-sorted point index)
  double *sd;      // [kSelCap]
  int *sid;
  int *saux;
  uint32_t *hc;    // [kBuckets] (cursor << 16) | count
  float *row;      // [row_pad]
};

__host__ __device__ inline int row_pad(int obs_width) { return (obs_width + 3) & ~3; }

size_t obs_smem_bytes(const ds_config &cfg, int max_agents, int warps, int obs_width) {
  (void)cfg;
  size_t agents = (size_t)max_agents * (6 * sizeof(double) + 1);
  agents = (agents + 15) & ~size_t(15);
  size_t per_warp = kCandCap * (sizeof(double) + 2 * sizeof(int)) +
                    kSelCap * (sizeof(double) + 2 * sizeof(int)) + kBuckets * sizeof(uint32_t) +
                    (size_t)row_pad(obs_width) * sizeof(float);
  per_warp = (per_warp + 15) & ~size_t(15);
  return agents + per_warp * warps;
}

__device__ __forceinline__ bool key_less(double da, int ia, double db, int ib) {
  return da < db || (da == db && ia < ib);
}

__device__ __forceinline__ int bucket_of(double d, double scale) {
  double b = d * scale;
  int k = (int)b;   // d >= 0
  return k < kBuckets ? k : kBuckets - 1;
}

// Direct rank of all n candidates: element with rank < k goes to s*[rank].
__device__ void rank_all(const WarpScratch &ws, int n, int k, int lane) {
  for (int p = lane; p < n; p += 32) {
    const double dp = ws.cd[p];
    const int ip = ws.cid[p];
    int rank = 0;
    for (int q = 0; q < n; ++q) rank += key_less(ws.cd[q], ws.cid[q], dp, ip) ? 1 : 0;
    if (rank < k) {
      ws.sd[rank] = dp;
      ws.sid[rank] = ip;
      ws.saux[rank] = ws.caux[p];
    }
  }
}

// Exact ascending top-min(n,k) of the candidate buffer, left in cd/cid/caux[0..m).
// k <= kSelCap.  Returns m.
__device__ int warp_topk(const WarpScratch &ws, int n, int k, double radius, int lane) {
  const int m = n < k ? n : k;
  if (m == 0) return 0;
  __syncwarp();
  if (n <= 64) {
    rank_all(ws, n, k, lane);
    __syncwarp();
    for (int p = lane; p < m; p += 32) {
      ws.cd[p] = ws.sd[p];
      ws.cid[p] = ws.sid[p];
      ws.caux[p] = ws.saux[p];
    }
    __syncwarp();
    return m;
  }
  const double scale = radius > 0.0 ? (double)kBuckets / radius : 0.0;
  for (int b = lane; b < kBuckets; b += 32) ws.hc[b] = 0u;
  __syncwarp();
  for (int p = lane; p < n; p += 32) atomicAdd(&ws.hc[bucket_of(ws.cd[p], scale)], 1u);
  __syncwarp();
  // Exclusive prefix of the counts; each lane owns 8 consecutive buckets.
  constexpr int kPer = kBuckets / 32;
  uint32_t cnt[kPer];
  uint32_t local = 0;
#pragma unroll
  for (int q = 0; q < kPer; ++q) {
    cnt[q] = ws.hc[lane * kPer + q];
    local += cnt[q];
  }
  uint32_t incl = local;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const uint32_t up = __shfl_up_sync(kFull, incl, off);
    if (lane >= off) incl += up;
  }
  uint32_t run = incl - local;
  // Threshold bucket b*: first bucket whose inclusive count reaches k.
  int bstar = kBuckets;
#pragma unroll
  for (int q = 0; q < kPer; ++q) {
    ws.hc[lane * kPer + q] = (run << 16) | cnt[q];
    if (bstar == kBuckets && run < (uint32_t)k && run + cnt[q] >= (uint32_t)k) bstar = lane * kPer + q;
    run += cnt[q];
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) bstar = min(bstar, __shfl_xor_sync(kFull, bstar, off));
  const uint32_t n_sel = bstar < kBuckets ? ((ws.hc[bstar] >> 16) + (ws.hc[bstar] & 0xffffu))
                                          : (uint32_t)n;
  __syncwarp();
  if (n_sel > (uint32_t)kSelCap) {
    // Pathological threshold bucket: exact O(n^2) rank of everything.
    rank_all(ws, n, k, lane);
    __syncwarp();
    for (int p = lane; p < m; p += 32) {
      ws.cd[p] = ws.sd[p];
      ws.cid[p] = ws.sid[p];
      ws.caux[p] = ws.saux[p];
    }
    __syncwarp();
    return m;
  }
  // Counting-sort scatter of buckets <= b*.
  for (int p = lane; p < n; p += 32) {
    const int b = bucket_of(ws.cd[p], scale);
    if (b <= bstar) {
      const uint32_t pos = atomicAdd(&ws.hc[b], 1u << 16) >> 16;
      ws.sd[pos] = ws.cd[p];
      ws.sid[pos] = ws.cid[p];
      ws.saux[pos] = ws.caux[p];
    }
  }
  __syncwarp();
  // Exact (d, id) rank inside each bucket; cursor now = start + count.
  for (int p = lane; p < (int)n_sel; p += 32) {
    const double dp = ws.sd[p];
    const int ip = ws.sid[p];
    const uint32_t hcv = ws.hc[bucket_of(dp, scale)];
    const int cntb = (int)(hcv & 0xffffu);
    const int start = (int)(hcv >> 16) - cntb;
    int rank = start;
    for (int q = start; q < start + cntb; ++q) rank += key_less(ws.sd[q], ws.sid[q], dp, ip) ? 1 : 0;
    if (rank < k) {
      ws.cd[rank] = dp;
      ws.cid[rank] = ip;
      ws.caux[rank] = ws.saux[p];
    }
  }
  __syncwarp();
  return m;
}

// Ballot-compacted push of one candidate per lane into the buffer.
__device__ __forceinline__ int warp_push(const WarpScratch &ws, int n, bool ok, double d, int id,
                                         int aux, int lane) {
  const unsigned bal = __ballot_sync(kFull, ok);
  if (ok) {
    const int pos = n + __popc(bal & ((1u << lane) - 1u));
    ws.cd[pos] = d;
    ws.cid[pos] = id;
    ws.caux[pos] = aux;
  }
  return n + __popc(bal);
}

__device__ __forceinline__ int clampi(double f, int lo, int hi) {
  if (f < (double)lo) return lo;
  if (f > (double)hi) return hi;
  return (int)f;
}

template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32) obs_radial_kernel(ds_tables T, ds_config C,
                                                              ds_state S, const uint8_t *mask,
                                                              float *obs, const float *scale,
                                                              int32_t *sel_idx, int obs_width) {
  const int w = blockIdx.x;
  if (mask && !mask[w]) return;
  const int64_t c0 = T.c_off[w];
  const int nrow = (int)(T.c_off[w + 1] - c0);
  if (nrow == 0) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int amax = T.max_agents;
  double *ax = reinterpret_cast<double *>(smem_raw);
  double *ay = ax + amax, *ah = ax + 2 * amax, *av = ax + 3 * amax, *al = ax + 4 * amax,
         *aw = ax + 5 * amax;
  uint8_t *avis = reinterpret_cast<uint8_t *>(ax + 6 * amax);
  size_t agents_bytes = ((size_t)amax * (6 * sizeof(double) + 1) + 15) & ~size_t(15);
  const int rp = row_pad(obs_width);
  size_t per_warp = kCandCap * (sizeof(double) + 2 * sizeof(int)) +
                    kSelCap * (sizeof(double) + 2 * sizeof(int)) + kBuckets * sizeof(uint32_t) +
                    (size_t)rp * sizeof(float);
  per_warp = (per_warp + 15) & ~size_t(15);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char *wb = smem_raw + agents_bytes + per_warp * warp;
  WarpScratch ws;
  ws.cd = reinterpret_cast<double *>(wb);
  ws.sd = ws.cd + kCandCap;
  ws.cid = reinterpret_cast<int *>(ws.sd + kSelCap);
  ws.caux = ws.cid + kCandCap;
  ws.sid = ws.caux + kCandCap;
  ws.saux = ws.sid + kSelCap;
  ws.hc = reinterpret_cast<uint32_t *>(ws.saux + kSelCap);
  ws.row = reinterpret_cast<float *>(ws.hc + kBuckets);

  const int64_t a0 = T.a_off[w];
  const int A = (int)(T.a_off[w + 1] - a0);
  for (int i = threadIdx.x; i < A; i += blockDim.x) {
    const int64_t g = a0 + i;
    ax[i] = S.x[g];
    ay[i] = S.y[g];
    ah[i] = S.heading[g];
    av[i] = S.speed[g];
    al[i] = T.length[g];
    aw[i] = T.width[g];
    const uint16_t f = S.flags[g];
    avis[i] = (f & DS_F_PRESENT) && !(f & DS_F_REMOVED);
  }
  __syncthreads();

  const double radius = C.radius;
  const double reach = radius + 1e-6;   // culling slack; membership is decided exactly
  const int cap_a = C.max_agents_obs, cap_r = C.max_road_points_obs;
  const int road_off = 7 + 7 * cap_a;
  const int sel_w = cap_a + cap_r;
  const int nx = T.grid_nx[w], ny = T.grid_ny[w];
  const double gx0 = T.grid_x0[w], gy0 = T.grid_y0[w], cs = C.grid_cell;
  const int64_t cbase = T.grid_cell_off[w];
  const int64_t p0 = T.p_off[w];

  for (int r = warp; r < nrow; r += WARPS) {
    const int64_t orow = c0 + r;
    float *out = obs + orow * (int64_t)obs_width;
    const int64_t g = T.row_agent[orow];
    const int i = (int)(g - a0);
    const uint16_t f = S.flags[g];
    if (f & (DS_F_DONE | DS_F_REMOVED)) {
      // finished / removed rows are zero-filled (engine.py:502-512)
      for (int c = lane; c < obs_width; c += 32) out[c] = 0.0f;
      if (sel_idx)
        for (int c = lane; c < sel_w; c += 32) sel_idx[orow * sel_w + c] = -1;
      continue;
    }
    for (int c = lane; c < rp; c += 32) ws.row[c] = 0.0f;
    const double px = ax[i], py = ay[i], h = ah[i];
    const double ch = cos(h), sh = sin(h);
    __syncwarp();
    if (lane == 0) {
      // ego block (fp:228-238)
      const double gx = T.goal_x[g] - px, gy = T.goal_y[g] - py;
      ws.row[0] = (float)av[i];
      ws.row[1] = (float)al[i];
      ws.row[2] = (float)aw[i];
      ws.row[3] = (float)(gx * ch + gy * sh);
      ws.row[4] = (float)(gy * ch - gx * sh);
      ws.row[5] = (float)hypot(gx, gy);
      ws.row[6] = (f & DS_F_COLLIDED) ? 1.0f : 0.0f;
    }

    // ---- partners: visible, j != i, hypot <= radius, k nearest (fp:240-272)
    int n = 0;
    for (int j0 = 0; j0 < A; j0 += 32) {
      const int j = j0 + lane;
      bool ok = j < A && j != i && avis[j];
      double d = 0.0;
      if (ok) {
        d = hypot(ax[j] - px, ay[j] - py);
        ok = d <= radius;
      }
      n = warp_push(ws, n, ok, d, j, j, lane);
      if (n > kCandCap - 32) n = warp_topk(ws, n, cap_a, radius, lane);
    }
    const int ma = warp_topk(ws, n, cap_a, radius, lane);
    for (int m = lane; m < ma; m += 32) {
      const int j = ws.cid[m];
      const double dx = ax[j] - px, dy = ay[j] - py;
      float *slot = ws.row + 7 + 7 * m;
      slot[0] = (float)(dx * ch + dy * sh);
      slot[1] = (float)(dy * ch - dx * sh);
      slot[2] = (float)wrap(ah[j] - h);
      slot[3] = (float)(av[j] - av[i]);
      slot[4] = (float)al[j];
      slot[5] = (float)aw[j];
      slot[6] = 1.0f;
      if (sel_idx) sel_idx[orow * sel_w + m] = j;
    }
    if (sel_idx)
      for (int m = ma + lane; m < cap_a; m += 32) sel_idx[orow * sel_w + m] = -1;
    __syncwarp();

    // ---- road points within the radius, k nearest (fp:274-302)
    n = 0;
    if (cap_r > 0 && nx > 0 && ny > 0) {
      const double fy0 = (py - reach - gy0) / cs, fy1 = (py + reach - gy0) / cs;
      if (fy1 >= 0.0 && fy0 < (double)ny) {
        const int iy0 = clampi(floor(fy0), 0, ny - 1), iy1 = clampi(floor(fy1), 0, ny - 1);
        for (int iy = iy0; iy <= iy1; ++iy) {
          const double ylo = gy0 + iy * cs, yhi = ylo + cs;
          double dyb = 0.0;
          if (py < ylo) dyb = ylo - py;
          else if (py > yhi) dyb = py - yhi;
          if (dyb > reach) continue;
          const double half = sqrt(reach * reach - dyb * dyb) + 1e-6;
          const double fx0 = (px - half - gx0) / cs, fx1 = (px + half - gx0) / cs;
          if (fx1 < 0.0 || fx0 >= (double)nx) continue;
          const int ix0 = clampi(floor(fx0), 0, nx - 1), ix1 = clampi(floor(fx1), 0, nx - 1);
          const int64_t cell = cbase + (int64_t)iy * nx;
          const int sb = T.pt_cell_start[cell + ix0], se = T.pt_cell_start[cell + ix1 + 1];
          for (int s0 = sb; s0 < se; s0 += 32) {
            const int s = s0 + lane;
            bool ok = s < se;
            double d = 0.0;
            int id = 0;
            if (ok) {
              const double dx = T.gpt_x[s] - px, dy = T.gpt_y[s] - py;
              ok = fabs(dx) <= reach && fabs(dy) <= reach;
              if (ok) {
                d = hypot(dx, dy);
                ok = d <= radius;
                id = T.gpt_id[s];
              }
            }
            n = warp_push(ws, n, ok, d, id, s, lane);
            if (n > kCandCap - 32) n = warp_topk(ws, n, cap_r, radius, lane);
          }
        }
      }
    }
    const int mr = warp_topk(ws, n, cap_r, radius, lane);
    for (int m = lane; m < mr; m += 32) {
      const int s = ws.caux[m];
      const double dx = T.gpt_x[s] - px, dy = T.gpt_y[s] - py;
      float *slot = ws.row + road_off + 11 * m;
      slot[0] = (float)(dx * ch + dy * sh);
      slot[1] = (float)(dy * ch - dx * sh);
      slot[2] = (float)wrap(T.gpt_h[s] - h);
      slot[3 + T.gpt_kind[s]] = 1.0f;
      slot[10] = 1.0f;
      if (sel_idx) sel_idx[orow * sel_w + cap_a + m] = ws.cid[m];
    }
    if (sel_idx)
      for (int m = mr + lane; m < cap_r; m += 32) sel_idx[orow * sel_w + cap_a + m] = -1;
    __syncwarp();
    if (scale) {
      for (int c = lane; c < obs_width; c += 32) out[c] = ws.row[c] / scale[c];
    } else {
      for (int c = lane; c < obs_width; c += 32) out[c] = ws.row[c];
    }
    __syncwarp();
  }
  (void)p0;
}

constexpr int kObsWarps = 8;

cudaError_t configure_kernels(int max_dynamic_smem) {
  cudaError_t e = cudaFuncSetAttribute(obs_radial_kernel<kObsWarps>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       max_dynamic_smem);
  if (e != cudaSuccess) return e;
  return configure_step_kernels(max_dynamic_smem);
}

cudaError_t launch_observe(const ds_handle *h, const uint8_t *mask, float *obs,
                           const float *scale, int32_t *sel_idx, cudaStream_t s) {
  if (h->cfg.obs_mode == DS_OBS_RADIAL) {
    obs_radial_kernel<kObsWarps><<<h->tab.n_worlds, kObsWarps * 32, h->obs_smem, s>>>(
        h->tab, h->cfg, h->st, mask, obs, scale, sel_idx, h->obs_width);
    return cudaGetLastError();
  }
  return cudaErrorNotSupported;
}

}  // namespace ds
