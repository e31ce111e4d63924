// ds_step.cu -- the fused per-world step kernel and the reset kernel.
//
// One CTA per world, one thread per agent (blockDim = A_max rounded up to a
// warp).  A world is share-nothing (engine.py:4-7), so a CTA owns it for the
// whole step and the four phases of World.step (engine.py:357-498) are
// separated by __syncthreads only:
//   A  dynamics of live controlled agents + expert replay   (engine.py:378-418)
//   B  SAT agent-agent and slab agent-road-edge collisions   (engine.py:420-459)
//   C  goal reward, removal, collision behaviour, horizon    (engine.py:461-492)
//   D  outputs, episode record, optional VecDriveEnv auto-reset
// State is FP64 in HBM (SURVEY.md §7 "hard parts").  The broad phases only
// prune, the exact FP64 narrow phases decide (the reference's BVH likewise
// only prunes: its results are pinned equal to brute force,
// tests/test_acceptance.py:193-219): agent pairs by sweep and prune over a
// counting sort of x-bins with a float circumcircle test, road edges by the
// world's uniform grid with float AABB and separating-axis filters whose
// margins bound their rounding.
#include "ds_internal.cuh"

namespace ds {

constexpr int kStepBins = 64;   // x-bins of the agent-agent sweep
constexpr int kStepStride = 128;   // table stride of the <= 128-agent variant

struct StepShared {
  double *x, *y, *c, *s, *hl, *hw, *cr;
  uint8_t *elig;
  uint8_t *hit;    // agent-agent collision flags (each pair tested once)
  // circumcircle prefilter: float position relative to the world's grid
  // origin, circumradius padded by the float rounding bound (> 0: eligible)
  float4 *pre;
  // sweep-and-prune order: the eligible agents' ids (sord) and x-bins (skey,
  // as int), counting-sorted by bin
  float *skey;
  int *sord;
  int *bcnt, *bstart;   // x-bin counts / starts (+ total) of the sweep
};

__host__ __device__ inline int pow2_at_least(int n) {
  int p = 1;
  while (p < n) p <<= 1;
  return p;
}

__device__ __forceinline__ StepShared carve_step(void *base, int amax) {
  StepShared sh;
  double *d = reinterpret_cast<double *>(base);
  sh.x = d;
  sh.y = d + amax;
  sh.c = d + 2 * amax;
  sh.s = d + 3 * amax;
  sh.hl = d + 4 * amax;
  sh.hw = d + 5 * amax;
  sh.cr = d + 6 * amax;
  sh.elig = reinterpret_cast<uint8_t *>(d + 7 * amax);
  sh.hit = sh.elig + amax;
  sh.pre = reinterpret_cast<float4 *>(
      (reinterpret_cast<uintptr_t>(sh.hit + amax) + 15) & ~uintptr_t(15));
  sh.skey = reinterpret_cast<float *>(sh.pre + amax);
  sh.sord = reinterpret_cast<int *>(sh.skey + pow2_at_least(amax));
  sh.bcnt = sh.sord + pow2_at_least(amax);
  sh.bstart = sh.bcnt + kStepBins;
  return sh;
}

size_t step_smem_bytes(int max_agents) {
  if (max_agents <= kStepStride) max_agents = kStepStride;   // the <= 128-agent variant's stride
  return (size_t)max_agents * (7 * sizeof(double) + 2) + 16 + (size_t)max_agents * sizeof(float4) +
         (size_t)pow2_at_least(max_agents) * (sizeof(float) + sizeof(int)) +
         (2 * kStepBins + 1) * sizeof(int);
}

// SAT over the 4 box axes, _fastpath.sat_pairs (fp:29-53); (i, j) with i < j.
__device__ __forceinline__ bool sat_hit(const StepShared &sh, int i, int j) {
  const double dx = sh.x[j] - sh.x[i];
  const double dy = sh.y[j] - sh.y[i];
  const double ci = sh.c[i], si = sh.s[i], cj = sh.c[j], sj = sh.s[j];
  const double hli = sh.hl[i], hwi = sh.hw[i], hlj = sh.hl[j], hwj = sh.hw[j];
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    double ax, ay;
    if (m == 0) { ax = ci; ay = si; }
    else if (m == 1) { ax = -si; ay = ci; }
    else if (m == 2) { ax = cj; ay = sj; }
    else { ax = -sj; ay = cj; }
    const double dist = fabs(dx * ax + dy * ay);
    const double ra = hli * fabs(ci * ax + si * ay) + hwi * fabs(ci * ay - si * ax);
    const double rb = hlj * fabs(cj * ax + sj * ay) + hwj * fabs(cj * ay - sj * ax);
    if (dist > ra + rb) return false;
  }
  return true;
}

// Segment vs oriented box slab clip in the box frame, _fastpath.seg_box_hits
// (fp:55-90); boundary contact counts as a hit.
__device__ __forceinline__ bool seg_box_hit(double cx, double cy, double ck, double sk,
                                            double hl, double hw, double sax, double say,
                                            double sbx, double sby) {
  const double rax = sax - cx, ray = say - cy, rbx = sbx - cx, rby = sby - cy;
  const double pax = rax * ck + ray * sk;
  const double pay = -rax * sk + ray * ck;
  const double pbx = rbx * ck + rby * sk;
  const double pby = -rbx * sk + rby * ck;
  double t0 = 0.0, t1 = 1.0;
#pragma unroll
  for (int axis = 0; axis < 2; ++axis) {
    const double p0 = axis == 0 ? pax : pay;
    const double d = axis == 0 ? (pbx - pax) : (pby - pay);
    const double h = axis == 0 ? hl : hw;
    if (d == 0.0) {
      if (p0 < -h || p0 > h) return false;
    } else {
      double ta = (-h - p0) / d;
      double tb = (h - p0) / d;
      if (ta > tb) { const double tmp = ta; ta = tb; tb = tmp; }
      if (ta > t0) t0 = ta;
      if (tb < t1) t1 = tb;
      if (t0 > t1) return false;
    }
  }
  return true;
}

// float prefilter loads in flight per pass of the off-road scan
#ifndef DS_OFF_INFLIGHT
#define DS_OFF_INFLIGHT 2
#endif

// Clamp a floating cell coordinate to [lo, hi] before converting.
__device__ __forceinline__ int cell_of(double v, int lo, int hi) {
  double f = floor(v);
  if (f < (double)lo) return lo;
  if (f > (double)hi) return hi;
  return (int)f;
}

// Any road-edge segment of world w touching box (cx, cy, ck, sk, hl, hw)?
// The box's FP64 values are read from the shared tables (sh, agent i): the
// float filter loop holds only floats, the exact phase re-reads the rest.
__device__ bool offroad_query(const ds_tables &T, const ds_config &C, int w, const StepShared &sh,
                              int i) {
  const double cx = sh.x[i], cy = sh.y[i], ck = sh.c[i], sk = sh.s[i], hl = sh.hl[i], hw = sh.hw[i];
  const int nx = T.grid_nx[w], ny = T.grid_ny[w];
  const double x0 = T.grid_x0[w], y0 = T.grid_y0[w], cs = C.grid_cell;
  const int64_t cbase = T.grid_cell_off[w];
  // AABB of the box (agent_aabbs_core fp:304-317) with 1.1 cm slack: the grid
  // only has to produce a superset, the slab test below decides.
  const double rx = hl * fabs(ck) + hw * fabs(sk) + 0.011;
  const double ry = hl * fabs(sk) + hw * fabs(ck) + 0.011;
  // float prefilter on the grid-relative copies (16 B per segment): widened
  // by a bound on its rounding, it only skips segments the FP64 test skips
  const float fcx = (float)(cx - x0), fcy = (float)(cy - y0);
  const float fm = 1e-3f + 2.4e-7f * (fabsf(fcx) + fabsf(fcy) + (float)(rx + ry));
  const float frx = (float)rx + fm, fry = (float)ry + fm;
  const float4 *erel = reinterpret_cast<const float4 *>(T.eseg_rel);
  // float separating-axis filter (box axes and the segment normal) on the
  // same copies: a separation by more than the margin (four times a bound on
  // the float error of the box-relative endpoints and their projections)
  // proves the exact slab test misses, so the FP64 record is not fetched
  const float cf = (float)ck, sf = (float)sk, hlf = (float)hl, hwf = (float)hw;
  const float e_c = 1.2e-7f * (fabsf(fcx) + fabsf(fcy)) + 1e-6f;
  const double gx0 = (cx - rx - x0) / cs, gx1 = (cx + rx - x0) / cs;
  const double gy0 = (cy - ry - y0) / cs, gy1 = (cy + ry - y0) / cs;
  if (gx1 < 0.0 || gy1 < 0.0 || gx0 >= (double)nx || gy0 >= (double)ny) return false;
  const int ix0 = cell_of(gx0, 0, nx - 1), ix1 = cell_of(gx1, 0, nx - 1);
  const int iy0 = cell_of(gy0, 0, ny - 1), iy1 = cell_of(gy1, 0, ny - 1);
  for (int iy = iy0; iy <= iy1; ++iy) {
    // the cells ix0..ix1 of one grid row are consecutive bins: one range
    const int64_t crow = cbase + (int64_t)iy * nx;
    const int b = T.eseg_cell_start[crow + ix0], e = T.eseg_cell_start[crow + ix1 + 1];
    for (int k0 = b; k0 < e; k0 += DS_OFF_INFLIGHT) {
      // four float prefilter loads in flight, then the tests
      float4 q[DS_OFF_INFLIGHT];
#pragma unroll
      for (int v = 0; v < DS_OFF_INFLIGHT; ++v)
        q[v] = k0 + v < e ? erel[k0 + v] : make_float4(INFINITY, INFINITY, INFINITY, INFINITY);
#pragma unroll
      for (int v = 0; v < DS_OFF_INFLIGHT; ++v) {
        if (fmaxf(q[v].x, q[v].z) < fcx - frx || fminf(q[v].x, q[v].z) > fcx + frx ||
            fmaxf(q[v].y, q[v].w) < fcy - fry || fminf(q[v].y, q[v].w) > fcy + fry)
          continue;
        {
          const float pax = q[v].x - fcx, pay = q[v].y - fcy, pbx = q[v].z - fcx, pby = q[v].w - fcy;
          // |float error| of the box-relative endpoints <= e_in (input
          // roundings of both copies and of the subtraction, long segments
          // included); four times that plus 0.1 mm on every axis
          const float e_in =
              e_c + 1.2e-7f * (fabsf(pax) + fabsf(pay) + fabsf(pbx) + fabsf(pby));
          const float mg = 4.0f * e_in + 1e-4f;
          const float ua = pax * cf + pay * sf, ub = pbx * cf + pby * sf;
          if (fminf(ua, ub) > hlf + mg || fmaxf(ua, ub) < -hlf - mg) continue;
          const float va = pay * cf - pax * sf, vb = pby * cf - pbx * sf;
          if (fminf(va, vb) > hwf + mg || fmaxf(va, vb) < -hwf - mg) continue;
          const float nxs = pay - pby, nys = pbx - pax;   // segment normal (unnormalised)
          const float dn = fabsf(pax * nxs + pay * nys);
          const float rn = hlf * fabsf(cf * nxs + sf * nys) + hwf * fabsf(cf * nys - sf * nxs);
          const float mn = mg * (fabsf(nxs) + fabsf(nys)) +
                           8.0f * e_in * (fabsf(pax) + fabsf(pay) + hlf + hwf);
          if (dn > rn + mn) continue;
        }
        // FP64 endpoints: one 32-B record (one sector) per entry
        const double2 *er = reinterpret_cast<const double2 *>(T.eseg_rec) + 2 * (int64_t)(k0 + v);
        const double2 e0 = er[0], e1 = er[1];
        const double ax = e0.x, ay = e0.y, bx = e1.x, by = e1.y;
        // the box from shared memory again (the same values as above; the
        // empty asm keeps the compiler from holding the first reads live)
        asm volatile("" ::: "memory");
        const double qx = sh.x[i], qy = sh.y[i], qk = sh.c[i], qs = sh.s[i];
        const double ql = sh.hl[i], qw = sh.hw[i];
        const double qrx = ql * fabs(qk) + qw * fabs(qs) + 0.011;
        const double qry = ql * fabs(qs) + qw * fabs(qk) + 0.011;
        // segment AABB vs box AABB (with slack): a superset prefilter
        if (fmax(ax, bx) < qx - qrx || fmin(ax, bx) > qx + qrx || fmax(ay, by) < qy - qry ||
            fmin(ay, by) > qy + qry)
          continue;
        if (seg_box_hit(qx, qy, qk, qs, ql, qw, ax, ay, bx, by)) return true;
      }
    }
  }
  return false;
}

// Reset one agent of world w to t = 0 (World.reset, engine.py:318-340).
__device__ __forceinline__ void reset_agent(const ds_tables &T, const ds_state &S, int64_t g,
                                            int64_t r0) {
  S.x[g] = T.rep_x[r0];
  S.y[g] = T.rep_y[r0];
  S.heading[g] = T.rep_h[r0];
  S.speed[g] = T.rep_v[r0];
  S.head_angle[g] = 0.0;
  const bool present = T.rep_present[r0] || (T.sflags[g] & DS_SF_CONTROLLED);
  S.flags[g] = present ? DS_F_PRESENT : 0;
}

// MAXT: the launch's thread bound (worlds of <= 256 agents get the 256
// variant: up to 255 registers, no spills of the FP64 state)
template <int MAXT, int MINB>
__global__ void __launch_bounds__(MAXT, MINB) step_kernel(ds_tables T, ds_config C, ds_state S,
                                                    ds_step_args a, const WorldStrides U) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int w = blockIdx.x;
  const int tid = threadIdx.x;
  const int64_t a0 = U.a0(T, w);
  const int A = (int)(U.a1(T, w) - a0);
  const int64_t r_w = U.r0(T, w);
  const int Tw = T.num_steps[w];
  const bool act_here = tid < A;
  const int64_t g = a0 + tid;
  const uint8_t sf = act_here ? T.sflags[g] : 0;
  const bool ctrl = sf & DS_SF_CONTROLLED;
  const int row = (act_here && ctrl) ? T.ctrl_row[g] : -1;
  const int n_rows = (int)(U.c1(T, w) - U.c0(T, w));

  if (S.episode_over[w]) {
    // Early return of World.step (engine.py:370-373): zero rewards/info,
    // dones = done[ids]; observation rows are all done -> zero.
    if (row >= 0) {
      a.rewards[row] = 0.0f;
      a.dones[row] = (S.flags[g] & DS_F_DONE) ? 1 : 0;
      a.info[row] = 0;
      a.info[T.n_rows + row] = 0;
      a.info[2 * T.n_rows + row] = 0;
    }
    if (a.auto_reset) {
      if (act_here) reset_agent(T, S, g, r_w + tid);
      if (row >= 0) a.rewards[row] = 0.0f;
      if (tid == 0) {
        S.t[w] = 0;
        S.episode_over[w] = 0;
      }
    }
    return;
  }

  // the <= 128-agent variant lays its tables out at the compile-time stride
  // 128 (every array at a constant offset; step_smem_bytes sizes it so)
  StepShared sh = carve_step(smem_raw, MAXT <= kStepStride ? kStepStride : T.max_agents);
  const int t = S.t[w];
  const int t_next = min(t + 1, Tw - 1);
  const double dt = T.dt[w];
  const int64_t rn = r_w + (int64_t)t_next * A + tid;   // replay cell at t_next

  uint16_t f = 0;
  double x = 0, y = 0, h = 0, v = 0;
  // statics, one 32-B record: half-extents and goal (length = 2 half_l and
  // the circumradius hypot(half_l, half_w) are exact functions of them)
  double2 st_hlw = make_double2(0.0, 0.0), st_goal = make_double2(0.0, 0.0);
  if (act_here) {
    const double2 *ar = reinterpret_cast<const double2 *>(T.agent_rec) + 2 * g;
    st_hlw = ar[0];
    st_goal = ar[1];
  }
  if (act_here) {
    f = S.flags[g];
    // (1) remove agents flagged last step (engine.py:379-380)
    if (f & DS_F_PENDING) f |= DS_F_REMOVED;
    f &= ~(DS_F_PENDING | DS_F_COLLIDED | DS_F_OFFROAD);
    x = S.x[g];
    y = S.y[g];
    h = S.heading[g];
    v = S.speed[g];
    const bool live = ctrl && !(f & (DS_F_REMOVED | DS_F_DONE));
    if (!a.replay && live) {
      // Action row (engine.py:392: float64 cast of the caller's values).
      double a0v = 0.0, a1v = 0.0, a2v = 0.0, a3v = 0.0;
      bool bad_action = false;
      if (a.actions) {
        const float *ar = a.actions + (int64_t)row * a.act_dim;
        a0v = ar[0];
        a1v = ar[1];
        if (a.act_dim > 2) a2v = ar[2];
        if (a.act_dim > 3) a3v = ar[3];
      } else {
        // VecDriveEnv.to_continuous (env.py:111-116): accel[i // n_steer],
        // steer[i % n_steer] with Python floor division and numpy indexing
        // (a negative accel index counts from the end; outside
        // [-n_accel, n_accel) numpy raises IndexError: flagged in the
        // status word, the agent's dynamics skipped, never clamped)
        const int idx = a.action_idx[row];
        int ai = idx >= 0 ? idx / a.n_steer : -((-idx + a.n_steer - 1) / a.n_steer);
        const int si = idx - ai * a.n_steer;
        if (ai < -a.n_accel || ai >= a.n_accel) {
          if (S.status) atomicOr(S.status, DS_STATUS_BAD_ACTION_INDEX);
          bad_action = true;
        } else {
          if (ai < 0) ai += a.n_accel;
          a0v = a.grid_accel[ai];
          a1v = a.grid_steer[si];
        }
      }
      const double L = 2.0 * st_hlw.x;   // == length exactly (half_l = 0.5 length)
      if (bad_action) {
        // pose held (the reference would have raised before stepping)
      } else if (C.dynamics == DS_DYN_CLASSIC) {
        // classic_core (fp:319-333), left-to-right, no FMA.
        const double acc = clip(a0v, C.accel_lo, C.accel_hi);
        const double delta = clip(a1v, C.steer_lo, C.steer_hi);
        const double v_bar = clip(v + 0.5 * acc * dt, -C.v_max, C.v_max);
        const double tdelta = tan(delta);
        const double beta = atan(0.5 * tdelta);
        const double ang = h + beta;
        x += v_bar * cos(ang) * dt;
        y += v_bar * sin(ang) * dt;
        h = wrap(h + v_bar * cos(beta) * tdelta / L * dt);
        v = clip(v + acc * dt, -C.v_max, C.v_max);
      } else if (C.dynamics == DS_DYN_INVERTIBLE) {
        // invertible_core (fp:335-342); actions are not clipped.
        const double d = v * dt + 0.5 * a0v * dt * dt;
        x += d * cos(h);
        y += d * sin(h);
        h = wrap(h + a1v * d);
        v = clip(v + a0v * dt, -C.v_max, C.v_max);
      } else {
        // delta_local: ego-frame displacement (dx, dy) and yaw
        // increment, clipped to SimConfig.delta_bounds; speed = |d| / dt.
        const double ddx = clip(a0v, C.delta_lo[0], C.delta_hi[0]);
        const double ddy = clip(a1v, C.delta_lo[1], C.delta_hi[1]);
        const double dyaw = clip(a2v, C.delta_lo[2], C.delta_hi[2]);
        const double ch = cos(h), shh = sin(h);
        x += ddx * ch - ddy * shh;
        y += ddx * shh + ddy * ch;
        h = wrap(h + dyaw);
        v = clip(hypot(ddx, ddy) / dt, -C.v_max, C.v_max);
      }
      // Head rotation (engine.py:408-411), column 2 (column 3 for delta_local).
      const int head_col = C.dynamics == DS_DYN_DELTA_LOCAL ? 3 : 2;
      if (a.actions && a.act_dim > head_col) {
        const double hr = head_col == 2 ? a2v : a3v;
        S.head_angle[g] = clip(S.head_angle[g] + hr * dt, -0.5 * kPi, 0.5 * kPi);
      }
    }
    // Expert replay (engine.py:383-385, 413-418).
    const bool replay_i = (sf & DS_SF_REPLAY_ONLY) || (a.replay && ctrl);
    if (replay_i && (sf & DS_SF_INSTANTIABLE) && !(f & DS_F_REMOVED)) {
      x = T.rep_x[rn];
      y = T.rep_y[rn];
      h = T.rep_h[rn];
      v = T.rep_v[rn];
      if (T.rep_present[rn]) f |= DS_F_PRESENT; else f &= ~DS_F_PRESENT;
    }
    S.x[g] = x;
    S.y[g] = y;
    S.heading[g] = h;
    S.speed[g] = v;
    // (2-3) collision inputs (engine.py:424-428)
    sh.x[tid] = x;
    sh.y[tid] = y;
    sh.c[tid] = cos(h);
    sh.s[tid] = sin(h);
    // np.hypot(half_l, half_w) (engine.py:189): the glibc-exact port
    const double cr = hypot(st_hlw.x, st_hlw.y);
    sh.hl[tid] = st_hlw.x;
    sh.hw[tid] = st_hlw.y;
    sh.cr[tid] = cr;
    const bool elig = (f & DS_F_PRESENT) && !(f & DS_F_REMOVED) &&
                      ((ctrl && !(f & DS_F_DONE)) || T.rep_valid[rn]);
    sh.elig[tid] = elig;
    // |fx - (x - x0)| <= 2^-24 |x - x0|: pad the radius by 2.4e-7 (|fx| + |fy|)
    // + 1 mm, so that float distances > the padded sum prove disjoint circles
    const float fx = (float)(x - T.grid_x0[w]), fy = (float)(y - T.grid_y0[w]);
    const float pr = (float)cr * (1.0f + 1e-6f) + 1e-3f +
                     2.4e-7f * (fabsf(fx) + fabsf(fy));
    sh.pre[tid] = make_float4(fx, fy, pr, elig ? 1.0f : 0.0f);
    sh.hit[tid] = 0;
  }
  for (int b0 = tid; b0 < kStepBins; b0 += blockDim.x) sh.bcnt[b0] = 0;
  __syncthreads();

  bool collided = false, offroad = false;
  // Agent-agent pairs by sweep and prune over x-bins: the eligible agents
  // are counting-sorted by the bin of their padded circle's left edge (bins
  // are monotone in x, so every agent after p in this order starts at or
  // beyond p's bin), then each position scans forward while the next
  // agent's bin is <= the bin of its own right edge -- every pair whose
  // circles can overlap is tested exactly once (within a bin, by the earlier
  // position), and both ends are flagged (SAT runs on (min, max) id, so
  // either end computes the same bits).  Four barriers instead of a bitonic
  // network's log^2 stages.
  const float ext = (float)T.grid_nx[w] * (float)C.grid_cell;
  const float inv_bw = ext > 0.0f ? (float)kStepBins / ext : 0.0f;
  auto bin_of = [&](float xr) {
    return (int)fminf(fmaxf(floorf(xr * inv_bw), 0.0f), (float)(kStepBins - 1));
  };
  int my_bin = -1, my_pos = 0;
  if (act_here) {
    const float4 pe = sh.pre[tid];
    if (pe.w != 0.0f) {
      my_bin = bin_of(pe.x - pe.z);
      my_pos = atomicAdd(&sh.bcnt[my_bin], 1);
    }
  }
  __syncthreads();
  if (tid < 32) {
    // exclusive scan of the bin counts (one warp)
    int carry = 0;
    for (int b0 = 0; b0 < kStepBins; b0 += 32) {
      const int c = sh.bcnt[b0 + tid];
      int incl = c;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int up = __shfl_up_sync(0xffffffffu, incl, off);
        if (tid >= off) incl += up;
      }
      sh.bstart[b0 + tid] = carry + incl - c;
      carry += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (tid == 0) sh.bstart[kStepBins] = carry;
  }
  __syncthreads();
  if (my_bin >= 0) {
    const int slot = sh.bstart[my_bin] + my_pos;
    sh.sord[slot] = tid;
    reinterpret_cast<int *>(sh.skey)[slot] = my_bin;
  }
  __syncthreads();
  const int n_elig = sh.bstart[kStepBins];
  const int *sbin = reinterpret_cast<const int *>(sh.skey);
  for (int p = tid; p < n_elig; p += blockDim.x) {
    const int i = sh.sord[p];
    const float4 pi = sh.pre[i];
    const int rbin = bin_of(pi.x + pi.z + 1e-4f * (1.0f + fabsf(pi.x)));
    bool hit_any = false;
    for (int q = p + 1; q < n_elig; ++q) {
      if (sbin[q] > rbin) break;            // this and all later circles start beyond i's
      const int j = sh.sord[q];
      // boxes lie inside their circumcircles: disjoint circles cannot collide
      // (float superset test on padded radii; SAT below decides exactly)
      const float4 pj = sh.pre[j];
      const float dx = pj.x - pi.x, dy = pj.y - pi.y, rr = pi.z + pj.z;
      if (fmaf(dx, dx, dy * dy) > rr * rr * (1.0f + 1e-5f)) continue;
      if (j > i ? sat_hit(sh, i, j) : sat_hit(sh, j, i)) {
        hit_any = true;
        sh.hit[j] = 1;
      }
    }
    if (hit_any) sh.hit[i] = 1;
  }
  __syncthreads();
  if (act_here && sh.elig[tid]) {
    collided = sh.hit[tid] != 0;
    if (!(sf & DS_SF_PEDESTRIAN))
      offroad = offroad_query(T, C, w, sh, tid);
  }
  if (collided) f |= DS_F_COLLIDED;
  if (offroad) f |= DS_F_OFFROAD;

  // (4) goal rewards, then terminations (engine.py:461-486).
  bool at_goal = false, live = false;
  if (n_rows > 0 && act_here) {
    live = ctrl && !(f & (DS_F_REMOVED | DS_F_DONE));
    if (live) {
      const double dgx = x - st_goal.x;
      const double dgy = y - st_goal.y;
      at_goal = hypot(dgx, dgy) <= C.goal_tolerance;
    }
    if (at_goal) f |= DS_F_GOAL_REACHED | DS_F_GOAL_EVER | DS_F_PENDING | DS_F_DONE;
    if (collided && live) f |= DS_F_COLL_EVER;
    if (offroad && live) f |= DS_F_OFF_EVER;
    if (C.collision_behavior == DS_COLL_REMOVE_AGENT && live && (collided || offroad))
      f |= DS_F_PENDING | DS_F_DONE;
  }
  // the CTA-wide OR only where it decides something (end_episode): other
  // behaviours let finished warps leave without waiting for the off-road
  // queries of the rest
  bool over = false;
  if (C.collision_behavior == DS_COLL_END_EPISODE)
    over = __syncthreads_or(live && (collided || offroad)) != 0;
  const int t1 = t + 1;
  if (t1 >= Tw) over = true;
  if (over && ctrl) f |= DS_F_DONE;

  if (row >= 0) {
    a.rewards[row] = at_goal ? 1.0f : 0.0f;
    a.dones[row] = (f & DS_F_DONE) ? 1 : 0;
    a.info[row] = at_goal;
    a.info[T.n_rows + row] = collided && live;
    a.info[2 * T.n_rows + row] = offroad && live;
  }
  if (act_here) S.flags[g] = f;

  if (over) {
    // EpisodeInfo at the episode's end (engine.py:521-528, 646-647).
    const int n_goal = __syncthreads_count(ctrl && (f & DS_F_GOAL_EVER));
    const int n_coll = __syncthreads_count(ctrl && (f & DS_F_COLL_EVER));
    const int n_off = __syncthreads_count(ctrl && (f & DS_F_OFF_EVER));
    if (tid == 0 && S.ring) {
      const uint32_t pos = atomicAdd(S.ring_head, 1u);
      if (pos < (uint32_t)S.ring_cap) {
        int32_t *rec = S.ring + (int64_t)pos * 6;
        rec[0] = a.serial;
        rec[1] = w;
        rec[2] = n_rows;
        rec[3] = n_goal;
        rec[4] = n_coll;
        rec[5] = n_off;
      }
    }
    if (a.auto_reset) {
      // VecDriveEnv.step auto-reset (env.py:105-107): World.reset of the
      // finished world; SimBatch.reset zeroes the rewards buffer rows the env
      // returns (engine.py:660), dones/infos were copied before.
      __syncthreads();
      if (act_here) reset_agent(T, S, g, r_w + tid);
      if (row >= 0) a.rewards[row] = 0.0f;
      if (tid == 0) {
        S.t[w] = 0;
        S.episode_over[w] = 0;
      }
      return;
    }
  }
  if (tid == 0) {
    S.t[w] = t1;
    S.episode_over[w] = over ? 1 : 0;
  }
}

__global__ void __launch_bounds__(1024) reset_kernel(ds_tables T, ds_state S, const uint8_t *mask,
                                                     float *rewards, uint8_t *dones) {
  const int w = blockIdx.x;
  if (mask && !mask[w]) return;
  const int64_t a0 = T.a_off[w];
  const int A = (int)(T.a_off[w + 1] - a0);
  for (int i = threadIdx.x; i < A; i += blockDim.x) {
    const int64_t g = a0 + i;
    reset_agent(T, S, g, T.r_off[w] + i);
    if (T.sflags[g] & DS_SF_CONTROLLED) {
      const int row = T.ctrl_row[g];
      if (rewards) rewards[row] = 0.0f;
      if (dones) dones[row] = 0;
    }
  }
  if (threadIdx.x == 0) {
    S.t[w] = 0;
    S.episode_over[w] = 0;
  }
}

// goal_seek_actions (engine.py:559-574): proportional steer-to-goal with the
// speed capped by the distance, one thread per controlled row, FP64 in the
// reference's operation order (distance: the glibc hypot port; err =
// floor-mod(atan2(dy, dx) - heading + pi, 2 pi) - pi, WITHOUT wrap()'s
// r <= -pi correction, as np.mod there).  Rows of done / removed agents get
// the same formula (the reference computes all controlled rows; the step
// ignores them).  Output: float32 [rows, 2] (accel, steer), the action format
// ds_step consumes.
__global__ void goal_seek_kernel(ds_tables T, ds_config C, ds_state S, float *out) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= T.n_rows) return;
  const int64_t g = T.row_agent[r];
  const double dx = T.goal_x[g] - S.x[g];
  const double dy = T.goal_y[g] - S.y[g];
  const double dist = hypot(dx, dy);
  const double err = floor_mod_2pi(atan2(dy, dx) - S.heading[g] + kPi) - kPi;
  const double steer = fmin(fmax(2.0 * err, C.steer_lo), C.steer_hi);
  const double target_v = fmin(0.8 * dist + 0.5, 15.0);
  const double accel = fmin(fmax(2.0 * (target_v - S.speed[g]), C.accel_lo), C.accel_hi);
  out[2 * (int64_t)r] = (float)accel;
  out[2 * (int64_t)r + 1] = (float)steer;
}

cudaError_t launch_goal_seek(const ds_handle *h, float *out, cudaStream_t s) {
  const int n = h->tab.n_rows;
  if (n <= 0) return cudaSuccess;
  goal_seek_kernel<<<(n + 127) / 128, 128, 0, s>>>(h->tab, h->cfg, h->st, out);
  return cudaGetLastError();
}

#ifndef DS_STEP_MINB
#define DS_STEP_MINB 8   // CTAs (x 4 warps) per SM of the <= 128-agent variant
#endif

cudaError_t configure_step_kernels(int max_dynamic_smem) {
  const void *ks[] = {(const void *)step_kernel<128, DS_STEP_MINB>, (const void *)step_kernel<256, 1>,
                      (const void *)step_kernel<1024, 1>};
  for (const void *k : ks) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         max_dynamic_smem);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t launch_step(const ds_handle *h, const ds_step_args *a, cudaStream_t s) {
  if (h->step_threads <= 128)   // 8 CTAs (32 warps) per SM at <= 64 registers
    step_kernel<128, DS_STEP_MINB><<<h->tab.n_worlds, h->step_threads, h->step_smem, s>>>(h->tab, h->cfg,
                                                                              h->st, *a, world_strides(h));
  else if (h->step_threads <= 256)
    step_kernel<256, 1><<<h->tab.n_worlds, h->step_threads, h->step_smem, s>>>(h->tab, h->cfg,
                                                                              h->st, *a, world_strides(h));
  else
    step_kernel<1024, 1><<<h->tab.n_worlds, h->step_threads, h->step_smem, s>>>(h->tab, h->cfg,
                                                                               h->st, *a, world_strides(h));
  return cudaGetLastError();
}

cudaError_t launch_reset(const ds_handle *h, const uint8_t *mask, float *rewards, uint8_t *dones,
                         cudaStream_t s) {
  int threads = h->step_threads;
  reset_kernel<<<h->tab.n_worlds, threads, 0, s>>>(h->tab, h->st, mask, rewards, dones);
  return cudaGetLastError();
}

}  // namespace ds
