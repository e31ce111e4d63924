/*
 * drivesim_oracle.c -- TEST INFRASTRUCTURE ONLY (the checker, never the product).
 *
 * A plain-C, FP64, glibc-libm restatement of the reference's batched world
 * step (/root/reference/pkg/src/drivesim), used by tests/ as the parity oracle
 * and by bench.py's cpu_baseline / --impl reference legs.  The product path
 * (paper_2408_01584_b200) never links, imports or calls this file.
 *
 * Followed line by line:
 *   World.step            engine.py:357-498   -> or_step_world()
 *   World.reset/observe   engine.py:318-340, 514-519
 *   classic_core          _fastpath.py:319-333, invertible_core 335-342
 *   _wrap                 _fastpath.py:206-212
 *   sat_pairs             _fastpath.py:29-53  (candidates: all eligible pairs,
 *                         equal to the BVH path, tests/test_acceptance.py:193-219)
 *   seg_box_hits          _fastpath.py:55-90  (candidates: edge segments whose
 *                         AABB overlaps the agent AABB with AABB_MARGIN, the
 *                         set Bvh.query_aabbs_arr returns, broadphase.py:247-276)
 *   radial_fill_core      _fastpath.py:214-302 (linear scan + insertion top-k)
 *   fill_lidar            observation.py:223-280 with raycast_obbs_arr
 *                         geometry.py:399-424 and raycast_segments_arr 380-396
 *                         (an exact distance tie between a road edge and another
 *                         kind goes to the edge; the reference breaks it in BVH
 *                         order).
 *   delta_local dynamics  (not in the reference; DESIGN.md definition)
 *
 * Compiled with -O2 -ffp-contract=off (no FMA contraction, like numba's
 * default) and linked against glibc libm, which is what numba's math.* and
 * numpy's float64 ufuncs resolve to on this image (tests/test_host_math.py).
 * Pinned against the real reference by tests/golden/ (make_golden.py).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define F_PRESENT 0x001
#define F_REMOVED 0x002
#define F_PENDING 0x004
#define F_GOAL_REACHED 0x008
#define F_COLLIDED 0x010
#define F_OFFROAD 0x020
#define F_GOAL_EVER 0x040
#define F_COLL_EVER 0x080
#define F_OFF_EVER 0x100
#define F_DONE 0x200
#define SF_CONTROLLED 1
#define SF_INSTANTIABLE 2
#define SF_REPLAY_ONLY 4
#define SF_PEDESTRIAN 8

typedef struct or_tables {
  int32_t n_worlds, n_agents, n_rows, reserved;
  const int64_t *a_off, *c_off, *r_off, *p_off, *s_off;
  const int32_t *num_steps;
  const double *dt;
  const int8_t *kind;
  const double *length, *width, *half_l, *half_w, *circumradius, *goal_x, *goal_y;
  const uint8_t *sflags;
  const int32_t *ctrl_row, *row_agent;
  const double *rep_x, *rep_y, *rep_h, *rep_v;
  const uint8_t *rep_valid, *rep_present;
  const double *pt_x, *pt_y, *pt_h;
  const int8_t *pt_kind;
  const double *seg_ax, *seg_ay, *seg_bx, *seg_by;
  const int8_t *seg_kind;
} or_tables;

typedef struct or_config {
  int32_t dynamics, collision_behavior, obs_mode, n_rays;
  int32_t max_agents_obs, max_road_points_obs, obs_width, reserved;
  double radius, fov, max_range, goal_tolerance;
  double accel_lo, accel_hi, steer_lo, steer_hi, v_max;
  double delta_lo[3], delta_hi[3];
} or_config;

typedef struct or_state {
  double *x, *y, *heading, *speed, *head_angle;
  uint16_t *flags;
  int32_t *t;
  uint8_t *episode_over;
} or_state;

static const double PI = 3.141592653589793;
static const double TWO_PI = 6.283185307179586;
static const double AABB_MARGIN = 0.01; /* engine.py:28 */
static const int ROAD_EDGE = 0;

static inline double wrap(double theta) {
  double r = fmod(theta + PI, TWO_PI);
  if (r != 0.0) {
    if (r < 0.0) r += TWO_PI;
  } else {
    r = 0.0;
  }
  r = r - PI;
  if (r <= -PI) r += TWO_PI;
  return r;
}

static inline double clip(double v, double lo, double hi) {
  double m = (lo > v) ? lo : v;
  return (m > hi) ? hi : m;
}

static int sat_hit(const double *x, const double *y, const double *c, const double *s,
                   const double *hl, const double *hw, int i, int j) {
  double dx = x[j] - x[i], dy = y[j] - y[i];
  double ci = c[i], si = s[i], cj = c[j], sj = s[j];
  for (int m = 0; m < 4; ++m) {
    double ax, ay;
    if (m == 0) { ax = ci; ay = si; }
    else if (m == 1) { ax = -si; ay = ci; }
    else if (m == 2) { ax = cj; ay = sj; }
    else { ax = -sj; ay = cj; }
    double dist = fabs(dx * ax + dy * ay);
    double ra = hl[i] * fabs(ci * ax + si * ay) + hw[i] * fabs(ci * ay - si * ax);
    double rb = hl[j] * fabs(cj * ax + sj * ay) + hw[j] * fabs(cj * ay - sj * ax);
    if (dist > ra + rb) return 0;
  }
  return 1;
}

static int seg_box_hit(double cx, double cy, double ck, double sk, double hl, double hw,
                       double sax, double say, double sbx, double sby) {
  double rax = sax - cx, ray = say - cy, rbx = sbx - cx, rby = sby - cy;
  double pax = rax * ck + ray * sk;
  double pay = -rax * sk + ray * ck;
  double pbx = rbx * ck + rby * sk;
  double pby = -rbx * sk + rby * ck;
  double t0 = 0.0, t1 = 1.0;
  for (int axis = 0; axis < 2; ++axis) {
    double p0 = axis == 0 ? pax : pay;
    double d = axis == 0 ? pbx - pax : pby - pay;
    double h = axis == 0 ? hl : hw;
    if (d == 0.0) {
      if (p0 < -h || p0 > h) return 0;
    } else {
      double ta = (-h - p0) / d, tb = (h - p0) / d;
      if (ta > tb) { double tmp = ta; ta = tb; tb = tmp; }
      if (ta > t0) t0 = ta;
      if (tb < t1) t1 = tb;
      if (t0 > t1) return 0;
    }
  }
  return 1;
}

/* ----- observations ------------------------------------------------------ */

/* radial_fill_core (fp:214-302) for one agent i of world w into out[width]. */
static void radial_row(const or_tables *T, const or_config *C, const or_state *S, int w, int i,
                       double *out, int32_t *sel, double *best_d, int64_t *best_j) {
  const int64_t a0 = T->a_off[w];
  const int n = (int)(T->a_off[w + 1] - a0);
  const int64_t p0 = T->p_off[w];
  const int n_pts = (int)(T->p_off[w + 1] - p0);
  const int cap_a = C->max_agents_obs, cap_r = C->max_road_points_obs;
  const int road_off = 7 + cap_a * 7;
  const double radius = C->radius;
  const int64_t g = a0 + i;
  for (int k = 0; k < C->obs_width; ++k) out[k] = 0.0;
  double px = S->x[g], py = S->y[g], h = S->heading[g];
  double ch = cos(h), sh = sin(h);
  double gx = T->goal_x[g] - px, gy = T->goal_y[g] - py;
  out[0] = S->speed[g];
  out[1] = T->length[g];
  out[2] = T->width[g];
  out[3] = gx * ch + gy * sh;
  out[4] = gy * ch - gx * sh;
  out[5] = hypot(gx, gy);
  out[6] = (S->flags[g] & F_COLLIDED) ? 1.0 : 0.0;

  int cnt = 0;
  for (int j = 0; j < n; ++j) {
    uint16_t fj = S->flags[a0 + j];
    if (j == i || !((fj & F_PRESENT) && !(fj & F_REMOVED))) continue;
    double d = hypot(S->x[a0 + j] - px, S->y[a0 + j] - py);
    if (d > radius) continue;
    int m;
    if (cnt < cap_a) { m = cnt; cnt++; }
    else if (cap_a > 0 && d < best_d[cap_a - 1]) m = cap_a - 1;
    else continue;
    while (m > 0 && best_d[m - 1] > d) {
      best_d[m] = best_d[m - 1];
      best_j[m] = best_j[m - 1];
      m--;
    }
    best_d[m] = d;
    best_j[m] = j;
  }
  for (int m = 0; m < cnt; ++m) {
    int64_t j = a0 + best_j[m];
    int base = 7 + m * 7;
    double dx = S->x[j] - px, dy = S->y[j] - py;
    out[base + 0] = dx * ch + dy * sh;
    out[base + 1] = dy * ch - dx * sh;
    out[base + 2] = wrap(S->heading[j] - h);
    out[base + 3] = S->speed[j] - S->speed[g];
    out[base + 4] = T->length[j];
    out[base + 5] = T->width[j];
    out[base + 6] = 1.0;
  }
  if (sel) {
    for (int m = 0; m < cap_a; ++m) sel[m] = m < cnt ? (int32_t)best_j[m] : -1;
  }

  cnt = 0;
  for (int j = 0; j < n_pts; ++j) {
    double d = hypot(T->pt_x[p0 + j] - px, T->pt_y[p0 + j] - py);
    if (d > radius) continue;
    int m;
    if (cnt < cap_r) { m = cnt; cnt++; }
    else if (cap_r > 0 && d < best_d[cap_r - 1]) m = cap_r - 1;
    else continue;
    while (m > 0 && best_d[m - 1] > d) {
      best_d[m] = best_d[m - 1];
      best_j[m] = best_j[m - 1];
      m--;
    }
    best_d[m] = d;
    best_j[m] = j;
  }
  for (int m = 0; m < cnt; ++m) {
    int64_t j = p0 + best_j[m];
    int base = road_off + m * 11;
    double dx = T->pt_x[j] - px, dy = T->pt_y[j] - py;
    out[base + 0] = dx * ch + dy * sh;
    out[base + 1] = dy * ch - dx * sh;
    out[base + 2] = wrap(T->pt_h[j] - h);
    out[base + 3 + T->pt_kind[j]] = 1.0;
    out[base + 10] = 1.0;
  }
  if (sel) {
    for (int m = 0; m < cap_r; ++m) sel[cap_a + m] = m < cnt ? (int32_t)best_j[m] : -1;
  }
}

/* exact-distance ties between a road edge and another road kind on a ray's
 * nearest segment hit (see lidar_row) since the last or_lidar_ties(1) */
static long long g_lidar_ties = 0;

long long or_lidar_ties(int reset) {
  long long v;
#pragma omp atomic read
  v = g_lidar_ties;
  if (reset) {
#pragma omp atomic write
    g_lidar_ties = 0;
  }
  return v;
}

/* fill_lidar (obs:223-280) for one agent. */
static void lidar_row(const or_tables *T, const or_config *C, const or_state *S, int w, int i,
                      double *out) {
  const int64_t a0 = T->a_off[w];
  const int n = (int)(T->a_off[w + 1] - a0);
  const int64_t s0 = T->s_off[w];
  const int n_seg = (int)(T->s_off[w + 1] - s0);
  const int64_t g = a0 + i;
  const int R = C->n_rays;
  const double max_range = C->max_range;
  for (int k = 0; k < C->obs_width; ++k) out[k] = 0.0;
  double px = S->x[g], py = S->y[g], h = S->heading[g];
  /* _fill_ego (obs:129-142) */
  double c = cos(h), s = sin(h);
  double gx = T->goal_x[g] - px, gy = T->goal_y[g] - py;
  out[0] = S->speed[g];
  out[1] = T->length[g];
  out[2] = T->width[g];
  out[3] = gx * c + gy * s;
  out[4] = -gx * s + gy * c;
  out[5] = hypot(gx, gy);
  out[6] = (S->flags[g] & F_COLLIDED) ? 1.0 : 0.0;

  double center = h;
  if (C->obs_mode == 2) center += S->head_angle[g];
  for (int k = 0; k < R; ++k) {
    double ang;
    if (C->obs_mode == 1 || C->fov >= TWO_PI) ang = center + (2.0 * PI * (double)k) / (double)R;
    else if (R == 1) ang = center;
    else ang = (center - 0.5 * C->fov) + (C->fov * (double)k) / (double)(R - 1);
    double dx = cos(ang), dy = sin(ang);
    double best = INFINITY;
    int best_type = 3;
    /* boxes: visible, != ego, hypot <= max_range + circumradius */
    double bmin = INFINITY;
    for (int j = 0; j < n; ++j) {
      int64_t gj = a0 + j;
      uint16_t fj = S->flags[gj];
      if (j == i || !((fj & F_PRESENT) && !(fj & F_REMOVED))) continue;
      double cdx = S->x[gj] - px, cdy = S->y[gj] - py;
      if (!(hypot(cdx, cdy) <= max_range + T->circumradius[gj])) continue;
      double cj = cos(S->heading[gj]), sj = sin(S->heading[gj]);
      double qx = (px - S->x[gj]) * cj + (py - S->y[gj]) * sj;
      double qy = -(px - S->x[gj]) * sj + (py - S->y[gj]) * cj;
      double rx = dx * cj + dy * sj;
      double ry = -dx * sj + dy * cj;
      double tmin = -INFINITY, tmax = INFINITY;
      int ok = 1;
      for (int axis = 0; axis < 2; ++axis) {
        double p = axis == 0 ? qx : qy, r = axis == 0 ? rx : ry;
        double hh = axis == 0 ? T->half_l[gj] : T->half_w[gj];
        if (r == 0.0) {
          if (!(p >= -hh && p <= hh)) ok = 0;
        } else {
          double ta = (-hh - p) / r, tb = (hh - p) / r;
          double lo = fmin(ta, tb), hi = fmax(ta, tb);
          tmin = fmax(tmin, lo);
          tmax = fmin(tmax, hi);
        }
      }
      if (ok && tmin <= tmax && tmax >= 0.0) {
        double d = tmin > 0.0 ? tmin : 0.0;
        if (d < bmin) bmin = d;
      }
    }
    if (bmin < best) { best = bmin; best_type = 0; }
    /* segments inside the +-max_range box, argmin = first minimal */
    double smin = INFINITY;
    int sedge = 0;
    double qx0 = px - max_range, qy0 = py - max_range, qx1 = px + max_range, qy1 = py + max_range;
    for (int j = 0; j < n_seg; ++j) {
      int64_t q = s0 + j;
      double ax = T->seg_ax[q], ay = T->seg_ay[q], bx = T->seg_bx[q], by = T->seg_by[q];
      double lx = ax < bx ? ax : bx, hx = ax < bx ? bx : ax;
      double ly = ay < by ? ay : by, hy = ay < by ? by : ay;
      if (lx > qx1 || qx0 > hx || ly > qy1 || qy0 > hy) continue;
      double ex = bx - ax, ey = by - ay, wx = ax - px, wy = ay - py;
      double denom = dx * ey - dy * ex;
      if (denom == 0.0) continue;
      double t = (wx * ey - wy * ex) / denom;
      double u = (wx * dy - wy * dx) / denom;
      if (!(t >= 0.0 && u >= 0.0 && u <= 1.0)) continue;
      /* nearest wins; an exact tie between a road edge and another kind goes
       * to the edge (the reference breaks such ties in BVH order) */
      const int is_edge = T->seg_kind[q] == ROAD_EDGE;
      if (t == smin && is_edge != sedge) {
        /* the one case where the reference's answer depends on its BVH
         * traversal order (obs:261-271): counted, reported by or_lidar_ties */
#pragma omp atomic
        g_lidar_ties++;
      }
      if (t < smin || (t == smin && is_edge && !sedge)) { smin = t; sedge = is_edge; }
    }
    if (smin < best) { best = smin; best_type = sedge ? 1 : 2; }
    if (best > max_range) { best = max_range; best_type = 3; }
    double *slot = out + 7 + 5 * k;
    slot[0] = best;
    slot[1 + best_type] = 1.0;
  }
}

static void fill_world_obs(const or_tables *T, const or_config *C, const or_state *S, int w,
                           double *obs, int32_t *sel_idx, double *best_d, int64_t *best_j) {
  const int64_t c0 = T->c_off[w];
  const int nrow = (int)(T->c_off[w + 1] - c0);
  const int sel_w = C->max_agents_obs + C->max_road_points_obs;
  for (int r = 0; r < nrow; ++r) {
    int64_t g = T->row_agent[c0 + r];
    double *out = obs + (c0 + r) * (int64_t)C->obs_width;
    int32_t *sel = sel_idx ? sel_idx + (c0 + r) * (int64_t)sel_w : NULL;
    uint16_t f = S->flags[g];
    if (f & (F_DONE | F_REMOVED)) {
      for (int k = 0; k < C->obs_width; ++k) out[k] = 0.0;
      if (sel) for (int k = 0; k < sel_w; ++k) sel[k] = -1;
      continue;
    }
    int i = (int)(g - T->a_off[w]);
    if (C->obs_mode == 0) radial_row(T, C, S, w, i, out, sel, best_d, best_j);
    else lidar_row(T, C, S, w, i, out);
  }
}

/* ----- world step --------------------------------------------------------- */

static void reset_world(const or_tables *T, or_state *S, int w) {
  const int64_t a0 = T->a_off[w];
  const int A = (int)(T->a_off[w + 1] - a0);
  const int64_t r0 = T->r_off[w];
  for (int i = 0; i < A; ++i) {
    int64_t g = a0 + i;
    S->x[g] = T->rep_x[r0 + i];
    S->y[g] = T->rep_y[r0 + i];
    S->heading[g] = T->rep_h[r0 + i];
    S->speed[g] = T->rep_v[r0 + i];
    S->head_angle[g] = 0.0;
    int present = T->rep_present[r0 + i] || (T->sflags[g] & SF_CONTROLLED);
    S->flags[g] = present ? F_PRESENT : 0;
  }
  S->t[w] = 0;
  S->episode_over[w] = 0;
}

/* World.step for world w.  ep[0..4] = (ended_now, n_controlled, n_goal,
 * n_veh_collision, n_offroad). */
static void step_world(const or_tables *T, const or_config *C, or_state *S, int w,
                       const double *actions, int act_dim, double *rewards, uint8_t *dones,
                       uint8_t *info, int32_t *ep, double *scratch) {
  const int64_t a0 = T->a_off[w];
  const int A = (int)(T->a_off[w + 1] - a0);
  const int64_t c0 = T->c_off[w];
  const int nrow = (int)(T->c_off[w + 1] - c0);
  const int NR = T->n_rows;
  ep[0] = 0;
  for (int r = 0; r < nrow; ++r) {
    rewards[c0 + r] = 0.0;
    info[c0 + r] = info[NR + c0 + r] = info[2 * NR + c0 + r] = 0;
  }
  if (S->episode_over[w]) {
    for (int r = 0; r < nrow; ++r) dones[c0 + r] = (S->flags[T->row_agent[c0 + r]] & F_DONE) != 0;
    return;
  }
  const int Tw = T->num_steps[w];
  const int t_next = (S->t[w] + 1 < Tw - 1) ? S->t[w] + 1 : Tw - 1;
  const double dt = T->dt[w];
  const int64_t rn = T->r_off[w] + (int64_t)t_next * A;
  double *cs = scratch, *sn = scratch + A;
  uint8_t *elig = (uint8_t *)(scratch + 2 * A);

  /* (1) removals, dynamics, head angle, replay */
  for (int i = 0; i < A; ++i) {
    int64_t g = a0 + i;
    uint16_t f = S->flags[g];
    if (f & F_PENDING) f |= F_REMOVED;
    f &= ~F_PENDING;
    uint8_t sf = T->sflags[g];
    int ctrl = sf & SF_CONTROLLED;
    if (actions && ctrl && !(f & (F_REMOVED | F_DONE))) {
      const double *a = actions + (int64_t)T->ctrl_row[g] * act_dim;
      double x = S->x[g], y = S->y[g], h = S->heading[g], v = S->speed[g];
      if (C->dynamics == 0) {
        double acc = clip(a[0], C->accel_lo, C->accel_hi);
        double delta = clip(a[1], C->steer_lo, C->steer_hi);
        double v_bar = clip(v + 0.5 * acc * dt, -C->v_max, C->v_max);
        double beta = atan(0.5 * tan(delta));
        double ang = h + beta;
        x += v_bar * cos(ang) * dt;
        y += v_bar * sin(ang) * dt;
        h = wrap(h + v_bar * cos(beta) * tan(delta) / T->length[g] * dt);
        v = clip(v + acc * dt, -C->v_max, C->v_max);
      } else if (C->dynamics == 1) {
        double d = v * dt + 0.5 * a[0] * dt * dt;
        x += d * cos(h);
        y += d * sin(h);
        h = wrap(h + a[1] * d);
        v = clip(v + a[0] * dt, -C->v_max, C->v_max);
      } else {
        double ddx = clip(a[0], C->delta_lo[0], C->delta_hi[0]);
        double ddy = clip(a[1], C->delta_lo[1], C->delta_hi[1]);
        double dyaw = clip(a[2], C->delta_lo[2], C->delta_hi[2]);
        double ch = cos(h), sh = sin(h);
        x += ddx * ch - ddy * sh;
        y += ddx * sh + ddy * ch;
        h = wrap(h + dyaw);
        v = clip(hypot(ddx, ddy) / dt, -C->v_max, C->v_max);
      }
      S->x[g] = x; S->y[g] = y; S->heading[g] = h; S->speed[g] = v;
      int head_col = C->dynamics == 2 ? 3 : 2;
      if (act_dim > head_col)
        S->head_angle[g] = clip(S->head_angle[g] + a[head_col] * dt, -0.5 * PI, 0.5 * PI);
    }
    int replay = (sf & SF_REPLAY_ONLY) || (!actions && ctrl);
    if (replay && (sf & SF_INSTANTIABLE) && !(f & F_REMOVED)) {
      S->x[g] = T->rep_x[rn + i];
      S->y[g] = T->rep_y[rn + i];
      S->heading[g] = T->rep_h[rn + i];
      S->speed[g] = T->rep_v[rn + i];
      if (T->rep_present[rn + i]) f |= F_PRESENT; else f &= ~F_PRESENT;
    }
    f &= ~(F_COLLIDED | F_OFFROAD);
    S->flags[g] = f;
  }
  /* (2-3) collisions */
  if (A) {
    for (int i = 0; i < A; ++i) {
      int64_t g = a0 + i;
      cs[i] = cos(S->heading[g]);
      sn[i] = sin(S->heading[g]);
      uint16_t f = S->flags[g];
      int ctrl = T->sflags[g] & SF_CONTROLLED;
      elig[i] = (f & F_PRESENT) && !(f & F_REMOVED) &&
                ((ctrl && !(f & F_DONE)) || T->rep_valid[rn + i]);
    }
    const double *X = S->x + a0, *Y = S->y + a0, *HL = T->half_l + a0, *HW = T->half_w + a0;
    for (int i = 0; i < A; ++i) {
      if (!elig[i]) continue;
      for (int j = i + 1; j < A; ++j) {
        if (!elig[j]) continue;
        if (sat_hit(X, Y, cs, sn, HL, HW, i, j)) {
          S->flags[a0 + i] |= F_COLLIDED;
          S->flags[a0 + j] |= F_COLLIDED;
        }
      }
    }
    const int64_t s0 = T->s_off[w];
    const int n_seg = (int)(T->s_off[w + 1] - s0);
    for (int i = 0; i < A; ++i) {
      int64_t g = a0 + i;
      if (!elig[i] || (T->sflags[g] & SF_PEDESTRIAN)) continue;
      double c = cs[i], s = sn[i];
      double rx = HL[i] * fabs(c) + HW[i] * fabs(s), ry = HL[i] * fabs(s) + HW[i] * fabs(c);
      double bx0 = X[i] - rx - AABB_MARGIN, by0 = Y[i] - ry - AABB_MARGIN;
      double bx1 = X[i] + rx + AABB_MARGIN, by1 = Y[i] + ry + AABB_MARGIN;
      for (int k = 0; k < n_seg; ++k) {
        int64_t q = s0 + k;
        if (T->seg_kind[q] != ROAD_EDGE) continue;
        double ax = T->seg_ax[q], ay = T->seg_ay[q], bx = T->seg_bx[q], by = T->seg_by[q];
        double lx = ax < bx ? ax : bx, hx = ax < bx ? bx : ax;
        double ly = ay < by ? ay : by, hy = ay < by ? by : ay;
        if (lx > bx1 || bx0 > hx || ly > by1 || by0 > hy) continue;
        if (seg_box_hit(X[i], Y[i], c, s, HL[i], HW[i], ax, ay, bx, by)) {
          S->flags[g] |= F_OFFROAD;
          break;
        }
      }
    }
  }
  /* (4) goal rewards, then terminations */
  if (nrow) {
    int any_end = 0;
    for (int i = 0; i < A; ++i) {
      int64_t g = a0 + i;
      uint16_t f = S->flags[g];
      int ctrl = T->sflags[g] & SF_CONTROLLED;
      int live = ctrl && !(f & (F_REMOVED | F_DONE));
      int at_goal = 0;
      if (live) at_goal = hypot(S->x[g] - T->goal_x[g], S->y[g] - T->goal_y[g]) <= C->goal_tolerance;
      int coll = (f & F_COLLIDED) != 0, off = (f & F_OFFROAD) != 0;
      if (at_goal) f |= F_GOAL_REACHED | F_GOAL_EVER | F_PENDING | F_DONE;
      if (coll && live) f |= F_COLL_EVER;
      if (off && live) f |= F_OFF_EVER;
      if (C->collision_behavior == 1 && live && (coll || off)) f |= F_PENDING | F_DONE;
      if (C->collision_behavior == 2 && live && (coll || off)) any_end = 1;
      S->flags[g] = f;
      if (ctrl) {
        int r = T->ctrl_row[g];
        if (at_goal) rewards[r] = 1.0;
        info[r] = (uint8_t)at_goal;
        info[NR + r] = (uint8_t)(coll && live);
        info[2 * NR + r] = (uint8_t)(off && live);
      }
    }
    if (any_end) S->episode_over[w] = 1;
  }
  S->t[w] += 1;
  if (S->t[w] >= Tw) S->episode_over[w] = 1;
  if (S->episode_over[w]) {
    for (int r = 0; r < nrow; ++r) S->flags[T->row_agent[c0 + r]] |= F_DONE;
    int ng = 0, nv = 0, no = 0;
    for (int r = 0; r < nrow; ++r) {
      uint16_t f = S->flags[T->row_agent[c0 + r]];
      ng += (f & F_GOAL_EVER) != 0;
      nv += (f & F_COLL_EVER) != 0;
      no += (f & F_OFF_EVER) != 0;
    }
    ep[0] = 1; ep[1] = nrow; ep[2] = ng; ep[3] = nv; ep[4] = no;
  }
  for (int r = 0; r < nrow; ++r) dones[c0 + r] = (S->flags[T->row_agent[c0 + r]] & F_DONE) != 0;
}

static int max_agents(const or_tables *T) {
  int m = 1;
  for (int w = 0; w < T->n_worlds; ++w) {
    int a = (int)(T->a_off[w + 1] - T->a_off[w]);
    if (a > m) m = a;
  }
  return m;
}

/* Batched step over all worlds (SimBatch.step, engine.py:626-649).  When
 * auto_reset, finished worlds are reset and rewards zeroed (VecDriveEnv.step,
 * env.py:95-109) before observations are filled. */
int or_step(const or_tables *T, const or_config *C, or_state *S, const double *actions,
            int act_dim, double *obs, double *rewards, uint8_t *dones, uint8_t *info,
            int32_t *sel_idx, int32_t *ep, int auto_reset, int n_threads) {
  int amax = max_agents(T);
  int kmax = C->max_agents_obs > C->max_road_points_obs ? C->max_agents_obs : C->max_road_points_obs;
  if (kmax < 1) kmax = 1;
#ifdef _OPENMP
  if (n_threads > 0) omp_set_num_threads(n_threads);
#else
  (void)n_threads;
#endif
#pragma omp parallel
  {
    double *scratch = (double *)malloc(sizeof(double) * (3 * (size_t)amax + 8));
    double *best_d = (double *)malloc(sizeof(double) * kmax);
    int64_t *best_j = (int64_t *)malloc(sizeof(int64_t) * kmax);
#pragma omp for schedule(dynamic, 1)
    for (int w = 0; w < T->n_worlds; ++w) {
      step_world(T, C, S, w, actions, act_dim, rewards, dones, info, ep + 5 * w, scratch);
      if (auto_reset && S->episode_over[w]) {
        reset_world(T, S, w);
        for (int64_t r = T->c_off[w]; r < T->c_off[w + 1]; ++r) rewards[r] = 0.0;
      }
      if (obs) fill_world_obs(T, C, S, w, obs, sel_idx, best_d, best_j);
    }
    free(scratch);
    free(best_d);
    free(best_j);
  }
  return 0;
}

/* SimBatch.reset(world_ids) (engine.py:651-663). */
int or_reset(const or_tables *T, const or_config *C, or_state *S, const uint8_t *mask,
             double *obs, double *rewards, uint8_t *dones, int32_t *sel_idx) {
  int kmax = C->max_agents_obs > C->max_road_points_obs ? C->max_agents_obs : C->max_road_points_obs;
  if (kmax < 1) kmax = 1;
  double *best_d = (double *)malloc(sizeof(double) * kmax);
  int64_t *best_j = (int64_t *)malloc(sizeof(int64_t) * kmax);
  for (int w = 0; w < T->n_worlds; ++w) {
    if (mask && !mask[w]) continue;
    reset_world(T, S, w);
    for (int64_t r = T->c_off[w]; r < T->c_off[w + 1]; ++r) {
      if (rewards) rewards[r] = 0.0;
      if (dones) dones[r] = 0;
    }
    if (obs) fill_world_obs(T, C, S, w, obs, sel_idx, best_d, best_j);
  }
  free(best_d);
  free(best_j);
  return 0;
}

int or_observe(const or_tables *T, const or_config *C, const or_state *S, double *obs,
               int32_t *sel_idx) {
  int kmax = C->max_agents_obs > C->max_road_points_obs ? C->max_agents_obs : C->max_road_points_obs;
  if (kmax < 1) kmax = 1;
  double *best_d = (double *)malloc(sizeof(double) * kmax);
  int64_t *best_j = (int64_t *)malloc(sizeof(int64_t) * kmax);
  for (int w = 0; w < T->n_worlds; ++w) fill_world_obs(T, C, S, w, obs, sel_idx, best_d, best_j);
  free(best_d);
  free(best_j);
  return 0;
}

int or_abi_version(void) { return 1; }
