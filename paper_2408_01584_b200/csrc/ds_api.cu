// ds_api.cu -- the extern "C" boundary (include/drivesim_b200.h).
#include <float.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <new>

#include <vector>

#include "ds_internal.cuh"

namespace {

thread_local char g_err[512] = "";

int fail(int code, const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

int cuda_fail(cudaError_t e, const char *where) {
  return fail(DS_E_CUDA, "%s: %s", where, cudaGetErrorString(e));
}

int expected_width(const ds_config &c) {
  if (c.obs_mode == DS_OBS_RADIAL) return 7 + 7 * c.max_agents_obs + 11 * c.max_road_points_obs;
  return 7 + 5 * c.n_rays;
}

}  // namespace

extern "C" {

int ds_abi_version(void) { return DS_ABI_VERSION; }

void ds_struct_sizes(int64_t out[4]) {
  out[0] = sizeof(ds_config);
  out[1] = sizeof(ds_tables);
  out[2] = sizeof(ds_state);
  out[3] = sizeof(ds_step_args);
}

const char *ds_last_error(void) { return g_err; }

int ds_create(const ds_tables *tables, const ds_config *cfg, ds_state *state, int device,
              ds_handle **out) {
  if (!tables || !cfg || !state || !out) return fail(DS_E_INVALID, "ds_create: null argument");
  *out = nullptr;
  const ds_config &c = *cfg;
  if (c.dynamics < 0 || c.dynamics > 2) return fail(DS_E_INVALID, "unknown dynamics %d", c.dynamics);
  if (c.collision_behavior < 0 || c.collision_behavior > 2)
    return fail(DS_E_INVALID, "unknown collision behavior %d", c.collision_behavior);
  if (c.obs_mode < 0 || c.obs_mode > 2) return fail(DS_E_INVALID, "unknown obs mode %d", c.obs_mode);
  if (c.obs_width != expected_width(c))
    return fail(DS_E_INVALID, "obs_width %d != layout width %d", c.obs_width, expected_width(c));
  if (c.max_agents_obs < 0 || c.max_agents_obs > ds::kSelCap || c.max_road_points_obs < 0 ||
      c.max_road_points_obs > ds::kSelCap)
    return fail(DS_E_CAPACITY, "slot caps must be in [0, %d]", ds::kSelCap);
  if (!(c.grid_cell > 0.0)) return fail(DS_E_INVALID, "grid_cell must be > 0");
  if (c.obs_mode == DS_OBS_RADIAL && 2.0 * (c.radius + 1e-6) / c.grid_cell + 2.0 > 32.0)
    return fail(DS_E_INVALID, "grid_cell %.3f too small for radius %.3f (> 32 cell rows)",
                c.grid_cell, c.radius);
  if (tables->max_agents < 0 || tables->max_agents > DS_MAX_AGENTS_PER_WORLD)
    return fail(DS_E_CAPACITY, "max agents per world %d > %d", tables->max_agents,
                DS_MAX_AGENTS_PER_WORLD);
  if (tables->n_worlds < 1) return fail(DS_E_INVALID, "need at least one world");
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
  ds_handle *h = new (std::nothrow) ds_handle();
  if (!h) return fail(DS_E_INVALID, "out of host memory");
  h->tab = *tables;
  h->cfg = c;
  h->st = *state;
  h->device = device;
  h->obs_width = c.obs_width;
  h->obs_dtype = DS_OBS_F32;
  h->obs_stride = c.obs_width;
  e = cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, device);
  if (e != cudaSuccess) {
    delete h;
    return cuda_fail(e, "cudaDeviceGetAttribute");
  }
  // uniform per-world strides (one host read of the offsets at creation)
  {
    const int W = tables->n_worlds;
    const int64_t *offs[4] = {tables->a_off, tables->c_off, tables->p_off, tables->r_off};
    int64_t *uni[4] = {&h->uni_a, &h->uni_c, &h->uni_p, &h->uni_r};
    std::vector<int64_t> hv((size_t)W + 1);
    for (int k = 0; k < 4; ++k) {
      *uni[k] = 0;
      if (W <= 0 || !offs[k] ||
          cudaMemcpy(hv.data(), offs[k], hv.size() * sizeof(int64_t), cudaMemcpyDeviceToHost) != cudaSuccess)
        continue;
      const int64_t st = hv[1] - hv[0];
      bool ok = hv[0] == 0 && st > 0;
      for (int w = 1; ok && w <= W; ++w) ok = hv[w] == (int64_t)w * st;
      if (ok) *uni[k] = st;
    }
    cudaGetLastError();
  }
  int amax = tables->max_agents < 1 ? 1 : tables->max_agents;
  h->step_threads = ((amax + 31) / 32) * 32;
  h->step_smem = ds::step_smem_bytes(amax);
  int max_optin = 0;
  cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  ds::obs_plan(h, max_optin);
  if ((int)h->obs_smem > max_optin || (int)h->step_smem > max_optin) {
    delete h;
    return fail(DS_E_CAPACITY, "shared memory %zu/%zu exceeds %d", h->obs_smem, h->step_smem,
                max_optin);
  }
  e = ds::configure_kernels(max_optin);
  if (e != cudaSuccess) {
    delete h;
    return cuda_fail(e, "cudaFuncSetAttribute");
  }
  *out = h;
  return DS_OK;
}

int ds_destroy(ds_handle *h) {
  delete h;
  return DS_OK;
}

int ds_set_obs_format(ds_handle *h, int dtype, int row_stride) {
  if (!h) return fail(DS_E_INVALID, "ds_set_obs_format: null handle");
  if (dtype != DS_OBS_F32 && dtype != DS_OBS_BF16)
    return fail(DS_E_INVALID, "unknown observation dtype %d", dtype);
  if (row_stride == 0) row_stride = h->obs_width;
  if (row_stride < h->obs_width)
    return fail(DS_E_INVALID, "row stride %d < observation width %d", row_stride, h->obs_width);
  h->obs_dtype = dtype;
  h->obs_stride = row_stride;
  return DS_OK;
}

int ds_sample_categorical(const void *logits, int dtype, int64_t rows, int32_t n, int64_t ld,
                          uint64_t seed, uint64_t counter, int32_t *out, void *stream) {
  if (rows < 0 || n < 1 || ld < n) return fail(DS_E_INVALID, "ds_sample_categorical: bad shape");
  if (dtype != DS_OBS_F32 && dtype != DS_OBS_BF16)
    return fail(DS_E_INVALID, "ds_sample_categorical: unknown dtype %d", dtype);
  if (rows == 0) return DS_OK;
  if (!logits || !out) return fail(DS_E_INVALID, "ds_sample_categorical: null argument");
  cudaError_t e = ds::launch_sample(logits, dtype, rows, n, ld, seed, counter, out,
                                    (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "sample kernel");
  return DS_OK;
}

int ds_status(ds_handle *h, uint32_t *out, int clear, void *stream) {
  if (!h || !out) return fail(DS_E_INVALID, "ds_status: null argument");
  *out = 0;
  if (!h->st.status) return DS_OK;
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = cudaMemcpyAsync(out, h->st.status, sizeof(uint32_t), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e == cudaSuccess && clear) e = cudaMemsetAsync(h->st.status, 0, sizeof(uint32_t), s);
  if (e != cudaSuccess) return cuda_fail(e, "status");
  return DS_OK;
}

int ds_gumbel_noise(const uint32_t *bits, int64_t n, float *out, void *stream) {
  if (n < 0) return fail(DS_E_INVALID, "ds_gumbel_noise: negative count");
  if (n > 0 && (!bits || !out)) return fail(DS_E_INVALID, "ds_gumbel_noise: null argument");
  cudaError_t e = ds::launch_gumbel(bits, n, out, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "gumbel kernel");
  return DS_OK;
}

int ds_goal_seek(ds_handle *h, float *actions, void *stream) {
  if (!h) return fail(DS_E_INVALID, "ds_goal_seek: null handle");
  if (h->tab.n_rows > 0 && !actions) return fail(DS_E_INVALID, "ds_goal_seek: null actions");
  cudaError_t e = ds::launch_goal_seek(h, actions, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "goal_seek kernel");
  return DS_OK;
}

int64_t ds_decimate_scratch_bytes(int64_t n_points) {
  return n_points < 0 ? 0 : n_points * (int64_t)(2 * sizeof(int32_t) + sizeof(double));
}

int ds_decimate_polylines(const double *x, const double *y, const int64_t *poly_off,
                          int64_t n_poly, const uint8_t *skip, double threshold, uint8_t *keep,
                          void *scratch, int64_t n_points, void *stream) {
  if (n_poly < 0 || n_points < 0) return fail(DS_E_INVALID, "ds_decimate_polylines: bad sizes");
  if (n_poly == 0 || n_points == 0) return DS_OK;
  if (!x || !y || !poly_off || !keep || !scratch)
    return fail(DS_E_INVALID, "ds_decimate_polylines: null argument");
  cudaError_t e = ds::launch_decimate(x, y, poly_off, n_poly, skip, threshold, keep, scratch,
                                      n_points, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "decimate kernel");
  return DS_OK;
}

int ds_reset(ds_handle *h, const uint8_t *world_mask, void *obs, float *rewards, uint8_t *dones,
             const float *obs_scale, int32_t *sel_idx, void *stream) {
  if (!h || !obs) return fail(DS_E_INVALID, "ds_reset: null argument");
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = ds::launch_reset(h, world_mask, rewards, dones, s);
  if (e != cudaSuccess) return cuda_fail(e, "reset_kernel");
  e = ds::launch_observe(h, world_mask, obs, obs_scale, sel_idx, s);
  if (e != cudaSuccess) return cuda_fail(e, "observe kernel");
  return DS_OK;
}

int ds_observe(ds_handle *h, const uint8_t *world_mask, void *obs, const float *obs_scale,
               int32_t *sel_idx, void *stream) {
  if (!h || !obs) return fail(DS_E_INVALID, "ds_observe: null argument");
  cudaError_t e = ds::launch_observe(h, world_mask, obs, obs_scale, sel_idx, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "observe kernel");
  return DS_OK;
}

int ds_step(ds_handle *h, const ds_step_args *a, void *stream) {
  if (!h || !a) return fail(DS_E_INVALID, "ds_step: null argument");
  if (!a->obs || !a->rewards || !a->dones || !a->info)
    return fail(DS_E_INVALID, "ds_step: null output buffer");
  if (!a->replay) {
    if (a->actions) {
      const int need = h->cfg.dynamics == DS_DYN_DELTA_LOCAL ? 3 : 2;
      if (a->act_dim < need) return fail(DS_E_INVALID, "act_dim %d < %d", a->act_dim, need);
    } else if (a->action_idx) {
      if (!a->grid_accel || !a->grid_steer || a->n_accel < 1 || a->n_steer < 1)
        return fail(DS_E_INVALID, "discrete actions need the action grid");
      if (h->cfg.dynamics == DS_DYN_DELTA_LOCAL)
        return fail(DS_E_INVALID, "discrete grid actions are (accel, steer) pairs");
    } else {
      return fail(DS_E_INVALID, "ds_step: no actions and replay == 0");
    }
  }
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e;
  if (a->events[0] && (e = cudaEventRecord((cudaEvent_t)a->events[0], s)) != cudaSuccess)
    return cuda_fail(e, "event");
  e = ds::launch_step(h, a, s);
  if (e != cudaSuccess) return cuda_fail(e, "step_kernel");
  if (a->events[1] && (e = cudaEventRecord((cudaEvent_t)a->events[1], s)) != cudaSuccess)
    return cuda_fail(e, "event");
  e = ds::launch_observe(h, nullptr, a->obs, a->obs_scale, a->sel_idx, s);
  if (e != cudaSuccess) return cuda_fail(e, "observe kernel");
  if (a->events[2] && (e = cudaEventRecord((cudaEvent_t)a->events[2], s)) != cudaSuccess)
    return cuda_fail(e, "event");
  return DS_OK;
}

int ds_episode_drain(ds_handle *h, int32_t *out, int32_t max_records, int32_t *n_out,
                     void *stream) {
  if (!h || !n_out) return fail(DS_E_INVALID, "ds_episode_drain: null argument");
  *n_out = 0;
  if (!h->st.ring || !h->st.ring_head) return DS_OK;
  cudaStream_t s = (cudaStream_t)stream;
  uint32_t head = 0;
  cudaError_t e = cudaMemcpyAsync(&head, h->st.ring_head, sizeof(head), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_fail(e, "drain head");
  const uint32_t avail = head < (uint32_t)h->st.ring_cap ? head : (uint32_t)h->st.ring_cap;
  const uint32_t n = avail < (uint32_t)max_records ? avail : (uint32_t)max_records;
  if (n && out) {
    e = cudaMemcpyAsync(out, h->st.ring, (size_t)n * 6 * sizeof(int32_t), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_fail(e, "drain copy");
  }
  e = cudaMemsetAsync(h->st.ring_head, 0, sizeof(uint32_t), s);
  if (e != cudaSuccess) return cuda_fail(e, "drain reset");
  *n_out = (int32_t)n;
  if (head > (uint32_t)h->st.ring_cap || n < avail)
    return fail(DS_E_OVERFLOW, "episode ring overflow: %u records, capacity %d", head,
                h->st.ring_cap);
  return DS_OK;
}

// ---------------------------------------------------------------------------
// Host helpers used by the packer (exact restatements of CPU libm paths).
// ---------------------------------------------------------------------------

int ds_host_hypot_libm(const double *x, const double *y, int64_t n, double *out) {
  for (int64_t i = 0; i < n; ++i) out[i] = ::hypot(x[i], y[i]);
  return DS_OK;
}

int ds_host_wrap_port(const double *x, int64_t n, double *out) {
  for (int64_t i = 0; i < n; ++i) out[i] = ds::wrap(x[i]);
  return DS_OK;
}

int ds_host_hypot_port(const double *x, const double *y, int64_t n, double *out) {
  for (int64_t i = 0; i < n; ++i) out[i] = ds::hypot(x[i], y[i]);
  return DS_OK;
}

// CPython's math.hypot (Modules/mathmodule.c vector_norm, 3.12) for two
// finite coordinates: lossless scaling, error-free squares and sums, one
// differential correction.  Used for World.__init__'s log speed (engine.py:205)
// and mark_controllable (scenario.py:382).
static inline void dl_mul(double x, double y, double *hi, double *lo) {
  const double z = x * y;
  *hi = z;
  *lo = fma(x, y, -z);
}

static inline void dl_fast_sum(double a, double b, double *hi, double *lo) {
  const double x = a + b;
  *hi = x;
  *lo = (a - x) + b;
}

static double cpython_hypot(double x, double y) {
  x = fabs(x);
  y = fabs(y);
  if (isinf(x) || isinf(y)) return INFINITY;
  if (isnan(x) || isnan(y)) return NAN;
  double mx = x > y ? x : y;
  if (mx == 0.0) return mx;
  int max_e;
  frexp(mx, &max_e);
  if (max_e < -1023) return DBL_MIN * cpython_hypot(x / DBL_MIN, y / DBL_MIN);
  const double scale = ldexp(1.0, -max_e);
  double csum = 1.0, frac1 = 0.0, frac2 = 0.0, hi, lo;
  const double v[2] = {x, y};
  for (int i = 0; i < 2; ++i) {
    const double s = v[i] * scale;
    double phi, plo;
    dl_mul(s, s, &phi, &plo);
    dl_fast_sum(csum, phi, &hi, &lo);
    csum = hi;
    frac1 += plo;
    frac2 += lo;
  }
  double h = sqrt(csum - 1.0 + (frac1 + frac2));
  double phi, plo;
  dl_mul(-h, h, &phi, &plo);
  dl_fast_sum(csum, phi, &hi, &lo);
  csum = hi;
  frac1 += plo;
  frac2 += lo;
  const double r = csum - 1.0 + (frac1 + frac2);
  h += r / (2.0 * h);
  return h / scale;
}

int ds_host_hypot_cpython(const double *x, const double *y, int64_t n, double *out) {
  for (int64_t i = 0; i < n; ++i) out[i] = cpython_hypot(x[i], y[i]);
  return DS_OK;
}

// Road point headings (engine.py:256-265): atan2 to the next point; the last
// point of a polyline uses its previous segment; a single point gives 0.
int ds_host_road_headings(const double *x, const double *y, const int64_t *poly_pt_off,
                          int64_t n_poly, double *out) {
  for (int64_t r = 0; r < n_poly; ++r) {
    const int64_t b = poly_pt_off[r], e = poly_pt_off[r + 1];
    if (e - b == 1) {
      out[b] = 0.0;
      continue;
    }
    for (int64_t j = b; j < e; ++j) {
      const int64_t q = j + 1 < e ? j + 1 : j;
      const int64_t p = j + 1 < e ? j : j - 1;
      out[j] = atan2(y[q] - y[p], x[q] - x[p]);
    }
  }
  return DS_OK;
}

}  // extern "C"
