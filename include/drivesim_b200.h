/*
 * drivesim_b200.h -- C ABI of the B200 batched world step (libdrivesim_b200.so).
 *
 * The reference has no native ABI: its seams are Python classes.  Each entry
 * point below replaces one reference call on the hot path (file:line under
 * /root/reference/pkg/src/drivesim/):
 *
 *   ds_create        SimBatch.__init__ / World.__init__   engine.py:591-621, 173-314
 *   ds_reset         SimBatch.reset(world_ids)            engine.py:651-663
 *                    (World.reset 318-340 + World.observe 514-519)
 *   ds_step          SimBatch.step(actions)               engine.py:626-649
 *                    (World.step 357-498 + _fill_obs 500-512 + fill_radial
 *                    observation.py:145-210 / fill_lidar 223-280), plus the
 *                    VecDriveEnv.step extras (pkg/rl/src/drivesim_rl/env.py:95-121):
 *                    discrete-action decode, obs normalisation, auto-reset
 *   ds_episode_drain SimBatch.episode_infos / World.episode_info engine.py:521-528, 646-647
 *   ds_destroy       SimBatch.close                        engine.py:668-671
 *   ds_last_error    (exception text of the above)
 *
 * Ownership: every device buffer (static tables, mutable state, outputs,
 * scratch) is allocated by the caller (torch) and passed as a raw pointer;
 * the library never allocates or frees device memory and keeps no pointer
 * beyond what ds_create copies into its handle.  All work is enqueued on the
 * caller's stream with no host synchronisation (except ds_episode_drain,
 * which is documented as synchronising).  A handle is single-caller.
 *
 * Errors: every function returns 0 on success or a negative DS_E* code, and
 * ds_last_error() returns a thread-local message for the last failure.
 */
#ifndef DRIVESIM_B200_H
#define DRIVESIM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DS_ABI_VERSION 4
#define DS_MAX_AGENTS_PER_WORLD 1024

/* error codes */
#define DS_OK 0
#define DS_E_INVALID (-1)        /* bad argument / config  -> ValueError            */
#define DS_E_ACTION_COUNT (-2)   /* action rows != controlled rows -> ActionCountMismatch */
#define DS_E_CUDA (-3)           /* CUDA runtime failure   -> RuntimeError          */
#define DS_E_CAPACITY (-4)       /* a compiled-in capacity was exceeded            */
#define DS_E_OVERFLOW (-5)       /* episode ring overflowed before a drain         */

/* enums (values mirror the order of the reference's tuples, engine.py:32-34) */
#define DS_DYN_CLASSIC 0
#define DS_DYN_INVERTIBLE 1
#define DS_DYN_DELTA_LOCAL 2
#define DS_COLL_IGNORE 0
#define DS_COLL_REMOVE_AGENT 1
#define DS_COLL_END_EPISODE 2
#define DS_OBS_RADIAL 0
#define DS_OBS_LIDAR 1
#define DS_OBS_VIEW_CONE 2
/* observation buffer element types (ds_set_obs_format) */
#define DS_OBS_F32 0
#define DS_OBS_BF16 1

/* static per-agent flags (ds_tables.sflags) */
#define DS_SF_CONTROLLED 1
#define DS_SF_INSTANTIABLE 2
#define DS_SF_REPLAY_ONLY 4
#define DS_SF_PEDESTRIAN 8

/* mutable per-agent flags (ds_state.flags), World attributes engine.py:296-305 */
#define DS_F_PRESENT 0x001
#define DS_F_REMOVED 0x002
#define DS_F_PENDING 0x004
#define DS_F_GOAL_REACHED 0x008
#define DS_F_COLLIDED 0x010
#define DS_F_OFFROAD 0x020
#define DS_F_GOAL_EVER 0x040
#define DS_F_COLL_EVER 0x080
#define DS_F_OFF_EVER 0x100
#define DS_F_DONE 0x200

typedef struct ds_config {
  int32_t dynamics;            /* DS_DYN_*   SimConfig.dynamics            */
  int32_t collision_behavior;  /* DS_COLL_*  SimConfig.collision_behavior  */
  int32_t obs_mode;            /* DS_OBS_*   ObsConfig.mode                */
  int32_t n_rays;              /* ObsConfig.n_rays                          */
  int32_t max_agents_obs;      /* ObsConfig.max_agents_obs                  */
  int32_t max_road_points_obs; /* ObsConfig.max_road_points_obs             */
  int32_t obs_width;           /* observation row width (checked)           */
  int32_t reserved0;
  double radius, fov, max_range, goal_tolerance;
  double accel_lo, accel_hi, steer_lo, steer_hi, v_max;
  double delta_lo[3], delta_hi[3]; /* delta_local (dx, dy, dyaw) bounds    */
  double grid_cell;            /* road grid cell size (metres)              */
} ds_config;

/* Static world tables (device pointers; layout documented in DESIGN.md and
 * paper_2408_01584_b200/packing.py + device_layout.py).  Offsets are int64
 * CSR arrays of length n_worlds+1 unless noted. */
typedef struct ds_tables {
  int32_t n_worlds, n_agents, n_rows, max_agents;
  int32_t max_points, reserved0;    /* largest road-point count of a world */
  const int64_t *a_off, *c_off, *r_off;
  const int32_t *num_steps;
  const double *dt;
  /* agents [n_agents] */
  const int8_t *kind;
  const double *length, *width, *half_l, *half_w, *circumradius, *goal_x, *goal_y;
  const uint8_t *sflags;
  const int32_t *ctrl_row;  /* -1 if not controlled */
  const int32_t *row_agent; /* [n_rows] */
  /* replay tables, time-major per world: r_off[w] + t*A_w + i */
  const double *rep_x, *rep_y, *rep_h, *rep_v;
  const uint8_t *rep_valid, *rep_present;
  /* road grid (shared by points and segments), per world */
  const double *grid_x0, *grid_y0; /* [n_worlds] */
  const int32_t *grid_nx, *grid_ny; /* [n_worlds] */
  const int64_t *grid_cell_off;     /* [n_worlds+1] offset into *_cell_start (ncell+1 per world) */
  /* road points, grid-sorted (cell-major, original index ascending inside a cell) */
  const int64_t *p_off;             /* [n_worlds+1] */
  const int32_t *pt_cell_start;     /* absolute index into gpt_* */
  const double *gpt_x, *gpt_y, *gpt_h;
  const int8_t *gpt_kind;
  const int32_t *gpt_id;            /* original point index inside its world */
  /* road-edge segments binned to every cell their AABB touches (duplicates) */
  const int32_t *eseg_cell_start;   /* absolute index into eseg_* */
  const double *eseg_ax, *eseg_ay, *eseg_bx, *eseg_by;
  /* all segments binned likewise (LiDAR / view-cone) */
  const int32_t *aseg_cell_start;
  const double *aseg_ax, *aseg_ay, *aseg_bx, *aseg_by;
  const int32_t *aseg_id;           /* original segment index inside its world */
  const uint8_t *aseg_edge;         /* 1 if road_edge */
  const int64_t *s_off;             /* [n_worlds+1] segments per world (original) */
  /* grid-sorted points as float2 relative to (grid_x0, grid_y0), and the
   * per-world max |float - exact| of those coordinates (shared-memory scan) */
  const float *gpt_xy;
  const double *grid_eps;
  /* grid-sorted points as 32-B records (ds_point_rec): one sector per point
   * for the observation kernel's gather of the selected points */
  const void *gpt_rec;
  /* road-edge segments of eseg_* as float (ax, ay, bx, by) relative to the
   * world's grid origin, 16 B per entry: the off-road AABB prefilter */
  const float *eseg_rel;
  /* per agent, one 32-B record (half_l, half_w, goal_x, goal_y) FP64: the
   * step kernel's statics in one sector (length = 2 half_l and the
   * circumradius = hypot(half_l, half_w) are exact functions of it) */
  const double *agent_rec;
  /* the FP64 endpoints of eseg_* as one 32-B record (ax, ay, bx, by) per
   * entry: the off-road slab test's exact phase reads one sector */
  const double *eseg_rec;
  /* the FP64 endpoints of aseg_* as one 32-B record (ax, ay, bx, by) per
   * entry: the LiDAR / view-cone segment fetch reads one sector */
  const double *aseg_rec;
} ds_tables;

/* One road point of gpt_rec: the gpt_x / gpt_y / gpt_h / gpt_id / gpt_kind
 * entries of the same grid-sorted index. */
typedef struct ds_point_rec {
  double x, y, heading;
  int32_t id;
  int8_t kind;
  int8_t pad[3];
} ds_point_rec;

/* Mutable simulation state (device pointers, torch-owned). */
typedef struct ds_state {
  double *x, *y, *heading, *speed, *head_angle; /* [n_agents] */
  uint16_t *flags;                              /* [n_agents] DS_F_* */
  int32_t *t;                                   /* [n_worlds] World.t */
  uint8_t *episode_over;                        /* [n_worlds] */
  /* episode record ring: [ring_cap][6] int32 (serial, world, n_controlled,
   * n_goal, n_veh_collision, n_offroad) + head counter */
  int32_t *ring;
  uint32_t *ring_head;
  int32_t ring_cap;
  int32_t reserved0;
  /* [n_agents][4] search hint of the radial observation: a bound on the
   * k-th road-point distance and the (grid-relative) position it was taken
   * at; results never depend on it (it only narrows a provably sufficient
   * search disc).  NULL disables it. */
  float *obs_hint;
  /* one device word of sticky DS_STATUS_* bits set by the kernels (read and
   * cleared with ds_status); NULL disables the reporting */
  uint32_t *status;
} ds_state;

/* ds_state.status bits */
#define DS_STATUS_BAD_ACTION_INDEX 1u  /* a joint action index outside the grid:
                                        * the reference's to_continuous raises
                                        * IndexError (env.py:111-116); the
                                        * agent's dynamics are skipped */

/* Per-call step arguments. */
typedef struct ds_step_args {
  const float *actions;      /* [n_rows, act_dim] continuous, or NULL */
  const int32_t *action_idx; /* [n_rows] discrete grid indices (used when actions==NULL and non-NULL) */
  int32_t act_dim;           /* columns of actions */
  int32_t replay;            /* 1: actions=None (expert replay for everyone) */
  const double *grid_accel;  /* [n_accel] ActionGrid.accelerations (discrete mode) */
  const double *grid_steer;  /* [n_steer] ActionGrid.steerings */
  int32_t n_accel, n_steer;
  void *obs;                 /* [n_rows, row_stride] in the handle's obs format (default float32, stride obs_width) */
  float *rewards;            /* [n_rows] */
  uint8_t *dones;            /* [n_rows] */
  uint8_t *info;             /* [3, n_rows]: goal, veh_collision, offroad */
  const float *obs_scale;    /* [obs_width] divide obs by this (VecDriveEnv normalisation), NULL = raw */
  int32_t auto_reset;        /* VecDriveEnv semantics: reset finished worlds */
  int32_t serial;            /* step serial number recorded in the episode ring */
  int32_t *sel_idx;          /* debug/parity: [n_rows, max_agents_obs+max_road_points_obs] selected ids, or NULL */
  int32_t reserved0;
  /* optional cudaEvent_t recorded on the stream: before the step kernel,
   * between step and observation kernels, after the observation kernel */
  void *events[3];
} ds_step_args;

typedef struct ds_handle ds_handle;

int ds_abi_version(void);
/* 1 when the LiDAR / view-cone observation kernel is built in */
int ds_lidar_supported(void);
/* sizeof(ds_config), sizeof(ds_tables), sizeof(ds_state), sizeof(ds_step_args) */
void ds_struct_sizes(int64_t out[4]);
const char *ds_last_error(void);

/* Bind packed world tables + mutable state (device pointers, caller-owned)
 * and a validated config to a handle: replaces SimBatch.__init__
 * (engine.py:591-624) over the World.__init__ tables (engine.py:173-314).
 * Rejects unknown dynamics / collision behaviour / sensor modes like
 * SimConfig / ObsConfig (engine.py:59-67, observation.py:61-67). */
int ds_create(const ds_tables *tables, const ds_config *cfg, ds_state *state,
              int device, ds_handle **out);
/* SimBatch.close (engine.py:669-671); frees only the handle. */
int ds_destroy(ds_handle *h);

/* Reset the worlds whose world_mask[w] != 0 (device [n_worlds] u8; NULL = all)
 * and write their observation rows; rewards/dones rows of those worlds are
 * zeroed (engine.py:657-662). */
int ds_reset(ds_handle *h, const uint8_t *world_mask, void *obs, float *rewards,
             uint8_t *dones, const float *obs_scale, int32_t *sel_idx,
             void *stream);

/* SimBatch.step (engine.py:626-649): World.step (engine.py:357-498) of every
 * world -- dynamics, replay, collisions, goal / removal / horizon -- then
 * _fill_obs (engine.py:500-512); with auto_reset, VecDriveEnv.step's reset of
 * finished worlds (env.py:95-124).  Two kernels on `stream`, no host sync.
 * Row-count mismatches are the caller's ActionCountMismatch (engine.py:37-38,
 * 629-631). */
int ds_step(ds_handle *h, const ds_step_args *args, void *stream);

/* Recompute observations from the current state only (World.observe). */
int ds_observe(ds_handle *h, const uint8_t *world_mask, void *obs,
               const float *obs_scale, int32_t *sel_idx, void *stream);

/* Observation buffer format for every later ds_step / ds_reset / ds_observe
 * of this handle: element type DS_OBS_F32 (default) or DS_OBS_BF16 and the
 * row stride in elements (0 = obs_width; otherwise >= obs_width).  Pad
 * columns [obs_width, row_stride) are written as zeros, so a bf16 buffer
 * with a stride padded to a multiple of 8 feeds a policy GEMM directly
 * (no cast, 16-B aligned rows).  The reference returns float64 rows
 * (engine.py:603-608); VecDriveEnv divides them by the scale (env.py:121). */
int ds_set_obs_format(ds_handle *h, int dtype, int row_stride);

/* Categorical sample per row by Gumbel-max: out[r] = argmax_j(logits[r, j] +
 * G(seed, counter, r, j)), G standard Gumbel noise from a counter-based hash
 * (deterministic for (seed, counter)).  logits: device [rows, ld] float32
 * (dtype DS_OBS_F32) or bfloat16 (DS_OBS_BF16), first n columns used.  The
 * reference trainer samples torch.distributions.Categorical(logits)
 * (ippo.py:136-142); this is the in-loop sampler of the device rollout. */
int ds_sample_categorical(const void *logits, int dtype, int64_t rows, int32_t n, int64_t ld,
                          uint64_t seed, uint64_t counter, int32_t *out, void *stream);

/* Copy the handle's sticky status word (DS_STATUS_* bits) to host *out,
 * optionally clearing it; synchronises `stream`.  *out = 0 when the state
 * has no status word. */
int ds_status(ds_handle *h, uint32_t *out, int clear, void *stream);

/* Gumbel noise of raw 32-bit hash values, out[i] = -log(-log u(bits[i])) with
 * u = (2 (bits >> 9) + 1) 2^-24 strictly inside (0, 1): the noise function
 * of ds_sample_categorical, exposed so tests can feed it the extreme hash
 * values.  bits, out: device arrays of n elements. */
int ds_gumbel_noise(const uint32_t *bits, int64_t n, float *out, void *stream);

/* goal_seek policy (make_policy("goal_seek"), engine.py:554-574): actions
 * [n_rows, 2] float32 (accel, steer) for every controlled row from the
 * handle's current device state -- proportional steer-to-goal, speed capped
 * by the distance to the goal -- written to device `actions` on `stream`,
 * ready for ds_step.  Stream-ordered, no host sync. */
int ds_goal_seek(ds_handle *h, float *actions, void *stream);

/* Batched polyline decimation (preprocess, scenario.py:387-411, with
 * decimate_polyline, geometry.py:84-127): for every polyline p (points
 * [poly_off[p], poly_off[p+1]) of the device FP64 arrays x, y) remove
 * interior points by iterative smallest-triangle-area removal (ties: smaller
 * index) while the minimum area is < threshold; keep[i] = 1 for survivors.
 * Polylines with skip[p] != 0 (stop signs), fewer than 3 points, or
 * threshold <= 0 are kept whole.  scratch: device buffer of
 * ds_decimate_scratch_bytes(n_points) bytes, 8-byte aligned. */
int64_t ds_decimate_scratch_bytes(int64_t n_points);
int ds_decimate_polylines(const double *x, const double *y, const int64_t *poly_off,
                          int64_t n_poly, const uint8_t *skip, double threshold, uint8_t *keep,
                          void *scratch, int64_t n_points, void *stream);

/* Copy up to max_records ring entries (6 int32 each) to host memory `out`,
 * in ring order, reset the ring, and return the count in *n_out.
 * Synchronises `stream`.  Returns DS_E_OVERFLOW if records were lost. */
int ds_episode_drain(ds_handle *h, int32_t *out, int32_t max_records,
                     int32_t *n_out, void *stream);

/* Host helpers (CPU, exact restatements of the scalar libm calls used by
 * World.__init__; used by the packer). */
int ds_host_hypot_libm(const double *x, const double *y, int64_t n, double *out);
int ds_host_hypot_cpython(const double *x, const double *y, int64_t n, double *out);
int ds_host_hypot_port(const double *x, const double *y, int64_t n, double *out);
int ds_host_wrap_port(const double *x, int64_t n, double *out);
int ds_host_road_headings(const double *x, const double *y, const int64_t *poly_pt_off,
                          int64_t n_poly, double *out);

#ifdef __cplusplus
}
#endif
#endif /* DRIVESIM_B200_H */
