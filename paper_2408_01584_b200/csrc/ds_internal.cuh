// ds_internal.cuh -- handle layout and kernel launchers shared by the .cu files.
#pragma once

#include <cuda_runtime.h>

#include "../../include/drivesim_b200.h"
#include "ds_math.cuh"

struct ds_handle {
  ds_tables tab;
  ds_config cfg;
  ds_state st;
  int device;
  int num_sms;
  int obs_width;
  int step_threads;     // threads per world CTA in the step kernel
  size_t step_smem;     // dynamic shared memory of the step kernel
  int obs_warps;        // warps per world CTA in the observation kernel
  int obs_shared_pts;   // 1: road points staged in shared memory
  size_t obs_smem;
  int obs_dtype;        // DS_OBS_F32 / DS_OBS_BF16
  int obs_stride;       // elements per observation row (>= obs_width)
  uint32_t ring_read;   // host mirror of entries already drained
  // per-world strides when every world has the same number of agents /
  // rows / road points (offset[w] = w * stride; 0: ragged): the observation
  // kernel then forms its offsets without a dependent load
  int64_t uni_a, uni_c, uni_p, uni_r;
};

namespace ds {

// Uniform per-world strides of the CSR offsets (0: ragged, read the offsets);
// see ds_handle::uni_*
struct WorldStrides {
  int64_t a, c, r;
  __device__ __forceinline__ int64_t a0(const ds_tables &T, int w) const { return a ? w * a : T.a_off[w]; }
  __device__ __forceinline__ int64_t a1(const ds_tables &T, int w) const { return a ? (w + 1) * a : T.a_off[w + 1]; }
  __device__ __forceinline__ int64_t c0(const ds_tables &T, int w) const { return c ? w * c : T.c_off[w]; }
  __device__ __forceinline__ int64_t c1(const ds_tables &T, int w) const { return c ? (w + 1) * c : T.c_off[w + 1]; }
  __device__ __forceinline__ int64_t r0(const ds_tables &T, int w) const { return r ? w * r : T.r_off[w]; }
};
inline WorldStrides world_strides(const ds_handle *h) { return WorldStrides{h->uni_a, h->uni_c, h->uni_r}; }

// Largest supported max_agents_obs / max_road_points_obs (selection set size).
constexpr int kSelCap = 128;

cudaError_t launch_step(const ds_handle *h, const ds_step_args *a, cudaStream_t s);
cudaError_t launch_reset(const ds_handle *h, const uint8_t *mask, float *rewards,
                         uint8_t *dones, cudaStream_t s);
cudaError_t launch_observe(const ds_handle *h, const uint8_t *mask, void *obs,
                           const float *scale, int32_t *sel_idx, cudaStream_t s);
void obs_plan(ds_handle *h, int max_dynamic_smem);
size_t lidar_smem_bytes(const ds_config &cfg, int max_agents, int obs_width);
int lidar_warps();
cudaError_t configure_lidar_kernels(int max_dynamic_smem);
cudaError_t launch_lidar(const ds_handle *h, const uint8_t *mask, void *obs, const float *scale,
                         cudaStream_t s);
cudaError_t launch_decimate(const double *x, const double *y, const int64_t *poly_off,
                            int64_t n_poly, const uint8_t *skip, double threshold, uint8_t *keep,
                            void *scratch, int64_t n_points, cudaStream_t s);
cudaError_t launch_sample(const void *logits, int dtype, int64_t rows, int n, int64_t ld,
                          uint64_t seed, uint64_t counter, int32_t *out, cudaStream_t s);
size_t step_smem_bytes(int max_agents);
cudaError_t launch_goal_seek(const ds_handle *h, float *out, cudaStream_t s);
cudaError_t launch_gumbel(const uint32_t *bits, int64_t n, float *out, cudaStream_t s);
cudaError_t configure_kernels(int max_dynamic_smem);
cudaError_t configure_step_kernels(int max_dynamic_smem);

}  // namespace ds
