// ds_obs_out.cuh -- write-out of one staged observation row (shared memory,
// float) into the caller's observation buffer in the handle's format:
// float32 (the reference's values rounded to float32) or bfloat16 (round to
// nearest even, the format an in-loop bf16 policy consumes), with a row
// stride >= the observation width whose pad columns are written as zeros.
#pragma once

#include <cuda_bf16.h>

#include "ds_internal.cuh"

namespace ds {

struct ObsOut {
  void *base;
  int dtype;    // DS_OBS_F32 / DS_OBS_BF16
  int stride;   // elements per row
};

// float phase (0..3) modulo 16 B that the staged row should have so that the
// float32 write-out can use 16-B vector stores (bf16 rows want phase 0)
__device__ __forceinline__ int out_row_phase(const ObsOut &o, int64_t orow) {
  if (o.dtype != DS_OBS_F32) return 0;
  const float *out = static_cast<const float *>(o.base) + orow * (int64_t)o.stride;
  return (int)((reinterpret_cast<uintptr_t>(out) >> 2) & 3);
}

// normalisation by the env's per-column divisors (env.py:50-63): IEEE
// round-to-nearest division, so a float32 result stays within 1.5 ulp of the
// reference's float64 quotient (the staged value's own rounding plus one),
// and a bfloat16 row is exactly the float32 row rounded to bf16
__device__ __forceinline__ float scaled(const float *row, const float *scale, int c) {
  return scale ? __fdiv_rn(row[c], scale[c]) : row[c];
}

// Bulk (TMA engine) shared -> global store of a staged row's 16-B aligned
// body: one instruction of one lane instead of a load / store per float4.
// The issuing lane must wait for the source to be read (bulk_row_wait)
// before the staging buffer is written again, and before the CTA exits.
__device__ __forceinline__ void bulk_row_store(float *gdst, const float *ssrc, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst),
               "r"((uint32_t)__cvta_generic_to_shared(ssrc)), "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_row_wait() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}


// Warp-collective float32 write-out of a staged row whose 16-B phase matches
// the output row's, without normalisation: head / tail floats by single
// stores of lanes 0-3 / 4-7, the aligned body by one bulk store of lane 0
// (call bulk_row_wait on lane 0 before reusing `row`).
__device__ __forceinline__ void write_row_bulk(const ObsOut &o, int64_t orow, const float *row,
                                               int width, int lane) {
  float *out = static_cast<float *>(o.base) + orow * (int64_t)o.stride;
  const int ph = (int)((reinterpret_cast<uintptr_t>(out) >> 2) & 3);
  const int head = min((4 - ph) & 3, width);
  const int nvec = (width - head) >> 2;
  const int tail0 = head + 4 * nvec;
  const int c = lane < 4 ? lane : tail0 + lane - 4;
  if (lane < 4 ? lane < head : (lane < 8 && c < width)) out[c] = row[c];
  // the staged row was written through the generic proxy: every writer
  // fences toward the async proxy, then one lane issues the copy
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  if (lane == 0 && nvec > 0) bulk_row_store(out + head, row + head, (uint32_t)nvec * 16u);
  if (o.stride > width) {
#pragma unroll 1
    for (int q = width + lane; q < o.stride; q += 32) out[q] = 0.0f;
  }
}

// Warp-collective: row[0, width) (divided by scale[c] when scale != NULL) to
// output row orow, zeros in [width, stride).
__device__ __forceinline__ void write_row(const ObsOut &o, int64_t orow, const float *row,
                                          int width, const float *scale, int lane) {
  if (o.dtype == DS_OBS_F32) {
    float *out = static_cast<float *>(o.base) + orow * (int64_t)o.stride;
    const int ph = (int)((reinterpret_cast<uintptr_t>(out) >> 2) & 3);
    if (((reinterpret_cast<uintptr_t>(row) >> 2) & 3) != (uintptr_t)ph) {
      // phases differ (callers stage rows phase-matched): scalar copy
#pragma unroll 1
      for (int c = lane; c < width; c += 32) out[c] = scaled(row, scale, c);
    } else {
      // <= 3 head floats up to the 16-B boundary, float4 body, <= 3 tail
      // floats: head and tail are one predicated store each (lanes 0-3 /
      // 4-7), the body one 16-B store per lane and pass
      const int head = min((4 - ph) & 3, width);
      const int nvec = (width - head) >> 2;
      const int tail0 = head + 4 * nvec;
      const int c = lane < 4 ? lane : tail0 + lane - 4;
      if (lane < 4 ? lane < head : (lane < 8 && c < width)) out[c] = scaled(row, scale, c);
      const float4 *rv = reinterpret_cast<const float4 *>(row + head) + lane;
      float4 *ov = reinterpret_cast<float4 *>(out + head) + lane;
      const int nv = nvec > lane ? (nvec - lane + 31) >> 5 : 0;   // this lane's vectors
      if (!scale) {
#pragma unroll 4
        for (int q = 0; q < nv; ++q) ov[32 * q] = rv[32 * q];
      } else {
#pragma unroll 1
        for (int q = 0; q < nv; ++q) {
          float4 x = rv[32 * q];
          const float *sc = scale + head + 4 * (lane + 32 * q);
          x.x = __fdiv_rn(x.x, sc[0]);
          x.y = __fdiv_rn(x.y, sc[1]);
          x.z = __fdiv_rn(x.z, sc[2]);
          x.w = __fdiv_rn(x.w, sc[3]);
          ov[32 * q] = x;
        }
      }
    }
    if (o.stride > width) {
#pragma unroll 1
      for (int c = width + lane; c < o.stride; c += 32) out[c] = 0.0f;
    }
    return;
  }
  __nv_bfloat16 *out = static_cast<__nv_bfloat16 *>(o.base) + orow * (int64_t)o.stride;
  const bool vec = ((reinterpret_cast<uintptr_t>(out) | reinterpret_cast<uintptr_t>(row)) & 15) == 0;
  const int nvec = vec ? width >> 3 : 0;
#pragma unroll 1
  for (int v = lane; v < nvec; v += 32) {
    float4 a = reinterpret_cast<const float4 *>(row)[2 * v];
    float4 b = reinterpret_cast<const float4 *>(row)[2 * v + 1];
    if (scale) {
      const float *sc = scale + 8 * v;
      a.x = __fdiv_rn(a.x, sc[0]);
      a.y = __fdiv_rn(a.y, sc[1]);
      a.z = __fdiv_rn(a.z, sc[2]);
      a.w = __fdiv_rn(a.w, sc[3]);
      b.x = __fdiv_rn(b.x, sc[4]);
      b.y = __fdiv_rn(b.y, sc[5]);
      b.z = __fdiv_rn(b.z, sc[6]);
      b.w = __fdiv_rn(b.w, sc[7]);
    }
    __nv_bfloat162 q[4] = {__floats2bfloat162_rn(a.x, a.y), __floats2bfloat162_rn(a.z, a.w),
                           __floats2bfloat162_rn(b.x, b.y), __floats2bfloat162_rn(b.z, b.w)};
    reinterpret_cast<uint4 *>(out)[v] = *reinterpret_cast<const uint4 *>(q);
  }
#pragma unroll 1
  for (int c = 8 * nvec + lane; c < width; c += 32) out[c] = __float2bfloat16_rn(scaled(row, scale, c));
#pragma unroll 1
  for (int c = width + lane; c < o.stride; c += 32) out[c] = __float2bfloat16_rn(0.0f);
}

// Warp-collective: a zero output row (done / removed agents, engine.py:502-512).
__device__ __forceinline__ void zero_row(const ObsOut &o, int64_t orow, int lane) {
  const size_t esz = o.dtype == DS_OBS_F32 ? 4 : 2;
  unsigned char *out = static_cast<unsigned char *>(o.base) + (size_t)orow * o.stride * esz;
  const size_t bytes = (size_t)o.stride * esz;
  const size_t head = ((16 - (reinterpret_cast<uintptr_t>(out) & 15)) & 15) < bytes
                          ? ((16 - (reinterpret_cast<uintptr_t>(out) & 15)) & 15)
                          : bytes;
  const size_t nvec = (bytes - head) >> 4;
  // element-sized head/tail stores (the buffer is element aligned)
  for (size_t c = lane * esz; c < head; c += 32 * esz) {
    if (esz == 4) *reinterpret_cast<float *>(out + c) = 0.0f;
    else *reinterpret_cast<uint16_t *>(out + c) = 0;
  }
#pragma unroll 1
  for (size_t v = lane; v < nvec; v += 32)
    reinterpret_cast<uint4 *>(out + head)[v] = make_uint4(0u, 0u, 0u, 0u);
  for (size_t c = head + 16 * nvec + lane * esz; c < bytes; c += 32 * esz) {
    if (esz == 4) *reinterpret_cast<float *>(out + c) = 0.0f;
    else *reinterpret_cast<uint16_t *>(out + c) = 0;
  }
}

}  // namespace ds
