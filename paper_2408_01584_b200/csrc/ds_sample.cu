// ds_sample.cu -- in-loop categorical action sampler of the device rollout
// (the reference trainer samples torch.distributions.Categorical(logits),
// pkg/rl/src/drivesim_rl/ippo.py:136-142).
//
// Gumbel-max: out[r] = argmax_j (logits[r, j] + G_rj), G_rj = -log(-log u_rj)
// with u_rj in (0, 1) from a counter-based hash of (seed, counter, r, j), so a
// rollout is reproducible from (seed, step) alone and needs no RNG state.
// One warp per row, lanes strided over the columns, warp argmax (ties to the
// smaller column).  One launch replaces the rand / log / log / add / argmax
// chain of the eager torch sampler.
#include <cuda_bf16.h>

#include "ds_internal.cuh"

namespace ds {

namespace {

constexpr int kSampleWarps = 8;

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

// 32-bit integer hash (lowbias32): one per logit; the 64-bit key and the row
// are folded into a per-row seed once
__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352du;
  x ^= x >> 15;
  x *= 0x846ca68bu;
  x ^= x >> 16;
  return x;
}

__device__ __forceinline__ uint32_t row_seed(uint64_t key, uint64_t r) {
  return hash32((uint32_t)key ^ hash32((uint32_t)(key >> 32) ^ hash32((uint32_t)r) ^
                                       (uint32_t)(r >> 32)));
}

__device__ __forceinline__ uint32_t hash_bits(uint32_t seed, uint32_t j) {
  return hash32(seed + j * 0x9e3779b9u);
}

// Gumbel noise -log(-log u) of one 32-bit hash.  u = (2m + 1) 2^-24 from the
// top 23 bits m: exactly representable and strictly inside (0, 1)
// (2^-24 <= u <= 1 - 2^-24).  The exponential variate -log u is formed as
// -log1p(-w) from w = 1 - u = (2^24 - 2m - 1) 2^-24, also exact, so it stays
// accurate (and > 0) right up to u = 1 - 2^-24 where -log u ~ 6e-8; the
// outer log is the accurate logf, never the fast __logf.
__device__ __forceinline__ float gumbel_of_bits(uint32_t h) {
  const uint32_t m = h >> 9;
  const float w = (float)(16777215u - 2u * m) * 5.9604644775390625e-8f;
  const float e = -log1pf(-w);
  return -logf(e);
}

template <typename T>
__device__ __forceinline__ float load_logit(const T *p);
template <>
__device__ __forceinline__ float load_logit<float>(const float *p) { return *p; }
template <>
__device__ __forceinline__ float load_logit<__nv_bfloat16>(const __nv_bfloat16 *p) {
  return __bfloat162float(*p);
}

template <typename T>
__global__ void __launch_bounds__(kSampleWarps * 32) sample_kernel(const T *logits, int64_t rows,
                                                                   int n, int64_t ld,
                                                                   uint64_t key, int32_t *out) {
  const int lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * kSampleWarps + (threadIdx.x >> 5);
  if (r >= rows) return;
  const T *row = logits + r * ld;
  float best = -INFINITY;
  int arg = 0x7fffffff;
  const uint32_t seed = row_seed(key, (uint64_t)r);
  for (int j = lane; j < n; j += 32) {
    const float v = load_logit(row + j) + gumbel_of_bits(hash_bits(seed, (uint32_t)j));
    if (v > best || (v == best && j < arg) || arg == 0x7fffffff) {
      best = v;
      arg = j;
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const float ob = __shfl_xor_sync(0xffffffffu, best, off);
    const int oa = __shfl_xor_sync(0xffffffffu, arg, off);
    if (ob > best || (ob == best && oa < arg)) {
      best = ob;
      arg = oa;
    }
  }
  if (lane == 0) out[r] = arg;
}

__global__ void gumbel_kernel(const uint32_t *bits, int64_t n, float *out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = gumbel_of_bits(bits[i]);
}

}  // namespace

cudaError_t launch_gumbel(const uint32_t *bits, int64_t n, float *out, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  gumbel_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(bits, n, out);
  return cudaGetLastError();
}

cudaError_t launch_sample(const void *logits, int dtype, int64_t rows, int n, int64_t ld,
                          uint64_t seed, uint64_t counter, int32_t *out, cudaStream_t s) {
  const uint64_t key = mix64(seed ^ mix64(counter + 0x632be59bd9b4e019ull));
  const int64_t blocks = (rows + kSampleWarps - 1) / kSampleWarps;
  if (dtype == DS_OBS_BF16)
    sample_kernel<__nv_bfloat16><<<(unsigned)blocks, kSampleWarps * 32, 0, s>>>(
        static_cast<const __nv_bfloat16 *>(logits), rows, n, ld, key, out);
  else
    sample_kernel<float><<<(unsigned)blocks, kSampleWarps * 32, 0, s>>>(
        static_cast<const float *>(logits), rows, n, ld, key, out);
  return cudaGetLastError();
}

}  // namespace ds
