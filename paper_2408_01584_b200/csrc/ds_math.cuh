// ds_math.cuh -- scalar FP64 helpers shared by the device kernels and the
// host helpers.  The whole library is compiled with --fmad=false /
// -ffp-contract=off: every a*b+c below is two roundings, exactly like the
// reference's numba kernels (no fast-math, pkg/src/drivesim/_fastpath.py).
#pragma once

#include <math.h>
#include <stdint.h>

#ifdef __CUDACC__
#define DS_HD __host__ __device__ __forceinline__
#define DS_HD_COLD static __host__ __device__ __noinline__
#else
#define DS_HD static inline
#define DS_HD_COLD static
#endif

namespace ds {

constexpr double kPi = 3.141592653589793;      // math.pi
constexpr double kTwoPi = 6.283185307179586;   // 2.0 * math.pi (exact doubling)

// Angle wrap of _fastpath._wrap (fp:206-212) / geometry.wrap_angle_arr
// (geo:70-72): r = (theta + pi) mod 2pi - pi with Python's floor-mod sign
// rule, then +2pi if r <= -pi.  fmod is exact, so this is bit-reproducible.
// floor-mod of a by 2pi outside [-2pi, 4pi) (fmod, then the sign rule)
DS_HD double wrap_far(double a) {
  double r = fmod(a, kTwoPi);
  if (r != 0.0) {
    if (r < 0.0) r += kTwoPi;
  } else {
    r = 0.0;  // copysign(0, 2pi)
  }
  return r;
}

// Branch-free on [-2pi, 4pi): fmod(a, 2pi) is a, a - 2pi (exact, Sterbenz)
// or a (a < 0, then the sign rule adds 2pi: one rounding, a + 2pi).
DS_HD double wrap(double theta) {
  const double a = theta + kPi;
  double r = a >= kTwoPi ? a - kTwoPi : a;
  r = a < 0.0 ? a + kTwoPi : r;
  if (!(a >= -kTwoPi && a < 2.0 * kTwoPi)) r = wrap_far(a);
  r = r - kPi;
  return r <= -kPi ? r + kTwoPi : r;
}

// np.mod(a, 2 pi) (numpy's npy_divmod: fmod, then +2pi for a negative
// remainder; fmod is exact), the first half of wrap() above.
DS_HD double floor_mod_2pi(double a) {
  if (a >= 0.0 && a < kTwoPi) return a;
  if (a >= kTwoPi && a < 2.0 * kTwoPi) return a - kTwoPi;
  if (a < 0.0 && a >= -kTwoPi) return a + kTwoPi;
  double r = fmod(a, kTwoPi);
  if (r != 0.0) {
    if (r < 0.0) r += kTwoPi;
  } else {
    r = 0.0;
  }
  return r;
}

// hypot with the exact arithmetic of glibc 2.39's non-FMA kernel
// (sysdeps/ieee754/dbl-64/e_hypot.c), which is what numba's math.hypot,
// numpy's np.hypot and the oracle's libm call resolve to on this image
// (verified bit-for-bit in tests/test_host_math.py).  CUDA's own hypot is a
// different (<=2 ulp) algorithm, which would flip exact distance ties and
// radius knife edges; this port makes device distances equal to the
// reference's bit for bit.
DS_HD double hypot_kernel(double ax, double ay) {
  double h = sqrt(ax * ax + ay * ay);
  double t1, t2;
  if (h <= 2.0 * ay) {
    double delta = h - ay;
    t1 = ax * (2.0 * delta - ax);
    t2 = (delta - 2.0 * (ax - ay)) * delta;
  } else {
    double delta = h - ax;
    t1 = 2.0 * delta * (ax - 2.0 * ay);
    t2 = (4.0 * delta - ay) * ay + delta * delta;
  }
  h -= (t1 + t2) / (2.0 * h);
  return h;
}

// scaled / non-finite / degenerate cases of hypot() below (out of line: they
// are cold, and keeping one inline copy of the common path keeps the
// observation kernels' code small)
DS_HD_COLD double hypot_slow(double x, double y) {
  const double kScale = 0x1p-600, kLarge = 0x1p+511, kTiny = 0x1p-511, kEps = 0x1p-54;
  if (!isfinite(x) || !isfinite(y)) {
    if ((isinf(x) || isinf(y)) && !isnan(x) && !isnan(y)) return INFINITY;
    if (isinf(x) || isinf(y)) return INFINITY;  // hypot(inf, nan) = inf
    return x + y;
  }
  x = fabs(x);
  y = fabs(y);
  double ax = x < y ? y : x;
  double ay = x < y ? x : y;
  if (ax > kLarge) {
    if (ay <= ax * kEps) return ax + ay;
    return hypot_kernel(ax * kScale, ay * kScale) / kScale;
  }
  if (ay < kTiny) {
    if (ax >= ay / kEps) return ax + ay;
    ax = hypot_kernel(ax / kScale, ay / kScale) * kScale;
    return ax;
  }
  if (ay <= ax * kEps) return ax + ay;
  return hypot_kernel(ax, ay);
}

DS_HD double hypot(double x, double y) {
  // common case (finite, unscaled, non-degenerate): glibc's branch order
  // reaches hypot_kernel(ax, ay) directly; NaN fails every comparison
  const double kLarge = 0x1p+511, kTiny = 0x1p-511, kEps = 0x1p-54;
  const double fx = fabs(x), fy = fabs(y);
  const double ax = fx < fy ? fy : fx, ay = fx < fy ? fx : fy;
  if (ax <= kLarge && ay >= kTiny && ay > ax * kEps) return hypot_kernel(ax, ay);
  return hypot_slow(x, y);
}

DS_HD double clip(double v, double lo, double hi) {
  // Python min(max(v, lo), hi) as in classic_core (fp:323-333)
  double m = (lo > v) ? lo : v;
  return (m > hi) ? hi : m;
}

}  // namespace ds
