// ds_obs.cu -- radial observation kernel (World._fill_obs, engine.py:500-512;
// fill_radial / radial_fill_core, observation.py:145-210, _fastpath.py:214-302).
//
// Layout: one CTA per world, one warp per controlled agent (rows handed to
// warps dynamically).  The world's road points (float2 relative to the world
// grid origin, 8 B/point) arrive in shared memory by one TMA bulk copy while
// the threads stage the agent tables and every per-agent selection parameter;
// each warp then scans them.  Road candidates come from the world's uniform
// grid: lane l owns cell row iy0 + l of the search disc, whose covered cells
// form ONE contiguous, cell-sorted point range.
//
// Exact top-k (the reference's insertion sort = ascending (distance, index)):
//  keys    every candidate gets a cheap float key a ~ d^2 with a proven
//          absolute error bound D (|a - d^2| <= D);
//  roads   a 128-bucket histogram of a over [0, rho^2] (rho: a hint-narrowed
//          radius that provably covers the k nearest, or the full disc)
//          gives the threshold bucket b*; the candidates of buckets <= b*+1
//          are counting-sort scattered into a small set G (about k+1
//          entries), sorted by odd-even transposition rounds (G is already
//          block-sorted by bucket), and each sorted position is the
//          reference's rank unless a neighbour lies within 2D of it (a near
//          tie) or its key may lie beyond the radius; only those get the
//          glibc-exact FP64 hypot (ds_math.cuh) and an exact (d, id) rank
//          inside their near-tie cluster.  Elements beyond b*+1 cannot reach
//          rank k;
//  partners at most 32 candidates, ranked by counting key compares over the
//          warp, the same neighbour checks.
// A set the fast paths cannot rank (G beyond its capacity, a key bound too
// loose for the bucket width, more than 32 partners, a near tie among the
// partners) falls back to the reference's serial insertion -- exact by
// construction.  Rows are staged in shared memory and leave by TMA bulk
// stores.
#include "ds_internal.cuh"
#include "ds_obs_out.cuh"
#include "ds_rows.cuh"

namespace ds {

// Dev-only path counters (a build with -DDS_OBS_STATS; tools/obs_stats.py).
#ifdef DS_OBS_STATS
__device__ unsigned long long g_obs_stats[8];
#define OBS_STAT(i, v) \
  do { if (lane == 0) atomicAdd(&g_obs_stats[i], (unsigned long long)(v)); } while (0)
#else
#define OBS_STAT(i, v) \
  do { } while (0)
#endif
// Dev-only CTA timeline (a build with -DDS_OBS_TIMES; tools/obs_times.py):
// per world [sm, start, prologue end, end of warp 0..31's row loop, thread 0
// staged, after the prologue barrier]
#ifdef DS_OBS_TIMES
constexpr int kTimesW = 37;
__device__ unsigned long long g_obs_times[8192 * kTimesW];
__device__ unsigned int g_row_dur[8192 * 128];   // per (world, row < 128): row time (ns)
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#endif

constexpr unsigned kFull = 0xffffffffu;
constexpr int kNB = 128;       // histogram buckets
constexpr int kCandGlobal = 640;  // buffered pass-1 candidates (global-points variant)
constexpr int kCandShared = 224;  // (shared-points variant: hint-narrowed scans)
// warps per world CTA: as many as the shared memory allows (occupancy is what
// hides this kernel's latencies: 16 / 24 / 28 / 32 warps measured 2.82 /
// 2.53 / 2.28 / 2.16 ms at C3 in round 1; 28 / 30 / 32 measured 1.356 /
// 1.401 / 1.292 ms in round 2); 32 fits the default caps with 10k points.
// DS_OBS_WARPS: A/B builds only (tools/build_variant.sh)
#ifndef DS_OBS_WARPS
#define DS_OBS_WARPS 32
#endif
constexpr int kWarpsShared = DS_OBS_WARPS;
constexpr int kWarpsSharedSmall = 24;
// batches of >= 2 x #SMs worlds of <= 64 agents whose tables fit twice per
// SM: two 16-warp CTAs per SM (the same 32 warps, but one world's staging
// overlaps the other's rows; C2 obs 0.193 -> 0.190 ms)
constexpr int kWarpsSharedPair = 16;
constexpr int kSmemPerSM = 228 * 1024;
constexpr int kWarpsGlobal = 12;
constexpr int kAgentStride = 128;   // compile-time agent-table stride (AMAX)
// static shared memory of the radial kernel (mbarrier, per-warp rounding
// maxima, row counter): an upper bound for the launch plan
constexpr size_t kStaticSmem = 256;

__host__ __device__ constexpr int kmax_of(int cap_a, int cap_r) {
  return (cap_a > cap_r ? cap_a : cap_r) < 1 ? 1 : (cap_a > cap_r ? cap_a : cap_r);
}

// Capacity of the exactly ranked set G.
__host__ __device__ constexpr int gcap_of(int cap_a, int cap_r) {
  return kmax_of(cap_a, cap_r) + 48;
}

__host__ __device__ constexpr size_t al16(size_t v) { return (v + 15) & ~size_t(15); }

// Per-warp shared scratch (byte offsets).  The observation row is staged
// contiguously: [ego | partner slots] sit right before `hc`, and the road
// block (11 floats per slot) aliases [hc ..), which is dead once the road
// selection has produced sel_pl.  constexpr: with compile-time slot caps the
// whole layout folds into immediate offsets off one base register.
//   R1 = the pass-1 candidate buffer (ca keys, cp payloads), dead once
//        scattered into G; then the sorted G (sa keys, spl payloads) and the
//        exact ids sid
//   R2 = G in bucket order (ga keys, gpl payloads), dead once sorted; then
//        the exact distances se of the sorted G
struct WarpLayout {
  size_t row, hc, ca, cp, sa, spl, sid, ga, gpl, se, sf, road_end, sel_pl, psel, fr, total;
};

__host__ __device__ constexpr WarpLayout make_layout(int cap_a, int cap_r, bool buffered) {
  WarpLayout L{};
  const int km = kmax_of(cap_a, cap_r), gc = gcap_of(cap_a, cap_r);
  // the staged row may sit up to 3 floats before `row` (it is shifted so
  // that its 16-B phase matches the output row's, for float4 write-out)
  const size_t head = (size_t)(7 + 7 * cap_a) * sizeof(float);
  size_t o = al16(head) + 16;
  L.row = o - head;
  L.hc = o; o = al16(o + kNB * sizeof(uint32_t));
  const int cc = buffered ? kCandGlobal : kCandShared;
  const size_t g4 = al16((size_t)gc * 4);
  L.ca = o;
  L.cp = al16(o + cc * sizeof(float));
  const size_t cand_end = al16(L.cp + cc * sizeof(uint16_t));
  L.sa = o;
  L.spl = o + g4;
  L.sid = o + 2 * g4;
  o = cand_end > o + 3 * g4 ? cand_end : o + 3 * g4;
  L.ga = o;
  L.gpl = o + g4;
  L.se = o;
  o = o + 2 * g4 > al16(o + (size_t)gc * sizeof(double)) ? o + 2 * g4 : al16(o + (size_t)gc * sizeof(double));
  L.sf = o; o = al16(o + gc);
  const size_t road_end = al16(L.hc + (size_t)cap_r * 11 * sizeof(float));
  L.road_end = road_end;
  if (o < road_end) o = road_end;
  L.sel_pl = o; o = al16(o + km * sizeof(int));
  L.psel = o; o = al16(o + (cap_a > 0 ? cap_a : 1) * sizeof(int));   // partner picks
  L.fr = o; o = al16(o + 32 * sizeof(int));   // FlatRows compaction scratch
  L.total = o;
  return L;
}

__host__ __device__ inline WarpLayout warp_layout(const ds_config &c, bool buffered) {
  return make_layout(c.max_agents_obs, c.max_road_points_obs, buffered);
}

// Per-agent tables staged once per world (structure of arrays):
//   x, y, heading, speed, cos, sin (f64) | length, width (f32: only their
//   float32 values are observed) | ego block (7
//   floats, padded to 8) | road-selection parameters (RoadPre) | partner
//   key positions (float2, padded to 32) | flags (u16) | row -> local agent
//   (u16)
// RoadPre: everything the road selection of one agent needs that does not
// depend on the candidates, formed by one thread per agent in the prologue
// (instead of by every lane of the agent's warp):
//   a = (prx, pry, marg, Df): grid-relative float position, the RowGeo float
//       margin, Df >= D
//   b = (r2hi, inv_w, two_d, r2lo): the first histogram range
//   c = (D, rho): the key error bound and the covered radius
//   d = (iy0, nrows, flags): the disc's cell rows; flags 1 = restricted
//       (hint-narrowed), 2 = serial
struct AgentTabs {
  double *x, *y, *h, *v, *c, *s;
  float *l, *w;
  float *ego;
  float4 *pa, *pb;
  double2 *pc;
  int4 *pd;
  float2 *pxy;
  uint16_t *flg, *rloc;
};

__host__ __device__ constexpr int pad32(int n) { return (n + 31) & ~31; }

__host__ __device__ inline size_t agents_bytes(int amax) {
  return (size_t)amax * (6 * sizeof(double) + 2 * sizeof(float) + 8 * sizeof(float) +
                         3 * sizeof(float4) + sizeof(double2)) +
         (size_t)pad32(amax) * sizeof(float2) + al16((size_t)amax * sizeof(uint16_t)) * 2;
}

__device__ inline AgentTabs agent_tabs(unsigned char *base, int amax) {
  AgentTabs t;
  unsigned char *o = base;
  t.pa = reinterpret_cast<float4 *>(o); o += (size_t)amax * sizeof(float4);
  t.pb = reinterpret_cast<float4 *>(o); o += (size_t)amax * sizeof(float4);
  t.pc = reinterpret_cast<double2 *>(o); o += (size_t)amax * sizeof(double2);
  t.pd = reinterpret_cast<int4 *>(o); o += (size_t)amax * sizeof(int4);
  double *d = reinterpret_cast<double *>(o);
  t.x = d; t.y = d + amax; t.h = d + 2 * amax; t.v = d + 3 * amax; t.c = d + 4 * amax; t.s = d + 5 * amax;
  o += (size_t)amax * 6 * sizeof(double);
  t.l = reinterpret_cast<float *>(o); o += (size_t)amax * sizeof(float);
  t.w = reinterpret_cast<float *>(o); o += (size_t)amax * sizeof(float);
  t.ego = reinterpret_cast<float *>(o); o += (size_t)amax * 8 * sizeof(float);
  t.pxy = reinterpret_cast<float2 *>(o); o += (size_t)pad32(amax) * sizeof(float2);
  t.flg = reinterpret_cast<uint16_t *>(o); o += al16((size_t)amax * sizeof(uint16_t));
  t.rloc = reinterpret_cast<uint16_t *>(o);
  return t;
}

// road points: float2, +2 entries of slack so the bulk copy's 16-B aligned
// body can start at an odd point offset
__host__ __device__ inline size_t points_bytes(int max_points) {
  return al16((size_t)(max_points + 2) * sizeof(float2));
}

size_t obs_smem_bytes_shared(const ds_config &cfg, int max_agents, int max_points, int warps) {
  return agents_bytes(max_agents) + points_bytes(max_points) +
         warp_layout(cfg, false).total * warps;
}

size_t obs_smem_bytes_global(const ds_config &cfg, int max_agents) {
  return agents_bytes(max_agents) + warp_layout(cfg, true).total * kWarpsGlobal;
}

// Per-warp selection scratch: one base pointer plus the layout's offsets
// (compile-time for the default caps, so every array is base + immediate).
struct Sel {
  unsigned char *wb;
  WarpLayout L;
  int gcap, ccap;
  __device__ __forceinline__ uint32_t *hc() const { return reinterpret_cast<uint32_t *>(wb + L.hc); }
  __device__ __forceinline__ float *ca() const { return reinterpret_cast<float *>(wb + L.ca); }
  __device__ __forceinline__ uint16_t *cp() const { return reinterpret_cast<uint16_t *>(wb + L.cp); }
  __device__ __forceinline__ float *ga() const { return reinterpret_cast<float *>(wb + L.ga); }
  __device__ __forceinline__ int *gpl() const { return reinterpret_cast<int *>(wb + L.gpl); }
  __device__ __forceinline__ float *sa() const { return reinterpret_cast<float *>(wb + L.sa); }
  __device__ __forceinline__ int *spl() const { return reinterpret_cast<int *>(wb + L.spl); }
  __device__ __forceinline__ int *sid() const { return reinterpret_cast<int *>(wb + L.sid); }
  __device__ __forceinline__ double *se() const { return reinterpret_cast<double *>(wb + L.se); }
  __device__ __forceinline__ uint8_t *sf() const { return wb + L.sf; }
  __device__ __forceinline__ int *sel_pl() const { return reinterpret_cast<int *>(wb + L.sel_pl); }
};

__device__ __forceinline__ bool key_less(double da, int ia, double db, int ib) {
  return da < db || (da == db && ia < ib);
}

__device__ __forceinline__ int bucket_of(float a, float inv_w) {
  const int b = (int)(a * inv_w);
  return b < kNB ? b : kNB - 1;
}

// Asynchronous copies.  The world's road points arrive by one bulk copy (TMA
// engine, completion counted on an mbarrier) while the threads stage the
// agent tables; the selected road-point records of a row are fetched with
// 16-B cp.async into dead scratch while the partner slots are formed.
__device__ __forceinline__ uint32_t sm_addr(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sm_addr(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sm_addr(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sm_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(sm_addr(bar)), "r"(parity)
        : "memory");
  } while (!done);
}
// global -> shared bulk copy (16-B aligned addresses, size a multiple of 16)
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          sm_addr(dst)),
      "l"(src), "r"(bytes), "r"(sm_addr(bar))
      : "memory");
}
__device__ __forceinline__ void cp_async16(void *dst, const void *src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sm_addr(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;" ::: "memory");
}

// ---------------------------------------------------------------------------
// Candidate sources.  visit(r2hi, lane, fn) calls fn(ok, key, payload)
// warp-collectively, one candidate per lane; exact(payload, id) returns the
// reference's distance (glibc hypot port) and the tie-break index.
// ---------------------------------------------------------------------------

// Agents of the world (partner slots, fp:240-272): keys from float2
// positions relative to the grid origin (shared memory, padded to a whole
// number of warps; absent / removed agents and the padding hold a far
// sentinel whose key is +inf), exact distances from the FP64 tables.
// |a - d^2| <= D as for the road points, with E = both positions' float
// rounding (the world's largest, measured in the prologue) + the float
// subtraction.
struct PartnerSrc {
  const float2 *pxy;
  const double *x, *y;
  int npad, self;
  float prx, pry;
  double px, py;
  __device__ __forceinline__ int pbase() const { return 0; }
  __device__ __forceinline__ bool small_payload() const { return true; }
  template <class F>
  __device__ __forceinline__ void visit(float r2hi, int lane, F &&fn) const {
    #pragma unroll 1
    for (int f0 = 0; f0 < npad; f0 += 32) {
      const int f = f0 + lane;
      const float2 q = pxy[f];
      const float dx = q.x - prx, dy = q.y - pry;
      const float a = fmaf(dx, dx, dy * dy);
      fn(f != self && a <= r2hi, a, f);
    }
  }
  __device__ __forceinline__ double exact(int pl, int &id) const {
    id = pl;
    return hypot(x[pl] - px, y[pl] - py);
  }
  __device__ __forceinline__ void restrict_to(double, int) {}
};

// Road points staged in shared memory as float2 relative to the grid origin.
// dx = fl32(xr - pr) with |xr - (x - x0)| <= eps_p (host-measured) and
// |pr - (px - x0)| measured per agent: see the bound D in the kernel.
struct RoadSrcShared {
  const float2 *pts;                 // shared, world-relative index
  const ds_point_rec *__restrict__ rec;
  int p0;
  float prx, pry;
  double px, py;
  const RowGeo *geo;
  int *fscr;
  FlatRows rows;
  __device__ __forceinline__ void cover(double rho, int lane) {
    int b, c;
    geo->range((float)rho, lane, b, c);
    rows.build(b - p0, c, lane, fscr);
  }
  // cover() from the raw cell-table values of RowGeo::range_issue_async
  __device__ __forceinline__ void cover_raw(int v0, int v1, int lane) {
    rows.build(v0 - p0, v1 - v0, lane, fscr);
  }
  __device__ __forceinline__ void restrict_to(double rho, int lane) { cover(rho, lane); }
  __device__ __forceinline__ int pbase() const { return 0; }
  __device__ __forceinline__ bool small_payload() const { return true; }
  template <class F>
  __device__ __forceinline__ void visit(float r2hi, int lane, F &&fn) const {
    #pragma unroll 1
    for (int f0 = 0; f0 < rows.total; f0 += 32) {
      const bool in = f0 + lane < rows.total;
      const int sm = rows.map(f0, lane);
      const int s = in ? sm : 0;   // branch-free: lanes past the end read point 0
      const float2 p = pts[s];
      const float dx = p.x - prx, dy = p.y - pry;
      const float a = fmaf(dx, dx, dy * dy);
      const bool ok = in && a <= r2hi;
      fn(ok, a, s);
    }
  }
  __device__ __forceinline__ double exact(int pl, int &id) const {
    const ds_point_rec &q = rec[p0 + pl];
    id = q.id;
    return hypot(q.x - px, q.y - py);
  }
};

// Road points read from global memory (worlds too large for shared memory).
struct RoadSrcGlobal {
  const double *__restrict__ gx, *__restrict__ gy;
  const int *__restrict__ gid;
  int p0, np;
  double px, py;
  const RowGeo *geo;
  int *fscr;
  FlatRows rows;
  __device__ __forceinline__ void cover(double rho, int lane) {
    int b, c;
    geo->range((float)rho, lane, b, c);
    rows.build(b, c, lane, fscr);
  }
  __device__ __forceinline__ void restrict_to(double rho, int lane) { cover(rho, lane); }
  __device__ __forceinline__ int pbase() const { return p0; }
  __device__ __forceinline__ bool small_payload() const { return np <= 0xffff; }
  template <class F>
  __device__ __forceinline__ void visit(float r2hi, int lane, F &&fn) const {
    #pragma unroll 1
    for (int f0 = 0; f0 < rows.total; f0 += 32) {
      const int s = rows.map(f0, lane);
      bool ok = f0 + lane < rows.total;
      float a = 0.0f;
      if (ok) {
        const double dx = gx[s] - px, dy = gy[s] - py;
        a = (float)fma(dx, dx, dy * dy);
        ok = a <= r2hi;
      }
      fn(ok, a, s);
    }
  }
  __device__ __forceinline__ double exact(int pl, int &id) const {
    id = gid[pl];
    return hypot(gx[pl] - px, gy[pl] - py);
  }
};

// Serial exact insertion (the reference's algorithm): the fallback.
template <class Src>
__device__ int select_serial(const Src &src, int k, double radius, float r2hi, const Sel &S,
                             int lane) {
  int cnt = 0;
  src.visit(r2hi, lane, [&](bool ok, float, int pl) {
    int id = 0;
    double e = 0.0;
    if (ok) {
      e = src.exact(pl, id);
      ok = e <= radius;
    }
    unsigned bal = __ballot_sync(kFull, ok);
    while (bal) {
      const int src_lane = __ffs(bal) - 1;
      bal &= bal - 1;
      const double ej = __shfl_sync(kFull, e, src_lane);
      const int idj = __shfl_sync(kFull, id, src_lane);
      const int plj = __shfl_sync(kFull, pl, src_lane);
      if (lane == 0) {
        int m;
        bool take = true;
        if (cnt < k) {
          m = cnt++;
        } else if (key_less(ej, idj, S.se()[k - 1], S.sid()[k - 1])) {
          m = k - 1;
        } else {
          take = false;
          m = 0;
        }
        if (take) {
          while (m > 0 && key_less(ej, idj, S.se()[m - 1], S.sid()[m - 1])) {
            S.se()[m] = S.se()[m - 1];
            S.sid()[m] = S.sid()[m - 1];
            S.spl()[m] = S.spl()[m - 1];
            --m;
          }
          S.se()[m] = ej;
          S.sid()[m] = idj;
          S.spl()[m] = plj;
        }
      }
      __syncwarp();
    }
  });
  cnt = __shfl_sync(kFull, cnt, 0);
  for (int m = lane; m < cnt; m += 32) {
    S.sel_pl()[m] = S.spl()[m];
  }
  __syncwarp();
  return cnt;
}


// Radius that provably contains the k nearest candidates given a hint that
// bounds the k-th distance (triangle inequality).  The narrowed selection
// histograms [0, rho^2] (bucket width w = rho^2 / kNB); the k-th key is
// <= hint^2 + D, so the bucket window b* + 1 (+1.01 slack) stays inside
// rho^2 - D when rho^2 (1 - 2.05 / kNB) >= hint^2 + 2D.  The floor
// rho^2 >= 10240 D keeps the edge band beta = 2 D kNB / rho^2 <= 0.05.
// (float arithmetic: any radius is correct here, the caller validates the
// narrowed window against the rho it actually uses)
__device__ __forceinline__ double hint_radius(float hint, double radius, double D) {
  if (!(hint > 0.0f)) return radius;
  const float Df = (float)D;
  const float r2n = fmaxf((hint * hint + 2.0f * Df) * (1.0f / (1.0f - 2.05f / kNB)) + 1e-3f,
                          10240.0f * Df);
  return fmin((double)sqrtf(r2n), radius);
}

// Rank the set G[0, n_g) (bucket order, n_g <= 32 EPL).  Returns
// min(#valid, k); payloads in S.sel_pl().
//  sort    G is block-sorted (buckets are contiguous and ordered, strictly by
//          key since bucket_of is monotone), so odd-even transposition rounds
//          over the whole array (EPL consecutive positions per lane, +inf
//          padding) sort it in cmax rounds, cmax = the largest bucket: a
//          compare-exchange across a bucket boundary never swaps, so every
//          bucket is sorted as its own segment;
//  check   two sorted neighbours more than 2D apart are ordered exactly like
//          their distances, so position t is the reference's rank unless t
//          and a neighbour are a near tie, or its key may lie beyond the
//          radius (a > r2 - D).  Every element before an unflagged t is
//          exactly nearer and inside the radius.
//  exact   (rare) flagged elements get the glibc-exact distance and id; a
//          valid one ranks as the start of its near-tie cluster (a maximal
//          run of neighbours <= 2D apart, all flagged) plus the valid
//          cluster members that are exactly less.  Out-of-radius elements
//          sort after every valid one, so they only reduce the count.
__device__ __forceinline__ void cswap(float &ka, int &va, float &kb, int &vb) {
  const bool sw = kb < ka;
  const float k0 = sw ? kb : ka, k1 = sw ? ka : kb;
  const int v0 = sw ? vb : va, v1 = sw ? va : vb;
  ka = k0; kb = k1; va = v0; vb = v1;
}

// The exact tail of rank_set (rare: a near tie or a possibly-out-of-radius
// key among the first k): G sorted in S.sa() / S.spl().
template <class Src>
__device__ int rank_exact(const Src &src, int n_g, float two_d, float r2lo,
                                       double radius, int k, const Sel &S, int lane) {
  const float *const sa = S.sa();
  const int *const spl = S.spl();
  // exact: flags over every position (clusters may run past k; the count of
  // valid elements needs the top), exact (distance, id) of the flagged ones
  int n_invalid = 0;
  for (int t = lane; t < n_g; t += 32) {
    const float at = sa[t];
    const bool amb = (t > 0 && at - sa[t - 1] <= two_d) || (t + 1 < n_g && sa[t + 1] - at <= two_d);
    uint8_t f = (amb ? 1 : 0) | (at > r2lo ? 2 : 0);
    if (f) {
      int id;
      const double e = src.exact(spl[t], id);
      S.se()[t] = e;
      S.sid()[t] = id;
      if (e > radius) {
        f |= 4;
        ++n_invalid;
      }
    }
    S.sf()[t] = f;
  }
  __syncwarp();
  for (int t = lane; t < n_g; t += 32) {
    const uint8_t f = S.sf()[t];
    if (!f || (f & 4)) continue;
    int c0 = t, c1 = t;
    while (c0 > 0 && sa[c0] - sa[c0 - 1] <= two_d) --c0;
    while (c1 + 1 < n_g && sa[c1 + 1] - sa[c1] <= two_d) ++c1;
    const double et = S.se()[t];
    const int it = S.sid()[t];
    int rank = c0;
    for (int q = c0; q <= c1; ++q)
      if (q != t && !(S.sf()[q] & 4) && key_less(S.se()[q], S.sid()[q], et, it)) ++rank;
    if (rank < k) S.sel_pl()[rank] = spl[t];
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) n_invalid += __shfl_xor_sync(kFull, n_invalid, off);
  __syncwarp();
  const int n_valid = n_g - n_invalid;
  return n_valid < k ? n_valid : k;
}

template <int EPL, class Src>
__device__ int rank_set(const Src &src, int n_g, int cmax, float two_d, float r2lo, double radius,
                        int k, const Sel &S, int lane) {
  static_assert(EPL % 2 == 0, "odd-even rounds pair positions inside a lane");
  float key[EPL];
  int val[EPL];
  const int base = EPL * lane;
  if constexpr (EPL % 4 == 0) {
#pragma unroll
    for (int e = 0; e < EPL; e += 4) {
      const float4 kv = *reinterpret_cast<const float4 *>(S.ga() + base + e);
      const int4 pv = *reinterpret_cast<const int4 *>(S.gpl() + base + e);
      key[e] = kv.x; key[e + 1] = kv.y; key[e + 2] = kv.z; key[e + 3] = kv.w;
      val[e] = pv.x; val[e + 1] = pv.y; val[e + 2] = pv.z; val[e + 3] = pv.w;
    }
  } else {
#pragma unroll
    for (int e = 0; e < EPL; ++e) {
      key[e] = S.ga()[base + e];
      val[e] = S.gpl()[base + e];
    }
  }
#pragma unroll
  for (int e = 0; e < EPL; ++e)
    if (base + e >= n_g) key[e] = INFINITY;
  for (int r = 0; r < cmax; ++r) {
    if ((r & 1) == 0) {
#pragma unroll
      for (int e = 0; e < EPL; e += 2) cswap(key[e], val[e], key[e + 1], val[e + 1]);
    } else {
      // lane boundary pair (EPL l + EPL - 1, EPL (l + 1)): both sides read
      // the other's value before either updates
      const float kn = __shfl_down_sync(kFull, key[0], 1);
      const int vn = __shfl_down_sync(kFull, val[0], 1);
      const float kp = __shfl_up_sync(kFull, key[EPL - 1], 1);
      const int vp = __shfl_up_sync(kFull, val[EPL - 1], 1);
#pragma unroll
      for (int e = 1; e + 1 < EPL; e += 2) cswap(key[e], val[e], key[e + 1], val[e + 1]);
      if (lane < 31 && kn < key[EPL - 1]) { key[EPL - 1] = kn; val[EPL - 1] = vn; }
      if (lane > 0 && kp > key[0]) { key[0] = kp; val[0] = vp; }
    }
  }
  // check the first min(n_g, k) positions against their sorted neighbours
  const int nk = n_g < k ? n_g : k;
  const float kprev = __shfl_up_sync(kFull, key[EPL - 1], 1);
  const float knext = __shfl_down_sync(kFull, key[0], 1);
  bool flagged = false;
#pragma unroll
  for (int e = 0; e < EPL; ++e) {
    const float lo = e > 0 ? key[e - 1] : (lane > 0 ? kprev : -INFINITY);
    const float hi = e + 1 < EPL ? key[e + 1] : (lane < 31 ? knext : INFINITY);
    const bool amb = key[e] - lo <= two_d || hi - key[e] <= two_d;
    if (base + e < nk) {
      if (amb || key[e] > r2lo) flagged = true;
      else S.sel_pl()[base + e] = val[e];
    }
  }
  if (!__any_sync(kFull, flagged)) {
    __syncwarp();
    return nk;
  }
  OBS_STAT(5, 1);
#pragma unroll
  for (int e = 0; e < EPL; ++e) {
    if (base + e < n_g) {
      S.sa()[base + e] = key[e];
      S.spl()[base + e] = val[e];
    }
  }
  __syncwarp();
  return rank_exact(src, n_g, two_d, r2lo, radius, k, S, lane);
}

// Histogram range [0, r2hi] in key units (the whole disc r^2 + D, or rho^2
// for a hint-narrowed scan): the bucket scale inv_w (any scale works here --
// histogram, scatter and ranking all bucket by a * inv_w; the edge bands are
// in those units and the window check keeps a 1 % slack on w, so the fast
// reciprocal), the edge band beta in bucket units (twice the key error plus
// float slack) and the near-tie band two_d (padded by the float rounding of
// a - 2D).
struct SelRange {
  float r2hi, inv_w, beta, two_d;
};

__host__ __device__ __forceinline__ SelRange range_of(double top, float Df) {
  SelRange R;
  R.r2hi = (float)(top * (1.0 + 1e-7) + 1e-30);
#ifdef __CUDA_ARCH__
  float rcp;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rcp) : "f"(R.r2hi));
#else
  const float rcp = 1.0f / R.r2hi;
#endif
  R.inv_w = R.r2hi > 0.0f ? (float)kNB * rcp : 0.0f;
  R.beta = 2.0f * Df * R.inv_w + 4e-5f;
  R.two_d = 2.0f * Df + 2.5e-7f * R.r2hi;
  return R;
}

// Per-selection parameters (formed once per agent in the prologue for the
// road points, once per launch on the host for the partners).
//  Df >= D and r2lo <= r2 - D: float thresholds rounded the conservative way
//  (wider bands, more keys get the exact radius test); R: the first range
//  (narrowed to rho when `restricted`); serial: the full-radius key bound is
//  too loose for the bucket width (beta >= 1/8): serial insertion.
struct SelParams {
  SelRange R;
  float Df, r2lo;
  double D, rho;
  bool restricted, serial;
};

// The selection's current histogram range (the first one of SelParams, or
// the full disc after a failed narrowing).
struct SelState {
  float r2hi, inv_w, two_d;
  __device__ __forceinline__ void set_full(double r2, double D, float Df) {
    const SelRange F = range_of(r2 + D, Df);
    r2hi = F.r2hi;
    inv_w = F.inv_w;
    two_d = F.two_d;
  }
};

// Small candidate sets (partners): compacted straight into G in visit order
// and ranked by counting; returns -1 when this fast path cannot decide (more
// than 32 candidates, or a near tie / a possibly-out-of-radius key among the
// first k).
template <class Src>
__device__ __forceinline__ int select_direct(const Src &src, int k, const SelParams &P,
                                             const SelState &R, const Sel &S, int lane,
                                             float &bound_out) {
  int n = 0;
  src.visit(R.r2hi, lane, [&](bool ok, float a, int pl) {
    const unsigned bal = __ballot_sync(kFull, ok);
    const int pos = n + __popc(bal & ((1u << lane) - 1u));
    if (ok && pos < S.gcap) {
      S.ga()[pos] = a;
      S.gpl()[pos] = pl;
    }
    n += __popc(bal);
  });
  bound_out = 0.0f;
  if (n == 0) return 0;
  if (n > 32) return -1;
  if (lane >= n && lane < ((n + 3) & ~3)) S.ga()[lane] = INFINITY;   // whole float4s below
  __syncwarp();
  // one candidate per lane, ranked by counting (key, payload) order over the
  // n broadcast keys; keys more than 2D apart order exactly like the
  // distances.  (key, payload) order = (key bits, lane): G was compacted in
  // visit order, so payloads ascend with the lane.  The keys are read back
  // by broadcast shared loads, four per load; equal keys are ranked by lane
  // with one match.
  const float a = lane < n ? S.ga()[lane] : INFINITY;
  const int pl = lane < n ? S.gpl()[lane] : 0x7fffffff;
  const unsigned ab = __float_as_uint(a);
  int rank = __popc(__match_any_sync(kFull, ab) & ((1u << lane) - 1u));
  // the n keys read back four at a time by broadcast shared loads (padded
  // with +inf, which never counts)
  const float4 *g4 = reinterpret_cast<const float4 *>(S.ga());
#pragma unroll 2
  for (int j = 0; j < n; j += 4) {
    const float4 q = g4[j >> 2];
    rank += (q.x < a ? 1 : 0) + (q.y < a ? 1 : 0) + (q.z < a ? 1 : 0) + (q.w < a ? 1 : 0);
  }
  // near ties between sorted neighbours, staged in the idle pass-1 buffer
  float *const srt = S.ca();
  if (lane < n) srt[rank] = a;
  __syncwarp();
  bool amb = false;
  if (lane < n)
    amb = (rank + 1 < n && srt[rank + 1] - a <= R.two_d) || (rank > 0 && a - srt[rank - 1] <= R.two_d);
  const bool bad = lane < n && rank < k && (amb || a > P.r2lo);
  if (__any_sync(kFull, bad)) return -1;
  if (lane < n && rank < k) S.sel_pl()[rank] = pl;
  __syncwarp();
  return n < k ? n : k;
}

// Larger sets (road points): histogram threshold, counting-sort scatter into
// G, rank_set.  Returns -1 when G would exceed its capacity.
//  * rho: the radius the source currently covers (< radius when the caller
//    narrowed it with a search hint, see hint_radius).  A narrowed pass 1 is
//    used only if every bucket the selection touches provably lies inside
//    the disc ((bmax + 1) w + D <= rho^2), else it reruns on the full radius.
//    bound_out: a bound on the k-th distance (0 when fewer than k candidates
//    exist).
//  * pass 1 keeps (key, payload) in shared memory when they fit.
template <int EPL, class Src>
__device__ __forceinline__ int select_hist(Src &src, int k, double radius, const SelParams &P,
                                           SelState &R, const Sel &S, int lane, float &bound_out) {
  const double r2 = radius * radius, D = P.D, rho = P.rho;
  bool restricted = P.restricted;
  const int pb = src.pbase();
  const bool small = src.small_payload();
  constexpr int kPer = kNB / 32;
  uint32_t total, n_g, incl, local;
  uint32_t cnt[kPer];
  int bstar, bmax, nbuf;
  double w;   // bucket width (key units)
  static_assert(kPer % 4 == 0, "the histogram is read / written as uint4 per lane");
  constexpr int kVec = kPer / 4;
  uint4 *const hc4 = reinterpret_cast<uint4 *>(S.hc());
  while (true) {
#pragma unroll
    for (int v = 0; v < kVec; ++v) hc4[lane + 32 * v] = make_uint4(0u, 0u, 0u, 0u);
    __syncwarp();
    nbuf = 0;
    const float inv_w = R.inv_w;
    src.visit(R.r2hi, lane, [&](bool ok, float a, int pl) {
      // branch-free: a lane without a candidate adds 0 (its key is finite
      // and >= 0, so its bucket index is in range)
      atomicAdd(&S.hc()[bucket_of(a, inv_w)], ok ? 1u : 0u);
      const unsigned bal = __ballot_sync(kFull, ok);
      const int pos = nbuf + __popc(bal & ((1u << lane) - 1u));
      if (ok && pos < S.ccap) {
        S.ca()[pos] = a;
        S.cp()[pos] = (uint16_t)(pl - pb);
      }
      nbuf += __popc(bal);
    });
    __syncwarp();
#pragma unroll
    for (int v = 0; v < kVec; ++v) {
      const uint4 c = hc4[kVec * lane + v];
      cnt[4 * v] = c.x; cnt[4 * v + 1] = c.y; cnt[4 * v + 2] = c.z; cnt[4 * v + 3] = c.w;
    }
    local = 0;
#pragma unroll
    for (int q = 0; q < kPer; ++q) local += cnt[q];
    incl = local;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const uint32_t up = __shfl_up_sync(kFull, incl, off);
      if (lane >= off) incl += up;
    }
    total = __shfl_sync(kFull, incl, 31);
    uint32_t run = incl - local;
    bstar = kNB - 1;
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
      if (run < (uint32_t)k && run + cnt[q] >= (uint32_t)k) bstar = lane * kPer + q;
      run += cnt[q];
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) bstar = min(bstar, __shfl_xor_sync(kFull, bstar, off));
    // G = buckets <= b*+1: an element of b*+2 has at least k elements
    // exactly nearer (all of buckets <= b*), so it never ranks below k
    bmax = min(bstar + 1, kNB - 1);
    w = (double)R.r2hi / kNB;
    // a narrowed scan is valid only if all buckets <= bmax lie inside the disc
    OBS_STAT(1, total);
    if (restricted && !((((double)bmax + 1.01) * w + D) <= rho * rho)) {
      OBS_STAT(2, 1);
      src.restrict_to(radius + 1e-6, lane);
      restricted = false;
      R.set_full(r2, D, P.Df);
      continue;
    }
    break;
  }
  bound_out = total >= (uint32_t)k ? sqrtf(((float)bstar + 1.0f) * (float)w + P.Df) * (1.0f + 1e-6f)
                                    : 0.0f;
  if (total == 0) return 0;
  uint32_t run2 = incl - local;
  uint32_t hv[kPer];
#pragma unroll
  for (int q = 0; q < kPer; ++q) {
    hv[q] = (run2 << 16) | cnt[q];
    run2 += cnt[q];
  }
#pragma unroll
  for (int v = 0; v < kVec; ++v)
    hc4[kVec * lane + v] = make_uint4(hv[4 * v], hv[4 * v + 1], hv[4 * v + 2], hv[4 * v + 3]);
  __syncwarp();
  {
    const uint32_t hb = S.hc()[bmax];   // (start << 16) | count of the last kept bucket
    n_g = (hb >> 16) + (hb & 0xffffu);
  }
  if (n_g > (uint32_t)S.gcap || total > 0xffffu) return -1;
  // largest kept bucket: the sort's round count
  int cmax = 0;
#pragma unroll
  for (int q = 0; q < kPer; ++q)
    if (lane * kPer + q <= bmax) cmax = max(cmax, (int)cnt[q]);
  cmax = (int)__reduce_max_sync(kFull, (unsigned)cmax);
  OBS_STAT(4, n_g);
  // pass 2: counting-sort scatter of buckets <= bmax into G
  const float inv_w = R.inv_w;
  auto scatter = [&](float a, int pl) {
    const int b = bucket_of(a, inv_w);
    if (b <= bmax) {
      const uint32_t pos = atomicAdd(&S.hc()[b], 1u << 16) >> 16;
      S.ga()[pos] = a;
      S.gpl()[pos] = pl;
    }
  };
  if (nbuf <= S.ccap && small) {
    // warp-uniform trip count; idle lanes of the last pass skip the scatter
    for (int p0 = 0; p0 < nbuf; p0 += 32) {
      const int p = p0 + lane < nbuf ? p0 + lane : p0;
      const float a = S.ca()[p];
      const int pl = pb + (int)S.cp()[p];
      if (p0 + lane < nbuf) scatter(a, pl);
    }
  } else {
    OBS_STAT(7, 1);
    // only keys in buckets <= bmax matter: a < (bmax + 1) w, so d^2 < that + D
    if (bmax < kNB - 1) src.restrict_to(sqrt(((double)bmax + 1.01) * w + D) + 1e-6, lane);
    src.visit(R.r2hi, lane, [&](bool ok, float a, int pl) {
      if (ok) scatter(a, pl);
    });
  }
  __syncwarp();
  return rank_set<EPL>(src, (int)n_g, cmax, R.two_d, P.r2lo, radius, k, S, lane);
}

// Exact ascending top-min(n_valid, k) by (distance, id) given candidate keys
// with |a - d^2| <= D.  Payloads land in S.sel_pl()[0..m).  Warp-collective.
// Direct: the partners' counting path, else the histogram path; ranking uses
// the float keys (two keys more than 2D apart are ordered exactly as the
// distances), the exact FP64 hypot only near ties and the radius.  Either
// path falls back to the reference's serial insertion -- exact by
// construction, one call site (code size) -- for a loose key bound
// (P.serial), a set the fast path cannot rank, or a G beyond capacity.
template <bool Direct, int EPL, class Src>
__device__ int select_topk(Src src, int k, double radius, const SelParams &P, const Sel &S,
                           int lane, float &bound_out) {
  if (k <= 0) return 0;
  SelState R{P.R.r2hi, P.R.inv_w, P.R.two_d};
  if (!P.serial) {
    int m;
    if constexpr (Direct) m = select_direct(src, k, P, R, S, lane, bound_out);
    else m = select_hist<EPL>(src, k, radius, P, R, S, lane, bound_out);
    if (m >= 0) return m;
    OBS_STAT(Direct ? 6 : 3, 1);
  } else {
    OBS_STAT(3, 1);
  }
  __syncwarp();
  R.set_full(radius * radius, P.D, P.Df);
  src.restrict_to(radius + 1e-6, lane);
  return select_serial(src, k, radius, R.r2hi, S, lane);
}

// ---------------------------------------------------------------------------
// The kernel.  SharedPts: road points staged in shared memory (float2).
// ---------------------------------------------------------------------------
// CAPA / CAPR > 0: compile-time slot caps (the ObsConfig default 16 / 64);
// 0: taken from the config at run time.
// Per-launch scalars derived from the config on the host: kernel parameters
// live in the constant bank, so the kernel uses them as operands instead of
// keeping (or rematerialising) them in registers.
struct RadialK {
  double radius, reach, r2, D_fp64, cs, inv_cs, key_e;
  int64_t uni_a, uni_c, uni_p;   // uniform per-world strides (0: read the offsets)
};

// AMAX > 0: the agent tables' stride as a compile-time constant (worlds of
// <= AMAX agents; every agent array then sits at a constant offset from one
// base instead of a dozen run-time pointers); 0: T.max_agents
template <int WARPS, bool SharedPts, int CAPA, int CAPR, int AMAX = 0>
__global__ void __launch_bounds__(WARPS * 32, (!SharedPts || WARPS <= 16) ? 2 : 1) obs_radial_kernel(
    ds_tables T, ds_config C, ds_state St, const RadialK K, const uint8_t *mask, const ObsOut O,
    const float *scale, int32_t *sel_idx, int obs_width) {
  const int w = blockIdx.x;
  if (mask && !mask[w]) return;
#ifdef DS_OBS_TIMES
  if (threadIdx.x == 0 && w < 8192) {
    unsigned sm;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
    g_obs_times[w * kTimesW] = sm;
    g_obs_times[w * kTimesW + 1] = gtimer();
  }
#endif
  // every per-world offset in one round of independent loads
  // (uniform worlds: formed from the strides, no dependent load)
  const int64_t c0 = K.uni_c ? w * K.uni_c : T.c_off[w], c1 = K.uni_c ? c0 + K.uni_c : T.c_off[w + 1];
  const int64_t a0 = K.uni_a ? w * K.uni_a : T.a_off[w], a1 = K.uni_a ? a0 + K.uni_a : T.a_off[w + 1];
  const int64_t p0 = K.uni_p ? w * K.uni_p : T.p_off[w], p1 = K.uni_p ? p0 + K.uni_p : T.p_off[w + 1];
  const int nrow = (int)(c1 - c0);
  if (nrow == 0) return;
  const int A = (int)(a1 - a0);
  const int np = (int)(p1 - p0);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ uint64_t pts_bar;
  __shared__ float e_max_w[WARPS];   // per warp: largest float rounding of an agent position
  __shared__ int next_row;
  __shared__ float bound_w[WARPS];   // per warp: the road selection's k-th distance bound           // rows are handed out dynamically (no tail imbalance)
  constexpr bool kFixed = CAPA > 0;
  // G positions per lane in the sort (even; runtime caps <= kSelCap: 6)
  constexpr int kEPL = kFixed ? ((gcap_of(CAPA, CAPR) + 63) / 64) * 2 : 2 * ((kSelCap + 48 + 63) / 64);
  static_assert(32 * kEPL >= (kFixed ? gcap_of(CAPA, CAPR) : kSelCap + 48), "sort capacity");
  const int cap_a = kFixed ? CAPA : C.max_agents_obs, cap_r = kFixed ? CAPR : C.max_road_points_obs;
  constexpr WarpLayout kWL = make_layout(CAPA, CAPR, !SharedPts);
  const WarpLayout WL = kFixed ? kWL : warp_layout(C, !SharedPts);
  // shared memory: [per-warp scratch x WARPS][road points][agent tables] --
  // the scratch and the points sit at (compile-time) constant offsets
  // lane / warp from opaque moves: the compiler keeps them in registers
  // instead of re-reading the special registers (S2R)
  int lane, warp;
  asm volatile("mov.u32 %0, %%laneid;" : "=r"(lane));
  warp = __shfl_sync(kFull, (int)threadIdx.x >> 5, 0);
  // the dynamic shared window's base (a 32-bit shared address that depends
  // on the CTA's cluster rank) taken once through an opaque move: otherwise
  // the compiler rematerialises it (S2R SR_CgaCtaId + LEA) at every use
  // under register pressure
  uint32_t smem_s = (uint32_t)__cvta_generic_to_shared(smem_raw);
  asm volatile("mov.u32 %0, %0;" : "+r"(smem_s));
  unsigned char *const sbase = static_cast<unsigned char *>(__cvta_shared_to_generic(smem_s));
  unsigned char *wb = sbase + WL.total * warp;
  unsigned char *after_scratch = sbase + WL.total * WARPS;
  const int amax = AMAX > 0 ? AMAX : T.max_agents;
  // points: the 16-B aligned body [pa, pb) of the world's range by one bulk
  // copy, an odd head / tail point by plain loads; pts[j] = point p0 + j
  float2 *const pbuf = reinterpret_cast<float2 *>(after_scratch);
  float2 *const pts = pbuf + (p0 & 1);
  if (threadIdx.x == 0) next_row = WARPS;   // rows 0..WARPS-1 start statically
  if (SharedPts && threadIdx.x == 0) {
    mbar_init(&pts_bar, 1);
    const int64_t pa = (p0 + 1) & ~int64_t(1), pb = p1 & ~int64_t(1);
    const float2 *src = reinterpret_cast<const float2 *>(T.gpt_xy);
    if (pb > pa) {
      const uint32_t bytes = (uint32_t)((pb - pa) * sizeof(float2));
      mbar_arrive_tx(&pts_bar, bytes);
      bulk_g2s(pbuf + (pa - (p0 & ~int64_t(1))), src + pa, bytes, &pts_bar);
    } else {
      mbar_arrive(&pts_bar);
    }
  }
  if (SharedPts && threadIdx.x == 32) {
    const float2 *src = reinterpret_cast<const float2 *>(T.gpt_xy);
    const int64_t pa = (p0 + 1) & ~int64_t(1), pb = p1 & ~int64_t(1);
    if (p0 < pa && p0 < p1) pts[0] = src[p0];
    if (pb < p1 && pb >= pa) pts[pb - p0] = src[pb];
  }
  const AgentTabs AT = agent_tabs(after_scratch + (SharedPts ? points_bytes(T.max_points) : 0), amax);
  Sel S;
  S.wb = wb;
  S.L = WL;
  S.gcap = gcap_of(cap_a, cap_r);
  S.ccap = SharedPts ? kCandShared : kCandGlobal;
  float *const row0 = reinterpret_cast<float *>(wb + WL.row);
  const int row0_phase = (int)((reinterpret_cast<uintptr_t>(row0) >> 2) & 3);

  const double radius = K.radius;
  const double reach = K.reach;         // culling slack; membership is decided exactly
  const int road_off = 7 + 7 * cap_a;
  const int sel_w = cap_a + cap_r;
  const int nx = T.grid_nx[w], ny = T.grid_ny[w];
  const double gx0 = T.grid_x0[w], gy0 = T.grid_y0[w], cs = K.cs;
  const double inv_cs = K.inv_cs;
  const int64_t cbase = T.grid_cell_off[w];
  const double eps_p = SharedPts ? T.grid_eps[w] : 0.0;
  const double D_fp64 = K.D_fp64;       // fl32 of an FP64 d^2

  // agent tables and the ego block of every agent (fp:228-238), then -- by
  // a second group of threads -- the road-selection parameters and partner
  // key positions: one thread per (agent, part), overlapping the points'
  // bulk copy (the parts split the prologue's critical path)
  // row -> agent loads issued first: in flight across the staging below
  const int ra_pre = (int)threadIdx.x < nrow ? T.row_agent[c0 + threadIdx.x] : 0;
  float e_own = 0.0f;
  // three parts per agent, one thread each: the tables and the rotation,
  // the goal distance (an FP64 hypot, independent of the rotation), the
  // road-selection parameters
  for (int u = threadIdx.x; u < 3 * A; u += blockDim.x) {
    const int part = u < A ? 0 : (u < 2 * A ? 1 : 2);
    const bool tabs = part == 0;
    const int i = u - part * A;
    const int64_t g = a0 + i;
    const double px = St.x[g], py = St.y[g];
    if (part == 1) {
      const double gx = T.goal_x[g] - px, gy = T.goal_y[g] - py;
      AT.ego[8 * i + 5] = (float)hypot(gx, gy);
      continue;
    }
    const uint16_t f = St.flags[g];
    if (tabs) {
      const double hd = St.heading[g], v = St.speed[g];
      const double ln = T.length[g], wd = T.width[g];
      const double gx = T.goal_x[g] - px, gy = T.goal_y[g] - py;
      double sh, ch;
      sincos(hd, &sh, &ch);
      AT.x[i] = px; AT.y[i] = py; AT.h[i] = hd; AT.v[i] = v;
      AT.l[i] = (float)ln; AT.w[i] = (float)wd; AT.c[i] = ch; AT.s[i] = sh;
      AT.flg[i] = f;
      float *e = AT.ego + 8 * i;
      e[0] = (float)v;
      e[1] = (float)ln;
      e[2] = (float)wd;
      e[3] = (float)(gx * ch + gy * sh);
      e[4] = (float)(gy * ch - gx * sh);
      e[6] = (f & DS_F_COLLIDED) ? 1.0f : 0.0f;
      continue;
    }
    const float4 hint = St.obs_hint ? reinterpret_cast<const float4 *>(St.obs_hint)[g]
                                    : make_float4(0.f, 0.f, 0.f, 0.f);
    // road selection: the bound on this step's k-th distance is the hint
    // plus the distance moved (float; the 1 mm slack exceeds the rounding of
    // the grid-relative floats)
    const double rx = px - gx0, ry = py - gy0;
    const float prx = (float)rx, pry = (float)ry;
    float rho_hint = 0.0f;
    if (hint.x > 0.0f) {
      const float mx = hint.y - prx, my = hint.z - pry;
      rho_hint = hint.x + sqrtf(mx * mx + my * my) + 1e-3f;
    }
    double D = D_fp64;
    if (SharedPts) {
      // key bound: |dx_f - dx| <= E; |a - d^2| <= 4 (r + 1) E + 2 E^2 + fl32 rounding
      const double E = eps_p + fmax(fabs((double)prx - rx), fabs((double)pry - ry)) + K.key_e;
      D = 4.0 * (radius + 1.0) * E + 2.0 * E * E + D_fp64;
    }
    const double rho = hint_radius(rho_hint, radius, D);
    const float Df = __double2float_ru(D);
    const SelRange full = range_of(K.r2 + D, Df);
    const bool restricted = rho < radius;
    const SelRange R = restricted ? range_of(rho * rho, Df) : full;
    RowGeo geo{nullptr, prx, pry, (float)cs, (float)inv_cs, 0.0f, nx, ny, 0, 0};
    geo.init((float)reach);
    AT.pa[i] = make_float4(prx, pry, geo.marg, Df);
    AT.pb[i] = make_float4(R.r2hi, R.inv_w, R.two_d, __double2float_rd(K.r2 - D));
    AT.pc[i] = make_double2(D, rho);
    AT.pd[i] = make_int4(geo.iy0, geo.nrows, (restricted ? 1 : 0) | (full.beta < 0.125f ? 0 : 2), 0);
    // partner key position: absent / removed agents get the far sentinel
    const bool vis = (f & DS_F_PRESENT) && !(f & DS_F_REMOVED);
    AT.pxy[i] = vis ? make_float2(prx, pry) : make_float2(1e30f, 1e30f);
    e_own = fmaxf(e_own, (float)fmax(fabs((double)prx - rx), fabs((double)pry - ry)) * (1.0f + 1e-6f));
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) e_own = fmaxf(e_own, __shfl_xor_sync(kFull, e_own, off));
  if (lane == 0) e_max_w[warp] = e_own;
  for (int i = A + (int)threadIdx.x; i < pad32(A); i += blockDim.x) AT.pxy[i] = make_float2(1e30f, 1e30f);
  // row -> local agent, so the row loop starts from shared memory
  if ((int)threadIdx.x < nrow) AT.rloc[threadIdx.x] = (uint16_t)(ra_pre - a0);
  for (int r = threadIdx.x + blockDim.x; r < nrow; r += blockDim.x)
    AT.rloc[r] = (uint16_t)(T.row_agent[c0 + r] - a0);
#ifdef DS_OBS_TIMES
  if (threadIdx.x == 0 && w < 8192) g_obs_times[w * kTimesW + 35] = gtimer();
#endif
  __syncthreads();
#ifdef DS_OBS_TIMES
  if (threadIdx.x == 0 && w < 8192) g_obs_times[w * kTimesW + 36] = gtimer();
#endif
  if (SharedPts) mbar_wait(&pts_bar, 0);
#ifdef DS_OBS_TIMES
  if (threadIdx.x == 0 && w < 8192) g_obs_times[w * kTimesW + 2] = gtimer();
#endif
  const double *ax = AT.x, *ay = AT.y, *ah = AT.h, *av = AT.v, *ac = AT.c, *as = AT.s;
  const float *al = AT.l, *aw = AT.w;
  // the partners' selection parameters (per world): E = both positions'
  // float rounding + the float subtraction
  // (kept in shared memory -- one copy per warp -- and read where used
  // instead of in registers held across the row loop)
  __shared__ SelParams PP_w[WARPS];
  {
    SelParams PP;
    float em = lane < WARPS ? e_max_w[lane] : 0.0f;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) em = fmaxf(em, __shfl_xor_sync(kFull, em, off));
    const double E = 2.0 * (double)em + K.key_e;
    const double D = 4.0 * (radius + 1.0) * E + 2.0 * E * E + D_fp64;
    PP.Df = __double2float_ru(D);
    PP.r2lo = __double2float_rd(K.r2 - D);
    PP.R = range_of(K.r2 + D, PP.Df);
    PP.D = D;
    PP.rho = radius;
    PP.restricted = false;
    PP.serial = !(PP.R.beta < 0.125f);
    if (lane == 0) PP_w[warp] = PP;
    __syncwarp();
  }
  const SelParams &PP = PP_w[warp];

  // float32 rows without normalisation leave by bulk stores
  const bool bulk_out = O.dtype == DS_OBS_F32 && scale == nullptr;
  auto grab_row = [&]() {
    int v = 0;
    if (lane == 0) v = atomicAdd(&next_row, 1);
    return __shfl_sync(kFull, v, 0);
  };
#ifdef DS_OBS_TIMES
  int prev_r = -1;
  unsigned long long t_prev = 0;
#endif
  for (int r = warp; r < nrow; r = grab_row()) {
#ifdef DS_OBS_TIMES
    {
      const unsigned long long t_now = gtimer();
      if (lane == 0 && prev_r >= 0 && prev_r < 128 && w < 8192) g_row_dur[w * 128 + prev_r] = (unsigned)(t_now - t_prev);
      prev_r = r;
      t_prev = t_now;
    }
#endif
    const int64_t orow = c0 + r;
    const int i = AT.rloc[r];
    const uint16_t f = AT.flg[i];
    if (f & (DS_F_DONE | DS_F_REMOVED)) {
      // finished / removed rows are zero-filled (engine.py:502-512)
      zero_row(O, orow, lane);
      if (sel_idx)
        #pragma unroll 1
        for (int c = lane; c < sel_w; c += 32) sel_idx[orow * sel_w + c] = -1;
      continue;
    }
    OBS_STAT(0, 1);
    if (bulk_out) {
      // the previous row's bulk store must have read the staging buffer
      if (lane == 0) bulk_row_wait();
      __syncwarp();
    }
    // the staged row copies the output row's 16-B phase (vector write-out)
    const int out_phase = out_row_phase(O, orow);
    float *const row = row0 - ((row0_phase - out_phase) & 3);   // contiguous staged row
    const double px = ax[i], py = ay[i];
    const float4 pa = AT.pa[i], pb = AT.pb[i];
    const double2 pc = AT.pc[i];
    const int4 pd = AT.pd[i];
    SelParams P;
    P.R = SelRange{pb.x, pb.y, 0.0f, pb.z};
    P.Df = pa.w;
    P.r2lo = pb.w;
    P.D = pc.x;
    P.rho = pc.y;
    P.restricted = pd.z & 1;
    P.serial = pd.z & 2;
    const RowGeo geo{T.pt_cell_start + cbase, pa.x, pa.y, (float)cs, (float)inv_cs, pa.z, nx, ny, pd.x, pd.y};
    // the road rows' cell-table loads stay in flight across the partners
    // (into the histogram words, unused until the road selection; no
    // registers are held across the partners)
    int *const cellv = reinterpret_cast<int *>(wb + WL.hc);
    if (SharedPts && cap_r > 0) geo.range_issue_async((float)(P.restricted ? P.rho : reach), lane, cellv);

    // ---- partners: the picks are kept aside (psel); their slots are formed
    // while the selected road records are in flight
    Sel SP = S;
    SP.L.sel_pl = WL.psel;
    PartnerSrc psrc{AT.pxy, ax, ay, pad32(A), i, pa.x, pa.y, px, py};
    float no_bound = 0.0f;
    const int ma = select_topk<true, kEPL>(psrc, cap_a, radius, PP, SP, lane, no_bound);
    int *const psel = reinterpret_cast<int *>(wb + WL.psel);
    if (lane < 7) row[lane] = AT.ego[8 * i + lane];   // ego block, formed in the prologue

    // ---- road points: lane l owns cell row iy0 + l of the disc
    int mr = 0;
    // the k-th distance bound goes to shared memory (one word per warp): it
    // is produced before the ranking and consumed after it
    float &bound = bound_w[warp];
    if (lane == 0) bound = 0.0f;
    if (cap_r > 0) {
      if (SharedPts) {
        RoadSrcShared rsrc{pts, static_cast<const ds_point_rec *>(T.gpt_rec), (int)p0, pa.x, pa.y, px,
                           py, &geo, reinterpret_cast<int *>(wb + WL.fr)};
        cp_async_wait_all();
        __syncwarp();
        rsrc.cover_raw(cellv[lane], cellv[32 + lane], lane);
        mr = select_topk<false, kEPL>(rsrc, cap_r, radius, P, S, lane, bound);
      } else {
        RoadSrcGlobal rsrc{T.gpt_x, T.gpt_y, T.gpt_id, (int)p0, np, px, py, &geo,
                           reinterpret_cast<int *>(wb + WL.fr)};
        rsrc.cover(P.restricted ? P.rho : reach, lane);
        mr = select_topk<false, kEPL>(rsrc, cap_r, radius, P, S, lane, bound);
      }
    }
    // the agent's index, heading and rotation re-read from the staged tables
    // after the selections (instead of held in registers across them)
    const int ii = AT.rloc[r];
    const double h = ah[ii], ch = ac[ii], sh = as[ii];
    if (St.obs_hint && lane == 0)
      // (pa.x, pa.y) = (float)(px - gx0), (float)(py - gy0)
      reinterpret_cast<float4 *>(St.obs_hint)[a0 + ii] =
          make_float4(bound, AT.pa[ii].x, AT.pa[ii].y, 0.0f);
    // the selected records (32 B, one sector each) are fetched into the dead
    // selection scratch at the END of the road block ([road_end - 32 cap_r,
    // road_end)): the slots of batch u (44 B each, written from the start)
    // never reach the records of batch u + 1.  Each lane fetches the records
    // of the slots it forms.
    float *rstage = row + road_off;
    const double2 *recs = reinterpret_cast<const double2 *>(wb + WL.road_end) - 2 * cap_r;
    const int sel_off = SharedPts ? (int)p0 : 0;
    if (SharedPts) {
      const double2 *grec = reinterpret_cast<const double2 *>(T.gpt_rec);
      for (int m = lane; m < mr; m += 32) {
        const int64_t s2 = 2 * (int64_t)(S.sel_pl()[m] + sel_off);
        cp_async16(const_cast<double2 *>(recs + 2 * m), grec + s2);
        cp_async16(const_cast<double2 *>(recs + 2 * m + 1), grec + s2 + 1);
      }
    }

    // ---- partner slots (fp:240-272) while the records arrive
    float *ps = row + 7;
    for (int m = lane; m < ma; m += 32) {
      const int j = psel[m];
      const double dx = ax[j] - px, dy = ay[j] - py;
      float *slot = ps + 7 * m;
      slot[0] = (float)(dx * ch + dy * sh);
      slot[1] = (float)(dy * ch - dx * sh);
      slot[2] = (float)wrap(ah[j] - h);
      slot[3] = (float)(av[j] - av[ii]);
      slot[4] = (float)al[j];
      slot[5] = (float)aw[j];
      slot[6] = 1.0f;
      if (sel_idx) sel_idx[orow * sel_w + m] = j;
    }
    // unused partner slots read 0 (uniform trip count: 7 cap_a floats)
    for (int q0 = 0; q0 < 7 * cap_a; q0 += 32)
      if (q0 + lane >= 7 * ma && q0 + lane < 7 * cap_a) ps[q0 + lane] = 0.0f;
    if (sel_idx)
      for (int m = ma + lane; m < cap_a; m += 32) sel_idx[orow * sel_w + m] = -1;

    // ---- road slots (fp:274-300), 32 per batch: read the batch's records,
    // sync, then overwrite the scratch with the slots
    if (SharedPts) cp_async_wait_all();
    for (int m0 = 0; m0 < cap_r; m0 += 32) {
      const int m = m0 + lane;
      double qx = 0.0, qy = 0.0, qh = 0.0;
      int qid = 0, kind = 0;
      if (m < mr) {
        if (SharedPts) {
          const double2 ra = recs[2 * m], rb = recs[2 * m + 1];
          qx = ra.x;
          qy = ra.y;
          qh = rb.x;
          qid = __double2loint(rb.y);
          kind = (int)(signed char)(__double2hiint(rb.y) & 0xff);
        } else {
          const int s = S.sel_pl()[m];
          qx = T.gpt_x[s];
          qy = T.gpt_y[s];
          qh = T.gpt_h[s];
          kind = T.gpt_kind[s];
          qid = T.gpt_id[s];
        }
      }
      __syncwarp();
      if (m < cap_r) {
        float *slot = rstage + 11 * m;
        if (m < mr) {
          const double dx = qx - px, dy = qy - py;
          slot[0] = (float)(dx * ch + dy * sh);
          slot[1] = (float)(dy * ch - dx * sh);
          slot[2] = (float)wrap(qh - h);
#pragma unroll
          for (int q = 0; q < 7; ++q) slot[3 + q] = 0.0f;
          slot[3 + kind] = 1.0f;                   // road kinds are 0..6
          slot[10] = 1.0f;
          if (sel_idx) sel_idx[orow * sel_w + cap_a + m] = qid;
        } else {
#pragma unroll
          for (int q = 0; q < 11; ++q) slot[q] = 0.0f;
          if (sel_idx) sel_idx[orow * sel_w + cap_a + m] = -1;
        }
      }
    }
    __syncwarp();
    // ---- coalesced write-out of the staged row
    if (bulk_out) {
      write_row_bulk(O, orow, row, obs_width, lane);
    } else {
      write_row(O, orow, row, obs_width, scale, lane);
      __syncwarp();
    }
  }
  if (bulk_out && lane == 0) bulk_row_wait();   // the staging must outlive the copies
#ifdef DS_OBS_TIMES
  {
    const unsigned long long t_now = gtimer();
    if (lane == 0 && prev_r >= 0 && prev_r < 128 && w < 8192) g_row_dur[w * 128 + prev_r] = (unsigned)(t_now - t_prev);
    if (lane == 0 && w < 8192) g_obs_times[w * kTimesW + 3 + warp] = t_now;
  }
#endif
}

#ifdef DS_OBS_STATS
}  // namespace ds
extern "C" int ds_debug_obs_stats(unsigned long long *out) {
  cudaMemcpyFromSymbol(out, ds::g_obs_stats, sizeof(ds::g_obs_stats));
  unsigned long long z[8] = {0};
  cudaMemcpyToSymbol(ds::g_obs_stats, z, sizeof(z));
  return 0;
}
namespace ds {
#endif
#ifdef DS_OBS_TIMES
}  // namespace ds
extern "C" int ds_debug_obs_times(unsigned long long *out) {
  return (int)cudaMemcpyFromSymbol(out, ds::g_obs_times, sizeof(ds::g_obs_times));
}
extern "C" int ds_debug_obs_row_dur(unsigned int *out) {
  return (int)cudaMemcpyFromSymbol(out, ds::g_row_dur, sizeof(ds::g_row_dur));
}
namespace ds {
#endif

cudaError_t configure_kernels(int max_dynamic_smem) {
  const void *ks[] = {(const void *)obs_radial_kernel<kWarpsShared, true, 16, 64, kAgentStride>,
                      (const void *)obs_radial_kernel<kWarpsSharedSmall, true, 16, 64, kAgentStride>,
                      (const void *)obs_radial_kernel<kWarpsSharedPair, true, 16, 64, kAgentStride>,
                      (const void *)obs_radial_kernel<kWarpsShared, true, 16, 64>,
                      (const void *)obs_radial_kernel<kWarpsShared, true, 0, 0>,
                      (const void *)obs_radial_kernel<kWarpsSharedSmall, true, 16, 64>,
                      (const void *)obs_radial_kernel<kWarpsSharedSmall, true, 0, 0>,
                      (const void *)obs_radial_kernel<kWarpsSharedPair, true, 16, 64>,
                      (const void *)obs_radial_kernel<kWarpsSharedPair, true, 0, 0>,
                      (const void *)obs_radial_kernel<kWarpsGlobal, false, 16, 64>,
                      (const void *)obs_radial_kernel<kWarpsGlobal, false, 0, 0>};
  for (const void *k : ks) {
    // the opt-in limit covers static + dynamic shared memory (the points'
    // mbarrier is static)
    cudaFuncAttributes fa;
    cudaError_t e = cudaFuncGetAttributes(&fa, k);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             max_dynamic_smem - (int)fa.sharedSizeBytes);
    if (e != cudaSuccess) return e;
  }
  cudaError_t e = configure_lidar_kernels(max_dynamic_smem);
  if (e != cudaSuccess) return e;
  return configure_step_kernels(max_dynamic_smem);
}

static bool obs_fixed_caps(const ds_handle *h) {
  return h->cfg.max_agents_obs == 16 && h->cfg.max_road_points_obs == 64;
}

// the agent-table stride of the shared-points kernels: kAgentStride when the
// fixed-cap variant runs on worlds of <= kAgentStride agents
static int obs_agent_stride(const ds_handle *h) {
  return obs_fixed_caps(h) && h->tab.max_agents <= kAgentStride ? kAgentStride : h->tab.max_agents;
}

void obs_plan(ds_handle *h, int max_optin) {
  if (h->cfg.obs_mode != DS_OBS_RADIAL) {
    h->obs_shared_pts = 0;
    h->obs_warps = lidar_warps();
    h->obs_smem = lidar_smem_bytes(h->cfg, h->tab.max_agents, h->obs_width);
    return;
  }
  const bool can = h->tab.gpt_xy && h->tab.grid_eps && h->tab.gpt_rec;
  const int am = obs_agent_stride(h);
  const size_t sh = obs_smem_bytes_shared(h->cfg, am, h->tab.max_points, kWarpsShared);
  const size_t sh_small = obs_smem_bytes_shared(h->cfg, am, h->tab.max_points, kWarpsSharedSmall);
  const size_t sh_pair = obs_smem_bytes_shared(h->cfg, am, h->tab.max_points, kWarpsSharedPair);
  if (can && h->tab.max_agents <= 64 && h->tab.n_worlds >= 2 * h->num_sms &&
      2 * (sh_pair + 1024) <= (size_t)kSmemPerSM) {
    h->obs_shared_pts = 1;
    h->obs_warps = kWarpsSharedPair;
    h->obs_smem = sh_pair;
  } else if (can && sh + kStaticSmem <= (size_t)max_optin) {
    h->obs_shared_pts = 1;
    h->obs_warps = kWarpsShared;
    h->obs_smem = sh;
  } else if (can && sh_small + kStaticSmem <= (size_t)max_optin) {
    h->obs_shared_pts = 1;
    h->obs_warps = kWarpsSharedSmall;
    h->obs_smem = sh_small;
  } else {
    h->obs_shared_pts = 0;
    h->obs_warps = kWarpsGlobal;
    h->obs_smem = obs_smem_bytes_global(h->cfg, h->tab.max_agents);
  }
}

struct ObsLaunch {
  const ds_handle *h;
  RadialK K;
  const uint8_t *mask;
  ObsOut O;
  const float *scale;
  int32_t *sel_idx;
  int W;
  bool fixed;
  cudaStream_t s;
};

template <int WARPS, bool SharedPts>
void launch_radial(const ObsLaunch &L) {
  const ds_handle *h = L.h;
  if (SharedPts && L.fixed && obs_agent_stride(h) == kAgentStride)
    obs_radial_kernel<WARPS, SharedPts, 16, 64, kAgentStride><<<L.W, WARPS * 32, h->obs_smem, L.s>>>(
        h->tab, h->cfg, h->st, L.K, L.mask, L.O, L.scale, L.sel_idx, h->obs_width);
  else if (L.fixed)
    obs_radial_kernel<WARPS, SharedPts, 16, 64><<<L.W, WARPS * 32, h->obs_smem, L.s>>>(
        h->tab, h->cfg, h->st, L.K, L.mask, L.O, L.scale, L.sel_idx, h->obs_width);
  else
    obs_radial_kernel<WARPS, SharedPts, 0, 0><<<L.W, WARPS * 32, h->obs_smem, L.s>>>(
        h->tab, h->cfg, h->st, L.K, L.mask, L.O, L.scale, L.sel_idx, h->obs_width);
}

cudaError_t launch_observe(const ds_handle *h, const uint8_t *mask, void *obs,
                           const float *scale, int32_t *sel_idx, cudaStream_t s) {
  if (h->cfg.obs_mode != DS_OBS_RADIAL) {
    if (sel_idx) return cudaErrorInvalidValue;   // selection indices are radial-only
    return launch_lidar(h, mask, obs, scale, s);
  }
  const bool fixed = h->cfg.max_agents_obs == 16 && h->cfg.max_road_points_obs == 64;
  const int W = h->tab.n_worlds;
  const ObsOut O{obs, h->obs_dtype, h->obs_stride};
  RadialK K;
  K.radius = h->cfg.radius;
  K.reach = K.radius + 1e-6;
  K.r2 = K.radius * K.radius;
  K.D_fp64 = (K.radius * K.radius + 1.0) * 2.4e-7;
  K.cs = h->cfg.grid_cell;
  K.inv_cs = 1.0 / K.cs;
  K.key_e = (K.radius + 1.0) * 1.2e-7;
  K.uni_a = h->uni_a;
  K.uni_c = h->uni_c;
  K.uni_p = h->uni_p;
  const ObsLaunch L{h, K, mask, O, scale, sel_idx, W, fixed, s};
  if (!h->obs_shared_pts) launch_radial<kWarpsGlobal, false>(L);
  else if (h->obs_warps == kWarpsShared) launch_radial<kWarpsShared, true>(L);
  else if (h->obs_warps == kWarpsSharedSmall) launch_radial<kWarpsSharedSmall, true>(L);
  else launch_radial<kWarpsSharedPair, true>(L);
  return cudaGetLastError();
}

}  // namespace ds
