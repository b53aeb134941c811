// gather_dev.cuh -- device functions shared by the gather kernels: hit-point
// setup, the banded fp32 predicates, the exact fp64 reference predicates,
// sector binning, F/chi2 statistics, the end-of-iteration policy and the
// per-region finalisation (pooled moments + decision + outputs).
#pragma once
#include "common.cuh"
#include "gather.cuh"

namespace fppm_b200 {

// ---------------------------------------------------------------- sectors
// n_s == 4: atan2 quadrant rule, equal to the reference's atan2 binning
// (SURVEY.md §8a exact-sector table) except when 0 < min/max < ~2^-50,
// where atan2 may round onto an axis; those are flagged ambiguous and
// resolved with the device atan2 as the best estimate.
static __device__ __forceinline__ int atan2_bin(double yu, double yv, int ns, bool &amb) {
  double theta = atan2(yv, yu);
  if (theta < 0.0) theta = da(theta, kTwoPi);
  const double t = dd(dm((double)ns, theta), kTwoPi);
  int s = (int)t;
  if (s > ns - 1) s = ns - 1;
  if (yu != 0.0 && yv != 0.0) {
    const double k = rint(t);
    if (k >= 1.0 && k <= (double)(ns - 1) && fabs(t - k) <= 1e-12 * t) amb = true;
  }
  return s;
}

static __device__ __forceinline__ int quadrant_bin(double yu, double yv, bool &amb) {
  if (yv == 0.0) return signbit(yu) ? 2 : 0;
  if (yu == 0.0) return yv > 0.0 ? 1 : 3;
  const double au = fabs(yu), av = fabs(yv);
  if (fmin(au, av) < fmax(au, av) * 0x1p-50) {
    amb = true;
    return atan2_bin(yu, yv, 4, amb);
  }
  if (yu > 0.0) return yv > 0.0 ? 0 : 3;
  return yv > 0.0 ? 1 : 2;
}

// gather.cpp:15-33 on exact fp64 plane coordinates (d2 <= r2 already holds).
static __device__ __forceinline__ int exact_sector(double yu, double yv, double r2, int na, int ns,
                                                   bool &amb) {
  const double d2 = da(dm(yu, yu), dm(yv, yv));
  int a = (int)dd(dm((double)na, d2), r2);
  if (a > na - 1) a = na - 1;
  const int s = ns == 4 ? quadrant_bin(yu, yv, amb) : atan2_bin(yu, yv, ns, amb);
  return a * ns + s;
}

// ---------------------------------------------------------------- hit point
// Full per-hit-point state (fp64 for the exact path, fp32 for the fast path).
struct Hit {
  double cx, cy, cz, nx, ny, nz;
  double3 u, v;
  double r, r2;
  double K0, K1, K2;  // throughput * albedo/pi (0 when cos_o <= 0)
  float chx, chy, chz, clx, cly, clz;  // center as float hi + lo
  float nfx, nfy, nfz, ufx, ufy, ufz, vfx, vfy, vfz;
  float r2f, lim_hi, lim_lo, band_y, guard_f;
  float guard_ceil;  // smallest float f with (double)f >= guard
  float qa_scale;  // n_a / r2 (fp32)
  uint32_t h, eye;
  bool fast, gray;
};

// Register-resident subset used by the candidate loops.
// fp64 subset of Hit for the exact path and pair values (sparse kernel smem)
struct HitX {
  double cx, cy, cz, nx, ny, nz;
  double3 u, v;
  double r, r2, K0, K1, K2;
};

struct HitF {
  float chx, chy, chz, clx, cly, clz;
  float nfx, nfy, nfz, ufx, ufy, ufz, vfx, vfy, vfz;
  float lim_hi, lim_lo, band_y, guard_f, qa_scale, r, guard_ceil;
  uint32_t eye;
  int na, ns;
  bool fast;
};

static __device__ __forceinline__ void make_hit(const GatherArgs &A, uint32_t h, Hit &H) {
  const double r = A.radius[h];
  H.h = h;
  H.r = r;
  H.r2 = dm(r, r);
  const double3 c = A.pos[h];
  const double3 n = A.nrm[h];
  H.cx = c.x; H.cy = c.y; H.cz = c.z;
  H.nx = n.x; H.ny = n.y; H.nz = n.z;
  eframe(n.x, n.y, n.z, H.u, H.v);  // move_to (gather.cpp:54-57)
  const double3 K = A.K[h];
  H.K0 = K.x; H.K1 = K.y; H.K2 = K.z;
  H.gray = K.x == K.y && K.y == K.z;
  H.eye = A.eye_depth[h];
  H.chx = __double2float_rn(c.x); H.chy = __double2float_rn(c.y); H.chz = __double2float_rn(c.z);
  H.clx = __double2float_rn(c.x - (double)H.chx);
  H.cly = __double2float_rn(c.y - (double)H.chy);
  H.clz = __double2float_rn(c.z - (double)H.chz);
  H.nfx = (float)n.x; H.nfy = (float)n.y; H.nfz = (float)n.z;
  H.ufx = (float)H.u.x; H.ufy = (float)H.u.y; H.ufz = (float)H.u.z;
  H.vfx = (float)H.v.x; H.vfy = (float)H.v.y; H.vfz = (float)H.v.z;
  H.r2f = (float)H.r2;
  H.band_y = 1e-5f * (float)r;
  H.guard_f = (float)A.guard;
  H.guard_ceil = __double2float_ru(A.guard);
  H.qa_scale = (float)A.na / H.r2f;
  const double cmax = fmax(fabs(c.x), fmax(fabs(c.y), fabs(c.z)));
  const double nn = edot(n.x, n.y, n.z, n.x, n.y, n.z);
  H.fast = H.r2f > 1e-30f && H.r2f < 1e30f && cmax <= 1e6 * r && nn > 0.999 && nn < 1.001;
  // certain-reject / certain-accept limits for squared distances
  H.lim_hi = H.fast ? H.r2f + 2e-5f * H.r2f : __int_as_float(0x7f800000);
  H.lim_lo = H.fast ? H.r2f - 2e-5f * H.r2f : -1.0f;
}

static __device__ __forceinline__ HitF hitf(const Hit &H, int na, int ns) {
  HitF F;
  F.chx = H.chx; F.chy = H.chy; F.chz = H.chz; F.clx = H.clx; F.cly = H.cly; F.clz = H.clz;
  F.nfx = H.nfx; F.nfy = H.nfy; F.nfz = H.nfz;
  F.ufx = H.ufx; F.ufy = H.ufy; F.ufz = H.ufz;
  F.vfx = H.vfx; F.vfy = H.vfy; F.vfz = H.vfz;
  F.lim_hi = H.lim_hi; F.lim_lo = H.lim_lo; F.band_y = H.band_y; F.guard_f = H.guard_f;
  F.qa_scale = H.qa_scale; F.r = (float)H.r; F.guard_ceil = H.guard_ceil;
  F.eye = H.eye; F.na = na; F.ns = ns; F.fast = H.fast;
  return F;
}

// Full reference evaluation of one candidate in fp64 (no FMA).
// Returns true when the photon is accepted; sets sector and cos_pos.
template <class HT>
static __device__ __noinline__ bool exact_pair(const HT &H, float4 a, float4 b, float4 c2, int na,
                                               int ns, double guard, int &sector, bool &cos_pos,
                                               bool &amb) {
  const double dx = ds((double)a.x, H.cx), dy = ds((double)a.y, H.cy),
               dz = ds((double)a.z, H.cz);
  if (!(edot(dx, dy, dz, dx, dy, dz) <= H.r2)) return false;                       // :76
  if (edot((double)b.x, (double)b.y, (double)b.z, H.nx, H.ny, H.nz) < guard) return false;  // :397
  const double yu = edot(dx, dy, dz, H.u.x, H.u.y, H.u.z);
  const double yv = edot(dx, dy, dz, H.v.x, H.v.y, H.v.z);
  if (da(dm(yu, yu), dm(yv, yv)) > H.r2) return false;                           // :399
  const double ci = edot((double)b.w, (double)c2.x, (double)c2.y, H.nx, H.ny, H.nz);
  cos_pos = !(ci <= 0.0);                                                        // bsdf.cpp:58
  sector = exact_sector(yu, yv, H.r2, na, ns, amb);
  return true;
}

// Same, returning packed flags (no address-taken locals at the call site):
// bit0 accepted, bit1 cos_i > 0, bit2 ambiguous sector, bits 8..15 sector.
static __device__ __noinline__ uint32_t exact_pair_packed(const Hit &H, float4 a, float4 b,
                                                         float4 c2, int na, int ns, double guard) {
  int sector = 0;
  bool cos_pos = false, amb = false;
  if (!exact_pair(H, a, b, c2, na, ns, guard, sector, cos_pos, amb)) return 0u;
  return 1u | (cos_pos ? 2u : 0u) | (amb ? 4u : 0u) | ((uint32_t)sector << 8);
}

// Candidate pre-test: false only when the reference certainly rejects the
// pair (ball, depth or disk).  fp32 with error bands; see flush_pair.
static __device__ __forceinline__ bool test_pair(const HitF &F, float4 a, uint32_t max_depth) {
  const float dx = (a.x - F.chx) - F.clx;
  const float dy = (a.y - F.chy) - F.cly;
  const float dz = (a.z - F.chz) - F.clz;
  const float d2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
  if (!(d2 <= F.lim_hi)) return false;                             // photon_map.cpp:76
  if (F.eye + __float_as_uint(a.w) > max_depth) return false;      // integrator.cpp:396
  const float yu = fmaf(dx, F.ufx, fmaf(dy, F.ufy, dz * F.ufz));
  const float yv = fmaf(dx, F.vfx, fmaf(dy, F.vfy, dz * F.vfz));
  return fmaf(yu, yu, yv * yv) <= F.lim_hi;                        // integrator.cpp:399
}

// Full decision for a pre-tested candidate: every predicate in fp32 with a
// rigorous error band; anything inside a band goes to the exact fp64 path.
template <class HT>
static __device__ __forceinline__ bool flush_pair(const HitF &F, const HT &Hs, float4 a, float4 b,
                                                  float4 c2, double guard, int &sector,
                                                  bool &cos_pos, uint32_t &n_exact,
                                                  uint32_t &n_amb) {
  const float dx = (a.x - F.chx) - F.clx;
  const float dy = (a.y - F.chy) - F.cly;
  const float dz = (a.z - F.chz) - F.clz;
  const float d2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
  const float yu = fmaf(dx, F.ufx, fmaf(dy, F.ufy, dz * F.ufz));
  const float yv = fmaf(dx, F.vfx, fmaf(dy, F.vfy, dz * F.vfz));
  const float yy = fmaf(yu, yu, yv * yv);
  bool ex = !F.fast || !(d2 < F.lim_lo) || !(yy < F.lim_lo);
  // normal guard (integrator.cpp:397)
  const float gd = fmaf(b.x, F.nfx, fmaf(b.y, F.nfy, b.z * F.nfz));
  const float gb = 2e-6f * (fabsf(b.x * F.nfx) + fabsf(b.y * F.nfy) + fabsf(b.z * F.nfz)) + 1e-30f;
  if (!ex && gd < F.guard_f - gb) return false;
  ex = ex || !(gd >= F.guard_f + gb);
  // cos_i > 0 of the Lambertian eval (bsdf.cpp:56-58)
  const float ci = fmaf(b.w, F.nfx, fmaf(c2.x, F.nfy, c2.y * F.nfz));
  const float cb = 2e-6f * (fabsf(b.w * F.nfx) + fabsf(c2.x * F.nfy) + fabsf(c2.y * F.nfz)) + 1e-30f;
  ex = ex || !(fabsf(ci) > cb);
  cos_pos = ci > 0.0f;
  // sector (gather.cpp:15-33)
  int s_ang;
  if (F.ns == 4) {
    ex = ex || !(fabsf(yu) > F.band_y) || !(fabsf(yv) > F.band_y);
    s_ang = yu > 0.0f ? (yv > 0.0f ? 0 : 3) : (yv > 0.0f ? 1 : 2);
  } else {
    const float ay = fmaxf(fabsf(yu), fabsf(yv));
    ex = ex || !(ay > 1e-3f * F.r);
    float th = atan2f(yv, yu);
    if (th < 0.0f) th += 6.2831853f;
    const float tt = (float)F.ns * th * 0.15915494f;
    const float kk = rintf(tt);
    ex = ex || (kk >= 1.0f && kk <= (float)(F.ns - 1) && fabsf(tt - kk) < 4e-3f);
    s_ang = min((int)tt, F.ns - 1);
  }
  int a_ring = 0;
  if (F.na > 1) {
    const float qa = yy * F.qa_scale;
    const float kq = rintf(qa);
    ex = ex || (kq >= 1.0f && kq <= (float)(F.na - 1) && fabsf(qa - kq) < 1e-4f * (float)F.na);
    a_ring = min((int)qa, F.na - 1);
  }
  sector = a_ring * F.ns + s_ang;
  if (ex) {
    ++n_exact;
    bool amb = false;
    if (!exact_pair(Hs, a, b, c2, F.na, F.ns, guard, sector, cos_pos, amb)) return false;
    if (amb) ++n_amb;
  }
  return true;
}

// Fast-path sector of a surviving candidate; false when any band is hit.
static __device__ __forceinline__ bool fast_sector(const HitF &F, float yu, float yv, float yy, int &sector) {
  bool ok;
  int s_ang;
  if (F.ns == 4) {
    ok = fabsf(yu) > F.band_y && fabsf(yv) > F.band_y;
    s_ang = yu > 0.0f ? (yv > 0.0f ? 0 : 3) : (yv > 0.0f ? 1 : 2);
  } else {
    ok = fmaxf(fabsf(yu), fabsf(yv)) > 1e-3f * F.r;
    float th = atan2f(yv, yu);
    if (th < 0.0f) th += 6.2831853f;
    const float tt = (float)F.ns * th * 0.15915494f;
    const float kk = rintf(tt);
    ok = ok && !(kk >= 1.0f && kk <= (float)(F.ns - 1) && fabsf(tt - kk) < 4e-3f);
    s_ang = min((int)tt, F.ns - 1);
  }
  int a_ring = 0;
  if (F.na > 1) {
    const float qa = yy * F.qa_scale;
    const float kq = rintf(qa);
    ok = ok && !(kq >= 1.0f && kq <= (float)(F.na - 1) && fabsf(qa - kq) < 1e-4f * (float)F.na);
    a_ring = min((int)qa, F.na - 1);
  }
  sector = a_ring * F.ns + s_ang;
  return ok;
}



// Test phase: ball and depth only (photon_map.cpp:76, integrator.cpp:396).
// False only when the reference certainly rejects the pair; disk, sector and
// the remaining filters are decided in the flush, where every lane holds a
// survivor.
static __device__ __forceinline__ bool ball_pass(const HitF &F, bool lo_zero, float4 a, uint32_t max_depth) {
  float dx = a.x - F.chx, dy = a.y - F.chy, dz = a.z - F.chz;
  if (!lo_zero) {
    dx -= F.clx;
    dy -= F.cly;
    dz -= F.clz;
  }
  const float d2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
  return d2 <= F.lim_hi && F.eye + __float_as_uint(a.w) <= max_depth;
}


// ---------------------------------------------------------------- accumulators
// Per-lane fp64 sector accumulators must stay in registers.  Written as
// "if (sector == k) acc[k] += v" the optimiser proves that exactly one k
// matches and rewrites the chain into acc[sector] += v, a dynamically indexed
// access that demotes the whole array to local memory.  Each case below uses
// a distinct inline-asm add (the case number is part of the asm text), so no
// two cases can be merged and every index stays a compile-time constant.
#define FPPM_ADD_F64(x, y, k) asm("add.rn.f64 %0, %0, %1; // acc " #k : "+d"(x) : "d"(y))
#define FPPM_ADD_U32(x, y, k) asm("add.u32 %0, %0, %1; // cnt " #k : "+r"(x) : "r"(y))

// warp-uniform sector g: an indirect branch to one case (no G-way predication)
#define FPPM_ACC_CASE(k)                    \
  case k:                                   \
    if constexpr ((k) < GMAX) {             \
      FPPM_ADD_F64(s[k], v, s##k);          \
      FPPM_ADD_F64(q[k], vv, q##k);         \
      FPPM_ADD_U32(c[k], n, c##k);          \
    }                                       \
    break;
template <int GMAX>
__device__ __forceinline__ void acc_uniform(double (&s)[GMAX], double (&q)[GMAX],
                                            uint32_t (&c)[GMAX], int g, double v, double vv,
                                            uint32_t n) {
  switch (g) {
    FPPM_ACC_CASE(0) FPPM_ACC_CASE(1) FPPM_ACC_CASE(2) FPPM_ACC_CASE(3)
    FPPM_ACC_CASE(4) FPPM_ACC_CASE(5) FPPM_ACC_CASE(6) FPPM_ACC_CASE(7)
    FPPM_ACC_CASE(8) FPPM_ACC_CASE(9) FPPM_ACC_CASE(10) FPPM_ACC_CASE(11)
    FPPM_ACC_CASE(12) FPPM_ACC_CASE(13) FPPM_ACC_CASE(14) FPPM_ACC_CASE(15)
    FPPM_ACC_CASE(16) FPPM_ACC_CASE(17) FPPM_ACC_CASE(18) FPPM_ACC_CASE(19)
    FPPM_ACC_CASE(20) FPPM_ACC_CASE(21) FPPM_ACC_CASE(22) FPPM_ACC_CASE(23)
    FPPM_ACC_CASE(24) FPPM_ACC_CASE(25) FPPM_ACC_CASE(26) FPPM_ACC_CASE(27)
    FPPM_ACC_CASE(28) FPPM_ACC_CASE(29) FPPM_ACC_CASE(30) FPPM_ACC_CASE(31)
    default: break;
  }
}
#undef FPPM_ACC_CASE

// per-lane sector: G predicated adds with distinct asm per case
#define FPPM_PRED_CASE(k)                                   \
  if constexpr ((k) < GMAX) {                               \
    if (sector == (k)) {                                    \
      FPPM_ADD_F64(s[k], v, p##k);                          \
      FPPM_ADD_F64(q[k], vv, pq##k);                        \
    }                                                       \
  }
template <int GMAX>
__device__ __forceinline__ void acc_pred(double (&s)[GMAX], double (&q)[GMAX], int sector, double v,
                                         double vv) {
  FPPM_PRED_CASE(0) FPPM_PRED_CASE(1) FPPM_PRED_CASE(2) FPPM_PRED_CASE(3)
  FPPM_PRED_CASE(4) FPPM_PRED_CASE(5) FPPM_PRED_CASE(6) FPPM_PRED_CASE(7)
  FPPM_PRED_CASE(8) FPPM_PRED_CASE(9) FPPM_PRED_CASE(10) FPPM_PRED_CASE(11)
  FPPM_PRED_CASE(12) FPPM_PRED_CASE(13) FPPM_PRED_CASE(14) FPPM_PRED_CASE(15)
  FPPM_PRED_CASE(16) FPPM_PRED_CASE(17) FPPM_PRED_CASE(18) FPPM_PRED_CASE(19)
  FPPM_PRED_CASE(20) FPPM_PRED_CASE(21) FPPM_PRED_CASE(22) FPPM_PRED_CASE(23)
  FPPM_PRED_CASE(24) FPPM_PRED_CASE(25) FPPM_PRED_CASE(26) FPPM_PRED_CASE(27)
  FPPM_PRED_CASE(28) FPPM_PRED_CASE(29) FPPM_PRED_CASE(30) FPPM_PRED_CASE(31)
}
#undef FPPM_PRED_CASE

static __device__ __forceinline__ double warp_sum(double x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(kFull, x, o);
  return x;
}
static __device__ __forceinline__ uint32_t warp_sum(uint32_t x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(kFull, x, o);
  return x;
}

// ---------------------------------------------------------------- VCM+ merge weight
// path.cpp:11-13
static __device__ __forceinline__ double mis_pow_dev(double beta, double x) {
  return beta == 1.0 ? x : pow(x, beta);
}
// path.cpp:103-111 with vc_factor (path.cpp:22-24) of eta_vm = n_vm pi r^2
// (integrator.cpp:503), in the reference's operation order without FMA.
static __device__ __forceinline__ double mis_weight_merge_dev(int n_vm, double beta, double r, double e_vcm,
                                                              double e_vm, double l_vcm, double l_vm,
                                                              double fwd, double rev) {
  const double eta = dm(dm(dm((double)n_vm, kPi), r), r);
  const double vcf = eta > 0.0 ? mis_pow_dev(beta, dd(1.0, eta)) : 0.0;
  const double w_light = da(dm(l_vcm, vcf), dm(l_vm, mis_pow_dev(beta, fwd)));
  const double w_camera = da(dm(e_vcm, vcf), dm(e_vm, mis_pow_dev(beta, rev)));
  return dd(1.0, da(da(w_light, 1.0), w_camera));
}

// ---------------------------------------------------------------- end_iteration
// f_statistic (stat_tests.cpp:12-44) with the reference's operation order.
static __device__ double f_statistic_dev(const double *sum, const double *sq, int n, uint64_t m) {
  const double md = (double)m;
  double grand = 0.0;
  for (int i = 0; i < n; ++i) grand = da(grand, sum[i]);
  const double grand_mean = dd(grand, dm(md, (double)n));
  double between = 0.0, within = 0.0;
  for (int i = 0; i < n; ++i) {
    const double mean = dd(sum[i], md);
    const double dev = ds(mean, grand_mean);
    between = da(between, dm(dm(md, dev), dev));
    within = da(within, ds(sq[i], dd(dm(sum[i], sum[i]), md)));
  }
  between = between < 0.0 ? 0.0 : between;
  within = within < 0.0 ? 0.0 : within;
  if (between == 0.0) return 0.0;
  if (within == 0.0) return __longlong_as_double(0x7ff0000000000000ll);
  const double d1 = (double)(n - 1);
  const double d2 = dm((double)n, ds(md, 1.0));
  return dd(dd(between, d1), dd(within, d2));
}

// stat_tests.cpp:100-116
static __device__ double chi2_statistic_dev(const unsigned long long *cnt, int n) {
  unsigned long long total = 0;
  for (int i = 0; i < n; ++i) total += cnt[i];
  const double expected = dd((double)total, (double)n);
  double chi2 = 0.0;
  for (int i = 0; i < n; ++i) {
    const double dev = ds((double)cnt[i], expected);
    chi2 = da(chi2, dd(dm(dev, dev), expected));
  }
  return chi2;
}

// gather.cpp:74-144. cnt/sum/sq hold the pooled moments [C][G]; they are
// cleared on rejection.  Returns the flags (bit0 tested, bit1 rejected).
static __device__ uint8_t end_of_iteration(const EndParams &P, int G, int C, double &r, uint32_t &t,
                                           unsigned long long *cnt, double *sum, double *sq,
                                           double &stat, double &critical) {
  stat = 0.0;
  critical = 0.0;
  if (P.policy == FPPM_POLICY_SCHEDULE) {  // :138-144
    r = P.sched_next;
    ++t;
    return 0;
  }
  bool reject = false, tested = false;
  if (P.override_decision != FPPM_OVERRIDE_NONE) {
    reject = P.override_decision == FPPM_OVERRIDE_ALWAYS_REJECT;
  } else if (P.policy == FPPM_POLICY_CHI2) {  // :114-136
    unsigned long long total = 0;
    for (int s = 0; s < G; ++s) total += cnt[s];
    if (total != 0) {
      stat = chi2_statistic_dev(cnt, G);
      critical = P.chi2_crit;
      reject = stat > critical;
      tested = true;
    }
  } else {  // F-test :90-112
    const unsigned long long m = (unsigned long long)t * P.J;
    if (m >= 2) {
      const uint32_t ti = t < P.crit_len ? t : P.crit_len - 1;
      const double crit = P.crit[ti];
      for (int c = 0; c < C; ++c) {
        const double f = f_statistic_dev(sum + c * G, sq + c * G, G, m);
        reject = reject || (f > crit);
        stat = stat < f ? f : stat;  // std::max(stat, f)
        critical = crit;
      }
      tested = true;
    }
  }
  if (reject) {  // apply_decision :74-88
    const double kr = dm(P.k, r);
    r = kr < P.floor_next ? P.floor_next : kr;
    for (int i = 0; i < G * C; ++i) {
      cnt[i] = 0;
      sum[i] = 0.0;
      sq[i] = 0.0;
    }
    t = 1;
  } else {
    ++t;
  }
  return (uint8_t)((tested ? 1 : 0) | (reject ? 2 : 0));
}

// Pools one region's iteration moments with its stored moments, runs the
// end-of-iteration policy and writes every output (one thread).  p0..p2 are
// the sums of photon power over accepted pairs with cos_i > 0; the flux is
// K * p (integrator.cpp:448-449).
template <int GMAX, int CH>
static __device__ __forceinline__ void finalize_hit(const GatherArgs &A, uint32_t h,
                                                 const uint32_t (&cnt)[GMAX],
                                                 const double (&sm)[CH][GMAX],
                                                 const double (&sq)[CH][GMAX], double p0, double p1,
                                                 double p2, uint32_t &n_tested, uint32_t &n_rejected,
                                                 double &rmax) {
  const int G = A.na * A.ns;
  const int CG = G * CH;
  if (A.delta_out) {  // option B: hand the partial sums to the owner
    double *d = A.delta_out + (size_t)h * (size_t)(G + 2 * CG + 3);
#pragma unroll
    for (int g = 0; g < GMAX; ++g)
      if (g < G) d[g] = (double)cnt[g];
#pragma unroll
    for (int c = 0; c < CH; ++c)
#pragma unroll
      for (int g = 0; g < GMAX; ++g)
        if (g < G) {
          d[G + c * G + g] = sm[c][g];
          d[G + CG + c * G + g] = sq[c][g];
        }
    d[G + 2 * CG] = p0;
    d[G + 2 * CG + 1] = p1;
    d[G + 2 * CG + 2] = p2;
    return;
  }
  const size_t base = (size_t)h * CG;
  const double r = A.radius[h];
  uint32_t t = A.t[h];
  const bool gathered = A.gathered == nullptr || A.gathered[h] != 0;
  const double3 K = A.K[h];
  // FPPM: p = sum of photon power over accepted pairs (flux = K p); VCM+:
  // p = sum of the weighted values themselves (integrator.cpp:617)
  const double fl0 = A.vcm ? p0 : dm(K.x, p0), fl1 = A.vcm ? p1 : dm(K.y, p1),
               fl2 = A.vcm ? p2 : dm(K.z, p2);
  double r_new = r;
  double stat = 0.0, critical = 0.0;
  uint8_t flags = 0;
  uint32_t accepted = 0;
  for (int g = 0; g < GMAX; ++g) accepted += g < G ? cnt[g] : 0u;
  if (gathered) {
    unsigned long long pc[GMAX * CH];
    double ps[GMAX * CH], pq[GMAX * CH];
    // compile-time indices into the register accumulators (runtime indexing
    // would demote them to local memory for the whole kernel)
#pragma unroll
    for (int c = 0; c < CH; ++c)
#pragma unroll
      for (int g = 0; g < GMAX; ++g) {
        if (g < G) {
          const size_t o = base + (size_t)c * G + g;
          pc[c * G + g] = A.st_cnt[o] + cnt[g];
          ps[c * G + g] = A.st_sum[o] + sm[c][g];
          pq[c * G + g] = A.st_sq[o] + sq[c][g];
        }
      }
    if (A.snap_cnt) {
      for (int i = 0; i < CG; ++i) {
        A.snap_cnt[base + i] = pc[i];
        A.snap_sum[base + i] = ps[i];
        A.snap_sq[base + i] = pq[i];
      }
    }
    flags = end_of_iteration(A.end, G, CH, r_new, t, pc, ps, pq, stat, critical);
    for (int i = 0; i < CG; ++i) {
      A.st_cnt[base + i] = pc[i];
      A.st_sum[base + i] = ps[i];
      A.st_sq[base + i] = pq[i];
    }
    A.radius[h] = r_new;
    A.t[h] = t;
  } else if (A.end.policy == FPPM_POLICY_SCHEDULE) {
    // the global schedule (SPPM / VCM: one radius for every pixel,
    // integrator.cpp:159-170 radius_now_) moves on whether or not the pixel
    // gathered: schedule_end_iteration (gather.cpp:138-144) for every region
    r_new = A.end.sched_next;
    A.radius[h] = r_new;
    A.t[h] = A.t[h] + 1;
    if (A.snap_cnt)
      for (int i = 0; i < CG; ++i) {
        A.snap_cnt[base + i] = A.st_cnt[base + i];
        A.snap_sum[base + i] = A.st_sum[base + i];
        A.snap_sq[base + i] = A.st_sq[base + i];
      }
  } else if (A.snap_cnt) {  // no observation: state holds (integrator.cpp:483-488)
    for (int i = 0; i < CG; ++i) {
      A.snap_cnt[base + i] = A.st_cnt[base + i];
      A.snap_sum[base + i] = A.st_sum[base + i];
      A.snap_sq[base + i] = A.st_sq[base + i];
    }
  }
  n_tested += flags & 1;
  n_rejected += (flags >> 1) & 1;
  rmax = fmax(rmax, r_new);
  if (A.o_gather_r) A.o_gather_r[h] = r;
  if (A.o_flags) A.o_flags[h] = flags;
  if (A.o_stat) A.o_stat[h] = stat;
  if (A.o_crit) A.o_crit[h] = critical;
  if (A.o_accepted) A.o_accepted[h] = accepted;
  if (A.o_flux) {
    A.o_flux[3 * (size_t)h] = fl0;
    A.o_flux[3 * (size_t)h + 1] = fl1;
    A.o_flux[3 * (size_t)h + 2] = fl2;
  }
  if (A.o_radiance) {
    const double denom = dm(dm(dm(kPi, r), r), (double)A.end.J);  // :452-453
    A.o_radiance[3 * (size_t)h] = gathered ? (float)dd(fl0, denom) : 0.0f;
    A.o_radiance[3 * (size_t)h + 1] = gathered ? (float)dd(fl1, denom) : 0.0f;
    A.o_radiance[3 * (size_t)h + 2] = gathered ? (float)dd(fl2, denom) : 0.0f;
  }
}

// ---------------------------------------------------------------- fine-cell geometry
// slab layout: S = kFineS fine cells per reference cell (planar photon sets)
static __device__ __forceinline__ bool slab_grid(const GridHeader &g) { return g.S == kFineS; }

// (fine boxes, runs clipped to the ball's chord; gather_fine.cu, gather.cu)
struct FBox {
  int x0, x1, y0, y1, z0, z1;
};

// fine-cell range of one axis: the box [c - m, c + m] intersected with the
// reference 27-neighbourhood of the home cell and the table.
static __device__ __forceinline__ bool fine_axis(const GridHeader &g, double c, double m,
                                                 long long o, long long n, int &lo, int &hi) {
  const double hc = dm(c, g.inv);
  if (!(fabs(hc) < 4.0e15)) return false;
  const long long h = (long long)floor(hc);
  const long long H = h >> g.shift;  // reference cell (floor division by S)
  long long a = (H - 1) * (long long)g.S, b = (H + 2) * (long long)g.S - 1;
  const long long a2 = (long long)floor(dm(ds(c, m), g.inv));
  const long long b2 = (long long)floor(dm(da(c, m), g.inv));
  a = (a > a2 ? a : a2) - o;
  b = (b < b2 ? b : b2) - o;
  if (a < 0) a = 0;
  if (b > n - 1) b = n - 1;
  lo = (int)a;
  hi = (int)b;
  return a <= b;
}

// Fine cells that can hold an accepted photon of the ball (c, r): the margin
// covers the rounding of the fp64 ball test (|p - c| <= r (1 + 2^-50)) and of
// c +- m.
static __device__ __forceinline__ bool fine_box(const GridHeader &g, double cx, double cy, double cz,
                                                double r, FBox &b) {
  if (g.n == 0) return false;
  const double cm = fmax(fabs(cx), fmax(fabs(cy), fabs(cz)));
  const double m = da(da(r, dm(r, 1e-9)), dm(cm, 4e-16));
  return fine_axis(g, cx, m, g.ix0, g.nx, b.x0, b.x1) && fine_axis(g, cy, m, g.iy0, g.ny, b.y0, b.y1) &&
         fine_axis(g, cz, m, g.iz0, g.nz, b.z0, b.z1);
}

static __device__ __forceinline__ unsigned long long fid(const GridHeader &g, long long x, long long y,
                                                         long long z) {
  return (unsigned long long)((x * g.ny + y) * g.nz + z);
}

// Key range of piece p of a union box (slab: one fine row over the union's y
// range and every z; otherwise one (x, y) column over the union's z range).
static __device__ __forceinline__ void piece_keys(const GridHeader &g, const FBox &u, int p,
                                                  unsigned long long &k0, unsigned long long &k1) {
  if (slab_grid(g)) {
    const long long x = u.x0 + p;
    k0 = fid(g, x, u.y0, 0);
    k1 = fid(g, x, u.y1, g.nz - 1);
  } else {
    const int nyu = u.y1 - u.y0 + 1;
    const long long x = u.x0 + p / nyu, y = u.y0 + p % nyu;
    k0 = fid(g, x, y, u.z0);
    k1 = fid(g, x, y, u.z1);
  }
}
static __device__ __forceinline__ int piece_count(const GridHeader &g, const FBox &u) {
  return slab_grid(g) ? u.x1 - u.x0 + 1 : (u.x1 - u.x0 + 1) * (u.y1 - u.y0 + 1);
}
// runs of a box: one fine row per x in the slab layout (S = kFineS, every z
// of the row), one (x, y) column otherwise (3D grids, S = 1 or 2)
static __device__ __forceinline__ int run_count(const GridHeader &g, const FBox &b) {
  return slab_grid(g) ? b.x1 - b.x0 + 1 : (b.x1 - b.x0 + 1) * (b.y1 - b.y0 + 1);
}

// Distance from c to the fine slab [X f, (X + 1) f) of one axis (f = 1 / inv),
// shortened by `slack` (never negative).  Photons stored in fine cell X
// satisfy floor(x * inv) = X in fp64; slack covers that rounding.
static __device__ __forceinline__ double slab_gap(double c, long long X, double f, double slack) {
  const double lo = (double)X * f, hi = (double)(X + 1) * f;  // f = 1 / inv (rounding << slack)
  const double d = c < lo ? lo - c : (c > hi ? c - hi : 0.0);
  return d > slack ? d - slack : 0.0;
}

// Run j of box b clipped to the chord of the ball (c, m) (m: fine_box's
// margin radius).  A photon accepted by the reference ball test lies within
// m of c in the plane of the two outer axes, so in column x (slab layout)
// only the rows |y - c.y| <= sqrt(m^2 - gap_x^2) can hold it, and in an
// (x, y) column (reference layout) only |z - c.z| <= sqrt(m^2 - gap_xy^2).
// The bounds are widened by `slack` (>> fp64 rounding) and mapped through the
// same monotone floor(v * inv) as the photons' own cells, so no accepted
// photon is ever cut.  Returns false when the run is empty.
static __device__ __forceinline__ bool run_keys_clipped(const GridHeader &g, const FBox &b, int j, double cx,
                                                        double cy, double cz, double m,
                                                        unsigned long long &k0, unsigned long long &k1) {
  const double cm = fmax(fabs(cx), fmax(fabs(cy), fabs(cz)));
  const double f = 1.0 / g.inv;
  const double slack = 1e-6 * f + m * 1e-7 + cm * 1e-12;
  const double m2 = m * m;
  if (slab_grid(g)) {
    const long long x = b.x0 + j;
    const double gx = slab_gap(cx, x + g.ix0, f, slack);
    const double h2 = m2 - gx * gx;
    if (!(h2 >= 0.0)) return false;
    const double hy = sqrt(h2) + slack;
    long long y0 = (long long)floor(dm(ds(cy, hy), g.inv)) - g.iy0;
    long long y1 = (long long)floor(dm(da(cy, hy), g.inv)) - g.iy0;
    if (y0 < b.y0) y0 = b.y0;
    if (y1 > b.y1) y1 = b.y1;
    if (y0 > y1) return false;
    k0 = fid(g, x, y0, 0);
    k1 = fid(g, x, y1, g.nz - 1);
    return true;
  }
  const int nyb = b.y1 - b.y0 + 1;
  const long long x = b.x0 + j / nyb, y = b.y0 + j % nyb;
  const double gx = slab_gap(cx, x + g.ix0, f, slack), gy = slab_gap(cy, y + g.iy0, f, slack);
  const double h2 = m2 - gx * gx - gy * gy;
  if (!(h2 >= 0.0)) return false;
  const double hz = sqrt(h2) + slack;
  long long z0 = (long long)floor(dm(ds(cz, hz), g.inv)) - g.iz0;
  long long z1 = (long long)floor(dm(da(cz, hz), g.inv)) - g.iz0;
  if (z0 < b.z0) z0 = b.z0;
  if (z1 > b.z1) z1 = b.z1;
  if (z0 > z1) return false;
  k0 = fid(g, x, y, z0);
  k1 = fid(g, x, y, z1);
  return true;
}

}  // namespace fppm_b200
