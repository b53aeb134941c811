// gather.cu -- warp-cooperative photon gather + streaming ANOVA F-test.
//
// One warp owns one hit point (GatherRegion) at a time, pulled from a global
// work counter.  The warp resolves the 27-cell neighbourhood of the hit
// point's cell (photon_map.cpp:65-77) as 9 contiguous sorted ranges (the
// three z-cells of each (dx, dy) column are adjacent in key order), flattens
// them, and each lane tests one candidate per round:
//
//   ball      |p - c|^2 <= r^2                      photon_map.cpp:76
//   depth     eye_depth + p.depth <= max_depth       integrator.cpp:396
//   guard     dot(p.n, n) >= cos 30 deg              integrator.cpp:397
//   disk      y.u^2 + y.v^2 <= r^2, y = map_to_unified(c, p, frame)  :398-399
//   value     (throughput * f) * p.power, f = albedo/pi if cos_o, cos_i > 0
//   sector    sector_index(y, r, n_a, n_s)           gather.cpp:15-33
//
// Every predicate is first evaluated in fp32 with a rigorous error band; a
// candidate whose fp32 value falls inside a band is re-evaluated on the
// exact path in fp64 without FMA, reproducing the reference's x86-64 fp64
// arithmetic bit for bit.  Per-sector {count, sum, sum^2} and the RGB flux
// are accumulated per lane in fp64 registers and reduced with warp shuffles
// in a fixed lane order (deterministic run to run).  Lane 0 then pools them
// with the region's stored moments and runs end_iteration
// (gather.cpp:90-112, apply_decision :74-88) in the same kernel.
#include "common.cuh"
#include "gather.cuh"

namespace fppm_b200 {

// ---------------------------------------------------------------- sectors
// n_s == 4: atan2 quadrant rule, equal to the reference's atan2 binning
// (SURVEY.md §8a exact-sector table) except when 0 < min/max < ~2^-50,
// where atan2 may round onto an axis; those are flagged ambiguous and
// resolved with the device atan2 as the best estimate.
__device__ __forceinline__ int atan2_bin(double yu, double yv, int ns, bool &amb) {
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

__device__ __forceinline__ int quadrant_bin(double yu, double yv, bool &amb) {
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
__device__ __forceinline__ int exact_sector(double yu, double yv, double r2, int na, int ns,
                                            bool &amb) {
  const double d2 = da(dm(yu, yu), dm(yv, yv));
  int a = (int)dd(dm((double)na, d2), r2);
  if (a > na - 1) a = na - 1;
  const int s = ns == 4 ? quadrant_bin(yu, yv, amb) : atan2_bin(yu, yv, ns, amb);
  return a * ns + s;
}

// ---------------------------------------------------------------- hit point
struct Hit {
  double cx, cy, cz, nx, ny, nz;
  double3 u, v;
  double r, r2;
  double K0, K1, K2;  // throughput * albedo/pi (0 when cos_o <= 0)
  float chx, chy, chz, clx, cly, clz;  // center as float hi + lo
  float nfx, nfy, nfz, ufx, ufy, ufz, vfx, vfy, vfz;
  float r2f, lim_hi, lim_lo, band_y, guard_f;
  float qa_scale;  // n_a / r2 (fp32)
  bool fast;
  uint32_t eye;
};

// Full reference evaluation of one candidate in fp64 (no FMA).
// Returns true when the photon is accepted; sets sector and cos_pos.
__device__ __noinline__ bool exact_pair(const Hit &H, float4 a, float4 b, float4 c2, int na,
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

__device__ __forceinline__ double warp_sum(double x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(kFull, x, o);
  return x;
}
__device__ __forceinline__ uint32_t warp_sum(uint32_t x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(kFull, x, o);
  return x;
}

// ---------------------------------------------------------------- end_iteration
// f_statistic (stat_tests.cpp:12-44) with the reference's operation order.
__device__ double f_statistic_dev(const double *sum, const double *sq, int n, uint64_t m) {
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
__device__ double chi2_statistic_dev(const unsigned long long *cnt, int n) {
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
__device__ uint8_t end_of_iteration(const EndParams &P, int G, int C, double &r, uint32_t &t,
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

// ---------------------------------------------------------------- fused kernel
template <int GMAX, int CH>
__global__ void __launch_bounds__(kGatherThreads)
    k_gather_test(const GatherArgs A) {
  const int lane = threadIdx.x & 31;
  const int G = A.na * A.ns;
  const int CG = G * CH;
  const GridHeader grid = *A.grid;
  unsigned long long my_cand = 0, my_exact = 0, my_amb = 0, my_acc = 0;
  double my_rmax = 0.0;
  uint32_t my_tested = 0, my_rejected = 0;

  for (;;) {
    uint32_t h = 0;
    if (lane == 0) h = atomicAdd(A.work, 1u);
    h = __shfl_sync(kFull, h, 0);
    if (h >= A.H) break;

    // ---------------------------------------------------- region + frame
    Hit H;
    const double r = A.radius[h];
    uint32_t t = A.t[h];
    const bool gathered = A.gathered == nullptr || A.gathered[h] != 0;
    H.r = r;
    H.r2 = dm(r, r);
    const double3 c = A.pos[h];
    const double3 n = A.nrm[h];
    H.cx = c.x; H.cy = c.y; H.cz = c.z;
    H.nx = n.x; H.ny = n.y; H.nz = n.z;
    eframe(n.x, n.y, n.z, H.u, H.v);
    const double3 K = A.K[h];
    H.K0 = K.x; H.K1 = K.y; H.K2 = K.z;
    H.eye = A.eye_depth[h];
    H.chx = __double2float_rn(c.x); H.chy = __double2float_rn(c.y); H.chz = __double2float_rn(c.z);
    H.clx = __double2float_rn(c.x - (double)H.chx);
    H.cly = __double2float_rn(c.y - (double)H.chy);
    H.clz = __double2float_rn(c.z - (double)H.chz);
    H.nfx = (float)n.x; H.nfy = (float)n.y; H.nfz = (float)n.z;
    H.ufx = (float)H.u.x; H.ufy = (float)H.u.y; H.ufz = (float)H.u.z;
    H.vfx = (float)H.v.x; H.vfy = (float)H.v.y; H.vfz = (float)H.v.z;
    H.r2f = (float)H.r2;
    H.lim_hi = H.r2f + 2e-5f * H.r2f;
    H.lim_lo = H.r2f - 2e-5f * H.r2f;
    H.band_y = 1e-5f * (float)r;
    H.guard_f = (float)A.guard;
    H.qa_scale = (float)A.na / H.r2f;
    {
      const double cmax = fmax(fabs(c.x), fmax(fabs(c.y), fabs(c.z)));
      const double nn = edot(n.x, n.y, n.z, n.x, n.y, n.z);
      H.fast = H.r2f > 1e-30f && H.r2f < 1e30f && cmax <= 1e6 * r && nn > 0.999 && nn < 1.001;
    }

    uint32_t cnt[GMAX];
    double sm[CH][GMAX], sq[CH][GMAX];
#pragma unroll
    for (int g = 0; g < GMAX; ++g) {
      cnt[g] = 0;
#pragma unroll
      for (int ch = 0; ch < CH; ++ch) { sm[ch][g] = 0.0; sq[ch][g] = 0.0; }
    }
    double fl0 = 0.0, fl1 = 0.0, fl2 = 0.0;

    if (gathered && grid.n > 0) {
      // ------------------------------------------------ 9 column ranges
      const long long ix = (long long)floor(dm(c.x, grid.inv)) - grid.ix0;
      const long long iy = (long long)floor(dm(c.y, grid.inv)) - grid.iy0;
      const long long iz = (long long)floor(dm(c.z, grid.inv)) - grid.iz0;
      uint32_t rbeg = 0, rlen = 0;
      if (lane < 9) {
        const long long X = ix + lane / 3 - 1, Y = iy + lane % 3 - 1;
        const long long z0 = iz - 1 < 0 ? 0 : iz - 1;
        const long long z1 = iz + 1 >= grid.nz ? grid.nz - 1 : iz + 1;
        if (X >= 0 && X < grid.nx && Y >= 0 && Y < grid.ny && z0 <= z1) {
          const unsigned long long k0 = (unsigned long long)((X * grid.ny + Y) * grid.nz + z0);
          const unsigned long long k1 = (unsigned long long)((X * grid.ny + Y) * grid.nz + z1);
          rbeg = A.cell_start[k0];
          rlen = A.cell_start[k1 + 1] - rbeg;
        }
      }
      // inclusive prefix over lanes 0..8
      uint32_t rend = rlen;
#pragma unroll
      for (int o = 1; o < 16; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, rend, o);
        if (lane >= o) rend += y;
      }
      const uint32_t total = __shfl_sync(kFull, rend, 8);
      const uint32_t rpre = rend - rlen;

      int cur = 0;
      for (uint32_t base = 0; base < total; base += 32) {
        const uint32_t idx = base + lane;
        for (;;) {
          const uint32_t e = __shfl_sync(kFull, rend, cur);
          const bool adv = idx >= e && cur < 8;
          if (!__any_sync(kFull, adv)) break;
          cur += adv ? 1 : 0;
        }
        const uint32_t pb = __shfl_sync(kFull, rbeg, cur);
        const uint32_t pp = __shfl_sync(kFull, rpre, cur);
        if (idx >= total) continue;
        const uint32_t i = pb + (idx - pp);
        ++my_cand;
        const float4 a = __ldg(&A.rec0[i]);
        const float dx = (a.x - H.chx) - H.clx;
        const float dy = (a.y - H.chy) - H.cly;
        const float dz = (a.z - H.chz) - H.clz;
        const float d2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
        if (H.fast && d2 > H.lim_hi) continue;
        if (H.eye + __float_as_uint(a.w) > A.max_depth) continue;  // :396 (u32 sum)
        bool ex = !H.fast || !(d2 < H.lim_lo);
        const float4 b = __ldg(&A.rec1[i]);
        const float gd = fmaf(b.x, H.nfx, fmaf(b.y, H.nfy, b.z * H.nfz));
        const float gb = 2e-6f * (fabsf(b.x * H.nfx) + fabsf(b.y * H.nfy) + fabsf(b.z * H.nfz)) + 1e-30f;
        if (!ex && gd < H.guard_f - gb) continue;
        ex = ex || !(gd >= H.guard_f + gb);
        const float yu = fmaf(dx, H.ufx, fmaf(dy, H.ufy, dz * H.ufz));
        const float yv = fmaf(dx, H.vfx, fmaf(dy, H.vfy, dz * H.vfz));
        const float yy = fmaf(yu, yu, yv * yv);
        if (!ex && yy > H.lim_hi) continue;
        ex = ex || !(yy < H.lim_lo);
        const float4 c2 = __ldg(&A.rec2[i]);
        const float ci = fmaf(b.w, H.nfx, fmaf(c2.x, H.nfy, c2.y * H.nfz));
        const float cb = 2e-6f * (fabsf(b.w * H.nfx) + fabsf(c2.x * H.nfy) + fabsf(c2.y * H.nfz)) + 1e-30f;
        ex = ex || !(fabsf(ci) > cb);
        bool cos_pos = ci > 0.0f;
        int sector;
        int s_ang;
        if (A.ns == 4) {
          ex = ex || !(fabsf(yu) > H.band_y) || !(fabsf(yv) > H.band_y);
          s_ang = yu > 0.0f ? (yv > 0.0f ? 0 : 3) : (yv > 0.0f ? 1 : 2);
        } else {
          const float ay = fmaxf(fabsf(yu), fabsf(yv));
          ex = ex || !(ay > 1e-3f * (float)r);
          float th = atan2f(yv, yu);
          if (th < 0.0f) th += 6.2831853f;
          const float tt = (float)A.ns * th * 0.15915494f;
          const float kk = rintf(tt);
          ex = ex || (kk >= 1.0f && kk <= (float)(A.ns - 1) && fabsf(tt - kk) < 4e-3f);
          s_ang = min((int)tt, A.ns - 1);
        }
        int a_ring = 0;
        if (A.na > 1) {
          const float qa = yy * H.qa_scale;
          const float kq = rintf(qa);
          ex = ex || (kq >= 1.0f && kq <= (float)(A.na - 1) && fabsf(qa - kq) < 1e-4f * (float)A.na);
          a_ring = min((int)qa, A.na - 1);
        }
        sector = a_ring * A.ns + s_ang;
        if (ex) {
          ++my_exact;
          bool amb = false;
          if (!exact_pair(H, a, b, c2, A.na, A.ns, A.guard, sector, cos_pos, amb)) continue;
          if (amb) ++my_amb;
        }
        // ---------------------------------------------- accumulate (gather.cpp:59-67)
        ++my_acc;
        const float4 c3 = __ldg(&A.rec3[i]);
        const double v0 = cos_pos ? dm(H.K0, (double)c2.z) : 0.0;
        const double v1 = cos_pos ? dm(H.K1, (double)c2.w) : 0.0;
        const double v2 = cos_pos ? dm(H.K2, (double)c3.x) : 0.0;
        fl0 += v0; fl1 += v1; fl2 += v2;
        if constexpr (CH == 1) {
          const double v = elum(v0, v1, v2);
          const double vv = v * v;
#pragma unroll
          for (int g = 0; g < GMAX; ++g)
            if (sector == g) { cnt[g] += 1; sm[0][g] += v; sq[0][g] += vv; }
        } else {
          const double vv0 = v0 * v0, vv1 = v1 * v1, vv2 = v2 * v2;
#pragma unroll
          for (int g = 0; g < GMAX; ++g)
            if (sector == g) {
              cnt[g] += 1;
              sm[0][g] += v0; sq[0][g] += vv0;
              sm[1][g] += v1; sq[1][g] += vv1;
              sm[2][g] += v2; sq[2][g] += vv2;
            }
        }
      }
    }

    // -------------------------------------------------- warp reduction
#pragma unroll
    for (int g = 0; g < GMAX; ++g) {
      cnt[g] = warp_sum(cnt[g]);
#pragma unroll
      for (int ch = 0; ch < CH; ++ch) {
        sm[ch][g] = warp_sum(sm[ch][g]);
        sq[ch][g] = warp_sum(sq[ch][g]);
      }
    }
    fl0 = warp_sum(fl0); fl1 = warp_sum(fl1); fl2 = warp_sum(fl2);

    // -------------------------------------------------- pool + end_iteration
    if (lane == 0) {
      const size_t base = (size_t)h * CG;
      double r_new = r;
      double stat = 0.0, critical = 0.0;
      uint8_t flags = 0;
      uint32_t accepted = 0;
      for (int g = 0; g < GMAX; ++g) accepted += g < G ? cnt[g] : 0u;
      if (gathered) {
        unsigned long long pc[GMAX * CH];
        double ps[GMAX * CH], pq[GMAX * CH];
#pragma unroll
        for (int ch = 0; ch < CH; ++ch)
#pragma unroll
          for (int g = 0; g < GMAX; ++g) {
            if (g < G) {
              const size_t o = base + (size_t)ch * G + g;
              pc[ch * G + g] = A.st_cnt[o] + cnt[g];
              ps[ch * G + g] = A.st_sum[o] + sm[ch][g];
              pq[ch * G + g] = A.st_sq[o] + sq[ch][g];
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
      } else if (A.snap_cnt) {
        for (int i = 0; i < CG; ++i) {
          A.snap_cnt[base + i] = A.st_cnt[base + i];
          A.snap_sum[base + i] = A.st_sum[base + i];
          A.snap_sq[base + i] = A.st_sq[base + i];
        }
      }
      my_tested += flags & 1;
      my_rejected += (flags >> 1) & 1;
      my_rmax = fmax(my_rmax, r_new);
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
  }

  // ------------------------------------------------------ block totals
  __shared__ unsigned long long s_c[4];
  __shared__ unsigned int s_tr[2];
  __shared__ unsigned long long s_rmax;
  if (threadIdx.x == 0) { s_c[0] = s_c[1] = s_c[2] = s_c[3] = 0; s_tr[0] = s_tr[1] = 0; s_rmax = 0; }
  __syncthreads();
  atomicAdd(&s_c[0], my_acc);
  atomicAdd(&s_c[1], my_cand);
  atomicAdd(&s_c[2], my_exact);
  atomicAdd(&s_c[3], my_amb);
  if (lane == 0) {
    atomicAdd(&s_tr[0], my_tested);
    atomicAdd(&s_tr[1], my_rejected);
    atomicMax(&s_rmax, (unsigned long long)__double_as_longlong(my_rmax));
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    atomicAdd(&A.counters[0], s_c[0]);
    atomicAdd(&A.counters[1], s_c[1]);
    atomicAdd(&A.counters[2], s_c[2]);
    atomicAdd(&A.counters[3], s_c[3]);
    atomicAdd(A.iter_tr, s_tr[0]);
    atomicAdd(A.iter_tr + 1, s_tr[1]);
    atomicMax(A.rmax_bits, s_rmax);
  }
}

// ---------------------------------------------------------------- explicit samples
// GatherRegion::accumulate on caller-supplied (region, y, value) samples.
__global__ void k_sample_sectors(const uint32_t *__restrict__ region, const double2 *__restrict__ y,
                                 uint32_t n, const double *__restrict__ radius, uint32_t H, int na,
                                 int ns, int *__restrict__ sectors, int *__restrict__ err) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint32_t h = region[i];
    if (h >= H) { atomicExch(err, FPPM_ERR_INVALID_ARGUMENT); sectors[i] = -1; continue; }
    const double r = radius[h];
    const double r2 = dm(r, r);
    const double d2 = da(dm(y[i].x, y[i].x), dm(y[i].y, y[i].y));
    if (d2 > dm(r2, 1.0 + 1e-9)) {  // gather.cpp:20-21
      atomicExch(err, FPPM_ERR_DOMAIN);
      sectors[i] = -1;
      continue;
    }
    bool amb = false;
    sectors[i] = exact_sector(y[i].x, y[i].y, r2, na, ns, amb);
  }
}

__global__ void k_sample_accumulate(const uint32_t *__restrict__ region,
                                    const double *__restrict__ value, const int *__restrict__ sectors,
                                    uint32_t n, int G, int C, unsigned long long *__restrict__ st_cnt,
                                    double *__restrict__ st_sum, double *__restrict__ st_sq) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int s = sectors[i];
    const size_t base = (size_t)region[i] * G * C;
    const double r = value[3 * (size_t)i], g = value[3 * (size_t)i + 1], b = value[3 * (size_t)i + 2];
    if (C == 1) {
      const double v = elum(r, g, b);
      atomicAdd(&st_cnt[base + s], 1ull);
      atomicAdd(&st_sum[base + s], v);
      atomicAdd(&st_sq[base + s], v * v);
    } else {
      const double vals[3] = {r, g, b};
      for (int c = 0; c < 3; ++c) {
        atomicAdd(&st_cnt[base + c * G + s], 1ull);
        atomicAdd(&st_sum[base + c * G + s], vals[c]);
        atomicAdd(&st_sq[base + c * G + s], vals[c] * vals[c]);
      }
    }
  }
}

// end_iteration over every region without a gather (gather.cpp:90-144).
__global__ void k_end_iteration(EndArgs A) {
  const int G = A.G, C = A.C, CG = G * C;
  for (uint32_t h = blockIdx.x * blockDim.x + threadIdx.x; h < A.H; h += gridDim.x * blockDim.x) {
    unsigned long long pc[kMaxCG];
    double ps[kMaxCG], pq[kMaxCG];
    const size_t base = (size_t)h * CG;
    for (int i = 0; i < CG; ++i) {
      pc[i] = A.st_cnt[base + i];
      ps[i] = A.st_sum[base + i];
      pq[i] = A.st_sq[base + i];
    }
    if (A.snap_cnt)
      for (int i = 0; i < CG; ++i) {
        A.snap_cnt[base + i] = pc[i];
        A.snap_sum[base + i] = ps[i];
        A.snap_sq[base + i] = pq[i];
      }
    double r = A.radius[h];
    uint32_t t = A.t[h];
    double stat, critical;
    const double r_old = r;
    const uint8_t flags = end_of_iteration(A.end, G, C, r, t, pc, ps, pq, stat, critical);
    for (int i = 0; i < CG; ++i) {
      A.st_cnt[base + i] = pc[i];
      A.st_sum[base + i] = ps[i];
      A.st_sq[base + i] = pq[i];
    }
    A.radius[h] = r;
    A.t[h] = t;
    if (A.o_gather_r) A.o_gather_r[h] = r_old;
    if (A.o_flags) A.o_flags[h] = flags;
    if (A.o_stat) A.o_stat[h] = stat;
    if (A.o_crit) A.o_crit[h] = critical;
  }
}

__global__ void k_hit_weights(const double3 *__restrict__ nrm, const double3 *__restrict__ wo,
                              const double3 *__restrict__ thr, const double3 *__restrict__ alb,
                              uint32_t H, double3 *__restrict__ K) {
  for (uint32_t h = blockIdx.x * blockDim.x + threadIdx.x; h < H; h += gridDim.x * blockDim.x) {
    const double3 n = nrm[h], w = wo[h], T = thr[h], a = alb[h];
    const double cos_o = edot(w.x, w.y, w.z, n.x, n.y, n.z);  // bsdf.cpp:34
    const bool off = cos_o <= 0.0;                             // bsdf.cpp:58
    K[h] = make_double3(dm(T.x, off ? 0.0 : dm(a.x, kInvPi)), dm(T.y, off ? 0.0 : dm(a.y, kInvPi)),
                        dm(T.z, off ? 0.0 : dm(a.z, kInvPi)));
  }
}

// ---------------------------------------------------------------- launchers
template <int GMAX, int CH>
static cudaError_t launch_one(cudaStream_t s, const GatherArgs &A, int sms) {
  int per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_gather_test<GMAX, CH>,
                                                                kGatherThreads, 0);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  unsigned blocks = (unsigned)(sms * per_sm);
  const unsigned need = (A.H + kGatherThreads / 32 - 1) / (kGatherThreads / 32);
  if (blocks > need) blocks = need ? need : 1;
  k_gather_test<GMAX, CH><<<blocks, kGatherThreads, 0, s>>>(A);
  note_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_gather_test(cudaStream_t s, const GatherArgs &A, int C, int sms) {
  const int G = A.na * A.ns;
  if (C == 1) {
    if (G <= 4) return launch_one<4, 1>(s, A, sms);
    if (G <= 8) return launch_one<8, 1>(s, A, sms);
    if (G <= 12) return launch_one<12, 1>(s, A, sms);
    if (G <= 16) return launch_one<16, 1>(s, A, sms);
    return launch_one<32, 1>(s, A, sms);
  }
  if (G <= 4) return launch_one<4, 3>(s, A, sms);
  if (G <= 8) return launch_one<8, 3>(s, A, sms);
  if (G <= 12) return launch_one<12, 3>(s, A, sms);
  return launch_one<32, 3>(s, A, sms);
}

cudaError_t launch_samples(cudaStream_t s, const uint32_t *region, const double2 *y,
                           const double *value, uint32_t n, const double *radius, uint32_t H, int na,
                           int ns, int C, int *sectors, int *err, unsigned long long *st_cnt,
                           double *st_sum, double *st_sq, int phase) {
  if (n == 0) return cudaSuccess;
  const int blocks = (int)((n + 255) / 256);
  if (phase == 0)
    k_sample_sectors<<<blocks, 256, 0, s>>>(region, y, n, radius, H, na, ns, sectors, err);
  else
    k_sample_accumulate<<<blocks, 256, 0, s>>>(region, value, sectors, n, na * ns, C, st_cnt,
                                               st_sum, st_sq);
  note_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_end_iteration(cudaStream_t s, const EndArgs &A) {
  if (A.H == 0) return cudaSuccess;
  const int blocks = (int)((A.H + 127) / 128);
  k_end_iteration<<<blocks, 128, 0, s>>>(A);
  note_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_hit_weights(cudaStream_t s, const double3 *nrm, const double3 *wo,
                               const double3 *thr, const double3 *alb, uint32_t H, double3 *K) {
  if (H == 0) return cudaSuccess;
  const int blocks = (int)((H + 255) / 256);
  k_hit_weights<<<blocks, 256, 0, s>>>(nrm, wo, thr, alb, H, K);
  note_launches(1);
  return cudaGetLastError();
}

}  // namespace fppm_b200
