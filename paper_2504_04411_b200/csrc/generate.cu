// generate.cu -- canonical synthetic inputs on the device.
//
// Counter-based PCG32 (one stream per (seed, iteration), photon j reads draws
// [16 j, 16 j + 16)) and transcendental-free deterministic math: only
// correctly rounded IEEE operations (+ - * / sqrt) and exact integer/bit
// manipulation, so any IEEE-conforming implementation (the C oracle on the
// host included) produces the same fp32 photons bit for bit.
#include "common.cuh"
#include "gather.cuh"

namespace fppm_b200 {
namespace gen {

constexpr uint64_t kMul = 6364136223846793005ull;
constexpr uint32_t kDraws = 16;

__device__ __forceinline__ uint64_t splitmix_fin(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

// O(log n) LCG jump (Brown, "Random number generation with arbitrary strides").
__device__ uint64_t jump(uint64_t state, uint64_t steps, uint64_t inc) {
  uint64_t g = kMul, c = inc, G = 1, Cc = 0;
  while (steps) {
    if (steps & 1u) {
      G *= g;
      Cc = Cc * g + c;
    }
    c = (g + 1) * c;
    g *= g;
    steps >>= 1;
  }
  return G * state + Cc;
}

__device__ __forceinline__ uint32_t xsh_rr(uint64_t s) {
  const uint32_t x = (uint32_t)(((s >> 18) ^ s) >> 27);
  const uint32_t r = (uint32_t)(s >> 59);
  return __funnelshift_r(x, x, r);
}

struct Stream {
  uint64_t inc, origin;
  __device__ Stream(uint64_t seed, uint64_t iteration, uint64_t kind) {
    const uint64_t sid = splitmix_fin(iteration + 0x9e3779b97f4a7c15ull * (kind + 1));
    inc = (sid << 1) | 1u;
    uint64_t s = inc;        // state 0 advanced once
    s += seed;
    origin = s * kMul + inc;  // pcg32_srandom_r
  }
};

__device__ __forceinline__ float unit24(uint32_t x) {
  return __uint2float_rn(x >> 8) * 0x1p-24f;
}
__device__ __forceinline__ double unit_open(uint32_t x) {
  return __dmul_rn(__dadd_rn((double)x, 0.5), 0x1p-32);
}

// sin/cos of 2*pi*u, u in [0,1]: exact quarter-turn reduction + Taylor.
__device__ void sincos_turns(double u, double &sn, double &cs) {
  const double q = floor(da(dm(u, 4.0), 0.5));
  const double x = ds(u, dm(q, 0.25));
  const double t = dm(x, 0x1.921fb54442d18p+2);
  const double z = dm(t, t);
  double ps = 0x1.952c77030ad4ap-49;
  ps = da(-0x1.ae7f3e733b81fp-41, dm(z, ps));
  ps = da(0x1.6124613a86d09p-33, dm(z, ps));
  ps = da(-0x1.ae64567f544e4p-26, dm(z, ps));
  ps = da(0x1.71de3a556c734p-19, dm(z, ps));
  ps = da(-0x1.a01a01a01a01ap-13, dm(z, ps));
  ps = da(0x1.1111111111111p-7, dm(z, ps));
  ps = da(-0x1.5555555555555p-3, dm(z, ps));
  const double s = da(t, dm(t, dm(z, ps)));
  double pc = -0x1.6827863b97d97p-53;
  pc = da(0x1.ae7f3e733b81fp-45, dm(z, pc));
  pc = da(-0x1.93974a8c07c9dp-37, dm(z, pc));
  pc = da(0x1.1eed8eff8d898p-29, dm(z, pc));
  pc = da(-0x1.27e4fb7789f5cp-22, dm(z, pc));
  pc = da(0x1.a01a01a01a01ap-16, dm(z, pc));
  pc = da(-0x1.6c16c16c16c17p-10, dm(z, pc));
  pc = da(0x1.5555555555555p-5, dm(z, pc));
  const double c = da(1.0, da(dm(z, -0.5), dm(z, dm(z, pc))));
  switch (((int)q) & 3) {
    case 0: sn = s; cs = c; break;
    case 1: sn = c; cs = -s; break;
    case 2: sn = -s; cs = -c; break;
    default: sn = -c; cs = s; break;
  }
}

// natural log for positive normal x: m in [sqrt(1/2), sqrt(2)), atanh series.
__device__ double log_pos(double x) {
  const unsigned long long bits = __double_as_longlong(x);
  int e = (int)((bits >> 52) & 0x7ff) - 1023;
  double m = __longlong_as_double((long long)((bits & 0x000fffffffffffffull) |
                                              0x3ff0000000000000ull));
  if (m > 0x1.6a09e667f3bcdp+0) {
    m = dm(m, 0.5);
    e += 1;
  }
  const double f = dd(ds(m, 1.0), da(m, 1.0));
  const double s = dm(f, f);
  double p = 0x1.2f684bda12f68p-4;
  p = da(0x1.47ae147ae147bp-4, dm(s, p));
  p = da(0x1.642c8590b2164p-4, dm(s, p));
  p = da(0x1.8618618618618p-4, dm(s, p));
  p = da(0x1.af286bca1af28p-4, dm(s, p));
  p = da(0x1.e1e1e1e1e1e1ep-4, dm(s, p));
  p = da(0x1.1111111111111p-3, dm(s, p));
  p = da(0x1.3b13b13b13b14p-3, dm(s, p));
  p = da(0x1.745d1745d1746p-3, dm(s, p));
  p = da(0x1.c71c71c71c71cp-3, dm(s, p));
  p = da(0x1.2492492492492p-2, dm(s, p));
  p = da(0x1.999999999999ap-2, dm(s, p));
  p = da(0x1.5555555555555p-1, dm(s, p));
  const double lm = da(da(f, f), dm(f, dm(s, p)));
  const double ed = (double)e;
  return da(dm(ed, 0x1.62e42fee00000p-1), da(dm(ed, 0x1.a39ef35793c76p-33), lm));
}

__global__ void k_photons(int workload, uint64_t seed, uint64_t iteration, uint64_t begin,
                          uint32_t n, float *__restrict__ pos, float *__restrict__ nrm,
                          float *__restrict__ wi, float *__restrict__ pw,
                          uint32_t *__restrict__ depth) {
  const Stream st(seed, iteration, 0);
  for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < n;
       k += gridDim.x * blockDim.x) {
    const uint64_t j = begin + k;
    uint64_t s = jump(st.origin, j * kDraws, st.inc);
    uint32_t d[12];
#pragma unroll
    for (int i = 0; i < 12; ++i) {
      d[i] = xsh_rr(s);
      s = s * kMul + st.inc;
    }
    double x, y;
    int pdraw, wdraw;
    if (workload == FPPM_WORKLOAD_C1) {
      x = (double)unit24(d[0]);
      y = (double)unit24(d[1]);
      pdraw = 2;
      wdraw = 5;
    } else {  // FPPM_WORKLOAD_C2: 70% step density (10:1), 30% Gaussian blob
      if (unit24(d[0]) < 0x1.6666660000000p-1f) {
        const double xs = (double)unit24(d[2]);
        x = unit24(d[1]) < 0x1.d1745e0000000p-1f ? da(0.5, dm(0.5, xs)) : dm(0.5, xs);
        y = (double)unit24(d[3]);
      } else {
        const double rad = __dsqrt_rn(dm(-2.0, log_pos(unit_open(d[4]))));
        double sn, cs;
        sincos_turns((double)unit24(d[5]), sn, cs);
        x = da(0.3, dm(0.03, dm(rad, cs)));
        y = da(0.7, dm(0.03, dm(rad, sn)));
      }
      pdraw = 6;
      wdraw = 9;
    }
    const size_t o = 3 * (size_t)k;
    pos[o] = __double2float_rn(x);
    pos[o + 1] = __double2float_rn(y);
    pos[o + 2] = 0.0f;
    nrm[o] = 0.0f;
    nrm[o + 1] = 0.0f;
    nrm[o + 2] = 1.0f;
    pw[o] = unit24(d[pdraw]);
    pw[o + 1] = unit24(d[pdraw + 1]);
    pw[o + 2] = unit24(d[pdraw + 2]);
    const double u1 = (double)unit24(d[wdraw]);
    double sn, cs;
    sincos_turns((double)unit24(d[wdraw + 1]), sn, cs);
    const double r = __dsqrt_rn(u1);
    const double zz = ds(1.0, u1);
    wi[o] = __double2float_rn(dm(r, cs));
    wi[o + 1] = __double2float_rn(dm(r, sn));
    wi[o + 2] = __double2float_rn(__dsqrt_rn(zz < 0.0 ? 0.0 : zz));
    depth[k] = 1;
  }
}

__global__ void k_raster_hitpoints(uint32_t W, double3 *__restrict__ pos,
                                   double3 *__restrict__ nrm, double3 *__restrict__ wo,
                                   double3 *__restrict__ thr, double3 *__restrict__ alb,
                                   uint32_t *__restrict__ eye_depth,
                                   uint8_t *__restrict__ gathered) {
  const uint32_t H = W * W;
  for (uint32_t h = blockIdx.x * blockDim.x + threadIdx.x; h < H;
       h += gridDim.x * blockDim.x) {
    const uint32_t i = h % W, j = h / W;
    const double x = (double)__double2float_rn(dd(da((double)i, 0.5), (double)W));
    const double y = (double)__double2float_rn(dd(da((double)j, 0.5), (double)W));
    pos[h] = make_double3(x, y, 0.0);
    nrm[h] = make_double3(0.0, 0.0, 1.0);
    wo[h] = make_double3(0.0, 0.0, 1.0);
    thr[h] = make_double3(1.0, 1.0, 1.0);
    alb[h] = make_double3(1.0, 1.0, 1.0);
    eye_depth[h] = 1;
    gathered[h] = 1;
  }
}

// ---------------------------------------------------------------- C5
// BASELINE configs[4]: hit points uniform in the unit cube
// with uniform random unit normals; photons from 64 isotropic Gaussian
// clusters (sigma log-uniform in [0.01, 0.05], Dirichlet(1) weights) plus 20 %
// uniform background, restricted to within 0.05 of the tangent plane of the
// nearest hit point (rejection, up to 8 attempts), deposit normal = that hit
// point's normal, wi cosine-distributed about it.

// exp for moderate x: round-to-nearest reduction by ln 2 + Taylor (the C
// oracle's orc_dm_exp, operation for operation)
__device__ double exp_dm(double x) {
  const double k = floor(da(dm(x, 0x1.71547652b82fep+0), 0.5));
  const double r = ds(ds(x, dm(k, 0x1.62e42fee00000p-1)), dm(k, 0x1.a39ef35793c76p-33));
  double p = 0x1.93974a8c07c9dp-37;
  p = da(0x1.6124613a86d09p-33, dm(r, p));
  p = da(0x1.1eed8eff8d898p-29, dm(r, p));
  p = da(0x1.ae64567f544e4p-26, dm(r, p));
  p = da(0x1.27e4fb7789f5cp-22, dm(r, p));
  p = da(0x1.71de3a556c734p-19, dm(r, p));
  p = da(0x1.a01a01a01a01ap-16, dm(r, p));
  p = da(0x1.a01a01a01a01ap-13, dm(r, p));
  p = da(0x1.6c16c16c16c17p-10, dm(r, p));
  p = da(0x1.1111111111111p-7, dm(r, p));
  p = da(0x1.5555555555555p-5, dm(r, p));
  p = da(0x1.5555555555555p-3, dm(r, p));
  p = da(0x1.0000000000000p-1, dm(r, p));
  const double er = da(1.0, da(r, dm(r, dm(r, p))));
  const unsigned long long sb = (unsigned long long)((long long)k + 1023) << 52;
  return dm(er, __longlong_as_double((long long)sb));
}

__device__ __forceinline__ void draws_at(uint64_t seed, uint64_t iteration, uint64_t kind, uint64_t idx,
                                         uint32_t *d, int n) {
  const Stream st(seed, iteration, kind);
  uint64_t s = jump(st.origin, idx * kDraws, st.inc);
  for (int i = 0; i < n; ++i) {
    d[i] = xsh_rr(s);
    s = s * kMul + st.inc;
  }
}

// clusters [k] = {cx, cy, cz, sigma, cumulative weight}; one thread
__global__ void k_c5_clusters(uint64_t seed, double *cl) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double w[kC5Clusters];
  double total = 0.0;
  for (int k = 0; k < kC5Clusters; ++k) {
    uint32_t d[5];
    draws_at(seed, 0, 3, k, d, 5);
    cl[5 * k] = (double)unit24(d[0]);
    cl[5 * k + 1] = (double)unit24(d[1]);
    cl[5 * k + 2] = (double)unit24(d[2]);
    cl[5 * k + 3] = dm(0.01, exp_dm(dm((double)unit24(d[3]), 0x1.9c041f7ed8d33p+0)));  // 0.01 * 5^u
    w[k] = -log_pos(unit_open(d[4]));                                                   // Dirichlet(1)
    total = da(total, w[k]);
  }
  double run = 0.0;
  for (int k = 0; k < kC5Clusters; ++k) {
    run = da(run, w[k]);
    cl[5 * k + 4] = dd(run, total);
  }
}

__global__ void k_c5_hitpoints(uint64_t seed, uint32_t H, double3 *__restrict__ pos, double3 *__restrict__ nrm) {
  for (uint32_t h = blockIdx.x * blockDim.x + threadIdx.x; h < H; h += gridDim.x * blockDim.x) {
    uint32_t d[5];
    draws_at(seed, 0, 2, h, d, 5);
    pos[h] = make_double3((double)unit24(d[0]), (double)unit24(d[1]), (double)unit24(d[2]));
    const double z = ds(1.0, dm(2.0, (double)unit24(d[3])));
    const double q = ds(1.0, dm(z, z));
    const double r = __dsqrt_rn(q > 0.0 ? q : 0.0);
    double sn, cs;
    sincos_turns((double)unit24(d[4]), sn, cs);
    nrm[h] = make_double3(dm(r, cs), dm(r, sn), z);
  }
}

__device__ __forceinline__ int c5_cell(double x, int G) {
  const double f = floor(dm(x, (double)G));
  return f < 0.0 ? 0 : (f > (double)(G - 1) ? G - 1 : (int)f);
}

__global__ void k_c5_count(const double3 *__restrict__ pos, uint32_t H, int G, uint32_t *__restrict__ cnt,
                           uint32_t *__restrict__ cell_of) {
  for (uint32_t h = blockIdx.x * blockDim.x + threadIdx.x; h < H; h += gridDim.x * blockDim.x) {
    const double3 p = pos[h];
    const uint32_t c = ((uint32_t)c5_cell(p.z, G) * (uint32_t)G + (uint32_t)c5_cell(p.y, G)) * (uint32_t)G +
                       (uint32_t)c5_cell(p.x, G);
    cell_of[h] = c;
    atomicAdd(&cnt[c], 1u);
  }
}

__global__ void k_c5_scatter(const uint32_t *__restrict__ cell_of, uint32_t H, const uint32_t *__restrict__ start,
                             uint32_t *__restrict__ fill, uint32_t *__restrict__ items) {
  for (uint32_t h = blockIdx.x * blockDim.x + threadIdx.x; h < H; h += gridDim.x * blockDim.x) {
    const uint32_t c = cell_of[h];
    items[start[c] + atomicAdd(&fill[c], 1u)] = h;  // order within a cell is irrelevant (ties -> lower index)
  }
}

// nearest hit point: rings of cells around the photon's (clamped) cell until
// the ring's lower distance bound k / G exceeds the best distance; ties go to
// the lower index, so the visiting order does not matter
__device__ uint32_t c5_nearest(const C5Args &C, double px, double py, double pz) {
  const int G = C.G;
  const int cx = c5_cell(px, G), cy = c5_cell(py, G), cz = c5_cell(pz, G);
  const double cs = dd(1.0, (double)G);
  double best = 1e300;
  uint32_t bi = 0xffffffffu;
  for (int k = 0; k <= G; ++k) {
    for (int z = cz - k; z <= cz + k; ++z) {
      if (z < 0 || z >= G) continue;
      for (int y = cy - k; y <= cy + k; ++y) {
        if (y < 0 || y >= G) continue;
        const bool face = z == cz - k || z == cz + k || y == cy - k || y == cy + k;
        for (int x = cx - k; x <= cx + k; x += (face ? 1 : (k > 0 ? 2 * k : 1))) {
          if (x < 0 || x >= G) continue;
          const uint32_t c = ((uint32_t)z * (uint32_t)G + (uint32_t)y) * (uint32_t)G + (uint32_t)x;
          for (uint32_t e = C.start[c]; e < C.start[c + 1]; ++e) {
            const uint32_t h = C.items[e];
            const double3 q = C.pos[h];
            const double dx = ds(px, q.x), dy = ds(py, q.y), dz = ds(pz, q.z);
            const double d2 = da(da(dm(dx, dx), dm(dy, dy)), dm(dz, dz));
            if (d2 < best || (d2 == best && h < bi)) {
              best = d2;
              bi = h;
            }
          }
        }
      }
    }
    const double b = dm((double)k, cs);
    if (bi != 0xffffffffu && best <= dm(b, b)) break;
  }
  return bi;
}

__global__ void k_c5_photons(const C5Args C, uint64_t iteration, uint64_t begin, uint32_t n,
                             float *__restrict__ pos, float *__restrict__ nrm, float *__restrict__ wi,
                             float *__restrict__ pw, uint32_t *__restrict__ depth) {
  for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    const uint64_t j = begin + k;
    uint32_t d[11];
    float fx = 0.f, fy = 0.f, fz = 0.f;
    uint32_t hn = 0;
    for (int a = 0; a < kC5Attempts; ++a) {
      draws_at(C.seed, iteration, a == 0 ? 0 : 7 + a, j, d, 11);
      double x, y, z;
      if (unit24(d[0]) < 0.2f) {
        x = (double)unit24(d[2]);
        y = (double)unit24(d[3]);
        z = (double)unit24(d[4]);
      } else {
        const double u = (double)unit24(d[1]);
        int c = 0;
        while (c < kC5Clusters - 1 && !(u < C.clusters[5 * c + 4])) ++c;
        const double *q = C.clusters + 5 * c;
        const double r1 = __dsqrt_rn(dm(-2.0, log_pos(unit_open(d[2]))));
        const double r2 = __dsqrt_rn(dm(-2.0, log_pos(unit_open(d[4]))));
        double s1, c1, s2, c2;
        sincos_turns((double)unit24(d[3]), s1, c1);
        sincos_turns((double)unit24(d[5]), s2, c2);
        x = da(q[0], dm(q[3], dm(r1, c1)));
        y = da(q[1], dm(q[3], dm(r1, s1)));
        z = da(q[2], dm(q[3], dm(r2, c2)));
      }
      fx = __double2float_rn(x);
      fy = __double2float_rn(y);
      fz = __double2float_rn(z);
      hn = c5_nearest(C, (double)fx, (double)fy, (double)fz);
      const double3 hp = C.pos[hn], hnv = C.nrm[hn];
      const double off = edot(ds((double)fx, hp.x), ds((double)fy, hp.y), ds((double)fz, hp.z), hnv.x, hnv.y,
                              hnv.z);
      if (fabs(off) <= 0.05) break;
    }
    const double3 nv = C.nrm[hn];
    const size_t o = 3 * (size_t)k;
    pos[o] = fx;
    pos[o + 1] = fy;
    pos[o + 2] = fz;
    nrm[o] = __double2float_rn(nv.x);
    nrm[o + 1] = __double2float_rn(nv.y);
    nrm[o + 2] = __double2float_rn(nv.z);
    pw[o] = unit24(d[6]);
    pw[o + 1] = unit24(d[7]);
    pw[o + 2] = unit24(d[8]);
    // cosine-distributed about the deposit normal (sampling.hpp:15-19, frame.cpp:5-14)
    const double u1 = (double)unit24(d[9]);
    double sn, cs;
    sincos_turns((double)unit24(d[10]), sn, cs);
    const double r = __dsqrt_rn(u1);
    const double zz = ds(1.0, u1);
    const double lx = dm(r, cs), ly = dm(r, sn), lz = __dsqrt_rn(zz < 0.0 ? 0.0 : zz);
    double3 fu, fv;
    eframe(nv.x, nv.y, nv.z, fu, fv);
    wi[o] = __double2float_rn(da(da(dm(fu.x, lx), dm(fv.x, ly)), dm(nv.x, lz)));
    wi[o + 1] = __double2float_rn(da(da(dm(fu.y, lx), dm(fv.y, ly)), dm(nv.y, lz)));
    wi[o + 2] = __double2float_rn(da(da(dm(fu.z, lx), dm(fv.z, ly)), dm(nv.z, lz)));
    depth[k] = 1;
  }
}

__global__ void k_c5_set_hitpoints(const double3 *__restrict__ tp, const double3 *__restrict__ tn, uint32_t h0,
                                   uint32_t n, double3 *__restrict__ pos, double3 *__restrict__ nrm,
                                   double3 *__restrict__ wo, double3 *__restrict__ thr, double3 *__restrict__ alb,
                                   uint32_t *__restrict__ eye_depth, uint8_t *__restrict__ gathered) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    pos[i] = tp[h0 + i];
    nrm[i] = tn[h0 + i];
    wo[i] = tn[h0 + i];
    thr[i] = make_double3(1.0, 1.0, 1.0);
    alb[i] = make_double3(1.0, 1.0, 1.0);
    eye_depth[i] = 1;
    gathered[i] = 1;
  }
}

}  // namespace gen

cudaError_t launch_c5_setup(cudaStream_t s, uint64_t seed, uint32_t H, int G, double *clusters, double3 *pos,
                            double3 *nrm, uint32_t *cnt, uint32_t *cell_of, uint32_t *start, uint32_t *fill,
                            uint32_t *items, uint32_t *scan_tmp, int sms) {
  const unsigned long long ncell = (unsigned long long)G * G * G;
  gen::k_c5_clusters<<<1, 32, 0, s>>>(seed, clusters);
  int blocks = (int)((H + 255) / 256);
  if (blocks > sms * 16) blocks = sms * 16;
  if (blocks < 1) blocks = 1;
  gen::k_c5_hitpoints<<<blocks, 256, 0, s>>>(seed, H, pos, nrm);
  cudaError_t e = cudaMemsetAsync(cnt, 0, sizeof(uint32_t) * (ncell + 1), s);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(fill, 0, sizeof(uint32_t) * ncell, s);
  if (e != cudaSuccess) return e;
  gen::k_c5_count<<<blocks, 256, 0, s>>>(pos, H, G, cnt, cell_of);
  note_launches(3);
  e = launch_exclusive_scan(s, cnt, (uint32_t)(ncell + 1), scan_tmp, start);
  if (e != cudaSuccess) return e;
  gen::k_c5_scatter<<<blocks, 256, 0, s>>>(cell_of, H, start, fill, items);
  note_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_c5_photons(cudaStream_t s, const C5Args &C, uint64_t iteration, uint64_t begin, uint32_t n,
                              float *pos, float *nrm, float *wi, float *pw, uint32_t *depth, int sms) {
  if (n == 0) return cudaSuccess;
  int blocks = (int)((n + 127) / 128);
  if (blocks > sms * 32) blocks = sms * 32;
  gen::k_c5_photons<<<blocks, 128, 0, s>>>(C, iteration, begin, n, pos, nrm, wi, pw, depth);
  note_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_c5_set_hitpoints(cudaStream_t s, const C5Args &C, uint32_t h0, uint32_t n, double3 *pos,
                                    double3 *nrm, double3 *wo, double3 *thr, double3 *alb, uint32_t *eye_depth,
                                    uint8_t *gathered, int sms) {
  if (n == 0) return cudaSuccess;
  int blocks = (int)((n + 255) / 256);
  if (blocks > sms * 16) blocks = sms * 16;
  gen::k_c5_set_hitpoints<<<blocks, 256, 0, s>>>(C.pos, C.nrm, h0, n, pos, nrm, wo, thr, alb, eye_depth,
                                                 gathered);
  note_launches(1);
  return cudaGetLastError();
}

void launch_generate_photons(cudaStream_t s, int workload, uint64_t seed, uint64_t iteration,
                             uint64_t begin, uint32_t n, float *pos, float *nrm, float *wi,
                             float *pw, uint32_t *depth, int sms) {
  if (n == 0) return;
  const int threads = 256;
  int blocks = (int)((n + threads - 1) / threads);
  if (blocks > sms * 16) blocks = sms * 16;
  gen::k_photons<<<blocks, threads, 0, s>>>(workload, seed, iteration, begin, n, pos, nrm, wi,
                                            pw, depth);
  note_launches(1);
}

void launch_raster_hitpoints(cudaStream_t s, uint32_t W, double3 *pos, double3 *nrm,
                             double3 *wo, double3 *thr, double3 *alb, uint32_t *eye_depth,
                             uint8_t *gathered, int sms) {
  const uint32_t H = W * W;
  if (H == 0) return;
  const int threads = 256;
  int blocks = (int)((H + threads - 1) / threads);
  if (blocks > sms * 16) blocks = sms * 16;
  gen::k_raster_hitpoints<<<blocks, threads, 0, s>>>(W, pos, nrm, wo, thr, alb, eye_depth,
                                                     gathered);
  note_launches(1);
}

}  // namespace fppm_b200
