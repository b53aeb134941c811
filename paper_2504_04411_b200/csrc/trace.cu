// trace.cu -- photon emission and light-subpath tracing on analytic geometry
// (Renderer::light_phase, integrator.cpp:230-265; trace_light_subpath,
// path.cpp:388-449), one thread per light path.
//
// Restated on the device in fp64 with the reference's operation order (no
// FMA): the counter-based RngStream (rng.hpp), area-light emission
// (path.cpp:180-195, 222-236), closest-hit intersection with spheres and quads
// (scene_geometry.cpp:11-45, 186-224), Lambertian / mirror / dielectric
// sampling (bsdf.cpp:94-182), Russian roulette from depth 5 (path.hpp:156) and
// the VCM MIS partials (path.cpp:28-76).  Deposits at non-delta hits are
// written per path, then compacted in path order, exactly as light_phase
// flattens paths_ -- the photon order the grid build and the reference see.
//
// sin/cos come from the device libm (<= 2 ulp) instead of glibc: directions
// differ in the last bits, which leaves every discrete decision of a path
// (hits, Fresnel and roulette choices) unchanged except with negligible
// probability; tests/test_gpu_trace.py checks paths against the reference's
// own trace_light_subpath.
#include "common.cuh"
#include "gather.cuh"

namespace fppm_b200 {

struct DVec {
  double x, y, z;
};
__device__ __forceinline__ DVec dv(double x, double y, double z) { return DVec{x, y, z}; }
__device__ __forceinline__ DVec add(DVec a, DVec b) { return dv(da(a.x, b.x), da(a.y, b.y), da(a.z, b.z)); }
__device__ __forceinline__ DVec sub(DVec a, DVec b) { return dv(ds(a.x, b.x), ds(a.y, b.y), ds(a.z, b.z)); }
__device__ __forceinline__ DVec mul(DVec a, double s) { return dv(dm(a.x, s), dm(a.y, s), dm(a.z, s)); }
__device__ __forceinline__ DVec divs(DVec a, double s) { return dv(dd(a.x, s), dd(a.y, s), dd(a.z, s)); }
__device__ __forceinline__ DVec neg(DVec a) { return dv(-a.x, -a.y, -a.z); }
__device__ __forceinline__ double dot(DVec a, DVec b) { return edot(a.x, a.y, a.z, b.x, b.y, b.z); }
__device__ __forceinline__ DVec cross(DVec a, DVec b) {
  return dv(ds(dm(a.y, b.z), dm(a.z, b.y)), ds(dm(a.z, b.x), dm(a.x, b.z)), ds(dm(a.x, b.y), dm(a.y, b.x)));
}
__device__ __forceinline__ DVec normalize(DVec a) { return divs(a, __dsqrt_rn(dot(a, a))); }

// rng.hpp RngStream
struct Rng {
  unsigned long long s;
  __device__ static unsigned long long mix(unsigned long long z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
  }
  __device__ Rng(unsigned long long seed, unsigned long long k1, unsigned long long k2,
                 unsigned long long k3) {
    s = mix(seed + 0x9e3779b97f4a7c15ull);
    s = mix(s ^ mix(k1 + 0xbf58476d1ce4e5b9ull));
    s = mix(s ^ mix(k2 + 0x94d049bb133111ebull));
    s = mix(s ^ mix(k3 + 0xd6e8feb86659fd93ull));
  }
  __device__ double next() {
    s += 0x9e3779b97f4a7c15ull;
    return dm((double)(mix(s) >> 11), 0x1.0p-53);
  }
};

// frame.cpp:5-14 (Duff et al.), to_world (frame.hpp:12-14)
struct Frame {
  DVec u, v, n;
};
__device__ __forceinline__ Frame make_frame(DVec n) {
  double3 u, v;
  eframe(n.x, n.y, n.z, u, v);
  return Frame{dv(u.x, u.y, u.z), dv(v.x, v.y, v.z), n};
}
__device__ __forceinline__ DVec to_world(const Frame &f, DVec l) {
  return add(add(mul(f.u, l.x), mul(f.v, l.y)), mul(f.n, l.z));
}

// sampling.hpp
__device__ __forceinline__ DVec sample_cosine_hemisphere(double u1, double u2) {
  const double r = __dsqrt_rn(u1);
  const double phi = dm(kTwoPi, u2);
  double sp, cp;
  sincos(phi, &sp, &cp);
  const double z2 = ds(1.0, u1);
  return dv(dm(r, cp), dm(r, sp), __dsqrt_rn(z2 > 0.0 ? z2 : 0.0));
}
__device__ __forceinline__ DVec sample_uniform_sphere(double u1, double u2) {
  const double z = ds(1.0, dm(2.0, u1));
  const double w = ds(1.0, dm(z, z));
  const double r = __dsqrt_rn(w > 0.0 ? w : 0.0);
  double sp, cp;
  sincos(dm(kTwoPi, u2), &sp, &cp);
  return dv(dm(r, cp), dm(r, sp), z);
}
__device__ __forceinline__ double cos_pdf(double c) { return c > 0 ? dm(c, kInvPi) : 0.0; }
__device__ __forceinline__ DVec reflect(DVec wi, DVec n) { return sub(mul(n, dm(2.0, dot(wi, n))), wi); }

// MIS (path.cpp:11-76)
struct Mis {
  double d_vcm, d_vc, d_vm;
};
__device__ __forceinline__ double mpow(double beta, double x) { return beta == 1.0 ? x : pow(x, beta); }

// intersect_sphere (scene_geometry.cpp:11-26)
__device__ __forceinline__ bool hit_sphere(const double *p, DVec o, DVec d, double tmin, double tmax,
                                           double &t) {
  const DVec c = dv(p[0], p[1], p[2]);
  const DVec oc = sub(o, c);
  const double b = dot(oc, d);
  const double cc = ds(dot(oc, oc), dm(p[3], p[3]));
  const double disc = ds(dm(b, b), cc);
  if (disc < 0.0) return false;
  const double sq = __dsqrt_rn(disc);
  const double q = b < 0.0 ? da(-b, sq) : ds(-b, sq);
  double t0 = q, t1 = q != 0.0 ? dd(cc, q) : 0.0;
  if (t0 > t1) {
    const double x = t0;
    t0 = t1;
    t1 = x;
  }
  if (t0 > tmin && t0 < tmax) { t = t0; return true; }
  if (t1 > tmin && t1 < tmax) { t = t1; return true; }
  return false;
}

// intersect_quad (scene_geometry.cpp:28-45)
__device__ __forceinline__ bool hit_quad(const double *p, DVec o, DVec d, double tmin, double tmax,
                                         double &t) {
  const DVec corner = dv(p[0], p[1], p[2]), e1 = dv(p[3], p[4], p[5]), e2 = dv(p[6], p[7], p[8]);
  const DVec n = cross(e1, e2);
  const double denom = dot(d, n);
  if (denom == 0.0) return false;
  const double tt = dd(dot(sub(corner, o), n), denom);
  if (tt <= tmin || tt >= tmax) return false;
  const DVec rel = sub(add(o, mul(d, tt)), corner);
  const double a11 = dot(e1, e1), a12 = dot(e1, e2), a22 = dot(e2, e2);
  const double b1 = dot(rel, e1), b2 = dot(rel, e2);
  const double det = ds(dm(a11, a22), dm(a12, a12));
  if (det == 0.0) return false;
  const double u = dd(ds(dm(b1, a22), dm(b2, a12)), det);
  const double v = dd(ds(dm(b2, a11), dm(b1, a12)), det);
  if (u < 0.0 || u > 1.0 || v < 0.0 || v > 1.0) return false;
  t = tt;
  return true;
}

struct HitD {
  double t;
  DVec point, gn, sn;
  bool front;
  int mat;
};

// intersect + fill_hit (scene_geometry.cpp:186-224, 263-315), closest hit
// over all primitives in declaration order.
__device__ bool intersect(const TraceScene &sc, DVec o, DVec d, HitD &h) {
  double tbest = 1e300;
  int best = -1;
  for (int i = 0; i < sc.n_prim; ++i) {
    const double *p = sc.prim + 9 * (size_t)i;
    double t;
    const bool ok = sc.prim_kind[i] == 0 ? hit_sphere(p, o, d, 1e-6, tbest, t)
                                         : hit_quad(p, o, d, 1e-6, tbest, t);
    if (ok && t < tbest) {
      tbest = t;
      best = i;
    }
  }
  if (best < 0) return false;
  const double *p = sc.prim + 9 * (size_t)best;
  h.t = tbest;
  h.point = add(o, mul(d, tbest));
  h.mat = sc.prim_mat[best];
  DVec outward;
  if (sc.prim_kind[best] == 0)
    outward = mul(sub(h.point, dv(p[0], p[1], p[2])), dd(1.0, p[3]));
  else
    outward = normalize(cross(dv(p[3], p[4], p[5]), dv(p[6], p[7], p[8])));
  h.front = dot(d, outward) < 0.0;
  h.gn = h.front ? outward : neg(outward);
  h.sn = dot(outward, h.gn) < 0.0 ? neg(outward) : outward;
  return true;
}

__device__ __forceinline__ double prim_area(const TraceScene &sc, int i) {
  const double *p = sc.prim + 9 * (size_t)i;
  if (sc.prim_kind[i] == 0) return dm(dm(dm(4.0, kPi), p[3]), p[3]);
  const DVec c = cross(dv(p[3], p[4], p[5]), dv(p[6], p[7], p[8]));
  return __dsqrt_rn(dot(c, c));
}

// bsdf.cpp:41-51 (min(1, max component))
__device__ __forceinline__ double cont_prob(const TraceScene &sc, int m) {
  const double *a = sc.mat_rgb + 3 * (size_t)m;
  const double m1 = a[1] < a[2] ? a[2] : a[1];
  const double mx = a[0] < m1 ? m1 : a[0];
  return mx < 1.0 ? mx : 1.0;
}

__global__ void __launch_bounds__(128) k_trace_paths(const TraceArgs A) {
  const TraceScene &sc = A.sc;
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < A.n_paths; j += gridDim.x * blockDim.x) {
    uint32_t nv = 0;
    Rng rng(A.seed, A.iteration, j, 0ull /* kLightStream */);
    const size_t slot = (size_t)j * A.light_depth;
    if (sc.n_emit > 0) {
      // emitter pick (path.cpp:392-397)
      const int n = sc.n_emit;
      int pick = (int)dm(rng.next(), (double)n);
      if (pick > n - 1) pick = n - 1;
      const double pick_prob = dd(1.0, (double)n);
      // area emission (path.cpp:180-195, 222-236)
      const int pi = sc.emit_prim[pick];
      const double *p = sc.prim + 9 * (size_t)pi;
      DVec pos, nrm;
      if (sc.prim_kind[pi] == 1) {
        const double u = rng.next(), v = rng.next();
        pos = add(add(dv(p[0], p[1], p[2]), mul(dv(p[3], p[4], p[5]), u)), mul(dv(p[6], p[7], p[8]), v));
        nrm = normalize(cross(dv(p[3], p[4], p[5]), dv(p[6], p[7], p[8])));
      } else {
        // f(rng.next_double(), rng.next_double()): the reference build (g++)
        // evaluates call arguments right to left, so the first draw is u2
        const double u2 = rng.next(), u1 = rng.next();
        const DVec dd_ = sample_uniform_sphere(u1, u2);
        pos = add(dv(p[0], p[1], p[2]), mul(dd_, p[3]));
        nrm = dd_;
      }
      const double pdf_a = dd(1.0, prim_area(sc, pi));
      const Frame fr = make_frame(nrm);
      const double u2 = rng.next(), u1 = rng.next();  // right-to-left arguments (see above)
      const DVec local = sample_cosine_hemisphere(u1, u2);
      DVec dir = to_world(fr, local);
      const double cos_at_light = local.z;
      const double emission_pdf = dm(pdf_a, cos_pdf(local.z));
      const double *rad = sc.emit_rad + 3 * (size_t)pick;
      const double wscale = dd(kPi, pdf_a);
      double t0 = dm(rad[0], wscale), t1 = dm(rad[1], wscale), t2 = dm(rad[2], wscale);
      const bool black = t0 == 0 && t1 == 0 && t2 == 0;
      if (!(emission_pdf <= 0.0) && !black) {
        // mis_light_origin (path.cpp:28-36)
        const double ep = dm(emission_pdf, pick_prob), dp = dm(pdf_a, pick_prob);
        const double vcf = A.eta_vm > 0.0 ? mpow(A.beta, dd(1.0, A.eta_vm)) : 0.0;
        const double vmf = A.eta_vm > 0.0 ? mpow(A.beta, A.eta_vm) : 0.0;
        Mis mis;
        mis.d_vcm = mpow(A.beta, dd(dp, ep));
        mis.d_vc = mpow(A.beta, dd(cos_at_light, ep));
        mis.d_vm = dm(mis.d_vc, vcf);
        t0 = dd(t0, pick_prob);
        t1 = dd(t1, pick_prob);
        t2 = dd(t2, pick_prob);
        DVec o = pos;
        for (uint32_t depth = 1; depth <= A.light_depth; ++depth) {
          HitD h;
          if (!intersect(sc, o, dir, h)) break;
          const DVec wi = neg(dir);
          const double cos_in = fabs(dot(h.sn, wi));
          if (cos_in == 0.0) break;
          // mis_arrive (path.cpp:45-50)
          {
            const double inv_cos = dd(1.0, mpow(A.beta, cos_in));
            mis.d_vcm = dm(mis.d_vcm, dm(mpow(A.beta, dm(h.t, h.t)), inv_cos));
            mis.d_vc = dm(mis.d_vc, inv_cos);
            mis.d_vm = dm(mis.d_vm, inv_cos);
          }
          const int mk = sc.mat_kind[h.mat];
          const double cont = cont_prob(sc, h.mat);
          const double cos_o = dot(wi, h.sn);  // Bsdf ctor (bsdf.cpp:34)
          if (mk == 0) {  // non-delta: deposit (path.cpp:414-428)
            const size_t o3 = 3 * (slot + nv);
            A.v_pos[o3] = (float)h.point.x; A.v_pos[o3 + 1] = (float)h.point.y; A.v_pos[o3 + 2] = (float)h.point.z;
            A.v_nrm[o3] = (float)h.sn.x; A.v_nrm[o3 + 1] = (float)h.sn.y; A.v_nrm[o3 + 2] = (float)h.sn.z;
            A.v_wi[o3] = (float)wi.x; A.v_wi[o3 + 1] = (float)wi.y; A.v_wi[o3 + 2] = (float)wi.z;
            A.v_pow[o3] = (float)t0; A.v_pow[o3 + 1] = (float)t1; A.v_pow[o3 + 2] = (float)t2;
            A.v_depth[slot + nv] = depth;
            if (A.v_mis) {
              A.v_mis[o3] = mis.d_vcm;
              A.v_mis[o3 + 1] = mis.d_vm;
              A.v_mis[o3 + 2] = cont;
            }
            ++nv;
          }
          if (depth == A.light_depth) break;
          // bsdf.sample (bsdf.cpp:94-182)
          DVec ndir;
          double s_cos, s_pdf, s_rev, w0, w1, w2;
          bool s_delta;
          const double *rgb = sc.mat_rgb + 3 * (size_t)h.mat;
          if (mk == 2) {  // dielectric (bsdf.cpp:147-180)
            const double eta = h.front ? sc.mat_ior[h.mat] : dd(1.0, sc.mat_ior[h.mat]);
            const double ci = cos_o;
            if (ci <= 0.0) break;
            const double sin2_t = dd(ds(1.0, dm(ci, ci)), dm(eta, eta));
            double frs;
            if (sin2_t >= 1.0) {
              frs = 1.0;
            } else {
              const double ct = __dsqrt_rn(ds(1.0, sin2_t));
              const double rs = dd(ds(ci, dm(eta, ct)), da(ci, dm(eta, ct)));
              const double rp = dd(ds(dm(eta, ci), ct), da(dm(eta, ci), ct));
              frs = dm(0.5, da(dm(rs, rs), dm(rp, rp)));
            }
            s_delta = true;
            if (rng.next() < frs) {
              ndir = reflect(wi, h.sn);
              s_cos = dot(ndir, h.sn);
              s_pdf = frs;
              s_rev = frs;
            } else {
              const double s2 = dd(ds(1.0, dm(ci, ci)), dm(eta, eta));
              const double x = ds(1.0, s2);
              const double ct = __dsqrt_rn(x > 0.0 ? x : 0.0);
              ndir = normalize(add(mul(wi, dd(-1.0, eta)), mul(h.sn, ds(dd(ci, eta), ct))));
              s_cos = ct;
              s_pdf = ds(1.0, frs);
              s_rev = ds(1.0, frs);
            }
            w0 = rgb[0]; w1 = rgb[1]; w2 = rgb[2];
          } else {
            if (cos_o <= 0.0) break;
            if (mk == 0) {  // lambertian
              const Frame sf = make_frame(h.sn);
              const double a2 = rng.next(), a1 = rng.next();  // right-to-left arguments
              const DVec l = sample_cosine_hemisphere(a1, a2);
              ndir = to_world(sf, l);
              s_cos = l.z;
              if (s_cos <= 0.0) break;
              s_pdf = cos_pdf(s_cos);
              s_rev = cos_pdf(cos_o);
              s_delta = false;
            } else {  // mirror
              ndir = reflect(wi, h.sn);
              s_cos = dot(ndir, h.sn);
              s_pdf = 1.0;
              s_rev = 1.0;
              s_delta = true;
            }
            w0 = rgb[0]; w1 = rgb[1]; w2 = rgb[2];
          }
          if (s_pdf <= 0.0 || (w0 == 0 && w1 == 0 && w2 == 0)) break;
          double q = 1.0;
          if (depth >= 5) {  // kRouletteDepth (path.hpp:156)
            q = cont;
            if (rng.next() >= q) break;
          }
          // mis_scatter (path.cpp:52-76)
          {
            const double pf = dm(s_pdf, cont), pr = dm(s_rev, cont);
            if (s_delta) {
              const double f = mpow(A.beta, dd(dm(s_cos, pr), pf));
              mis.d_vcm = 0.0;
              mis.d_vc = dm(mis.d_vc, f);
              mis.d_vm = dm(mis.d_vm, f);
            } else {
              const double ratio = mpow(A.beta, dd(s_cos, pf));
              const double rev = mpow(A.beta, pr);
              const double d_vc = dm(ratio, da(da(dm(mis.d_vc, rev), mis.d_vcm), vmf));
              const double d_vm = dm(ratio, da(da(dm(mis.d_vm, rev), dm(mis.d_vcm, vcf)), 1.0));
              mis.d_vc = d_vc;
              mis.d_vm = d_vm;
              mis.d_vcm = mpow(A.beta, dd(1.0, pf));
            }
          }
          t0 = dd(dm(t0, w0), q);
          t1 = dd(dm(t1, w1), q);
          t2 = dd(dm(t2, w2), q);
          o = h.point;
          dir = ndir;
        }
      }
    }
    A.count[j] = nv;
  }
}

// flatten the per-path slots in path order (light_phase, integrator.cpp:250-258)
__global__ void k_trace_compact(const TraceArgs A, const uint32_t *__restrict__ base, float *pos, float *nrm,
                                float *wi, float *pw, uint32_t *depth, double *mis_vcm, double *mis_vm,
                                double *mis_cont) {
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < A.n_paths; j += gridDim.x * blockDim.x) {
    const uint32_t n = A.count[j], b = base[j];
    const size_t slot = (size_t)j * A.light_depth;
    for (uint32_t k = 0; k < n; ++k) {
      const size_t s3 = 3 * (slot + k), d3 = 3 * (size_t)(b + k);
      for (int c = 0; c < 3; ++c) {
        pos[d3 + c] = A.v_pos[s3 + c];
        nrm[d3 + c] = A.v_nrm[s3 + c];
        wi[d3 + c] = A.v_wi[s3 + c];
        pw[d3 + c] = A.v_pow[s3 + c];
      }
      depth[b + k] = A.v_depth[slot + k];
      if (mis_vcm) {
        mis_vcm[b + k] = A.v_mis[s3];
        mis_vm[b + k] = A.v_mis[s3 + 1];
        mis_cont[b + k] = A.v_mis[s3 + 2];
      }
    }
  }
}

cudaError_t launch_trace(cudaStream_t s, const TraceArgs &A, int sms) {
  if (A.n_paths == 0) return cudaSuccess;
  unsigned blocks = (A.n_paths + 127) / 128;
  if (blocks > (unsigned)sms * 16) blocks = sms * 16;
  k_trace_paths<<<blocks, 128, 0, s>>>(A);
  note_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_trace_compact(cudaStream_t s, const TraceArgs &A, const uint32_t *base, float *pos,
                                 float *nrm, float *wi, float *pw, uint32_t *depth, double *mv, double *mm,
                                 double *mc, int sms) {
  if (A.n_paths == 0) return cudaSuccess;
  unsigned blocks = (A.n_paths + 255) / 256;
  if (blocks > (unsigned)sms * 16) blocks = sms * 16;
  k_trace_compact<<<blocks, 256, 0, s>>>(A, base, pos, nrm, wi, pw, depth, mv, mm, mc);
  note_launches(1);
  return cudaGetLastError();
}

}  // namespace fppm_b200
