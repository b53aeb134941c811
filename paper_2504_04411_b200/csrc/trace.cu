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
  Rng() = default;
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

// Per-primitive constants hoisted out of the hit tests: every value is the
// same IEEE expression the reference evaluates per call (cross(e1, e2), the
// Gram entries, r * r, 1 / r, 1 / area), so hoisting changes no bit.
struct PrimD {
  int kind, mat, emitter, pad;  // emitter: area emitter on this primitive, -1 if none
  double c[3], e1[3], e2[3];
  double n[3];   // quad: cross(e1, e2)
  double on[3];  // quad: normalize(cross(e1, e2))
  double a11, a12, a22, det;
  double r, r2, inv_r;
  double inv_area;  // 1 / primitive_area (scene_geometry.cpp:320-338)
};
constexpr int kMaxTracePrims = 96;

__global__ void k_scene_prep(const TraceScene sc, PrimD *out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= sc.n_prim) return;
  const double *p = sc.prim + 9 * (size_t)i;
  PrimD d;
  d.kind = sc.prim_kind[i];
  d.mat = sc.prim_mat[i];
  d.emitter = -1;
  d.pad = 0;
  for (int e = 0; e < sc.n_emit; ++e)
    if (sc.emit_prim[e] == i) d.emitter = e;
  for (int k = 0; k < 3; ++k) {
    d.c[k] = p[k];
    d.e1[k] = p[3 + k];
    d.e2[k] = p[6 + k];
  }
  d.r = p[3];
  d.r2 = dm(p[3], p[3]);
  d.inv_r = dd(1.0, p[3]);
  const DVec e1 = dv(p[3], p[4], p[5]), e2 = dv(p[6], p[7], p[8]);
  const DVec n = cross(e1, e2);
  d.n[0] = n.x; d.n[1] = n.y; d.n[2] = n.z;
  const DVec on = normalize(n);
  d.on[0] = on.x; d.on[1] = on.y; d.on[2] = on.z;
  d.a11 = dot(e1, e1);
  d.a12 = dot(e1, e2);
  d.a22 = dot(e2, e2);
  d.det = ds(dm(d.a11, d.a22), dm(d.a12, d.a12));
  const double area = d.kind == 0 ? dm(dm(dm(4.0, kPi), p[3]), p[3]) : __dsqrt_rn(dot(n, n));
  d.inv_area = dd(1.0, area);
  out[i] = d;
}

// intersect_sphere (scene_geometry.cpp:11-26)
__device__ __forceinline__ bool hit_sphere(const PrimD &p, DVec o, DVec d, double tmin, double tmax,
                                           double &t) {
  const DVec oc = sub(o, dv(p.c[0], p.c[1], p.c[2]));
  const double b = dot(oc, d);
  const double cc = ds(dot(oc, oc), p.r2);
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
__device__ __forceinline__ bool hit_quad(const PrimD &p, DVec o, DVec d, double tmin, double tmax,
                                         double &t) {
  const DVec n = dv(p.n[0], p.n[1], p.n[2]);
  const double denom = dot(d, n);
  if (denom == 0.0) return false;
  const DVec corner = dv(p.c[0], p.c[1], p.c[2]);
  const double num = dot(sub(corner, o), n);
  // Division-free rejections that the IEEE quotient num / denom would also
  // reject: t <= 0 (opposite signs or num == 0) and t >= tmax when |num|
  // exceeds tmax |denom| by more than the rounding of both operations.
  if (num == 0.0 || ((num < 0.0) != (denom < 0.0))) return false;
  if (fabs(num) > dm(dm(tmax, fabs(denom)), 1.0 + 0x1p-50)) return false;
  const double tt = dd(num, denom);
  if (tt <= tmin || tt >= tmax) return false;
  const DVec e1 = dv(p.e1[0], p.e1[1], p.e1[2]), e2 = dv(p.e2[0], p.e2[1], p.e2[2]);
  const DVec rel = sub(add(o, mul(d, tt)), corner);
  const double b1 = dot(rel, e1), b2 = dot(rel, e2);
  if (p.det == 0.0) return false;
  const double u = dd(ds(dm(b1, p.a22), dm(b2, p.a12)), p.det);
  const double v = dd(ds(dm(b2, p.a11), dm(b1, p.a12)), p.det);
  if (u < 0.0 || u > 1.0 || v < 0.0 || v > 1.0) return false;
  t = tt;
  return true;
}

struct HitD {
  double t;
  DVec point, sn;
  bool front;
  int mat, prim;
};

// intersect + fill_hit (scene_geometry.cpp:186-224, 263-315): closest hit
// over all primitives in declaration order (strict '<' keeps the first of
// equal distances; the reference's BVH visits leaves in a fixed order, so a
// tie between two primitives at bit-identical t is the only case that could
// pick differently).
__device__ __forceinline__ bool intersect(const PrimD *P, int np, DVec o, DVec d, HitD &h) {
  double tbest = 1e300;
  int best = -1;
  for (int i = 0; i < np; ++i) {
    double t;
    const bool ok = P[i].kind == 0 ? hit_sphere(P[i], o, d, 1e-6, tbest, t) : hit_quad(P[i], o, d, 1e-6, tbest, t);
    if (ok && t < tbest) {
      tbest = t;
      best = i;
    }
  }
  if (best < 0) return false;
  const PrimD &p = P[best];
  h.t = tbest;
  h.point = add(o, mul(d, tbest));
  h.mat = p.mat;
  h.prim = best;
  DVec outward;
  if (p.kind == 0)
    outward = mul(sub(h.point, dv(p.c[0], p.c[1], p.c[2])), p.inv_r);
  else
    outward = dv(p.on[0], p.on[1], p.on[2]);
  h.front = dot(d, outward) < 0.0;
  const DVec gn = h.front ? outward : neg(outward);
  h.sn = dot(outward, gn) < 0.0 ? neg(outward) : outward;
  return true;
}

// bsdf.cpp:41-51 (min(1, max component))
__device__ __forceinline__ double cont_prob(const TraceScene &sc, int m) {
  const double *a = sc.mat_rgb + 3 * (size_t)m;
  const double m1 = a[1] < a[2] ? a[2] : a[1];
  const double mx = a[0] < m1 ? m1 : a[0];
  return mx < 1.0 ? mx : 1.0;
}

struct PathState {
  Rng rng;
  DVec o, dir;
  double t0, t1, t2;
  Mis mis;
  uint32_t depth, nv, j;
};

// Emission (trace_light_subpath prologue, path.cpp:392-407; sample_emission
// area branch, path.cpp:180-195, 222-236).  False: the path deposits nothing.
__device__ __forceinline__ bool start_path(const TraceArgs &A, const PrimD *P, PathState &s, uint32_t j,
                                           double vcf) {
  const TraceScene &sc = A.sc;
  s.rng = Rng(A.seed, A.iteration, A.path0 + j, 0ull /* kLightStream */);
  s.j = j;
  s.nv = 0;
  s.depth = 1;
  if (sc.n_emit <= 0 || A.light_depth == 0) return false;  // no loop iteration (path.cpp:409)
  const int n = sc.n_emit;
  int pick = (int)dm(s.rng.next(), (double)n);
  if (pick > n - 1) pick = n - 1;
  const double pick_prob = dd(1.0, (double)n);
  const int pi = sc.emit_prim[pick];
  const PrimD &p = P[pi];
  DVec pos, nrm;
  if (p.kind == 1) {
    const double u = s.rng.next(), v = s.rng.next();
    pos = add(add(dv(p.c[0], p.c[1], p.c[2]), mul(dv(p.e1[0], p.e1[1], p.e1[2]), u)),
              mul(dv(p.e2[0], p.e2[1], p.e2[2]), v));
    nrm = dv(p.on[0], p.on[1], p.on[2]);
  } else {
    // f(rng.next_double(), rng.next_double()): the reference build (g++)
    // evaluates call arguments right to left, so the first draw is u2
    const double u2 = s.rng.next(), u1 = s.rng.next();
    const DVec dd_ = sample_uniform_sphere(u1, u2);
    pos = add(dv(p.c[0], p.c[1], p.c[2]), mul(dd_, p.r));
    nrm = dd_;
  }
  const double pdf_a = p.inv_area;
  const Frame fr = make_frame(nrm);
  const double u2 = s.rng.next(), u1 = s.rng.next();  // right-to-left arguments (see above)
  const DVec local = sample_cosine_hemisphere(u1, u2);
  s.dir = to_world(fr, local);
  const double cos_at_light = local.z;
  const double emission_pdf = dm(pdf_a, cos_pdf(local.z));
  const double *rad = sc.emit_rad + 3 * (size_t)pick;
  const double wscale = dd(kPi, pdf_a);
  s.t0 = dm(rad[0], wscale);
  s.t1 = dm(rad[1], wscale);
  s.t2 = dm(rad[2], wscale);
  if (emission_pdf <= 0.0 || (s.t0 == 0 && s.t1 == 0 && s.t2 == 0)) return false;
  // mis_light_origin (path.cpp:28-36)
  const double ep = dm(emission_pdf, pick_prob), dp = dm(pdf_a, pick_prob);
  s.mis.d_vcm = mpow(A.beta, dd(dp, ep));
  s.mis.d_vc = mpow(A.beta, dd(cos_at_light, ep));
  s.mis.d_vm = dm(s.mis.d_vc, vcf);
  s.t0 = dd(s.t0, pick_prob);
  s.t1 = dd(s.t1, pick_prob);
  s.t2 = dd(s.t2, pick_prob);
  s.o = pos;
  return true;
}

// Bsdf::sample (bsdf.cpp:94-182) for the analytic materials: Lambertian
// (cosine lobe), mirror, dielectric (Fresnel pick).  wi is the Bsdf's stored
// direction (toward the previous vertex), cos_o = dot(wi, sn).  False: no
// sample (the path ends).
__device__ __forceinline__ bool bsdf_sample(const TraceScene &sc, int mk, int mat, DVec sn, DVec wi, bool front,
                                            double cos_o, Rng &rng, DVec &ndir, double &s_cos, double &s_pdf,
                                            double &s_rev, bool &s_delta) {
  if (mk == 2) {  // dielectric (bsdf.cpp:147-180)
    const double eta = front ? sc.mat_ior[mat] : dd(1.0, sc.mat_ior[mat]);
    const double ci = cos_o;
    if (ci <= 0.0) return false;
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
      ndir = reflect(wi, sn);
      s_cos = dot(ndir, sn);
      s_pdf = frs;
      s_rev = frs;
    } else {
      const double x = ds(1.0, sin2_t);
      const double ct = __dsqrt_rn(x > 0.0 ? x : 0.0);
      ndir = normalize(add(mul(wi, dd(-1.0, eta)), mul(sn, ds(dd(ci, eta), ct))));
      s_cos = ct;
      s_pdf = ds(1.0, frs);
      s_rev = ds(1.0, frs);
    }
  } else {
    if (cos_o <= 0.0) return false;
    if (mk == 0) {  // lambertian
      const Frame sf = make_frame(sn);
      const double a2 = rng.next(), a1 = rng.next();  // right-to-left arguments
      const DVec l = sample_cosine_hemisphere(a1, a2);
      ndir = to_world(sf, l);
      s_cos = l.z;
      if (s_cos <= 0.0) return false;
      s_pdf = cos_pdf(s_cos);
      s_rev = cos_pdf(cos_o);
      s_delta = false;
    } else {  // mirror
      ndir = reflect(wi, sn);
      s_cos = dot(ndir, sn);
      s_pdf = 1.0;
      s_rev = 1.0;
      s_delta = true;
    }
  }
  return true;
}

// One segment of trace_light_subpath's loop (path.cpp:409-447).  False: the
// path ended.
__device__ __forceinline__ bool bounce(const TraceArgs &A, const PrimD *P, int np, PathState &s, double vcf,
                                       double vmf) {
  const TraceScene &sc = A.sc;
  HitD h;
  if (!intersect(P, np, s.o, s.dir, h)) return false;
  const DVec wi = neg(s.dir);
  const double cos_in = fabs(dot(h.sn, wi));
  if (cos_in == 0.0) return false;
  {  // mis_arrive (path.cpp:45-50)
    const double inv_cos = dd(1.0, mpow(A.beta, cos_in));
    s.mis.d_vcm = dm(s.mis.d_vcm, dm(mpow(A.beta, dm(h.t, h.t)), inv_cos));
    s.mis.d_vc = dm(s.mis.d_vc, inv_cos);
    s.mis.d_vm = dm(s.mis.d_vm, inv_cos);
  }
  const int mk = sc.mat_kind[h.mat];
  const double cont = cont_prob(sc, h.mat);
  const double cos_o = dot(wi, h.sn);  // Bsdf ctor (bsdf.cpp:34)
  if (mk == 0) {  // non-delta: deposit (path.cpp:414-428)
    const size_t slot = (size_t)s.j * A.light_depth + s.nv;
    const size_t o3 = 3 * slot;
    A.v_pos[o3] = (float)h.point.x; A.v_pos[o3 + 1] = (float)h.point.y; A.v_pos[o3 + 2] = (float)h.point.z;
    A.v_nrm[o3] = (float)h.sn.x; A.v_nrm[o3 + 1] = (float)h.sn.y; A.v_nrm[o3 + 2] = (float)h.sn.z;
    A.v_wi[o3] = (float)wi.x; A.v_wi[o3 + 1] = (float)wi.y; A.v_wi[o3 + 2] = (float)wi.z;
    A.v_pow[o3] = (float)s.t0; A.v_pow[o3 + 1] = (float)s.t1; A.v_pow[o3 + 2] = (float)s.t2;
    A.v_depth[slot] = s.depth;
    if (A.v_mis) {
      A.v_mis[o3] = s.mis.d_vcm;
      A.v_mis[o3 + 1] = s.mis.d_vm;
      A.v_mis[o3 + 2] = cont;
    }
    if (A.b_pos) {  // fp64 LightVertex for connections and camera splats
      A.b_pos[o3] = h.point.x; A.b_pos[o3 + 1] = h.point.y; A.b_pos[o3 + 2] = h.point.z;
      A.b_sn[o3] = h.sn.x; A.b_sn[o3 + 1] = h.sn.y; A.b_sn[o3 + 2] = h.sn.z;
      A.b_wi[o3] = wi.x; A.b_wi[o3 + 1] = wi.y; A.b_wi[o3 + 2] = wi.z;
      A.b_thr[o3] = s.t0; A.b_thr[o3 + 1] = s.t1; A.b_thr[o3 + 2] = s.t2;
      A.b_mis[o3] = s.mis.d_vcm; A.b_mis[o3 + 1] = s.mis.d_vc; A.b_mis[o3 + 2] = s.mis.d_vm;
      A.b_mat[slot] = h.mat;
    }
    ++s.nv;
  }
  if (s.depth == A.light_depth) return false;
  // bsdf.sample (bsdf.cpp:94-182)
  DVec ndir;
  double s_cos, s_pdf, s_rev;
  bool s_delta;
  const double *rgb = sc.mat_rgb + 3 * (size_t)h.mat;
  if (!bsdf_sample(sc, mk, h.mat, h.sn, wi, h.front, cos_o, s.rng, ndir, s_cos, s_pdf, s_rev, s_delta))
    return false;
  const double w0 = rgb[0], w1 = rgb[1], w2 = rgb[2];
  if (s_pdf <= 0.0 || (w0 == 0 && w1 == 0 && w2 == 0)) return false;
  double q = 1.0;
  if (s.depth >= 5) {  // kRouletteDepth (path.hpp:156)
    q = cont;
    if (s.rng.next() >= q) return false;
  }
  {  // mis_scatter (path.cpp:52-76)
    const double pf = dm(s_pdf, cont), pr = dm(s_rev, cont);
    if (s_delta) {
      const double f = mpow(A.beta, dd(dm(s_cos, pr), pf));
      s.mis.d_vcm = 0.0;
      s.mis.d_vc = dm(s.mis.d_vc, f);
      s.mis.d_vm = dm(s.mis.d_vm, f);
    } else {
      const double ratio = mpow(A.beta, dd(s_cos, pf));
      const double rev = mpow(A.beta, pr);
      const double d_vc = dm(ratio, da(da(dm(s.mis.d_vc, rev), s.mis.d_vcm), vmf));
      const double d_vm = dm(ratio, da(da(dm(s.mis.d_vm, rev), dm(s.mis.d_vcm, vcf)), 1.0));
      s.mis.d_vc = d_vc;
      s.mis.d_vm = d_vm;
      s.mis.d_vcm = mpow(A.beta, dd(1.0, pf));
    }
  }
  s.t0 = dd(dm(s.t0, w0), q);
  s.t1 = dd(dm(s.t1, w1), q);
  s.t2 = dd(dm(s.t2, w2), q);
  s.o = h.point;
  s.dir = ndir;
  ++s.depth;
  return true;
}

// Persistent warps with path regeneration: a lane whose path ended takes the
// next path id from a warp-local chunk (refilled by one atomic per kTraceChunk
// paths), so lanes stay busy instead of idling until the warp's longest path
// ends.  Output slots are indexed by path id, so the processing order does
// not change the flattened photon order.
constexpr uint32_t kTraceChunk = 64;

#ifndef FPPM_TRACE_MINB
#define FPPM_TRACE_MINB 3
#endif
__global__ void __launch_bounds__(256, FPPM_TRACE_MINB) k_trace_paths(const TraceArgs A, const PrimD *__restrict__ prims) {
  __shared__ PrimD P[kMaxTracePrims];
  const int np = A.sc.n_prim;
  for (int i = threadIdx.x; i < np; i += blockDim.x) P[i] = prims[i];
  __syncthreads();
  const unsigned lane = threadIdx.x & 31;
  const double vcf = A.eta_vm > 0.0 ? mpow(A.beta, dd(1.0, A.eta_vm)) : 0.0;  // vc_factor (path.cpp:22-24)
  const double vmf = A.eta_vm > 0.0 ? mpow(A.beta, A.eta_vm) : 0.0;           // vm_factor (path.cpp:19-21)
  uint32_t q_next = 0, q_end = 0;  // warp-uniform chunk of path ids
  bool alive = false, done = false;
  PathState st;
  for (;;) {
    unsigned need = __ballot_sync(~0u, !alive && !done);
    while (need) {
      if (q_next >= q_end) {
        uint32_t b = 0;
        if (lane == 0) b = atomicAdd(A.path_counter, kTraceChunk);
        b = __shfl_sync(~0u, b, 0);
        q_next = b < A.n_paths ? b : A.n_paths;
        q_end = b + kTraceChunk < A.n_paths ? b + kTraceChunk : A.n_paths;
        if (q_next >= q_end) {  // no paths left
          if (!alive) done = true;
          break;
        }
      }
      const uint32_t avail = q_end - q_next;
      const uint32_t rank = __popc(need & ((1u << lane) - 1u));
      if (((need >> lane) & 1u) && rank < avail) {
        const uint32_t j = q_next + rank;
        alive = start_path(A, P, st, j, vcf);
        if (!alive) A.count[j] = 0;
      }
      const uint32_t took = __popc(need) < avail ? __popc(need) : avail;
      q_next += took;
      need = __ballot_sync(~0u, !alive && !done);
    }
    if (__all_sync(~0u, done)) break;
    if (alive && !bounce(A, P, np, st, vcf, vmf)) {
      A.count[st.j] = st.nv;
      alive = false;
    }
  }
}

// Flatten the per-path slots in path order (light_phase, integrator.cpp:
// 250-258).  One warp per 32 consecutive paths: their outputs form one
// contiguous range, copied lane-per-photon with the owning path found by a
// shuffle binary search over the warp's exclusive offsets.
__global__ void __launch_bounds__(256) k_trace_compact(const TraceArgs A, const uint32_t *__restrict__ base,
                                                       float *pos, float *nrm, float *wi, float *pw,
                                                       uint32_t *depth, double *mis_vcm, double *mis_vm,
                                                       double *mis_cont) {
  const unsigned lane = threadIdx.x & 31;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w * 32u < A.n_paths; w += nwarps) {
    const uint32_t p = w * 32u + lane;
    const uint32_t cnt = p < A.n_paths ? A.count[p] : 0u;
    const uint32_t b = p < A.n_paths ? base[p] : 0xffffffffu;
    const uint32_t start = __shfl_sync(~0u, b, 0);
    const uint32_t total = __reduce_add_sync(~0u, cnt);
    const uint32_t rel = b - start;  // lanes past n_paths: huge, never selected
    for (uint32_t o0 = 0; o0 < total; o0 += 32) {
      const uint32_t o = o0 + lane;
      uint32_t L = 0, rv = 0;  // rel of lane 0 is 0
#pragma unroll
      for (uint32_t step = 16; step; step >>= 1) {
        const uint32_t v = __shfl_sync(~0u, rel, L + step);
        if (v <= o) {
          L += step;
          rv = v;
        }
      }
      if (o < total) {
        const uint32_t k = o - rv;
        const size_t s = (size_t)(w * 32u + L) * A.light_depth + k;
        const size_t s3 = 3 * s, d3 = 3 * (size_t)(start + o);
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          pos[d3 + c] = A.v_pos[s3 + c];
          nrm[d3 + c] = A.v_nrm[s3 + c];
          wi[d3 + c] = A.v_wi[s3 + c];
          pw[d3 + c] = A.v_pow[s3 + c];
        }
        depth[start + o] = A.v_depth[s];
        if (mis_vcm) {
          mis_vcm[start + o] = A.v_mis[s3];
          mis_vm[start + o] = A.v_mis[s3 + 1];
          mis_cont[start + o] = A.v_mis[s3 + 2];
        }
      }
    }
  }
}

// ---------------------------------------------------------------- eye pass
// Renderer::pixel_pm's camera walk (integrator.cpp:407-474) up to the gather:
// jittered pinhole ray (make_camera_ray, path.cpp:135-142) with
// RngStream(seed, iteration, px, kEyeStream = 1), emitted radiance of
// front-facing emitter hits, delta bounces (mirror / dielectric) with Russian
// roulette from depth 5, and the first non-delta hit becomes the pixel's hit
// point (GatherRegion::move_to, eye Bsdf, eye depth).
__global__ void __launch_bounds__(128) k_trace_eye(const EyeArgs E, const PrimD *__restrict__ prims) {
  __shared__ PrimD P[kMaxTracePrims];
  const TraceScene &sc = E.sc;
  const int np = sc.n_prim;
  for (int i = threadIdx.x; i < np; i += blockDim.x) P[i] = prims[i];
  __syncthreads();
  const CamD &cam = E.cam;
  for (uint32_t px = blockIdx.x * blockDim.x + threadIdx.x; px < E.npix; px += gridDim.x * blockDim.x) {
    Rng rng(E.seed, E.iteration, px, 1ull /* kEyeStream */);
    const double sx = da((double)(px % (uint32_t)cam.width), rng.next());
    const double sy = da((double)(px / (uint32_t)cam.width), rng.next());
    DVec dir = normalize(add(add(mul(dv(cam.fwd[0], cam.fwd[1], cam.fwd[2]), cam.plane_dist),
                                 mul(dv(cam.right[0], cam.right[1], cam.right[2]),
                                     ds(sx, dm(0.5, (double)cam.width)))),
                             mul(dv(cam.up[0], cam.up[1], cam.up[2]), ds(dm(0.5, (double)cam.height), sy))));
    DVec o = dv(cam.pos[0], cam.pos[1], cam.pos[2]);
    double t0 = 1.0, t1 = 1.0, t2 = 1.0;
    double e0 = 0.0, e1 = 0.0, e2 = 0.0;
    uint8_t gathered = 0;
    uint32_t eye_depth = 0;
    HitD hp{};
    DVec hwo = dv(0, 0, 0);
    for (uint32_t depth = 1; depth <= E.max_depth; ++depth) {
      HitD h;
      if (!intersect(P, np, o, dir, h)) break;
      const DVec wo = neg(dir);
      const int em = P[h.prim].emitter;
      if (em >= 0 && h.front) {  // out += throughput * radiance
        const double *L = sc.emit_rad + 3 * (size_t)em;
        e0 = da(e0, dm(t0, L[0]));
        e1 = da(e1, dm(t1, L[1]));
        e2 = da(e2, dm(t2, L[2]));
      }
      const int mk = sc.mat_kind[h.mat];
      if (mk == 0) {  // first rough surface: gather here
        hp = h;
        hwo = wo;
        eye_depth = depth;
        gathered = 1;
        break;
      }
      if (depth == E.max_depth) break;
      const double cos_o = dot(wo, h.sn);
      DVec ndir;
      double pdf;
      if (mk == 2) {  // sample_dielectric (bsdf.cpp:147-180)
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
        if (rng.next() < frs) {
          ndir = reflect(wo, h.sn);
          pdf = frs;
        } else {
          const double x = ds(1.0, sin2_t);
          const double ct = __dsqrt_rn(x > 0.0 ? x : 0.0);
          ndir = normalize(add(mul(wo, dd(-1.0, eta)), mul(h.sn, ds(dd(ci, eta), ct))));
          pdf = ds(1.0, frs);
        }
      } else {  // mirror (bsdf.cpp:108-116)
        if (cos_o <= 0.0) break;
        ndir = reflect(wo, h.sn);
        pdf = 1.0;
      }
      const double *w = sc.mat_rgb + 3 * (size_t)h.mat;
      if (pdf <= 0.0 || (w[0] == 0 && w[1] == 0 && w[2] == 0)) break;
      double q = 1.0;
      if (depth >= 5) {  // kRouletteDepth
        q = cont_prob(sc, h.mat);
        if (rng.next() >= q) break;
      }
      t0 = dd(dm(t0, w[0]), q);
      t1 = dd(dm(t1, w[1]), q);
      t2 = dd(dm(t2, w[2]), q);
      o = h.point;
      dir = ndir;
    }
    E.emitted[px] = make_double3(e0, e1, e2);
    E.gathered[px] = gathered;
    E.eye_depth[px] = eye_depth;
    if (gathered) {
      const double *a = sc.mat_rgb + 3 * (size_t)hp.mat;
      E.pos[px] = make_double3(hp.point.x, hp.point.y, hp.point.z);
      E.nrm[px] = make_double3(hp.sn.x, hp.sn.y, hp.sn.z);
      E.wo[px] = make_double3(hwo.x, hwo.y, hwo.z);
      E.thr[px] = make_double3(t0, t1, t2);
      E.alb[px] = make_double3(a[0], a[1], a[2]);
    } else {
      E.pos[px] = make_double3(0, 0, 0);
      E.nrm[px] = make_double3(0, 0, 1);
      E.wo[px] = make_double3(0, 0, 1);
      E.thr[px] = make_double3(0, 0, 0);
      E.alb[px] = make_double3(0, 0, 0);
    }
  }
}

// Film::add_iteration (film.cpp:21-26) of the pixel estimate
// out = emitted + sum / (pi r^2 J) (integrator.cpp:452-455).
// Film::add_iteration + add_split (film.cpp:21-34; integrator.cpp:452-474):
// vc = luminance of the emitted radiance along the chain, vm = luminance of
// the kernel estimate c = sum / (pi r^2 J).
__global__ void k_film_add(uint32_t npix, const double3 *__restrict__ emitted, const uint8_t *__restrict__ gathered,
                           const double *__restrict__ flux, const double *__restrict__ gather_r, double J,
                           double3 *__restrict__ film, double2 *__restrict__ vcvm) {
  for (uint32_t px = blockIdx.x * blockDim.x + threadIdx.x; px < npix; px += gridDim.x * blockDim.x) {
    double3 est = emitted[px];
    double vm = 0.0;
    if (gathered[px]) {
      const double r = gather_r[px];
      const double denom = dm(dm(dm(kPi, r), r), J);
      const double c0 = dd(flux[3 * (size_t)px], denom), c1 = dd(flux[3 * (size_t)px + 1], denom),
                   c2 = dd(flux[3 * (size_t)px + 2], denom);
      vm = elum(c0, c1, c2);
      est.x = da(est.x, c0);
      est.y = da(est.y, c1);
      est.z = da(est.z, c2);
    }
    if (vcvm) {
      double2 v = vcvm[px];
      v.x = da(v.x, elum(emitted[px].x, emitted[px].y, emitted[px].z));
      v.y = da(v.y, vm);
      vcvm[px] = v;
    }
    double3 f = film[px];
    f.x = da(f.x, est.x);
    f.y = da(f.y, est.y);
    f.z = da(f.z, est.z);
    film[px] = f;
  }
}

__global__ void k_film_mean(uint32_t npix, const double3 *__restrict__ film, double iters, double *__restrict__ out) {
  for (uint32_t px = blockIdx.x * blockDim.x + threadIdx.x; px < npix; px += gridDim.x * blockDim.x) {
    const double3 f = film[px];
    out[3 * (size_t)px] = iters > 0 ? dd(f.x, iters) : 0.0;
    out[3 * (size_t)px + 1] = iters > 0 ? dd(f.y, iters) : 0.0;
    out[3 * (size_t)px + 2] = iters > 0 ? dd(f.z, iters) : 0.0;
  }
}

cudaError_t launch_trace_eye(cudaStream_t s, const EyeArgs &E, const void *prep, int sms) {
  if (E.npix == 0) return cudaSuccess;
  unsigned blocks = (E.npix + 127) / 128;
  if (blocks > (unsigned)sms * 16) blocks = sms * 16;
  k_trace_eye<<<blocks, 128, 0, s>>>(E, static_cast<const PrimD *>(prep));
  note_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_film(cudaStream_t s, int op, uint32_t npix, const double3 *emitted, const uint8_t *gathered,
                        const double *flux, const double *gather_r, double J, double3 *film, double *mean_out,
                        int sms, double2 *vcvm) {
  if (npix == 0) return cudaSuccess;
  unsigned blocks = (npix + 255) / 256;
  if (blocks > (unsigned)sms * 8) blocks = sms * 8;
  if (op == 0)
    k_film_add<<<blocks, 256, 0, s>>>(npix, emitted, gathered, flux, gather_r, J, film, vcvm);
  else
    k_film_mean<<<blocks, 256, 0, s>>>(npix, film, J, mean_out);
  note_launches(1);
  return cudaGetLastError();
}


// ---------------------------------------------------------------- VCM+ bidirectional remainder
// Renderer::pixel_bidir (integrator.cpp:492-653) for vcm_plus and the light
// sub-paths' camera connections (light_phase / camera_connect,
// integrator.cpp:236-301), restated in fp64 without FMA in the reference's
// operation order.  The merges themselves run on the gather kernels: the
// primary rough vertex becomes the pixel's region hit point (tested,
// integrator.cpp:596-602), the others are merge queries gathered without a
// region (the same kernel in delta-row mode).

// any hit in (tmin, tmax): occluded (scene_geometry.cpp:308-318)
__device__ __forceinline__ bool occluded(const PrimD *P, int np, DVec a, DVec b) {
  const DVec d = sub(b, a);
  const double dist = __dsqrt_rn(dot(d, d));
  if (dist == 0.0) return false;
  const DVec dir = mul(d, dd(1.0, dist));
  const double tmin = dm(1e-6, dist), tmax = dm(ds(1.0, 1e-6), dist);  // kShadowEps (scene.hpp:121)
  for (int i = 0; i < np; ++i) {
    double t;
    const bool ok = P[i].kind == 0 ? hit_sphere(P[i], a, dir, tmin, tmax, t) : hit_quad(P[i], a, dir, tmin, tmax, t);
    if (ok) return true;
  }
  return false;
}

// Lambertian Bsdf::eval (bsdf.cpp:53-63): f = albedo / pi when cos_o > 0 and
// cos_i > 0, with the forward / reverse cosine pdfs; black otherwise (mirror
// and dielectric have no non-delta lobe).
struct Eval {
  double f0, f1, f2, pf, pr;
  bool black;
};
__device__ __forceinline__ Eval bsdf_eval(const TraceScene &sc, int mat, DVec sn, double cos_o, DVec wi) {
  Eval e{0, 0, 0, 0, 0, true};
  const double cos_i = dot(wi, sn);
  if (cos_o <= 0.0 || cos_i <= 0.0) return e;
  if (sc.mat_kind[mat] != 0) return e;
  const double *a = sc.mat_rgb + 3 * (size_t)mat;
  e.pf = cos_pdf(cos_i);
  e.pr = cos_pdf(cos_o);
  e.f0 = dm(a[0], kInvPi);
  e.f1 = dm(a[1], kInvPi);
  e.f2 = dm(a[2], kInvPi);
  e.black = e.f0 == 0 && e.f1 == 0 && e.f2 == 0;
  return e;
}

struct MisC {  // MisContext (path.hpp:30-36) with the factors hoisted
  double beta, vmf, vcf;
};
__device__ __forceinline__ MisC mis_ctx(double beta, double eta) {
  MisC c;
  c.beta = beta;
  c.vmf = eta > 0.0 ? mpow(beta, eta) : 0.0;           // vm_factor (path.cpp:19-21)
  c.vcf = eta > 0.0 ? mpow(beta, dd(1.0, eta)) : 0.0;  // vc_factor (path.cpp:22-24)
  return c;
}

// Eye vertex of trace_eye_subpath (path.cpp:337-386), as the vertex loop
// reads it back (cos_exit = dot(gn, wo) replaces the geometric normal, which
// is only read for emitter hits, integrator.cpp:520-531).
struct EyeV {
  DVec pos, sn, wo;
  double t0, t1, t2, cos_exit;
  Mis mis;
  int mat, emitter;
  uint32_t depth;
  bool delta, front;
};

// The eye sub-paths live in HBM between the walk and the vertex loop:
// [field][vertex k][pixel] fp64 planes (16 fields) and one int4 plane
// (mat, emitter, depth, flags), so a warp's accesses at the same k are
// coalesced; a per-thread vertex array would sit in local memory and
// (at ~2.6 KB per thread) miss L1 on every access.
constexpr int kEyeVFields = 16;
__device__ __forceinline__ size_t eyev_at(const BidirArgs &B, int f, uint32_t k, uint32_t px) {
  return ((size_t)f * B.max_depth + k) * B.npix + px;
}
__device__ __forceinline__ void eyev_store(const BidirArgs &B, uint32_t k, uint32_t px, const EyeV &v) {
  const double f[kEyeVFields] = {v.pos.x, v.pos.y, v.pos.z, v.sn.x, v.sn.y, v.sn.z, v.wo.x, v.wo.y,
                                 v.wo.z, v.t0, v.t1, v.t2, v.mis.d_vcm, v.mis.d_vc, v.mis.d_vm, v.cos_exit};
#pragma unroll
  for (int i = 0; i < kEyeVFields; ++i) B.vtx_d[eyev_at(B, i, k, px)] = f[i];
  B.vtx_i[(size_t)k * B.npix + px] =
      make_int4(v.mat, v.emitter, (int)v.depth, (v.delta ? 1 : 0) | (v.front ? 2 : 0));
}
__device__ __forceinline__ EyeV eyev_load(const BidirArgs &B, uint32_t k, uint32_t px) {
  EyeV v;
  double f[kEyeVFields];
#pragma unroll
  for (int i = 0; i < kEyeVFields; ++i) f[i] = B.vtx_d[eyev_at(B, i, k, px)];
  v.pos = dv(f[0], f[1], f[2]);
  v.sn = dv(f[3], f[4], f[5]);
  v.wo = dv(f[6], f[7], f[8]);
  v.t0 = f[9]; v.t1 = f[10]; v.t2 = f[11];
  v.mis.d_vcm = f[12]; v.mis.d_vc = f[13]; v.mis.d_vm = f[14];
  v.cos_exit = f[15];
  const int4 q = B.vtx_i[(size_t)k * B.npix + px];
  v.mat = q.x;
  v.emitter = q.y;
  v.depth = (uint32_t)q.z;
  v.delta = (q.w & 1) != 0;
  v.front = (q.w & 2) != 0;
  return v;
}

#ifndef FPPM_EYE_MINB
#define FPPM_EYE_MINB 4   // walk: 120 registers, no spills
#endif
#ifndef FPPM_BIDIR_MINB
#define FPPM_BIDIR_MINB 4  // vertex loop: 128 registers + a small spill beat 166 at 3 CTAs (C4: 2.56 vs 2.64 ms)
#endif
// trace_eye_subpath (path.cpp:331-386) for every pixel: the vertices to HBM,
// the vertex count and the RNG state the vertex loop continues from.
__global__ void __launch_bounds__(128, FPPM_EYE_MINB) k_eye_walk(const BidirArgs B, const PrimD *__restrict__ prims) {
  __shared__ PrimD P[kMaxTracePrims];
  const TraceScene &sc = B.sc;
  const int np = sc.n_prim;
  for (int i = threadIdx.x; i < np; i += blockDim.x) P[i] = prims[i];
  __syncthreads();
  const CamD &cam = B.cam;
  const DVec fwd = dv(cam.fwd[0], cam.fwd[1], cam.fwd[2]);
  for (uint32_t px = blockIdx.x * blockDim.x + threadIdx.x; px < B.npix; px += gridDim.x * blockDim.x) {
    Rng rng(B.seed, B.iteration, px, 1ull /* kEyeStream */);
    const double r = B.radius[px];
    const double eta = dm(dm(dm((double)B.n_vm, kPi), r), r);  // n_vm * kPi * r * r (integrator.cpp:503)
    const MisC ctx = mis_ctx(B.beta, eta);
    const double sx = da((double)(px % (uint32_t)cam.width), rng.next());
    const double sy = da((double)(px / (uint32_t)cam.width), rng.next());
    DVec dir = normalize(add(add(mul(fwd, cam.plane_dist),
                                 mul(dv(cam.right[0], cam.right[1], cam.right[2]),
                                     ds(sx, dm(0.5, (double)cam.width)))),
                             mul(dv(cam.up[0], cam.up[1], cam.up[2]), ds(dm(0.5, (double)cam.height), sy))));
    DVec o = dv(cam.pos[0], cam.pos[1], cam.pos[2]);
    Mis mis;
    {  // mis_camera_origin (path.cpp:38-43) with camera_pdf_w (path.cpp:144-148)
      const double ct = dot(dir, fwd);
      const double cpdf = ct <= 0.0 ? 0.0 : dd(dm(cam.plane_dist, cam.plane_dist), dm(dm(ct, ct), ct));
      mis.d_vcm = mpow(B.beta, dd((double)B.n_paths, cpdf));
      mis.d_vc = 0.0;
      mis.d_vm = 0.0;
    }
    double t0 = 1.0, t1 = 1.0, t2 = 1.0;
    uint32_t nv = 0;
    for (uint32_t depth = 1; depth <= B.max_depth; ++depth) {
      HitD h;
      if (!intersect(P, np, o, dir, h)) break;
      const DVec wo = neg(dir);
      const double cos_in = fabs(dot(h.sn, wo));
      if (cos_in == 0.0) break;
      {  // mis_arrive
        const double inv_cos = dd(1.0, mpow(B.beta, cos_in));
        mis.d_vcm = dm(mis.d_vcm, dm(mpow(B.beta, dm(h.t, h.t)), inv_cos));
        mis.d_vc = dm(mis.d_vc, inv_cos);
        mis.d_vm = dm(mis.d_vm, inv_cos);
      }
      const int mk = sc.mat_kind[h.mat];
      EyeV v;
      v.pos = h.point;
      v.sn = h.sn;
      {  // fill_hit's geometric normal (gn = front ? outward : -outward)
        const PrimD &pp = P[h.prim];
        const DVec outward = pp.kind == 0 ? mul(sub(h.point, dv(pp.c[0], pp.c[1], pp.c[2])), pp.inv_r)
                                          : dv(pp.on[0], pp.on[1], pp.on[2]);
        const DVec gn = h.front ? outward : neg(outward);
        v.cos_exit = dot(gn, wo);  // emitter_hit_pdfs' cos_exit (path.cpp:320-329)
      }
      v.wo = wo;
      v.t0 = t0; v.t1 = t1; v.t2 = t2;
      v.mat = h.mat;
      v.emitter = P[h.prim].emitter;
      v.delta = mk != 0;
      v.front = h.front;
      v.depth = depth;
      v.mis = mis;
      eyev_store(B, nv++, px, v);
      if (depth == B.max_depth) break;
      const double cos_o = dot(wo, h.sn);
      DVec ndir;
      double s_cos, s_pdf, s_rev;
      bool s_delta;
      if (!bsdf_sample(sc, mk, h.mat, h.sn, wo, h.front, cos_o, rng, ndir, s_cos, s_pdf, s_rev, s_delta)) break;
      const double *w = sc.mat_rgb + 3 * (size_t)h.mat;
      if (s_pdf <= 0.0 || (w[0] == 0 && w[1] == 0 && w[2] == 0)) break;
      double q = 1.0;
      const double cont = cont_prob(sc, h.mat);
      if (depth >= 5) {  // kRouletteDepth
        q = cont;
        if (rng.next() >= q) break;
      }
      {  // mis_scatter with pdfs x continuation (path.cpp:52-76, 374-380)
        const double pf = dm(s_pdf, cont), pr = dm(s_rev, cont);
        if (s_delta) {
          const double f = mpow(B.beta, dd(dm(s_cos, pr), pf));
          mis.d_vcm = 0.0;
          mis.d_vc = dm(mis.d_vc, f);
          mis.d_vm = dm(mis.d_vm, f);
        } else {
          const double ratio = mpow(B.beta, dd(s_cos, pf));
          const double rev = mpow(B.beta, pr);
          const double d_vc = dm(ratio, da(da(dm(mis.d_vc, rev), mis.d_vcm), ctx.vmf));
          const double d_vm = dm(ratio, da(da(dm(mis.d_vm, rev), dm(mis.d_vcm, ctx.vcf)), 1.0));
          mis.d_vc = d_vc;
          mis.d_vm = d_vm;
          mis.d_vcm = mpow(B.beta, dd(1.0, pf));
        }
      }
      t0 = dd(dm(t0, w[0]), q);
      t1 = dd(dm(t1, w[1]), q);
      t2 = dd(dm(t2, w[2]), q);
      o = h.point;
      dir = ndir;
    }
    B.vtx_n[px] = nv;
    B.vtx_rng[px] = rng.s;
  }
}

// pixel_bidir's vertex loop (integrator.cpp:519-625) over the stored eye
// sub-path, continuing the pixel's RNG stream where the walk left it.
__global__ void __launch_bounds__(128, FPPM_BIDIR_MINB) k_eye_bidir(const BidirArgs B, const PrimD *__restrict__ prims) {
  __shared__ PrimD P[kMaxTracePrims];
  const TraceScene &sc = B.sc;
  const int np = sc.n_prim;
  for (int i = threadIdx.x; i < np; i += blockDim.x) P[i] = prims[i];
  __syncthreads();
  const uint32_t nq = B.max_depth > 1 ? B.max_depth - 1 : 1;
  const int n_emit = sc.n_emit;
  const double pick_prob = n_emit ? dd(1.0, (double)n_emit) : 0.0;
  for (uint32_t px = blockIdx.x * blockDim.x + threadIdx.x; px < B.npix; px += gridDim.x * blockDim.x) {
    Rng rng;
    rng.s = B.vtx_rng[px];
    const uint32_t nv = B.vtx_n[px];
    const double r = B.radius[px];
    const double eta = dm(dm(dm((double)B.n_vm, kPi), r), r);  // n_vm * kPi * r * r (integrator.cpp:503)
    const MisC ctx = mis_ctx(B.beta, eta);
    // ---- pixel_bidir's vertex loop (integrator.cpp:519-625)
    double o0 = 0.0, o1 = 0.0, o2 = 0.0;
    const uint32_t lp = px % B.n_paths;
    const size_t lbase = (size_t)lp * B.light_depth;
    const uint32_t lcount = B.l_count[lp];
    bool primary_seen = false;
    uint32_t nsec = 0;
    B.gathered[px] = 0;
    for (uint32_t k = 0; k < nv; ++k) {
      const EyeV v = eyev_load(B, k, px);
      if (v.emitter >= 0 && v.front) {  // emitted radiance (integrator.cpp:520-531)
        double w = 1.0;
        if (v.depth > 1) {
          // emitter_hit_pdfs (path.cpp:320-329): area emitters, cos_exit = dot(n, -ray_dir)
          const double cos_exit = v.cos_exit;
          if (cos_exit <= 0.0) {
            w = 0.0;
          } else {
            const double dpa = P[sc.emit_prim[v.emitter]].inv_area;
            const double epdf = dm(dpa, cos_pdf(cos_exit));
            const double a = dm(pick_prob, dpa), e = dm(pick_prob, epdf);
            // mis_weight_emitter_hit (path.cpp:78-83)
            const double wc = da(dm(mpow(B.beta, a), v.mis.d_vcm), dm(mpow(B.beta, e), v.mis.d_vc));
            w = dd(1.0, da(1.0, wc));
          }
        }
        const double *L = sc.emit_rad + 3 * (size_t)v.emitter;
        o0 = da(o0, dm(dm(v.t0, L[0]), w));
        o1 = da(o1, dm(dm(v.t1, L[1]), w));
        o2 = da(o2, dm(dm(v.t2, L[2]), w));
      }
      if (v.delta) continue;
      const double cos_o = dot(v.wo, v.sn);  // Bsdf ctor (bsdf.cpp:34)
      const double cont = cont_prob(sc, v.mat);
      // ---- next-event estimation (integrator.cpp:537-561)
      if (n_emit && v.depth + 1 <= B.max_depth) {
        int pick = (int)dm(rng.next(), (double)n_emit);
        if (pick > n_emit - 1) pick = n_emit - 1;
        // sample_direct, area emitters (path.cpp:262-277) via sample_area_point (path.cpp:172-189)
        const PrimD &ep = P[sc.emit_prim[pick]];
        DVec apos, anrm;
        if (ep.kind == 1) {
          const double u = rng.next(), w2 = rng.next();
          apos = add(add(dv(ep.c[0], ep.c[1], ep.c[2]), mul(dv(ep.e1[0], ep.e1[1], ep.e1[2]), u)),
                     mul(dv(ep.e2[0], ep.e2[1], ep.e2[2]), w2));
          anrm = dv(ep.on[0], ep.on[1], ep.on[2]);
        } else {
          const double u2 = rng.next(), u1 = rng.next();  // right-to-left arguments
          const DVec d_ = sample_uniform_sphere(u1, u2);
          apos = add(dv(ep.c[0], ep.c[1], ep.c[2]), mul(d_, ep.r));
          anrm = d_;
        }
        const double pdf_a = ep.inv_area;
        const DVec lv = sub(apos, v.pos);
        const double dist2 = dot(lv, lv);
        if (dist2 != 0.0) {
          const double dist = __dsqrt_rn(dist2);
          const DVec to_light = mul(lv, dd(1.0, dist));
          const double cos_at_light = dot(anrm, neg(to_light));
          const double *Le = sc.emit_rad + 3 * (size_t)pick;
          if (cos_at_light > 0.0 && !(Le[0] == 0 && Le[1] == 0 && Le[2] == 0)) {
            const double direct_pdf_w = dd(dm(pdf_a, dist2), cos_at_light);
            const double emission_pdf = dm(pdf_a, cos_pdf(cos_at_light));
            const Eval f = bsdf_eval(sc, v.mat, v.sn, cos_o, to_light);
            const double cos_v = fabs(dot(v.sn, to_light));
            if (!f.black && cos_v > 0.0 && !occluded(P, np, v.pos, add(v.pos, mul(to_light, dist)))) {
              // mis_weight_nee (path.cpp:85-95), delta_light = false
              const double dpw = dm(pick_prob, direct_pdf_w), epw = dm(pick_prob, emission_pdf);
              const double w_light = mpow(B.beta, dd(dm(f.pf, cont), dpw));
              const double w_camera =
                  dm(mpow(B.beta, dd(dm(epw, cos_v), dm(dpw, cos_at_light))),
                     da(da(ctx.vmf, v.mis.d_vcm), dm(v.mis.d_vc, mpow(B.beta, dm(f.pr, cont)))));
              const double w = dd(1.0, da(da(w_light, 1.0), w_camera));
              const double sc_ = dd(dm(w, cos_v), dpw);
              o0 = da(o0, dm(dm(dm(v.t0, f.f0), Le[0]), sc_));
              o1 = da(o1, dm(dm(dm(v.t1, f.f1), Le[1]), sc_));
              o2 = da(o2, dm(dm(dm(v.t2, f.f2), Le[2]), sc_));
            }
          }
        }
      }
      // ---- connections to light sub-path px % J (integrator.cpp:563-588)
      for (uint32_t li = 0; li < lcount; ++li) {
        const size_t sl = lbase + li, s3 = 3 * sl;
        if (v.depth + B.l_depth[sl] + 1 > B.max_depth) continue;
        const DVec lpos = dv(B.l_pos[s3], B.l_pos[s3 + 1], B.l_pos[s3 + 2]);
        DVec d = sub(lpos, v.pos);
        const double d2 = dot(d, d);
        if (d2 == 0.0) continue;
        const double dist = __dsqrt_rn(d2);
        d = divs(d, dist);
        const Eval fe = bsdf_eval(sc, v.mat, v.sn, cos_o, d);
        if (fe.black) continue;
        const DVec lsn = dv(B.l_sn[s3], B.l_sn[s3 + 1], B.l_sn[s3 + 2]);
        const DVec lwi = dv(B.l_wi[s3], B.l_wi[s3 + 1], B.l_wi[s3 + 2]);
        const int lmat = B.l_mat[sl];
        const Eval fl = bsdf_eval(sc, lmat, lsn, dot(lwi, lsn), neg(d));
        if (fl.black) continue;
        if (occluded(P, np, v.pos, lpos)) continue;
        const double lcont = cont_prob(sc, lmat);
        const double cos_e = fabs(dot(v.sn, d)), cos_l = fabs(dot(lsn, d));
        // mis_weight_connect (path.cpp:97-108)
        const double efa = dd(dm(dm(fe.pf, cont), cos_l), d2), erw = dm(fe.pr, cont);
        const double lfa = dd(dm(dm(fl.pf, lcont), cos_e), d2), lrw = dm(fl.pr, lcont);
        const double w_light = dm(mpow(B.beta, efa), da(da(ctx.vmf, B.l_mis[s3]), dm(B.l_mis[s3 + 1], mpow(B.beta, lrw))));
        const double w_camera = dm(mpow(B.beta, lfa), da(da(ctx.vmf, v.mis.d_vcm), dm(v.mis.d_vc, mpow(B.beta, erw))));
        const double w = dd(1.0, da(da(w_light, 1.0), w_camera));
        const double g = dd(dm(dm(w, cos_e), cos_l), d2);
        o0 = da(o0, dm(dm(dm(dm(v.t0, fe.f0), fl.f0), B.l_thr[s3]), g));
        o1 = da(o1, dm(dm(dm(dm(v.t1, fe.f1), fl.f1), B.l_thr[s3 + 1]), g));
        o2 = da(o2, dm(dm(dm(dm(v.t2, fe.f2), fl.f2), B.l_thr[s3 + 2]), g));
      }
      // ---- merge vertex (integrator.cpp:590-623)
      const bool primary = !primary_seen;
      primary_seen = true;
      const double *alb = sc.mat_rgb + 3 * (size_t)v.mat;
      if (primary) {
        B.pos[px] = make_double3(v.pos.x, v.pos.y, v.pos.z);
        B.nrm[px] = make_double3(v.sn.x, v.sn.y, v.sn.z);
        B.wo[px] = make_double3(v.wo.x, v.wo.y, v.wo.z);
        B.thr[px] = make_double3(v.t0, v.t1, v.t2);
        B.alb[px] = make_double3(alb[0], alb[1], alb[2]);
        B.eye_depth[px] = v.depth;
        B.eye_mis[px] = make_double2(v.mis.d_vcm, v.mis.d_vm);
        B.gathered[px] = 1;
      } else if (nsec < nq) {
        const size_t q = (size_t)px * nq + nsec++;
        B.q_pos[q] = make_double3(v.pos.x, v.pos.y, v.pos.z);
        B.q_nrm[q] = make_double3(v.sn.x, v.sn.y, v.sn.z);
        B.q_wo[q] = make_double3(v.wo.x, v.wo.y, v.wo.z);
        B.q_thr[q] = make_double3(v.t0, v.t1, v.t2);
        B.q_alb[q] = make_double3(alb[0], alb[1], alb[2]);
        B.q_eye[q] = v.depth;
        B.q_mis[q] = make_double2(v.mis.d_vcm, v.mis.d_vm);
        B.q_radius[q] = r;
        B.q_gathered[q] = 1;
      }
    }
    for (uint32_t k = nsec; k < nq; ++k) B.q_gathered[(size_t)px * nq + k] = 0;
    if (!primary_seen) {  // the region holds (integrator.cpp:627-631); placeholders
      B.pos[px] = make_double3(0, 0, 0);
      B.nrm[px] = make_double3(0, 0, 1);
      B.wo[px] = make_double3(0, 0, 1);
      B.thr[px] = make_double3(0, 0, 0);
      B.alb[px] = make_double3(0, 0, 0);
      B.eye_depth[px] = 0;
      B.eye_mis[px] = make_double2(0.0, 0.0);
    }
    B.direct[px] = make_double3(o0, o1, o2);
  }
}


// camera_connect (integrator.cpp:270-301) for every light vertex with
// depth + 1 <= max_depth: project_to_camera (path.cpp:150-170), the light
// vertex's Bsdf toward the camera, visibility, mis_weight_camera_connect
// (path.cpp:119-126) with the light sub-paths' context; the splat goes to the
// pixel the vertex projects to (fp64 atomics: the reference adds the splats
// serially in path order, so sums agree to rounding).
__global__ void __launch_bounds__(128) k_light_splat(const BidirArgs B, const PrimD *__restrict__ prims) {
  __shared__ PrimD P[kMaxTracePrims];
  const TraceScene &sc = B.sc;
  const int np = sc.n_prim;
  for (int i = threadIdx.x; i < np; i += blockDim.x) P[i] = prims[i];
  __syncthreads();
  const CamD &cam = B.cam;
  const DVec cpos = dv(cam.pos[0], cam.pos[1], cam.pos[2]), fwd = dv(cam.fwd[0], cam.fwd[1], cam.fwd[2]);
  const DVec right = dv(cam.right[0], cam.right[1], cam.right[2]), up = dv(cam.up[0], cam.up[1], cam.up[2]);
  const MisC ctx = mis_ctx(B.beta, B.eta_light);
  const double n_paths = (double)B.n_paths;
  const size_t nslots = (size_t)B.n_paths * B.light_depth;
  for (size_t sl = blockIdx.x * (size_t)blockDim.x + threadIdx.x; sl < nslots; sl += (size_t)gridDim.x * blockDim.x) {
    const uint32_t j = (uint32_t)(sl / B.light_depth), k = (uint32_t)(sl % B.light_depth);
    if (k >= B.l_count[j]) continue;
    if (B.l_depth[sl] + 1 > B.max_depth) continue;
    const size_t s3 = 3 * sl;
    const DVec p = dv(B.l_pos[s3], B.l_pos[s3 + 1], B.l_pos[s3 + 2]);
    // project_to_camera
    const DVec vv = sub(p, cpos);
    const double dist = __dsqrt_rn(dot(vv, vv));
    if (dist == 0.0) continue;
    const DVec d = mul(vv, dd(1.0, dist));
    const double ct = dot(d, fwd);
    if (ct <= 1e-9) continue;
    const DVec on_plane = mul(d, dd(cam.plane_dist, ct));
    const double sx = da(dm(0.5, (double)cam.width), dot(on_plane, right));
    const double sy = ds(dm(0.5, (double)cam.height), dot(on_plane, up));
    if (sx < 0.0 || sx >= (double)cam.width || sy < 0.0 || sy >= (double)cam.height) continue;
    const DVec to_cam = neg(d);
    const double pdf_w = dd(dm(cam.plane_dist, cam.plane_dist), dm(dm(ct, ct), ct));
    const DVec sn = dv(B.l_sn[s3], B.l_sn[s3 + 1], B.l_sn[s3 + 2]);
    const DVec wi = dv(B.l_wi[s3], B.l_wi[s3 + 1], B.l_wi[s3 + 2]);
    const int mat = B.l_mat[sl];
    const Eval f = bsdf_eval(sc, mat, sn, dot(wi, sn), to_cam);
    if (f.black) continue;
    if (occluded(P, np, p, cpos)) continue;
    const double cos_v = fabs(dot(sn, to_cam));
    const double dist2 = dm(dist, dist);
    const double cam_pdf_a = dd(dm(pdf_w, cos_v), dist2);
    const double rev = dm(f.pr, cont_prob(sc, mat));
    const double w_light = dm(mpow(B.beta, dd(cam_pdf_a, n_paths)),
                              da(da(ctx.vmf, B.l_mis[s3]), dm(B.l_mis[s3 + 1], mpow(B.beta, rev))));
    const double w = dd(1.0, da(w_light, 1.0));
    const double g = dd(dm(dm(w, pdf_w), cos_v), dm(dist2, n_paths));
    const double v0 = dm(dm(B.l_thr[s3], f.f0), g), v1 = dm(dm(B.l_thr[s3 + 1], f.f1), g),
                 v2 = dm(dm(B.l_thr[s3 + 2], f.f2), g);
    if (v0 == 0 && v1 == 0 && v2 == 0) continue;
    int x = (int)sx, y = (int)sy;
    x = x < 0 ? 0 : (x > cam.width - 1 ? cam.width - 1 : x);
    y = y < 0 ? 0 : (y > cam.height - 1 ? cam.height - 1 : y);
    double *o = reinterpret_cast<double *>(B.splat + (size_t)y * (uint32_t)cam.width + (uint32_t)x);
    atomicAdd(o, v0);
    atomicAdd(o + 1, v1);
    atomicAdd(o + 2, v2);
  }
}

// Film::add_iteration of the VCM+ estimate: out = direct + sum_k merge_k *
// vm_norm in vertex order (vm_norm = 1 / (pi r^2 J), integrator.cpp:505-506,
// 620) + the splats (integrator.cpp:205-211).
__global__ void k_film_vcm(uint32_t npix, uint32_t nq, const double3 *__restrict__ direct,
                           const uint8_t *__restrict__ gathered, const double *__restrict__ flux,
                           const double *__restrict__ gather_r, const double *__restrict__ q_rows, uint32_t q_stride,
                           const uint8_t *__restrict__ q_gathered, const double *__restrict__ q_radius,
                           const double3 *__restrict__ splat, double J, double3 *__restrict__ film,
                           double2 *__restrict__ vcvm) {
  for (uint32_t px = blockIdx.x * blockDim.x + threadIdx.x; px < npix; px += gridDim.x * blockDim.x) {
    double3 est = direct[px];
    // add_split (integrator.cpp:205-211, 623-624): vm = luminance of the
    // merges, vc = luminance of everything else (direct + camera splats)
    double vm = 0.0;
    if (gathered[px]) {
      const double r = gather_r[px];
      const double vn = dd(1.0, dm(dm(dm(kPi, r), r), J));
      const double c0 = dm(flux[3 * (size_t)px], vn), c1 = dm(flux[3 * (size_t)px + 1], vn),
                   c2 = dm(flux[3 * (size_t)px + 2], vn);
      vm = da(vm, elum(c0, c1, c2));
      est.x = da(est.x, c0);
      est.y = da(est.y, c1);
      est.z = da(est.z, c2);
    }
    for (uint32_t k = 0; k < nq; ++k) {
      const size_t q = (size_t)px * nq + k;
      if (!q_gathered[q]) break;
      const double r = q_radius[q];
      const double vn = dd(1.0, dm(dm(dm(kPi, r), r), J));
      const double *row = q_rows + q * q_stride + (q_stride - 3);
      const double c0 = dm(row[0], vn), c1 = dm(row[1], vn), c2 = dm(row[2], vn);
      vm = da(vm, elum(c0, c1, c2));
      est.x = da(est.x, c0);
      est.y = da(est.y, c1);
      est.z = da(est.z, c2);
    }
    const double3 sp = splat[px];
    if (vcvm) {
      double2 v = vcvm[px];
      v.x = da(v.x, da(elum(direct[px].x, direct[px].y, direct[px].z), elum(sp.x, sp.y, sp.z)));
      v.y = da(v.y, vm);
      vcvm[px] = v;
    }
    est.x = da(est.x, sp.x);
    est.y = da(est.y, sp.y);
    est.z = da(est.z, sp.z);
    double3 f = film[px];
    f.x = da(f.x, est.x);
    f.y = da(f.y, est.y);
    f.z = da(f.z, est.z);
    film[px] = f;
  }
}

cudaError_t launch_eye_bidir(cudaStream_t s, const BidirArgs &B, const void *prep, int sms) {
  if (B.npix == 0) return cudaSuccess;
  if (B.max_depth > kMaxBidirDepth) return cudaErrorInvalidValue;
  unsigned blocks = (B.npix + 127) / 128;
  if (blocks > (unsigned)sms * 16) blocks = sms * 16;
  k_eye_walk<<<blocks, 128, 0, s>>>(B, static_cast<const PrimD *>(prep));
  k_eye_bidir<<<blocks, 128, 0, s>>>(B, static_cast<const PrimD *>(prep));
  note_launches(2);
  return cudaGetLastError();
}

cudaError_t launch_light_splat(cudaStream_t s, const BidirArgs &B, const void *prep, int sms) {
  const unsigned long long n = (unsigned long long)B.n_paths * B.light_depth;
  if (n == 0) return cudaSuccess;
  unsigned long long blocks = (n + 127) / 128;
  if (blocks > (unsigned long long)sms * 16) blocks = (unsigned long long)sms * 16;
  k_light_splat<<<(unsigned)blocks, 128, 0, s>>>(B, static_cast<const PrimD *>(prep));
  note_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_film_vcm(cudaStream_t s, uint32_t npix, uint32_t nq_per_px, const double3 *direct,
                            const uint8_t *gathered, const double *flux, const double *gather_r,
                            const double *q_rows, uint32_t q_stride, const uint8_t *q_gathered,
                            const double *q_radius, const double3 *splat, double J, double3 *film, int sms,
                            double2 *vcvm) {
  if (npix == 0) return cudaSuccess;
  unsigned blocks = (npix + 255) / 256;
  if (blocks > (unsigned)sms * 8) blocks = sms * 8;
  k_film_vcm<<<blocks, 256, 0, s>>>(npix, nq_per_px, direct, gathered, flux, gather_r, q_rows, q_stride,
                                    q_gathered, q_radius, splat, J, film, vcvm);
  note_launches(1);
  return cudaGetLastError();
}

size_t trace_prep_bytes(int n_prim) { return sizeof(PrimD) * (size_t)(n_prim > 0 ? n_prim : 1); }
int trace_max_prims() { return kMaxTracePrims; }

cudaError_t launch_scene_prep(cudaStream_t s, const TraceScene &sc, void *prep) {
  if (sc.n_prim <= 0) return cudaSuccess;
  k_scene_prep<<<(sc.n_prim + 63) / 64, 64, 0, s>>>(sc, static_cast<PrimD *>(prep));
  note_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_trace(cudaStream_t s, const TraceArgs &A, const void *prep, int sms) {
  if (A.n_paths == 0) return cudaSuccess;
  cudaError_t e = cudaMemsetAsync(A.path_counter, 0, sizeof(uint32_t), s);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_trace_paths, 256, 0);
  if (e != cudaSuccess) return e;
  unsigned blocks = (unsigned)sms * (unsigned)(per_sm > 0 ? per_sm : 1);
  const unsigned need = (A.n_paths + 255) / 256;
  if (blocks > need) blocks = need;
  k_trace_paths<<<blocks, 256, 0, s>>>(A, static_cast<const PrimD *>(prep));
  note_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_trace_compact(cudaStream_t s, const TraceArgs &A, const uint32_t *base, float *pos,
                                 float *nrm, float *wi, float *pw, uint32_t *depth, double *mv, double *mm,
                                 double *mc, int sms) {
  if (A.n_paths == 0) return cudaSuccess;
  unsigned blocks = (A.n_paths + 255) / 256;
  if (blocks > (unsigned)sms * 8) blocks = sms * 8;
  k_trace_compact<<<blocks, 256, 0, s>>>(A, base, pos, nrm, wi, pw, depth, mv, mm, mc);
  note_launches(1);
  return cudaGetLastError();
}

}  // namespace fppm_b200
