// ref_driver.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" driver over the reference's OWN public C++ API
// (fppm::PhotonGrid, fppm::GatherRegion, fppm::Bsdf, the stat/special
// functions), compiled together with the unmodified reference sources from
// /root/reference/proj/core/src into oracle/_ref/libfppm_ref.so by
// oracle/Makefile.  It is the "reference" CPU arm of bench.py and the pin for
// the C restatement in fppm_oracle.c.
//
// The only reference logic restated here is Renderer::gather_disk's filter
// chain (proj/core/src/integrator.cpp:388-402) and the pixel_pm callback
// (:445-451, :452-455, :476-489), which live in a private class of
// integrator.cpp and cannot be called from outside.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <functional>
#include <limits>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <thread>
#include <unordered_map>
#include <utility>
#include <vector>

// Read-only access to PhotonGrid's private order_/keys_/cells_ so grid
// parity can be checked on keys and permutation, not only on query results.
#define private public
#include "fppm/photon_map.hpp"
#undef private
#include "fppm/bsdf.hpp"
#include "fppm/frame.hpp"
#include "fppm/gather.hpp"
#include "fppm/path.hpp"
#include "fppm/scene.hpp"
#include "fppm/integrator.hpp"
#include "fppm/film.hpp"
#include "fppm/sampling.hpp"
#include "fppm/special_functions.hpp"
#include "fppm/stat_tests.hpp"

using namespace fppm;

namespace {
constexpr double kNormalGuardCos = 0.86602540378443865; // integrator.cpp:47

template <typename F>
double guarded(int* err, F&& f) {
  try {
    return f();
  } catch (const std::invalid_argument&) {
    if (err) *err = 1;
  } catch (const std::domain_error&) {
    if (err) *err = 2;
  } catch (...) {
    if (err) *err = 9;
  }
  return 0.0;
}

// Same static split as parallel_ranges (integrator.cpp:55-70).
template <typename F>
void parallel_ranges(int threads, std::size_t count, F&& fn) {
  const std::size_t t =
      std::min<std::size_t>(std::max(threads, 1), std::max<std::size_t>(count, 1));
  if (t <= 1) {
    fn(std::size_t{0}, count);
    return;
  }
  std::vector<std::thread> pool;
  for (std::size_t w = 1; w < t; ++w)
    pool.emplace_back([&fn, w, t, count] { fn(count * w / t, count * (w + 1) / t); });
  fn(std::size_t{0}, count / t);
  for (auto& th : pool) th.join();
}
} // namespace

extern "C" {

// ---------------------------------------------------------------- scalars
int ref_sector_index(double u, double v, double r, int na, int ns, int* err) {
  return static_cast<int>(guarded(err, [&] {
    return static_cast<double>(sector_index(UnifiedPoint{u, v}, r, na, ns));
  }));
}
double ref_schedule_radius(double base, double alpha, uint64_t i) {
  return schedule_radius(base, alpha, i);
}
double ref_f_quantile(double p, double d1, double d2, int* err) {
  return guarded(err, [&] { return f_quantile(p, d1, d2); });
}
double ref_chi2_quantile(double p, double df, int* err) {
  return guarded(err, [&] { return chi2_quantile(p, df); });
}
double ref_f_cdf(double x, double d1, double d2, int* err) {
  return guarded(err, [&] { return f_cdf(x, d1, d2); });
}
double ref_chi2_cdf(double x, double df, int* err) {
  return guarded(err, [&] { return chi2_cdf(x, df); });
}
double ref_reg_inc_beta(double a, double b, double x, int* err) {
  return guarded(err, [&] { return reg_inc_beta(a, b, x); });
}
double ref_reg_lower_gamma(double a, double x, int* err) {
  return guarded(err, [&] { return reg_lower_gamma(a, x); });
}
static std::vector<SectorStats> make_stats(const uint64_t* c, const double* s,
                                           const double* q, int n) {
  std::vector<SectorStats> v(static_cast<std::size_t>(n));
  for (int i = 0; i < n; ++i) v[i] = SectorStats{c ? c[i] : 0, s[i], q[i]};
  return v;
}
double ref_f_statistic(const uint64_t* c, const double* s, const double* q, int n,
                       uint64_t m, int* err) {
  return guarded(err, [&] { return f_statistic(make_stats(c, s, q, n), m); });
}
// out: [f, critical, reject, d1, d2]
void ref_anova_f_test(const uint64_t* c, const double* s, const double* q, int n,
                      uint64_t m, double alpha, double* out, int* err) {
  guarded(err, [&] {
    const FTestResult r = anova_f_test(make_stats(c, s, q, n), m, alpha);
    out[0] = r.f;
    out[1] = r.critical;
    out[2] = r.reject ? 1.0 : 0.0;
    out[3] = static_cast<double>(r.d1);
    out[4] = static_cast<double>(r.d2);
    return 0.0;
  });
}
double ref_chi2_statistic(const uint64_t* c, int n, int* err) {
  return guarded(err, [&] {
    return chi2_statistic(std::span<const std::uint64_t>(c, static_cast<std::size_t>(n)));
  });
}
void ref_build_frame(const double* n, double* u, double* v) {
  const TangentFrame f = build_tangent_frame(Normal3{n[0], n[1], n[2]});
  u[0] = f.u.x; u[1] = f.u.y; u[2] = f.u.z;
  v[0] = f.v.x; v[1] = f.v.y; v[2] = f.v.z;
}

// ---------------------------------------------------------------- grid
void* ref_grid_build(const double* pos, size_t n, double cell, int* err) {
  try {
    std::vector<LightVertex> vs(n);
    for (size_t i = 0; i < n; ++i) {
      vs[i].position = Point3{pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]};
      vs[i].path_index = static_cast<uint32_t>(i);
    }
    return new PhotonGrid(std::move(vs), cell);
  } catch (const std::invalid_argument&) {
    if (err) *err = 1;
  }
  return nullptr;
}
void ref_grid_free(void* g) { delete static_cast<PhotonGrid*>(g); }
size_t ref_grid_cell_count(void* g) { return static_cast<PhotonGrid*>(g)->keys_.size(); }
void ref_grid_export(void* gp, uint64_t* keys, uint32_t* begin, uint32_t* end,
                     uint32_t* order) {
  const PhotonGrid* g = static_cast<PhotonGrid*>(gp);
  for (size_t i = 0; i < g->keys_.size(); ++i) {
    if (keys) keys[i] = g->keys_[i];
    if (begin) begin[i] = g->cells_[i].begin;
    if (end) end[i] = g->cells_[i].end;
  }
  if (order) std::memcpy(order, g->order_.data(), sizeof(uint32_t) * g->order_.size());
}
size_t ref_grid_query_ball(void* gp, const double* c, double r, uint32_t* out,
                           size_t cap, int* err) {
  std::vector<uint32_t> found;
  try {
    static_cast<PhotonGrid*>(gp)->query_ball(Point3{c[0], c[1], c[2]}, r, found);
  } catch (const std::invalid_argument&) {
    if (err) *err = 1;
    return 0;
  }
  for (size_t i = 0; i < found.size() && i < cap; ++i) out[i] = found[i];
  return found.size();
}

// ---------------------------------------------------------------- session
struct RefConfig { // identical layout to orc_config (fppm_oracle.h)
  int n_annuli, n_sectors;
  double alpha_f;
  int channels;
  int override_decision;
  double k, alpha, r_min_base;
  double initial_radius;
  uint64_t samples_per_iteration;
  uint32_t max_depth;
  double normal_guard_cos;
  int threads;
  double alpha_chi2;
  int policy;  // 0 end_iteration, 1 chi2_end_iteration, 2 schedule_end_iteration
  int vcm_plus;
  int mis_n_vm;
  double mis_beta;
};

struct RefIterOut { // identical layout to orc_iter_out
  double* radius;
  double* gather_r;
  uint64_t* t;
  uint8_t* tested;
  uint8_t* rejected;
  double* statistic;
  double* critical;
  double* flux;
  double* radiance;
  uint64_t* accepted;
  uint64_t* stat_count;
  double* stat_sum;
  double* stat_sum_sq;
};

struct RefSession {
  RefConfig cfg;
  std::vector<GatherRegion> regions;
  std::vector<Point3> pos;
  std::vector<Normal3> nrm;
  std::vector<Vec3> wo;
  std::vector<Rgb> thr;
  std::vector<Material> mat;
  std::vector<uint32_t> eye_depth;
  std::vector<uint8_t> gathered;
  std::vector<MisPartials> eye_mis;            // VCM+ (PathVertex::mis)
  const double *ph_d_vcm = nullptr, *ph_d_vm = nullptr, *ph_cont = nullptr;  // VCM+
};

void* ref_session_create(const RefConfig* cfg, size_t H, const double* pos,
                         const double* nrm, const double* wo, const double* thr,
                         const double* alb, const uint32_t* eye_depth,
                         const uint8_t* gathered, int* err) {
  try {
    auto* s = new RefSession;
    s->cfg = *cfg;
    TestConfig test;
    test.n_annuli = cfg->n_annuli;
    test.n_sectors = cfg->n_sectors;
    test.alpha_f = cfg->alpha_f;
    test.alpha_chi2 = cfg->alpha_chi2;
    test.channels = cfg->channels == 3 ? TestChannels::rgb : TestChannels::luminance;
    test.override_decision = cfg->override_decision == 1   ? TestOverride::always_reject
                             : cfg->override_decision == 2 ? TestOverride::never_reject
                                                           : TestOverride::none;
    const RadiusSchedule sched{cfg->k, cfg->alpha, cfg->r_min_base};
    s->regions.assign(H, GatherRegion(test, sched, cfg->initial_radius));
    for (size_t h = 0; h < H; ++h) {
      s->pos.push_back({pos[3 * h], pos[3 * h + 1], pos[3 * h + 2]});
      s->nrm.push_back({nrm[3 * h], nrm[3 * h + 1], nrm[3 * h + 2]});
      s->wo.push_back({wo[3 * h], wo[3 * h + 1], wo[3 * h + 2]});
      s->thr.push_back({thr[3 * h], thr[3 * h + 1], thr[3 * h + 2]});
      Material m;
      m.kind = MaterialKind::lambertian;
      m.albedo = Rgb{alb[3 * h], alb[3 * h + 1], alb[3 * h + 2]};
      s->mat.push_back(m);
      s->eye_depth.push_back(eye_depth[h]);
      s->gathered.push_back(gathered ? gathered[h] : 1);
    }
    s->eye_mis.assign(H, MisPartials{});
    return s;
  } catch (const std::invalid_argument&) {
    if (err) *err = 1;
  }
  return nullptr;
}

void ref_session_free(void* s) { delete static_cast<RefSession*>(s); }

void ref_session_set_hitpoints(void* sp, const double* pos, const double* nrm, const double* wo,
                               const double* thr, const double* alb, const uint32_t* eye_depth,
                               const uint8_t* gathered) {
  auto* s = static_cast<RefSession*>(sp);
  for (size_t h = 0; h < s->pos.size(); ++h) {
    s->pos[h] = {pos[3 * h], pos[3 * h + 1], pos[3 * h + 2]};
    s->nrm[h] = {nrm[3 * h], nrm[3 * h + 1], nrm[3 * h + 2]};
    s->wo[h] = {wo[3 * h], wo[3 * h + 1], wo[3 * h + 2]};
    s->thr[h] = {thr[3 * h], thr[3 * h + 1], thr[3 * h + 2]};
    s->mat[h].albedo = Rgb{alb[3 * h], alb[3 * h + 1], alb[3 * h + 2]};
    s->eye_depth[h] = eye_depth[h];
    s->gathered[h] = gathered ? gathered[h] : 1;
  }
}

void ref_session_set_eye_mis(void* sp, const double* d_vcm, const double* d_vm) {
  auto* s = static_cast<RefSession*>(sp);
  for (size_t h = 0; h < s->eye_mis.size(); ++h) {
    s->eye_mis[h].d_vcm = d_vcm ? d_vcm[h] : 0.0;
    s->eye_mis[h].d_vm = d_vm ? d_vm[h] : 0.0;
  }
}

void ref_session_set_photon_mis(void* sp, const double* d_vcm, const double* d_vm, const double* cont,
                                size_t) {
  auto* s = static_cast<RefSession*>(sp);
  s->ph_d_vcm = d_vcm;
  s->ph_d_vm = d_vm;
  s->ph_cont = cont;
}

double ref_mis_weight_merge(int n_vm, double beta, double r, double eye_d_vcm, double eye_d_vm,
                            double light_d_vcm, double light_d_vm, double fwd, double rev) {
  MisContext ctx{1, n_vm, beta, 0.0};
  ctx.eta_vm = ctx.n_vm * kPi * r * r;  // integrator.cpp:503
  MisPartials e, l;
  e.d_vcm = eye_d_vcm;
  e.d_vm = eye_d_vm;
  l.d_vcm = light_d_vcm;
  l.d_vm = light_d_vm;
  return mis_weight_merge(ctx, e, l, fwd, rev);
}

double ref_session_max_radius(void* sp) {
  auto* s = static_cast<RefSession*>(sp);
  double r = 0.0;
  for (const GatherRegion& g : s->regions) r = std::max(r, g.radius());
  return r;
}

// Builds the reference PhotonGrid from canonical fp32 photons widened to
// double, then gathers + tests every selected hit point exactly as
// Renderer::pixel_pm does (integrator.cpp:407-490) for a first-hit diffuse
// gather point.  grid_seconds / gather_seconds receive steady-clock timings.
// Photon fields as float (the device's canonical records) or double (the
// reference tracer's own LightVertex values, for attributing fp32 narrowing).
}  // extern "C"
template <typename T>
static int session_iterate(void* sp, uint64_t iteration, const T* ppos, const T* pnrm, const T* pwi,
                           const T* ppow, const uint32_t* pdepth, size_t N, double cell_size,
                           const uint32_t* subset, size_t nsub, RefIterOut* out,
                           double* grid_seconds, double* gather_seconds) {
  auto* s = static_cast<RefSession*>(sp);
  const RefConfig& cfg = s->cfg;
  double cell = cell_size;
  if (!(cell > 0)) cell = ref_session_max_radius(sp); // integrator.cpp:159-161
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<LightVertex> flat(N);
  for (size_t i = 0; i < N; ++i) {
    LightVertex& v = flat[i];
    v.position = {ppos[3 * i], ppos[3 * i + 1], ppos[3 * i + 2]};
    v.shading_normal = {pnrm[3 * i], pnrm[3 * i + 1], pnrm[3 * i + 2]};
    v.geom_normal = v.shading_normal;
    v.wi = {pwi[3 * i], pwi[3 * i + 1], pwi[3 * i + 2]};
    v.throughput = {ppow[3 * i], ppow[3 * i + 1], ppow[3 * i + 2]};
    v.path_index = static_cast<uint32_t>(i);
    v.depth = pdepth[i];
    if (cfg.vcm_plus && s->ph_d_vcm) {
      v.mis.d_vcm = s->ph_d_vcm[i];
      v.mis.d_vm = s->ph_d_vm[i];
      v.cont = s->ph_cont[i];
    }
  }
  PhotonGrid grid;
  try {
    grid = PhotonGrid(std::move(flat), cell); // integrator.cpp:262-264
  } catch (const std::invalid_argument&) {
    return 1;
  }
  const auto t1 = std::chrono::steady_clock::now();
  const std::vector<LightVertex>& photons = grid.vertices();
  const size_t count = subset ? nsub : s->regions.size();
  const int CG = cfg.n_annuli * cfg.n_sectors * (cfg.channels == 3 ? 3 : 1);
  int failure = 0;

  parallel_ranges(cfg.threads, count, [&](size_t begin, size_t end) {
    std::vector<uint32_t> query;
    for (size_t slot = begin; slot < end; ++slot) {
      const size_t h = subset ? subset[slot] : slot;
      GatherRegion* region = &s->regions[h];
      const double r = region->radius(); // :411
      if (out && out->gather_r) out->gather_r[slot] = r;
      Rgb sum;
      uint64_t accepted = 0;
      const bool gathered = s->gathered[h] != 0;
      try {
        if (gathered) {
          const Point3& center = s->pos[h];
          const Normal3& normal = s->nrm[h];
          region->move_to(center, normal); // :438
          const TangentFrame frame = region->frame();
          const Bsdf bsdf(s->mat[h], normal, s->wo[h], true);
          const Rgb throughput = s->thr[h];
          // gather_disk (:388-402)
          grid.query_ball(center, r, query);
          const double r2 = r * r;
          for (const uint32_t id : query) {
            const LightVertex& p = photons[id];
            if (s->eye_depth[h] + p.depth > cfg.max_depth) continue;
            if (dot(p.shading_normal, normal) < cfg.normal_guard_cos) continue;
            const UnifiedPoint y = map_to_unified(center, p.position, frame);
            if (y.u * y.u + y.v * y.v > r2) continue;
            // callback (:445-451); VCM+ merge callback (:609-616)
            double pf = 0, pr = 0;
            const Rgb f = bsdf.eval(p.wi, pf, pr);
            Rgb val = throughput * f * p.throughput;
            if (cfg.vcm_plus) {
              MisContext ctx{1, cfg.mis_n_vm, cfg.mis_beta, 0.0};
              ctx.eta_vm = ctx.n_vm * kPi * r * r;  // :503
              const double w = mis_weight_merge(ctx, s->eye_mis[h], p.mis,
                                                pf * bsdf.continuation_prob(), pr * p.cont);
              val = throughput * f * p.throughput * w;
            }
            sum += val;
            region->accumulate({y, val});
            ++accepted;
          }
        }
      } catch (...) {
        failure = 2;
        return;
      }
      if (out && out->flux) {
        out->flux[3 * slot] = sum.r; out->flux[3 * slot + 1] = sum.g; out->flux[3 * slot + 2] = sum.b;
      }
      if (out && out->radiance) {
        const Rgb c = gathered ? sum / (kPi * r * r * static_cast<double>(cfg.samples_per_iteration))
                               : Rgb{};
        out->radiance[3 * slot] = c.r; out->radiance[3 * slot + 1] = c.g; out->radiance[3 * slot + 2] = c.b;
      }
      if (out && out->accepted) out->accepted[slot] = accepted;
      if (out && (out->stat_count || out->stat_sum || out->stat_sum_sq)) {
        for (int c = 0; c < region->channel_count(); ++c) {
          const auto st = region->sector_stats(c);
          for (size_t g = 0; g < st.size(); ++g) {
            const size_t o = static_cast<size_t>(CG) * slot + static_cast<size_t>(c) * st.size() + g;
            if (out->stat_count) out->stat_count[o] = st[g].count;
            if (out->stat_sum) out->stat_sum[o] = st[g].sum;
            if (out->stat_sum_sq) out->stat_sum_sq[o] = st[g].sum_sq;
          }
        }
      }
      RadiusUpdate up;
      if (cfg.policy == 2) {
        // the global schedule moves every region (integrator.cpp:159-164, 213-217)
        up = region->schedule_end_iteration(iteration);
      } else if (gathered) {
        // :478-480 (CPPM uses chi2_end_iteration); schedule policy: gather.cpp:138
        up = cfg.policy == 1   ? region->chi2_end_iteration(iteration, cfg.samples_per_iteration)
             : cfg.policy == 2 ? region->schedule_end_iteration(iteration)
                               : region->end_iteration(iteration, cfg.samples_per_iteration);
      } else {
        up.radius = region->radius(); // :486
      }
      if (out && out->radius) out->radius[slot] = up.radius;
      if (out && out->t) out->t[slot] = region->held_iterations();
      if (out && out->tested) out->tested[slot] = up.tested ? 1 : 0;
      if (out && out->rejected) out->rejected[slot] = up.rejected ? 1 : 0;
      if (out && out->statistic) out->statistic[slot] = up.statistic;
      if (out && out->critical) out->critical[slot] = up.critical;
    }
  });
  const auto t2 = std::chrono::steady_clock::now();
  if (grid_seconds) *grid_seconds = std::chrono::duration<double>(t1 - t0).count();
  if (gather_seconds) *gather_seconds = std::chrono::duration<double>(t2 - t1).count();
  return failure;
}
extern "C" {

int ref_session_iterate(void* sp, uint64_t iteration, const float* ppos, const float* pnrm, const float* pwi,
                        const float* ppow, const uint32_t* pdepth, size_t N, double cell_size,
                        const uint32_t* subset, size_t nsub, RefIterOut* out, double* grid_seconds,
                        double* gather_seconds) {
  return session_iterate<float>(sp, iteration, ppos, pnrm, pwi, ppow, pdepth, N, cell_size, subset, nsub, out,
                                grid_seconds, gather_seconds);
}

int ref_session_iterate_f64(void* sp, uint64_t iteration, const double* ppos, const double* pnrm,
                            const double* pwi, const double* ppow, const uint32_t* pdepth, size_t N,
                            double cell_size, const uint32_t* subset, size_t nsub, RefIterOut* out,
                            double* grid_seconds, double* gather_seconds) {
  return session_iterate<double>(sp, iteration, ppos, pnrm, pwi, ppow, pdepth, N, cell_size, subset, nsub, out,
                                 grid_seconds, gather_seconds);
}

// ---- light phase (Renderer::light_phase, integrator.cpp:230-265) ----------
// Scene arrays mirror fppm_scene (include/fppm_gpu.h): materials kind 0
// lambertian / 1 mirror / 2 dielectric with one rgb (albedo / reflectance /
// tint) and ior; shapes kind 0 sphere (center, radius) / 1 quad (corner, e1,
// e2) packed in 9 doubles; area emitters (shape, radiance).
struct RefScene {
  Scene scene;
};

void* ref_scene_create(uint32_t nm, const int32_t* mkind, const double* mrgb, const double* mior, uint32_t np,
                       const int32_t* skind, const double* shape, const int32_t* smat, uint32_t ne,
                       const int32_t* eshape, const double* erad) {
  auto* rs = new RefScene;
  Scene& sc = rs->scene;
  for (uint32_t i = 0; i < nm; ++i) {
    Material m;
    const Rgb c{mrgb[3 * i], mrgb[3 * i + 1], mrgb[3 * i + 2]};
    m.kind = mkind[i] == 0 ? MaterialKind::lambertian
                           : (mkind[i] == 1 ? MaterialKind::mirror : MaterialKind::dielectric);
    m.albedo = c;
    m.reflectance = c;
    m.tint = c;
    m.ior = mior[i];
    sc.materials.push_back(m);
  }
  for (uint32_t i = 0; i < np; ++i) {
    Primitive p;
    const double* q = shape + 9 * i;
    if (skind[i] == 0) {
      p.kind = ShapeKind::sphere;
      p.sphere.center = {q[0], q[1], q[2]};
      p.sphere.radius = q[3];
    } else {
      p.kind = ShapeKind::quad;
      p.quad.corner = {q[0], q[1], q[2]};
      p.quad.e1 = {q[3], q[4], q[5]};
      p.quad.e2 = {q[6], q[7], q[8]};
    }
    p.material = smat[i];
    sc.primitives.push_back(p);
  }
  for (uint32_t i = 0; i < ne; ++i) {
    Emitter e;
    e.kind = EmitterKind::area;
    e.primitive = eshape[i];
    e.radiance = Rgb{erad[3 * i], erad[3 * i + 1], erad[3 * i + 2]};
    sc.primitives[static_cast<std::size_t>(eshape[i])].emitter = static_cast<int>(i);
    sc.emitters.push_back(e);
  }
  build_accel(sc);
  return rs;
}

void ref_scene_free(void* s) { delete static_cast<RefScene*>(s); }

// The reference's own parser (scene_parse.cpp parse_scene): a RefScene, or
// nullptr with the ParseError message in `err` (cap bytes).
void* ref_scene_parse(const char* text, char* err, size_t cap) {
  try {
    auto* rs = new RefScene;
    rs->scene = parse_scene(text, "", "<scene>");
    return rs;
  } catch (const std::exception& e) {
    if (err && cap) {
      std::strncpy(err, e.what(), cap - 1);
      err[cap - 1] = 0;
    }
  }
  return nullptr;
}

// counts: [materials, primitives, emitters, has_camera]; then the arrays in
// the fppm_scene layout (NULL to query counts only) and the camera
// (pos, look, up, vfov, width, height).
void ref_scene_export(void* sp, int* counts, int* mkind, double* mrgb, double* mior, int* skind, double* shape,
                      int* smat, int* eshape, double* erad, double* cam) {
  const Scene& sc = static_cast<RefScene*>(sp)->scene;
  counts[0] = (int)sc.materials.size();
  counts[1] = (int)sc.primitives.size();
  counts[2] = (int)sc.emitters.size();
  counts[3] = sc.has_camera ? 1 : 0;
  if (!mkind) return;
  for (size_t i = 0; i < sc.materials.size(); ++i) {
    const Material& m = sc.materials[i];
    const Rgb c = m.kind == MaterialKind::lambertian ? m.albedo
                  : m.kind == MaterialKind::mirror   ? m.reflectance
                                                     : m.tint;
    mkind[i] = m.kind == MaterialKind::lambertian ? 0 : m.kind == MaterialKind::mirror ? 1
               : m.kind == MaterialKind::dielectric ? 2 : 3;
    mrgb[3 * i] = c.r; mrgb[3 * i + 1] = c.g; mrgb[3 * i + 2] = c.b;
    mior[i] = m.ior;
  }
  for (size_t i = 0; i < sc.primitives.size(); ++i) {
    const Primitive& p = sc.primitives[i];
    double* q = shape + 9 * i;
    for (int k = 0; k < 9; ++k) q[k] = 0.0;
    if (p.kind == ShapeKind::sphere) {
      skind[i] = 0;
      q[0] = p.sphere.center.x; q[1] = p.sphere.center.y; q[2] = p.sphere.center.z; q[3] = p.sphere.radius;
    } else {
      skind[i] = p.kind == ShapeKind::quad ? 1 : 2;
      q[0] = p.quad.corner.x; q[1] = p.quad.corner.y; q[2] = p.quad.corner.z;
      q[3] = p.quad.e1.x; q[4] = p.quad.e1.y; q[5] = p.quad.e1.z;
      q[6] = p.quad.e2.x; q[7] = p.quad.e2.y; q[8] = p.quad.e2.z;
    }
    smat[i] = p.material;
  }
  for (size_t i = 0; i < sc.emitters.size(); ++i) {
    eshape[i] = sc.emitters[i].primitive;
    erad[3 * i] = sc.emitters[i].radiance.r;
    erad[3 * i + 1] = sc.emitters[i].radiance.g;
    erad[3 * i + 2] = sc.emitters[i].radiance.b;
  }
  if (sc.has_camera && cam) {
    const Camera& c = sc.camera;
    const double v[12] = {c.position.x, c.position.y, c.position.z, c.look_at.x, c.look_at.y, c.look_at.z,
                          c.up.x, c.up.y, c.up.z, c.vfov_deg, (double)c.width, (double)c.height};
    for (int k = 0; k < 12; ++k) cam[k] = v[k];
  }
}

// Traces light paths [begin, end) of `iteration` with RngStream(seed,
// iteration, j, kLightStream = 0) and light_depth = max_depth - 1, then
// flattens the vertices in path order.  Writes up to `cap` vertices (fp64
// pos/nrm/wi/pow [.][3], depth, path index, mis [.][3] = d_vcm, d_vm, cont)
// and returns the total count (call again with a larger cap if it exceeds).
size_t ref_trace_photons(void* sp, uint64_t seed, uint64_t iteration, uint32_t begin, uint32_t end,
                         uint32_t max_depth, int n_vm, double beta, double eta_vm, int threads, size_t cap,
                         double* pos, double* nrm, double* wi, double* pw, uint32_t* depth, uint32_t* path,
                         double* mis) {
  const Scene& sc = static_cast<RefScene*>(sp)->scene;
  MisContext ctx;
  ctx.n_vm = n_vm;
  ctx.beta = beta;
  ctx.eta_vm = eta_vm;
  const uint32_t light_depth = max_depth > 0 ? max_depth - 1 : 0;
  std::vector<LightPath> paths(end - begin);
  parallel_ranges(threads, paths.size(), [&](std::size_t b, std::size_t e) {
    for (std::size_t k = b; k < e; ++k) {
      const std::size_t j = begin + k;
      RngStream rng(seed, iteration, j, 0 /* kLightStream */);
      paths[k] = trace_light_subpath(sc, ctx, static_cast<std::uint32_t>(j), light_depth, rng);
    }
  });
  size_t n = 0;
  for (const LightPath& p : paths)
    for (const LightVertex& v : p.vertices) {
      if (n < cap && pos) {
        const double a[4][3] = {{v.position.x, v.position.y, v.position.z},
                                {v.shading_normal.x, v.shading_normal.y, v.shading_normal.z},
                                {v.wi.x, v.wi.y, v.wi.z},
                                {v.throughput.r, v.throughput.g, v.throughput.b}};
        double* dst[4] = {pos, nrm, wi, pw};
        for (int f = 0; f < 4; ++f)
          for (int c = 0; c < 3; ++c) dst[f][3 * n + c] = a[f][c];
        depth[n] = v.depth;
        path[n] = v.path_index;
        mis[3 * n] = v.mis.d_vcm;
        mis[3 * n + 1] = v.mis.d_vm;
        mis[3 * n + 2] = v.cont;
      }
      ++n;
    }
  return n;
}

// ---- eye pass + full render ------------------------------------------------
static Camera make_cam(const double* c9, double vfov, int w, int h) {
  Camera cam;
  cam.position = {c9[0], c9[1], c9[2]};
  cam.look_at = {c9[3], c9[4], c9[5]};
  cam.up = {c9[6], c9[7], c9[8]};
  cam.vfov_deg = vfov;
  cam.width = w;
  cam.height = h;
  return cam;
}

// Renderer::pixel_pm's camera walk (integrator.cpp:407-474) up to the gather,
// restated on the reference's public pieces (the Renderer is private):
// make_camera_frame / make_camera_ray, intersect, Bsdf, RngStream with
// kEyeStream = 1.  Per pixel: hit point (pos, shading normal, wo, throughput,
// albedo, eye depth, gathered) and the emitted radiance collected on the way.
void ref_eye_pass(void* sp, const double* cam9, double vfov, int w, int h, uint64_t seed, uint64_t iteration,
                  uint32_t max_depth, double* pos, double* nrm, double* wo_out, double* thr, double* alb,
                  uint32_t* eye_depth, uint8_t* gathered, double* emitted) {
  const Scene& scene = static_cast<RefScene*>(sp)->scene;
  const CameraFrame cam = make_camera_frame(make_cam(cam9, vfov, w, h));
  const std::size_t npix = static_cast<std::size_t>(w) * h;
  for (std::size_t px = 0; px < npix; ++px) {
    RngStream rng(seed, iteration, px, 1 /* kEyeStream */);
    const double sx = static_cast<double>(px % cam.width) + rng.next_double();
    const double sy = static_cast<double>(px / cam.width) + rng.next_double();
    Ray ray = make_camera_ray(cam, sx, sy);
    Rgb throughput{1.0, 1.0, 1.0};
    Rgb out;
    gathered[px] = 0;
    eye_depth[px] = 0;
    for (int k = 0; k < 3; ++k) pos[3 * px + k] = nrm[3 * px + k] = wo_out[3 * px + k] = thr[3 * px + k] = alb[3 * px + k] = 0.0;
    nrm[3 * px + 2] = wo_out[3 * px + 2] = 1.0;
    for (std::uint32_t depth = 1; depth <= max_depth; ++depth) {
      const auto hit = intersect(scene, ray);
      if (!hit) break;
      const Vec3 wo = -ray.dir;
      if (hit->emitter >= 0 && hit->front_face)
        out += throughput * scene.emitters[static_cast<std::size_t>(hit->emitter)].radiance;
      const Material& mat = scene.materials[static_cast<std::size_t>(hit->material)];
      const Bsdf bsdf(mat, hit->shading_normal, wo, hit->front_face);
      if (!bsdf.is_delta_only()) {
        const double p3[5][3] = {{hit->point.x, hit->point.y, hit->point.z},
                                 {hit->shading_normal.x, hit->shading_normal.y, hit->shading_normal.z},
                                 {wo.x, wo.y, wo.z},
                                 {throughput.r, throughput.g, throughput.b},
                                 {mat.albedo.r, mat.albedo.g, mat.albedo.b}};
        double* dst[5] = {pos, nrm, wo_out, thr, alb};
        for (int f = 0; f < 5; ++f)
          for (int k = 0; k < 3; ++k) dst[f][3 * px + k] = p3[f][k];
        eye_depth[px] = depth;
        gathered[px] = 1;
        break;
      }
      if (depth == max_depth) break;
      const auto s = bsdf.sample(rng);
      if (!s || s->pdf_w <= 0.0 || s->weight.is_black()) break;
      double q = 1.0;
      if (depth >= kRouletteDepth) {
        q = bsdf.continuation_prob();
        if (rng.next_double() >= q) break;
      }
      throughput = throughput * s->weight / q;
      ray = Ray{hit->point, s->dir};
    }
    emitted[3 * px] = out.r;
    emitted[3 * px + 1] = out.g;
    emitted[3 * px + 2] = out.b;
  }
}

// The reference's own render() (integrator.cpp:669-...) with the FPPM
// algorithm: film mean [npix][3] and the last iteration's radii [npix].
static int render_algo(Algorithm algo, void* sp, const double* cam9, double vfov, int w, int h, uint64_t seed,
                       uint64_t iterations, uint32_t max_depth, uint64_t light_paths, double r0_frac, int na, int ns,
                       double alpha_f, int threads, double* film_mean, double* radius, double* seconds) {
  RefScene* rs = static_cast<RefScene*>(sp);
  Scene scene = rs->scene;
  scene.has_camera = true;
  scene.camera = make_cam(cam9, vfov, w, h);
  IntegratorConfig cfg;
  cfg.algorithm = algo;
  cfg.iterations = iterations;
  cfg.seed = seed;
  cfg.max_depth = max_depth;
  cfg.threads = threads;
  cfg.r0_frac = r0_frac;
  cfg.light_paths = light_paths;
  cfg.test.n_annuli = na;
  cfg.test.n_sectors = ns;
  cfg.test.alpha_f = alpha_f;
  try {
    const auto t0 = std::chrono::steady_clock::now();
    RenderResult res = render(scene, cfg);
    if (seconds) *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    const Image img = res.film.image();
    for (std::size_t i = 0; i < img.pixels.size(); ++i) {
      film_mean[3 * i] = img.pixels[i].r;
      film_mean[3 * i + 1] = img.pixels[i].g;
      film_mean[3 * i + 2] = img.pixels[i].b;
    }
    if (radius && !res.reports.empty()) {
      const auto& r = res.reports.back().radius;
      for (std::size_t i = 0; i < r.size(); ++i) radius[i] = r[i];
    }
  } catch (const std::exception&) {
    return 1;
  }
  return 0;
}

int ref_render_fppm(void* sp, const double* cam9, double vfov, int w, int h, uint64_t seed, uint64_t iterations,
                    uint32_t max_depth, uint64_t light_paths, double r0_frac, int na, int ns, double alpha_f,
                    int threads, double* film_mean, double* radius, double* seconds) {
  return render_algo(Algorithm::fppm, sp, cam9, vfov, w, h, seed, iterations, max_depth, light_paths, r0_frac, na,
                     ns, alpha_f, threads, film_mean, radius, seconds);
}

// The same with Algorithm::vcm_plus (bidirectional, tested per-pixel radii).
int ref_render_vcm_plus(void* sp, const double* cam9, double vfov, int w, int h, uint64_t seed,
                        uint64_t iterations, uint32_t max_depth, uint64_t light_paths, double r0_frac, int na,
                        int ns, double alpha_f, int threads, double* film_mean, double* radius, double* seconds) {
  return render_algo(Algorithm::vcm_plus, sp, cam9, vfov, w, h, seed, iterations, max_depth, light_paths, r0_frac,
                     na, ns, alpha_f, threads, film_mean, radius, seconds);
}


// ---- formats and film outputs (film.cpp, scene_parse.cpp): the reference's
// own functions for the host-side format tests (tests/test_formats.py)
long ref_serialize_scene(const char* text, char* out, size_t cap) {
  try {
    const Scene sc = parse_scene(text, "", "<scene>");
    const std::string s = serialize_scene(sc);
    if (out && cap) {
      std::strncpy(out, s.c_str(), cap - 1);
      out[cap - 1] = 0;
    }
    return static_cast<long>(s.size());
  } catch (const std::exception&) {
    return -1;
  }
}

static std::vector<ConvergenceRow> conv_rows(size_t n, const uint64_t* it, const double* sec, const double* m,
                                             const double* rad, const double* vms) {
  std::vector<ConvergenceRow> rows(n);
  for (size_t i = 0; i < n; ++i) rows[i] = ConvergenceRow{it[i], sec[i], m[i], rad[i], vms[i]};
  return rows;
}

int ref_write_convergence_csv(const char* path, size_t n, const uint64_t* it, const double* sec, const double* m,
                              const double* rad, const double* vms) {
  try {
    write_convergence_csv(path, conv_rows(n, it, sec, m, rad, vms));
  } catch (const std::exception&) {
    return 1;
  }
  return 0;
}

// rows read (<= cap) or -1 with the message in err
long ref_read_convergence_csv(const char* path, size_t cap, uint64_t* it, double* sec, double* m, double* rad,
                              double* vms, char* err, size_t errcap) {
  try {
    const auto rows = read_convergence_csv(path);
    for (size_t i = 0; i < rows.size() && i < cap; ++i) {
      it[i] = rows[i].iteration; sec[i] = rows[i].seconds; m[i] = rows[i].mse;
      rad[i] = rows[i].mean_radius; vms[i] = rows[i].vm_share;
    }
    return static_cast<long>(rows.size());
  } catch (const std::exception& e) {
    if (err && errcap) {
      std::strncpy(err, e.what(), errcap - 1);
      err[errcap - 1] = 0;
    }
    return -1;
  }
}

static Image make_image(int w, int h, const double* rgb) {
  Image img{w, h, {}};
  img.pixels.resize(static_cast<size_t>(w) * h);
  for (size_t i = 0; i < img.pixels.size(); ++i) img.pixels[i] = Rgb{rgb[3 * i], rgb[3 * i + 1], rgb[3 * i + 2]};
  return img;
}

static void put_image(const Image& img, double* rgb) {
  for (size_t i = 0; i < img.pixels.size(); ++i) {
    rgb[3 * i] = img.pixels[i].r; rgb[3 * i + 1] = img.pixels[i].g; rgb[3 * i + 2] = img.pixels[i].b;
  }
}

int ref_write_pfm(const char* path, int w, int h, const double* rgb) {
  try {
    write_pfm(path, make_image(w, h, rgb));
  } catch (const std::exception&) {
    return 1;
  }
  return 0;
}

double ref_mse(int w, int h, const double* a, const double* b) { return mse(make_image(w, h, a), make_image(w, h, b)); }

double ref_fit_slope(size_t n, const uint64_t* it, const double* m, uint64_t lo, uint64_t hi, int* err) {
  try {
    *err = 0;
    return fit_convergence_slope(std::span<const uint64_t>(it, n), std::span<const double>(m, n), lo, hi);
  } catch (const std::exception&) {
    *err = 1;
    return 0.0;
  }
}

// A Film holding one iteration `mean`, splits vc / vm and a radius channel:
// its radius / vc-share / vm-share / squared-error images ([npix][3] each).
void ref_film_aux(int w, int h, const double* mean, const double* vc, const double* vm, const double* radius,
                  double r_min, double r_1, const double* ref, double* o_rad, double* o_vcs, double* o_vms,
                  double* o_sq) {
  Film film(w, h);
  const size_t n = static_cast<size_t>(w) * h;
  std::vector<Rgb> est(n);
  for (size_t i = 0; i < n; ++i) est[i] = Rgb{mean[3 * i], mean[3 * i + 1], mean[3 * i + 2]};
  film.add_iteration(est);
  for (size_t i = 0; i < n; ++i) film.add_split(i, vc[i], vm[i]);
  film.set_radius_channel(std::span<const double>(radius, n));
  put_image(film.radius_image(r_min, r_1), o_rad);
  put_image(film.vc_share_image(), o_vcs);
  put_image(film.vm_share_image(), o_vms);
  put_image(film.squared_error_image(make_image(w, h, ref)), o_sq);
}

// render() for any algorithm (0 fppm, 1 vcm_plus, 2 sppm, 3 vcm, 4 cppm) with
// the test override and r_min_base, returning the film mean, the last radii
// and the per-pixel split totals (Film::vc_total / vm_total)
int ref_render_ex(void* sp, int algo, const double* cam9, double vfov, int w, int h, uint64_t seed,
                  uint64_t iterations, uint32_t max_depth, uint64_t light_paths, double r0_frac, int na, int ns,
                  double alpha_f, int override_decision, double r_min_base, int threads, double* film_mean,
                  double* radius, double* vc, double* vm) {
  RefScene* rs = static_cast<RefScene*>(sp);
  Scene scene = rs->scene;
  scene.has_camera = true;
  scene.camera = make_cam(cam9, vfov, w, h);
  IntegratorConfig cfg;
  const Algorithm algos[] = {Algorithm::fppm, Algorithm::vcm_plus, Algorithm::sppm, Algorithm::vcm,
                             Algorithm::cppm};
  cfg.algorithm = algos[algo];
  cfg.iterations = iterations;
  cfg.seed = seed;
  cfg.max_depth = max_depth;
  cfg.threads = threads;
  cfg.r0_frac = r0_frac;
  cfg.light_paths = light_paths;
  cfg.test.n_annuli = na;
  cfg.test.n_sectors = ns;
  cfg.test.alpha_f = alpha_f;
  cfg.test.override_decision = override_decision == 1   ? TestOverride::always_reject
                               : override_decision == 2 ? TestOverride::never_reject
                                                        : TestOverride::none;
  if (r_min_base > 0) cfg.schedule.r_min_base = r_min_base;
  try {
    RenderResult res = render(scene, cfg);
    const Image img = res.film.image();
    for (size_t i = 0; i < img.pixels.size(); ++i) {
      film_mean[3 * i] = img.pixels[i].r;
      film_mean[3 * i + 1] = img.pixels[i].g;
      film_mean[3 * i + 2] = img.pixels[i].b;
      if (vc) vc[i] = res.film.vc_total(i);
      if (vm) vm[i] = res.film.vm_total(i);
    }
    if (radius && !res.reports.empty()) {
      const auto& r = res.reports.back().radius;
      for (size_t i = 0; i < r.size(); ++i) radius[i] = r[i];
    }
  } catch (const std::exception&) {
    return 1;
  }
  return 0;
}

// bounding_radius (scene_geometry.cpp:341-362): the initial radius is
// r0_frac times this (integrator.cpp:121).
double ref_bounding_radius(void* sp) { return bounding_radius(static_cast<RefScene*>(sp)->scene); }

unsigned ref_hardware_threads() { return std::thread::hardware_concurrency(); }

} // extern "C"
