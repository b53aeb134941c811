// fppm_gpu.hpp -- header-only C++ view of the C ABI (fppm_gpu.h) shaped like
// the reference's in-process interface, so reference-side C++ callers and the
// reference's own unit tests can switch to the GPU path:
//
//   fppm::PhotonGrid  (photon_map.hpp:15-42)  -> fppm_gpu::PhotonGrid
//   fppm::GatherRegion (gather.hpp:69-112)    -> fppm_gpu::GatherRegionBatch
//                                               (N regions in one device context)
//   Renderer::pixel_pm gather block           -> fppm_gpu::Context::iterate
//
// Status codes are rethrown as the reference's exception classes:
// FPPM_ERR_INVALID_ARGUMENT -> std::invalid_argument, FPPM_ERR_DOMAIN ->
// std::domain_error, everything else -> std::runtime_error.
#ifndef FPPM_GPU_HPP
#define FPPM_GPU_HPP

#include <array>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "fppm_gpu.h"

namespace fppm_gpu {

inline void check(int status, const fppm_gpu_ctx *ctx = nullptr) {
  if (status == FPPM_OK) return;
  std::string msg = fppm_gpu_status_string(status);
  if (ctx) {
    const char *e = fppm_gpu_last_error(ctx);
    if (e && *e) msg += std::string(": ") + e;
  }
  if (status == FPPM_ERR_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  if (status == FPPM_ERR_DOMAIN) throw std::domain_error(msg);
  throw std::runtime_error(msg);
}

// TestConfig (gather.hpp:34-41) + RadiusSchedule (gather.hpp:16-20).
struct TestConfig {
  int n_annuli = 2, n_sectors = 6;
  double alpha_f = 0.01, alpha_chi2 = 0.01;
  int channels = FPPM_CHANNELS_LUMINANCE;
  int override_decision = FPPM_OVERRIDE_NONE;
};
struct RadiusSchedule {
  double k = 0.7, alpha = 0.75, r_min_base = 0.0;
};

// RAII owner of one device context.
class Context {
 public:
  explicit Context(const fppm_gpu_config &cfg) { check(fppm_gpu_create(&cfg, &ctx_)); }
  Context(const Context &) = delete;
  Context &operator=(const Context &) = delete;
  Context(Context &&o) noexcept : ctx_(std::exchange(o.ctx_, nullptr)) {}
  ~Context() {
    if (ctx_) fppm_gpu_destroy(ctx_);
  }
  fppm_gpu_ctx *get() const { return ctx_; }
  void ok(int status) const { check(status, ctx_); }

  void set_hitpoints(const fppm_hitpoints &hp, uint32_t n) { ok(fppm_gpu_set_hitpoints(ctx_, &hp, n)); }
  void set_photons(const fppm_photons &ph, uint32_t n) { ok(fppm_gpu_set_photons(ctx_, &ph, n)); }
  void build_grid(double cell_size) { ok(fppm_gpu_build_grid(ctx_, cell_size)); }
  fppm_gpu_summary iterate(uint64_t i, fppm_gpu_iter_out *out = nullptr) {
    fppm_gpu_summary s{};
    ok(fppm_gpu_iterate(ctx_, i, out, &s));
    return s;
  }
  // (summary != NULL synchronizes, so `out` is complete on return)
  fppm_gpu_summary gather_test(uint64_t i, fppm_gpu_iter_out *out = nullptr) {
    fppm_gpu_summary s{};
    ok(fppm_gpu_gather_test(ctx_, i, out, &s));
    return s;
  }
  double max_radius() {
    double r = 0;
    ok(fppm_gpu_max_radius(ctx_, &r));
    return r;
  }

 private:
  fppm_gpu_ctx *ctx_ = nullptr;
};

// PhotonGrid(std::vector<LightVertex>, double cell) + query_ball (photon_map.hpp:18-27).
// Positions are the canonical fp32 photon positions; query results are indices
// into the constructor's vertex order, in the reference's visit order.
class PhotonGrid {
 public:
  PhotonGrid(const std::vector<std::array<float, 3>> &positions, double cell_size, int device = 0)
      : n_(static_cast<uint32_t>(positions.size())), cell_(cell_size), ctx_(config(n_, device)) {
    if (!(cell_size > 0)) throw std::invalid_argument("PhotonGrid requires a positive cell size");
    std::vector<float> pos(3 * (size_t)n_), nrm(3 * (size_t)n_, 0.f), pw(3 * (size_t)n_, 0.f);
    std::vector<uint32_t> depth(n_, 1u);
    for (uint32_t i = 0; i < n_; ++i)
      for (int c = 0; c < 3; ++c) pos[3 * (size_t)i + c] = positions[i][c];
    for (uint32_t i = 0; i < n_; ++i) nrm[3 * (size_t)i + 2] = 1.f;
    fppm_photons ph{pos.data(), nrm.data(), nrm.data(), pw.data(), depth.data()};
    ctx_.set_photons(ph, n_);
    ctx_.build_grid(cell_size);
  }
  std::size_t size() const { return n_; }
  double cell_size() const { return cell_; }
  void query_ball(const std::array<double, 3> &c, double r, std::vector<uint32_t> &out) const {
    uint64_t offsets[2] = {0, 0}, total = 0;
    ctx_.ok(fppm_gpu_query_ball(ctx_.get(), c.data(), &r, 1, offsets, nullptr, 0, &total));
    out.assign(total, 0u);
    if (total)
      ctx_.ok(fppm_gpu_query_ball(ctx_.get(), c.data(), &r, 1, offsets, out.data(), total, &total));
  }

 private:
  static fppm_gpu_config config(uint32_t n, int device) {
    fppm_gpu_config c{};
    c.n_annuli = 2;
    c.n_sectors = 6;
    c.alpha_f = c.alpha_chi2 = 0.01;
    c.channels = FPPM_CHANNELS_LUMINANCE;
    c.k = 0.7;
    c.alpha = 0.75;
    c.r_min_base = 1.0;
    c.initial_radius = 1.0;
    c.samples_per_iteration = 1;
    c.max_depth = 10;
    c.normal_guard_cos = 0.86602540378443865;
    c.max_hitpoints = 1;
    c.max_photons = n ? n : 1;
    c.device = device;
    return c;
  }
  uint32_t n_;
  double cell_;
  mutable Context ctx_;
};

// `count` GatherRegion objects (same TestConfig / RadiusSchedule / r_1) on one GPU.
class GatherRegionBatch {
 public:
  GatherRegionBatch(const TestConfig &test, const RadiusSchedule &sched, double initial_radius,
                    uint32_t count, uint64_t samples_per_iteration,
                    int policy = FPPM_POLICY_FTEST, int device = 0)
      : count_(count), G_(test.n_annuli * test.n_sectors),
        C_(test.channels == FPPM_CHANNELS_RGB ? 3 : 1),
        ctx_(config(test, sched, initial_radius, count, samples_per_iteration, policy, device)) {
    std::vector<double> z(3 * (size_t)count, 0.0), n(3 * (size_t)count, 0.0),
        one(3 * (size_t)count, 1.0);
    std::vector<uint32_t> eye(count, 1u);
    for (uint32_t i = 0; i < count; ++i) n[3 * (size_t)i + 2] = 1.0;
    fppm_hitpoints hp{z.data(), n.data(), n.data(), one.data(), one.data(), eye.data(), nullptr};
    ctx_.set_hitpoints(hp, count);
  }
  // GatherRegion::accumulate (gather.cpp:59-67) for a batch of samples.
  void accumulate(const std::vector<uint32_t> &region, const std::vector<double> &y_uv,
                  const std::vector<double> &rgb) {
    ctx_.ok(fppm_gpu_accumulate(ctx_.get(), region.data(), y_uv.data(), rgb.data(),
                                static_cast<uint32_t>(region.size())));
  }
  // end_iteration / chi2_end_iteration / schedule_end_iteration per `policy`.
  void end_iteration(uint64_t i, uint64_t samples_per_iteration, fppm_gpu_iter_out *out = nullptr) {
    ctx_.ok(fppm_gpu_set_samples_per_iteration(ctx_.get(), samples_per_iteration));
    ctx_.ok(fppm_gpu_end_iteration(ctx_.get(), i, out));
    if (out) ctx_.ok(fppm_gpu_synchronize(ctx_.get()));
  }
  std::vector<double> radius() const {
    std::vector<double> r(count_);
    ctx_.ok(fppm_gpu_get_regions(ctx_.get(), r.data(), nullptr, nullptr, nullptr, nullptr));
    return r;
  }
  std::vector<uint64_t> held_iterations() const {
    std::vector<uint64_t> t(count_);
    ctx_.ok(fppm_gpu_get_regions(ctx_.get(), nullptr, t.data(), nullptr, nullptr, nullptr));
    return t;
  }
  int sector_count() const { return G_; }
  int channel_count() const { return C_; }

 private:
  static fppm_gpu_config config(const TestConfig &t, const RadiusSchedule &s, double r1,
                                uint32_t count, uint64_t J, int policy, int device) {
    fppm_gpu_config c{};
    c.n_annuli = t.n_annuli;
    c.n_sectors = t.n_sectors;
    c.alpha_f = t.alpha_f;
    c.alpha_chi2 = t.alpha_chi2;
    c.channels = t.channels;
    c.override_decision = t.override_decision;
    c.policy = policy;
    c.k = s.k;
    c.alpha = s.alpha;
    c.r_min_base = s.r_min_base;
    c.initial_radius = r1;
    c.samples_per_iteration = J;
    c.max_depth = 10;
    c.normal_guard_cos = 0.86602540378443865;
    c.max_hitpoints = count;
    c.max_photons = 1;
    c.device = device;
    return c;
  }
  uint32_t count_;
  int G_, C_;
  mutable Context ctx_;
};

}  // namespace fppm_gpu

#endif  // FPPM_GPU_HPP
