// compat/fppm/gather.hpp -- fppm::GatherRegion and its free functions
// (reference gather.hpp:11-112) re-expressed over the C ABI (fppm_gpu.h).
// A reference-side C++ caller puts include/compat ahead of its own include
// directory and links libfppm_gpu.so.
//
// Each GatherRegion owns a one-region device context: accumulate() bins the
// sample on the device (sector_index with the region's current radius, the
// luminance or RGB channel values), the three end-of-iteration policies run
// the device policy kernel (fppm_gpu_set_policy + fppm_gpu_end_iteration),
// and radius / held_iterations / sector_stats read the device state back.
// A renderer drives many regions through one context instead
// (fppm_gpu::GatherRegionBatch, or the batched hot path fppm_gpu_iterate).
#pragma once

#include <cstdint>
#include <memory>
#include <span>
#include <stdexcept>
#include <vector>

#include "fppm/frame.hpp"
#include "fppm/stat_tests.hpp"
#include "fppm/vec.hpp"
#include "fppm_gpu.hpp"

namespace fppm {

/// gather.hpp:16-20
struct RadiusSchedule {
  double k = 0.7;
  double alpha = 0.75;
  double r_min_base = 0;
};

/// gather.hpp:25 (gather.cpp:9-13): the device and host share one expression.
inline double schedule_radius(double base, double alpha, std::uint64_t i) {
  return fppm_gpu_schedule_radius(base, alpha, i);
}

enum class TestChannels { auto_detect, luminance, rgb };
enum class TestOverride { none, always_reject, never_reject };

struct TestConfig {
  int n_annuli = 2;
  int n_sectors = 6;
  double alpha_f = 0.01;
  double alpha_chi2 = 0.01;
  TestChannels channels = TestChannels::auto_detect;
  TestOverride override_decision = TestOverride::none;
};

struct ContributionSample {
  UnifiedPoint y;
  Rgb value;
};

/// gather.hpp:50-53: throws std::domain_error outside the disk and
/// std::invalid_argument for bin counts < 1.
inline int sector_index(const UnifiedPoint &y, double radius, int n_annuli, int n_sectors) {
  int32_t s = 0;
  fppm_gpu::check(fppm_gpu_sector_index(y.u, y.v, radius, n_annuli, n_sectors, &s));
  return s;
}

struct RadiusUpdate {
  double radius = 0;
  bool tested = false;
  bool rejected = false;
  double statistic = 0;
  double critical = 0;
};

inline TangentFrame build_tangent_frame_gpu_abi(const Normal3 &n) {
  const double nn[3] = {n.x, n.y, n.z};
  double u[3], v[3];
  fppm_gpu::check(fppm_gpu_build_frame(nn, u, v));
  TangentFrame f;
  f.u = Vec3{u[0], u[1], u[2]};
  f.v = Vec3{v[0], v[1], v[2]};
  f.n = n;
  return f;
}

class GatherRegion {
 public:
  GatherRegion(const TestConfig &test, const RadiusSchedule &schedule, double initial_radius)
      : test_(test), schedule_(schedule), initial_radius_(initial_radius),
        n_sectors_total_(test.n_annuli * test.n_sectors),
        channels_(test.channels == TestChannels::rgb ? 3 : 1) {
    fppm_gpu_config c{};
    c.n_annuli = test.n_annuli;
    c.n_sectors = test.n_sectors;
    c.alpha_f = test.alpha_f;
    c.alpha_chi2 = test.alpha_chi2;
    c.channels = channels_ == 3 ? FPPM_CHANNELS_RGB : FPPM_CHANNELS_LUMINANCE;
    c.override_decision = test.override_decision == TestOverride::always_reject ? FPPM_OVERRIDE_ALWAYS_REJECT
                          : test.override_decision == TestOverride::never_reject ? FPPM_OVERRIDE_NEVER_REJECT
                                                                                 : FPPM_OVERRIDE_NONE;
    c.policy = FPPM_POLICY_FTEST;
    c.k = schedule.k;
    c.alpha = schedule.alpha;
    c.r_min_base = schedule.r_min_base;
    c.initial_radius = initial_radius;
    c.samples_per_iteration = 1;
    c.max_depth = 10;
    c.normal_guard_cos = 0.86602540378443865;
    c.max_hitpoints = 1;
    c.max_photons = 1;
    ctx_ = std::make_unique<fppm_gpu::Context>(c);  // invalid_argument per gather.cpp:41-50
    const double zero[3] = {0, 0, 0}, nz[3] = {0, 0, 1}, one[3] = {1, 1, 1};
    const uint32_t depth = 1;
    const fppm_hitpoints hp{zero, nz, nz, one, one, &depth, nullptr};
    ctx_->set_hitpoints(hp, 1);
  }

  /// New gather point for this iteration; keeps the pooled statistics.
  void move_to(const Point3 &center, const Normal3 &normal) {
    center_ = center;
    frame_ = build_tangent_frame_gpu_abi(normal);
  }

  void accumulate(const ContributionSample &sample) {
    const uint32_t region = 0;
    const double y[2] = {sample.y.u, sample.y.v};
    const double v[3] = {sample.value.r, sample.value.g, sample.value.b};
    ctx_->ok(fppm_gpu_accumulate(ctx_->get(), &region, y, v, 1));
  }

  RadiusUpdate end_iteration(std::uint64_t i, std::uint64_t samples_per_iteration) {
    return run(FPPM_POLICY_FTEST, i, samples_per_iteration);
  }
  RadiusUpdate chi2_end_iteration(std::uint64_t i, std::uint64_t samples_per_iteration) {
    return run(FPPM_POLICY_CHI2, i, samples_per_iteration);
  }
  RadiusUpdate schedule_end_iteration(std::uint64_t i) { return run(FPPM_POLICY_SCHEDULE, i, 0); }

  double radius() const {
    double r = 0;
    ctx_->ok(fppm_gpu_get_regions(ctx_->get(), &r, nullptr, nullptr, nullptr, nullptr));
    return r;
  }
  double initial_radius() const { return initial_radius_; }
  std::uint64_t held_iterations() const {
    uint64_t t = 0;
    ctx_->ok(fppm_gpu_get_regions(ctx_->get(), nullptr, &t, nullptr, nullptr, nullptr));
    return t;
  }
  const Point3 &center() const { return center_; }
  const TangentFrame &frame() const { return frame_; }
  int sector_count() const { return n_sectors_total_; }
  int channel_count() const { return channels_; }

  /// The pooled moments of one channel, read back from the device.
  std::span<const SectorStats> sector_stats(int channel) const {
    const size_t n = static_cast<size_t>(channels_) * n_sectors_total_;
    std::vector<uint64_t> cnt(n);
    std::vector<double> sum(n), sq(n);
    ctx_->ok(fppm_gpu_get_regions(ctx_->get(), nullptr, nullptr, cnt.data(), sum.data(), sq.data()));
    stats_.assign(n, SectorStats{});
    for (size_t k = 0; k < n; ++k) {
      stats_[k].count = cnt[k];
      stats_[k].sum = sum[k];
      stats_[k].sum_sq = sq[k];
    }
    return {stats_.data() + static_cast<size_t>(channel) * n_sectors_total_,
            static_cast<size_t>(n_sectors_total_)};
  }

 private:
  RadiusUpdate run(int policy, std::uint64_t i, std::uint64_t J) {
    ctx_->ok(fppm_gpu_set_policy(ctx_->get(), policy));
    if (policy != FPPM_POLICY_SCHEDULE) ctx_->ok(fppm_gpu_set_samples_per_iteration(ctx_->get(), J));
    double radius = 0, stat = 0, crit = 0;
    uint8_t tested = 0, rejected = 0;
    fppm_gpu_iter_out out{};
    out.radius = &radius;
    out.tested = &tested;
    out.rejected = &rejected;
    out.statistic = &stat;
    out.critical = &crit;
    ctx_->ok(fppm_gpu_end_iteration(ctx_->get(), i, &out));
    ctx_->ok(fppm_gpu_synchronize(ctx_->get()));
    RadiusUpdate up;
    up.radius = radius;
    up.tested = tested != 0;
    up.rejected = rejected != 0;
    up.statistic = stat;
    up.critical = crit;
    return up;
  }

  TestConfig test_;
  RadiusSchedule schedule_;
  double initial_radius_;
  int n_sectors_total_;
  int channels_;
  Point3 center_{};
  TangentFrame frame_{};
  std::unique_ptr<fppm_gpu::Context> ctx_;
  mutable std::vector<SectorStats> stats_;
};

}  // namespace fppm
