// compat/fppm/photon_map.hpp -- fppm::PhotonGrid (reference photon_map.hpp:15-42)
// re-expressed over the C ABI (fppm_gpu.h): a reference-side C++ caller puts
// include/compat ahead of its own include directory and links libfppm_gpu.so;
// the rest of its tree (vec.hpp, path.hpp, ...) is unchanged.
//
// One device context per grid.  Light vertices are handed to the device as
// canonical fp32 photons (fppm_gpu.h, fppm_photons); query results are vertex
// indices in the reference's visit order (cells in the fixed 27-cell order,
// vertices in insertion order inside a cell), so ordered comparisons against
// the reference hold.  Exceptions follow photon_map.cpp:29 and :58.
#pragma once

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <utility>
#include <vector>

#include "fppm/path.hpp"
#include "fppm/vec.hpp"
#include "fppm_gpu.hpp"

namespace fppm {

class PhotonGrid {
 public:
  PhotonGrid() = default;
  PhotonGrid(std::vector<LightVertex> vertices, double cell_size)
      : vertices_(std::move(vertices)), cell_size_(cell_size) {
    if (!(cell_size > 0)) throw std::invalid_argument("PhotonGrid: cell size must be positive");
    const uint32_t n = static_cast<uint32_t>(vertices_.size());
    ctx_ = std::make_shared<fppm_gpu::Context>(config(n));
    std::vector<float> pos(3 * (size_t)n), nrm(3 * (size_t)n), wi(3 * (size_t)n), pw(3 * (size_t)n);
    std::vector<uint32_t> depth(n);
    for (uint32_t i = 0; i < n; ++i) {
      const LightVertex &v = vertices_[i];
      const double p[3] = {v.position.x, v.position.y, v.position.z};
      const double s[3] = {v.shading_normal.x, v.shading_normal.y, v.shading_normal.z};
      const double w[3] = {v.wi.x, v.wi.y, v.wi.z};
      const double t[3] = {v.throughput.r, v.throughput.g, v.throughput.b};
      for (int c = 0; c < 3; ++c) {
        pos[3 * (size_t)i + c] = static_cast<float>(p[c]);
        nrm[3 * (size_t)i + c] = static_cast<float>(s[c]);
        wi[3 * (size_t)i + c] = static_cast<float>(w[c]);
        pw[3 * (size_t)i + c] = static_cast<float>(t[c]);
      }
      depth[i] = v.depth;
    }
    const fppm_photons ph{pos.data(), nrm.data(), wi.data(), pw.data(), depth.data()};
    ctx_->set_photons(ph, n);
    ctx_->build_grid(cell_size);
  }

  std::size_t size() const { return vertices_.size(); }
  const std::vector<LightVertex> &vertices() const { return vertices_; }
  double cell_size() const { return cell_size_; }

  /// Indices of stored vertices with |pos - center| <= r (closed ball).
  void query_ball(const Point3 &center, double r, std::vector<std::uint32_t> &out) const {
    if (r > cell_size_) throw std::invalid_argument("PhotonGrid: query radius exceeds cell size");
    out.clear();
    if (!ctx_) return;
    const double c[3] = {center.x, center.y, center.z};
    uint64_t offsets[2] = {0, 0}, total = 0;
    ctx_->ok(fppm_gpu_query_ball(ctx_->get(), c, &r, 1, offsets, nullptr, 0, &total));
    out.assign(total, 0u);
    if (total) ctx_->ok(fppm_gpu_query_ball(ctx_->get(), c, &r, 1, offsets, out.data(), total, &total));
  }

 private:
  static fppm_gpu_config config(uint32_t n) {
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
    return c;
  }

  std::vector<LightVertex> vertices_;
  double cell_size_ = 0.0;
  std::shared_ptr<fppm_gpu::Context> ctx_;  // copies share the device grid (immutable)
};

}  // namespace fppm
