// C++ drop-in check of include/fppm_gpu.hpp against the reference's own unit
// test expectations (proj/tests/test_photon_map.cpp, test_gather.cpp), with
// the reference's exception classes.  Built and run by tests/test_cpp_wrapper.py.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <random>
#include <stdexcept>

#include "fppm_gpu.hpp"

#define REQUIRE(c)                                                  \
  do {                                                              \
    if (!(c)) {                                                     \
      std::fprintf(stderr, "FAILED %s:%d: %s\n", __FILE__, __LINE__, #c); \
      return 1;                                                     \
    }                                                               \
  } while (0)

template <class E, class F>
static bool throws(F f) {
  try {
    f();
  } catch (const E &) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

int main() {
  // ---- PhotonGrid: brute force agreement, closed ball, r > cell throws
  std::mt19937 rng(7);
  std::uniform_real_distribution<float> U(-1.f, 1.f);
  std::vector<std::array<float, 3>> pos(2500);
  for (auto &p : pos) p = {U(rng), U(rng), U(rng)};
  const double cell = 0.3;
  fppm_gpu::PhotonGrid grid(pos, cell);
  REQUIRE(grid.size() == pos.size());
  std::vector<uint32_t> out;
  for (int q = 0; q < 200; ++q) {
    const std::array<double, 3> c = {U(rng) * 1.2, U(rng) * 1.2, U(rng) * 1.2};
    const double r = cell * std::fabs(U(rng));
    grid.query_ball(c, r, out);
    std::vector<uint32_t> want;
    for (uint32_t i = 0; i < pos.size(); ++i) {
      const double dx = (double)pos[i][0] - c[0], dy = (double)pos[i][1] - c[1],
                   dz = (double)pos[i][2] - c[2];
      if (dx * dx + dy * dy + dz * dz <= r * r) want.push_back(i);
    }
    std::vector<uint32_t> got = out;
    std::sort(got.begin(), got.end());
    REQUIRE(got == want);
  }
  REQUIRE(throws<std::invalid_argument>([&] { grid.query_ball({0, 0, 0}, cell * 1.5, out); }));
  REQUIRE(throws<std::invalid_argument>([&] { fppm_gpu::PhotonGrid bad(pos, 0.0); }));

  // ---- GatherRegionBatch: hold keeps stats / reject clears (test_gather.cpp:66-96)
  fppm_gpu::TestConfig hold;
  hold.override_decision = FPPM_OVERRIDE_NEVER_REJECT;
  fppm_gpu::RadiusSchedule sched{0.7, 0.75, 0.001};
  fppm_gpu::GatherRegionBatch holder(hold, sched, 1.0, 1, 10);
  holder.accumulate({0u}, {0.1, 0.2}, {2.0, 2.0, 2.0});
  holder.end_iteration(1, 10);
  REQUIRE(holder.radius()[0] == 1.0);
  REQUIRE(holder.held_iterations()[0] == 2);
  fppm_gpu::TestConfig shrink;
  shrink.override_decision = FPPM_OVERRIDE_ALWAYS_REJECT;
  fppm_gpu::GatherRegionBatch shrinker(shrink, sched, 1.0, 1, 10);
  shrinker.end_iteration(1, 10);
  REQUIRE(std::fabs(shrinker.radius()[0] - 0.7) < 1e-15);
  REQUIRE(shrinker.held_iterations()[0] == 1);
  // sector_index domain error outside the disk (gather.cpp:20-21)
  REQUIRE(throws<std::domain_error>([&] { holder.accumulate({0u}, {1.1, 0.0}, {1, 1, 1}); }));
  // constructor validation (test_gather.cpp:259-268)
  REQUIRE(throws<std::invalid_argument>(
      [&] { fppm_gpu::GatherRegionBatch b(fppm_gpu::TestConfig{}, {0.7, 0.75, 2.0}, 1.0, 1, 10); }));
  REQUIRE(throws<std::invalid_argument>(
      [&] { fppm_gpu::GatherRegionBatch b(fppm_gpu::TestConfig{}, {1.5, 0.75, 0.001}, 1.0, 1, 10); }));
  REQUIRE(throws<std::invalid_argument>(
      [&] { fppm_gpu::GatherRegionBatch b(fppm_gpu::TestConfig{}, {0.7, 0.3, 0.001}, 1.0, 1, 10); }));
  REQUIRE(throws<std::invalid_argument>(
      [&] { fppm_gpu::GatherRegionBatch b(fppm_gpu::TestConfig{}, sched, 0.0, 1, 10); }));
  std::printf("wrapper_check OK\n");
  return 0;
}
