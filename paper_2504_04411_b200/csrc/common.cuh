// common.cuh -- shared device/host definitions for the B200 gather + F-test path.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "fppm_gpu.h"

namespace fppm_b200 {

constexpr int kWarp = 32;
constexpr unsigned kFull = 0xffffffffu;
constexpr double kPi = 3.141592653589793;      // std::numbers::pi
constexpr double kInvPi = 0.3183098861837907;  // std::numbers::inv_pi
constexpr double kTwoPi = 2.0 * 3.141592653589793;  // sampling.hpp:11

// ---------------------------------------------------------------------------
// IEEE fp64 helpers that the compiler may not contract into FMA.  Every
// predicate that decides membership or a sector is evaluated with these so it
// reproduces the reference's x86-64 (no-FMA) fp64 arithmetic bit for bit.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double dm(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double da(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double ds(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dd(double a, double b) { return __ddiv_rn(a, b); }

// vec.hpp:463 dot: (a.x*b.x + a.y*b.y) + a.z*b.z
__device__ __forceinline__ double edot(double ax, double ay, double az, double bx,
                                       double by, double bz) {
  return da(da(dm(ax, bx), dm(ay, by)), dm(az, bz));
}

// frame.cpp:5-14 (Duff et al. branchless basis), evaluated without FMA.
__device__ __forceinline__ void eframe(double nx, double ny, double nz, double3 &u,
                                       double3 &v) {
  const double sign = copysign(1.0, nz);
  const double a = dd(-1.0, da(sign, nz));
  const double b = dm(dm(nx, ny), a);
  u = make_double3(da(1.0, dm(dm(dm(sign, nx), nx), a)), dm(sign, b), dm(-sign, nx));
  v = make_double3(b, da(sign, dm(dm(ny, ny), a)), -ny);
}

// vec.hpp:79-81 luminance: (0.2126 r + 0.7152 g) + 0.0722 b
__device__ __forceinline__ double elum(double r, double g, double b) {
  return da(da(dm(0.2126, r), dm(0.7152, g)), dm(0.0722, b));
}

// ---------------------------------------------------------------------------
// Grid header (device resident; also mirrored on the host after each build).
// Dense cell id = ((ix - ix0) * ny + (iy - iy0)) * nz + (iz - iz0), which
// preserves the reference's key order (photon_map.cpp:19-24: x major, z minor).
// ---------------------------------------------------------------------------
struct GridHeader {
  double cell;     // cell size (photon_map.cpp:26)
  double inv;      // 1 / cell (photon_map.cpp:29)
  long long ix0, iy0, iz0;
  long long nx, ny, nz;
  unsigned long long ncells;
  uint32_t key_bits;
  uint32_t n;      // photons in the grid
  uint32_t ok;     // 1 when dims fit the dense table
  uint32_t pad;
};

// Sorted photon record, 4 x 16 B vectors (SoA of float4):
//   rec0 = (x, y, z, depth bits)     -- the only vector read per candidate
//   rec1 = (nx, ny, nz, wi.x)
//   rec2 = (wi.y, wi.z, pow.r, pow.g)
//   rec3 = (pow.b, 0, 0, 0)
struct PhotonRecs {
  float4 *rec0, *rec1, *rec2, *rec3;
};

}  // namespace fppm_b200

#define FPPM_CUDA_OK(expr)                                                  \
  do {                                                                      \
    cudaError_t _e = (expr);                                                \
    if (_e != cudaSuccess) return ::fppm_b200::cuda_fail(ctx, _e, #expr);  \
  } while (0)
