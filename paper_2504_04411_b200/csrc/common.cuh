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
  uint32_t S;      // fine cells per reference cell and axis (power of two; 1 = reference cells)
  uint32_t shift;  // log2(S)
  uint32_t lean;   // 1: lean planar records (rec0 = x, y, z, meta; rec1 = L, b; rec2 = r, g; fp64 pairs)
                   // 2: flat lean records, 32 B (every photon has z == zflat; flat_record)
  float zflat;     // lean == 2: the photons' common z
  uint32_t pad_;
};
// With S > 1 the dense table indexes FINE cells of size cell / S ("slab"
// layout, used when the photons span few reference cells along z): inv is
// S / cell and ix0.. / nx.. are fine-cell coordinates.  Because S is a power
// of two, floor(x * (S / cell)) = S * floor-part of x * (1 / cell) exactly, so
// the reference cell of a fine cell is its coordinate >> shift.

// Sorted photon record, 4 x 16 B vectors (SoA of float4).
// Layout used by the fine gather (gather_fine.cu):
//   rec0 = (x, y, z, depth bits), rec1 = (n.z, wi.z, lum(pow) as fp64 lo/hi),
//   rec2 = (pow.r, pow.g, pow.b, flags), rec3 = (n.x, n.y, wi.x, wi.y)
//   flags bit0: n.x, n.y, wi.x, wi.y all finite (planar-shortcut exactness)
// Lean layout (GridHeader::lean; slab grids whose gathered hit points are all
// planar and gray, C = 1, n_a <= 2, n_s = 4; gather_fine.cu lean path):
//   rec0 = (x, y, z, meta), rec1 = (lum(pow), pow.b), rec2 = (pow.r, pow.g)
//   in fp64; no rec3 (lean_record)
// Layout used by the tile / warp / lanes kernels:
//   rec0 = (x, y, z, depth bits)     -- the only vector read per candidate
//   rec1 = (nx, ny, nz, wi.x)
//   rec2 = (wi.y, wi.z, pow.r, pow.g)
//   rec3 = (pow.b, 0, lum(pow) as fp64 lo/hi words)
struct PhotonRecs {
  float4 *rec0, *rec1, *rec2, *rec3;
  float4 *pack;  // fine layout: 64-B records in input order (permutation source)
};

// One input photon (fppm_photons SoA fields).
struct PhotonIn {
  float p[3], n[3], w[3], c[3];
  uint32_t d;
};
__device__ __forceinline__ PhotonIn load_photon(const float *__restrict__ pos, const float *__restrict__ nrm,
                                                const float *__restrict__ wi, const float *__restrict__ pw,
                                                const uint32_t *__restrict__ depth, size_t j) {
  PhotonIn P;
  const size_t o = 3 * j;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    P.p[a] = pos[o + a];
    P.n[a] = nrm[o + a];
    P.w[a] = wi[o + a];
    P.c[a] = pw[o + a];
  }
  P.d = depth[j];
  return P;
}
// Photons j .. j + 3 (j % 4 == 0, 16-B aligned arrays) with 16-B loads:
// three per float[3] array, one for the depths.
__device__ __forceinline__ void load_photons4(const float *__restrict__ pos, const float *__restrict__ nrm,
                                              const float *__restrict__ wi, const float *__restrict__ pw,
                                              const uint32_t *__restrict__ depth, size_t j, PhotonIn (&P)[4]) {
  const float *src[4] = {pos, nrm, wi, pw};
#pragma unroll
  for (int f = 0; f < 4; ++f) {
    const float4 *q = reinterpret_cast<const float4 *>(src[f] + 3 * j);
    const float4 a = __ldcs(q), b = __ldcs(q + 1), c = __ldcs(q + 2);
    const float v[12] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w, c.x, c.y, c.z, c.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      float *dst = f == 0 ? P[k].p : (f == 1 ? P[k].n : (f == 2 ? P[k].w : P[k].c));
      dst[0] = v[3 * k];
      dst[1] = v[3 * k + 1];
      dst[2] = v[3 * k + 2];
    }
  }
  const uint4 d = __ldcs(reinterpret_cast<const uint4 *>(depth + j));
  P[0].d = d.x; P[1].d = d.y; P[2].d = d.z; P[3].d = d.w;
}

// Fine-layout records packed in input order (coalesced reads of the SoA input
// and 64-B contiguous writes); the permutation then moves whole 64-B records.
__device__ __forceinline__ void fine_record(const PhotonIn &P, float4 &q0, float4 &q1, float4 &q2, float4 &q3) {
  const float nx = P.n[0], ny = P.n[1], wx = P.w[0], wy = P.w[1];
  const double L = elum((double)P.c[0], (double)P.c[1], (double)P.c[2]);
  const unsigned long long Lb = (unsigned long long)__double_as_longlong(L);
  const uint32_t flags =
      (fabsf(nx) < INFINITY && fabsf(ny) < INFINITY && fabsf(wx) < INFINITY && fabsf(wy) < INFINITY) ? 1u
                                                                                                     : 0u;
  q0 = make_float4(P.p[0], P.p[1], P.p[2], __uint_as_float(P.d));
  q1 = make_float4(P.n[2], P.w[2], __uint_as_float((uint32_t)Lb), __uint_as_float((uint32_t)(Lb >> 32)));
  q2 = make_float4(P.c[0], P.c[1], P.c[2], __uint_as_float(flags));
  q3 = make_float4(nx, ny, wx, wy);
}
__device__ __forceinline__ void fine_record(const float *__restrict__ pos, const float *__restrict__ nrm,
                                            const float *__restrict__ wi, const float *__restrict__ pw,
                                            const uint32_t *__restrict__ depth, size_t j, float4 &q0,
                                            float4 &q1, float4 &q2, float4 &q3) {
  fine_record(load_photon(pos, nrm, wi, pw, depth, j), q0, q1, q2, q3);
}

// Lean record (GridHeader::lean): 48 B with the photon-only parts of the
// planar predicates folded in.  Against a hit normal n = +z the guard and
// cos_i dots are n.z and wi.z exactly when n.x, n.y, wi.x, wi.y are finite
// (frame.cpp:5-14, integrator.cpp:397, bsdf.cpp:56-58), so:
//   meta = depth << 8 | guard_fail << 31: eye + depth <= max_depth and the
//          guard in one unsigned compare against the hit point's limit
//          (< 2^31); depth < 2^23;
//   cos_i <= 0: the pair is counted with value 0 (f = 0) -> L = r = g = b = 0;
//   a non-finite n.x/n.y/wi.x/wi.y or power, or depth >= 2^23: x = NaN, meta = 0, which
//          lands every pair with the photon in the exact fp64 path (it reads
//          the input photon, not this record).
__device__ __forceinline__ void lean_record(const PhotonIn &P, double guard, float4 &q0, float4 &q1, float4 &q2) {
  const float nx = P.n[0], ny = P.n[1], wx = P.w[0], wy = P.w[1];
  const uint32_t d = P.d;
  double r = (double)P.c[0], g = (double)P.c[1], b = (double)P.c[2];
  double L = elum(r, g, b);
  const bool exact = !(fabsf(nx) < INFINITY && fabsf(ny) < INFINITY && fabsf(wx) < INFINITY &&
                       fabsf(wy) < INFINITY) || d >= (1u << 23) || !(fabs(L) < INFINITY) ||
                     !(fabs(r) < INFINITY && fabs(g) < INFINITY && fabs(b) < INFINITY);
  const bool guard_fail = (double)P.n[2] < guard;
  const bool cos_pos = !(P.w[2] <= 0.0f);
  if (!cos_pos) r = g = b = L = 0.0;
  const uint32_t meta = exact ? 0u : ((d << 8) | (guard_fail ? 0x80000000u : 0u));
  q0 = make_float4(exact ? __int_as_float(0x7fffffff) : P.p[0], P.p[1], P.p[2], __uint_as_float(meta));
  q1 = make_float4(__uint_as_float((uint32_t)__double_as_longlong(L)),
                   __uint_as_float((uint32_t)((unsigned long long)__double_as_longlong(L) >> 32)),
                   __uint_as_float((uint32_t)__double_as_longlong(b)),
                   __uint_as_float((uint32_t)((unsigned long long)__double_as_longlong(b) >> 32)));
  q2 = make_float4(__uint_as_float((uint32_t)__double_as_longlong(r)),
                   __uint_as_float((uint32_t)((unsigned long long)__double_as_longlong(r) >> 32)),
                   __uint_as_float((uint32_t)__double_as_longlong(g)),
                   __uint_as_float((uint32_t)((unsigned long long)__double_as_longlong(g) >> 32)));
}
__device__ __forceinline__ void lean_record(const float *__restrict__ pos, const float *__restrict__ nrm,
                                            const float *__restrict__ wi, const float *__restrict__ pw,
                                            const uint32_t *__restrict__ depth, size_t j, double guard, float4 &q0,
                                            float4 &q1, float4 &q2) {
  lean_record(load_photon(pos, nrm, wi, pw, depth, j), guard, q0, q1, q2);
}

// Flat lean record (GridHeader::lean == 2): the lean record of a frame whose
// photons all share one z (bit-identical fp32, k_cell_bounds): z leaves the
// record (the ball's dz is a per-hit-point constant) and the power stays in
// the ABI's fp32, widened exactly in the gather:
//   rec0 = (x, y, meta, pow.r), rec1 = (lum(pow) as fp64 lo/hi, pow.g, pow.b)
// with meta, the cos_i zeroing and the exact flag (x = NaN) of lean_record.
__device__ __forceinline__ void flat_record(const PhotonIn &P, double guard, float4 &q0, float4 &q1) {
  const float nx = P.n[0], ny = P.n[1], wx = P.w[0], wy = P.w[1];
  const uint32_t d = P.d;
  float r = P.c[0], g = P.c[1], b = P.c[2];
  double L = elum((double)r, (double)g, (double)b);
  const bool exact = !(fabsf(nx) < INFINITY && fabsf(ny) < INFINITY && fabsf(wx) < INFINITY &&
                       fabsf(wy) < INFINITY) || d >= (1u << 23) || !(fabs(L) < INFINITY) ||
                     !(fabsf(r) < INFINITY && fabsf(g) < INFINITY && fabsf(b) < INFINITY);
  const bool guard_fail = (double)P.n[2] < guard;
  const bool cos_pos = !(P.w[2] <= 0.0f);
  if (!cos_pos) {
    r = g = b = 0.0f;
    L = 0.0;
  }
  const uint32_t meta = exact ? 0u : ((d << 8) | (guard_fail ? 0x80000000u : 0u));
  q0 = make_float4(exact ? __int_as_float(0x7fffffff) : P.p[0], P.p[1], __uint_as_float(meta), r);
  q1 = make_float4(__uint_as_float((uint32_t)__double_as_longlong(L)),
                   __uint_as_float((uint32_t)((unsigned long long)__double_as_longlong(L) >> 32)), g, b);
}

// exclusive scan of one value per thread over a 256-thread block; returns the
// block total through *total.
__device__ __forceinline__ uint32_t block_exclusive_scan_256(uint32_t v, uint32_t *s_warp,
                                                             uint32_t *total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(kFull, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_warp[warp] = x;
  __syncthreads();
  if (warp == 0) {
    uint32_t w = lane < 8 ? s_warp[lane] : 0u;
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, w, o);
      if (lane >= o) w += y;
    }
    if (lane < 8) s_warp[lane] = w;  // inclusive warp totals
  }
  __syncthreads();
  const uint32_t before = warp == 0 ? 0u : s_warp[warp - 1];
  *total = s_warp[7];
  __syncthreads();
  return before + x - v;
}

// ---------------------------------------------------------------------------
// TMA 1D bulk copies (cp.async.bulk, SASS UBLKCP) completing on an mbarrier.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// L2 prefetch of a global range (bytes: multiple of 16), no completion tracking
__device__ __forceinline__ void bulk_prefetch_l2(const void *src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

}  // namespace fppm_b200

#define FPPM_CUDA_OK(expr)                                                \
  do {                                                                      \
    cudaError_t _e = (expr);                                                \
    if (_e != cudaSuccess) return ::fppm_b200::cuda_fail(ctx, _e, #expr);  \
  } while (0)
