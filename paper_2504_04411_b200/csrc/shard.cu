// Multi-GPU photon staging (DESIGN.md §7 option A).
//
// Each rank owns a band of hit points and receives every rank's photon share
// in ONE collective (a packed [part][13][stride] 32-bit layout: position,
// shading normal, wi, power, depth).  fppm_gpu_set_photons_packed unpacks it
// into the staging SoA keeping only the photons that can reach this rank's
// hit points: those inside the hit points' bounding box grown by the cell
// size (>= every gather radius, integrator.cpp:159-161).  A photon outside
// that box is farther than r_max from every local hit point, so it is never
// accepted (photon_map.cpp:76) and dropping it changes no result; the kept
// photons stay in global order (parts in rank order, each in input order),
// so the reference's insertion order inside every cell is preserved.
#include "gather.cuh"

namespace fppm_b200 {

constexpr int kPackedFields = 13;

// hit-point bounding box: six doubles (min xyz, max xyz), one block
__global__ void __launch_bounds__(1024) k_hp_box(const double3 *__restrict__ pos, uint32_t n, double *__restrict__ box) {
  double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
    const double3 p = pos[i];
    lo[0] = fmin(lo[0], p.x); hi[0] = fmax(hi[0], p.x);
    lo[1] = fmin(lo[1], p.y); hi[1] = fmax(hi[1], p.y);
    lo[2] = fmin(lo[2], p.z); hi[2] = fmax(hi[2], p.z);
  }
  __shared__ double s[6][32];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    for (int o = 16; o; o >>= 1) {
      lo[a] = fmin(lo[a], __shfl_xor_sync(kFull, lo[a], o));
      hi[a] = fmax(hi[a], __shfl_xor_sync(kFull, hi[a], o));
    }
  }
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0)
    for (int a = 0; a < 3; ++a) { s[a][w] = lo[a]; s[3 + a][w] = hi[a]; }
  __syncthreads();
  if (threadIdx.x < 6) {
    const int nw = (blockDim.x + 31) >> 5;
    double v = s[threadIdx.x][0];
    for (int k = 1; k < nw; ++k) v = threadIdx.x < 3 ? fmin(v, s[threadIdx.x][k]) : fmax(v, s[threadIdx.x][k]);
    box[threadIdx.x] = v;
  }
}

struct PackedParts {
  const uint32_t *data;
  unsigned long long stride;
  uint32_t parts;
  uint32_t off[kMaxPackedParts + 1];  // exclusive prefix of the part counts
};

__device__ __forceinline__ void packed_locate(const PackedParts &P, uint32_t g, uint32_t &p, uint32_t &i) {
  uint32_t lo = 0, hi = P.parts;  // last part with off[p] <= g
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (P.off[mid] <= g) lo = mid; else hi = mid;
  }
  p = lo;
  i = g - P.off[lo];
}

__device__ __forceinline__ uint32_t packed_word(const PackedParts &P, uint32_t p, int f, uint32_t i) {
  return P.data[((unsigned long long)p * kPackedFields + f) * P.stride + i];
}

// keep[g] = photon g lies in the box grown by the margin (all kept without a box)
__global__ void __launch_bounds__(256) k_cull_flags(const PackedParts P, uint32_t total, const double *__restrict__ box,
                                                    const double *__restrict__ margin, uint32_t *__restrict__ keep) {
  double lo[3] = {-INFINITY, -INFINITY, -INFINITY}, hi[3] = {INFINITY, INFINITY, INFINITY};
  if (box) {
    // a relative slack keeps the box conservative under rounding of lo - m
    const double m = *margin;
    for (int a = 0; a < 3; ++a) {
      const double sl = 1e-9 * (fabs(box[a]) + fabs(box[3 + a]) + m) + 1e-300;
      lo[a] = box[a] - m - sl;
      hi[a] = box[3 + a] + m + sl;
    }
  }
  for (uint32_t g = blockIdx.x * blockDim.x + threadIdx.x; g < total; g += gridDim.x * blockDim.x) {
    uint32_t p, i;
    packed_locate(P, g, p, i);
    bool in = true;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const double x = (double)__uint_as_float(packed_word(P, p, a, i));
      in = in && !(x < lo[a]) && !(x > hi[a]);  // NaN positions are kept (the exact path decides)
    }
    keep[g] = in ? 1u : 0u;
  }
}

__global__ void __launch_bounds__(256) k_cull_scatter(const PackedParts P, uint32_t total, const uint32_t *__restrict__ keep,
                                                      const uint32_t *__restrict__ dst, float *__restrict__ pos,
                                                      float *__restrict__ nrm, float *__restrict__ wi,
                                                      float *__restrict__ pw, uint32_t *__restrict__ depth) {
  for (uint32_t g = blockIdx.x * blockDim.x + threadIdx.x; g < total; g += gridDim.x * blockDim.x) {
    if (!keep[g]) continue;
    uint32_t p, i;
    packed_locate(P, g, p, i);
    const size_t o = 3 * (size_t)dst[g];
    float *out[4] = {pos, nrm, wi, pw};
#pragma unroll
    for (int f = 0; f < 12; ++f) out[f / 3][o + f % 3] = __uint_as_float(packed_word(P, p, f, i));
    depth[dst[g]] = packed_word(P, p, 12, i);
  }
}

cudaError_t launch_hp_box(cudaStream_t s, const double3 *pos, uint32_t n, double *box) {
  k_hp_box<<<1, 1024, 0, s>>>(pos, n, box);
  note_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_cull_packed(cudaStream_t s, const uint32_t *data, unsigned long long stride, uint32_t parts,
                               const uint32_t *part_n, const double *box, const double *margin, uint32_t *keep,
                               uint32_t *dst, uint32_t *scan_tmp, float *pos, float *nrm, float *wi, float *pw,
                               uint32_t *depth, int sms) {
  if (parts > (uint32_t)kMaxPackedParts) return cudaErrorInvalidValue;
  PackedParts P;
  P.data = data;
  P.stride = stride;
  P.parts = parts;
  P.off[0] = 0;
  for (uint32_t p = 0; p < parts; ++p) P.off[p + 1] = P.off[p] + part_n[p];
  for (uint32_t p = parts + 1; p <= (uint32_t)kMaxPackedParts; ++p) P.off[p] = P.off[parts];
  const uint32_t total = P.off[parts];
  unsigned blocks = (total + 255) / 256;
  if (blocks > (unsigned)sms * 8) blocks = sms * 8;
  if (blocks == 0) blocks = 1;
  k_cull_flags<<<blocks, 256, 0, s>>>(P, total, box, margin, keep);
  cudaMemsetAsync(keep + total, 0, sizeof(uint32_t), s);
  cudaError_t e = launch_exclusive_scan(s, keep, total + 1, scan_tmp, dst);
  if (e != cudaSuccess) return e;
  k_cull_scatter<<<blocks, 256, 0, s>>>(P, total, keep, dst, pos, nrm, wi, pw, depth);
  note_launches(2);
  return cudaGetLastError();
}

}  // namespace fppm_b200
