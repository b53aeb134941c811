// grid.cu -- uniform hash-grid build on the device (PhotonGrid, photon_map.cpp:26-51).
//
//  1. k_cell_bounds: per-photon fp64 cell coordinates floor(x * (1/cell))
//     (photon_map.cpp:13-15), block-reduced min/max -> grid bounding box.
//  2. k_grid_header: dense dims; dense id = ((x*ny + y)*nz + z) preserves the
//     reference key order (x major, z minor; photon_map.cpp:19-24).
//  3. k_dense_keys + hand-written LSD radix sort of (dense id, photon index)
//     pairs.  Stable, so ties keep insertion order exactly like std::sort on
//     (key, index) pairs (photon_map.cpp:39-40).  Per pass: tile digit
//     histograms, a two-kernel digit-major scan, and a stable scatter whose
//     tile is staged in shared memory in sorted order and streamed out
//     coalesced.
//  4. k_cell_start: start offset per dense cell (the cells_ ranges).
//  5. k_permute: 64-B photon records written in sorted order as four
//     coalesced float4 SoA streams (the gather reads rec0 per candidate).
#include "common.cuh"
#include "gather.cuh"

namespace fppm_b200 {

std::atomic<unsigned long long> g_kernel_launches{0};

// ------------------------------------------------------------------ block helpers
template <typename T, typename Op>
__device__ __forceinline__ T warp_reduce(T v, Op op) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = op(v, __shfl_xor_sync(kFull, v, o));
  return v;
}

// ------------------------------------------------------------------ bounds
__global__ void __launch_bounds__(256)
    k_cell_bounds(const float *__restrict__ pos, uint32_t n, const double *__restrict__ cell_ptr,
                  uint32_t S, long long *__restrict__ bounds /* [8]: min xyz, max xyz, z bits min / max */) {
  const double inv = dm(dd(1.0, *cell_ptr), (double)S);  // photon_map.cpp:29, x S exactly
  long long mn[3] = {LLONG_MAX, LLONG_MAX, LLONG_MAX};
  long long mx[3] = {LLONG_MIN, LLONG_MIN, LLONG_MIN};
  // the photons' z as raw bit patterns (min == max <=> one bit-identical z:
  // the flat lean layout, common.cuh)
  uint32_t zlo = 0xffffffffu, zhi = 0u;
  // 4 photons (12 floats) per thread with 16-B loads when aligned; axis of
  // float k of a quad = k % 3
  const uint32_t nq = (reinterpret_cast<uintptr_t>(pos) & 15u) == 0u ? n / 4 : 0;
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < nq; t += gridDim.x * blockDim.x) {
    const float4 *q = reinterpret_cast<const float4 *>(pos + 12 * (size_t)t);
    const float4 a = q[0], b = q[1], c = q[2];
    const float v[12] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w, c.x, c.y, c.z, c.w};
#pragma unroll
    for (int k = 0; k < 12; ++k) {
      const long long cc = (long long)floor(dm((double)v[k], inv));
      mn[k % 3] = min(mn[k % 3], cc);
      mx[k % 3] = max(mx[k % 3], cc);
      if (k % 3 == 2) {
        zlo = min(zlo, __float_as_uint(v[k]));
        zhi = max(zhi, __float_as_uint(v[k]));
      }
    }
  }
  for (uint32_t i = 4 * nq + blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const long long c = (long long)floor(dm((double)pos[3 * (size_t)i + a], inv));
      mn[a] = min(mn[a], c);
      mx[a] = max(mx[a], c);
    }
    const uint32_t zb = __float_as_uint(pos[3 * (size_t)i + 2]);
    zlo = min(zlo, zb);
    zhi = max(zhi, zb);
  }
  __shared__ long long s[6][8];
  __shared__ uint32_t s_z[2][8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const long long wmin = warp_reduce(mn[a], [](long long x, long long y) { return min(x, y); });
    const long long wmax = warp_reduce(mx[a], [](long long x, long long y) { return max(x, y); });
    if (lane == 0) {
      s[a][warp] = wmin;
      s[3 + a][warp] = wmax;
    }
  }
  {
    const uint32_t wlo = warp_reduce(zlo, [](uint32_t x, uint32_t y) { return min(x, y); });
    const uint32_t whi = warp_reduce(zhi, [](uint32_t x, uint32_t y) { return max(x, y); });
    if (lane == 0) {
      s_z[0][warp] = wlo;
      s_z[1][warp] = whi;
    }
  }
  __syncthreads();
  if (threadIdx.x == 3) {
    uint32_t blo = 0xffffffffu, bhi = 0u;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      blo = min(blo, s_z[0][w]);
      bhi = max(bhi, s_z[1][w]);
    }
    atomicMin(&bounds[6], (long long)blo);
    atomicMax(&bounds[7], (long long)bhi);
  }
  if (threadIdx.x < 3) {
    const int a = threadIdx.x;
    long long bmin = LLONG_MAX, bmax = LLONG_MIN;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      bmin = min(bmin, s[a][w]);
      bmax = max(bmax, s[3 + a][w]);
    }
    atomicMin(&bounds[a], bmin);
    atomicMax(&bounds[3 + a], bmax);
  }
}

// bounds are in cells of size cell / S_req.  The fine (slab) layout is kept
// when the z extent is at most 3 reference cells and the dense table fits;
// otherwise the bounds are folded back to reference cells (>> shift, exact).
__global__ void k_grid_header(const long long *__restrict__ bounds, const double *__restrict__ cell_ptr,
                              uint32_t n, unsigned long long max_cells, uint32_t S_req,
                              const uint32_t *__restrict__ lean_ok, int allow_flat,
                              GridHeader *__restrict__ hdr) {
  GridHeader g;
  g.cell = *cell_ptr;
  g.n = n;
  g.lean = 0;
  g.zflat = 0.0f;
  g.pad_ = 0;
  uint32_t shift = 0;
  while ((1u << shift) < S_req) ++shift;
  long long b[6];
  for (int i = 0; i < 6; ++i) b[i] = bounds[i];
  if (n > 0 && S_req > 1) {
    const double fx = (double)(b[3] - b[0] + 1), fy = (double)(b[4] - b[1] + 1),
                 fz = (double)(b[5] - b[2] + 1);
    if (!(fz <= 3.0 * S_req && fx * fy * fz <= (double)max_cells)) {
      // not a slab: 3D fine cells (S = 2) when the dense table fits, else
      // reference cells.  b holds fine coordinates at S_req; floor division
      // by a power of two is an arithmetic shift.
      long long r[6];
      for (int i = 0; i < 6; ++i) r[i] = b[i] >> shift;  // reference cells
      const double rc = (double)(r[3] - r[0] + 1) * (double)(r[4] - r[1] + 1) * (double)(r[5] - r[2] + 1);
      if (shift >= 1 && 8.0 * rc <= (double)max_cells) {
        for (int i = 0; i < 6; ++i) b[i] >>= (shift - 1);
        shift = 1;
      } else {
        for (int i = 0; i < 6; ++i) b[i] = r[i];
        shift = 0;
      }
    }
  } else {
    shift = 0;
  }
  g.S = 1u << shift;
  g.shift = shift;
  g.lean = (shift > 0 && lean_ok != nullptr && *lean_ok != 0u) ? 1u : 0u;
  if (g.lean != 0u && allow_flat && n > 0 && bounds[6] == bounds[7]) {  // one z: 32-B flat records
    g.lean = 2u;
    g.zflat = __uint_as_float((uint32_t)bounds[6]);
  }
  g.inv = dm(dd(1.0, g.cell), (double)g.S);
  if (n == 0) {
    g.ix0 = g.iy0 = g.iz0 = 0;
    g.nx = g.ny = g.nz = 1;
    g.ncells = 1;
    g.key_bits = 1;
    g.ok = 1;
  } else {
    g.ix0 = b[0];
    g.iy0 = b[1];
    g.iz0 = b[2];
    g.nx = b[3] - b[0] + 1;
    g.ny = b[4] - b[1] + 1;
    g.nz = b[5] - b[2] + 1;
    double dcells = (double)g.nx * (double)g.ny * (double)g.nz;
    // A dense table that would not fit (many tiny cells over a large box,
    // e.g. a global radius schedule late in a render): coarsen the cell by
    // powers of two.  floor(x * inv / 2) = floor(floor(x * inv) / 2), so the
    // bounds shift exactly; every radius stays <= the cell, so each hit
    // point's accepted set is unchanged -- only the candidates' visit order
    // (the fp64 summation order) differs from the reference's r_max grid.
    for (int k = 0; k < 24 && !(dcells <= (double)max_cells); ++k) {
      for (int i = 0; i < 6; ++i) b[i] >>= 1;
      g.cell = dm(g.cell, 2.0);
      g.inv = dm(g.inv, 0.5);
      g.ix0 = b[0]; g.iy0 = b[1]; g.iz0 = b[2];
      g.nx = b[3] - b[0] + 1; g.ny = b[4] - b[1] + 1; g.nz = b[5] - b[2] + 1;
      dcells = (double)g.nx * (double)g.ny * (double)g.nz;
    }
    g.ok = (g.nx > 0 && g.ny > 0 && g.nz > 0 && dcells <= (double)max_cells) ? 1u : 0u;
    g.ncells = g.ok ? (unsigned long long)g.nx * (unsigned long long)g.ny * (unsigned long long)g.nz : 0;
    uint32_t bits = 1;
    while (bits < 32 && (1ull << bits) < g.ncells) ++bits;
    g.key_bits = bits;
  }
  *hdr = g;
}

__global__ void __launch_bounds__(256)
    k_dense_keys(const float *__restrict__ pos, uint32_t n, const GridHeader *__restrict__ hdr,
                 uint32_t *__restrict__ keys, uint32_t *__restrict__ vals) {
  const GridHeader g = *hdr;
  auto key = [&](float x, float y, float z) {
    const long long X = (long long)floor(dm((double)x, g.inv)) - g.ix0;
    const long long Y = (long long)floor(dm((double)y, g.inv)) - g.iy0;
    const long long Z = (long long)floor(dm((double)z, g.inv)) - g.iz0;
    return (uint32_t)((X * g.ny + Y) * g.nz + Z);
  };
  // 4 photons per thread with three 16-B position loads when aligned
  const uint32_t nq = (reinterpret_cast<uintptr_t>(pos) & 15u) == 0u ? n / 4 : 0;
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < nq; t += stride) {
    const float4 *q = reinterpret_cast<const float4 *>(pos + 12 * (size_t)t);
    const float4 a = q[0], b = q[1], c = q[2];
    const uint4 k = make_uint4(key(a.x, a.y, a.z), key(a.w, b.x, b.y), key(b.z, b.w, c.x), key(c.y, c.z, c.w));
    reinterpret_cast<uint4 *>(keys)[t] = k;
    reinterpret_cast<uint4 *>(vals)[t] = make_uint4(4 * t, 4 * t + 1, 4 * t + 2, 4 * t + 3);
  }
  for (uint32_t i = 4 * nq + blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const size_t o = 3 * (size_t)i;
    keys[i] = key(pos[o], pos[o + 1], pos[o + 2]);
    vals[i] = i;
  }
}

static __device__ __forceinline__ bool aligned16(const void *p) {
  return (reinterpret_cast<uintptr_t>(p) & 15u) == 0u;
}

// Block of 256 consecutive photons: the SoA input is staged through shared
// memory with 16-B loads (3.25 per thread instead of 13 scalar loads), then
// each thread builds its photon's record (written 64 B apart).
__global__ void __launch_bounds__(256)
    k_pack_fine(const float *__restrict__ pos, const float *__restrict__ nrm, const float *__restrict__ wi,
                const float *__restrict__ pw, const uint32_t *__restrict__ depth, uint32_t n,
                const GridHeader *__restrict__ hdr, double guard, float4 *__restrict__ pack) {
  __shared__ float4 s_in[4][192];
  __shared__ uint4 s_d[64];
  const bool lean = hdr->lean != 0u, flat = hdr->lean == 2u;
  const bool vec = aligned16(pos) && aligned16(nrm) && aligned16(wi) && aligned16(pw) && aligned16(depth);
  const float *src[4] = {pos, nrm, wi, pw};
  for (uint32_t b0 = blockIdx.x * 256u; b0 < n; b0 += gridDim.x * 256u) {
    const uint32_t i = b0 + threadIdx.x;
    PhotonIn P;
    if (vec && b0 + 256u <= n) {
      __syncthreads();
      if (threadIdx.x < 192) {
#pragma unroll
        for (int f = 0; f < 4; ++f)
          s_in[f][threadIdx.x] = __ldcs(reinterpret_cast<const float4 *>(src[f] + 3 * (size_t)b0) + threadIdx.x);
      } else {
        s_d[threadIdx.x - 192] = __ldcs(reinterpret_cast<const uint4 *>(depth + b0) + (threadIdx.x - 192));
      }
      __syncthreads();
#pragma unroll
      for (int f = 0; f < 4; ++f) {
        const float *sf = reinterpret_cast<const float *>(s_in[f]) + 3 * threadIdx.x;
        float *dst = f == 0 ? P.p : (f == 1 ? P.n : (f == 2 ? P.w : P.c));
        dst[0] = sf[0];
        dst[1] = sf[1];
        dst[2] = sf[2];
      }
      P.d = reinterpret_cast<const uint32_t *>(s_d)[threadIdx.x];
    } else if (i < n) {
      P = load_photon(pos, nrm, wi, pw, depth, i);
    }
    if (i < n) {
      float4 q0, q1, q2, q3;
      if (flat) {  // flat lean records packed 32 B apart
        flat_record(P, guard, q0, q1);
        pack[2 * (size_t)i] = q0;
        pack[2 * (size_t)i + 1] = q1;
        continue;
      }
      float4 *d = pack + (lean ? 3 : 4) * (size_t)i;  // lean records packed 48 B apart
      if (lean) {
        lean_record(P, guard, q0, q1, q2);
      } else {
        fine_record(P, q0, q1, q2, q3);
        d[3] = q3;
      }
      d[0] = q0;
      d[1] = q1;
      d[2] = q2;
    }
  }
}

__global__ void __launch_bounds__(256)
    k_permute_packed(const uint32_t *__restrict__ order, uint32_t n, const float4 *__restrict__ pack,
                     float4 *__restrict__ rec0, float4 *__restrict__ rec1, float4 *__restrict__ rec2,
                     float4 *__restrict__ rec3, const GridHeader *__restrict__ hdr) {
  if (hdr != nullptr && hdr->lean != 0u) rec3 = nullptr;  // lean records: 48 B
  if (hdr != nullptr && hdr->lean == 2u) {                // flat lean records: 32 B
    constexpr uint32_t V = 6;
    const uint32_t st = gridDim.x * blockDim.x;
    for (uint32_t i0 = blockIdx.x * blockDim.x + threadIdx.x; i0 < n; i0 += V * st) {
      uint32_t o[V];
#pragma unroll
      for (uint32_t u = 0; u < V; ++u) o[u] = i0 + u * st < n ? __ldg(&order[i0 + u * st]) : 0u;
      float4 q[V][2];
#pragma unroll
      for (uint32_t u = 0; u < V; ++u) {
        const float4 *src = pack + 2 * (size_t)o[u];
        if (i0 + u * st < n) {
          q[u][0] = __ldg(&src[0]);
          q[u][1] = __ldg(&src[1]);
        }
      }
#pragma unroll
      for (uint32_t u = 0; u < V; ++u) {
        const uint32_t i = i0 + u * st;
        if (i < n) {
          __stcs(&rec0[i], q[u][0]);
          __stcs(&rec1[i], q[u][1]);
        }
      }
    }
    return;
  }
  // U records per thread per round, all loads issued before the stores
  // (random 64-B record reads: latency bound without the extra parallelism)
  constexpr uint32_t U = 4;
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t i0 = blockIdx.x * blockDim.x + threadIdx.x; i0 < n; i0 += U * stride) {
    uint32_t o[U];
#pragma unroll
    for (uint32_t u = 0; u < U; ++u) o[u] = i0 + u * stride < n ? __ldg(&order[i0 + u * stride]) : 0u;
    float4 q[U][4];
#pragma unroll
    for (uint32_t u = 0; u < U; ++u) {
      const float4 *src = pack + (rec3 ? 4 : 3) * (size_t)o[u];
      if (i0 + u * stride < n) {
        q[u][0] = __ldg(&src[0]); q[u][1] = __ldg(&src[1]); q[u][2] = __ldg(&src[2]);
        if (rec3) q[u][3] = __ldg(&src[3]);
      }
    }
#pragma unroll
    for (uint32_t u = 0; u < U; ++u) {
      const uint32_t i = i0 + u * stride;
      if (i < n) {
        __stcs(&rec0[i], q[u][0]);
        __stcs(&rec1[i], q[u][1]);
        __stcs(&rec2[i], q[u][2]);
        if (rec3) __stcs(&rec3[i], q[u][3]);
      }
    }
  }
}

// ------------------------------------------------------------------ radix sort
constexpr int kSortThreads = 256;
constexpr int kSortItems = 12;
constexpr int kTile = kSortThreads * kSortItems;  // 3072 keys per tile
constexpr int kRadixBits = 9;                     // digits of up to 9 bits: 18-bit keys in 2 passes
constexpr int kRadixMax = 1 << kRadixBits;
static_assert(kRadixMax == 2 * kSortThreads, "two digits per thread in the tile scans");

__global__ void __launch_bounds__(kSortThreads)
    k_radix_upsweep(const uint32_t *__restrict__ keys, uint32_t n, int shift, uint32_t mask,
                    uint32_t *__restrict__ hist /* [digit][tile] */, uint32_t tiles) {
  // per-warp sub-histograms: clustered keys (a photon blob) contend only
  // within a warp; all loads are issued before the counting
  constexpr int kWarps = kSortThreads / kWarp;
  __shared__ uint32_t s_h[kWarps][kRadixMax];
  for (int d = threadIdx.x; d < kWarps * kRadixMax; d += blockDim.x) (&s_h[0][0])[d] = 0;
  __syncthreads();
  const uint32_t base = blockIdx.x * kTile;
  const int warp = threadIdx.x / kWarp;
  uint32_t k[kSortItems];
#pragma unroll
  for (int it = 0; it < kSortItems; ++it) {
    const uint32_t i = base + it * kSortThreads + threadIdx.x;
    k[it] = i < n ? __ldcs(&keys[i]) : 0xffffffffu;
  }
#pragma unroll
  for (int it = 0; it < kSortItems; ++it) {
    const uint32_t i = base + it * kSortThreads + threadIdx.x;
    if (i < n) atomicAdd(&s_h[warp][(k[it] >> shift) & mask], 1u);
  }
  __syncthreads();
  for (uint32_t d = threadIdx.x; d <= mask; d += blockDim.x) {
    uint32_t c = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) c += s_h[w][d];
    hist[d * tiles + blockIdx.x] = c;
  }
}

// block d: total of digit d over all tiles
__global__ void __launch_bounds__(256)
    k_digit_totals(const uint32_t *__restrict__ hist, uint32_t tiles, uint32_t *__restrict__ totals) {
  const uint32_t *row = hist + (size_t)blockIdx.x * tiles;
  uint32_t s = 0;
  for (uint32_t i = threadIdx.x; i < tiles; i += blockDim.x) s += row[i];
  s = warp_reduce(s, [](uint32_t x, uint32_t y) { return x + y; });
  __shared__ uint32_t sw[8];
  if ((threadIdx.x & 31) == 0) sw[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (int w = 0; w < 8; ++w) t += sw[w];
    totals[blockIdx.x] = t;
  }
}

// block d: hist[d][*] <- exclusive digit-major prefix (all tiles of digits < d
// first, then tiles of digit d in order).
__global__ void __launch_bounds__(256)
    k_hist_scan(uint32_t *__restrict__ hist, uint32_t tiles, const uint32_t *__restrict__ totals) {
  __shared__ uint32_t s_warp[8];
  uint32_t part = 0;
  for (uint32_t d = threadIdx.x; d < blockIdx.x; d += blockDim.x) part += totals[d];
  uint32_t base_total;
  (void)block_exclusive_scan_256(part, s_warp, &base_total);
  uint32_t carry = base_total;
  uint32_t *row = hist + (size_t)blockIdx.x * tiles;
  for (uint32_t c = 0; c < tiles; c += blockDim.x) {
    const uint32_t i = c + threadIdx.x;
    const uint32_t v = i < tiles ? row[i] : 0u;
    uint32_t tot;
    const uint32_t ex = block_exclusive_scan_256(v, s_warp, &tot);
    if (i < tiles) row[i] = carry + ex;
    carry += tot;
  }
}

// Stable tile ranking: warp w owns tile elements [w*32*ITEMS, (w+1)*32*ITEMS)
// in rounds of 32 consecutive keys; __match_any_sync groups equal digits, so
// rank = per-warp running count + earlier peers in the round.  Per-digit
// prefixes over warps keep warp order (= index order).
__global__ void __launch_bounds__(kSortThreads)
    k_radix_downsweep(const uint32_t *__restrict__ keys_in, const uint32_t *__restrict__ vals_in,
                      uint32_t *__restrict__ keys_out, uint32_t *__restrict__ vals_out,
                      uint32_t n, int shift, uint32_t mask,
                      const uint32_t *__restrict__ hist_scan, uint32_t tiles) {
  constexpr int kWarps = kSortThreads / kWarp;
  __shared__ uint32_t s_wcnt[kWarps][kRadixMax];
  __shared__ uint32_t s_dstart[kRadixMax];
  __shared__ uint32_t s_gbase[kRadixMax];
  __shared__ uint32_t s_keys[kTile];
  __shared__ uint32_t s_vals[kTile];
  __shared__ uint32_t s_warp[8];
  const int warp = threadIdx.x / kWarp, lane = threadIdx.x % kWarp;
  for (int i = threadIdx.x; i < kWarps * kRadixMax; i += blockDim.x) (&s_wcnt[0][0])[i] = 0;
  __syncthreads();
  const uint32_t tile_base = blockIdx.x * kTile;
  const uint32_t lt_mask = (1u << lane) - 1u;
  uint32_t k[kSortItems], v[kSortItems], rank[kSortItems];
  // all loads issued before the ranking (its warp-synchronous shared-memory
  // updates would otherwise serialise them)
#pragma unroll
  for (int it = 0; it < kSortItems; ++it) {
    const uint32_t i = tile_base + (warp * kSortItems + it) * kWarp + lane;
    const bool valid = i < n;
    k[it] = valid ? __ldcs(&keys_in[i]) : 0u;
    v[it] = valid ? __ldcs(&vals_in[i]) : 0u;
  }
#pragma unroll
  for (int it = 0; it < kSortItems; ++it) {
    const uint32_t i = tile_base + (warp * kSortItems + it) * kWarp + lane;
    const bool valid = i < n;
    const uint32_t d = valid ? ((k[it] >> shift) & mask) : (uint32_t)kRadixMax;
    const uint32_t peers = __match_any_sync(kFull, d);
    const uint32_t before = valid ? s_wcnt[warp][d] : 0u;
    __syncwarp();
    if (valid && (__ffs(peers) - 1) == lane) s_wcnt[warp][d] = before + __popc(peers);
    __syncwarp();
    rank[it] = before + __popc(peers & lt_mask);
  }
  __syncthreads();
  // thread t owns digits 2t, 2t + 1: per-warp prefixes (warp order = index
  // order), global bases, and the tile's digit starts
  uint32_t tot2[2];
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const uint32_t d = 2 * threadIdx.x + j;
    uint32_t total = 0;
    for (int w = 0; w < kWarps; ++w) {
      const uint32_t c = s_wcnt[w][d];
      s_wcnt[w][d] = total;
      total += c;
    }
    tot2[j] = total;
    s_gbase[d] = d <= mask ? hist_scan[d * tiles + blockIdx.x] : 0u;
  }
  uint32_t tile_total;
  const uint32_t start = block_exclusive_scan_256(tot2[0] + tot2[1], s_warp, &tile_total);
  s_dstart[2 * threadIdx.x] = start;
  s_dstart[2 * threadIdx.x + 1] = start + tot2[0];
  __syncthreads();
#pragma unroll
  for (int it = 0; it < kSortItems; ++it) {
    const uint32_t i = tile_base + (warp * kSortItems + it) * kWarp + lane;
    if (i < n) {
      const uint32_t d = (k[it] >> shift) & mask;
      const uint32_t lp = s_dstart[d] + s_wcnt[warp][d] + rank[it];
      s_keys[lp] = k[it];
      s_vals[lp] = v[it];
    }
  }
  __syncthreads();
  const uint32_t valid_n = min((uint32_t)kTile, n - tile_base);
  for (uint32_t i = threadIdx.x; i < valid_n; i += blockDim.x) {
    const uint32_t key = s_keys[i];
    const uint32_t d = (key >> shift) & mask;
    const uint32_t o = s_gbase[d] + (i - s_dstart[d]);
    keys_out[o] = key;
    vals_out[o] = s_vals[i];
  }
}

// ------------------------------------------------------------------ cell table
// start[c] = first sorted position with dense id >= c, c in [0, ncells].
// Dense tables (every gap short): thread per photon writes its own gap.
__global__ void k_cell_start_dense(const uint32_t *__restrict__ skeys, uint32_t n, unsigned long long ncells,
                                   uint32_t *__restrict__ start) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const unsigned long long k = skeys[i];
    const unsigned long long prev = i == 0 ? 0ull : (unsigned long long)skeys[i - 1] + 1ull;
    for (unsigned long long c = prev; c <= k; ++c) start[c] = i;
    if (i == n - 1)
      for (unsigned long long c = k + 1; c <= ncells; ++c) start[c] = n;
  }
}

// Any table: photon i owns the cells (key[i - 1], key[i]] (start = i) and the
// last photon also (key[n - 1], ncells] (start = n).  Short gaps are written
// by their owner lane; long ones (empty stretches of a sparse or clustered
// photon set) by the whole warp with coalesced stores, so no thread walks a
// long gap and no binary search is needed.
__global__ void __launch_bounds__(256) k_cell_start_gaps(const uint32_t *__restrict__ skeys, uint32_t n,
                                                         unsigned long long ncells, uint32_t *__restrict__ start) {
  constexpr unsigned long long kShort = 8;
  const int lane = threadIdx.x & 31;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t base = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 32; base < n; base += nwarps * 32) {
    const uint32_t i = base + lane;
    const bool valid = i < n;
    unsigned long long lo = 0, hi = 0;  // cells [lo, hi) get start = i
    if (valid) {
      const unsigned long long k = __ldg(&skeys[i]);
      lo = i == 0 ? 0ull : (unsigned long long)__ldg(&skeys[i - 1]) + 1ull;
      hi = k + 1;
    }
    if (hi - lo <= kShort)
      for (unsigned long long c = lo; c < hi; ++c) start[c] = i;
    uint32_t big = __ballot_sync(kFull, hi - lo > kShort);
    while (big) {
      const int j = __ffs(big) - 1;
      big &= big - 1;
      const unsigned long long a = __shfl_sync(kFull, lo, j), b = __shfl_sync(kFull, hi, j);
      for (unsigned long long c = a + lane; c < b; c += 32) start[c] = base + j;
    }
    // cells after the last photon's
    const unsigned long long tl = __shfl_sync(kFull, (valid && i == n - 1) ? hi : 0ull, (n - 1 - base) & 31);
    if (n - 1 >= base && n - 1 < base + 32)
      for (unsigned long long c = tl + lane; c <= ncells; c += 32) start[c] = n;
  }
}

__global__ void k_cell_start_empty(uint32_t *__restrict__ start, unsigned long long ncells) {
  for (unsigned long long c = blockIdx.x * blockDim.x + threadIdx.x; c <= ncells;
       c += gridDim.x * blockDim.x)
    start[c] = 0;
}

// ------------------------------------------------------------------ permute
__global__ void __launch_bounds__(256)
    k_permute(const uint32_t *__restrict__ order, uint32_t n, const float *__restrict__ pos,
              const float *__restrict__ nrm, const float *__restrict__ wi,
              const float *__restrict__ pw, const uint32_t *__restrict__ depth,
              float4 *__restrict__ rec0, float4 *__restrict__ rec1, float4 *__restrict__ rec2,
              float4 *__restrict__ rec3) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const size_t j = order[i];
    const size_t o = 3 * j;
    rec0[i] = make_float4(pos[o], pos[o + 1], pos[o + 2], __uint_as_float(depth[j]));
    rec1[i] = make_float4(nrm[o], nrm[o + 1], nrm[o + 2], wi[o]);
    rec2[i] = make_float4(wi[o + 1], wi[o + 2], pw[o], pw[o + 1]);
    // luminance of the photon power in fp64 (vec.hpp:79-81), for gray hit-point weights
    const double L = elum((double)pw[o], (double)pw[o + 1], (double)pw[o + 2]);
    const unsigned long long Lb = (unsigned long long)__double_as_longlong(L);
    rec3[i] = make_float4(pw[o + 2], 0.f, __uint_as_float((uint32_t)Lb),
                          __uint_as_float((uint32_t)(Lb >> 32)));
  }
}

// warp / sparse kernel layout, packed in input order (coalesced) so the
// permute moves whole 64-B records
__global__ void __launch_bounds__(256)
    k_pack_std(const float *__restrict__ pos, const float *__restrict__ nrm, const float *__restrict__ wi,
               const float *__restrict__ pw, const uint32_t *__restrict__ depth, uint32_t n,
               float4 *__restrict__ pack) {
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    const size_t o = 3 * (size_t)j;
    float4 *d = pack + 4 * (size_t)j;
    d[0] = make_float4(pos[o], pos[o + 1], pos[o + 2], __uint_as_float(depth[j]));
    d[1] = make_float4(nrm[o], nrm[o + 1], nrm[o + 2], wi[o]);
    d[2] = make_float4(wi[o + 1], wi[o + 2], pw[o], pw[o + 1]);
    const double L = elum((double)pw[o], (double)pw[o + 1], (double)pw[o + 2]);
    const unsigned long long Lb = (unsigned long long)__double_as_longlong(L);
    d[3] = make_float4(pw[o + 2], 0.f, __uint_as_float((uint32_t)Lb), __uint_as_float((uint32_t)(Lb >> 32)));
  }
}

// fine-gather layout (common.cuh): the planar fast path reads rec0..rec2 only
__global__ void __launch_bounds__(256)
    k_permute_fine(const uint32_t *__restrict__ order, uint32_t n, const float *__restrict__ pos,
                   const float *__restrict__ nrm, const float *__restrict__ wi,
                   const float *__restrict__ pw, const uint32_t *__restrict__ depth,
                   float4 *__restrict__ rec0, float4 *__restrict__ rec1, float4 *__restrict__ rec2,
                   float4 *__restrict__ rec3) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const size_t j = order[i];
    const size_t o = 3 * j;
    const float nx = nrm[o], ny = nrm[o + 1], wx = wi[o], wy = wi[o + 1];
    const double L = elum((double)pw[o], (double)pw[o + 1], (double)pw[o + 2]);
    const unsigned long long Lb = (unsigned long long)__double_as_longlong(L);
    const uint32_t flags =
        (fabsf(nx) < INFINITY && fabsf(ny) < INFINITY && fabsf(wx) < INFINITY && fabsf(wy) < INFINITY)
            ? 1u : 0u;
    rec0[i] = make_float4(pos[o], pos[o + 1], pos[o + 2], __uint_as_float(depth[j]));
    rec1[i] = make_float4(nrm[o + 2], wi[o + 2], __uint_as_float((uint32_t)Lb),
                          __uint_as_float((uint32_t)(Lb >> 32)));
    rec2[i] = make_float4(pw[o], pw[o + 1], pw[o + 2], __uint_as_float(flags));
    rec3[i] = make_float4(nx, ny, wx, wy);
  }
}

// ------------------------------------------------------------------ query_ball
// photon_map.cpp:53-78: 27 cells in (dx, dy, dz) nested order, each cell in
// sorted (= insertion) order, closed fp64 ball test.  pass 0 counts, pass 1 fills.
__global__ void k_query_ball(const double *__restrict__ centers, const double *__restrict__ radii,
                             uint32_t nq, const GridHeader *__restrict__ hdr,
                             const uint32_t *__restrict__ start, const float4 *__restrict__ rec0,
                             const uint32_t *__restrict__ order,
                             unsigned long long *__restrict__ counts,
                             const unsigned long long *__restrict__ offsets,
                             uint32_t *__restrict__ out, int fill) {
  const GridHeader g = *hdr;
  for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < nq; q += gridDim.x * blockDim.x) {
    const double cx = centers[3 * (size_t)q], cy = centers[3 * (size_t)q + 1],
                 cz = centers[3 * (size_t)q + 2];
    const double r = radii[q];
    const double r2 = dm(r, r);
    const long long ix = (long long)floor(dm(cx, g.inv)) - g.ix0;
    const long long iy = (long long)floor(dm(cy, g.inv)) - g.iy0;
    const long long iz = (long long)floor(dm(cz, g.inv)) - g.iz0;
    unsigned long long cnt = 0;
    const unsigned long long o = fill ? offsets[q] : 0ull;
    for (int dx = -1; dx <= 1; ++dx)
      for (int dy = -1; dy <= 1; ++dy)
        for (int dz = -1; dz <= 1; ++dz) {
          const long long X = ix + dx, Y = iy + dy, Z = iz + dz;
          if (g.n == 0 || X < 0 || Y < 0 || Z < 0 || X >= g.nx || Y >= g.ny || Z >= g.nz) continue;
          const unsigned long long c = (unsigned long long)((X * g.ny + Y) * g.nz + Z);
          for (uint32_t i = start[c]; i < start[c + 1]; ++i) {
            const float4 p = rec0[i];
            const double ddx = ds((double)p.x, cx), ddy = ds((double)p.y, cy),
                         ddz = ds((double)p.z, cz);
            if (edot(ddx, ddy, ddz, ddx, ddy, ddz) <= r2) {
              if (fill) out[o + cnt] = order[i];
              ++cnt;
            }
          }
        }
    if (!fill) counts[q] = cnt;
  }
}

// ------------------------------------------------------------------ launchers
static inline int cap_blocks(unsigned long long work, int threads, int sms, int per_sm) {
  unsigned long long b = (work + threads - 1) / threads;
  const unsigned long long cap = (unsigned long long)sms * per_sm;
  if (b > cap) b = cap;
  return (int)(b ? b : 1);
}

size_t radix_hist_entries(uint32_t n) {
  const uint32_t tiles = (n + kTile - 1) / kTile;
  return (size_t)kRadixMax * (tiles ? tiles : 1) + kRadixMax;  // + digit totals
}

// Sorts (keys_a, vals_a) by the low `bits` bits; returns the buffers holding
// the result (a or b) through the out pointers.
cudaError_t radix_sort_pairs(cudaStream_t s, SortScratch &sc, uint32_t n, uint32_t bits,
                             uint32_t **keys_sorted, uint32_t **vals_sorted) {
  uint32_t *ki = sc.keys_a, *vi = sc.vals_a, *ko = sc.keys_b, *vo = sc.vals_b;
  if (n > 1) {
    const uint32_t tiles = (n + kTile - 1) / kTile;
    const uint32_t passes = (bits + kRadixBits - 1) / kRadixBits;
    const uint32_t width = (bits + passes - 1) / passes;
    uint32_t *totals = sc.hist + (size_t)kRadixMax * tiles;
    for (uint32_t p = 0; p < passes; ++p) {
      const int shift = (int)(p * width);
      const uint32_t w = min(width, bits - p * width);
      const uint32_t mask = (1u << w) - 1u;
      k_radix_upsweep<<<tiles, kSortThreads, 0, s>>>(ki, n, shift, mask, sc.hist, tiles);
      k_digit_totals<<<mask + 1, 256, 0, s>>>(sc.hist, tiles, totals);
      k_hist_scan<<<mask + 1, 256, 0, s>>>(sc.hist, tiles, totals);
      k_radix_downsweep<<<tiles, kSortThreads, 0, s>>>(ki, vi, ko, vo, n, shift, mask, sc.hist,
                                                       tiles);
      note_launches(4);
      uint32_t *t;
      t = ki; ki = ko; ko = t;
      t = vi; vi = vo; vo = t;
    }
  }
  *keys_sorted = ki;
  *vals_sorted = vi;
  return cudaGetLastError();
}

void launch_cell_bounds(cudaStream_t s, const float *pos, uint32_t n, const double *cell,
                        uint32_t S, long long *bounds, int sms) {
  if (n == 0) return;
  k_cell_bounds<<<cap_blocks(n, 256, sms, 8), 256, 0, s>>>(pos, n, cell, S, bounds);
  note_launches(1);
}

void launch_grid_header(cudaStream_t s, const long long *bounds, const double *cell, uint32_t n,
                        unsigned long long max_cells, uint32_t S, const uint32_t *lean_ok, bool allow_flat,
                        GridHeader *hdr) {
  k_grid_header<<<1, 1, 0, s>>>(bounds, cell, n, max_cells, S, lean_ok, allow_flat ? 1 : 0, hdr);
  note_launches(1);
}

void launch_pack_fine(cudaStream_t s, const float *pos, const float *nrm, const float *wi, const float *pw,
                      const uint32_t *depth, uint32_t n, const GridHeader *hdr, double guard, float4 *pack,
                      int sms) {
  if (n == 0) return;
  k_pack_fine<<<cap_blocks(n, 256, sms, 16), 256, 0, s>>>(pos, nrm, wi, pw, depth, n, hdr, guard, pack);
  note_launches(1);
}

// VCM+ per-photon MIS data into sorted order
__global__ void k_permute_f64x3(const uint32_t *__restrict__ order, uint32_t n, const double *__restrict__ a,
                                const double *__restrict__ b, const double *__restrict__ c,
                                double *__restrict__ oa, double *__restrict__ ob, double *__restrict__ oc) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint32_t j = order[i];
    oa[i] = a[j];
    ob[i] = b[j];
    oc[i] = c[j];
  }
}

void launch_permute_f64x3(cudaStream_t s, const uint32_t *order, uint32_t n, const double *a,
                          const double *b, const double *c, double *oa, double *ob, double *oc, int sms) {
  if (n == 0) return;
  k_permute_f64x3<<<cap_blocks(n, 256, sms, 16), 256, 0, s>>>(order, n, a, b, c, oa, ob, oc);
  note_launches(1);
}

void launch_dense_keys(cudaStream_t s, const float *pos, uint32_t n, const GridHeader *hdr,
                       uint32_t *keys, uint32_t *vals, int sms) {
  if (n == 0) return;
  k_dense_keys<<<cap_blocks(n, 256, sms, 16), 256, 0, s>>>(pos, n, hdr, keys, vals);
  note_launches(1);
}

void launch_cell_start(cudaStream_t s, const uint32_t *skeys, uint32_t n, const GridHeader *hdr,
                       uint32_t *start, unsigned long long ncells, int sms) {
  if (n == 0) {
    k_cell_start_empty<<<1, 32, 0, s>>>(start, ncells);
  } else if ((unsigned long long)n >= 4ull * ncells) {
    // >= 4 photons per cell on average: thread per photon (a long gap at the
    // end is walked by the last photon, so only for tables this dense)
    k_cell_start_dense<<<cap_blocks(n, 256, sms, 16), 256, 0, s>>>(skeys, n, ncells, start);
  } else {
    k_cell_start_gaps<<<cap_blocks(n, 256, sms, 16), 256, 0, s>>>(skeys, n, ncells, start);
  }
  note_launches(1);
}

void launch_permute(cudaStream_t s, const uint32_t *order, uint32_t n, const float *pos,
                    const float *nrm, const float *wi, const float *pw, const uint32_t *depth,
                    const PhotonRecs &r, int fine_layout, const GridHeader *hdr, int sms) {
  if (n == 0) return;
  if (fine_layout && r.pack)
    k_permute_packed<<<cap_blocks(n, 256, sms, 16), 256, 0, s>>>(order, n, r.pack, r.rec0, r.rec1, r.rec2,
                                                                  r.rec3, hdr);
  else if (fine_layout)
    k_permute_fine<<<cap_blocks(n, 256, sms, 16), 256, 0, s>>>(order, n, pos, nrm, wi, pw, depth,
                                                                r.rec0, r.rec1, r.rec2, r.rec3);
  else if (r.pack) {
    k_pack_std<<<cap_blocks(n, 256, sms, 16), 256, 0, s>>>(pos, nrm, wi, pw, depth, n, r.pack);
    note_launches(1);
    k_permute_packed<<<cap_blocks(n, 256, sms, 16), 256, 0, s>>>(order, n, r.pack, r.rec0, r.rec1, r.rec2,
                                                                  r.rec3, nullptr);
  } else
    k_permute<<<cap_blocks(n, 256, sms, 16), 256, 0, s>>>(order, n, pos, nrm, wi, pw, depth,
                                                           r.rec0, r.rec1, r.rec2, r.rec3);
  note_launches(1);
}

void launch_query_ball(cudaStream_t s, const double *centers, const double *radii, uint32_t nq,
                       const GridHeader *hdr, const uint32_t *start, const float4 *rec0,
                       const uint32_t *order, unsigned long long *counts,
                       const unsigned long long *offsets, uint32_t *out, int fill) {
  if (nq == 0) return;
  k_query_ball<<<(int)((nq + 127) / 128), 128, 0, s>>>(centers, radii, nq, hdr, start, rec0, order,
                                                       counts, offsets, out, fill);
  note_launches(1);
}

}  // namespace fppm_b200
