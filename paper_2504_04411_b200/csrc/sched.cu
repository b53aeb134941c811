// sched.cu -- hit-point scheduling shared by the gather kernels: home-cell
// binning and ordering of hit points, bucket starts, exclusive scans, and the
// fine kernel's per-item partial rows pooled into the end of iteration
// (k_tile_finalize).
#include "common.cuh"
#include "gather.cuh"
#include "gather_dev.cuh"

namespace fppm_b200 {

// 10-bit coordinate spread to every third bit (Morton order)
static __device__ __forceinline__ uint32_t spread3(uint32_t v) {
  v &= 0x3ffu;
  v = (v | (v << 16)) & 0x030000FFu;
  v = (v | (v << 8)) & 0x0300F00Fu;
  v = (v | (v << 4)) & 0x030C30C3u;
  v = (v | (v << 2)) & 0x09249249u;
  return v;
}

// Hit points keyed by their cell: Morton order when every extended axis fits
// 10 bits (spatially compact runs of hit points share records in L2), else
// the dense cell index; key `none` = no candidates (outside / not gathered).
__global__ void k_hp_bin(const double3 *__restrict__ pos, const uint8_t *__restrict__ gathered,
                         uint32_t H, const GridHeader *__restrict__ hdr, uint32_t none, int morton,
                         uint32_t *__restrict__ keys, uint32_t *__restrict__ vals) {
  const GridHeader g = *hdr;
  const long long ex = g.nx + 2, ey = g.ny + 2, ez = g.nz + 2;
  for (uint32_t h = blockIdx.x * blockDim.x + threadIdx.x; h < H; h += gridDim.x * blockDim.x) {
    uint32_t key = none;
    const double3 c = pos[h];
    if (g.n > 0 && (gathered == nullptr || gathered[h])) {
      const long long X = (long long)floor(dm(c.x, g.inv)) - g.ix0 + 1;
      const long long Y = (long long)floor(dm(c.y, g.inv)) - g.iy0 + 1;
      const long long Z = (long long)floor(dm(c.z, g.inv)) - g.iz0 + 1;
      if (X >= 0 && Y >= 0 && Z >= 0 && X < ex && Y < ey && Z < ez)
        key = morton ? (spread3((uint32_t)X) << 2) | (spread3((uint32_t)Y) << 1) | spread3((uint32_t)Z)
                     : (uint32_t)((X * ey + Y) * ez + Z);
    }
    keys[h] = key;
    vals[h] = h;
  }
}

// start[b] = first sorted position with key >= b, b in [0, nb]
__global__ void k_bucket_start(const uint32_t *__restrict__ skeys, uint32_t n, uint32_t nb,
                               uint32_t *__restrict__ start) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint32_t k = skeys[i];
    const uint32_t prev = i == 0 ? 0u : skeys[i - 1] + 1u;
    for (uint32_t b = prev; b <= k; ++b) start[b] = i;
    if (i == n - 1)
      for (uint32_t b = k + 1; b <= nb; ++b) start[b] = n;
  }
}

__global__ void k_bucket_start_bsearch(const uint32_t *__restrict__ skeys, uint32_t n, uint32_t nb,
                                       uint32_t *__restrict__ start) {
  for (uint32_t b = blockIdx.x * blockDim.x + threadIdx.x; b <= nb; b += gridDim.x * blockDim.x) {
    uint32_t lo = 0, hi = n;
    while (lo < hi) {
      const uint32_t mid = lo + (hi - lo) / 2;
      if (skeys[mid] < b) lo = mid + 1; else hi = mid;
    }
    start[b] = lo;
  }
}

// The 9 (dx, dy) columns of photon-grid cell (ix, iy, iz): each column's three
// z cells are contiguous in key order.  Returns the candidate count.

// Exclusive scan: tiles of 4096 = 256 threads x 16 consecutive values (one
// block scan per tile), tile sums scanned by one block, then applied.
constexpr int kScanTile = 4096;
constexpr int kScanPer = kScanTile / 256;
static __device__ __forceinline__ void scan_load16(const uint32_t *__restrict__ in, uint32_t n, uint32_t i0,
                                                   uint32_t (&v)[kScanPer]) {
  if (i0 + kScanPer <= n && (i0 & 3u) == 0u) {
    const uint4 *q = reinterpret_cast<const uint4 *>(in + i0);
#pragma unroll
    for (int k = 0; k < kScanPer / 4; ++k) {
      const uint4 w = q[k];
      v[4 * k] = w.x; v[4 * k + 1] = w.y; v[4 * k + 2] = w.z; v[4 * k + 3] = w.w;
    }
  } else {
#pragma unroll
    for (int k = 0; k < kScanPer; ++k) v[k] = i0 + k < n ? in[i0 + k] : 0u;
  }
}
__global__ void __launch_bounds__(256) k_scan_tiles(const uint32_t *__restrict__ in, uint32_t n,
                                                    uint32_t *__restrict__ tile_sum) {
  __shared__ uint32_t s_warp[8];
  uint32_t v[kScanPer];
  scan_load16(in, n, blockIdx.x * kScanTile + threadIdx.x * kScanPer, v);
  uint32_t s = 0;
#pragma unroll
  for (int k = 0; k < kScanPer; ++k) s += v[k];
  uint32_t tot;
  (void)block_exclusive_scan_256(s, s_warp, &tot);
  if (threadIdx.x == 0) tile_sum[blockIdx.x] = tot;
}
__global__ void __launch_bounds__(256) k_scan_top(uint32_t *__restrict__ tile_sum, uint32_t nt) {
  __shared__ uint32_t s_warp[8];
  uint32_t carry = 0;
  for (uint32_t c = 0; c < nt; c += 256) {
    const uint32_t i = c + threadIdx.x;
    const uint32_t v = i < nt ? tile_sum[i] : 0u;
    uint32_t tot;
    const uint32_t ex = block_exclusive_scan_256(v, s_warp, &tot);
    if (i < nt) tile_sum[i] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0) tile_sum[nt] = carry;
}
__global__ void __launch_bounds__(256) k_scan_apply(const uint32_t *__restrict__ in, uint32_t n,
                                                    const uint32_t *__restrict__ tile_sum,
                                                    uint32_t *__restrict__ out) {
  __shared__ uint32_t s_warp[8];
  const uint32_t i0 = blockIdx.x * kScanTile + threadIdx.x * kScanPer;
  uint32_t v[kScanPer];
  scan_load16(in, n, i0, v);
  uint32_t s = 0;
#pragma unroll
  for (int k = 0; k < kScanPer; ++k) s += v[k];
  uint32_t tot;
  uint32_t run = tile_sum[blockIdx.x] + block_exclusive_scan_256(s, s_warp, &tot);
#pragma unroll
  for (int k = 0; k < kScanPer; ++k) {
    if (i0 + k < n) out[i0 + k] = run;
    run += v[k];
  }
}

// Ring schedule: a hit point's rows are contiguous and allocated in hit-point
// order, so the 32 hit points of a warp own one contiguous run of rows.  The
// warp copies it through shared memory in chunks with coalesced 16-B loads and
// each lane sums its own rows in order (same order as k_tile_finalize).
constexpr int kFinChunk = 48;  // rows per warp and chunk
template <int GMAX, int CH>
__global__ void __launch_bounds__(128) k_tile_finalize_contig(const GatherArgs A, const TileArgs T) {
  constexpr int PS = partial_size(GMAX, CH);
  extern __shared__ __align__(16) double s_fin[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double2 *s2 = reinterpret_cast<double2 *>(s_fin + (size_t)warp * kFinChunk * PS);
  const double *sw = s_fin + (size_t)warp * kFinChunk * PS;
  const double2 *src2 = reinterpret_cast<const double2 *>(T.partials);
  double my_rmax = 0.0;
  uint32_t my_tested = 0, my_rejected = 0;
  for (uint32_t hb = blockIdx.x * blockDim.x + warp * 32; hb < A.H; hb += gridDim.x * blockDim.x) {
    const uint32_t h = hb + lane;
    const bool valid = h < A.H;
    const uint32_t rb = valid ? T.hp_map[3 * (size_t)h] : 0u, nc = valid ? T.hp_map[3 * (size_t)h + 1] : 0u;
    const uint32_t r_lo = __shfl_sync(kFull, rb, 0), r_hi = __reduce_max_sync(kFull, valid ? rb + nc : 0u);
    uint32_t cnt[GMAX];
    double sm[CH][GMAX], sq[CH][GMAX];
    double p0 = 0.0, p1 = 0.0, p2 = 0.0;
#pragma unroll
    for (int g = 0; g < GMAX; ++g) {
      cnt[g] = 0;
#pragma unroll
      for (int c = 0; c < CH; ++c) sm[c][g] = sq[c][g] = 0.0;
    }
    for (uint32_t c0 = r_lo; c0 < r_hi; c0 += kFinChunk) {
      const uint32_t c1 = min(r_hi, c0 + (uint32_t)kFinChunk);
      const uint32_t nv = (c1 - c0) * (PS / 2);
      {  // 8 loads in flight per lane
        const double2 *g2 = src2 + (size_t)c0 * (PS / 2);
        for (uint32_t k0 = 0; k0 < nv; k0 += 8 * 32) {
          double2 v[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const uint32_t k = k0 + u * 32 + lane;
            if (k < nv) v[u] = __ldcs(&g2[k]);
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const uint32_t k = k0 + u * 32 + lane;
            if (k < nv) s2[k] = v[u];
          }
        }
      }
      __syncwarp();
      const uint32_t a = max(rb, c0), e = min(rb + nc, c1);
      for (uint32_t r = a; r < e; ++r) {
        const double *pp = sw + (size_t)(r - c0) * PS;
#pragma unroll
        for (int g = 0; g < GMAX; ++g) cnt[g] += (uint32_t)pp[g];
#pragma unroll
        for (int c = 0; c < CH; ++c)
#pragma unroll
          for (int g = 0; g < GMAX; ++g) {
            sm[c][g] += pp[GMAX + c * GMAX + g];
            sq[c][g] += pp[GMAX + CH * GMAX + c * GMAX + g];
          }
        p0 += pp[GMAX + 2 * CH * GMAX];
        p1 += pp[GMAX + 2 * CH * GMAX + 1];
        p2 += pp[GMAX + 2 * CH * GMAX + 2];
      }
      __syncwarp();
    }
    if (valid) finalize_hit<GMAX, CH>(A, h, cnt, sm, sq, p0, p1, p2, my_tested, my_rejected, my_rmax);
  }
  __shared__ unsigned int s_tr[2];
  __shared__ unsigned long long s_rmax;
  if (threadIdx.x == 0) { s_tr[0] = s_tr[1] = 0; s_rmax = 0; }
  __syncthreads();
  atomicAdd(&s_tr[0], my_tested);
  atomicAdd(&s_tr[1], my_rejected);
  atomicMax(&s_rmax, (unsigned long long)__double_as_longlong(my_rmax));
  __syncthreads();
  if (threadIdx.x == 0) {
    atomicAdd(A.iter_tr, s_tr[0]);
    atomicAdd(A.iter_tr + 1, s_tr[1]);
    atomicMax(A.rmax_bits, s_rmax);
  }
}

template <int GMAX, int CH>
__global__ void __launch_bounds__(128) k_tile_finalize(const GatherArgs A, const TileArgs T) {
  constexpr int PS = partial_size(GMAX, CH);
  double my_rmax = 0.0;
  uint32_t my_tested = 0, my_rejected = 0;
  for (uint32_t h = blockIdx.x * blockDim.x + threadIdx.x; h < A.H; h += gridDim.x * blockDim.x) {
    const uint32_t pbase = T.hp_map[3 * (size_t)h], nch = T.hp_map[3 * (size_t)h + 1],
                   stride = T.hp_map[3 * (size_t)h + 2];
    uint32_t cnt[GMAX];
    double sm[CH][GMAX], sq[CH][GMAX];
    double p0 = 0.0, p1 = 0.0, p2 = 0.0;
#pragma unroll
    for (int g = 0; g < GMAX; ++g) {
      cnt[g] = 0;
#pragma unroll
      for (int c = 0; c < CH; ++c) sm[c][g] = sq[c][g] = 0.0;
    }
    for (uint32_t ch = 0; ch < nch; ++ch) {
      // 16-B loads of the (even-sized, 16-B aligned) row
      const double2 *pp2 = reinterpret_cast<const double2 *>(T.partials + ((size_t)pbase + (size_t)ch * stride) * PS);
      double pp[PS];
#pragma unroll
      for (int f = 0; f < PS / 2; ++f) {
        const double2 v = pp2[f];
        pp[2 * f] = v.x;
        pp[2 * f + 1] = v.y;
      }
#pragma unroll
      for (int g = 0; g < GMAX; ++g) cnt[g] += (uint32_t)pp[g];
#pragma unroll
      for (int c = 0; c < CH; ++c)
#pragma unroll
        for (int g = 0; g < GMAX; ++g) {
          sm[c][g] += pp[GMAX + c * GMAX + g];
          sq[c][g] += pp[GMAX + CH * GMAX + c * GMAX + g];
        }
      p0 += pp[GMAX + 2 * CH * GMAX];
      p1 += pp[GMAX + 2 * CH * GMAX + 1];
      p2 += pp[GMAX + 2 * CH * GMAX + 2];
    }
    finalize_hit<GMAX, CH>(A, h, cnt, sm, sq, p0, p1, p2, my_tested, my_rejected, my_rmax);
  }
  __shared__ unsigned int s_tr[2];
  __shared__ unsigned long long s_rmax;
  if (threadIdx.x == 0) { s_tr[0] = s_tr[1] = 0; s_rmax = 0; }
  __syncthreads();
  atomicAdd(&s_tr[0], my_tested);
  atomicAdd(&s_tr[1], my_rejected);
  atomicMax(&s_rmax, (unsigned long long)__double_as_longlong(my_rmax));
  __syncthreads();
  if (threadIdx.x == 0) {
    atomicAdd(A.iter_tr, s_tr[0]);
    atomicAdd(A.iter_tr + 1, s_tr[1]);
    atomicMax(A.rmax_bits, s_rmax);
  }
}


static inline unsigned blocks_for(unsigned long long n, int threads, int sms, int per_sm) {
  unsigned long long b = (n + threads - 1) / threads;
  const unsigned long long cap = (unsigned long long)sms * per_sm;
  if (b > cap) b = cap;
  return (unsigned)(b ? b : 1);
}

// Hit points sorted by home cell (k_hp_bin keys): the sparse kernel walks
// them in this order so a warp's hit points share candidate records.
cudaError_t hp_cell_order(cudaStream_t s, const GatherArgs &A, TileSched &S, const GridHeader &g, int sms,
                          const uint32_t **order) {
  S.bins_valid = false;  // the sort scratch is reused here
  const unsigned long long n_ext =
      (unsigned long long)(g.nx + 2) * (unsigned long long)(g.ny + 2) * (unsigned long long)(g.nz + 2);
  if (n_ext + 1 >= 0xffffffffull) return cudaErrorInvalidValue;
  const bool morton = g.nx + 2 <= 1024 && g.ny + 2 <= 1024 && g.nz + 2 <= 1024;
  const uint32_t none = morton ? (1u << 30) : (uint32_t)n_ext;
  k_hp_bin<<<blocks_for(A.H, 256, sms, 16), 256, 0, s>>>(A.pos, A.gathered, A.H, A.grid, none, morton ? 1 : 0,
                                                         S.sort.keys_a, S.sort.vals_a);
  note_launches(1);
  uint32_t bits = 1;
  while (bits < 32 && (1ull << bits) < (unsigned long long)none + 1) ++bits;
  uint32_t *skeys, *svals;
  cudaError_t e = radix_sort_pairs(s, S.sort, A.H, bits, &skeys, &svals);
  *order = svals;
  return e;
}


cudaError_t launch_bucket_start(cudaStream_t s, const uint32_t *skeys, uint32_t n, uint32_t nb,
                                uint32_t *start, int sms) {
  if ((unsigned long long)nb > 4ull * n)
    k_bucket_start_bsearch<<<blocks_for(nb + 1, 256, sms, 16), 256, 0, s>>>(skeys, n, nb, start);
  else
    k_bucket_start<<<blocks_for(n, 256, sms, 16), 256, 0, s>>>(skeys, n, nb, start);
  note_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_exclusive_scan(cudaStream_t s, const uint32_t *in, uint32_t n, uint32_t *tmp,
                                  uint32_t *out) {
  const uint32_t nt = (n + kScanTile - 1) / kScanTile;
  k_scan_tiles<<<nt, 256, 0, s>>>(in, n, tmp);
  k_scan_top<<<1, 256, 0, s>>>(tmp, nt);
  k_scan_apply<<<nt, 256, 0, s>>>(in, n, tmp, out);
  note_launches(3);
  return cudaGetLastError();
}


template <int GMAX, int CH>
static cudaError_t launch_fin(cudaStream_t s, const GatherArgs &A, const TileArgs &T, int sms) {
  if (A.H == 0) return cudaSuccess;
  if (T.contig) {
    const size_t smem = (size_t)4 * kFinChunk * partial_size(GMAX, CH) * sizeof(double);
    cudaError_t e = cudaFuncSetAttribute(k_tile_finalize_contig<GMAX, CH>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_tile_finalize_contig<GMAX, CH><<<blocks_for(A.H, 128, sms, 8), 128, smem, s>>>(A, T);
  } else {
    k_tile_finalize<GMAX, CH><<<blocks_for(A.H, 128, sms, 8), 128, 0, s>>>(A, T);
  }
  note_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_tile_finalize(cudaStream_t s, const GatherArgs &A, const TileArgs &T, int C,
                                 int sms) {
  // the fine kernel's instantiations (fine_supported: GMAX * C <= 24)
  const int G = A.na * A.ns;
  if (C == 1) {
    if (G <= 4) return launch_fin<4, 1>(s, A, T, sms);
    if (G <= 8) return launch_fin<8, 1>(s, A, T, sms);
    if (G <= 12) return launch_fin<12, 1>(s, A, T, sms);
    if (G <= 16) return launch_fin<16, 1>(s, A, T, sms);
    return cudaErrorInvalidValue;
  }
  if (G <= 4) return launch_fin<4, 3>(s, A, T, sms);
  if (G <= 8) return launch_fin<8, 3>(s, A, T, sms);
  return cudaErrorInvalidValue;
}

size_t tile_partial_doubles(int G, int C) {
  const int gmax = G <= 4 ? 4 : G <= 8 ? 8 : G <= 12 ? 12 : 16;
  return (size_t)partial_size(gmax, C) * 32;
}

}  // namespace fppm_b200
