// gather_fine.cu -- fine-cell tiled gather + F-test (the default kernel).
//
// Same work decomposition as gather_tile.cu -- item = (home reference cell,
// wave of <= 32 hit points, window of the wave's staged candidates) -- with
// three changes that cut the instruction count per accepted pair:
//
//  * fine culling.  The photon table is built on fine cells of size
//    cell / S (S = 4 when the photons span <= 3 reference cells in z, the
//    "slab" layout; grid.cu).  Every hit point tests only the fine cells of
//    its own bounding box [c - r, c + r] clipped to the reference
//    27-neighbourhood of its home cell (photon_map.cpp:65-77): the candidate
//    area follows the hit point's own radius instead of 9 r_max^2.  The wave
//    stages the union of its members' boxes (one contiguous piece per fine
//    row) with TMA bulk copies; each hit point walks its own runs inside it.
//  * specialised flush.  Hit points with n = +z, an fp32-exact center and
//    n_s = 4 (every canonical workload) take a flush that needs no frame
//    projection: plane coordinates are (dx, dy), guard and cos_i are p.n.z and
//    wi.z (exact when the other components are finite, precomputed flag), and
//    the photon luminance comes precomputed in fp64 from the record.
//  * shared-memory accumulators.  Each lane adds its pair's value into its own
//    (sector, lane) slot {sum, sum_sq} in shared memory (one LDS.128 + two
//    DADD + one STS.128 per pair instead of G predicated adds); per-sector
//    counts come from one ballot per sector per flush.  Slots are reduced in
//    a fixed order at the end of each fragment, so results are deterministic.
//
// Pairs whose fp32 predicates fall inside an error band are deferred to a
// per-warp list and decided on the exact fp64 path (exact_pair, gather_dev.cuh)
// outside the hot loop.  Partials and k_tile_finalize are shared with the
// tiled kernel.
#include <climits>
#include <type_traits>
#include <cstdlib>

#include "common.cuh"
#include "gather.cuh"
#include "gather_dev.cuh"

namespace fppm_b200 {

#ifndef FPPM_EXPERIMENT
#define FPPM_EXPERIMENT 0
#endif
#ifndef FPPM_FINE_WARPS
#define FPPM_FINE_WARPS 8
#endif
constexpr int kFWarps = FPPM_FINE_WARPS;
constexpr int kFThreads = kFWarps * kWarp;
constexpr int kFWave = 32;      // hit points per wave (= kWave of the partial layout)
constexpr int kFExact = 128;    // deferred exact pairs per warp (<= 31 + 64 pending)

__device__ __forceinline__ float4 lds128_f(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(addr));
  return v;
}

// Compact per-hit-point state staged in shared memory per item (the full
// Hit state stays in global memory for the exact path).
struct alignas(16) FineHot {
  HitF F;
  double K0, K1, K2;
  uint32_t planar, gray;
  int32_t bx0, by0, by1;  // fine box (fine_box); bx1, bz0, bz1 in the fbox array
  uint32_t nruns;
  uint2 run[kFMaxPieces];  // sorted-record range [begin, end) of each run (clipped to the chord)
  uint32_t mlim;           // lean layout: meta <= mlim <=> eye + depth <= max_depth (integrator.cpp:396)
  uint32_t pad_[3];        // ring schedule: row of window 0, first window, end window (k_fine_desc)
};
static_assert(sizeof(FineHot) % 16 == 0, "FineHot must be a multiple of 16 B (TMA)");

// Per hit point, once per gather, in wave order (position in hp_order): the
// staged state, its fine box and the sorted-record range of each run.
// Tiles of kPrepThreads hit points: the per-thread structs are assembled in
// shared memory and written out as contiguous 16-B vectors (coalesced).
constexpr int kPrepThreads = 128;
constexpr size_t kPrepSmem = (size_t)kPrepThreads * (sizeof(FineHot) + sizeof(Hit));
static_assert(sizeof(Hit) % 16 == 0, "Hit must be a multiple of 16 B");

static __device__ __forceinline__ void copy_out16(const void *src, void *dst, uint32_t bytes) {
  const int4 *s = static_cast<const int4 *>(src);
  int4 *d = static_cast<int4 *>(dst);
  for (uint32_t k = threadIdx.x; k < bytes / 16; k += blockDim.x) d[k] = s[k];
}

__global__ void __launch_bounds__(kPrepThreads)
    k_fine_prep(const GatherArgs A, const uint32_t *__restrict__ hp_order, FineHot *__restrict__ hot,
                int4 *__restrict__ fbox, Hit *__restrict__ hits) {
  extern __shared__ __align__(16) unsigned char prep_smem[];
  FineHot *s_hot = reinterpret_cast<FineHot *>(prep_smem);
  Hit *s_hit = reinterpret_cast<Hit *>(prep_smem + (size_t)kPrepThreads * sizeof(FineHot));
  const GridHeader g = *A.grid;
  for (uint32_t t0 = blockIdx.x * kPrepThreads; t0 < A.H; t0 += gridDim.x * kPrepThreads) {
    const uint32_t i = t0 + threadIdx.x;
    const uint32_t nt = min((uint32_t)kPrepThreads, A.H - t0);
    if (i < A.H) {
    const uint32_t h = hp_order[i];
    Hit P;
    make_hit(A, h, P);
    FBox b = {0, -1, 0, -1, 0, -1};
    const bool gathered = A.gathered == nullptr || A.gathered[h] != 0;
    const bool ok = gathered && fine_box(g, P.cx, P.cy, P.cz, P.r, b);
    const int nr = ok ? run_count(g, b) : 0;
    FineHot Q;
    Q.F = hitf(P, A.na, A.ns);
    Q.K0 = P.K0;
    Q.K1 = P.K1;
    Q.K2 = P.K2;
    // n = +z, fp32-exact center, 4 bins: the planar fast path (gather_dev.cuh)
    Q.planar = (P.fast && P.nx == 0.0 && P.ny == 0.0 && P.nz == 1.0 && A.ns == 4 &&
                P.clx == 0.0f && P.cly == 0.0f && P.clz == 0.0f) ? 1u : 0u;
    // bit0: K0 = K1 = K2; bit1: the lean path (planar, gray, finite K: the
    // lane slots hold photon-luminance moments, scaled by K0 at the end)
    Q.gray = (P.gray ? 1u : 0u) |
             ((Q.planar && P.gray && isfinite(P.K0) && A.na <= 2 && A.ns == 4 && P.eye <= A.max_depth) ? 2u : 0u);
    {
      // lean meta (lean_record): depth < 2^23 in bits 8..30, guard failure in bit 31
      unsigned long long dm_ = P.eye <= A.max_depth ? (unsigned long long)(A.max_depth - P.eye) : 0ull;
      if (dm_ > (1ull << 23) - 1) dm_ = (1ull << 23) - 1;
      Q.mlim = (uint32_t)((dm_ << 8) | 0xffu);
      Q.pad_[0] = Q.pad_[1] = Q.pad_[2] = 0u;
    }
    Q.bx0 = b.x0; Q.by0 = b.y0; Q.by1 = b.y1;
    fbox[i] = make_int4(b.x1, b.z0, b.z1, 0);
    Q.nruns = (uint32_t)nr;
    // runs clipped to the ball's chord (same margin radius as fine_box)
    const double cm = fmax(fabs(P.cx), fmax(fabs(P.cy), fabs(P.cz)));
    const double m = da(da(P.r, dm(P.r, 1e-9)), dm(cm, 4e-16));
    for (int j = 0; j < kFMaxPieces; ++j) {
      uint2 r = make_uint2(0u, 0u);
      unsigned long long k0, k1;
      if (j < nr && run_keys_clipped(g, b, j, P.cx, P.cy, P.cz, m, k0, k1))
        r = make_uint2(A.cell_start[k0], A.cell_start[k1 + 1]);
      Q.run[j] = r;
    }
    s_hot[threadIdx.x] = Q;
    s_hit[threadIdx.x] = P;
    }
    __syncthreads();
    copy_out16(s_hot, hot + t0, nt * (uint32_t)sizeof(FineHot));
    copy_out16(s_hit, hits + t0, nt * (uint32_t)sizeof(Hit));
    __syncthreads();
  }
}

// ------------------------------------------------------------------ scheduling
// bucket = home reference cell in the table's reference box extended by one
// cell on every side; key n_ext = "no candidates" (outside / not gathered /
// empty photon set).
struct RefBox {
  long long x0, y0, z0, ex, ey, ez;
};
static __device__ __forceinline__ RefBox ref_box(const GridHeader &g) {
  RefBox b;
  b.x0 = g.ix0 >> g.shift;
  b.y0 = g.iy0 >> g.shift;
  b.z0 = g.iz0 >> g.shift;
  b.ex = ((g.ix0 + g.nx - 1) >> g.shift) - b.x0 + 3;
  b.ey = ((g.iy0 + g.ny - 1) >> g.shift) - b.y0 + 3;
  b.ez = ((g.iz0 + g.nz - 1) >> g.shift) - b.z0 + 3;
  return b;
}

__global__ void k_fine_bin(const double3 *__restrict__ pos, const uint8_t *__restrict__ gathered,
                           uint32_t H, const GridHeader *__restrict__ hdr,
                           uint32_t *__restrict__ keys, uint32_t *__restrict__ vals) {
  const GridHeader g = *hdr;
  const RefBox rb = ref_box(g);
  const uint32_t n_ext = (uint32_t)(rb.ex * rb.ey * rb.ez);
  for (uint32_t h = blockIdx.x * blockDim.x + threadIdx.x; h < H; h += gridDim.x * blockDim.x) {
    uint32_t key = n_ext;
    const double3 c = pos[h];
    if (g.n > 0 && (gathered == nullptr || gathered[h])) {
      const double hx = dm(c.x, g.inv), hy = dm(c.y, g.inv), hz = dm(c.z, g.inv);
      if (fabs(hx) < 4.0e15 && fabs(hy) < 4.0e15 && fabs(hz) < 4.0e15) {
        const long long X = ((long long)floor(hx) >> g.shift) - rb.x0 + 1;
        const long long Y = ((long long)floor(hy) >> g.shift) - rb.y0 + 1;
        const long long Z = ((long long)floor(hz) >> g.shift) - rb.z0 + 1;
        if (X >= 0 && Y >= 0 && Z >= 0 && X < rb.ex && Y < rb.ey && Z < rb.ez)
          key = (uint32_t)((X * rb.ey + Y) * rb.ez + Z);
      }
    }
    keys[h] = key;
    vals[h] = h;
  }
}

// One wave of a bucket, evaluated by a full warp (lane j = member j): union of
// the members' fine boxes (from k_fine_prep), its pieces' key ranges (lane p
// = piece p), candidate total and whether every member takes the planar path.
struct WaveInfo {
  FBox u;
  int np;          // pieces (0: no member has candidates)
  uint32_t T;      // staged candidates (union size)
  uint32_t src;    // lane p: first sorted record of piece p
  uint32_t pre;    // lane p: exclusive offset of piece p
  bool planar;
};
static __device__ __forceinline__ WaveInfo wave_info(const GatherArgs &A, const GridHeader &g,
                                                     const FineHot *__restrict__ hot,
                                                     const int4 *__restrict__ fbox, uint32_t b0, uint32_t n,
                                                     bool real) {
  const int lane = threadIdx.x & 31;
  WaveInfo W;
  bool valid = false, pl = true;
  int x0 = INT_MAX, x1 = INT_MIN, y0 = INT_MAX, y1 = INT_MIN, z0 = INT_MAX, z1 = INT_MIN;
  if ((uint32_t)lane < n) {
    const FineHot &P = hot[b0 + lane];
    valid = real && P.nruns > 0;
    if (valid) {
      const int4 B = fbox[b0 + lane];
      x0 = P.bx0; x1 = B.x; y0 = P.by0; y1 = P.by1; z0 = B.y; z1 = B.z;
    }
    pl = P.planar != 0u;
  }
  W.planar = __all_sync(kFull, pl);
  W.u.x0 = __reduce_min_sync(kFull, x0); W.u.x1 = __reduce_max_sync(kFull, x1);
  W.u.y0 = __reduce_min_sync(kFull, y0); W.u.y1 = __reduce_max_sync(kFull, y1);
  W.u.z0 = __reduce_min_sync(kFull, z0); W.u.z1 = __reduce_max_sync(kFull, z1);
  W.np = __any_sync(kFull, valid) ? piece_count(g, W.u) : 0;
  uint32_t c = 0;
  W.src = 0;
  if (lane < W.np) {
    unsigned long long k0, k1;
    piece_keys(g, W.u, lane, k0, k1);
    W.src = A.cell_start[k0];
    c = A.cell_start[k1 + 1] - W.src;
  }
  uint32_t incl = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(kFull, incl, o);
    if (lane >= o) incl += y;
  }
  W.pre = incl - c;
  W.T = __shfl_sync(kFull, incl, 31);
  if (W.np == 0) W.u = FBox{0, -1, 0, -1, 0, -1};
  return W;
}

// Ring schedule: the windows [c_first, c_first + nc) of a wave that hold a
// member's candidates (lane j = member j, W from wave_info): its runs mapped
// into the union's flattened order (min / max over runs), divided by the
// window capacity.  nc = 0: no candidates.
static __device__ __forceinline__ void member_windows(const GridHeader &g, const FineHot *__restrict__ hot,
                                                      uint32_t b0, uint32_t n, const WaveInfo &W, uint32_t chunk,
                                                      uint32_t &c_first, uint32_t &nc, uint32_t *span = nullptr) {
  const int lane = threadIdx.x & 31;
  uint32_t fmin = 0xffffffffu, fmax = 0u;
  const bool mine = (uint32_t)lane < n;
  const FineHot *P = mine ? &hot[b0 + lane] : nullptr;
  const int nr = mine && W.np > 0 ? (int)P->nruns : 0;
#pragma unroll 1
  for (int r = 0; r < kFMaxPieces; ++r) {
    int pc = 0;
    if (r < nr) {
      if (slab_grid(g)) {
        pc = P->bx0 + r - W.u.x0;
      } else {
        const int nyb = P->by1 - P->by0 + 1, nyu = W.u.y1 - W.u.y0 + 1;
        pc = (P->bx0 + r / nyb - W.u.x0) * nyu + (P->by0 + r % nyb - W.u.y0);
      }
    }
    const uint32_t pre = __shfl_sync(kFull, W.pre, pc & 31), src = __shfl_sync(kFull, W.src, pc & 31);
    if (r < nr) {
      const uint2 R = P->run[r];
      if (R.y > R.x) {
        const uint32_t fa = pre + (R.x - src);
        fmin = min(fmin, fa);
        fmax = max(fmax, fa + (R.y - R.x));
      }
    }
  }
  if (fmin < fmax) {
    c_first = fmin / chunk;
    nc = (fmax - 1) / chunk - c_first + 1;
  } else {
    c_first = 0;
    nc = 0;
  }
  if (span) {
    span[0] = fmin;
    span[1] = fmax;
  }
}

// Warp-wide bitonic sort of one key per lane, descending.
static __device__ __forceinline__ uint32_t warp_sort_desc(uint32_t key) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 2; k <= 32; k <<= 1)
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      const uint32_t other = __shfl_xor_sync(kFull, key, j);
      const bool lower = (lane & j) == 0, desc = (lane & k) == 0;
      key = (lower == desc) ? max(key, other) : min(key, other);
    }
  return key;
}

// per bucket (one warp each): items (runs of <= fsub windows of
// ceil(union / chunk)) and partial rows (items x wave size)
__global__ void k_fine_items(const GatherArgs A, const uint32_t *__restrict__ hp_start, uint32_t nb,
                             const FineHot *__restrict__ hot, const int4 *__restrict__ fbox,
                             uint32_t *__restrict__ items, uint32_t *__restrict__ prows, uint32_t cap64,
                             uint32_t cap48, uint32_t fsub, uint32_t *__restrict__ nonempty,
                             const uint32_t *__restrict__ hp_order, uint32_t *__restrict__ hp_nc) {
  const GridHeader g = *A.grid;
  const int lane = threadIdx.x & 31;
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t b = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; b <= nb; b += nw) {
    const uint32_t h0 = b < nb ? hp_start[b] : 0u;
    const uint32_t nhp = b < nb ? hp_start[b + 1] - h0 : 0u;
    uint32_t it = 0, pr = 0;
    if (nhp && lane == 0) atomicAdd(nonempty, 1u);
    for (uint32_t w = 0; w * kFWave < nhp; ++w) {
      const uint32_t n = min((uint32_t)kFWave, nhp - w * kFWave);
      const WaveInfo W = wave_info(A, g, hot, fbox, h0 + w * kFWave, n, b + 1 < nb);
      const uint32_t chunk = (W.planar || g.lean) ? cap48 : cap64;
      const uint32_t nwin = W.T == 0 ? 1u : (W.T + chunk - 1) / chunk;
      const uint32_t nsub = (nwin + fsub - 1) / fsub;
      it += nsub;
      if (fsub == 1) {  // ring: one row per (hit point, window it has candidates in)
        uint32_t c_first, nc;
        member_windows(g, hot, h0 + w * kFWave, n, W, chunk, c_first, nc);
        pr += __reduce_add_sync(kFull, nc);
        if ((uint32_t)lane < n) hp_nc[hp_order[h0 + w * kFWave + lane]] = nc;  // rows in hit-point order
      } else {
        pr += nsub * n;
      }
    }
    if (lane == 0) {
      items[b] = it;
      prows[b] = pr;
    }
  }
}

__global__ void k_fine_desc(const GatherArgs A, const uint32_t *__restrict__ hp_start, uint32_t nb,
                            const uint32_t *__restrict__ hp_order, FineHot *__restrict__ hot,
                            const int4 *__restrict__ fbox, const uint32_t *__restrict__ item_base,
                            const uint32_t *__restrict__ prow_base, FineDesc *__restrict__ desc,
                            uint32_t *__restrict__ hp_map, uint32_t cap64, uint32_t cap48, uint32_t fsub,
                            const uint32_t *__restrict__ hp_rbase, uint2 *__restrict__ hp_span,
                            unsigned long long item_cap) {
  constexpr int kWarps = 4;  // 128 threads
  constexpr int kWords = (int)(sizeof(FineDesc) / 4);
  __shared__ __align__(16) uint32_t s_d[kWarps][kWords];
  const GridHeader g = *A.grid;
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  FineDesc &d = *reinterpret_cast<FineDesc *>(&s_d[wl][0]);  // (d.pbase unused by the ring)
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t b = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; b < nb; b += nw) {
    const uint32_t h0 = hp_start[b], nhp = hp_start[b + 1] - h0;
    uint32_t item = item_base[b], prow = prow_base[b];
    for (uint32_t w = 0; w * kFWave < nhp; ++w) {
      const uint32_t n = min((uint32_t)kFWave, nhp - w * kFWave);
      const uint32_t lo = h0 + w * kFWave;
      const WaveInfo W = wave_info(A, g, hot, fbox, lo, n, b + 1 < nb);
      const uint32_t chunk = (W.planar || g.lean) ? cap48 : cap64;
      const uint32_t nwin = W.T == 0 ? 1u : (W.T + chunk - 1) / chunk;
      const uint32_t nsub = (nwin + fsub - 1) / fsub;
      __syncwarp();
      if (lane < kFMaxPieces) {
        d.src[lane] = lane < W.np ? W.src : 0u;
        d.pre[lane] = lane < W.np ? W.pre : W.T;
      }
      if (lane == 0) {
        d.hp_lo = lo;
        d.hp_n = n;
        d.nwin = nwin;
        d.npieces = (uint32_t)W.np;
        d.pre[kFMaxPieces] = W.T;
        d.pad0 = (W.planar || g.lean) ? 1u : 0u;  // flags: bit0 = 48-B records (no rec3 staged)
        d.ux0 = W.u.x0; d.ux1 = W.u.x1; d.uy0 = W.u.y0; d.uy1 = W.u.y1; d.uz0 = W.u.z0; d.uz1 = W.u.z1;
      }
      uint32_t rows_used = nsub * n;
      uint32_t m_span[2] = {0u, 0u};  // ring: this lane's member span (k_fine_order)
      if (fsub == 1) {
        // ring: member j's rows are contiguous, one per window of its range,
        // allocated in hit-point order (scan of k_fine_items' counts) so the
        // finalize reads them coalesced; the fragment of window c writes row
        // pad_[0] + c (FineHot, staged by TMA)
        uint32_t c_first, nc;
        member_windows(g, hot, lo, n, W, chunk, c_first, nc, m_span);
        if ((uint32_t)lane < n) hp_span[lo + lane] = make_uint2(m_span[0], m_span[1]);
        rows_used = __reduce_add_sync(kFull, nc);
        if ((uint32_t)lane < n) {
          const uint32_t h = hp_order[lo + lane];
          const uint32_t r0 = hp_rbase[h];
          hp_map[3 * (size_t)h] = r0;  // finalize: rows r0 .. r0 + nc - 1
          hp_map[3 * (size_t)h + 1] = nc;
          hp_map[3 * (size_t)h + 2] = 1u;
          hot[lo + lane].pad_[0] = r0 - c_first;
          hot[lo + lane].pad_[1] = c_first;
          hot[lo + lane].pad_[2] = c_first + nc;
        }
      } else if ((uint32_t)lane < n) {
        const uint32_t h = hp_order[lo + lane];
        hp_map[3 * (size_t)h] = prow + lane;  // finalize: rows prow + j + sub * n
        hp_map[3 * (size_t)h + 1] = nsub;
        hp_map[3 * (size_t)h + 2] = n;
      }
      __syncwarp();
      for (uint32_t sb = 0; sb < nsub; ++sb, ++item) {
        if (lane == 0) {
          d.c0 = sb * fsub;
          d.c1 = min(nwin, d.c0 + fsub);
          d.pbase = prow + sb * n;
        }
        if (lane == 0) d.nclaim = n;  // ring: claim order filled by k_fine_order
        __syncwarp();
        if (item < item_cap) {  // a speculative build skips items past the capacity (the host rebuilds)
          uint32_t *dst = reinterpret_cast<uint32_t *>(desc + item);
          for (int k = lane; k < kWords; k += 32) dst[k] = s_d[wl][k];
        }
        __syncwarp();
      }
      prow += rows_used;
    }
  }
}

// Ring schedule: one warp per item (= one window c of a wave) orders the
// wave's hit points for claiming: those whose window range holds c, the
// largest share of the window first (span [first run, last run) of the hit
// point clipped to the window -- a proxy of its fragment), ties by index.
// Longest-first claiming shortens the tail of an item, and the buffer is
// released (refilled) when the last warp leaves it.
__global__ void __launch_bounds__(128) k_fine_order(FineDesc *__restrict__ desc, const uint32_t *__restrict__ total,
                                                    const FineHot *__restrict__ hot, const uint2 *__restrict__ hp_span,
                                                    uint32_t cap, unsigned long long item_cap) {
  const int lane = threadIdx.x & 31;
  const uint32_t nitems = (uint32_t)min((unsigned long long)*total, item_cap);
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t it = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; it < nitems; it += nw) {
    FineDesc &D = desc[it];
    const uint32_t hp_lo = D.hp_lo, n = D.hp_n, c = D.c0, T = D.pre[kFMaxPieces];
    uint32_t key = 0;
    if ((uint32_t)lane < n) {
      const FineHot &P = hot[hp_lo + lane];
      if (c >= P.pad_[1] && c < P.pad_[2]) {
        const uint2 sp = hp_span[hp_lo + lane];
        const uint32_t wlo = c * cap, whi = min(T, wlo + cap);
        const uint32_t sa = max(sp.x, wlo), se = min(sp.y, whi);
        const uint32_t cnt = se > sa ? se - sa : 0u;
        key = ((min(cnt, 0x3fffffu) + 1u) << 5) | (31u - (uint32_t)lane);
      }
    }
    const uint32_t sorted = warp_sort_desc(key);
    const uint32_t ncl = __popc(__ballot_sync(kFull, key != 0u));
    D.order[lane] = (uint8_t)(31u - (sorted & 31u));
    if (lane == 0) D.nclaim = ncl;
  }
}

// ------------------------------------------------------------------ kernel
template <int GMAX, int CH>
struct FineLayout {
  static constexpr int NC = GMAX * CH;                  // accumulator columns
  static constexpr int NQ = 32 / NC;                    // lane groups in the slot reduction
  static constexpr int PS = partial_size(GMAX, CH);
  // lane slots [NC + 1][32] {sum, sum_sq} per warp; row NC: the lean path's
  // spare row for rejected pairs (never reduced)
  static constexpr size_t kSlotBytes = (size_t)kFWarps * (NC + 1) * 32 * 16;
  static constexpr size_t kHotBytes = (size_t)kFWave * sizeof(FineHot);
  // the item's partial rows, accumulated in shared memory over its windows
  // and written out once at the end of the item
  static constexpr size_t kRowBytes = (size_t)kFWave * PS * 8;
  static constexpr int kMinBlocks = NC <= 8 ? 2 : 1;
  // dynamic shared memory: records + lane slots + staged hit points;
  // kMinBlocks CTAs share the SM's 228 KB, each with 1 KB reserved and the
  // static arrays of the kernel
  static constexpr size_t kStatic = (size_t)kFWarps * kFExact * 4 + 2 * sizeof(FineDesc) + 64;
  static constexpr size_t kBudget = (size_t)233472 / kMinBlocks - 1024 - kStatic - 256;
  static constexpr size_t kRecBytes = kBudget - kSlotBytes - kHotBytes - kRowBytes;
  // window capacity: 64 B per candidate, or 48 B for planar waves (no rec3)
  static constexpr uint32_t kCap64 = (uint32_t)((kRecBytes / 64) & ~(size_t)31);
  static constexpr uint32_t kCap48 = (uint32_t)((kRecBytes / 48) & ~(size_t)31);
  static constexpr size_t kDynBytes = kRecBytes + kSlotBytes + kHotBytes + kRowBytes;
};

struct FineState {
  uint32_t eh, et, pad0, pad1;  // exact ring (warp-uniform)
  uint32_t n_cand, n_exact, n_amb, n_acc;
};

// Per-hit-point weights held in registers for the fragment.
struct HitV {
  double K0, K1, K2;
  double Kz, Kz0, Kz1, Kz2;  // value of an accepted pair with cos_i <= 0 (K * 0: NaN for inf K)
  bool gray;
};

// Per-sector pair counts of one lane, packed as bytes (a lane adds at most
// one pair per flush or exact batch: <= 2 * chunk / 32 < 256 per fragment).
template <int GMAX>
struct PackedCounts {
  static constexpr int NP = (GMAX + 3) / 4;
  uint32_t w[NP];
};
#define FPPM_PK_CASE(r)                                                          \
  if constexpr ((r) < PackedCounts<GMAX>::NP) {                                  \
    if ((sector >> 2) == (r)) asm("add.u32 %0, %0, %1; // pk " #r : "+r"(c.w[r]) : "r"(inc)); \
  }
template <int GMAX>
static __device__ __forceinline__ void pk_add(PackedCounts<GMAX> &c, int sector) {
  if constexpr (GMAX == 8) {
    // one 64-bit shift-add over the two words
    unsigned long long wd = ((unsigned long long)c.w[1] << 32) | c.w[0];
    wd += 1ull << (sector * 8);
    c.w[0] = (uint32_t)wd;
    c.w[1] = (uint32_t)(wd >> 32);
  } else {
    const uint32_t inc = 1u << ((sector & 3) * 8);
    FPPM_PK_CASE(0) FPPM_PK_CASE(1) FPPM_PK_CASE(2) FPPM_PK_CASE(3)
  }
}
#undef FPPM_PK_CASE

static __device__ __forceinline__ void sts_u32(uint32_t addr, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
static __device__ __forceinline__ uint32_t lds_u32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
  return v;
}
static __device__ __forceinline__ double2 lds_f64x2(uint32_t addr) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(addr) : "memory");
  return v;
}
static __device__ __forceinline__ void sts_f64x2(uint32_t addr, double2 v) {
  asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(addr), "d"(v.x), "d"(v.y) : "memory");
}

// Value of an accepted pair (integrator.cpp:445-451, gather.cpp:59-67) added
// to the lane's (sector, lane) slot; flux sums; packed sector counts.
// Branch-free: a lane without an accepted pair adds zeros to a valid slot.
// slots = shared address of this warp's [C][GMAX][32] {sum, sum_sq} slots.
// GRAY: K0 = K1 = K2, so lum(K * pow) is taken as K0 * lum(pow) with the
// photon luminance precomputed in fp64 (same value to ~1 ulp).
template <int GMAX, int CH, bool GRAY>
static __device__ __forceinline__ void fine_accumulate(const HitV &K, bool acc, bool cos_pos, int sector,
                                                       float4 pw, double L, uint32_t slots, int lane,
                                                       PackedCounts<GMAX> &cnt, double &p0, double &p1,
                                                       double &p2) {
  const bool on = acc && cos_pos;
  const double pr = (double)pw.x, pg = (double)pw.y, pb = (double)pw.z;
#if FPPM_EXPERIMENT != 3
  if (on) {  // predicated: flux sums (integrator.cpp:449)
    p0 += pr;
    p1 += pg;
    p2 += pb;
  }
#endif
#if FPPM_EXPERIMENT != 4
  if (acc) pk_add<GMAX>(cnt, sector);
#endif
  if constexpr (CH == 1) {
    double v;
    if constexpr (GRAY) {
      const double kv = cos_pos ? dm(K.K0, L) : K.Kz;  // bsdf.cpp:58: f = 0 when cos_i <= 0
      v = acc ? kv : 0.0;
    } else {
      const double kv = cos_pos ? elum(dm(K.K0, pr), dm(K.K1, pg), dm(K.K2, pb)) : K.Kz;  // pr.. unselected: cos_pos
      v = acc ? kv : 0.0;
    }
    const uint32_t a = slots + (uint32_t)(sector * 32 + lane) * 16u;
    double2 o = lds_f64x2(a);
    o.x = da(o.x, v);          // SectorStats::add: sum += v; sum_sq += v * v
    o.y = da(o.y, dm(v, v));   // (stat_tests.hpp:18-22), v * v rounded alone
    sts_f64x2(a, o);
  } else {
    const double v[3] = {acc ? (cos_pos ? dm(K.K0, pr) : K.Kz0) : 0.0,
                         acc ? (cos_pos ? dm(K.K1, pg) : K.Kz1) : 0.0,
                         acc ? (cos_pos ? dm(K.K2, pb) : K.Kz2) : 0.0};
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const uint32_t a = slots + (uint32_t)((c * GMAX + sector) * 32 + lane) * 16u;
      double2 o = lds_f64x2(a);
      o.x = da(o.x, v[c]);
      o.y = da(o.y, dm(v[c], v[c]));
      sts_f64x2(a, o);
    }
  }
}

// Where the staged window lives: smem addresses of the record arrays and,
// for 48-B windows, how to find rec3 of a candidate in global memory.
struct FineWin {
  uint32_t r0, r1, r2, r3;  // r3 = 0: rec3 not staged
  uint32_t lo;               // window start in the union's flattened order
  const FineDesc *d;
  const float4 *grec3;
};

// One fp64-exact evaluation of a deferred pair (fine record layout -> the
// tile layout expected by exact_pair).
static __device__ __forceinline__ uint32_t fine_exact(const Hit &Hs, const FineWin &Wn, uint32_t i, int na,
                                                      int ns, double guard, float4 &pw, double &L) {
  const float4 a = lds128_f(Wn.r0 + i * 16u), B = lds128_f(Wn.r1 + i * 16u), Cc = lds128_f(Wn.r2 + i * 16u);
  float4 D;
  if (Wn.r3) {
    D = lds128_f(Wn.r3 + i * 16u);
  } else {  // flattened position -> piece -> sorted record
    const uint32_t f = i + Wn.lo;
    uint32_t p = 0;
    while (p + 1 < Wn.d->npieces && Wn.d->pre[p + 1] <= f) ++p;
    D = Wn.grec3[Wn.d->src[p] + (f - Wn.d->pre[p])];
  }
  pw = Cc;
  L = __longlong_as_double(((long long)__float_as_uint(B.w) << 32) | __float_as_uint(B.z));
  const float4 b_old = make_float4(D.x, D.y, B.x, D.z);
  const float4 c2_old = make_float4(D.w, B.y, Cc.x, Cc.y);
  return exact_pair_packed(Hs, a, b_old, c2_old, na, ns, guard);
}

template <int GMAX, int CH, bool GRAY>
static __device__ __forceinline__ void fine_exact_batch(const GatherArgs &A, const Hit &Hs, const HitV &K,
                                                     uint32_t n, uint32_t ex, uint32_t slots,
                                                     PackedCounts<GMAX> &cnt, double &p0, double &p1,
                                                     double &p2, const FineWin &Wn, FineState &st) {
  const int lane = threadIdx.x & 31;
  __syncwarp();
  const bool have = (uint32_t)lane < n;
  const uint32_t i = have ? lds_u32(ex + ((st.eh + lane) & (kFExact - 1)) * 4u) : 0u;
  st.eh += n;
  float4 pw = make_float4(0.f, 0.f, 0.f, 0.f);
  double L = 0.0;
  uint32_t fl = 0;
  if (have) {
    fl = fine_exact(Hs, Wn, i, A.na, A.ns, A.guard, pw, L);
    st.n_exact += 1;
    st.n_amb += (fl >> 2) & 1u;
  }
  fine_accumulate<GMAX, CH, GRAY>(K, (fl & 1u) != 0, (fl & 2u) != 0, (int)(fl >> 8), pw, L, slots, lane, cnt,
                                  p0, p1, p2);
  __syncwarp();
}

// Full fp32 evaluation of candidate i against the hit point (ball, depth,
// guard, disk, sector, cos_i; integrator.cpp:394-401, gather.cpp:15-33).
// acc: certainly accepted; need: inside an error band -> exact fp64 path.
template <bool PLANAR>
static __device__ __forceinline__ void fine_eval(const HitF &F, bool lo_zero, uint32_t max_depth, bool valid,
                                                 uint32_t i, uint32_t r0, uint32_t r1, uint32_t r2,
                                                 uint32_t r3, bool &acc, bool &need, bool &cos_pos,
                                                 int &sector, float4 &pw, double &L) {
  const float4 p = lds128_f(r0 + i * 16u);
  const float4 B = lds128_f(r1 + i * 16u);
  pw = lds128_f(r2 + i * 16u);
  L = __longlong_as_double(((long long)__float_as_uint(B.w) << 32) | __float_as_uint(B.z));
  const bool dep_ok = F.eye + __float_as_uint(p.w) <= max_depth;  // integrator.cpp:396
  if constexpr (PLANAR) {
    // n = +z: y = (dx, dy) exactly; guard = p.n.z, cos_i = wi.z (finite flag)
    const float dx = p.x - F.chx, dy = p.y - F.chy, dz = p.z - F.chz;
    const float yy = fmaf(dx, dx, dy * dy);
    const float d2 = fmaf(dz, dz, yy);
    const bool maybe = valid && dep_ok && d2 <= F.lim_hi;  // photon_map.cpp:76 (certain reject above)
    bool band = !(d2 < F.lim_lo) || !(fabsf(dx) > F.band_y) || !(fabsf(dy) > F.band_y) ||
                (__float_as_uint(pw.w) & 1u) == 0u;
    const int quad = dx > 0.0f ? (dy > 0.0f ? 0 : 3) : (dy > 0.0f ? 1 : 2);
    int ring = 0;
    if (F.na == 2) {  // one annulus edge at d2 = r2 / 2
      const float qa = yy * F.qa_scale;
      band = band || fabsf(qa - 1.0f) < 2e-4f;
      ring = qa >= 1.0f ? 1 : 0;
    } else if (F.na > 2) {
      const float qa = yy * F.qa_scale;
      const float kq = rintf(qa);
      band = band || (kq >= 1.0f && kq <= (float)(F.na - 1) && fabsf(qa - kq) < 1e-4f * (float)F.na);
      ring = min((int)qa, F.na - 1);
    }
    sector = ring * 4 + quad;
    cos_pos = !(B.y <= 0.0f);                        // bsdf.cpp:56-58
    need = maybe && band;
    acc = maybe && !band && !(B.x < F.guard_ceil);   // integrator.cpp:397
  } else {
    const float4 D = lds128_f(r3 + i * 16u);
    float dx = p.x - F.chx, dy = p.y - F.chy, dz = p.z - F.chz;
    if (!lo_zero) {
      dx -= F.clx;
      dy -= F.cly;
      dz -= F.clz;
    }
    const float d2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
    const float yu = fmaf(dx, F.ufx, fmaf(dy, F.ufy, dz * F.ufz));
    const float yv = fmaf(dx, F.vfx, fmaf(dy, F.vfy, dz * F.vfz));
    const float yy = fmaf(yu, yu, yv * yv);
    const bool maybe = valid && dep_ok && d2 <= F.lim_hi && yy <= F.lim_hi;  // ball, disk
    bool band = !(F.fast && d2 < F.lim_lo && yy < F.lim_lo);
    band = !fast_sector(F, yu, yv, yy, sector) || band;
    const float gd = fmaf(D.x, F.nfx, fmaf(D.y, F.nfy, B.x * F.nfz));
    const float gb = 2e-6f * (fabsf(D.x * F.nfx) + fabsf(D.y * F.nfy) + fabsf(B.x * F.nfz)) + 1e-30f;
    const bool guard_ok = !(gd < F.guard_f - gb);
    band = band || (guard_ok && !(gd >= F.guard_f + gb));
    const float ci = fmaf(D.z, F.nfx, fmaf(D.w, F.nfy, B.y * F.nfz));
    const float cb = 2e-6f * (fabsf(D.z * F.nfx) + fabsf(D.w * F.nfy) + fabsf(B.y * F.nfz)) + 1e-30f;
    band = band || !(fabsf(ci) > cb);
    cos_pos = ci > 0.0f;
    need = maybe && band;
    acc = maybe && !band && guard_ok;
  }
}

// All candidates of one hit point inside the staged window, one per lane per
// step (no compaction: at the fine boxes' pass rates a survivor queue costs
// more than the idle lanes).  Runs are held by lanes (lane j: smem start rs,
// length rl of run j).
template <int GMAX, int CH, bool PLANAR, bool GRAY>
static __device__ __forceinline__ void fine_fragment(const GatherArgs &A, const FineHot &Hh, const Hit &Hs,
                                                     uint32_t rs, uint32_t rl, int nruns, uint32_t ex,
                                                     uint32_t slots, PackedCounts<GMAX> &cnt, double &p0,
                                                     double &p1, double &p2, const FineWin &Wn,
                                                     FineState &st) {
  const int lane = threadIdx.x & 31;
  const uint32_t lt = (1u << lane) - 1u;
  const HitF F = Hh.F;
  const uint32_t r0 = Wn.r0, r1 = Wn.r1, r2 = Wn.r2, r3 = Wn.r3;
  HitV K;
  K.K0 = Hh.K0;
  K.K1 = Hh.K1;
  K.K2 = Hh.K2;
  K.gray = GRAY;
  K.Kz0 = dm(Hh.K0, 0.0);
  K.Kz1 = dm(Hh.K1, 0.0);
  K.Kz2 = dm(Hh.K2, 0.0);
  K.Kz = elum(K.Kz0, K.Kz1, K.Kz2);
  const uint32_t max_depth = A.max_depth;
  const bool lo_zero = PLANAR || (F.clx == 0.0f && F.cly == 0.0f && F.clz == 0.0f);
  // Runs are concatenated into one virtual index space [0, total) walked 64
  // slots per step with no per-run tails: lane j holds the inclusive end
  // `incl` of run j and the offset smem index - virtual index of that run.
  uint32_t incl = rl;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(kFull, incl, o);
    if (lane >= o) incl += y;
  }
  const uint32_t off = rs - (incl - rl);
  const uint32_t total = __shfl_sync(kFull, incl, 31);
  if (lane == 0) st.n_cand += total;
  int jlo = 0;  // first run ending after `base` (warp-uniform)
  for (uint32_t base = 0; base < total; base += 64) {
    while (__shfl_sync(kFull, incl, jlo) <= base) ++jlo;
    const uint32_t v0 = base + lane, v1 = v0 + 32;
    int j0 = jlo, j1 = jlo;
    for (int k = jlo; k < nruns; ++k) {  // run ends inside this step
      const uint32_t e = __shfl_sync(kFull, incl, k);
      if (e >= base + 64) break;
      j0 += e <= v0 ? 1 : 0;
      j1 += e <= v1 ? 1 : 0;
    }
    const bool ok0 = v0 < total, ok1 = v1 < total;
    const uint32_t o0 = __shfl_sync(kFull, off, j0 & 31), o1 = __shfl_sync(kFull, off, j1 & 31);
    const uint32_t i0 = ok0 ? v0 + o0 : rs, i1 = ok1 ? v1 + o1 : rs;
    bool acc0, need0, cp0, acc1, need1, cp1;
    int sec0, sec1;
    float4 pw0, pw1;
    double L0, L1;
#if FPPM_EXPERIMENT == 2  // timing experiment: loads only
    {
      const float4 q0 = lds128_f(r0 + i0 * 16u), q1 = lds128_f(r0 + i1 * 16u);
      acc0 = ok0 && q0.x > F.chx; acc1 = ok1 && q1.x > F.chx;
      need0 = need1 = false; cp0 = cp1 = true; sec0 = sec1 = 0;
      pw0 = pw1 = make_float4(0.f, 0.f, 0.f, 0.f); L0 = L1 = 0.0;
    }
#else
    fine_eval<PLANAR>(F, lo_zero, max_depth, ok0, i0, r0, r1, r2, r3, acc0, need0, cp0, sec0, pw0, L0);
    fine_eval<PLANAR>(F, lo_zero, max_depth, ok1, i1, r0, r1, r2, r3, acc1, need1, cp1, sec1, pw1, L1);
#endif
#if FPPM_EXPERIMENT >= 1  // timing experiment: no accumulation
    if (acc0) pk_add<GMAX>(cnt, sec0);
    if (acc1) pk_add<GMAX>(cnt, sec1);
#else
    fine_accumulate<GMAX, CH, GRAY>(K, acc0, cp0, sec0, pw0, L0, slots, lane, cnt, p0, p1, p2);
    fine_accumulate<GMAX, CH, GRAY>(K, acc1, cp1, sec1, pw1, L1, slots, lane, cnt, p0, p1, p2);
#endif
    // banded pairs (rare) go to the exact ring
    const uint32_t m0 = __ballot_sync(kFull, need0), m1 = __ballot_sync(kFull, need1);
    if (m0 | m1) {
      if (need0) sts_u32(ex + ((st.et + __popc(m0 & lt)) & (kFExact - 1)) * 4u, i0);
      st.et += __popc(m0);
      if (need1) sts_u32(ex + ((st.et + __popc(m1 & lt)) & (kFExact - 1)) * 4u, i1);
      st.et += __popc(m1);
      while (st.et - st.eh >= 32)
        fine_exact_batch<GMAX, CH, GRAY>(A, Hs, K, 32u, ex, slots, cnt, p0, p1, p2, Wn, st);
    }
  }
  while (st.et != st.eh)
    fine_exact_batch<GMAX, CH, GRAY>(A, Hs, K, min(32u, st.et - st.eh), ex, slots, cnt, p0, p1, p2, Wn, st);
  __syncwarp();
}


// ------------------------------------------------------------------ lean path
// Lean record layout (GridHeader::lean, common.cuh): every gathered hit point
// of the frame is planar and gray, C = 1, n_a <= 2, n_s = 4 -- every
// canonical workload.  A record is 48 B: (x, y, z, meta) with depth, guard
// and cos_i bits precomputed for n = +z, then (L, b) and (r, g) in fp64, so a
// pair needs no conversions.  The pair value is v = K0 * L, so a lane's slot
// accumulates the photon moments {sum L, sum L^2} of its accepted pairs and
// the fragment's sector sums are K0 * sum L and K0^2 * sum L^2
// (SectorStats::add, stat_tests.hpp:18-22; equal to the per-pair products up
// to fp64 reassociation, within the 1e-12 sum tolerance).  Per-sector counts
// are nibbles of one register per candidate slot (sector s at bits 4s..4s+3),
// spilled to byte words every 15 steps.  Pairs inside an fp32 error band take
// the exact fp64 path on the input photon (order[] -> fppm_photons arrays).
struct LeanCnt {
  uint32_t n0, n1, be, bo;  // nibble counts (candidate 0 / 1 of a step); byte words: sectors 0,2,4,6 / 1,3,5,7
};
static __device__ __forceinline__ void lean_spill(LeanCnt &c) {
  c.be += (c.n0 & 0x0F0F0F0Fu) + (c.n1 & 0x0F0F0F0Fu);
  c.bo += ((c.n0 >> 4) & 0x0F0F0F0Fu) + ((c.n1 >> 4) & 0x0F0F0F0Fu);
  c.n0 = c.n1 = 0u;
}

struct LeanPair {
  bool acc, need;
  uint32_t s4;  // 4 * sector
  double L, r, g, b;
};

// Hit-point constants of the lean loop.
struct LeanHit {
  float chx, chy, chz, lim_hi, lim_lo, band_y, qa_edge, qa_eps;  // annulus edge yy = r2 / 2 and its band
                                                                 // (FLAT: chz holds dz = zflat - centre z)
  uint32_t mlim;
};

// fp32 evaluation of one candidate (records at a0, a0 + d1, a0 + d2): ball,
// depth, guard, disk, annulus, quadrant, cos_i with the error bands of
// fine_eval<PLANAR>; band or exact-flagged photons -> need.
template <int NA, bool FLAT>
static __device__ __forceinline__ LeanPair lean_eval(const LeanHit &F, bool valid, uint32_t a0, uint32_t d1,
                                                     uint32_t d2) {
  LeanPair q;
  const float4 p = lds128_f(a0);
  float dz;
  uint32_t meta;
  if constexpr (FLAT) {  // (x, y, meta, r) | (L, g, b): the power widens exactly
    const float4 w = lds128_f(a0 + d1);
    q.L = __hiloint2double(__float_as_int(w.y), __float_as_int(w.x));
    q.r = (double)p.w;
    q.g = (double)w.z;
    q.b = (double)w.w;
    dz = F.chz;  // zflat - centre z, the same subtraction for every record
    meta = __float_as_uint(p.z);
  } else {
    const double2 LB = lds_f64x2(a0 + d1);
    const double2 RG = lds_f64x2(a0 + d2);
    q.L = LB.x;
    q.b = LB.y;
    q.r = RG.x;
    q.g = RG.y;
    dz = p.z - F.chz;
    meta = __float_as_uint(p.w);
  }
  const float dx = p.x - F.chx, dy = p.y - F.chy;
  const float yy = fmaf(dx, dx, dy * dy);
  const float r2 = fmaf(dz, dz, yy);
  // depth (integrator.cpp:396) + guard (:397) in one compare; ball
  // (photon_map.cpp:76): NaN (an exact-flagged record) passes into the band
  const bool maybe = valid && meta <= F.mlim && !(r2 > F.lim_hi);
  bool band = !(r2 < F.lim_lo) || !(fabsf(dx) > F.band_y) || !(fabsf(dy) > F.band_y);
  // quadrant (exact-sector table): +x+y 0, -x+y 1, -x-y 2, +x-y 3
  uint32_t s4 = dy > 0.0f ? (dx > 0.0f ? 0u : 4u) : (dx > 0.0f ? 12u : 8u);
  if constexpr (NA == 2) {  // one annulus edge at d2 = r2 / 2 (relative band 2e-4)
    const float de = yy - F.qa_edge;
    band = band || fabsf(de) < F.qa_eps;
    if (de >= 0.0f) s4 += 16u;
  }
  q.need = maybe && band;
  q.acc = maybe && !band;
  q.s4 = q.acc ? s4 : 16u * NA;  // a rejected pair adds into the lane's spare slot row (row 4 * NA)
  return q;
}

// Predicated add of the packed sector counts.
static __device__ __forceinline__ void padd_u32(uint32_t &acc, uint32_t v, bool p) {
  asm("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q add.u32 %0, %0, %1;\n\t}"
      : "+r"(acc) : "r"(v), "r"((uint32_t)p));
}

// Slot row 4 * n_a is the spare row of rejected pairs (never reduced), so the
// moments need no value select; cos_i <= 0 photons carry L = r = g = b = 0.
static __device__ __forceinline__ void lean_add(const LeanPair &q, uint32_t slot_lane, uint32_t &nib,
                                                double &p0, double &p1, double &p2) {
  const double v = q.L;
  const uint32_t a = slot_lane + q.s4 * (32u * 16u / 4u);  // [sector][lane] {sum, sum_sq}
  double2 o = lds_f64x2(a);
  o.x = da(o.x, v);
  o.y = da(o.y, dm(v, v));
  sts_f64x2(a, o);
  padd_u32(nib, 1u << q.s4, q.acc);
  // flux (integrator.cpp:449): fma(x, 1, p) = p + x and fma(x, 0, p) = p
  // exactly for the finite powers of lean records -- one DFMA per channel
  // (a predicated add is if-converted by ptxas into DADD + two FSEL)
  const double m = q.acc ? 1.0 : 0.0;
  p0 = __fma_rn(q.r, m, p0);
  p1 = __fma_rn(q.g, m, p1);
  p2 = __fma_rn(q.b, m, p2);
}

// Exact fp64 evaluation of the candidate at window index i of a lean window:
// the input photon (sorted -> input order) in the reference's operation order.
static __device__ __forceinline__ uint32_t lean_exact(const GatherArgs &A, const Hit &Hs, const FineWin &Wn,
                                                      uint32_t i, float4 &pw, double &L) {
  const uint32_t f = i + Wn.lo;  // flattened position -> piece -> sorted record -> input photon
  uint32_t p = 0;
  while (p + 1 < Wn.d->npieces && Wn.d->pre[p + 1] <= f) ++p;
  const uint32_t j = A.order[Wn.d->src[p] + (f - Wn.d->pre[p])];
  float4 a, B, Cc, D;
  fine_record(A.in_pos, A.in_nrm, A.in_wi, A.in_pow, A.in_depth, j, a, B, Cc, D);
  pw = Cc;
  L = __longlong_as_double(((long long)__float_as_uint(B.w) << 32) | __float_as_uint(B.z));
  const float4 b_old = make_float4(D.x, D.y, B.x, D.z);
  const float4 c2_old = make_float4(D.w, B.y, Cc.x, Cc.y);
  return exact_pair_packed(Hs, a, b_old, c2_old, A.na, A.ns, A.guard);
}

// Deferred pairs of a lean fragment (same ring as fine_exact_batch).
static __device__ __forceinline__ void lean_exact_batch(const GatherArgs &A, const Hit &Hs, uint32_t n, uint32_t ex,
                                                        uint32_t slot_lane, LeanCnt &c, double &p0, double &p1,
                                                        double &p2, const FineWin &Wn, FineState &st) {
  const int lane = threadIdx.x & 31;
  __syncwarp();
  lean_spill(c);
  const bool have = (uint32_t)lane < n;
  const uint32_t i = have ? lds_u32(ex + ((st.eh + lane) & (kFExact - 1)) * 4u) : 0u;
  st.eh += n;
  float4 pw = make_float4(0.f, 0.f, 0.f, 0.f);
  LeanPair q;
  q.L = 0.0;
  uint32_t fl = 0;
  if (have) {
    fl = lean_exact(A, Hs, Wn, i, pw, q.L);
    st.n_exact += 1;
    st.n_amb += (fl >> 2) & 1u;
  }
  q.acc = (fl & 1u) != 0;
  const bool on = q.acc && (fl & 2u) != 0;  // cos_i > 0 (bsdf.cpp:56-58): else the value is 0
  q.r = on ? (double)pw.x : 0.0;
  q.g = on ? (double)pw.y : 0.0;
  q.b = on ? (double)pw.z : 0.0;
  q.L = on ? q.L : 0.0;
  q.s4 = q.acc ? (fl >> 8) * 4u : 16u * (uint32_t)A.na;
  lean_add(q, slot_lane, c.n0, p0, p1, p2);
  lean_spill(c);
  __syncwarp();
}

// All candidates of one hit point inside the staged window, two per lane
// per step.  Virtual index v in [0, total) over the concatenated runs maps to
// the smem index v + off[j] of run j; the run is tracked warp-uniformly and a
// step only resolves per lane when a run ends inside it.
template <int NA, bool FLAT = false>
static __device__ __forceinline__ void lean_fragment(const GatherArgs &A, const FineHot &Hh, const Hit &Hs,
                                                     uint32_t rs, uint32_t rl, int nruns, uint32_t ex,
                                                     uint32_t slot_lane, LeanCnt &c, double &p0, double &p1,
                                                     double &p2, const FineWin &Wn, FineState &st,
                                                     float zflat = 0.0f) {
  const int lane = threadIdx.x & 31;
  const uint32_t lt = (1u << lane) - 1u;
  LeanHit F;
  F.chx = Hh.F.chx; F.chy = Hh.F.chy; F.chz = Hh.F.chz;
  if constexpr (FLAT) F.chz = zflat - Hh.F.chz;
  F.lim_hi = Hh.F.lim_hi; F.lim_lo = Hh.F.lim_lo; F.band_y = Hh.F.band_y;
  // n_a = 2: the annulus edge yy = r2 / 2, from lim_hi + lim_lo = 2 r2 (up to
  // an ulp; the 2e-4 band covers it; without the fp32 fast path every pair
  // is banded by the ball test anyway)
  F.qa_edge = 0.25f * (Hh.F.lim_hi + Hh.F.lim_lo);
  F.qa_eps = 2e-4f * F.qa_edge;
  F.mlim = Hh.mlim;
  const uint32_t d1 = Wn.r1 - Wn.r0, d2 = Wn.r2 - Wn.r0;
  uint32_t incl = rl;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(kFull, incl, o);
    if (lane >= o) incl += y;
  }
  const uint32_t off = rs - (incl - rl);  // smem index - virtual index within run `lane`
  const uint32_t total = __shfl_sync(kFull, incl, 31);
  if (lane == 0) st.n_cand += total;
  // the runs that meet this window are consecutive (the window is a range of
  // the flattened union): track from the first to the last non-empty one
  const uint32_t nem = __ballot_sync(kFull, rl != 0u);
  int j = nem ? __ffs(nem) - 1 : 0;
  nruns = nem ? 32 - __clz(nem) : 0;
  uint32_t e = __shfl_sync(kFull, incl, j), o = __shfl_sync(kFull, off, j);
  // candidates v0 = base + lane and v1 = v0 + 32 of a step -> window indices
  auto index = [&](uint32_t base, uint32_t &i0, uint32_t &i1) {
    const uint32_t v0 = base + lane, v1 = v0 + 32u;
    i0 = v0 + o;
    i1 = v1 + o;
    if (e < base + 64u) {  // a run ends before base + 64 (warp-uniform)
      while (e <= base) {  // skip runs that ended (incl. empty ones)
        ++j;
        e = __shfl_sync(kFull, incl, j);
        o = __shfl_sync(kFull, off, j);
      }
      i0 = v0 + o;
      i1 = v1 + o;
      int k = j;
      uint32_t ek = e, okk = o;
      while (ek < base + 64u && k + 1 < nruns) {
        ++k;
        okk = __shfl_sync(kFull, off, k);
        if (v0 >= ek) i0 = v0 + okk;
        if (v1 >= ek) i1 = v1 + okk;
        ek = __shfl_sync(kFull, incl, k);
      }
      // carry on from the run that holds the step's last slot
      j = k;
      e = ek;
      o = okk;
    }
  };
  // evaluate + accumulate the two candidates; their band flags out
  auto eval_add = [&](uint32_t i0, uint32_t i1, bool ok0, bool ok1, bool &n0, bool &n1) {
    const LeanPair q0 = lean_eval<NA, FLAT>(F, ok0, Wn.r0 + i0 * 16u, d1, d2);
    const LeanPair q1 = lean_eval<NA, FLAT>(F, ok1, Wn.r0 + i1 * 16u, d1, d2);
    lean_add(q0, slot_lane, c.n0, p0, p1, p2);
    lean_add(q1, slot_lane, c.n1, p0, p1, p2);
    n0 = q0.need;
    n1 = q1.need;
  };
  // banded pairs (rare) go to the exact ring
  auto push = [&](bool n0, uint32_t i0, bool n1, uint32_t i1) {
    const uint32_t m0 = __ballot_sync(kFull, n0), m1 = __ballot_sync(kFull, n1);
    if (n0) sts_u32(ex + ((st.et + __popc(m0 & lt)) & (kFExact - 1)) * 4u, i0);
    st.et += __popc(m0);
    if (n1) sts_u32(ex + ((st.et + __popc(m1 & lt)) & (kFExact - 1)) * 4u, i1);
    st.et += __popc(m1);
    while (st.et - st.eh >= 32)
      lean_exact_batch(A, Hs, 32u, ex, slot_lane, c, p0, p1, p2, Wn, st);
  };
  // two full steps per iteration: one spill count, one band vote (a nibble
  // takes <= 2 increments per iteration: spill every 7)
  const uint32_t full = total & ~63u, full2 = total & ~127u;
  for (uint32_t blk = 0; blk < full2; blk += 7u * 128u) {  // 7 iterations between spills
    const uint32_t blk_end = min(full2, blk + 7u * 128u);
    for (uint32_t base = blk; base < blk_end; base += 128) {
      uint32_t a0, a1, b0, b1;
      bool na0, na1, nb0, nb1;
      index(base, a0, a1);
      eval_add(a0, a1, true, true, na0, na1);
      index(base + 64u, b0, b1);
      eval_add(b0, b1, true, true, nb0, nb1);
      if (__any_sync(kFull, na0 || na1 || nb0 || nb1)) {
        push(na0, a0, na1, a1);
        push(nb0, b0, nb1, b1);
      }
    }
    lean_spill(c);
  }
  lean_spill(c);  // <= 2 more steps below
  if (full2 < full) {
    uint32_t a0, a1;
    bool na0, na1;
    index(full2, a0, a1);
    eval_add(a0, a1, true, true, na0, na1);
    if (__any_sync(kFull, na0 || na1)) push(na0, a0, na1, a1);
  }
  if (full < total) {  // the last, partial step: slots past the end read the window, never added
    uint32_t a0, a1;
    bool na0, na1;
    index(full, a0, a1);
    const bool ok0 = full + lane < total, ok1 = full + 32u + lane < total;
    if (!ok0) a0 = rs;
    if (!ok1) a1 = rs;
    eval_add(a0, a1, ok0, ok1, na0, na1);
    if (__any_sync(kFull, na0 || na1)) push(na0, a0, na1, a1);
  }
  while (st.et != st.eh)
    lean_exact_batch(A, Hs, min(32u, st.et - st.eh), ex, slot_lane, c, p0, p1, p2, Wn, st);
  lean_spill(c);
  __syncwarp();
}

// A hit point of a lean-layout frame that is not itself lean (another
// normal, a non-gray weight, ...): every candidate on the exact fp64 path,
// its full value v = lum(K * pw) accumulated in the lean slots (reduced with
// scale 1), counts in nibbles.
template <int NA>
static __device__ __forceinline__ void exact_fragment_lean(const GatherArgs &A, const FineHot &Hh, const Hit &Hs,
                                                           uint32_t rs, uint32_t rl, uint32_t slot_lane,
                                                           LeanCnt &c, double &p0, double &p1, double &p2,
                                                           const FineWin &Wn, FineState &st) {
  const int lane = threadIdx.x & 31;
  const double Kz = elum(dm(Hh.K0, 0.0), dm(Hh.K1, 0.0), dm(Hh.K2, 0.0));  // bsdf.cpp:58 (f = 0)
  uint32_t incl = rl;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(kFull, incl, o);
    if (lane >= o) incl += y;
  }
  const uint32_t off = rs - (incl - rl);
  const uint32_t total = __shfl_sync(kFull, incl, 31);
  if (lane == 0) st.n_cand += total;
  uint32_t spill = 15;
  for (uint32_t base = 0; base < total; base += 32) {
    const uint32_t v = base + lane;
    int j = 0;
    for (int k = 0; k < 32; ++k) j += __shfl_sync(kFull, incl, k) <= v ? 1 : 0;  // run of v
    const uint32_t i = v + __shfl_sync(kFull, off, j & 31);
    const bool have = v < total;
    float4 pw = make_float4(0.f, 0.f, 0.f, 0.f);
    double L = 0.0;
    uint32_t fl = 0;
    if (have) {
      fl = lean_exact(A, Hs, Wn, i, pw, L);
      st.n_exact += 1;
      st.n_amb += (fl >> 2) & 1u;
    }
    if (--spill == 0) {
      lean_spill(c);
      spill = 15;
    }
    LeanPair q;
    q.acc = (fl & 1u) != 0;
    const bool on = q.acc && (fl & 2u) != 0;
    q.L = on ? elum(dm(Hh.K0, (double)pw.x), dm(Hh.K1, (double)pw.y), dm(Hh.K2, (double)pw.z)) : Kz;
    q.r = on ? (double)pw.x : 0.0;
    q.g = on ? (double)pw.y : 0.0;
    q.b = on ? (double)pw.z : 0.0;
    q.s4 = q.acc ? (fl >> 8) * 4u : 16u * NA;
    lean_add(q, slot_lane, c.n0, p0, p1, p2);
  }
  lean_spill(c);
  __syncwarp();
}

// End of a lean fragment: the lane slots reduced in the fixed rotated order
// of the general path, scaled by K0 / K0^2, counts from the byte words, flux;
// added to the hit point's partial row [count G | sum G | sum_sq G | power 3].
// STORE: acc is the fragment's own row in HBM (ring kernel: one fragment per
// (hit point, item)), written instead of accumulated.
template <bool STORE>
static __device__ __forceinline__ void row_put(double &d, double v) {
  if constexpr (STORE) d = v; else d += v;
}
template <int GMAX, bool STORE = false>
static __device__ __forceinline__ void lean_reduce(uint32_t slots, int lane, double K0, const LeanCnt &c,
                                                   double p0, double p1, double p2, double *acc,
                                                   FineState &st, size_t fs = 1) {
  constexpr int NC = GMAX, NQ = 32 / NC, R = 32 / NQ;
  const int col = lane % NC, grp = lane / NC;
  double sm = 0.0, sq = 0.0;
  {
    // rows visited in an XOR-swizzled fixed order (lanes of different
    // columns hit different rows at each step: no bank conflicts); the
    // group's R rows are R * 16-B aligned, so the swizzle is one LOP3 per row
    static_assert(R == NC && (R & (R - 1)) == 0, "slot groups of R = NC rows, a power of two");
    const uint32_t base = (slots + (uint32_t)(col * 32 + grp * R) * 16u) | ((uint32_t)col * 16u);
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const uint32_t a = base ^ ((uint32_t)i * 16u);
      const double2 v = lds_f64x2(a);
      sm += v.x;
      sq += v.y;
      sts_f64x2(a, make_double2(0.0, 0.0));
    }
  }
#pragma unroll
  for (int o = (NQ / 2) * NC; o >= NC && o > 0; o >>= 1) {
    sm += __shfl_down_sync(kFull, sm, o);
    sq += __shfl_down_sync(kFull, sq, o);
  }
  // flux: transposed butterfly (12 shuffles instead of 30): after it lane 0
  // holds sum p0, lane 8 sum p1, lane 16 sum p2
  {
    const bool hi16 = (lane & 16) != 0, hi8 = (lane & 8) != 0;
    const double s0 = hi16 ? p0 : p2, k0 = hi16 ? p2 : p0;  // send / keep
    const double s1 = hi16 ? p1 : 0.0, k1 = hi16 ? 0.0 : p1;
    const double a = k0 + __shfl_xor_sync(kFull, s0, 16);   // lo: p0 | hi: p2
    const double b = k1 + __shfl_xor_sync(kFull, s1, 16);   // lo: p1 | hi: 0
    double c = (hi8 ? b : a) + __shfl_xor_sync(kFull, hi8 ? a : b, 8);
    c += __shfl_xor_sync(kFull, c, 4);
    c += __shfl_xor_sync(kFull, c, 2);
    c += __shfl_xor_sync(kFull, c, 1);
    p0 = __shfl_sync(kFull, c, 0);
    p1 = __shfl_sync(kFull, c, 8);
    p2 = __shfl_sync(kFull, c, 16);
  }
  // byte words -> 16-bit halves -> warp sums: even word bytes = sectors 0,2,4,6
  const uint32_t e02 = __reduce_add_sync(kFull, c.be & 0x00ff00ffu);         // s0 | s4 << 16
  const uint32_t e26 = __reduce_add_sync(kFull, (c.be >> 8) & 0x00ff00ffu);  // s2 | s6 << 16
  const uint32_t o15 = __reduce_add_sync(kFull, c.bo & 0x00ff00ffu);         // s1 | s5 << 16
  const uint32_t o37 = __reduce_add_sync(kFull, (c.bo >> 8) & 0x00ff00ffu);  // s3 | s7 << 16
  if (lane == 0)
    st.n_acc += (e02 & 0xffffu) + (e02 >> 16) + (e26 & 0xffffu) + (e26 >> 16) + (o15 & 0xffffu) + (o15 >> 16) +
                (o37 & 0xffffu) + (o37 >> 16);
  if (lane < NC) {
    row_put<STORE>(acc[(GMAX + lane) * fs], dm(K0, sm));
    row_put<STORE>(acc[(2 * GMAX + lane) * fs], dm(dm(K0, K0), sq));
  } else if (lane >= 32 - GMAX) {
    const int g = lane - (32 - GMAX);
    const uint32_t w = (g & 1) ? ((g & 2) ? o37 : o15) : ((g & 2) ? e26 : e02);
    row_put<STORE>(acc[g * fs], (double)((g & 4) ? (w >> 16) : (w & 0xffffu)));
  }
  if (lane == 0) {
    row_put<STORE>(acc[(3 * GMAX) * fs], p0);
    row_put<STORE>(acc[(3 * GMAX + 1) * fs], p1);
    row_put<STORE>(acc[(3 * GMAX + 2) * fs], p2);
  }
  if constexpr (STORE && partial_size(GMAX, 1) > 3 * GMAX + 3) {
    if (lane == 1) acc[(3 * GMAX + 3) * fs] = 0.0;  // the pad field: whole sectors written
  }
  __syncwarp();
}

// LEAN: the lean-layout instantiation (GridHeader::lean): only the lean
// fragment and its exact fallback are compiled in (register budget).
template <int GMAX, int CH, bool LEAN>
__global__ void __launch_bounds__(kFThreads, FineLayout<GMAX, CH>::kMinBlocks)
    k_gather_fine(const GatherArgs A, const FineArgs T) {
  using Lay = FineLayout<GMAX, CH>;
  constexpr int NC = Lay::NC, NQ = Lay::NQ, PS = Lay::PS;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double *s_slots = reinterpret_cast<double *>(smem_raw + Lay::kRecBytes);
  FineHot *s_hot = reinterpret_cast<FineHot *>(smem_raw + Lay::kRecBytes + Lay::kSlotBytes);
  double *s_rows = reinterpret_cast<double *>(smem_raw + Lay::kRecBytes + Lay::kSlotBytes + Lay::kHotBytes);
  __shared__ uint32_t s_ex[kFWarps][kFExact];
  __shared__ FineDesc s_descs[2];
  __shared__ __align__(8) uint64_t s_bar, s_dbar[2];  // records; descriptor buffer 0 / 1
  __shared__ uint32_t s_cur, s_next;

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t r0 = smem_u32(smem_raw);
  double *slots_p = s_slots + (size_t)warp * (NC + 1) * 32 * 2;
  for (int i = lane; i < (NC + 1) * 32 * 2; i += 32) slots_p[i] = 0.0;
  const uint32_t slots = smem_u32(slots_p);
  const uint32_t exa = smem_u32(&s_ex[warp][0]);
  const uint32_t total_items = *T.total_items;
  const GridHeader g = *A.grid;
  // Items are claimed one ahead and their descriptors prefetched by TMA, so
  // the work-counter atomic and the descriptor load overlap the current item.
  uint32_t nxt = 0;
  if (threadIdx.x == 0) {
    mbar_init(&s_bar, 1);
    mbar_init(&s_dbar[0], 1);
    mbar_init(&s_dbar[1], 1);
    fence_mbar_init();
    const uint32_t first = atomicAdd(A.work, 1u);
    if (first < total_items) {
      mbar_arrive_expect_tx(&s_dbar[0], (uint32_t)sizeof(FineDesc));
      bulk_g2s(&s_descs[0], T.desc + first, (uint32_t)sizeof(FineDesc), &s_dbar[0]);
    }
    s_cur = first;
    nxt = atomicAdd(A.work, 1u);
  }
  __syncthreads();
  uint32_t phase = 0, dphase = 0, b = 0;
  FineState st = {0, 0, 0, 0, 0, 0, 0, 0};

  for (;;) {
    const uint32_t item = s_cur;
    if (item >= total_items) break;
    mbar_wait(&s_dbar[b], (dphase >> b) & 1u);
    dphase ^= 1u << b;
    const FineDesc &s_desc = s_descs[b];
    uint32_t nxt2 = 0;
    if (threadIdx.x == 0) {
      if (nxt < total_items) {
        fence_proxy_async_smem();
        mbar_arrive_expect_tx(&s_dbar[b ^ 1u], (uint32_t)sizeof(FineDesc));
        bulk_g2s(&s_descs[b ^ 1u], T.desc + nxt, (uint32_t)sizeof(FineDesc), &s_dbar[b ^ 1u]);
      }
      nxt2 = atomicAdd(A.work, 1u);  // consumed at the end of this item
    }
    const uint32_t hp_n = s_desc.hp_n, Tu = s_desc.pre[kFMaxPieces];
    // per-hp sums over the item's windows accumulate in its partial rows
    double *out = s_rows;
    for (uint32_t i = threadIdx.x; i < hp_n * PS; i += kFThreads) out[i] = 0.0;
    __syncthreads();  // zeroed rows before any warp adds to them
    if (Tu != 0) {
      // window layout: 48-B records for planar waves (rec3 stays in HBM)
      const bool r48 = (s_desc.pad0 & 1u) != 0;
      const uint32_t cap = r48 ? Lay::kCap48 : Lay::kCap64;
      FineWin Wn;
      Wn.r0 = r0;
      Wn.r1 = r0 + cap * 16u;
      Wn.r2 = Wn.r1 + cap * 16u;
      Wn.r3 = r48 ? 0u : Wn.r2 + cap * 16u;
      Wn.d = &s_desc;
      Wn.grec3 = A.rec3;
      unsigned char *rec1 = smem_raw + (size_t)cap * 16, *rec2 = rec1 + (size_t)cap * 16,
                    *rec3 = rec2 + (size_t)cap * 16;
      // ---- the item's windows in order
      for (uint32_t c = s_desc.c0; c < s_desc.c1; ++c) {
        const uint32_t lo = c * cap, hi = min(Tu, lo + cap);
        const uint32_t ncand = hi - lo;
        Wn.lo = lo;
        if (warp == 0) {
          // lane 0 arms the barrier; lane p copies piece p, lane 31 the hit points
          const uint32_t hot_bytes = c == s_desc.c0 ? hp_n * (uint32_t)sizeof(FineHot) : 0u;
          if (lane == 0) {
            s_next = 0;
            fence_proxy_async_smem();
            mbar_arrive_expect_tx(&s_bar, ncand * (r48 ? 48u : 64u) + hot_bytes);
          }
          __syncwarp();
          if (lane == 31 && hot_bytes) bulk_g2s(s_hot, T.hot + s_desc.hp_lo, hot_bytes, &s_bar);
          if ((uint32_t)lane < s_desc.npieces) {
            const uint32_t p = lane;
            const uint32_t a = max(s_desc.pre[p], lo), e = min(s_desc.pre[p + 1], hi);
            if (e > a) {
              const uint32_t src = s_desc.src[p] + (a - s_desc.pre[p]), dst = a - lo, n = e - a;
              bulk_g2s(smem_raw + (size_t)dst * 16, A.rec0 + src, n * 16u, &s_bar);
              bulk_g2s(rec1 + (size_t)dst * 16, A.rec1 + src, n * 16u, &s_bar);
              bulk_g2s(rec2 + (size_t)dst * 16, A.rec2 + src, n * 16u, &s_bar);
              if (!r48) bulk_g2s(rec3 + (size_t)dst * 16, A.rec3 + src, n * 16u, &s_bar);
            }
#ifndef FPPM_NO_L2_PREFETCH
            // the item's next window into L2 while this one is processed
            if (c + 1 < s_desc.c1) {
              const uint32_t lo2 = lo + cap, hi2 = min(Tu, lo2 + cap);
              const uint32_t a2 = max(s_desc.pre[p], lo2), e2 = min(s_desc.pre[p + 1], hi2);
              if (e2 > a2) {
                const uint32_t src2 = s_desc.src[p] + (a2 - s_desc.pre[p]), n2 = e2 - a2;
                bulk_prefetch_l2(A.rec0 + src2, n2 * 16u);
                bulk_prefetch_l2(A.rec1 + src2, n2 * 16u);
                bulk_prefetch_l2(A.rec2 + src2, n2 * 16u);
                if (!r48) bulk_prefetch_l2(A.rec3 + src2, n2 * 16u);
              }
            }
#endif
          }
        }
        mbar_wait(&s_bar, phase);
        phase ^= 1u;

        // ---- warps take whole hit points (one fragment per hit point and window)
        for (;;) {
          uint32_t k = 0;
          if (lane == 0) k = atomicAdd(&s_next, 1u);
          k = __shfl_sync(kFull, k, 0);
          if (k >= hp_n) break;
          const FineHot &Hh = s_hot[k];
          // runs of this hit point inside the window (lane j = run j)
          const int nr = (int)Hh.nruns;
          uint32_t rs = 0, rl = 0;
          if (lane < nr) {
            int pc;
            if (slab_grid(g)) {
              pc = Hh.bx0 + lane - s_desc.ux0;
            } else {
              const int nyb = Hh.by1 - Hh.by0 + 1, nyu = s_desc.uy1 - s_desc.uy0 + 1;
              pc = (Hh.bx0 + lane / nyb - s_desc.ux0) * nyu + (Hh.by0 + lane % nyb - s_desc.uy0);
            }
            const uint2 R = Hh.run[lane];
            const uint32_t fa = s_desc.pre[pc] + (R.x - s_desc.src[pc]), fb = fa + (R.y - R.x);
            const uint32_t ca = max(fa, lo), cb = min(fb, hi);
            if (cb > ca) {
              rs = ca - lo;
              rl = cb - ca;
            }
          }
          if (!__any_sync(kFull, rl != 0)) continue;
          const Hit &Hs = T.hits[s_desc.hp_lo + k];  // full state: exact path only
          double *acc = out + (size_t)k * PS;  // windows of an item run in order in one CTA
          double p0 = 0.0, p1 = 0.0, p2 = 0.0;
          if constexpr (LEAN) {
            constexpr int NA = GMAX / 4;
            LeanCnt lc = {0u, 0u, 0u, 0u};
            const uint32_t slot_lane = slots + (uint32_t)lane * 16u;
            if (Hh.gray & 2u) {
              lean_fragment<NA>(A, Hh, Hs, rs, rl, nr, exa, slot_lane, lc, p0, p1, p2, Wn, st);
              lean_reduce<GMAX>(slots, lane, Hh.K0, lc, p0, p1, p2, acc, st);
            } else {
              exact_fragment_lean<NA>(A, Hh, Hs, rs, rl, slot_lane, lc, p0, p1, p2, Wn, st);
              lean_reduce<GMAX>(slots, lane, 1.0, lc, p0, p1, p2, acc, st);
            }
            continue;
          } else {
          PackedCounts<GMAX> cnt;
#pragma unroll
          for (int r = 0; r < PackedCounts<GMAX>::NP; ++r) cnt.w[r] = 0;
          if (Hh.planar && (Hh.gray & 1u))
            fine_fragment<GMAX, CH, true, true>(A, Hh, Hs, rs, rl, nr, exa, slots, cnt, p0, p1, p2, Wn, st);
          else if (Hh.planar)
            fine_fragment<GMAX, CH, true, false>(A, Hh, Hs, rs, rl, nr, exa, slots, cnt, p0, p1, p2, Wn, st);
          else if (Hh.gray & 1u)
            fine_fragment<GMAX, CH, false, true>(A, Hh, Hs, rs, rl, nr, exa, slots, cnt, p0, p1, p2, Wn, st);
          else
            fine_fragment<GMAX, CH, false, false>(A, Hh, Hs, rs, rl, nr, exa, slots, cnt, p0, p1, p2, Wn, st);

          // ---- fixed-order reduction of the lane slots, added to the hp's row
          const int col = lane % NC, grp = lane / NC;
          double sm = 0.0, sq = 0.0;
          if (grp < NQ) {
            // rows rotated by the column: the 16-B slots a warp touches per step
            // fall in distinct bank groups (fixed order, so still deterministic)
            constexpr int R = 32 / NQ;
            const uint32_t base = slots + (uint32_t)(col * 32 + grp * R) * 16u;
#pragma unroll 4
            for (int i = 0; i < R; ++i) {
              const uint32_t a = base + (uint32_t)((i + col) % R) * 16u;
              const double2 v = lds_f64x2(a);
              sm += v.x;
              sq += v.y;
              sts_f64x2(a, make_double2(0.0, 0.0));
            }
          }
#pragma unroll
          for (int o = (NQ / 2) * NC; o >= NC && o > 0; o >>= 1) {
            sm += __shfl_down_sync(kFull, sm, o);
            sq += __shfl_down_sync(kFull, sq, o);
          }
          p0 = warp_sum(p0);
          p1 = warp_sum(p1);
          p2 = warp_sum(p2);
          // packed byte counts -> 16-bit halves -> warp sums (<= 32 * 255 per half)
          uint32_t csum[2 * PackedCounts<GMAX>::NP];
#pragma unroll
          for (int r = 0; r < PackedCounts<GMAX>::NP; ++r) {
            csum[2 * r] = __reduce_add_sync(kFull, cnt.w[r] & 0x00ff00ffu);
            csum[2 * r + 1] = __reduce_add_sync(kFull, (cnt.w[r] >> 8) & 0x00ff00ffu);
          }
          if (lane == 0) {
            uint32_t tot = 0;
#pragma unroll
            for (int r = 0; r < 2 * PackedCounts<GMAX>::NP; ++r) tot += (csum[r] & 0xffffu) + (csum[r] >> 16);
            st.n_acc += tot;
          }
          if (lane < NC) {
            const int cc = lane / GMAX, gg = lane % GMAX;
            acc[GMAX + cc * GMAX + gg] += sm;
            acc[GMAX + CH * GMAX + cc * GMAX + gg] += sq;
          } else if (lane >= 32 - GMAX) {
            const int gg = lane - (32 - GMAX);
            const uint32_t wd = csum[2 * (gg >> 2) + (gg & 1)];
            acc[gg] += (double)((gg & 2) ? (wd >> 16) : (wd & 0xffffu));
          }
          if (lane == 0) {
            acc[GMAX + 2 * CH * GMAX] += p0;
            acc[GMAX + 2 * CH * GMAX + 1] += p1;
            acc[GMAX + 2 * CH * GMAX + 2] += p2;
          }
          __syncwarp();
          }
        }
        __syncthreads();  // the window buffer and s_next are reused by the next window
      }
    }
    {  // the item's rows, summed over its windows in order, out to HBM
      double *dst = T.partials + (size_t)s_desc.pbase * PS;
      for (uint32_t i = threadIdx.x; i < hp_n * PS; i += kFThreads) dst[i] = s_rows[i];
    }
    if (threadIdx.x == 0) {
      s_cur = nxt;
      nxt = nxt2;
    }
    b ^= 1u;
    __syncthreads();
  }

  // ------------------------------------------------------ block totals
  __shared__ unsigned long long s_c[4];
  if (threadIdx.x == 0) s_c[0] = s_c[1] = s_c[2] = s_c[3] = 0;
  __syncthreads();
  atomicAdd(&s_c[0], (unsigned long long)st.n_acc);
  atomicAdd(&s_c[1], (unsigned long long)st.n_cand);
  atomicAdd(&s_c[2], (unsigned long long)st.n_exact);
  atomicAdd(&s_c[3], (unsigned long long)st.n_amb);
  __syncthreads();
  if (threadIdx.x == 0) {
    atomicAdd(&A.counters[0], s_c[0]);
    atomicAdd(&A.counters[1], s_c[1]);
    atomicAdd(&A.counters[2], s_c[2]);
    atomicAdd(&A.counters[3], s_c[3]);
  }
}

// ------------------------------------------------------------------ ring kernel
// k_gather_ring: the lean fine gather with its windows in a ring of NB
// buffers.  k_gather_fine stages one window per CTA, so every window costs
// the CTA a barrier (warps wait for the one with the longest hit point) plus
// the TMA latency of the next window (ncu: 15 % + 6 % of the stall samples).
// Here one CTA per SM (16 warps) owns NB item buffers; an item is ONE window
// of a wave (schedule with fsub = 1).  Warps walk the items in sequence
// (position q in buffer q % NB), claiming hit points of each; the last warp
// to leave position q refills its buffer with position q + NB while the
// other buffers are consumed: no CTA-wide barrier, loads overlap the gather.
// Every buffer keeps one item claimed ahead with its descriptor already
// prefetched by TMA, so a refill issues its record copies at once.  Each
// (hit point, item) fragment writes its own partial row to HBM;
// k_tile_finalize sums a hit point's rows in window order, so the result is
// deterministic and identical to k_gather_fine's.
#ifndef FPPM_RING_WARPS
#define FPPM_RING_WARPS 16  // warps per CTA (12: 1.47 ms, larger windows but fewer warps)
#endif
#ifndef FPPM_RING_CAPDIV
#define FPPM_RING_CAPDIV 48  // measurement knob: > 48 shrinks the windows (records stay 48 B)
#endif
constexpr int kRWarps = FPPM_RING_WARPS;
constexpr int kRThreads = kRWarps * kWarp;

template <int GMAX, int NB, bool FLAT = false>
struct RingLayout {
  static constexpr uint32_t kRec = FLAT ? 32u : 48u;  // staged bytes per record
  static constexpr int NC = GMAX;  // lean: C = 1
  static constexpr int PS = partial_size(GMAX, 1);
  static constexpr size_t kSlotBytes = (size_t)kRWarps * (NC + 1) * 32 * 16;
  static constexpr size_t kHotBytes = (size_t)kFWave * sizeof(FineHot);
  static constexpr size_t kStatic = (size_t)kRWarps * kFExact * 4 + 2 * NB * sizeof(FineDesc) + 64 * NB + 64;
  static constexpr size_t kBudget = (size_t)233472 - 1024 - kStatic - 256;
  static constexpr uint32_t kCap =
      (uint32_t)((((kBudget - kSlotBytes - NB * kHotBytes) / NB) / (FLAT ? 32 : FPPM_RING_CAPDIV)) & ~(size_t)31);
  static constexpr size_t kBufBytes = (size_t)kCap * kRec;  // rec0 | rec1 [| rec2], 16 B each
  static constexpr size_t kDynBytes = NB * kBufBytes + kSlotBytes + NB * kHotBytes;
};

static __device__ __forceinline__ uint32_t atom_add_smem(uint32_t *p, uint32_t v) {
  uint32_t r;
  asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(v) : "memory");
  return r;
}

template <int NB>
struct RingShared {
  FineDesc desc[NB];   // descriptor of the item in buffer b
  FineDesc pdesc[NB];  // descriptor of buffer b's next item (TMA prefetch)
  uint64_t full[NB];   // records + hit points of buffer b landed
  uint64_t dbar[NB];   // pdesc[b] landed
  uint32_t item[NB], pitem[NB], next[NB], left[NB], dphase[NB];  // dphase: parity of dbar[b]
};

// Claim an item for buffer b's next turn and prefetch its descriptor (lane 0).
template <int NB>
static __device__ __forceinline__ void ring_preclaim(uint32_t b, const GatherArgs &A, const FineArgs &T,
                                                     uint32_t total_items, RingShared<NB> &R) {
  const uint32_t item = atomicAdd(A.work, 1u);
  R.pitem[b] = item;
  if (item < total_items) {
    fence_proxy_async_smem();
    mbar_arrive_expect_tx(&R.dbar[b], (uint32_t)sizeof(FineDesc));
    bulk_g2s(&R.pdesc[b], T.desc + item, (uint32_t)sizeof(FineDesc), &R.dbar[b]);
  }
}

// One warp: put buffer b's pre-claimed item into b (descriptor from pdesc,
// hit points + record pieces by TMA, completing on full[b]), then pre-claim
// the item for b's following turn.  An item past the end arrives without
// data: the consumers read R.item and skip it.
template <int GMAX, int NB, bool FLAT>
static __device__ __forceinline__ void ring_fill(uint32_t b, const GatherArgs &A, const FineArgs &T,
                                                 uint32_t total_items, RingShared<NB> &R,
                                                 unsigned char *buf, FineHot *hot) {
  using Lay = RingLayout<GMAX, NB, FLAT>;
  const int lane = threadIdx.x & 31;
  const uint32_t item = R.pitem[b];
  if (lane == 0) {
    R.item[b] = item;
    R.next[b] = 0;
    R.left[b] = 0;
  }
  if (item < total_items) {
    mbar_wait(&R.dbar[b], R.dphase[b]);
    constexpr int kWords = (int)(sizeof(FineDesc) / 4);
    const uint32_t *src = reinterpret_cast<const uint32_t *>(&R.pdesc[b]);
    uint32_t *dst = reinterpret_cast<uint32_t *>(&R.desc[b]);
    for (int k = lane; k < kWords; k += 32) dst[k] = src[k];
    __syncwarp();
    const FineDesc &D = R.desc[b];
    const uint32_t Tu = D.pre[kFMaxPieces];
    const uint32_t lo = D.c0 * Lay::kCap, hi = min(Tu, lo + Lay::kCap);
    const uint32_t hot_bytes = D.hp_n * (uint32_t)sizeof(FineHot);
    if (lane == 0) {
      R.dphase[b] ^= 1u;
      fence_proxy_async_smem();
      mbar_arrive_expect_tx(&R.full[b], (hi - lo) * Lay::kRec + hot_bytes);
    }
    __syncwarp();
    if (lane == 31) bulk_g2s(hot, T.hot + D.hp_lo, hot_bytes, &R.full[b]);
    if ((uint32_t)lane < D.npieces) {
      const uint32_t p = lane;
      const uint32_t a = max(D.pre[p], lo), e = min(D.pre[p + 1], hi);
      if (e > a) {
        const uint32_t sp = D.src[p] + (a - D.pre[p]), dp = a - lo, n = e - a;
        bulk_g2s(buf + (size_t)dp * 16, A.rec0 + sp, n * 16u, &R.full[b]);
        bulk_g2s(buf + (size_t)(Lay::kCap + dp) * 16, A.rec1 + sp, n * 16u, &R.full[b]);
        if constexpr (!FLAT)
          bulk_g2s(buf + (size_t)(2 * Lay::kCap + dp) * 16, A.rec2 + sp, n * 16u, &R.full[b]);
      }
    }
    __syncwarp();
    if (lane == 0) ring_preclaim<NB>(b, A, T, total_items, R);
  } else {
    __syncwarp();
    if (lane == 0) mbar_arrive_expect_tx(&R.full[b], 0u);  // items past the end stay past the end
  }
  __syncwarp();
}

template <int GMAX, int NB, bool FLAT>
__global__ void __launch_bounds__(kRThreads, 1) k_gather_ring(const GatherArgs A, const FineArgs T) {
  using Lay = RingLayout<GMAX, NB, FLAT>;
  constexpr int NC = Lay::NC, PS = Lay::PS, NA = GMAX / 4;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double *s_slots = reinterpret_cast<double *>(smem_raw + NB * Lay::kBufBytes);
  FineHot *s_hot = reinterpret_cast<FineHot *>(smem_raw + NB * Lay::kBufBytes + Lay::kSlotBytes);
  __shared__ uint32_t s_ex[kRWarps][kFExact];
  __shared__ __align__(16) RingShared<NB> R;

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double *slots_p = s_slots + (size_t)warp * (NC + 1) * 32 * 2;
  for (int i = lane; i < (NC + 1) * 32 * 2; i += 32) slots_p[i] = 0.0;
  const uint32_t slots = smem_u32(slots_p);
  const uint32_t exa = smem_u32(&s_ex[warp][0]);
  const uint32_t total_items = *T.total_items;
  const GridHeader g = *A.grid;
  if (threadIdx.x == 0) {
    for (int b = 0; b < NB; ++b) {
      mbar_init(&R.full[b], 1);
      mbar_init(&R.dbar[b], 1);
      R.dphase[b] = 0;
    }
    fence_mbar_init();
    for (int b = 0; b < NB; ++b) ring_preclaim<NB>(b, A, T, total_items, R);  // positions 0 .. NB - 1
  }
  __syncthreads();
  if (warp == 0)
    for (int b = 0; b < NB; ++b)
      ring_fill<GMAX, NB, FLAT>(b, A, T, total_items, R, smem_raw + b * Lay::kBufBytes, s_hot + b * kFWave);
  FineState st = {0, 0, 0, 0, 0, 0, 0, 0};

  uint32_t dead = 0;  // consecutive positions past the end
  for (uint32_t q = 0;; ++q) {
    const uint32_t b = q % NB;
    mbar_wait(&R.full[b], (q / NB) & 1u);
    const uint32_t item = *reinterpret_cast<volatile uint32_t *>(&R.item[b]);
    if (item < total_items) {
      dead = 0;
      const FineDesc &D = R.desc[b];
      const uint32_t hp_n = D.hp_n, Tu = D.pre[kFMaxPieces];
      const uint32_t lo = D.c0 * Lay::kCap, hi = min(Tu, lo + Lay::kCap);
      const uint32_t rb = smem_u32(smem_raw + b * Lay::kBufBytes);
      FineWin Wn;
      Wn.r0 = rb;
      Wn.r1 = rb + Lay::kCap * 16u;
      Wn.r2 = Wn.r1 + Lay::kCap * 16u;
      Wn.r3 = 0u;
      Wn.lo = lo;
      Wn.d = &D;
      Wn.grec3 = A.rec3;
      const FineHot *hot = s_hot + b * kFWave;
      const uint32_t nclaim = D.nclaim;
      (void)hp_n;
      for (;;) {
        uint32_t kc = 0;
        if (lane == 0) kc = atom_add_smem(&R.next[b], 1u);
        kc = __shfl_sync(kFull, kc, 0);
        if (kc >= nclaim) break;
        const uint32_t k = D.order[kc];  // largest fragment first (k_fine_desc)
        const FineHot &Hh = hot[k];
        const int nr = (int)Hh.nruns;
        uint32_t rs = 0, rl = 0;
        if (lane < nr) {
          int pc;
          if (slab_grid(g)) {
            pc = Hh.bx0 + lane - D.ux0;
          } else {
            const int nyb = Hh.by1 - Hh.by0 + 1, nyu = D.uy1 - D.uy0 + 1;
            pc = (Hh.bx0 + lane / nyb - D.ux0) * nyu + (Hh.by0 + lane % nyb - D.uy0);
          }
          const uint2 Rr = Hh.run[lane];
          const uint32_t fa = D.pre[pc] + (Rr.x - D.src[pc]), fb = fa + (Rr.y - Rr.x);
          const uint32_t ca = max(fa, lo), cb = min(fb, hi);
          if (cb > ca) {
            rs = ca - lo;
            rl = cb - ca;
          }
        }
        // this fragment's own row: the hit point's rows are contiguous, one per
        // window of its range [pad_[1], pad_[2]) (k_fine_desc); a window
        // outside the range holds none of its candidates and has no row
        const uint32_t c = D.c0;
        if (c < Hh.pad_[1] || c >= Hh.pad_[2]) continue;
        double *acc = T.partials + (size_t)(Hh.pad_[0] + c) * PS;
        constexpr size_t fs = 1;
        if (!__any_sync(kFull, rl != 0)) {
          if (lane < PS) acc[lane] = 0.0;
          continue;
        }
        const Hit &Hs = T.hits[D.hp_lo + k];  // full state: exact path only
        double p0 = 0.0, p1 = 0.0, p2 = 0.0;
        LeanCnt lc = {0u, 0u, 0u, 0u};
        const uint32_t slot_lane = slots + (uint32_t)lane * 16u;
        if (Hh.gray & 2u) {
          lean_fragment<NA, FLAT>(A, Hh, Hs, rs, rl, nr, exa, slot_lane, lc, p0, p1, p2, Wn, st, g.zflat);
          lean_reduce<GMAX, true>(slots, lane, Hh.K0, lc, p0, p1, p2, acc, st, fs);
        } else {
          exact_fragment_lean<NA>(A, Hh, Hs, rs, rl, slot_lane, lc, p0, p1, p2, Wn, st);
          lean_reduce<GMAX, true>(slots, lane, 1.0, lc, p0, p1, p2, acc, st, fs);
        }
      }
    } else {
      ++dead;
    }
    // leave the position; the last warp out refills its buffer (position q + NB)
    __syncwarp();
    uint32_t left = 0;
    if (lane == 0) left = atom_add_smem(&R.left[b], 1u);
    left = __shfl_sync(kFull, left, 0);
    if (left == kRWarps - 1)
      ring_fill<GMAX, NB, FLAT>(b, A, T, total_items, R, smem_raw + b * Lay::kBufBytes, s_hot + b * kFWave);
    // A position's item was claimed when position q - 2 NB was left, and every
    // claim after one past the end is past the end: after 2 NB dead positions
    // in a row no later position holds an item.
    if (dead == 2 * NB) break;
  }

  __shared__ unsigned long long s_c[4];
  if (threadIdx.x == 0) s_c[0] = s_c[1] = s_c[2] = s_c[3] = 0;
  __syncthreads();
  atomicAdd(&s_c[0], (unsigned long long)st.n_acc);
  atomicAdd(&s_c[1], (unsigned long long)st.n_cand);
  atomicAdd(&s_c[2], (unsigned long long)st.n_exact);
  atomicAdd(&s_c[3], (unsigned long long)st.n_amb);
  __syncthreads();
  if (threadIdx.x == 0) {
    atomicAdd(&A.counters[0], s_c[0]);
    atomicAdd(&A.counters[1], s_c[1]);
    atomicAdd(&A.counters[2], s_c[2]);
    atomicAdd(&A.counters[3], s_c[3]);
  }
}

// ------------------------------------------------------------------ launchers
static inline unsigned fblocks(unsigned long long n, int threads, int sms, int per_sm) {
  unsigned long long b = (n + threads - 1) / threads;
  const unsigned long long cap = (unsigned long long)sms * per_sm;
  if (b > cap) b = cap;
  return (unsigned)(b ? b : 1);
}

bool fine_supported(int G, int C) {
  const int gmax = G <= 4 ? 4 : G <= 8 ? 8 : G <= 12 ? 12 : G <= 16 ? 16 : 32;
  return gmax * C <= 24;
}

void fine_caps(int G, int C, int lean, uint32_t *cap64, uint32_t *cap48, uint32_t *fsub) {
#define FPPM_CAPS(gm, ch) \
  do {                    \
    *cap64 = FineLayout<gm, ch>::kCap64; \
    *cap48 = FineLayout<gm, ch>::kCap48; \
  } while (0)
  *fsub = kFSub;
  if (lean && ring_enabled()) {  // k_gather_ring: items of one window, 48-B records
    if (lean == 2) *cap48 = *cap64 = (G <= 4) ? RingLayout<4, 2, true>::kCap : RingLayout<8, 2, true>::kCap;
    else *cap48 = *cap64 = (G <= 4) ? RingLayout<4, 2>::kCap : RingLayout<8, 2>::kCap;
    *fsub = 1;
    return;
  }
  if (C == 1) {
    if (G <= 4) FPPM_CAPS(4, 1);
    else if (G <= 8) FPPM_CAPS(8, 1);
    else if (G <= 12) FPPM_CAPS(12, 1);
    else FPPM_CAPS(16, 1);
  } else {
    if (G <= 4) FPPM_CAPS(4, 3);
    else FPPM_CAPS(8, 3);
  }
#undef FPPM_CAPS
}

cudaError_t fine_schedule_bins(cudaStream_t s, const GatherArgs &A, TileSched &S, const GridHeader &g,
                               int sms, uint32_t cap64, uint32_t cap48, uint32_t fsub, uint32_t *nb_out,
                               unsigned long long hp_version) {
  const long long x0 = g.ix0 >> g.shift, y0 = g.iy0 >> g.shift, z0 = g.iz0 >> g.shift;
  const unsigned long long ex = (unsigned long long)(((g.ix0 + g.nx - 1) >> g.shift) - x0 + 3);
  const unsigned long long ey = (unsigned long long)(((g.iy0 + g.ny - 1) >> g.shift) - y0 + 3);
  const unsigned long long ez = (unsigned long long)(((g.iz0 + g.nz - 1) >> g.shift) - z0 + 3);
  const unsigned long long n_ext = ex * ey * ez;
  if (n_ext + 1 >= 0xffffffffull) return cudaErrorInvalidValue;
  const uint32_t nb = (uint32_t)n_ext + 1;
  *nb_out = nb;
  const long long dims[7] = {g.ix0, g.iy0, g.iz0, g.nx, g.ny, g.nz, (long long)g.shift};
  bool same = S.bins_valid && S.bins_version == hp_version && S.bins_H == A.H && S.bins_nb == nb &&
              S.bins_inv == g.inv;
  for (int k = 0; k < 7 && same; ++k) same = S.bins_dims[k] == dims[k];
  cudaError_t e = cudaSuccess;
  if (!same) {
    S.bins_valid = false;
    k_fine_bin<<<fblocks(A.H, 256, sms, 16), 256, 0, s>>>(A.pos, A.gathered, A.H, A.grid,
                                                          S.sort.keys_a, S.sort.vals_a);
    note_launches(1);
    uint32_t bits = 1;
    while (bits < 32 && (1ull << bits) < (unsigned long long)nb) ++bits;
    uint32_t *skeys, *svals;
    e = radix_sort_pairs(s, S.sort, A.H, bits, &skeys, &svals);
    if (e != cudaSuccess) return e;
    S.hp_order = svals;
    e = launch_bucket_start(s, skeys, A.H, nb, S.hp_start, sms);
    if (e != cudaSuccess) return e;
    S.bins_valid = true;
    S.bins_version = hp_version;
    S.bins_H = A.H;
    S.bins_nb = nb;
    S.bins_inv = g.inv;
    for (int k = 0; k < 7; ++k) S.bins_dims[k] = dims[k];
  }
  // per hit point state in wave order (needed by the window sizing below)
  e = cudaFuncSetAttribute(k_fine_prep, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kPrepSmem);
  if (e != cudaSuccess) return e;
  k_fine_prep<<<fblocks(A.H, kPrepThreads, sms, 8), kPrepThreads, kPrepSmem, s>>>(
      A, S.hp_order, static_cast<FineHot *>(S.fhot),
                                                        S.fbox, static_cast<Hit *>(S.fhit));
  note_launches(1);
  k_fine_items<<<fblocks((unsigned long long)(nb + 1) * 32, 128, sms, 16), 128, 0, s>>>(
      A, S.hp_start, nb, static_cast<const FineHot *>(S.fhot), S.fbox, S.items,
      S.chunks, cap64, cap48, fsub, S.nonempty, S.hp_order, S.hp_nc);
  note_launches(1);
  e = launch_exclusive_scan(s, S.items, nb + 1, S.scan_tmp, S.item_base);
  if (e != cudaSuccess) return e;
  if (fsub == 1) {  // ring rows in hit-point order (hp_nc[H] = 0: rbase[H] = rows)
    e = cudaMemsetAsync(S.hp_nc + A.H, 0, sizeof(uint32_t), s);
    if (e != cudaSuccess) return e;
    e = launch_exclusive_scan(s, S.hp_nc, A.H + 1, S.hp_scan_tmp, S.hp_rbase);
    if (e != cudaSuccess) return e;
  }
  return launch_exclusive_scan(s, S.chunks, nb + 1, S.scan_tmp, S.pbase);
}

cudaError_t fine_schedule_items(cudaStream_t s, const GatherArgs &A, TileSched &S, uint32_t nb, int sms,
                                uint32_t cap64, uint32_t cap48, uint32_t fsub) {
  k_fine_desc<<<fblocks((unsigned long long)nb * 32, 128, sms, 16), 128, 0, s>>>(
      A, S.hp_start, nb, S.hp_order, static_cast<FineHot *>(S.fhot), S.fbox,
      S.item_base, S.pbase, S.fdesc, S.hp_map, cap64, cap48, fsub, S.hp_rbase, S.hp_span, S.item_cap);
  note_launches(1);
  if (fsub == 1) {
    k_fine_order<<<(unsigned)sms * 8, 128, 0, s>>>(S.fdesc, S.item_base + nb, static_cast<const FineHot *>(S.fhot),
                                                 S.hp_span, cap48, S.item_cap);
    note_launches(1);
  }
  return cudaGetLastError();
}

template <int GMAX, int CH, bool LEAN>
static cudaError_t launch_fine_t(cudaStream_t s, const GatherArgs &A, const FineArgs &T, int sms) {
  using Lay = FineLayout<GMAX, CH>;
  const size_t smem = Lay::kDynBytes;
  cudaError_t e = cudaFuncSetAttribute(k_gather_fine<GMAX, CH, LEAN>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_gather_fine<GMAX, CH, LEAN>, kFThreads, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  k_gather_fine<GMAX, CH, LEAN><<<sms * per_sm, kFThreads, smem, s>>>(A, T);
  note_launches(1);
  return cudaGetLastError();
}

size_t fine_hot_bytes() { return sizeof(FineHot); }
size_t fine_hit_bytes() { return sizeof(Hit); }

template <int GMAX, int NB, bool FLAT>
static cudaError_t launch_ring_t(cudaStream_t s, const GatherArgs &A, const FineArgs &T, int sms) {
  using Lay = RingLayout<GMAX, NB, FLAT>;
  const size_t smem = Lay::kDynBytes;
  cudaError_t e = cudaFuncSetAttribute(k_gather_ring<GMAX, NB, FLAT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  k_gather_ring<GMAX, NB, FLAT><<<sms, kRThreads, smem, s>>>(A, T);
  note_launches(1);
  return cudaGetLastError();
}

// FPPM_RING=0 selects the one-window-per-CTA kernel for lean frames (A/B)
bool ring_enabled() {
  static const bool on = [] {
    const char *e = std::getenv("FPPM_RING");
    return !(e && e[0] == '0');
  }();
  return on;
}
// FPPM_FLAT=0 keeps 48-B lean records for frames whose photons share one z (A/B)
bool flat_records_enabled() {
  static const bool on = [] {
    const char *e = std::getenv("FPPM_FLAT");
    return ring_enabled() && !(e && e[0] == '0');
  }();
  return on;
}

cudaError_t launch_gather_fine(cudaStream_t s, const GatherArgs &A, const FineArgs &T, int C, int sms, int lean) {
  const int G = A.na * A.ns;
  if (lean) {  // C = 1, n_s = 4, n_a <= 2 (lean_config)
    if (C != 1 || A.ns != 4 || A.na > 2) return cudaErrorInvalidValue;
    if (ring_enabled()) {
      if (lean == 2)
        return A.na == 1 ? launch_ring_t<4, 2, true>(s, A, T, sms) : launch_ring_t<8, 2, true>(s, A, T, sms);
      return A.na == 1 ? launch_ring_t<4, 2, false>(s, A, T, sms) : launch_ring_t<8, 2, false>(s, A, T, sms);
    }
    if (lean == 2) return cudaErrorInvalidValue;  // flat records are staged by the ring kernel only
    return A.na == 1 ? launch_fine_t<4, 1, true>(s, A, T, sms) : launch_fine_t<8, 1, true>(s, A, T, sms);
  }
  if (C == 1) {
    if (G <= 4) return launch_fine_t<4, 1, false>(s, A, T, sms);
    if (G <= 8) return launch_fine_t<8, 1, false>(s, A, T, sms);
    if (G <= 12) return launch_fine_t<12, 1, false>(s, A, T, sms);
    if (G <= 16) return launch_fine_t<16, 1, false>(s, A, T, sms);
    return cudaErrorInvalidValue;
  }
  if (G <= 4) return launch_fine_t<4, 3, false>(s, A, T, sms);
  if (G <= 8) return launch_fine_t<8, 3, false>(s, A, T, sms);
  return cudaErrorInvalidValue;
}

}  // namespace fppm_b200
