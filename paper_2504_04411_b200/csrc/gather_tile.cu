// gather_tile.cu -- tiled gather + F-test: one CTA per (home cell, candidate chunk).
//
// The reference visits, for every hit point, the 27 cells around its own cell
// (photon_map.cpp:65-77).  All hit points whose center falls in the same
// grid cell ("home cell") share that candidate set, so the work is organised
// as items:
//
//   item = (home cell, wave of <= 32 hit points, chunk of <= kChunk candidates)
//
// Per item a CTA pulls the chunk's photon records (4 x 16 B SoA vectors) into
// shared memory with TMA bulk copies (cp.async.bulk, one per contiguous
// piece of the 9 (dx, dy) columns, completing on an mbarrier), then each warp
// owns one hit point at a time:
//
//   test   lanes stride over the chunk (LDS.128 of rec0), fp32 ball + disk test
//          with rigorous error bands; survivors go to a per-warp queue
//   flush  whenever 32 survivors are queued, all 32 lanes take one each:
//          guard, cos_i, sector in fp32 with bands (fp64 exact path otherwise),
//          then fp64 accumulation into per-lane sector registers
//   reduce fixed-order warp shuffles; fragments of one hit point (the
//          (hit point x candidate) space is split evenly over the warps)
//          are combined in warp order and written as the item's partial.
//
// Items are scheduled by a persistent grid through a global work counter.
// Every item writes one partial per hit point of its wave; k_tile_finalize
// (one thread per hit point) sums a wave's chunk partials in chunk order and
// runs the fused end_iteration, so no CTA waits on the serial epilogue.
#include "common.cuh"
#include "gather.cuh"
#include "gather_dev.cuh"

namespace fppm_b200 {

constexpr int kTileWarps = 8;
constexpr int kTileThreads = kTileWarps * kWarp;
constexpr int kWave = 32;  // hit points per item
constexpr int kUnroll = 4;                  // candidates per lane per test round
constexpr int kQueue = 256;               // survivor ring per warp (holds <= 31 + 128)
constexpr int kMaxFrag = kWave + kTileWarps;


// ------------------------------------------------------------------ scheduling
// bucket of a hit point: its home cell in the photon grid extended by one cell
// on every side, or the "no candidates" bucket n_ext (outside / not gathered /
// empty photon set).
__global__ void k_hp_bin(const double3 *__restrict__ pos, const uint8_t *__restrict__ gathered,
                         uint32_t H, const GridHeader *__restrict__ hdr,
                         uint32_t *__restrict__ keys, uint32_t *__restrict__ vals) {
  const GridHeader g = *hdr;
  const long long ex = g.nx + 2, ey = g.ny + 2, ez = g.nz + 2;
  const uint32_t n_ext = (uint32_t)(ex * ey * ez);
  for (uint32_t h = blockIdx.x * blockDim.x + threadIdx.x; h < H; h += gridDim.x * blockDim.x) {
    uint32_t key = n_ext;
    const double3 c = pos[h];
    if (g.n > 0 && (gathered == nullptr || gathered[h])) {
      const long long X = (long long)floor(dm(c.x, g.inv)) - g.ix0 + 1;
      const long long Y = (long long)floor(dm(c.y, g.inv)) - g.iy0 + 1;
      const long long Z = (long long)floor(dm(c.z, g.inv)) - g.iz0 + 1;
      if (X >= 0 && Y >= 0 && Z >= 0 && X < ex && Y < ey && Z < ez)
        key = (uint32_t)((X * ey + Y) * ez + Z);
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
__device__ __forceinline__ uint32_t column_ranges(const GridHeader &g, const uint32_t *cell_start,
                                                  long long ix, long long iy, long long iz,
                                                  uint32_t *beg, uint32_t *len) {
  uint32_t total = 0;
  const long long z0 = iz - 1 < 0 ? 0 : iz - 1;
  const long long z1 = iz + 1 >= g.nz ? g.nz - 1 : iz + 1;
  for (int c = 0; c < 9; ++c) {
    const long long X = ix + c / 3 - 1, Y = iy + c % 3 - 1;
    beg[c] = 0;
    len[c] = 0;
    if (g.n > 0 && X >= 0 && X < g.nx && Y >= 0 && Y < g.ny && z0 <= z1) {
      const unsigned long long k0 = (unsigned long long)((X * g.ny + Y) * g.nz + z0);
      const unsigned long long k1 = (unsigned long long)((X * g.ny + Y) * g.nz + z1);
      beg[c] = cell_start[k0];
      len[c] = cell_start[k1 + 1] - beg[c];
    }
    total += len[c];
  }
  return total;
}

__device__ __forceinline__ void bucket_cell(const GridHeader &g, uint32_t b, long long &ix,
                                            long long &iy, long long &iz) {
  const long long ey = g.ny + 2, ez = g.nz + 2;
  const long long X = (long long)b / (ey * ez);
  const long long Y = ((long long)b / ez) % ey;
  const long long Z = (long long)b % ez;
  ix = X - 1;
  iy = Y - 1;
  iz = Z - 1;
}

__global__ void k_bucket_items(const uint32_t *__restrict__ hp_start, uint32_t nb,
                               const GridHeader *__restrict__ hdr,
                               const uint32_t *__restrict__ cell_start,
                               uint32_t *__restrict__ items, uint32_t *__restrict__ chunks,
                               uint32_t chunk, uint32_t *__restrict__ nonempty) {
  const GridHeader g = *hdr;
  for (uint32_t b = blockIdx.x * blockDim.x + threadIdx.x; b <= nb; b += gridDim.x * blockDim.x) {
    const uint32_t nhp = b < nb ? hp_start[b + 1] - hp_start[b] : 0u;
    uint32_t ch = 0, it = 0;
    if (nhp) {
      atomicAdd(nonempty, 1u);
      uint32_t T = 0;
      if (b + 1 < nb) {  // bucket nb-1 is the "no candidates" bucket
        long long ix, iy, iz;
        bucket_cell(g, b, ix, iy, iz);
        uint32_t beg[9], len[9];
        T = column_ranges(g, cell_start, ix, iy, iz, beg, len);
      }
      ch = T == 0 ? 1u : (T + chunk - 1) / chunk;
      it = ch * ((nhp + kWave - 1) / kWave);
    }
    items[b] = it;
    chunks[b] = ch;
  }
}

// exclusive scan, 3 phases over tiles of 4096 (block_exclusive_scan_256 x 16)
constexpr int kScanTile = 4096;
__global__ void __launch_bounds__(256) k_scan_tiles(const uint32_t *__restrict__ in, uint32_t n,
                                                    uint32_t *__restrict__ tile_sum) {
  __shared__ uint32_t s_warp[8];
  const uint32_t base = blockIdx.x * kScanTile;
  uint32_t s = 0;
  for (int k = 0; k < kScanTile / 256; ++k) {
    const uint32_t i = base + k * 256 + threadIdx.x;
    s += i < n ? in[i] : 0u;
  }
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
  const uint32_t base = blockIdx.x * kScanTile;
  uint32_t carry = tile_sum[blockIdx.x];
  for (int k = 0; k < kScanTile / 256; ++k) {
    const uint32_t i = base + k * 256 + threadIdx.x;
    const uint32_t v = i < n ? in[i] : 0u;
    uint32_t tot;
    const uint32_t ex = block_exclusive_scan_256(v, s_warp, &tot);
    if (i < n) out[i] = carry + ex;
    carry += tot;
  }
}

__global__ void k_item_desc(const uint32_t *__restrict__ hp_start, uint32_t nb,
                            const GridHeader *__restrict__ hdr,
                            const uint32_t *__restrict__ cell_start,
                            const uint32_t *__restrict__ items, const uint32_t *__restrict__ chunks,
                            const uint32_t *__restrict__ item_base, const uint32_t *__restrict__ hp_order,
                            ItemDesc *__restrict__ desc, uint32_t *__restrict__ hp_map,
                            uint32_t kChunk) {
  const GridHeader g = *hdr;
  for (uint32_t b = blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += gridDim.x * blockDim.x) {
    if (items[b] == 0) continue;
    const uint32_t nch = chunks[b];
    uint32_t beg[9], len[9], T = 0;
    if (b + 1 < nb) {
      long long ix, iy, iz;
      bucket_cell(g, b, ix, iy, iz);
      T = column_ranges(g, cell_start, ix, iy, iz, beg, len);
    } else {
      for (int c = 0; c < 9; ++c) beg[c] = len[c] = 0;
    }
    const uint32_t h0 = hp_start[b], nhp = hp_start[b + 1] - h0;
    const uint32_t waves = (nhp + kWave - 1) / kWave;
    uint32_t item = item_base[b];
    for (uint32_t w = 0; w < waves; ++w) {
      const uint32_t first = item;
      for (uint32_t j = w * kWave; j < min(nhp, (w + 1) * kWave); ++j) {
        const uint32_t h = hp_order[h0 + j];
        // finalize reads partials (base + ch * stride) for ch < nch
        hp_map[3 * (size_t)h] = first * kWave + (j - w * kWave);
        hp_map[3 * (size_t)h + 1] = nch;
        hp_map[3 * (size_t)h + 2] = kWave;
      }
      for (uint32_t ch = 0; ch < nch; ++ch, ++item) {
        ItemDesc d;
        d.hp_lo = h0 + w * kWave;
        d.hp_n = min((uint32_t)kWave, nhp - w * kWave);
        d.first = first;
        d.nchunks = nch;
        const uint32_t lo = ch * kChunk, hi = min(T, lo + kChunk);
        d.ncand = hi > lo ? hi - lo : 0u;
        d.chunk = ch;
        uint32_t np = 0, pre = 0;
        for (int c = 0; c < 9; ++c) {
          const uint32_t a = max(pre, lo), e = min(pre + len[c], hi);
          if (e > a) {
            d.src[np] = beg[c] + (a - pre);
            d.len[np] = e - a;
            ++np;
          }
          pre += len[c];
        }
        for (uint32_t p = np; p < 9; ++p) d.src[p] = d.len[p] = 0;
        d.npieces = np;
        d.pad = 0;
        d.pad2[0] = d.pad2[1] = 0;
        desc[item] = d;
      }
    }
  }
}

// ------------------------------------------------------------------ the kernel
#ifndef FPPM_TILE_MINB
#define FPPM_TILE_MINB 2
#endif
#ifndef FPPM_TILE_MINB
#define FPPM_TILE_MINB 2
#endif


template <int GMAX, int CH>
__host__ __device__ constexpr size_t tile_dyn_smem_bytes() {
  return (size_t)kChunk * 64 + (size_t)kMaxFrag * partial_size(GMAX, CH) * sizeof(double);
}

constexpr uint32_t kNoEntry = 0xffffffffu;

__device__ __forceinline__ float4 lds128(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(addr));
  return v;
}

template <int GMAX, int CH>
__global__ void __launch_bounds__(kTileThreads, FPPM_TILE_MINB) k_gather_tiles(const GatherArgs A,
                                                                              const TileArgs T) {
  constexpr int PS = partial_size(GMAX, CH);
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float4 *s_rec0 = reinterpret_cast<float4 *>(smem_raw);
  double *s_frag = reinterpret_cast<double *>(smem_raw + (size_t)kChunk * 64);
  __shared__ Hit s_hit[kWave];
  __shared__ uint32_t s_q[kTileWarps][kQueue];  // ring: survivor = index | (sector or exact) << 16
  __shared__ uint32_t s_frag_hp[kMaxFrag];
  __shared__ ItemDesc s_desc;
  __shared__ __align__(8) uint64_t s_bar;
  __shared__ uint32_t s_item;

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t lt = (1u << lane) - 1u;
  uint32_t *q = s_q[warp];
  const uint32_t r0 = smem_u32(smem_raw);       // rec0 .. rec3 in 16-B strides
  const uint32_t r1 = r0 + kChunk * 16u, r2 = r1 + kChunk * 16u, r3 = r2 + kChunk * 16u;
  const uint32_t total_items = *T.total_items;
  if (threadIdx.x == 0) {
    mbar_init(&s_bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  uint32_t phase = 0;
  uint32_t my_cand = 0, my_exact = 0, my_amb = 0, my_acc = 0;

  for (;;) {
    if (threadIdx.x == 0) s_item = atomicAdd(A.work, 1u);
    __syncthreads();
    const uint32_t item = s_item;
    if (item >= total_items) break;
    if (threadIdx.x < sizeof(ItemDesc) / 4)
      reinterpret_cast<uint32_t *>(&s_desc)[threadIdx.x] =
          reinterpret_cast<const uint32_t *>(T.desc + item)[threadIdx.x];
    if (threadIdx.x < kMaxFrag) s_frag_hp[threadIdx.x] = kNoEntry;
    __syncthreads();
    const uint32_t ncand = s_desc.ncand, hp_n = s_desc.hp_n;
    if (threadIdx.x == 0 && ncand) {
      fence_proxy_async_smem();
      mbar_arrive_expect_tx(&s_bar, ncand * 64u);
      uint32_t off = 0;
      for (uint32_t p = 0; p < s_desc.npieces; ++p) {
        const uint32_t src = s_desc.src[p], n = s_desc.len[p];
        bulk_g2s(s_rec0 + off, A.rec0 + src, n * 16u, &s_bar);
        bulk_g2s(s_rec0 + kChunk + off, A.rec1 + src, n * 16u, &s_bar);
        bulk_g2s(s_rec0 + 2 * kChunk + off, A.rec2 + src, n * 16u, &s_bar);
        bulk_g2s(s_rec0 + 3 * kChunk + off, A.rec3 + src, n * 16u, &s_bar);
        off += n;
      }
    }
    if (threadIdx.x < hp_n) make_hit(A, T.hp_order[s_desc.hp_lo + threadIdx.x], s_hit[threadIdx.x]);
    __syncthreads();
    if (ncand) {
      mbar_wait(&s_bar, phase);
      phase ^= 1u;
    }

    // ---- balanced split of the (hit point x candidate) space over warps:
    // warp w owns flattened positions [w*W/8, (w+1)*W/8), i.e. a few
    // contiguous (hit point, candidate range) fragments.
    const uint32_t W = hp_n * ncand;
    const uint32_t f0 = (uint32_t)(((unsigned long long)W * warp) / kTileWarps);
    const uint32_t f1 = (uint32_t)(((unsigned long long)W * (warp + 1)) / kTileWarps);
    for (uint32_t f = f0; f < f1;) {
      const uint32_t k = f / ncand;
      const uint32_t ib = f - k * ncand;
      const uint32_t ie = min(ncand, f1 - k * ncand);
      f = k * ncand + ie;
      const Hit &Hs = s_hit[k];
      const HitF F = hitf(Hs, A.na, A.ns);
      // n = +z gives u = (1,-0,-0), v = (-0,1,-0): the fp32 plane coordinates
      // are exactly (dx, dy); an fp32-exact center has a zero low part.
      const bool planar = F.fast && Hs.nx == 0.0 && Hs.ny == 0.0 && Hs.nz == 1.0;
      const bool lo_zero = F.clx == 0.0f && F.cly == 0.0f && F.clz == 0.0f;
      uint32_t cnt[GMAX];
      double sm[CH][GMAX], sq[CH][GMAX];
#pragma unroll
      for (int g = 0; g < GMAX; ++g) {
        cnt[g] = 0;
#pragma unroll
        for (int c = 0; c < CH; ++c) { sm[c][g] = 0.0; sq[c][g] = 0.0; }
      }
      double p0 = 0.0, p1 = 0.0, p2 = 0.0;
      uint32_t qh = 0, qt = 0, base = ib;  // ring head / tail (warp-uniform)

      // One loop, one flush site: test rounds (kUnroll candidates per lane)
      // append survivors to the warp queue while fewer than 32 are pending;
      // otherwise 32 survivors are flushed with all lanes busy.
      for (;;) {
        if (qt - qh < 32 && base < ie) {
          uint32_t ent[kUnroll];
          float4 a[kUnroll];
#pragma unroll
          for (int u = 0; u < kUnroll; ++u) {
            const uint32_t i = base + u * 32 + lane;
            a[u] = lds128(r0 + (i < ie ? i : ib) * 16u);
          }
#pragma unroll
          for (int u = 0; u < kUnroll; ++u) {
            const uint32_t i = base + u * 32 + lane;
            ent[u] = i < ie && ball_pass(F, lo_zero, a[u], A.max_depth) ? i : kNoEntry;
            my_cand += i < ie ? 1u : 0u;
          }
          base += 32 * kUnroll;
#pragma unroll
          for (int u = 0; u < kUnroll; ++u) {
            const uint32_t m = __ballot_sync(kFull, ent[u] != kNoEntry);
            if (ent[u] != kNoEntry) q[(qt + __popc(m & lt)) & (kQueue - 1)] = ent[u];
            qt += __popc(m);
          }
          continue;
        }
        if (qt == qh) break;
        // ---- flush min(qn, 32) survivors, one per lane
        __syncwarp();
        const uint32_t n = qt - qh < 32 ? qt - qh : 32u;
        bool acc = false, cos_pos = false;
        int sector = 0;
        float4 c2 = make_float4(0.f, 0.f, 0.f, 0.f), c3 = c2;
        if ((uint32_t)lane < n) {
          const uint32_t i = q[(qh + lane) & (kQueue - 1)];
          const float4 a = lds128(r0 + i * 16u);
          const float4 b = lds128(r1 + i * 16u);
          c2 = lds128(r2 + i * 16u);
          c3 = lds128(r3 + i * 16u);
          float dx = a.x - F.chx, dy = a.y - F.chy, dz = a.z - F.chz;
          if (!lo_zero) {
            dx -= F.clx;
            dy -= F.cly;
            dz -= F.clz;
          }
          const float d2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
          float yu = dx, yv = dy;
          if (!planar) {
            yu = fmaf(dx, F.ufx, fmaf(dy, F.ufy, dz * F.ufz));
            yv = fmaf(dx, F.vfx, fmaf(dy, F.vfy, dz * F.vfz));
          }
          const float yy = fmaf(yu, yu, yv * yv);
          // disk (integrator.cpp:399): certain reject above the band
          const bool keep = yy <= F.lim_hi;
          bool ex = !(F.fast && d2 < F.lim_lo && yy < F.lim_lo);
          ex = !fast_sector(F, yu, yv, yy, sector) || ex;
          bool guard_ok = true;
          if (planar) {
            // n = +z: dot(p.n, n) = p.n.z and dot(wi, n) = wi.z exactly in fp64
            // when the x, y components are finite (integrator.cpp:397, bsdf.cpp:56)
            ex = ex || !(fabsf(b.x) < INFINITY && fabsf(b.y) < INFINITY && fabsf(b.w) < INFINITY &&
                         fabsf(c2.x) < INFINITY);
            guard_ok = !(b.z < F.guard_ceil);
            cos_pos = !(c2.y <= 0.0f);
          } else {
            const float gd = fmaf(b.x, F.nfx, fmaf(b.y, F.nfy, b.z * F.nfz));
            const float gb =
                2e-6f * (fabsf(b.x * F.nfx) + fabsf(b.y * F.nfy) + fabsf(b.z * F.nfz)) + 1e-30f;
            guard_ok = !(gd < F.guard_f - gb);
            ex = ex || (guard_ok && !(gd >= F.guard_f + gb));
            const float ci = fmaf(b.w, F.nfx, fmaf(c2.x, F.nfy, c2.y * F.nfz));
            const float cb =
                2e-6f * (fabsf(b.w * F.nfx) + fabsf(c2.x * F.nfy) + fabsf(c2.y * F.nfz)) + 1e-30f;
            ex = ex || !(fabsf(ci) > cb);
            cos_pos = ci > 0.0f;
          }
          ex = ex && keep;  // a certain disk reject needs no exact check
          if (ex) {
            ++my_exact;
            const uint32_t fl = exact_pair_packed(Hs, a, b, c2, F.na, F.ns, A.guard);
            acc = (fl & 1u) != 0;
            cos_pos = (fl & 2u) != 0;
            my_amb += (fl >> 2) & 1u;
            sector = (int)(fl >> 8);
          } else {
            acc = keep && guard_ok;
          }
        }
        if (acc) {
          ++my_acc;
          const double pr = cos_pos ? (double)c2.z : 0.0, pg = cos_pos ? (double)c2.w : 0.0,
                       pb = cos_pos ? (double)c3.x : 0.0;
          p0 += pr;
          p1 += pg;
          p2 += pb;
          if constexpr (CH == 1) {
            double v;
            if (Hs.gray) {
              const double L = __longlong_as_double(((long long)__float_as_uint(c3.w) << 32) |
                                                    __float_as_uint(c3.z));
              v = cos_pos ? Hs.K0 * L : 0.0;
            } else {
              v = elum(dm(Hs.K0, pr), dm(Hs.K1, pg), dm(Hs.K2, pb));
            }
            acc_pred<GMAX>(sm[0], sq[0], sector, v, v * v);
          } else {
            const double v0 = dm(Hs.K0, pr), v1 = dm(Hs.K1, pg), v2 = dm(Hs.K2, pb);
            acc_pred<GMAX>(sm[0], sq[0], sector, v0, v0 * v0);
            acc_pred<GMAX>(sm[1], sq[1], sector, v1, v1 * v1);
            acc_pred<GMAX>(sm[2], sq[2], sector, v2, v2 * v2);
          }
#pragma unroll
          for (int g = 0; g < GMAX; ++g) cnt[g] += sector == g ? 1u : 0u;
        }
        qh += n;
        __syncwarp();
      }

      // ---- fragment partial: fixed-order warp reduction into smem slot k + warp
#pragma unroll
      for (int g = 0; g < GMAX; ++g) {
        cnt[g] = warp_sum(cnt[g]);
#pragma unroll
        for (int c = 0; c < CH; ++c) {
          sm[c][g] = warp_sum(sm[c][g]);
          sq[c][g] = warp_sum(sq[c][g]);
        }
      }
      p0 = warp_sum(p0);
      p1 = warp_sum(p1);
      p2 = warp_sum(p2);
      if (lane == 0) {
        const uint32_t slot = k + warp;
        double *pp = s_frag + (size_t)slot * PS;
#pragma unroll
        for (int g = 0; g < GMAX; ++g) pp[g] = (double)cnt[g];
#pragma unroll
        for (int c = 0; c < CH; ++c)
#pragma unroll
          for (int g = 0; g < GMAX; ++g) {
            pp[GMAX + c * GMAX + g] = sm[c][g];
            pp[GMAX + CH * GMAX + c * GMAX + g] = sq[c][g];
          }
        pp[GMAX + 2 * CH * GMAX] = p0;
        pp[GMAX + 2 * CH * GMAX + 1] = p1;
        pp[GMAX + 2 * CH * GMAX + 2] = p2;
        s_frag_hp[slot] = k;
      }
      __syncwarp();
    }
    __syncthreads();

    // ---- combine fragments per hit point (slots k .. k+7, warp order) into
    // this item's partial; k_tile_finalize sums the wave's chunks in order.
    if (threadIdx.x < hp_n) {
      const uint32_t k = threadIdx.x;
      double *out = T.partials + ((size_t)item * kWave + k) * PS;
      for (int j = 0; j < PS; ++j) {
        double x = 0.0;
        for (int w = 0; w < kTileWarps; ++w)
          if (s_frag_hp[k + w] == k) x += s_frag[(size_t)(k + w) * PS + j];
        out[j] = x;
      }
    }
    __syncthreads();  // smem (records, hit points, descriptor) reused by the next item
  }

  // ------------------------------------------------------ block totals
  __shared__ unsigned long long s_c[4];
  if (threadIdx.x == 0) s_c[0] = s_c[1] = s_c[2] = s_c[3] = 0;
  __syncthreads();
  atomicAdd(&s_c[0], (unsigned long long)my_acc);
  atomicAdd(&s_c[1], (unsigned long long)my_cand);
  atomicAdd(&s_c[2], (unsigned long long)my_exact);
  atomicAdd(&s_c[3], (unsigned long long)my_amb);
  __syncthreads();
  if (threadIdx.x == 0) {
    atomicAdd(&A.counters[0], s_c[0]);
    atomicAdd(&A.counters[1], s_c[1]);
    atomicAdd(&A.counters[2], s_c[2]);
    atomicAdd(&A.counters[3], s_c[3]);
  }
}

// One thread per hit point: sum the wave's chunk partials in chunk order
// (deterministic), pool with the region state and run end_iteration.
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
      const double *pp = T.partials + ((size_t)pbase + (size_t)ch * stride) * PS;
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

// ------------------------------------------------------------------ launchers
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
  const unsigned long long n_ext =
      (unsigned long long)(g.nx + 2) * (unsigned long long)(g.ny + 2) * (unsigned long long)(g.nz + 2);
  if (n_ext + 1 >= 0xffffffffull) return cudaErrorInvalidValue;
  k_hp_bin<<<blocks_for(A.H, 256, sms, 16), 256, 0, s>>>(A.pos, A.gathered, A.H, A.grid, S.sort.keys_a,
                                                         S.sort.vals_a);
  note_launches(1);
  uint32_t bits = 1;
  while (bits < 32 && (1ull << bits) < n_ext + 1) ++bits;
  uint32_t *skeys, *svals;
  cudaError_t e = radix_sort_pairs(s, S.sort, A.H, bits, &skeys, &svals);
  *order = svals;
  return e;
}

cudaError_t tile_schedule_bins(cudaStream_t s, const GatherArgs &A, TileSched &S,
                               const GridHeader &g, int sms, uint32_t chunk, uint32_t *nb_out) {
  const unsigned long long n_ext =
      (unsigned long long)(g.nx + 2) * (unsigned long long)(g.ny + 2) * (unsigned long long)(g.nz + 2);
  if (n_ext + 1 >= 0xffffffffull) return cudaErrorInvalidValue;
  const uint32_t nb = (uint32_t)n_ext + 1;  // + "no candidates" bucket (key n_ext)
  *nb_out = nb;
  k_hp_bin<<<blocks_for(A.H, 256, sms, 16), 256, 0, s>>>(A.pos, A.gathered, A.H, A.grid,
                                                         S.sort.keys_a, S.sort.vals_a);
  note_launches(1);
  uint32_t bits = 1;
  while (bits < 32 && (1ull << bits) < (unsigned long long)nb) ++bits;
  uint32_t *skeys, *svals;
  cudaError_t e = radix_sort_pairs(s, S.sort, A.H, bits, &skeys, &svals);
  if (e != cudaSuccess) return e;
  S.hp_order = svals;
  if ((unsigned long long)nb > 4ull * A.H)
    k_bucket_start_bsearch<<<blocks_for(nb + 1, 256, sms, 16), 256, 0, s>>>(skeys, A.H, nb, S.hp_start);
  else
    k_bucket_start<<<blocks_for(A.H, 256, sms, 16), 256, 0, s>>>(skeys, A.H, nb, S.hp_start);
  k_bucket_items<<<blocks_for(nb + 1, 256, sms, 16), 256, 0, s>>>(
      S.hp_start, nb, A.grid, A.cell_start, S.items, S.chunks, chunk, S.nonempty);
  const uint32_t nt = (nb + 1 + kScanTile - 1) / kScanTile;
  k_scan_tiles<<<nt, 256, 0, s>>>(S.items, nb + 1, S.scan_tmp);
  k_scan_top<<<1, 256, 0, s>>>(S.scan_tmp, nt);
  k_scan_apply<<<nt, 256, 0, s>>>(S.items, nb + 1, S.scan_tmp, S.item_base);
  note_launches(5);
  return cudaGetLastError();
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

cudaError_t tile_schedule_items(cudaStream_t s, const GatherArgs &A, TileSched &S, uint32_t nb,
                                int sms, uint32_t chunk) {
  k_item_desc<<<blocks_for(nb, 128, sms, 16), 128, 0, s>>>(S.hp_start, nb, A.grid, A.cell_start,
                                                           S.items, S.chunks, S.item_base,
                                                           S.hp_order, S.desc, S.hp_map, chunk);
  note_launches(1);
  return cudaGetLastError();
}

template <int GMAX, int CH>
static cudaError_t launch_tiles(cudaStream_t s, const GatherArgs &A, const TileArgs &T, int sms) {
  const size_t smem = tile_dyn_smem_bytes<GMAX, CH>();
  cudaError_t e = cudaFuncSetAttribute(k_gather_tiles<GMAX, CH>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_gather_tiles<GMAX, CH>, kTileThreads,
                                                    smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  k_gather_tiles<GMAX, CH><<<sms * per_sm, kTileThreads, smem, s>>>(A, T);
  note_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_gather_tiles(cudaStream_t s, const GatherArgs &A, const TileArgs &T, int C,
                                int sms) {
  const int G = A.na * A.ns;
  if (C == 1) {
    if (G <= 4) return launch_tiles<4, 1>(s, A, T, sms);
    if (G <= 8) return launch_tiles<8, 1>(s, A, T, sms);
    if (G <= 12) return launch_tiles<12, 1>(s, A, T, sms);
    if (G <= 16) return launch_tiles<16, 1>(s, A, T, sms);
    return launch_tiles<32, 1>(s, A, T, sms);
  }
  if (G <= 4) return launch_tiles<4, 3>(s, A, T, sms);
  if (G <= 8) return launch_tiles<8, 3>(s, A, T, sms);
  if (G <= 12) return launch_tiles<12, 3>(s, A, T, sms);
  return launch_tiles<32, 3>(s, A, T, sms);
}

template <int GMAX, int CH>
static cudaError_t launch_fin(cudaStream_t s, const GatherArgs &A, const TileArgs &T, int sms) {
  if (A.H == 0) return cudaSuccess;
  k_tile_finalize<GMAX, CH><<<blocks_for(A.H, 128, sms, 8), 128, 0, s>>>(A, T);
  note_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_tile_finalize(cudaStream_t s, const GatherArgs &A, const TileArgs &T, int C,
                                 int sms) {
  const int G = A.na * A.ns;
  if (C == 1) {
    if (G <= 4) return launch_fin<4, 1>(s, A, T, sms);
    if (G <= 8) return launch_fin<8, 1>(s, A, T, sms);
    if (G <= 12) return launch_fin<12, 1>(s, A, T, sms);
    if (G <= 16) return launch_fin<16, 1>(s, A, T, sms);
    return launch_fin<32, 1>(s, A, T, sms);
  }
  if (G <= 4) return launch_fin<4, 3>(s, A, T, sms);
  if (G <= 8) return launch_fin<8, 3>(s, A, T, sms);
  if (G <= 12) return launch_fin<12, 3>(s, A, T, sms);
  return launch_fin<32, 3>(s, A, T, sms);
}

size_t tile_partial_doubles(int G, int C) {
  const int gmax = G <= 4 ? 4 : G <= 8 ? 8 : G <= 12 ? 12 : G <= 16 && C == 1 ? 16 : 32;
  return (size_t)partial_size(gmax, C) * kWave;
}

}  // namespace fppm_b200
