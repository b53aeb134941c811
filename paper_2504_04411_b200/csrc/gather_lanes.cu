// gather_lanes.cu -- gather + F-test for dense frames: lanes = hit points.
//
// All hit points whose center falls in one grid cell (a "home cell") share
// the same 27-cell candidate set (photon_map.cpp:65-77).  When cells hold tens
// of hit points (raster gather points on a surface, BASELINE configs 1-2),
// one warp takes an item = (home cell, <= 32 hit points, <= kLaneChunk
// candidates) and gives every lane one hit point:
//
//   stage   the warp streams its candidates through a private shared-memory
//           window (kLSub records of 4 x 16 B), one TMA bulk copy per
//           contiguous piece, completing on the warp's own mbarrier;
//   test    candidates are read with broadcast ld.shared (one wavefront per
//           candidate for the whole warp) and ball/depth-tested by every lane
//           against its own hit point in fp32 with error bands; survivors are
//           appended to the lane's private queue;
//   flush   whenever a queue may overflow, every lane drains its own queue:
//           disk, sector, guard, cos_i in fp32 with bands (the fp64 exact
//           path otherwise) and fp64 accumulation into the lane's sector
//           registers -- no cross-lane reduction is ever needed.
//
// Each item writes one partial per hit point; k_tile_finalize (gather_tile.cu)
// sums a wave's chunk partials in chunk order and runs end_iteration.  Warps
// are fully independent (no CTA barriers); items come from a global counter.
#include "common.cuh"
#include "gather.cuh"
#include "gather_dev.cuh"

namespace fppm_b200 {

constexpr int kLWarps = 8;
constexpr int kLThreads = kLWarps * kWarp;
constexpr int kLSub = 160;    // candidates staged per warp window (10 KB)
constexpr int kLQueue = 16;   // survivor queue depth per lane
constexpr int kLStep = 4;     // candidates tested per step
constexpr int kLWave = 32;

constexpr size_t kLWarpBytes = (size_t)kLSub * 64 + (size_t)kLQueue * 32 * 4 + sizeof(ItemDesc) + 16;
constexpr size_t lanes_smem_bytes() { return kLWarpBytes * kLWarps; }

__device__ __forceinline__ float4 lds128_l(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(addr));
  return v;
}
__device__ __forceinline__ void sts32(uint32_t addr, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(addr), "r"(v));
}
__device__ __forceinline__ uint32_t lds32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}

// fp32 parameters of one hit point (HitF subset of make_hit; gather_dev.cuh)
__device__ __forceinline__ void lane_hit(const GatherArgs &A, uint32_t h, HitF &F, bool &planar,
                                         bool &lo_zero, bool &gray, double &K0) {
  const double r = A.radius[h];
  const double r2 = dm(r, r);
  const double3 c = A.pos[h];
  const double3 n = A.nrm[h];
  double3 u, v;
  eframe(n.x, n.y, n.z, u, v);
  const double3 K = A.K[h];
  K0 = K.x;
  gray = K.x == K.y && K.y == K.z;
  F.eye = A.eye_depth[h];
  F.chx = __double2float_rn(c.x);
  F.chy = __double2float_rn(c.y);
  F.chz = __double2float_rn(c.z);
  F.clx = __double2float_rn(c.x - (double)F.chx);
  F.cly = __double2float_rn(c.y - (double)F.chy);
  F.clz = __double2float_rn(c.z - (double)F.chz);
  F.nfx = (float)n.x; F.nfy = (float)n.y; F.nfz = (float)n.z;
  F.ufx = (float)u.x; F.ufy = (float)u.y; F.ufz = (float)u.z;
  F.vfx = (float)v.x; F.vfy = (float)v.y; F.vfz = (float)v.z;
  const float r2f = (float)r2;
  F.band_y = 1e-5f * (float)r;
  F.guard_f = (float)A.guard;
  F.guard_ceil = __double2float_ru(A.guard);
  F.qa_scale = (float)A.na / r2f;
  F.r = (float)r;
  F.na = A.na;
  F.ns = A.ns;
  const double cmax = fmax(fabs(c.x), fmax(fabs(c.y), fabs(c.z)));
  const double nn = edot(n.x, n.y, n.z, n.x, n.y, n.z);
  F.fast = r2f > 1e-30f && r2f < 1e30f && cmax <= 1e6 * r && nn > 0.999 && nn < 1.001;
  F.lim_hi = F.fast ? r2f + 2e-5f * r2f : __int_as_float(0x7f800000);
  F.lim_lo = F.fast ? r2f - 2e-5f * r2f : -1.0f;
  planar = F.fast && n.x == 0.0 && n.y == 0.0 && n.z == 1.0;
  lo_zero = F.clx == 0.0f && F.cly == 0.0f && F.clz == 0.0f;
}

// exact path on demand: rebuild the full fp64 hit state (rare)
static __device__ __noinline__ uint32_t lane_exact(const GatherArgs &A, uint32_t h, float4 a,
                                                  float4 b, float4 c2) {
  Hit H;
  make_hit(A, h, H);
  return exact_pair_packed(H, a, b, c2, A.na, A.ns, A.guard);
}

template <int GMAX, int CH>
__global__ void __launch_bounds__(kLThreads, 2) k_gather_lanes(const GatherArgs A, const TileArgs T) {
  constexpr int PS = partial_size(GMAX, CH);
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned char *wb = smem_raw + (size_t)warp * kLWarpBytes;
  float4 *w_rec = reinterpret_cast<float4 *>(wb);
  ItemDesc *w_desc = reinterpret_cast<ItemDesc *>(wb + (size_t)kLSub * 64 + (size_t)kLQueue * 128);
  uint64_t *w_bar = reinterpret_cast<uint64_t *>(w_desc + 1);
  const uint32_t r0 = smem_u32(w_rec);
  const uint32_t r1 = r0 + kLSub * 16u, r2 = r1 + kLSub * 16u, r3 = r2 + kLSub * 16u;
  const uint32_t qa = r0 + kLSub * 64u + lane * 4u;  // lane's queue column, stride 128 B
  const uint32_t total_items = *T.total_items;
  if (lane == 0) {
    mbar_init(w_bar, 1);
    fence_mbar_init();
  }
  __syncwarp();
  uint32_t phase = 0;
  uint32_t my_cand = 0, my_exact = 0, my_amb = 0, my_acc = 0;

  for (;;) {
    uint32_t item = 0;
    if (lane == 0) item = atomicAdd(A.work, 1u);
    item = __shfl_sync(kFull, item, 0);
    if (item >= total_items) break;
    if (lane < (int)(sizeof(ItemDesc) / 4))
      reinterpret_cast<uint32_t *>(w_desc)[lane] =
          reinterpret_cast<const uint32_t *>(T.desc + item)[lane];
    __syncwarp();
    const uint32_t hp_n = w_desc->hp_n, ncand = w_desc->ncand;
    const bool active = (uint32_t)lane < hp_n;
    const uint32_t h = active ? T.hp_order[w_desc->hp_lo + lane] : 0u;
    HitF F;
    bool planar = false, lo_zero = false, gray = false;
    double K0 = 0.0;
    lane_hit(A, h, F, planar, lo_zero, gray, K0);
    if (!active) F.lim_hi = -1.0f;  // rejects everything
    uint32_t cnt[GMAX];
    double sm[CH][GMAX], sq[CH][GMAX];
#pragma unroll
    for (int g = 0; g < GMAX; ++g) {
      cnt[g] = 0;
#pragma unroll
      for (int c = 0; c < CH; ++c) { sm[c][g] = 0.0; sq[c][g] = 0.0; }
    }
    double p0 = 0.0, p1 = 0.0, p2 = 0.0;

    for (uint32_t sub = 0; sub < ncand; sub += kLSub) {
      const uint32_t ns = min((uint32_t)kLSub, ncand - sub);
      __syncwarp();  // the previous window is fully consumed
      if (lane == 0) {
        fence_proxy_async_smem();
        mbar_arrive_expect_tx(w_bar, ns * 64u);
        uint32_t pre = 0, off = 0;
        for (uint32_t p = 0; p < w_desc->npieces; ++p) {
          const uint32_t plen = w_desc->len[p];
          const uint32_t lo = max(pre, sub), hi = min(pre + plen, sub + ns);
          if (hi > lo) {
            const uint32_t src = w_desc->src[p] + (lo - pre), n = hi - lo;
            bulk_g2s(w_rec + off, A.rec0 + src, n * 16u, w_bar);
            bulk_g2s(w_rec + kLSub + off, A.rec1 + src, n * 16u, w_bar);
            bulk_g2s(w_rec + 2 * kLSub + off, A.rec2 + src, n * 16u, w_bar);
            bulk_g2s(w_rec + 3 * kLSub + off, A.rec3 + src, n * 16u, w_bar);
            off += n;
          }
          pre += plen;
        }
      }
      mbar_wait(w_bar, phase);
      phase ^= 1u;

      uint32_t qn = 0;  // this lane's queue length
      for (uint32_t c = 0;; c += kLStep) {
        const bool more = c < ns;
        if (more) {
#pragma unroll
          for (int u = 0; u < kLStep; ++u) {
            const uint32_t i = c + u;
            const float4 a = lds128_l(r0 + (i < ns ? i : 0u) * 16u);  // broadcast
            if (i < ns && ball_pass(F, lo_zero, a, A.max_depth)) {
              sts32(qa + qn * 128u, i);
              ++qn;
            }
          }
          my_cand += active ? (uint32_t)min((uint32_t)kLStep, ns - c) : 0u;
        }
        const bool flush_now = __any_sync(kFull, qn > kLQueue - kLStep) || (!more && __any_sync(kFull, qn > 0));
        if (flush_now) {
          const uint32_t qmax = __reduce_max_sync(kFull, qn);
          for (uint32_t j = 0; j < qmax; ++j) {
            bool acc = false, cos_pos = false;
            int sector = 0;
            float4 c2 = make_float4(0.f, 0.f, 0.f, 0.f), c3 = c2;
            if (j < qn) {
              const uint32_t i = lds32(qa + j * 128u);
              const float4 a = lds128_l(r0 + i * 16u);
              const float4 b = lds128_l(r1 + i * 16u);
              c2 = lds128_l(r2 + i * 16u);
              c3 = lds128_l(r3 + i * 16u);
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
              const bool keep = yy <= F.lim_hi;  // disk (integrator.cpp:399)
              bool ex = !(F.fast && d2 < F.lim_lo && yy < F.lim_lo);
              ex = !fast_sector(F, yu, yv, yy, sector) || ex;
              bool guard_ok = true;
              if (planar) {
                // n = +z: dot(p.n, n) = p.n.z and dot(wi, n) = wi.z exactly in
                // fp64 when the x, y components are finite
                ex = ex || !(fabsf(b.x) < INFINITY && fabsf(b.y) < INFINITY &&
                             fabsf(b.w) < INFINITY && fabsf(c2.x) < INFINITY);
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
              ex = ex && keep;
              if (ex) {
                ++my_exact;
                const uint32_t fl = lane_exact(A, h, a, b, c2);
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
                if (gray) {
                  const double L = __longlong_as_double(((long long)__float_as_uint(c3.w) << 32) |
                                                        __float_as_uint(c3.z));
                  v = cos_pos ? K0 * L : 0.0;
                } else {
                  const double3 K = A.K[h];
                  v = elum(dm(K.x, pr), dm(K.y, pg), dm(K.z, pb));
                }
                acc_pred<GMAX>(sm[0], sq[0], sector, v, v * v);
              } else {
                const double3 K = A.K[h];
                const double v0 = dm(K.x, pr), v1 = dm(K.y, pg), v2 = dm(K.z, pb);
                acc_pred<GMAX>(sm[0], sq[0], sector, v0, v0 * v0);
                acc_pred<GMAX>(sm[1], sq[1], sector, v1, v1 * v1);
                acc_pred<GMAX>(sm[2], sq[2], sector, v2, v2 * v2);
              }
#pragma unroll
              for (int g = 0; g < GMAX; ++g) cnt[g] += sector == g ? 1u : 0u;
            }
          }
          qn = 0;
        }
        if (!more) break;
      }
    }

    // ---- this item's partial for the lane's hit point
    if (active) {
      double *pp = T.partials + ((size_t)item * kLWave + lane) * PS;
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
    }
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

template <int GMAX, int CH>
static cudaError_t launch_l(cudaStream_t s, const GatherArgs &A, const TileArgs &T, int sms) {
  const size_t smem = lanes_smem_bytes();
  cudaError_t e = cudaFuncSetAttribute(k_gather_lanes<GMAX, CH>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_gather_lanes<GMAX, CH>, kLThreads, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  k_gather_lanes<GMAX, CH><<<sms * per_sm, kLThreads, smem, s>>>(A, T);
  note_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_gather_lanes(cudaStream_t s, const GatherArgs &A, const TileArgs &T, int C,
                                int sms) {
  const int G = A.na * A.ns;
  if (C == 1) {
    if (G <= 4) return launch_l<4, 1>(s, A, T, sms);
    if (G <= 8) return launch_l<8, 1>(s, A, T, sms);
    if (G <= 12) return launch_l<12, 1>(s, A, T, sms);
    if (G <= 16) return launch_l<16, 1>(s, A, T, sms);
    return launch_l<32, 1>(s, A, T, sms);
  }
  if (G <= 4) return launch_l<4, 3>(s, A, T, sms);
  if (G <= 8) return launch_l<8, 3>(s, A, T, sms);
  if (G <= 12) return launch_l<12, 3>(s, A, T, sms);
  return launch_l<32, 3>(s, A, T, sms);
}

}  // namespace fppm_b200
