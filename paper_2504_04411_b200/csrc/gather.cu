#include <algorithm>
// gather.cu -- warp-per-hit-point gather (the "warp" variant) + the
// explicit-sample / end_iteration kernels of the GatherRegion mirror.
//
// Warp variant: one warp owns one hit point (GatherRegion) at a time, pulled
// from a global work counter, and streams the 9 contiguous (dx, dy) column
// ranges of the hit point's 27-cell neighbourhood (photon_map.cpp:65-77)
// straight from global memory, one candidate per lane.  It needs no
// scheduling pass, which suits sparse 3D frames with a few hit points per
// cell; the tiled kernel (gather_tile.cu) is the default for dense frames.
// Predicates, sectors and the fused end-of-iteration are shared with the
// tiled kernel (gather_dev.cuh).
#include "common.cuh"
#include "gather.cuh"
#include "gather_dev.cuh"

namespace fppm_b200 {

// One candidate of a hit point (photon_map.cpp:65-77 ball, gather_disk
// filters integrator.cpp:388-402, value :445-451 / VCM+ :607-615, sector and
// SectorStats::add); shared by the warp-per-hit-point and
// thread-per-hit-point kernels.
struct EyeVcm {
  double cos_o, cont, d_vcm, d_vm;
};

// Evaluates one candidate: false when the reference rejects it; otherwise the
// sector, the statistic values (luminance, or RGB for CH = 3) with their
// squares, and the flux addends (photon power for FPPM, the weighted value
// for VCM+).
template <int CH, class HT>
static __device__ __forceinline__ bool pair_tail(const GatherArgs &A, const HitF &F, const HT &Hs, uint32_t i,
                                                 const EyeVcm &E, float4 a, float4 b, float4 c2, float4 c3,
                                                 int &sector, double (&sv)[CH], double (&sw)[CH], double &f0,
                                                 double &f1, double &f2, uint32_t &my_exact, uint32_t &my_amb);

template <int CH>
static __device__ __forceinline__ bool pair_eval(const GatherArgs &A, const HitF &F, const Hit &Hs, uint32_t i,
                                                 const EyeVcm &E, int &sector, double (&sv)[CH],
                                                 double (&sw)[CH], double &f0, double &f1, double &f2,
                                                 uint32_t &my_exact, uint32_t &my_amb) {
  const float4 a = __ldg(&A.rec0[i]);
  if (!test_pair(F, a, A.max_depth)) return false;
  const float4 b = __ldg(&A.rec1[i]);
  const float4 c2 = __ldg(&A.rec2[i]);
  const float4 c3 = __ldg(&A.rec3[i]);
  return pair_tail<CH, Hit>(A, F, Hs, i, E, a, b, c2, c3, sector, sv, sw, f0, f1, f2, my_exact, my_amb);
}

// flush_pair + value of a candidate whose records are loaded
template <int CH, class HT>
static __device__ __forceinline__ bool pair_tail(const GatherArgs &A, const HitF &F, const HT &Hs, uint32_t i,
                                                 const EyeVcm &E, float4 a, float4 b, float4 c2, float4 c3,
                                                 int &sector, double (&sv)[CH], double (&sw)[CH], double &f0,
                                                 double &f1, double &f2, uint32_t &my_exact, uint32_t &my_amb) {
  bool cos_pos;
  if (!flush_pair(F, Hs, a, b, c2, A.guard, sector, cos_pos, my_exact, my_amb)) return false;
  double v0, v1, v2;
  if (A.vcm) {
    // merge callback (integrator.cpp:609-616): f and the pdfs of
    // Bsdf::eval (bsdf.cpp:53-63), merge weight, val = thr * f * p.thr * w
    const double ci = edot((double)b.w, (double)c2.x, (double)c2.y, Hs.nx, Hs.ny, Hs.nz);
    const bool black = E.cos_o <= 0.0 || ci <= 0.0;
    const double pf = black ? 0.0 : (ci > 0.0 ? dm(ci, kInvPi) : 0.0);
    const double prv = black ? 0.0 : (E.cos_o > 0.0 ? dm(E.cos_o, kInvPi) : 0.0);
    const double w = mis_weight_merge_dev(A.mis_n_vm, A.mis_beta, Hs.r, E.d_vcm, E.d_vm, A.p_vcm[i],
                                          A.p_vm[i], dm(pf, E.cont), dm(prv, A.p_cont[i]));
    const double k0 = ci <= 0.0 ? dm(Hs.K0, 0.0) : Hs.K0, k1 = ci <= 0.0 ? dm(Hs.K1, 0.0) : Hs.K1,
                 k2 = ci <= 0.0 ? dm(Hs.K2, 0.0) : Hs.K2;
    v0 = dm(dm(k0, (double)c2.z), w);
    v1 = dm(dm(k1, (double)c2.w), w);
    v2 = dm(dm(k2, (double)c3.x), w);
    f0 = v0; f1 = v1; f2 = v2;
  } else {
    const double pr = cos_pos ? (double)c2.z : 0.0, pg = cos_pos ? (double)c2.w : 0.0,
                 pb_ = cos_pos ? (double)c3.x : 0.0;
    f0 = pr; f1 = pg; f2 = pb_;
    v0 = dm(Hs.K0, pr);
    v1 = dm(Hs.K1, pg);
    v2 = dm(Hs.K2, pb_);
  }
  if constexpr (CH == 1) {
    sv[0] = elum(v0, v1, v2);
    sw[0] = dm(sv[0], sv[0]);
  } else {
    sv[0] = v0; sv[1] = v1; sv[2] = v2;
    sw[0] = dm(v0, v0); sw[1] = dm(v1, v1); sw[2] = dm(v2, v2);
  }
  return true;
}

template <int GMAX, int CH>
static __device__ __forceinline__ void pair_accumulate(const GatherArgs &A, const HitF &F, const Hit &Hs,
                                                       uint32_t i, const EyeVcm &E, uint32_t (&cnt)[GMAX],
                                                       double (&sm)[CH][GMAX], double (&sq)[CH][GMAX],
                                                       double &p0, double &p1, double &p2, uint32_t &my_acc,
                                                       uint32_t &my_exact, uint32_t &my_amb) {
  int sector;
  double sv[CH], sw[CH], f0, f1, f2;
  if (!pair_eval<CH>(A, F, Hs, i, E, sector, sv, sw, f0, f1, f2, my_exact, my_amb)) return;
  ++my_acc;
  p0 = da(p0, f0); p1 = da(p1, f1); p2 = da(p2, f2);
#pragma unroll
  for (int g = 0; g < GMAX; ++g) cnt[g] += sector == g ? 1u : 0u;
#pragma unroll
  for (int c = 0; c < CH; ++c) acc_pred<GMAX>(sm[c], sq[c], sector, sv[c], sw[c]);
}

template <int GMAX, int CH>
__global__ void __launch_bounds__(kGatherThreads) k_gather_test(const GatherArgs A) {
  const int lane = threadIdx.x & 31;
  const GridHeader grid = *A.grid;
  __shared__ Hit s_hit[kGatherThreads / 32];
  Hit &Hs = s_hit[threadIdx.x >> 5];
  uint32_t my_cand = 0, my_exact = 0, my_amb = 0, my_acc = 0;
  double my_rmax = 0.0;
  uint32_t my_tested = 0, my_rejected = 0;

  for (;;) {
    uint32_t h = 0;
    if (lane == 0) h = atomicAdd(A.work, 1u);
    h = __shfl_sync(kFull, h, 0);
    if (h >= A.H) break;
    if (lane == 0) make_hit(A, h, Hs);
    __syncwarp();
    const HitF F = hitf(Hs, A.na, A.ns);
    const bool gathered = A.gathered == nullptr || A.gathered[h] != 0;

    uint32_t cnt[GMAX];
    double sm[CH][GMAX], sq[CH][GMAX];
#pragma unroll
    for (int g = 0; g < GMAX; ++g) {
      cnt[g] = 0;
#pragma unroll
      for (int c = 0; c < CH; ++c) { sm[c][g] = 0.0; sq[c][g] = 0.0; }
    }
    double p0 = 0.0, p1 = 0.0, p2 = 0.0;

    // VCM+ eye Bsdf terms: cos_o (bsdf.cpp:34) and continuation probability
    // (bsdf.cpp:42-51, std::max / std::min semantics)
    double v_cos_o = 0.0, v_cont = 0.0, v_vcm = 0.0, v_vm = 0.0;
    if (A.vcm) {
      const double3 wo = A.wo[h], al = A.alb[h];
      v_cos_o = edot(wo.x, wo.y, wo.z, Hs.nx, Hs.ny, Hs.nz);
      const double m1 = al.y < al.z ? al.z : al.y;
      const double amax = al.x < m1 ? m1 : al.x;
      v_cont = amax < 1.0 ? amax : 1.0;
      const double2 em = A.eye_mis[h];
      v_vcm = em.x;
      v_vm = em.y;
    }
    const EyeVcm eye{v_cos_o, v_cont, v_vcm, v_vm};
    if (gathered && grid.n > 0) {
      const long long ix = (long long)floor(dm(Hs.cx, grid.inv)) - grid.ix0;
      const long long iy = (long long)floor(dm(Hs.cy, grid.inv)) - grid.iy0;
      const long long iz = (long long)floor(dm(Hs.cz, grid.inv)) - grid.iz0;
      uint32_t rbeg = 0, rlen = 0;
      if (lane < 9) {
        const long long X = ix + lane / 3 - 1, Y = iy + lane % 3 - 1;
        const long long z0 = iz - 1 < 0 ? 0 : iz - 1;
        const long long z1 = iz + 1 >= grid.nz ? grid.nz - 1 : iz + 1;
        if (X >= 0 && X < grid.nx && Y >= 0 && Y < grid.ny && z0 <= z1) {
          const unsigned long long k0 = (unsigned long long)((X * grid.ny + Y) * grid.nz + z0);
          const unsigned long long k1 = (unsigned long long)((X * grid.ny + Y) * grid.nz + z1);
          rbeg = A.cell_start[k0];
          rlen = A.cell_start[k1 + 1] - rbeg;
        }
      }
      uint32_t rend = rlen;
#pragma unroll
      for (int o = 1; o < 16; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, rend, o);
        if (lane >= o) rend += y;
      }
      const uint32_t total = __shfl_sync(kFull, rend, 8);
      const uint32_t rpre = rend - rlen;
      int cur = 0;
      for (uint32_t base = 0; base < total; base += 32) {
        const uint32_t idx = base + lane;
        for (;;) {
          const uint32_t e = __shfl_sync(kFull, rend, cur);
          const bool adv = idx >= e && cur < 8;
          if (!__any_sync(kFull, adv)) break;
          cur += adv ? 1 : 0;
        }
        const uint32_t pb = __shfl_sync(kFull, rbeg, cur);
        const uint32_t pp = __shfl_sync(kFull, rpre, cur);
        if (idx >= total) continue;
        const uint32_t i = pb + (idx - pp);
        ++my_cand;
        pair_accumulate<GMAX, CH>(A, F, Hs, i, eye, cnt, sm, sq, p0, p1, p2, my_acc, my_exact, my_amb);
      }
    }

#pragma unroll
    for (int g = 0; g < GMAX; ++g) {
      cnt[g] = warp_sum(cnt[g]);
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        sm[c][g] = warp_sum(sm[c][g]);
        sq[c][g] = warp_sum(sq[c][g]);
      }
    }
    p0 = warp_sum(p0); p1 = warp_sum(p1); p2 = warp_sum(p2);
    if (lane == 0)
      finalize_hit<GMAX, CH>(A, h, cnt, sm, sq, p0, p1, p2, my_tested, my_rejected, my_rmax);
    __syncwarp();
  }

  __shared__ unsigned long long s_c[4];
  __shared__ unsigned int s_tr[2];
  __shared__ unsigned long long s_rmax;
  if (threadIdx.x == 0) { s_c[0] = s_c[1] = s_c[2] = s_c[3] = 0; s_tr[0] = s_tr[1] = 0; s_rmax = 0; }
  __syncthreads();
  atomicAdd(&s_c[0], (unsigned long long)my_acc);
  atomicAdd(&s_c[1], (unsigned long long)my_cand);
  atomicAdd(&s_c[2], (unsigned long long)my_exact);
  atomicAdd(&s_c[3], (unsigned long long)my_amb);
  if (lane == 0) {
    atomicAdd(&s_tr[0], my_tested);
    atomicAdd(&s_tr[1], my_rejected);
    atomicMax(&s_rmax, (unsigned long long)__double_as_longlong(my_rmax));
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    atomicAdd(&A.counters[0], s_c[0]);
    atomicAdd(&A.counters[1], s_c[1]);
    atomicAdd(&A.counters[2], s_c[2]);
    atomicAdd(&A.counters[3], s_c[3]);
    atomicAdd(A.iter_tr, s_tr[0]);
    atomicAdd(A.iter_tr + 1, s_tr[1]);
    atomicMax(A.rmax_bits, s_rmax);
  }
}

// ---------------------------------------------------------------- sparse frames
// Thread per hit point, for sparse 3D frames (C3 / C4 camera hit points on
// the walls, a few candidates each): a warp's fixed cost per hit point
// (runs, reductions) would exceed its candidates, so here each thread walks
// the chord-clipped columns of its own fine box with the same pair code.
// Neighbouring threads hold nearby hit points (cell order), so their photon
// records share L1/L2 lines.
constexpr int kSparseThreads = 128;
// Candidates per step (U): 4 for the FPPM value, whose record loads then
// overlap; 1 for the VCM+ value, whose MIS weight makes the unrolled body
// outgrow the instruction cache (measured on C3 / C4: 3.45 vs 4.04 ms and
// 2.98 vs 5.23 ms per iteration's gathers).
template <int GMAX, int CH, int kSparseU>
#ifndef FPPM_SPARSE_MINB
#define FPPM_SPARSE_MINB 4
#endif
__global__ void __launch_bounds__(kSparseThreads, FPPM_SPARSE_MINB) k_gather_sparse(const GatherArgs A, const uint32_t *__restrict__ order,
                                                                   double *__restrict__ rows) {
  // per thread: its Hit (exact path) and its sector accumulators, indexed
  // [slot][thread] so a lane's dynamic sector index costs one LDS/STS
  extern __shared__ __align__(16) unsigned char s_raw[];
  const int G = A.na * A.ns, CG = G * CH;
  const int t = threadIdx.x;
  HitX *s_hit = reinterpret_cast<HitX *>(s_raw);
  double *s_sum = reinterpret_cast<double *>(s_hit + kSparseThreads);   // [CG][T]
  double *s_sq = s_sum + (size_t)CG * kSparseThreads;                     // [CG][T]
  uint32_t *s_cnt = reinterpret_cast<uint32_t *>(s_sq + (size_t)CG * kSparseThreads);  // [G][T]
  HitX &Hs = s_hit[t];
  const GridHeader grid = *A.grid;
  uint32_t my_cand = 0, my_exact = 0, my_amb = 0, my_acc = 0;
  for (uint32_t q = blockIdx.x * blockDim.x + t; q < A.H; q += gridDim.x * blockDim.x) {
    const uint32_t h = order ? order[q] : q;
    HitF F;
    {
      Hit H;
      make_hit(A, h, H);
      F = hitf(H, A.na, A.ns);
      Hs.cx = H.cx; Hs.cy = H.cy; Hs.cz = H.cz;
      Hs.nx = H.nx; Hs.ny = H.ny; Hs.nz = H.nz;
      Hs.u = H.u; Hs.v = H.v;
      Hs.r = H.r; Hs.r2 = H.r2;
      Hs.K0 = H.K0; Hs.K1 = H.K1; Hs.K2 = H.K2;
    }
    const bool gathered = A.gathered == nullptr || A.gathered[h] != 0;
    for (int k = 0; k < CG; ++k) {
      s_sum[k * kSparseThreads + t] = 0.0;
      s_sq[k * kSparseThreads + t] = 0.0;
    }
    for (int g = 0; g < G; ++g) s_cnt[g * kSparseThreads + t] = 0u;
    double p0 = 0.0, p1 = 0.0, p2 = 0.0;
    EyeVcm eye{0.0, 0.0, 0.0, 0.0};
    if (A.vcm) {
      const double3 wo = A.wo[h], al = A.alb[h];
      eye.cos_o = edot(wo.x, wo.y, wo.z, Hs.nx, Hs.ny, Hs.nz);
      const double m1 = al.y < al.z ? al.z : al.y;
      const double amax = al.x < m1 ? m1 : al.x;
      eye.cont = amax < 1.0 ? amax : 1.0;
      const double2 em = A.eye_mis[h];
      eye.d_vcm = em.x;
      eye.d_vm = em.y;
    }
    FBox fb = {0, -1, 0, -1, 0, -1};
    if (gathered && fine_box(grid, Hs.cx, Hs.cy, Hs.cz, Hs.r, fb)) {
      // the box's columns (27-neighbourhood, chord-clipped: gather_dev.cuh)
      const int ncol = run_count(grid, fb);
      const double cm = fmax(fabs(Hs.cx), fmax(fabs(Hs.cy), fabs(Hs.cz)));
      const double mrad = da(da(Hs.r, dm(Hs.r, 1e-9)), dm(cm, 4e-16));
#pragma unroll 1
      for (int col = 0; col < ncol; ++col) {
        unsigned long long k0, k1;
        if (!run_keys_clipped(grid, fb, col, Hs.cx, Hs.cy, Hs.cz, mrad, k0, k1)) continue;
        const uint32_t beg = __ldg(&A.cell_start[k0]), end = __ldg(&A.cell_start[k1 + 1]);
        my_cand += end - beg;
        // kSparseU candidates per step: their record loads are issued
        // together (the loop is latency bound, one chain per thread)
        for (uint32_t i0 = beg; i0 < end; i0 += kSparseU) {
          float4 ra[kSparseU], rb[kSparseU], rc[kSparseU], rd[kSparseU];
          bool live[kSparseU];
#pragma unroll
          for (int u = 0; u < kSparseU; ++u) {
            live[u] = i0 + u < end;
            ra[u] = live[u] ? __ldg(&A.rec0[i0 + u]) : make_float4(0.f, 0.f, 0.f, 0.f);
          }
#pragma unroll
          for (int u = 0; u < kSparseU; ++u) live[u] = live[u] && test_pair(F, ra[u], A.max_depth);
#pragma unroll
          for (int u = 0; u < kSparseU; ++u)
            if (live[u]) {
              rb[u] = __ldg(&A.rec1[i0 + u]);
              rc[u] = __ldg(&A.rec2[i0 + u]);
              rd[u] = __ldg(&A.rec3[i0 + u]);
            }
#pragma unroll
          for (int u = 0; u < kSparseU; ++u) {
            if (!live[u]) continue;
            int sector;
            double sv[CH], sw[CH], f0, f1, f2;
            if (!pair_tail<CH, HitX>(A, F, Hs, i0 + u, eye, ra[u], rb[u], rc[u], rd[u], sector, sv, sw, f0, f1, f2,
                               my_exact, my_amb))
              continue;
            ++my_acc;
            p0 = da(p0, f0); p1 = da(p1, f1); p2 = da(p2, f2);
            s_cnt[sector * kSparseThreads + t] += 1u;
#pragma unroll
            for (int c = 0; c < CH; ++c) {
              double &x = s_sum[(c * G + sector) * kSparseThreads + t];
              double &y = s_sq[(c * G + sector) * kSparseThreads + t];
              x = da(x, sv[c]);
              y = da(y, sw[c]);
            }
          }
        }
      }
    }
    // option-B row layout [count G | sum C*G | sum_sq C*G | power 3]; the
    // end of iteration runs in k_apply_deltas (thread per hit point)
    double *d = rows + (size_t)h * (size_t)(G + 2 * CG + 3);
    for (int g = 0; g < G; ++g) d[g] = (double)s_cnt[g * kSparseThreads + t];
    for (int k = 0; k < CG; ++k) {
      d[G + k] = s_sum[k * kSparseThreads + t];
      d[G + CG + k] = s_sq[k * kSparseThreads + t];
    }
    d[G + 2 * CG] = p0;
    d[G + 2 * CG + 1] = p1;
    d[G + 2 * CG + 2] = p2;
  }
  unsigned long long c4[4] = {my_acc, my_cand, my_exact, my_amb};
#pragma unroll
  for (int o = 16; o; o >>= 1)
#pragma unroll
    for (int k = 0; k < 4; ++k) c4[k] += __shfl_xor_sync(~0u, c4[k], o);
  if ((t & 31) == 0)
#pragma unroll
    for (int k = 0; k < 4; ++k) atomicAdd(&A.counters[k], c4[k]);
}

size_t thread_smem_bytes(int G, int C) {
  return sizeof(HitX) * kSparseThreads + (size_t)kSparseThreads * (16 * (size_t)G * C + 4 * (size_t)G);
}

template <int GMAX, int CH, int U>
static cudaError_t launch_sparse_u(cudaStream_t s, const GatherArgs &A, const uint32_t *order, double *rows,
                                   int sms) {
  const int G = A.na * A.ns;
  const size_t smem = thread_smem_bytes(G, CH);
  cudaError_t e = cudaFuncSetAttribute(k_gather_sparse<GMAX, CH, U>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_gather_sparse<GMAX, CH, U>, kSparseThreads, smem);
  if (e != cudaSuccess) return e;
  unsigned blocks = (unsigned)sms * (unsigned)(per_sm > 0 ? per_sm : 1) * 8u;
  const unsigned need = (A.H + kSparseThreads - 1) / kSparseThreads;
  if (blocks > need) blocks = need;
  if (blocks == 0) blocks = 1;
  k_gather_sparse<GMAX, CH, U><<<blocks, kSparseThreads, smem, s>>>(A, order, rows);
  note_launches(1);
  return cudaGetLastError();
}

template <int GMAX, int CH>
static cudaError_t launch_sparse_one(cudaStream_t s, const GatherArgs &A, const uint32_t *order, double *rows,
                                     int sms) {
  return A.vcm ? launch_sparse_u<GMAX, CH, 1>(s, A, order, rows, sms)
               : launch_sparse_u<GMAX, CH, 4>(s, A, order, rows, sms);
}

// ---------------------------------------------------------------- 3D gather
// Dense 3D frames (the C5 clusters: ~100 candidates per hit point): a warp
// owns one hit point at a time (visited in cell order, so consecutive warps
// share cells in L1/L2).  k_prep_3d first stages every hit point's state
// thread-parallel (make_hit, the fp32 predicate constants, the VCM+ eye
// terms); the warp then computes its runs lane-parallel -- the (x, y)
// columns of its fine box (S = 2 fine cells where the dense table fits, else
// reference cells), clipped to the 27-neighbourhood and to the ball's chord
// (gather_dev.cuh) -- and walks the concatenated runs one candidate per lane,
// reading the sorted records straight from L2 (coalesced within a run) in
// three stages: ball + depth + disk on rec0 (test_pair), the normal guard on
// rec1 (certain rejections only), then the full banded decision and value
// (pair_tail, exact fp64 path inside).  Accepted values go to the lane's
// shared-memory slot [(c * G + sector)][lane] {sum, sum_sq} (a spare row for
// the others), counts in 4-bit fields; the slots are reduced in a fixed order
// into the hit point's option-B row (k_apply_deltas pools it and runs the end
// of iteration).
struct alignas(16) Hot3 {
  EyeVcm eye;
  HitF F;
  uint32_t h, nruns;  // runs3[q][0 .. nruns): sorted-record [begin, begin + len)
};
constexpr int kG3MaxRuns = 32;
#ifndef FPPM_G3_BATCH
#define FPPM_G3_BATCH 2  // 1: 56 / 46 / 41 ms on C5 iterations 1..3, 4: 53 / 40 / 33, 2: 47 / 37 / 32 (8 CTAs per SM)
#endif
#ifndef FPPM_G3_MINB
#define FPPM_G3_MINB 10  // CTAs per SM the register cap aims at (5: 96 registers, 8: 64, 10: 48, 12: 40 and slower)
#endif
constexpr int kG3Batch = FPPM_G3_BATCH;  // consecutive hit points per claim
static __device__ __forceinline__ void prefetch_l1(const void *p) {
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}

__global__ void __launch_bounds__(128) k_prep_3d(const GatherArgs A, const uint32_t *__restrict__ order,
                                               Hot3 *__restrict__ hot, HitX *__restrict__ hits,
                                               uint2 *__restrict__ runs) {
  const GridHeader g = *A.grid;
  for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < A.H; q += gridDim.x * blockDim.x) {
    const uint32_t h = order ? order[q] : q;
    Hit H;
    make_hit(A, h, H);
    HitX X;  // the fp64 subset the exact path and the pair values read
    X.cx = H.cx; X.cy = H.cy; X.cz = H.cz; X.nx = H.nx; X.ny = H.ny; X.nz = H.nz;
    X.u = H.u; X.v = H.v; X.r = H.r; X.r2 = H.r2; X.K0 = H.K0; X.K1 = H.K1; X.K2 = H.K2;
    hits[q] = X;
    Hot3 o;
    o.F = hitf(H, A.na, A.ns);
    o.h = h;
    o.eye = EyeVcm{0.0, 0.0, 0.0, 0.0};
    if (A.vcm) {  // bsdf.cpp:42-51 continuation, eye MIS partials
      const double3 wo = A.wo[h], al = A.alb[h];
      o.eye.cos_o = edot(wo.x, wo.y, wo.z, H.nx, H.ny, H.nz);
      const double m1 = al.y < al.z ? al.z : al.y;
      const double amax = al.x < m1 ? m1 : al.x;
      o.eye.cont = amax < 1.0 ? amax : 1.0;
      const double2 em = A.eye_mis[h];
      o.eye.d_vcm = em.x;
      o.eye.d_vm = em.y;
    }
    // the box's (x, y) columns clipped to the chord, non-empty ones only
    uint32_t nr = 0;
    FBox b = {0, -1, 0, -1, 0, -1};
    const bool gathered = A.gathered == nullptr || A.gathered[h] != 0;
    if (gathered && fine_box(g, H.cx, H.cy, H.cz, H.r, b)) {
      const int n = run_count(g, b);
      const double cm = fmax(fabs(H.cx), fmax(fabs(H.cy), fabs(H.cz)));
      const double m = da(da(H.r, dm(H.r, 1e-9)), dm(cm, 4e-16));
      uint2 *dst = runs + (size_t)q * kG3MaxRuns;
      // blocks of 12 columns: keys first, then all their table loads in
      // flight together, then the compaction (the loads are the latency)
      constexpr int kB = 12;
      for (int j0 = 0; j0 < n; j0 += kB) {
        unsigned long long ka[kB], kb[kB];
        bool ok[kB];
#pragma unroll
        for (int u = 0; u < kB; ++u) {
          ok[u] = j0 + u < n && run_keys_clipped(g, b, j0 + u, H.cx, H.cy, H.cz, m, ka[u], kb[u]);
          if (!ok[u]) ka[u] = kb[u] = 0;
        }
        uint32_t rb[kB], re[kB];
#pragma unroll
        for (int u = 0; u < kB; ++u) {
          rb[u] = ok[u] ? __ldg(&A.cell_start[ka[u]]) : 0u;
          re[u] = ok[u] ? __ldg(&A.cell_start[kb[u] + 1]) : 0u;
        }
        // at most 23 columns of a radius-2-fine-cell disk intersect it (S = 2;
        // 9 at S = 1), so the 32 slots always suffice
#pragma unroll
        for (int u = 0; u < kB; ++u)
          if (re[u] > rb[u] && nr < (uint32_t)kG3MaxRuns) dst[nr++] = make_uint2(rb[u], re[u] - rb[u]);
      }
    }
    o.nruns = nr;
    hot[q] = o;
  }
}

// slot columns padded to a power of two (compile-time reduction shape)
template <int GMAX, int CH>
struct G3Lay {
  static constexpr int NC = GMAX * CH;
  static constexpr int NCP = NC <= 8 ? 8 : NC <= 16 ? 16 : NC <= 32 ? 32 : NC <= 64 ? 64 : 128;
  static constexpr int W = NCP <= 32 ? 4 : NCP <= 64 ? 2 : 1;  // warps per CTA (shared memory)
  static constexpr int NW = (GMAX + 7) / 8;                      // 4-bit count words
  static constexpr size_t kSmem = (size_t)W * (NCP + 1) * 32 * 16;
  // the kernel is latency bound (ncu: 58 % long-scoreboard stalls at 20 warps
  // per SM): the register cap follows the CTAs per SM shared memory allows
  static constexpr int kBySmem = (int)((size_t)220 * 1024 / kSmem);
  static constexpr int kMinBlocks = kBySmem < FPPM_G3_MINB ? (kBySmem < 1 ? 1 : kBySmem) : FPPM_G3_MINB;
};

// 4-bit counts (sector 8w + k at bits 4k of nib[w]) spilled every 15 steps
// into 16-bit fields: q[w][k & 3] holds sector 8w + k in half k >> 2
template <int NW>
static __device__ __forceinline__ void g3_spill(uint32_t (&nib)[NW], uint32_t (&q)[NW][4]) {
#pragma unroll
  for (int w = 0; w < NW; ++w) {
#pragma unroll
    for (int k = 0; k < 4; ++k) q[w][k] += (nib[w] >> (4 * k)) & 0x000F000Fu;
    nib[w] = 0u;
  }
}

template <int GMAX, int CH>
__global__ void __launch_bounds__(G3Lay<GMAX, CH>::W * 32, G3Lay<GMAX, CH>::kMinBlocks)
    k_gather_3d(const GatherArgs A, const Hot3 *__restrict__ hot, const HitX *__restrict__ hits,
                const uint2 *__restrict__ runs, double *__restrict__ rows) {
  using L = G3Lay<GMAX, CH>;
  constexpr int NW = L::NW, NCP = L::NCP;
  extern __shared__ __align__(16) unsigned char s_raw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int G = A.na * A.ns, CG = G * CH;
  double *slot_base = reinterpret_cast<double *>(s_raw) + (size_t)warp * (NCP + 1) * 64;
  for (int i = lane; i < (NCP + 1) * 64; i += 32) slot_base[i] = 0.0;
  const uint32_t slots = smem_u32(slot_base);
  const uint32_t slot_lane = slots + (uint32_t)lane * 16u;
  uint32_t my_cand = 0, my_exact = 0, my_amb = 0, my_acc = 0;
  // a warp claims kG3Batch consecutive hit points (neighbours in cell order:
  // they share their cells' records in L1) and prefetches the next one's
  // state into L1 while it walks the current one
  for (uint32_t q = 0, q_end = 0;; ++q) {
    if (q == q_end) {
      if (lane == 0) q = atomicAdd(A.work, (uint32_t)kG3Batch);
      q = __shfl_sync(kFull, q, 0);
      if (q >= A.H) break;
      q_end = min(q + (uint32_t)kG3Batch, A.H);
    }
    if (q + 1 < q_end) {
      const char *nh = reinterpret_cast<const char *>(hot + q + 1);
      const char *nx = reinterpret_cast<const char *>(hits + q + 1);
      const char *nr = reinterpret_cast<const char *>(runs + (size_t)(q + 1) * kG3MaxRuns);
      if (lane * 128u < sizeof(Hot3) + 127u) prefetch_l1(nh + lane * 128u);
      else if (lane >= 8 && (lane - 8) * 128u < sizeof(HitX) + 127u) prefetch_l1(nx + (lane - 8) * 128u);
      else if (lane >= 16 && lane < 18) prefetch_l1(nr + (lane - 16) * 128u);
    }
    const Hot3 &Hq = hot[q];
    const HitX &Hs = hits[q];  // fp64 state: exact path and pair values
    const HitF F = Hq.F;
    const EyeVcm eye = Hq.eye;
    const uint32_t h = Hq.h;
    const uint32_t nruns = Hq.nruns;
    uint32_t rs = 0, rl = 0;  // lane j = run j (k_prep_3d)
    if ((uint32_t)lane < nruns) {
      const uint2 R = runs[(size_t)q * kG3MaxRuns + lane];
      rs = R.x;
      rl = R.y;
    }
    uint32_t incl = rl;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl += y;
    }
    const uint32_t off = rs - (incl - rl);  // sorted index - virtual index within run `lane`
    const uint32_t total = __shfl_sync(kFull, incl, 31);
    if (lane == 0) my_cand += total;
    uint32_t nib[NW], cq[NW][4];
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      nib[w] = 0u;
#pragma unroll
      for (int k = 0; k < 4; ++k) cq[w][k] = 0u;
    }
    double p0 = 0.0, p1 = 0.0, p2 = 0.0;
    uint32_t spill = 15;
    for (uint32_t base = 0; base < total; base += 32) {
      const uint32_t v = base + lane;
      // run of v: binary search over the lanes' inclusive ends
      int j = 0;
#pragma unroll
      for (int st = 16; st > 0; st >>= 1)
        if (__shfl_sync(kFull, incl, j + st - 1) <= v) j += st;
      if (__shfl_sync(kFull, incl, j & 31) <= v) ++j;
      const uint32_t i = v + __shfl_sync(kFull, off, j & 31);
      bool live = v < total;
      float4 a = make_float4(0.f, 0.f, 0.f, 0.f), bb = a, c2 = a, c3 = a;
      if (live) {
        a = __ldg(&A.rec0[i]);
        bb = __ldg(&A.rec1[i]);  // rec0 and rec1 in flight together (one latency, not two)
        live = test_pair(F, a, A.max_depth);  // ball (photon_map.cpp:76), depth (:396), disk (:399)
      }
      if (live) {
        // normal guard (integrator.cpp:397): certain rejections only
        const float gd = fmaf(bb.x, F.nfx, fmaf(bb.y, F.nfy, bb.z * F.nfz));
        const float gb = 2e-6f * (fabsf(bb.x * F.nfx) + fabsf(bb.y * F.nfy) + fabsf(bb.z * F.nfz)) + 1e-30f;
        live = !(F.fast && gd < F.guard_f - gb);
      }
      int sector = 0;
      double sv[CH], sw[CH], f0 = 0.0, f1 = 0.0, f2 = 0.0;
#pragma unroll
      for (int c = 0; c < CH; ++c) sv[c] = sw[c] = 0.0;
      if (live) {
        c2 = __ldg(&A.rec2[i]);
        c3 = __ldg(&A.rec3[i]);
        live = pair_tail<CH, HitX>(A, F, Hs, i, eye, a, bb, c2, c3, sector, sv, sw, f0, f1, f2, my_exact, my_amb);
      }
      if (!live) {
#pragma unroll
        for (int c = 0; c < CH; ++c) sv[c] = sw[c] = 0.0;
        f0 = f1 = f2 = 0.0;
      }
      if (--spill == 0) {
        g3_spill<NW>(nib, cq);
        spill = 15;
      }
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        const uint32_t row = live ? (uint32_t)(c * G + sector) : (uint32_t)NCP;  // spare row
        const uint32_t ad = slot_lane + row * 512u;
        double2 o;
        asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(o.x), "=d"(o.y) : "r"(ad) : "memory");
        o.x = da(o.x, sv[c]);
        o.y = da(o.y, sw[c]);
        asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(ad), "d"(o.x), "d"(o.y) : "memory");
      }
      if (live) {
        ++my_acc;
#pragma unroll
        for (int w = 0; w < NW; ++w)
          if ((sector >> 3) == w) nib[w] += 1u << ((sector & 7) * 4);
      }
      p0 = da(p0, f0);
      p1 = da(p1, f1);
      p2 = da(p2, f2);
    }
    g3_spill<NW>(nib, cq);
    // ---- the hit point's option-B row [count G | sum CG | sum_sq CG | power 3]
    double *d = rows + (size_t)h * (size_t)(G + 2 * CG + 3);
    // slots: lane (col, grp) sums R rows of column col in a fixed, rotated order
#pragma unroll
    for (int c0 = 0; c0 < NCP; c0 += 32) {
      constexpr int ncol = NCP < 32 ? NCP : 32;
      constexpr int nq = 32 / ncol, R = 32 / nq;
      const int col = lane % ncol, grp = lane / ncol;
      double sm = 0.0, sq = 0.0;
      const uint32_t bse = slots + (uint32_t)((c0 + col) * 32 + grp * R) * 16u;
#pragma unroll 4
      for (int k = 0; k < R; ++k) {
        const uint32_t ad = bse + (uint32_t)((k + col) % R) * 16u;
        double2 o;
        asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(o.x), "=d"(o.y) : "r"(ad) : "memory");
        sm += o.x;
        sq += o.y;
        asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(ad), "d"(0.0), "d"(0.0) : "memory");
      }
#pragma unroll
      for (int o = (nq / 2) * ncol; o >= ncol && o > 0; o >>= 1) {
        sm += __shfl_down_sync(kFull, sm, o);
        sq += __shfl_down_sync(kFull, sq, o);
      }
      if (lane < ncol && c0 + lane < CG) {
        d[G + c0 + lane] = sm;
        d[G + CG + c0 + lane] = sq;
      }
    }
    // counts: 16-bit fields -> warp sums (halves reduced separately)
#pragma unroll
    for (int w = 0; w < NW; ++w)
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t c_lo = __reduce_add_sync(kFull, cq[w][k] & 0xffffu);  // sector 8w + k
        const uint32_t c_hi = __reduce_add_sync(kFull, cq[w][k] >> 16);      // sector 8w + k + 4
        if (lane == 0) {
          if (8 * w + k < G) d[8 * w + k] = (double)c_lo;
          if (8 * w + k + 4 < G) d[8 * w + k + 4] = (double)c_hi;
        }
      }
    // flux: transposed butterfly; lane 0 / 8 / 16 end with p0 / p1 / p2
    {
      const bool hi16 = (lane & 16) != 0, hi8 = (lane & 8) != 0;
      const double s0 = hi16 ? p0 : p2, k0 = hi16 ? p2 : p0;
      const double s1 = hi16 ? p1 : 0.0, k1 = hi16 ? 0.0 : p1;
      const double x = k0 + __shfl_xor_sync(kFull, s0, 16);
      const double y = k1 + __shfl_xor_sync(kFull, s1, 16);
      double c = (hi8 ? y : x) + __shfl_xor_sync(kFull, hi8 ? x : y, 8);
      c += __shfl_xor_sync(kFull, c, 4);
      c += __shfl_xor_sync(kFull, c, 2);
      c += __shfl_xor_sync(kFull, c, 1);
      if (lane == 0) d[G + 2 * CG] = c;
      if (lane == 8) d[G + 2 * CG + 1] = c;
      if (lane == 16) d[G + 2 * CG + 2] = c;
    }
    __syncwarp();
  }
  unsigned long long c4[4] = {my_acc, my_cand, my_exact, my_amb};
#pragma unroll
  for (int o = 16; o; o >>= 1)
#pragma unroll
    for (int k = 0; k < 4; ++k) c4[k] += __shfl_xor_sync(~0u, c4[k], o);
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < 4; ++k) atomicAdd(&A.counters[k], c4[k]);
}

size_t hot3_bytes() { return sizeof(Hot3) + kG3MaxRuns * sizeof(uint2); }

template <int GMAX, int CH>
static cudaError_t launch_3d_one(cudaStream_t s, const GatherArgs &A, const uint32_t *order, void *hot,
                                 void *hits, double *rows, int sms) {
  using L = G3Lay<GMAX, CH>;
  if (A.H == 0) return cudaSuccess;
  // one buffer: Hot3[H] then the runs [H][kG3MaxRuns]
  Hot3 *h3 = static_cast<Hot3 *>(hot);
  uint2 *runs = reinterpret_cast<uint2 *>(h3 + A.H);
  k_prep_3d<<<(unsigned)std::min<unsigned long long>((A.H + 127) / 128, (unsigned long long)sms * 16), 128, 0, s>>>(
      A, order, h3, static_cast<HitX *>(hits), runs);
  note_launches(1);
  const size_t smem = L::kSmem;
  cudaError_t e = cudaFuncSetAttribute(k_gather_3d<GMAX, CH>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_gather_3d<GMAX, CH>, L::W * 32, smem);
  if (e != cudaSuccess) return e;
  unsigned blocks = (unsigned)sms * (unsigned)(per_sm > 0 ? per_sm : 1);
  const unsigned need = (A.H + L::W - 1) / L::W;
  if (blocks > need) blocks = need;
  if (blocks == 0) blocks = 1;
  k_gather_3d<GMAX, CH><<<blocks, L::W * 32, smem, s>>>(A, h3, static_cast<const HitX *>(hits), runs, rows);
  note_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_gather_sparse(cudaStream_t s, const GatherArgs &A, int C, const uint32_t *order,
                                 double *rows, int sms, void *hot3, void *hits) {
  const int G = A.na * A.ns;
  if (hot3 == nullptr)  // few candidates per hit point: one thread each
    return C == 1 ? launch_sparse_one<32, 1>(s, A, order, rows, sms) : launch_sparse_one<32, 3>(s, A, order, rows, sms);
  if (C == 1) {
    if (G <= 8) return launch_3d_one<8, 1>(s, A, order, hot3, hits, rows, sms);
    if (G <= 16) return launch_3d_one<16, 1>(s, A, order, hot3, hits, rows, sms);
    return launch_3d_one<32, 1>(s, A, order, hot3, hits, rows, sms);
  }
  if (G <= 8) return launch_3d_one<8, 3>(s, A, order, hot3, hits, rows, sms);
  if (G <= 16) return launch_3d_one<16, 3>(s, A, order, hot3, hits, rows, sms);
  return launch_3d_one<32, 3>(s, A, order, hot3, hits, rows, sms);
}

// ---------------------------------------------------------------- explicit samples
// GatherRegion::accumulate on caller-supplied (region, y, value) samples.
__global__ void k_sample_sectors(const uint32_t *__restrict__ region, const double2 *__restrict__ y,
                                 uint32_t n, const double *__restrict__ radius, uint32_t H, int na,
                                 int ns, int *__restrict__ sectors, int *__restrict__ err) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint32_t h = region[i];
    if (h >= H) { atomicExch(err, FPPM_ERR_INVALID_ARGUMENT); sectors[i] = -1; continue; }
    const double r = radius[h];
    const double r2 = dm(r, r);
    const double d2 = da(dm(y[i].x, y[i].x), dm(y[i].y, y[i].y));
    if (d2 > dm(r2, 1.0 + 1e-9)) {  // gather.cpp:20-21
      atomicExch(err, FPPM_ERR_DOMAIN);
      sectors[i] = -1;
      continue;
    }
    bool amb = false;
    sectors[i] = exact_sector(y[i].x, y[i].y, r2, na, ns, amb);
  }
}

__global__ void k_sample_accumulate(const uint32_t *__restrict__ region,
                                    const double *__restrict__ value, const int *__restrict__ sectors,
                                    uint32_t n, int G, int C, unsigned long long *__restrict__ st_cnt,
                                    double *__restrict__ st_sum, double *__restrict__ st_sq) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int s = sectors[i];
    const size_t base = (size_t)region[i] * G * C;
    const double r = value[3 * (size_t)i], g = value[3 * (size_t)i + 1], b = value[3 * (size_t)i + 2];
    if (C == 1) {
      const double v = elum(r, g, b);
      atomicAdd(&st_cnt[base + s], 1ull);
      atomicAdd(&st_sum[base + s], v);
      atomicAdd(&st_sq[base + s], v * v);
    } else {
      const double vals[3] = {r, g, b};
      for (int c = 0; c < 3; ++c) {
        atomicAdd(&st_cnt[base + c * G + s], 1ull);
        atomicAdd(&st_sum[base + c * G + s], vals[c]);
        atomicAdd(&st_sq[base + c * G + s], vals[c] * vals[c]);
      }
    }
  }
}

// end_iteration over every region without a gather (gather.cpp:90-144).
__global__ void k_end_iteration(EndArgs A) {
  const int G = A.G, C = A.C, CG = G * C;
  for (uint32_t h = blockIdx.x * blockDim.x + threadIdx.x; h < A.H; h += gridDim.x * blockDim.x) {
    unsigned long long pc[kMaxCG];
    double ps[kMaxCG], pq[kMaxCG];
    const size_t base = (size_t)h * CG;
    for (int i = 0; i < CG; ++i) {
      pc[i] = A.st_cnt[base + i];
      ps[i] = A.st_sum[base + i];
      pq[i] = A.st_sq[base + i];
    }
    if (A.snap_cnt)
      for (int i = 0; i < CG; ++i) {
        A.snap_cnt[base + i] = pc[i];
        A.snap_sum[base + i] = ps[i];
        A.snap_sq[base + i] = pq[i];
      }
    double r = A.radius[h];
    uint32_t t = A.t[h];
    double stat, critical;
    const double r_old = r;
    const uint8_t flags = end_of_iteration(A.end, G, C, r, t, pc, ps, pq, stat, critical);
    for (int i = 0; i < CG; ++i) {
      A.st_cnt[base + i] = pc[i];
      A.st_sum[base + i] = ps[i];
      A.st_sq[base + i] = pq[i];
    }
    A.radius[h] = r;
    A.t[h] = t;
    if (A.o_gather_r) A.o_gather_r[h] = r_old;
    if (A.o_flags) A.o_flags[h] = flags;
    if (A.o_stat) A.o_stat[h] = stat;
    if (A.o_crit) A.o_crit[h] = critical;
  }
}

__global__ void k_hit_weights(const double3 *__restrict__ nrm, const double3 *__restrict__ wo,
                              const double3 *__restrict__ thr, const double3 *__restrict__ alb,
                              uint32_t H, double3 *__restrict__ K) {
  for (uint32_t h = blockIdx.x * blockDim.x + threadIdx.x; h < H; h += gridDim.x * blockDim.x) {
    const double3 n = nrm[h], w = wo[h], T = thr[h], a = alb[h];
    const double cos_o = edot(w.x, w.y, w.z, n.x, n.y, n.z);  // bsdf.cpp:34
    const bool off = cos_o <= 0.0;                             // bsdf.cpp:58
    K[h] = make_double3(dm(T.x, off ? 0.0 : dm(a.x, kInvPi)), dm(T.y, off ? 0.0 : dm(a.y, kInvPi)),
                        dm(T.z, off ? 0.0 : dm(a.z, kInvPi)));
  }
}

// ---------------------------------------------------------------- launchers
template <int GMAX, int CH>
static cudaError_t launch_one(cudaStream_t s, const GatherArgs &A, int sms) {
  int per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_gather_test<GMAX, CH>,
                                                                kGatherThreads, 0);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  unsigned blocks = (unsigned)(sms * per_sm);
  const unsigned need = (A.H + kGatherThreads / 32 - 1) / (kGatherThreads / 32);
  if (blocks > need) blocks = need ? need : 1;
  k_gather_test<GMAX, CH><<<blocks, kGatherThreads, 0, s>>>(A);
  note_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_gather_test(cudaStream_t s, const GatherArgs &A, int C, int sms) {
  const int G = A.na * A.ns;
  if (C == 1) {
    if (G <= 4) return launch_one<4, 1>(s, A, sms);
    if (G <= 8) return launch_one<8, 1>(s, A, sms);
    if (G <= 12) return launch_one<12, 1>(s, A, sms);
    if (G <= 16) return launch_one<16, 1>(s, A, sms);
    return launch_one<32, 1>(s, A, sms);
  }
  if (G <= 4) return launch_one<4, 3>(s, A, sms);
  if (G <= 8) return launch_one<8, 3>(s, A, sms);
  if (G <= 12) return launch_one<12, 3>(s, A, sms);
  return launch_one<32, 3>(s, A, sms);
}

// Owner side of option B: rows summed over all ranks' photon shares are
// pooled exactly like a local gather's sums (finalize_hit).
template <int GMAX, int CH>
__global__ void __launch_bounds__(128) k_apply_deltas(const GatherArgs A, uint32_t h0, uint32_t n,
                                                      const double *__restrict__ delta) {
  const int G = A.na * A.ns, CG = G * CH;
  unsigned int my_tested = 0, my_rejected = 0;
  double my_rmax = 0.0;
  unsigned long long my_acc = 0;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const double *d = delta + (size_t)i * (size_t)(G + 2 * CG + 3);
    uint32_t cnt[GMAX];
    double sm[CH][GMAX], sq[CH][GMAX];
#pragma unroll
    for (int g = 0; g < GMAX; ++g) {
      cnt[g] = g < G ? (uint32_t)d[g] : 0u;
      my_acc += cnt[g];
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        sm[c][g] = g < G ? d[G + c * G + g] : 0.0;
        sq[c][g] = g < G ? d[G + CG + c * G + g] : 0.0;
      }
    }
    finalize_hit<GMAX, CH>(A, h0 + i, cnt, sm, sq, d[G + 2 * CG], d[G + 2 * CG + 1], d[G + 2 * CG + 2],
                           my_tested, my_rejected, my_rmax);
  }
  for (int o = 16; o; o >>= 1) {
    my_tested += __shfl_xor_sync(~0u, my_tested, o);
    my_rejected += __shfl_xor_sync(~0u, my_rejected, o);
    my_rmax = fmax(my_rmax, __shfl_xor_sync(~0u, my_rmax, o));
    my_acc += __shfl_xor_sync(~0u, my_acc, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(A.iter_tr, my_tested);
    atomicAdd(A.iter_tr + 1, my_rejected);
    atomicMax(A.rmax_bits, (unsigned long long)__double_as_longlong(my_rmax));
  }
}

template <int GMAX, int CH>
static cudaError_t launch_apply(cudaStream_t s, const GatherArgs &A, uint32_t h0, uint32_t n,
                                const double *delta) {
  const unsigned blocks = (unsigned)std::min<uint32_t>((n + 127) / 128, 4096u);
  k_apply_deltas<GMAX, CH><<<blocks, 128, 0, s>>>(A, h0, n, delta);
  note_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_apply_deltas(cudaStream_t s, const GatherArgs &A, int C, uint32_t h0, uint32_t n,
                                const double *delta) {
  if (n == 0) return cudaSuccess;
  const int G = A.na * A.ns;
  if (C == 1) {
    if (G <= 4) return launch_apply<4, 1>(s, A, h0, n, delta);
    if (G <= 8) return launch_apply<8, 1>(s, A, h0, n, delta);
    if (G <= 16) return launch_apply<16, 1>(s, A, h0, n, delta);
    return launch_apply<32, 1>(s, A, h0, n, delta);
  }
  if (G <= 4) return launch_apply<4, 3>(s, A, h0, n, delta);
  if (G <= 8) return launch_apply<8, 3>(s, A, h0, n, delta);
  return launch_apply<32, 3>(s, A, h0, n, delta);
}

cudaError_t launch_samples(cudaStream_t s, const uint32_t *region, const double2 *y,
                           const double *value, uint32_t n, const double *radius, uint32_t H, int na,
                           int ns, int C, int *sectors, int *err, unsigned long long *st_cnt,
                           double *st_sum, double *st_sq, int phase) {
  if (n == 0) return cudaSuccess;
  const int blocks = (int)((n + 255) / 256);
  if (phase == 0)
    k_sample_sectors<<<blocks, 256, 0, s>>>(region, y, n, radius, H, na, ns, sectors, err);
  else
    k_sample_accumulate<<<blocks, 256, 0, s>>>(region, value, sectors, n, na * ns, C, st_cnt,
                                               st_sum, st_sq);
  note_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_end_iteration(cudaStream_t s, const EndArgs &A) {
  if (A.H == 0) return cudaSuccess;
  const int blocks = (int)((A.H + 127) / 128);
  k_end_iteration<<<blocks, 128, 0, s>>>(A);
  note_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_hit_weights(cudaStream_t s, const double3 *nrm, const double3 *wo,
                               const double3 *thr, const double3 *alb, uint32_t H, double3 *K) {
  if (H == 0) return cudaSuccess;
  const int blocks = (int)((H + 255) / 256);
  k_hit_weights<<<blocks, 256, 0, s>>>(nrm, wo, thr, alb, H, K);
  note_launches(1);
  return cudaGetLastError();
}

__global__ void k_lean_check(const double3 *__restrict__ pos, const double3 *__restrict__ nrm,
                             const double3 *__restrict__ K, const uint8_t *__restrict__ gathered, uint32_t H,
                             uint32_t *__restrict__ flag) {
  bool ok = true;
  for (uint32_t h = blockIdx.x * blockDim.x + threadIdx.x; h < H; h += gridDim.x * blockDim.x) {
    if (gathered != nullptr && gathered[h] == 0) continue;
    const double3 c = pos[h], n = nrm[h], k = K[h];
    ok = ok && n.x == 0.0 && n.y == 0.0 && n.z == 1.0 && (double)(float)c.x == c.x &&
         (double)(float)c.y == c.y && (double)(float)c.z == c.z && k.x == k.y && k.y == k.z && isfinite(k.x);
  }
  if (!__all_sync(0xffffffffu, ok) && (threadIdx.x & 31) == 0) atomicAnd(flag, 0u);
}

cudaError_t launch_lean_check(cudaStream_t s, const double3 *pos, const double3 *nrm, const double3 *K,
                              const uint8_t *gathered, uint32_t H, uint32_t *flag) {
  cudaError_t e = cudaMemsetAsync(flag, 0xff, sizeof(uint32_t), s);  // nonzero: lean until a lane objects
  if (e != cudaSuccess || H == 0) return e;
  k_lean_check<<<(int)std::min<uint32_t>((H + 255) / 256, 1184u), 256, 0, s>>>(pos, nrm, K, gathered, H, flag);
  note_launches(1);
  return cudaGetLastError();
}

}  // namespace fppm_b200
