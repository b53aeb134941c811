// context.cu -- the C ABI (include/fppm_gpu.h): device buffers, the per-iteration
// orchestration and host<->device plumbing around the kernels in grid.cu,
// gather.cu and generate.cu.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "common.cuh"
#include "gather.cuh"

struct fppm_gpu_ctx {
  fppm_gpu_config cfg{};
  int sms = 148;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  // grid records: the fine layout's pack + permute run on gstream, forked
  // after the grid header / the sort and joined before the next consumer, so
  // they overlap the sort and the gather's scheduling kernels
  cudaStream_t gstream = nullptr;
  cudaEvent_t ev_g_hdr = nullptr, ev_g_sorted = nullptr, ev_g_recs = nullptr;
  cudaEvent_t ev_hdr = nullptr;  // the grid header's copy to the host
  cudaEvent_t ev_sched = nullptr;  // the fine schedule's totals copied to the host
  bool last_fork = false;        // the last build packed records on gstream (speculated for the next)
  bool recs_pending = false;
  unsigned long long hp_version = 0;  // bumped whenever hit points change
  std::string err;
  int G = 0, C = 1;

  // regions
  uint32_t H = 0;
  double3 *d_pos = nullptr, *d_nrm = nullptr, *d_wo = nullptr, *d_thr = nullptr,
          *d_alb = nullptr, *d_K = nullptr;
  uint32_t *d_eye = nullptr;
  uint8_t *d_gathered = nullptr;
  double *d_radius = nullptr;
  uint32_t *d_t = nullptr;
  unsigned long long *d_st_cnt = nullptr;
  double *d_st_sum = nullptr, *d_st_sq = nullptr;

  // photon staging (canonical [n][3] fp32)
  uint32_t N = 0;
  float *d_ppos = nullptr, *d_pnrm = nullptr, *d_pwi = nullptr, *d_ppow = nullptr;
  uint32_t *d_pdepth = nullptr;
  // second staging set: host uploads alternate between the two sets on a copy
  // stream, so the upload of the next batch overlaps the current iteration
  float *d_ppos2 = nullptr, *d_pnrm2 = nullptr, *d_pwi2 = nullptr, *d_ppow2 = nullptr;
  uint32_t *d_pdepth2 = nullptr;
  cudaStream_t cstream = nullptr;
  cudaEvent_t ev_copied[2] = {}, ev_free[2] = {};
  int stage_cur = 0;       // staging set the current photons live in
  int stage_pending = -1;  // set whose upload the next grid build must wait for
  // fppm_gpu_prefetch_photons: an upload of the NEXT batch into the free set,
  // made current without a copy by fppm_gpu_adopt_photons(token)
  int pf_set = -1;
  fppm_photons pf_src{};
  uint32_t pf_n = 0;
  uint64_t pf_digest = 0, pf_token = 0, pf_counter = 0;
  bool free_recorded[2] = {false, false};
  // photons the next grid build reads: the staging buffers, or caller-owned
  // device buffers registered by fppm_gpu_set_photons_device (zero copy)
  const float *in_pos = nullptr, *in_nrm = nullptr, *in_wi = nullptr, *in_pow = nullptr;
  const uint32_t *in_depth = nullptr;

  // light phase: scene on the device + per-path deposit slots
  // C5 workload: all hit points, their NN grid and the cluster table
  fppm_b200::C5Args c5{};
  void *c5_mem[8] = {};
  fppm_b200::CamD cam{};
  bool has_camera = false;
  double3 *d_emit = nullptr, *d_film = nullptr;  // per pixel: emitted radiance, film sum
  double2 *d_vcvm = nullptr;  // per pixel cumulative {vc, vm} luminance (Film::add_split)
  uint64_t film_iters = 0;
  fppm_b200::TraceScene scene{};
  void *scene_mem[9] = {};  // [8]: per-primitive constants (k_scene_prep)
  uint32_t *t_ctr = nullptr;
  double *d_rows = nullptr;  // sparse gather: per-hit-point sums before the end of iteration
  size_t rows_cap = 0;
  bool has_scene = false;
  float *t_pos = nullptr, *t_nrm = nullptr, *t_wi = nullptr, *t_pow = nullptr;
  uint32_t *t_depth = nullptr, *t_count = nullptr, *t_base = nullptr, *t_scan = nullptr;
  double *t_mis = nullptr;
  unsigned long long t_slot_cap = 0, t_path_cap = 0;
  // VCM+ bidirectional remainder: fp64 light vertices in the trace slots,
  // splats, secondary merge vertices and their delta rows
  bool bidir_trace = false;
  double last_eta_light = 0.0;
  double *b_pos = nullptr, *b_sn = nullptr, *b_wi = nullptr, *b_thr = nullptr, *b_mis = nullptr;
  int *b_mat = nullptr;
  unsigned long long b_slot_cap = 0;
  double3 *d_splat = nullptr;
  double3 *q_pos = nullptr, *q_nrm = nullptr, *q_wo = nullptr, *q_thr = nullptr, *q_alb = nullptr, *q_K = nullptr;
  uint32_t *q_eye = nullptr;
  uint8_t *q_gathered = nullptr;
  double *q_radius = nullptr, *q_rows = nullptr;
  double2 *q_mis = nullptr;
  unsigned long long q_cap = 0, q_rows_cap = 0;
  fppm_b200::SortScratch q_sort{};  // home-cell order of the merge queries
  // eye sub-paths between the walk and the vertex loop (BidirArgs::vtx_*)
  double *v_d = nullptr;
  int4 *v_i = nullptr;
  // fppm_gpu_set_photons_packed: keep flags, destinations, scan scratch, hit-point box
  uint32_t *d_keep = nullptr, *d_keep_dst = nullptr, *d_keep_scan = nullptr;
  unsigned long long keep_cap = 0;
  double *d_hpbox = nullptr;
  uint32_t *v_n = nullptr;
  unsigned long long *v_rng = nullptr;
  unsigned long long v_cap = 0;

  // VCM+ merge stage inputs
  double2 *d_eye_mis = nullptr;                                   // [H] {d_vcm, d_vm}
  double *d_pmis_in[3] = {nullptr, nullptr, nullptr};             // [N] photon order
  double *d_pmis[3] = {nullptr, nullptr, nullptr};                // [N] sorted order
  bool pmis_set = false;

  // grid
  fppm_b200::PhotonRecs recs{};
  fppm_b200::SortScratch sort{};
  uint32_t *d_skeys = nullptr, *d_order = nullptr;  // alias into sort buffers
  uint32_t *d_cell_start = nullptr;
  unsigned long long cell_cap = 0;
  fppm_b200::GridHeader *d_hdr = nullptr, *h_hdr = nullptr;
  long long *d_bounds = nullptr, *h_bounds_init = nullptr;
  double *d_cell = nullptr, *h_cell = nullptr, *d_cell_chk = nullptr;
  bool grid_valid = false;
  // the reference throws when a query radius exceeds the cell size
  // (photon_map.cpp:57-58); checked before the next gather whenever the cell
  // did not come from the max live radius or radii were raised (set_regions)
  bool grid_explicit = false, rcheck = false;
  // lean record layout: every gathered hit point planar and gray (device
  // flag from k_lean_check), config C = 1, n_a <= 2, n_s = 4, fine kernel
  uint32_t *d_lean_ok = nullptr;
  // 3D kernel staging (k_prep_3d): Hot3 and full Hit per hit point
  void *hot3 = nullptr, *hot3_hits = nullptr;
  uint32_t hot3_cap = 0;
  // staging set the current grid's input photons live in (the lean layout's
  // exact path reads them during the gather: released after it), -1 none
  int grid_set = -1;

  // outputs
  double *o_gather_r = nullptr, *o_stat = nullptr, *o_crit = nullptr, *o_flux = nullptr;
  uint8_t *o_flags = nullptr;
  uint8_t *o_tested = nullptr, *o_rejected = nullptr;  // unpacked flags (async outputs)
  unsigned long long *o_t64 = nullptr;
  float *o_rad = nullptr;
  uint32_t *o_acc = nullptr;
  unsigned long long *snap_cnt = nullptr;
  double *snap_sum = nullptr, *snap_sq = nullptr;

  // counters
  unsigned long long *d_counters = nullptr, *h_counters = nullptr;
  unsigned long long last_counters[4] = {0, 0, 0, 0};
  unsigned int *d_iter_tr = nullptr, *d_work = nullptr;
  unsigned long long *d_rmax_bits = nullptr;

  // critical-value table by t
  std::vector<double> crit;
  double *d_crit = nullptr;
  uint32_t crit_cap = 0;
  uint64_t end_calls = 0;
  double chi2_crit = 0.0;

  // scratch for explicit-sample / query APIs
  void *d_scratch = nullptr;
  size_t scratch_bytes = 0;

  // tiled-gather schedule (home-cell items)
  fppm_b200::TileSched tile{};
  // CUDA events around the dominant gather kernel of recent gathers (ring)
  static constexpr int kEvRing = 64;
  cudaEvent_t ev_k[kEvRing][2] = {};
  uint32_t ev_head = 0, ev_count = 0;
  uint32_t *h_total = nullptr;
};

namespace fppm_b200 {

int cuda_fail(fppm_gpu_ctx *ctx, cudaError_t e, const char *what) {
  if (ctx) {
    ctx->err = std::string("CUDA error ") + cudaGetErrorString(e) + " in " + what;
  }
  return FPPM_ERR_CUDA;
}

static int fail(fppm_gpu_ctx *ctx, int code, const std::string &msg) {
  if (ctx) ctx->err = msg;
  return code;
}

template <typename T>
static cudaError_t dalloc(T **p, size_t count) {
  *p = nullptr;
  if (count == 0) count = 1;
  return cudaMalloc(reinterpret_cast<void **>(p), sizeof(T) * count);
}

// gather kernel variant: 1 warp per hit point over reference cells (the
// reference query order; kept selectable as a cross-check), 4 fine (slab
// grids, the default where G * C <= 24), 5 the 3D warp-per-hit-point kernel
// over fine columns (every other grid and configuration, VCM+ merges)
static int gather_variant(const fppm_gpu_ctx *ctx) {
  if (ctx->cfg.gather_kernel == 1) return 1;
  if (ctx->cfg.vcm_plus) return 5;
  if (ctx->cfg.gather_kernel == 5) return 5;
  return fine_supported(ctx->G, ctx->C) ? 4 : 5;
}

// The kernel that will gather this grid: the fine kernel on slab (planar)
// grids, the 3D kernel on 3D grids (S = 1 or 2).
static int effective_variant(const fppm_gpu_ctx *ctx, uint32_t S) {
  const int v = gather_variant(ctx);
  if (v == 4 && S != kFineS) return 5;  // 3D grid (S = 1 or 2): the warp-per-hit-point 3D kernel
  return v;
}

// 3D frames: a warp per hit point pays off once the 27-cell neighbourhood
// holds tens of photons (C5: ~200); sparser frames (the C3 / C4 camera hit
// points: ~3) take one thread per hit point
static bool dense_3d(const GridHeader &g) {
  if (const char *e = std::getenv("FPPM_3D")) return e[0] == '1';  // measurement knob
  const double ref_cells = (double)g.ncells / ((double)g.S * g.S * g.S);
  return ref_cells > 0.0 && 27.0 * (double)g.n / ref_cells >= 48.0;
}

// per-hit-point staging of the 3D kernel (Hot3 + full Hit for the exact path)
static int ensure_hot3(fppm_gpu_ctx *ctx, uint32_t n) {
  if (n <= ctx->hot3_cap) return FPPM_OK;
  if (ctx->hot3) cudaFree(ctx->hot3);
  if (ctx->hot3_hits) cudaFree(ctx->hot3_hits);
  ctx->hot3 = ctx->hot3_hits = nullptr;
  ctx->hot3_cap = 0;
  FPPM_CUDA_OK(cudaMalloc(&ctx->hot3, hot3_bytes() * std::max<uint32_t>(n, 1)));
  FPPM_CUDA_OK(cudaMalloc(&ctx->hot3_hits, fine_hit_bytes() * std::max<uint32_t>(n, 1)));
  ctx->hot3_cap = n;
  return FPPM_OK;
}

static cudaError_t ensure_scratch(fppm_gpu_ctx *ctx, size_t bytes) {
  if (bytes <= ctx->scratch_bytes) return cudaSuccess;
  if (ctx->d_scratch) cudaFree(ctx->d_scratch);
  ctx->scratch_bytes = 0;
  cudaError_t e = cudaMalloc(&ctx->d_scratch, bytes);
  if (e == cudaSuccess) ctx->scratch_bytes = bytes;
  return e;
}

__global__ void k_max_radius(const double *__restrict__ radius, uint32_t H,
                             double *__restrict__ out, const uint8_t *__restrict__ gathered = nullptr) {
  __shared__ unsigned long long s;
  if (threadIdx.x == 0) s = 0;
  __syncthreads();
  double m = 0.0;
  for (uint32_t h = blockIdx.x * blockDim.x + threadIdx.x; h < H; h += gridDim.x * blockDim.x)
    if (gathered == nullptr || gathered[h]) m = fmax(m, radius[h]);
  atomicMax(&s, (unsigned long long)__double_as_longlong(m));
  __syncthreads();
  if (threadIdx.x == 0) atomicMax(reinterpret_cast<unsigned long long *>(out), s);
}

__global__ void k_fill_regions(double *radius, uint32_t *t, uint32_t H, double r0) {
  for (uint32_t h = blockIdx.x * blockDim.x + threadIdx.x; h < H; h += gridDim.x * blockDim.x) {
    radius[h] = r0;
    t[h] = 1;
  }
}

// grow the F critical table so that every t <= need is covered
// Orders the context stream after the forked record build (see gstream).
static int join_recs(fppm_gpu_ctx *ctx) {
  if (!ctx->recs_pending) return FPPM_OK;
  ctx->recs_pending = false;
  FPPM_CUDA_OK(cudaStreamWaitEvent(ctx->stream, ctx->ev_g_recs, 0));
  return FPPM_OK;
}
#define JOIN_RECS(ctx)                      \
  do {                                      \
    if (int jr_ = join_recs(ctx)) return jr_; \
  } while (0)

static int ensure_crit(fppm_gpu_ctx *ctx, uint64_t need) {
  const fppm_gpu_config &c = ctx->cfg;
  if (c.policy != FPPM_POLICY_FTEST || c.override_decision != FPPM_OVERRIDE_NONE) {
    if (ctx->crit.empty()) ctx->crit.assign(2, 0.0);
  }
  if (ctx->crit.empty()) ctx->crit.push_back(0.0);  // t = 0 unused
  const size_t old = ctx->crit.size();
  if (ctx->crit.size() <= need && c.policy == FPPM_POLICY_FTEST &&
      c.override_decision == FPPM_OVERRIDE_NONE) {
    const long long d1 = (long long)ctx->G - 1;
    while (ctx->crit.size() <= need) {
      const uint64_t t = ctx->crit.size();
      const uint64_t m = t * c.samples_per_iteration;
      double v = 0.0;
      if (m >= 2) {
        const long long d2 = (long long)ctx->G * (long long)(m - 1);
        // chi-squared limit is constant in d2 (special_functions.cpp:157)
        if ((double)d2 > 2e7 && ctx->crit.size() > 1 &&
            (double)((long long)ctx->G * (long long)((t - 1) * c.samples_per_iteration - 1)) > 2e7) {
          v = ctx->crit.back();
        } else {
          int st = 0;
          v = fppm_b200::host_f_quantile(1.0 - c.alpha_f, (double)d1, (double)d2, &st);
        }
      }
      ctx->crit.push_back(v);
    }
  }
  if (ctx->crit.size() > ctx->crit_cap) {
    uint32_t cap = std::max<uint32_t>(64, ctx->crit_cap * 2);
    while (cap < ctx->crit.size()) cap *= 2;
    double *p = nullptr;
    FPPM_CUDA_OK(cudaMalloc(&p, sizeof(double) * cap));
    if (ctx->d_crit) {
      FPPM_CUDA_OK(cudaStreamSynchronize(ctx->stream));
      cudaFree(ctx->d_crit);
    }
    ctx->d_crit = p;
    ctx->crit_cap = cap;
    FPPM_CUDA_OK(cudaMemcpyAsync(p, ctx->crit.data(), sizeof(double) * ctx->crit.size(),
                                 cudaMemcpyHostToDevice, ctx->stream));
    FPPM_CUDA_OK(cudaStreamSynchronize(ctx->stream));
  } else if (ctx->crit.size() > old) {
    FPPM_CUDA_OK(cudaMemcpyAsync(ctx->d_crit + old, ctx->crit.data() + old,
                                 sizeof(double) * (ctx->crit.size() - old),
                                 cudaMemcpyHostToDevice, ctx->stream));
    FPPM_CUDA_OK(cudaStreamSynchronize(ctx->stream));
  }
  return FPPM_OK;
}

static EndParams end_params(fppm_gpu_ctx *ctx, uint64_t iteration) {
  const fppm_gpu_config &c = ctx->cfg;
  EndParams P;
  P.policy = c.policy;
  P.override_decision = c.override_decision;
  P.J = c.samples_per_iteration;
  P.k = c.k;
  P.floor_next = host_schedule_radius(c.r_min_base, c.alpha, iteration + 1);
  P.sched_next = host_schedule_radius(c.initial_radius, c.alpha, iteration + 1);
  P.crit = ctx->d_crit;
  P.crit_len = (uint32_t)ctx->crit.size();
  P.chi2_crit = ctx->chi2_crit;
  return P;
}

static int copy_out(fppm_gpu_ctx *ctx, void *dst, const void *src, size_t bytes) {
  if (!dst || bytes == 0) return FPPM_OK;
  FPPM_CUDA_OK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, ctx->stream));
  return FPPM_OK;
}

// Split the decision flags and widen t on the device, so every output is a
// plain asynchronous copy (the call does not block the host).
__global__ void k_unpack_outputs(const uint8_t *__restrict__ flags, const uint32_t *__restrict__ t,
                                 uint32_t n, uint8_t *__restrict__ tested, uint8_t *__restrict__ rejected,
                                 unsigned long long *__restrict__ t64) {
  for (uint32_t h = blockIdx.x * blockDim.x + threadIdx.x; h < n; h += gridDim.x * blockDim.x) {
    const uint8_t f = flags[h];
    tested[h] = f & 1u;
    rejected[h] = (f >> 1) & 1u;
    t64[h] = t[h];
  }
}

static int copy_iter_out(fppm_gpu_ctx *ctx, fppm_gpu_iter_out *out, bool with_gather, size_t h0 = 0,
                         size_t n = ~size_t(0)) {
  if (!out) return FPPM_OK;
  const size_t H = std::min<size_t>(ctx->H - h0, n), CG = (size_t)ctx->G * ctx->C;
  int rc;
  if (!ctx->o_tested) {
    const size_t Hc = std::max<uint32_t>(ctx->cfg.max_hitpoints, 1);
    FPPM_CUDA_OK(dalloc(&ctx->o_tested, Hc));
    FPPM_CUDA_OK(dalloc(&ctx->o_rejected, Hc));
    FPPM_CUDA_OK(dalloc(&ctx->o_t64, Hc));
  }
  if (H && (out->tested || out->rejected || out->t)) {
    k_unpack_outputs<<<(unsigned)std::min<size_t>((H + 255) / 256, 1024), 256, 0, ctx->stream>>>(
        ctx->o_flags + h0, ctx->d_t + h0, (uint32_t)H, ctx->o_tested + h0, ctx->o_rejected + h0, ctx->o_t64 + h0);
    fppm_b200::note_launches(1);
    FPPM_CUDA_OK(cudaGetLastError());
  }
  if ((rc = copy_out(ctx, out->radius, ctx->d_radius + h0, sizeof(double) * H))) return rc;
  if ((rc = copy_out(ctx, out->gather_radius, ctx->o_gather_r + h0, sizeof(double) * H))) return rc;
  if ((rc = copy_out(ctx, out->tested, ctx->o_tested + h0, H))) return rc;
  if ((rc = copy_out(ctx, out->rejected, ctx->o_rejected + h0, H))) return rc;
  if ((rc = copy_out(ctx, out->t, ctx->o_t64 + h0, sizeof(uint64_t) * H))) return rc;
  if ((rc = copy_out(ctx, out->statistic, ctx->o_stat + h0, sizeof(double) * H))) return rc;
  if ((rc = copy_out(ctx, out->critical, ctx->o_crit + h0, sizeof(double) * H))) return rc;
  if (with_gather) {
    if ((rc = copy_out(ctx, out->flux, ctx->o_flux + 3 * h0, sizeof(double) * 3 * H))) return rc;
    if ((rc = copy_out(ctx, out->radiance, ctx->o_rad + 3 * h0, sizeof(float) * 3 * H))) return rc;
    if ((rc = copy_out(ctx, out->accepted, ctx->o_acc + h0, sizeof(uint32_t) * H))) return rc;
  }
  if ((rc = copy_out(ctx, out->stat_count, ctx->snap_cnt + CG * h0, sizeof(unsigned long long) * CG * H))) return rc;
  if ((rc = copy_out(ctx, out->stat_sum, ctx->snap_sum + CG * h0, sizeof(double) * CG * H))) return rc;
  if ((rc = copy_out(ctx, out->stat_sum_sq, ctx->snap_sq + CG * h0, sizeof(double) * CG * H))) return rc;
  return FPPM_OK;
}

}  // namespace fppm_b200

using namespace fppm_b200;

#define UPLOAD_OK(x)                                                       \
  do {                                                                     \
    cudaError_t e_ = (x);                                                  \
    if (e_ != cudaSuccess) return fail(ctx, FPPM_ERR_CUDA, cudaGetErrorString(e_)); \
  } while (0)
template <typename T>
static int upload(fppm_gpu_ctx *ctx, void *&slot, const T *src, size_t n) {
  if (slot) cudaFree(slot);
  slot = nullptr;
  UPLOAD_OK(cudaMalloc(&slot, sizeof(T) * (n ? n : 1)));
  if (n) UPLOAD_OK(cudaMemcpy(slot, src, sizeof(T) * n, cudaMemcpyHostToDevice));
  return FPPM_OK;
}

#undef UPLOAD_OK

extern "C" {

int fppm_gpu_abi_version(void) { return FPPM_GPU_ABI_VERSION; }

const char *fppm_gpu_status_string(int status) {
  switch (status) {
    case FPPM_OK: return "ok";
    case FPPM_ERR_INVALID_ARGUMENT: return "invalid argument";
    case FPPM_ERR_DOMAIN: return "domain error";
    case FPPM_ERR_CUDA: return "CUDA error";
    case FPPM_ERR_CAPACITY: return "capacity exceeded";
    case FPPM_ERR_STATE: return "invalid call order";
    case FPPM_ERR_NO_DEVICE: return "no sm_100 device";
  }
  return "unknown status";
}

const char *fppm_gpu_last_error(const fppm_gpu_ctx *ctx) { return ctx ? ctx->err.c_str() : ""; }

int fppm_gpu_create(const fppm_gpu_config *config, fppm_gpu_ctx **out) {
  if (!config || !out) return FPPM_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  const fppm_gpu_config &c = *config;
  // GatherRegion ctor validation (gather.cpp:41-50)
  if (!(c.initial_radius > 0)) return FPPM_ERR_INVALID_ARGUMENT;
  if (!(c.k > 0 && c.k < 1)) return FPPM_ERR_INVALID_ARGUMENT;
  if (!(c.alpha >= 0.5 && c.alpha < 1)) return FPPM_ERR_INVALID_ARGUMENT;
  if (!(c.r_min_base > 0 && c.r_min_base <= c.initial_radius)) return FPPM_ERR_INVALID_ARGUMENT;
  if (c.n_annuli < 1 || c.n_sectors < 1 || (long long)c.n_annuli * c.n_sectors < 2) return FPPM_ERR_INVALID_ARGUMENT;
  // deliberate deviation: the reference accepts any n_a * n_s >= 2
  // (gather.cpp:49-50); the device keeps at most 32 sectors per region
  if ((long long)c.n_annuli * c.n_sectors > 32) return FPPM_ERR_CAPACITY;
  if (c.channels != FPPM_CHANNELS_LUMINANCE && c.channels != FPPM_CHANNELS_RGB) return FPPM_ERR_INVALID_ARGUMENT;
  if (c.policy < FPPM_POLICY_FTEST || c.policy > FPPM_POLICY_SCHEDULE) return FPPM_ERR_INVALID_ARGUMENT;
  // gather_kernel: 0 auto, 1 warp (reference cells), 4 fine, 5 3D
  if (c.gather_kernel < 0 || c.gather_kernel > 5 || c.gather_kernel == 2 || c.gather_kernel == 3)
    return FPPM_ERR_INVALID_ARGUMENT;
  if (c.vcm_plus && (c.gather_kernel == 4 || c.mis_n_vm < 0 || !(c.mis_beta > 0.0)))
    return FPPM_ERR_INVALID_ARGUMENT;
  if (c.policy == FPPM_POLICY_FTEST && c.override_decision == FPPM_OVERRIDE_NONE &&
      !(c.alpha_f > 0.0 && c.alpha_f < 1.0)) return FPPM_ERR_INVALID_ARGUMENT;  // stat_tests.cpp:88
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return FPPM_ERR_NO_DEVICE;
  if (c.device < 0 || c.device >= ndev) return FPPM_ERR_NO_DEVICE;
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, c.device) != cudaSuccess || prop.major != 10) return FPPM_ERR_NO_DEVICE;
  if (cudaSetDevice(c.device) != cudaSuccess) return FPPM_ERR_NO_DEVICE;

  auto *ctx = new (std::nothrow) fppm_gpu_ctx;
  if (!ctx) return FPPM_ERR_CAPACITY;
  ctx->cfg = c;
  if (ctx->cfg.max_cells == 0) ctx->cfg.max_cells = 1u << 28;
  ctx->sms = prop.multiProcessorCount;
  ctx->G = c.n_annuli * c.n_sectors;
  ctx->C = c.channels;
  if (c.stream) {
    ctx->stream = static_cast<cudaStream_t>(c.stream);
  } else {
    if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess) {
      delete ctx;
      return FPPM_ERR_CUDA;
    }
    ctx->own_stream = true;
  }
  const size_t Hc = std::max<uint32_t>(c.max_hitpoints, 1);
  const size_t Nc = std::max<uint32_t>(c.max_photons, 1);
  const size_t CG = (size_t)ctx->G * ctx->C;
  cudaError_t e = cudaSuccess;
  auto A = [&](cudaError_t r) { if (e == cudaSuccess) e = r; };
  A(dalloc(&ctx->d_pos, Hc)); A(dalloc(&ctx->d_nrm, Hc)); A(dalloc(&ctx->d_wo, Hc));
  A(dalloc(&ctx->d_thr, Hc)); A(dalloc(&ctx->d_alb, Hc)); A(dalloc(&ctx->d_K, Hc));
  A(dalloc(&ctx->d_eye, Hc)); A(dalloc(&ctx->d_gathered, Hc));
  A(dalloc(&ctx->d_radius, Hc)); A(dalloc(&ctx->d_t, Hc));
  A(dalloc(&ctx->d_st_cnt, Hc * CG)); A(dalloc(&ctx->d_st_sum, Hc * CG)); A(dalloc(&ctx->d_st_sq, Hc * CG));
  A(dalloc(&ctx->d_ppos, Nc * 3)); A(dalloc(&ctx->d_pnrm, Nc * 3)); A(dalloc(&ctx->d_pwi, Nc * 3));
  A(dalloc(&ctx->d_ppos2, Nc * 3)); A(dalloc(&ctx->d_pnrm2, Nc * 3)); A(dalloc(&ctx->d_pwi2, Nc * 3));
  A(dalloc(&ctx->d_ppow2, Nc * 3)); A(dalloc(&ctx->d_pdepth2, Nc));
  A(dalloc(&ctx->d_ppow, Nc * 3)); A(dalloc(&ctx->d_pdepth, Nc));
  A(dalloc(&ctx->recs.rec0, Nc)); A(dalloc(&ctx->recs.rec1, Nc));
  A(dalloc(&ctx->recs.rec2, Nc)); A(dalloc(&ctx->recs.rec3, Nc));
  A(dalloc(&ctx->recs.pack, 4 * Nc));  // records packed in input order, then permuted whole
  A(dalloc(&ctx->sort.keys_a, Nc)); A(dalloc(&ctx->sort.vals_a, Nc));
  A(dalloc(&ctx->sort.keys_b, Nc)); A(dalloc(&ctx->sort.vals_b, Nc));
  A(dalloc(&ctx->sort.hist, radix_hist_entries((uint32_t)Nc)));
  A(dalloc(&ctx->d_hdr, 1)); A(dalloc(&ctx->d_bounds, 8)); A(dalloc(&ctx->d_cell, 1));
  A(dalloc(&ctx->d_cell_chk, 1));
  A(dalloc(&ctx->d_lean_ok, 1));
  A(cudaMemset(ctx->d_lean_ok, 0, sizeof(uint32_t)));
  A(cudaMallocHost(&ctx->h_hdr, sizeof(GridHeader)));
  A(cudaMallocHost(&ctx->h_bounds_init, sizeof(long long) * 8));
  A(cudaMallocHost(&ctx->h_cell, sizeof(double)));
  A(cudaMallocHost(&ctx->h_counters, sizeof(unsigned long long) * 8));
  A(dalloc(&ctx->o_gather_r, Hc)); A(dalloc(&ctx->o_stat, Hc)); A(dalloc(&ctx->o_crit, Hc));
  A(dalloc(&ctx->o_flux, Hc * 3)); A(dalloc(&ctx->o_flags, Hc)); A(dalloc(&ctx->o_rad, Hc * 3));
  A(dalloc(&ctx->o_acc, Hc));
  A(dalloc(&ctx->d_counters, 4)); A(dalloc(&ctx->d_iter_tr, 2)); A(dalloc(&ctx->d_work, 1));
  A(dalloc(&ctx->d_rmax_bits, 1));
  A(dalloc(&ctx->tile.sort.keys_a, Hc)); A(dalloc(&ctx->tile.sort.vals_a, Hc));
  A(dalloc(&ctx->tile.sort.keys_b, Hc)); A(dalloc(&ctx->tile.sort.vals_b, Hc));
  A(dalloc(&ctx->tile.sort.hist, radix_hist_entries((uint32_t)Hc)));
  A(dalloc(&ctx->tile.hp_map, 3 * Hc));
  A(dalloc(&ctx->tile.hp_nc, Hc + 1)); A(dalloc(&ctx->tile.hp_rbase, Hc + 1));
  A(dalloc(&ctx->tile.hp_scan_tmp, Hc / 4096 + 8));
  A(dalloc(&ctx->tile.hp_span, Hc));
  A(cudaMemset(ctx->tile.hp_nc, 0, sizeof(uint32_t) * (Hc + 1)));
  if (c.vcm_plus) {
    A(dalloc(&ctx->d_eye_mis, Hc));
    A(cudaMemset(ctx->d_eye_mis, 0, sizeof(double2) * Hc));
    for (int i = 0; i < 3; ++i) {
      A(dalloc(&ctx->d_pmis_in[i], Nc));
      A(dalloc(&ctx->d_pmis[i], Nc));
    }
  }
  A(dalloc(reinterpret_cast<char **>(&ctx->tile.fhot), fine_hot_bytes() * Hc));
  A(dalloc(&ctx->tile.fbox, Hc));
  A(dalloc(reinterpret_cast<char **>(&ctx->tile.fhit), fine_hit_bytes() * Hc));
  A(dalloc(&ctx->tile.nonempty, 1));
  A(cudaMallocHost(&ctx->h_total, 2 * sizeof(uint32_t)));
  if (e != cudaSuccess) {
    int rc = cuda_fail(ctx, e, "fppm_gpu_create allocation");
    fppm_gpu_destroy(ctx);
    return rc == FPPM_ERR_CUDA ? FPPM_ERR_CAPACITY : rc;
  }
  for (int a = 0; a < 3; ++a) {
    ctx->h_bounds_init[a] = LLONG_MAX;
    ctx->h_bounds_init[3 + a] = LLONG_MIN;
  }
  ctx->h_bounds_init[6] = LLONG_MAX;  // the photons' z bit patterns (k_cell_bounds)
  ctx->h_bounds_init[7] = LLONG_MIN;
  cudaMemsetAsync(ctx->d_counters, 0, sizeof(unsigned long long) * 4, ctx->stream);
  if (c.policy == FPPM_POLICY_CHI2) {
    int st = 0;
    ctx->chi2_crit = host_chi2_quantile(1.0 - c.alpha_chi2, (double)(ctx->G - 1), &st);
    if (st) {
      fppm_gpu_destroy(ctx);
      return FPPM_ERR_INVALID_ARGUMENT;
    }
  }
  int rc = ensure_crit(ctx, std::max<uint64_t>(64, 2));
  if (rc) {
    fppm_gpu_destroy(ctx);
    return rc;
  }
  *out = ctx;
  return FPPM_OK;
}

int fppm_gpu_destroy(fppm_gpu_ctx *ctx) {
  if (!ctx) return FPPM_OK;
  if (ctx->gstream) cudaStreamSynchronize(ctx->gstream);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  void *dev[] = {ctx->d_pos, ctx->d_nrm, ctx->d_wo, ctx->d_thr, ctx->d_alb, ctx->d_K, ctx->d_eye,
                 ctx->d_gathered, ctx->d_radius, ctx->d_t, ctx->d_st_cnt, ctx->d_st_sum,
                 ctx->d_st_sq, ctx->d_ppos, ctx->d_pnrm, ctx->d_pwi, ctx->d_ppow, ctx->d_pdepth,
                 ctx->d_ppos2, ctx->d_pnrm2, ctx->d_pwi2, ctx->d_ppow2, ctx->d_pdepth2,
                 ctx->recs.rec0, ctx->recs.rec1, ctx->recs.rec2, ctx->recs.rec3, ctx->recs.pack,
                 ctx->sort.keys_a,
                 ctx->sort.vals_a, ctx->sort.keys_b, ctx->sort.vals_b, ctx->sort.hist,
                 ctx->d_cell_start, ctx->d_hdr, ctx->d_bounds, ctx->d_cell, ctx->d_cell_chk, ctx->d_lean_ok,
                 ctx->o_gather_r, ctx->o_stat, ctx->o_crit, ctx->o_flux, ctx->o_flags, ctx->o_rad,
                 ctx->o_acc, ctx->o_tested, ctx->o_rejected, ctx->o_t64,
                 ctx->snap_cnt, ctx->snap_sum, ctx->snap_sq, ctx->d_counters,
                 ctx->d_iter_tr, ctx->d_work, ctx->d_rmax_bits, ctx->d_crit, ctx->d_scratch};
  for (void *p : dev)
    if (p) cudaFree(p);
  const TileSched &T = ctx->tile;
  void *tdev[] = {T.sort.keys_a, T.sort.vals_a, T.sort.keys_b, T.sort.vals_b, T.sort.hist,
                  T.hp_start, T.items, T.chunks, T.item_base, T.scan_tmp, T.fdesc, T.fhot, T.fbox, T.fhit, T.pbase, T.partials,
                  T.hp_map, T.nonempty, T.hp_nc, T.hp_rbase, T.hp_scan_tmp, T.hp_span};
  for (void *p : tdev)
    if (p) cudaFree(p);
  if (ctx->cstream) cudaStreamSynchronize(ctx->cstream);
  if (ctx->d_eye_mis) cudaFree(ctx->d_eye_mis);
  if (ctx->d_emit) cudaFree(ctx->d_emit);
  {
    void *bq[] = {ctx->b_pos, ctx->b_sn, ctx->b_wi, ctx->b_thr, ctx->b_mis, ctx->b_mat, ctx->d_splat,
                  ctx->q_sort.keys_a, ctx->q_sort.vals_a, ctx->q_sort.keys_b, ctx->q_sort.vals_b, ctx->q_sort.hist,
                  ctx->q_pos, ctx->q_nrm, ctx->q_wo, ctx->q_thr, ctx->q_alb, ctx->q_K, ctx->q_eye,
                  ctx->q_gathered, ctx->q_radius, ctx->q_rows, ctx->q_mis, ctx->v_d, ctx->v_i, ctx->v_n,
                  ctx->v_rng, ctx->d_keep, ctx->d_keep_dst, ctx->d_keep_scan, ctx->d_hpbox};
    for (void *p : bq)
      if (p) cudaFree(p);
  }
  if (ctx->d_rows) cudaFree(ctx->d_rows);
  if (ctx->hot3) cudaFree(ctx->hot3);
  if (ctx->hot3_hits) cudaFree(ctx->hot3_hits);
  for (void *p : ctx->c5_mem)
    if (p) cudaFree(p);
  if (ctx->d_film) cudaFree(ctx->d_film);
  if (ctx->d_vcvm) cudaFree(ctx->d_vcvm);
  for (void *p : ctx->scene_mem)
    if (p) cudaFree(p);
  {
    void *tp[] = {ctx->t_pos, ctx->t_nrm, ctx->t_wi, ctx->t_pow, ctx->t_depth, ctx->t_count, ctx->t_base,
                  ctx->t_scan, ctx->t_mis, ctx->t_ctr};
    for (void *p : tp)
      if (p) cudaFree(p);
  }
  for (int i = 0; i < 3; ++i) {
    if (ctx->d_pmis_in[i]) cudaFree(ctx->d_pmis_in[i]);
    if (ctx->d_pmis[i]) cudaFree(ctx->d_pmis[i]);
  }
  for (int i = 0; i < 2; ++i) {
    if (ctx->ev_copied[i]) cudaEventDestroy(ctx->ev_copied[i]);
    if (ctx->ev_free[i]) cudaEventDestroy(ctx->ev_free[i]);
  }
  if (ctx->cstream) cudaStreamDestroy(ctx->cstream);
  for (cudaEvent_t e : {ctx->ev_g_hdr, ctx->ev_g_sorted, ctx->ev_g_recs, ctx->ev_hdr, ctx->ev_sched})
    if (e) cudaEventDestroy(e);
  if (ctx->gstream) cudaStreamDestroy(ctx->gstream);
  for (auto &pr : ctx->ev_k)
    for (cudaEvent_t e : pr)
      if (e) cudaEventDestroy(e);
  if (ctx->h_total) cudaFreeHost(ctx->h_total);
  if (ctx->h_hdr) cudaFreeHost(ctx->h_hdr);
  if (ctx->h_bounds_init) cudaFreeHost(ctx->h_bounds_init);
  if (ctx->h_cell) cudaFreeHost(ctx->h_cell);
  if (ctx->h_counters) cudaFreeHost(ctx->h_counters);
  if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
  return FPPM_OK;
}

int fppm_gpu_synchronize(fppm_gpu_ctx *ctx) {
  if (!ctx) return FPPM_ERR_INVALID_ARGUMENT;
  JOIN_RECS(ctx);
  if (ctx->cstream) FPPM_CUDA_OK(cudaStreamSynchronize(ctx->cstream));
  FPPM_CUDA_OK(cudaStreamSynchronize(ctx->stream));
  return FPPM_OK;
}

void *fppm_gpu_stream(fppm_gpu_ctx *ctx) {
  if (!ctx) return nullptr;
  (void)join_recs(ctx);  // work the caller enqueues follows the record build
  return (void *)ctx->stream;
}

int fppm_gpu_device_view_get(fppm_gpu_ctx *ctx, fppm_gpu_device_view *v) {
  if (!ctx || !v) return FPPM_ERR_INVALID_ARGUMENT;
  JOIN_RECS(ctx);
  v->photon_pos = ctx->d_ppos;
  v->photon_normal = ctx->d_pnrm;
  v->photon_wi = ctx->d_pwi;
  v->photon_power = ctx->d_ppow;
  v->photon_depth = ctx->d_pdepth;
  v->radius = ctx->d_radius;
  v->counters = reinterpret_cast<uint64_t *>(ctx->d_counters);
  return FPPM_OK;
}

// ------------------------------------------------------------------ regions
static bool lean_config(const fppm_gpu_ctx *ctx) {
  const fppm_gpu_config &c = ctx->cfg;
  return ctx->C == 1 && c.n_annuli <= 2 && c.n_sectors == 4 && !c.vcm_plus && gather_variant(ctx) == 4;
}

static int finish_hitpoints(fppm_gpu_ctx *ctx, uint32_t n, bool has_gathered) {
  ++ctx->hp_version;  // cached hit-point bins are stale
  if (!has_gathered) FPPM_CUDA_OK(cudaMemsetAsync(ctx->d_gathered, 1, std::max<uint32_t>(n, 1), ctx->stream));
  FPPM_CUDA_OK(launch_hit_weights(ctx->stream, ctx->d_nrm, ctx->d_wo, ctx->d_thr, ctx->d_alb, n, ctx->d_K));
  if (lean_config(ctx))
    FPPM_CUDA_OK(launch_lean_check(ctx->stream, ctx->d_pos, ctx->d_nrm, ctx->d_K, ctx->d_gathered, n, ctx->d_lean_ok));
  else
    FPPM_CUDA_OK(cudaMemsetAsync(ctx->d_lean_ok, 0, sizeof(uint32_t), ctx->stream));
  const bool reset = n != ctx->H;
  ctx->H = n;
  if (ctx->grid_explicit) ctx->rcheck = true;  // a newly gathered region may exceed the cell
  if (reset) return fppm_gpu_reset_regions(ctx);
  return FPPM_OK;
}

static int set_hitpoints(fppm_gpu_ctx *ctx, const fppm_hitpoints *hp, uint32_t n, cudaMemcpyKind kind) {
  if (ctx) JOIN_RECS(ctx);
  if (!ctx || !hp) return FPPM_ERR_INVALID_ARGUMENT;
  if (n > ctx->cfg.max_hitpoints) return fail(ctx, FPPM_ERR_CAPACITY, "hit points exceed max_hitpoints");
  if (n && (!hp->pos || !hp->normal || !hp->wo || !hp->throughput || !hp->albedo || !hp->eye_depth))
    return fail(ctx, FPPM_ERR_INVALID_ARGUMENT, "null hit point array");
  const size_t b3 = sizeof(double3) * n;
  cudaStream_t s = ctx->stream;
  if (n) {
    FPPM_CUDA_OK(cudaMemcpyAsync(ctx->d_pos, hp->pos, b3, kind, s));
    FPPM_CUDA_OK(cudaMemcpyAsync(ctx->d_nrm, hp->normal, b3, kind, s));
    FPPM_CUDA_OK(cudaMemcpyAsync(ctx->d_wo, hp->wo, b3, kind, s));
    FPPM_CUDA_OK(cudaMemcpyAsync(ctx->d_thr, hp->throughput, b3, kind, s));
    FPPM_CUDA_OK(cudaMemcpyAsync(ctx->d_alb, hp->albedo, b3, kind, s));
    FPPM_CUDA_OK(cudaMemcpyAsync(ctx->d_eye, hp->eye_depth, sizeof(uint32_t) * n, kind, s));
    if (hp->gathered) FPPM_CUDA_OK(cudaMemcpyAsync(ctx->d_gathered, hp->gathered, n, kind, s));
  }
  return finish_hitpoints(ctx, n, hp->gathered != nullptr);
}

int fppm_gpu_set_hitpoints(fppm_gpu_ctx *ctx, const fppm_hitpoints *host, uint32_t n) {
  return set_hitpoints(ctx, host, n, cudaMemcpyHostToDevice);
}

int fppm_gpu_set_hitpoints_device(fppm_gpu_ctx *ctx, const fppm_hitpoints *dev, uint32_t n) {
  return set_hitpoints(ctx, dev, n, cudaMemcpyDeviceToDevice);
}

int fppm_gpu_generate_raster_hitpoints(fppm_gpu_ctx *ctx, uint32_t W) {
  if (!ctx) return FPPM_ERR_INVALID_ARGUMENT;
  JOIN_RECS(ctx);
  const uint64_t n = (uint64_t)W * W;
  if (n > ctx->cfg.max_hitpoints) return fail(ctx, FPPM_ERR_CAPACITY, "raster exceeds max_hitpoints");
  launch_raster_hitpoints(ctx->stream, W, ctx->d_pos, ctx->d_nrm, ctx->d_wo, ctx->d_thr, ctx->d_alb,
                          ctx->d_eye, ctx->d_gathered, ctx->sms);
  FPPM_CUDA_OK(cudaGetLastError());
  return finish_hitpoints(ctx, (uint32_t)n, true);
}

int fppm_gpu_c5_setup(fppm_gpu_ctx *ctx, uint64_t seed, uint32_t n_hitpoints) {
  if (!ctx || n_hitpoints == 0) return FPPM_ERR_INVALID_ARGUMENT;
  JOIN_RECS(ctx);
  for (void *&p : ctx->c5_mem) {
    if (p) cudaFree(p);
    p = nullptr;
  }
  int G = 1;  // NN grid: about 2 hit points per cell
  while ((unsigned long long)(G + 1) * (G + 1) * (G + 1) * 2ull <= n_hitpoints) ++G;
  const unsigned long long nc = (unsigned long long)G * G * G;
  const size_t H = n_hitpoints;
  const size_t sizes[8] = {sizeof(double) * 5 * kC5Clusters, sizeof(double3) * H, sizeof(double3) * H,
                           sizeof(uint32_t) * (nc + 1), sizeof(uint32_t) * H, sizeof(uint32_t) * (nc + 2),
                           sizeof(uint32_t) * nc, sizeof(uint32_t) * H};
  for (int i = 0; i < 8; ++i) FPPM_CUDA_OK(cudaMalloc(&ctx->c5_mem[i], sizes[i]));
  uint32_t *scan_tmp = nullptr;
  FPPM_CUDA_OK(dalloc(&scan_tmp, (nc + 1) / 4096 + 8));
  C5Args &C = ctx->c5;
  C.seed = seed;
  C.H = n_hitpoints;
  C.G = G;
  C.clusters = static_cast<double *>(ctx->c5_mem[0]);
  C.pos = static_cast<double3 *>(ctx->c5_mem[1]);
  C.nrm = static_cast<double3 *>(ctx->c5_mem[2]);
  C.start = static_cast<uint32_t *>(ctx->c5_mem[5]);
  C.items = static_cast<uint32_t *>(ctx->c5_mem[7]);
  cudaError_t e = launch_c5_setup(ctx->stream, seed, n_hitpoints, G, static_cast<double *>(ctx->c5_mem[0]),
                                  static_cast<double3 *>(ctx->c5_mem[1]), static_cast<double3 *>(ctx->c5_mem[2]),
                                  static_cast<uint32_t *>(ctx->c5_mem[3]), static_cast<uint32_t *>(ctx->c5_mem[4]),
                                  static_cast<uint32_t *>(ctx->c5_mem[5]), static_cast<uint32_t *>(ctx->c5_mem[6]),
                                  static_cast<uint32_t *>(ctx->c5_mem[7]), scan_tmp, ctx->sms);
  cudaError_t e2 = cudaStreamSynchronize(ctx->stream);
  cudaFree(scan_tmp);
  FPPM_CUDA_OK(e);
  FPPM_CUDA_OK(e2);
  return FPPM_OK;
}

int fppm_gpu_c5_hitpoints(fppm_gpu_ctx *ctx, uint32_t h0, uint32_t n) {
  if (!ctx) return FPPM_ERR_INVALID_ARGUMENT;
  JOIN_RECS(ctx);
  if (!ctx->c5.pos) return fail(ctx, FPPM_ERR_STATE, "c5_hitpoints before c5_setup");
  if ((uint64_t)h0 + n > ctx->c5.H) return fail(ctx, FPPM_ERR_INVALID_ARGUMENT, "hit point range exceeds C5 set");
  if (n > ctx->cfg.max_hitpoints) return fail(ctx, FPPM_ERR_CAPACITY, "hit points exceed max_hitpoints");
  FPPM_CUDA_OK(launch_c5_set_hitpoints(ctx->stream, ctx->c5, h0, n, ctx->d_pos, ctx->d_nrm, ctx->d_wo, ctx->d_thr,
                                       ctx->d_alb, ctx->d_eye, ctx->d_gathered, ctx->sms));
  return finish_hitpoints(ctx, n, true);
}

int fppm_gpu_reset_regions(fppm_gpu_ctx *ctx) {
  if (!ctx) return FPPM_ERR_INVALID_ARGUMENT;
  JOIN_RECS(ctx);
  const size_t H = std::max<uint32_t>(ctx->H, 1), CG = (size_t)ctx->G * ctx->C;
  k_fill_regions<<<(unsigned)((H + 255) / 256), 256, 0, ctx->stream>>>(ctx->d_radius, ctx->d_t, ctx->H,
                                                                     ctx->cfg.initial_radius);
  note_launches(1);
  FPPM_CUDA_OK(cudaGetLastError());
  FPPM_CUDA_OK(cudaMemsetAsync(ctx->d_st_cnt, 0, sizeof(unsigned long long) * H * CG, ctx->stream));
  FPPM_CUDA_OK(cudaMemsetAsync(ctx->d_st_sum, 0, sizeof(double) * H * CG, ctx->stream));
  FPPM_CUDA_OK(cudaMemsetAsync(ctx->d_st_sq, 0, sizeof(double) * H * CG, ctx->stream));
  ctx->end_calls = 0;
  return FPPM_OK;
}

int fppm_gpu_get_regions(fppm_gpu_ctx *ctx, double *radius, uint64_t *t, uint64_t *stat_count,
                         double *stat_sum, double *stat_sum_sq) {
  if (!ctx) return FPPM_ERR_INVALID_ARGUMENT;
  JOIN_RECS(ctx);
  const size_t H = ctx->H, CG = (size_t)ctx->G * ctx->C;
  int rc;
  if ((rc = copy_out(ctx, radius, ctx->d_radius, sizeof(double) * H))) return rc;
  if ((rc = copy_out(ctx, stat_count, ctx->d_st_cnt, sizeof(unsigned long long) * H * CG))) return rc;
  if ((rc = copy_out(ctx, stat_sum, ctx->d_st_sum, sizeof(double) * H * CG))) return rc;
  if ((rc = copy_out(ctx, stat_sum_sq, ctx->d_st_sq, sizeof(double) * H * CG))) return rc;
  std::vector<uint32_t> t32(t ? H : 0);
  if (t && (rc = copy_out(ctx, t32.data(), ctx->d_t, sizeof(uint32_t) * H))) return rc;
  FPPM_CUDA_OK(cudaStreamSynchronize(ctx->stream));
  for (size_t h = 0; t && h < H; ++h) t[h] = t32[h];
  return FPPM_OK;
}

int fppm_gpu_set_regions(fppm_gpu_ctx *ctx, const double *radius, const uint64_t *t,
                         const uint64_t *stat_count, const double *stat_sum,
                         const double *stat_sum_sq) {
  if (!ctx) return FPPM_ERR_INVALID_ARGUMENT;
  JOIN_RECS(ctx);
  const size_t H = ctx->H, CG = (size_t)ctx->G * ctx->C;
  cudaStream_t s = ctx->stream;
  if (radius) {
    FPPM_CUDA_OK(cudaMemcpyAsync(ctx->d_radius, radius, sizeof(double) * H, cudaMemcpyHostToDevice, s));
    ctx->rcheck = true;  // radii may now exceed the built grid's cell
  }
  if (stat_count) FPPM_CUDA_OK(cudaMemcpyAsync(ctx->d_st_cnt, stat_count, 8 * H * CG, cudaMemcpyHostToDevice, s));
  if (stat_sum) FPPM_CUDA_OK(cudaMemcpyAsync(ctx->d_st_sum, stat_sum, 8 * H * CG, cudaMemcpyHostToDevice, s));
  if (stat_sum_sq) FPPM_CUDA_OK(cudaMemcpyAsync(ctx->d_st_sq, stat_sum_sq, 8 * H * CG, cudaMemcpyHostToDevice, s));
  if (t) {
    std::vector<uint32_t> t32(H);
    uint64_t tmax = 0;
    for (size_t h = 0; h < H; ++h) {
      if (t[h] < 1 || t[h] > 0xffffffffull) return fail(ctx, FPPM_ERR_INVALID_ARGUMENT, "t out of range");
      t32[h] = (uint32_t)t[h];
      tmax = std::max<uint64_t>(tmax, t[h]);
    }
    FPPM_CUDA_OK(cudaMemcpyAsync(ctx->d_t, t32.data(), sizeof(uint32_t) * H, cudaMemcpyHostToDevice, s));
    FPPM_CUDA_OK(cudaStreamSynchronize(s));
    if (tmax > ctx->end_calls + 1) ctx->end_calls = tmax - 1;
  }
  FPPM_CUDA_OK(cudaStreamSynchronize(s));
  return FPPM_OK;
}

static int device_max_radius(fppm_gpu_ctx *ctx, double *dst, const uint8_t *gathered = nullptr) {
  FPPM_CUDA_OK(cudaMemsetAsync(dst, 0, sizeof(double), ctx->stream));
  if (ctx->H) {
    unsigned blocks = (ctx->H + 255) / 256;
    blocks = std::min<unsigned>(blocks, (unsigned)ctx->sms * 4);
    k_max_radius<<<blocks, 256, 0, ctx->stream>>>(ctx->d_radius, ctx->H, dst, gathered);
    note_launches(1);
    FPPM_CUDA_OK(cudaGetLastError());
  }
  return FPPM_OK;
}

int fppm_gpu_max_radius_device(fppm_gpu_ctx *ctx, double *d_r_max) {
  if (!ctx || !d_r_max) return FPPM_ERR_INVALID_ARGUMENT;
  JOIN_RECS(ctx);
  return device_max_radius(ctx, d_r_max);
}

int fppm_gpu_max_radius(fppm_gpu_ctx *ctx, double *r_max) {
  if (!ctx || !r_max) return FPPM_ERR_INVALID_ARGUMENT;
  JOIN_RECS(ctx);
  int rc = device_max_radius(ctx, ctx->d_cell);
  if (rc) return rc;
  FPPM_CUDA_OK(cudaMemcpyAsync(ctx->h_cell, ctx->d_cell, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  FPPM_CUDA_OK(cudaStreamSynchronize(ctx->stream));
  *r_max = *ctx->h_cell;
  return FPPM_OK;
}

// ------------------------------------------------------------------ photons + grid
static void use_staging(fppm_gpu_ctx *ctx, int set = 0) {
  ctx->stage_cur = set;
  ctx->in_pos = set ? ctx->d_ppos2 : ctx->d_ppos;
  ctx->in_nrm = set ? ctx->d_pnrm2 : ctx->d_pnrm;
  ctx->in_wi = set ? ctx->d_pwi2 : ctx->d_pwi;
  ctx->in_pow = set ? ctx->d_ppow2 : ctx->d_ppow;
  ctx->in_depth = set ? ctx->d_pdepth2 : ctx->d_pdepth;
}

// Host uploads go to the staging set not holding the current photons, on the
// copy stream: the copy waits only until the grid build that last read that
// set has consumed it (ev_free), and the next grid build waits for the copy
// (ev_copied).  With pinned host memory the call returns immediately.
// Sampled digest of a host photon batch: every field of up to 4096 records
// spread evenly over the batch (plus the last one).  fppm_gpu_adopt_photons
// recomputes it to catch arrays rewritten after fppm_gpu_prefetch_photons.
static uint64_t photon_digest(const fppm_photons &p, uint32_t n) {
  uint64_t h = 1469598103934665603ull ^ n;
  auto mix = [&h](const void *src, size_t bytes) {
    const unsigned char *b = static_cast<const unsigned char *>(src);
    for (size_t i = 0; i < bytes; ++i) h = (h ^ b[i]) * 1099511628211ull;
  };
  if (n == 0) return h;
  const uint32_t m = std::min<uint32_t>(n, 4096u);
  for (uint32_t k = 0; k <= m; ++k) {
    const uint32_t i = k == m ? n - 1 : (uint32_t)(((uint64_t)k * n) / m);
    mix(p.pos + 3 * (size_t)i, 12);
    mix(p.normal + 3 * (size_t)i, 12);
    mix(p.wi + 3 * (size_t)i, 12);
    mix(p.power + 3 * (size_t)i, 12);
    mix(p.depth + i, 4);
  }
  return h;
}

// upload n photons into staging set `set` on the copy stream (ev_copied[set])
static int upload_set(fppm_gpu_ctx *ctx, const fppm_photons *p, uint32_t n, cudaMemcpyKind kind, int set);

static int set_photons(fppm_gpu_ctx *ctx, const fppm_photons *p, uint32_t n, cudaMemcpyKind kind) {
  if (ctx) JOIN_RECS(ctx);
  if (!ctx || !p) return FPPM_ERR_INVALID_ARGUMENT;
  if (n > ctx->cfg.max_photons) return fail(ctx, FPPM_ERR_CAPACITY, "photons exceed max_photons");
  if (n && (!p->pos || !p->normal || !p->wi || !p->power || !p->depth))
    return fail(ctx, FPPM_ERR_INVALID_ARGUMENT, "null photon array");
  ctx->pf_set = -1;  // any explicit upload supersedes the prefetch
  const int set = ctx->stage_cur ^ 1;
  int rc = upload_set(ctx, p, n, kind, set);
  if (rc) return rc;
  ctx->stage_pending = set;
  ctx->N = n;
  ctx->grid_valid = false;
  use_staging(ctx, set);
  return FPPM_OK;
}

// Next batch into the staging set not holding the current photons, while the
// current iteration runs; fppm_gpu_adopt_photons(token) makes it current.
int fppm_gpu_set_photons_packed(fppm_gpu_ctx *ctx, const void *d_packed, uint32_t parts, uint64_t part_stride,
                                const uint32_t *part_n, const double *d_margin, uint32_t *n_kept) {
  if (!ctx || (parts && (!d_packed || !part_n))) return FPPM_ERR_INVALID_ARGUMENT;
  JOIN_RECS(ctx);
  if (parts > (uint32_t)kMaxPackedParts) return fail(ctx, FPPM_ERR_INVALID_ARGUMENT, "more than 64 packed parts");
  unsigned long long total = 0;
  for (uint32_t p = 0; p < parts; ++p) {
    if (part_n[p] > part_stride) return fail(ctx, FPPM_ERR_INVALID_ARGUMENT, "part count exceeds the part stride");
    total += part_n[p];
  }
  if (total >= 0xffffffffull) return fail(ctx, FPPM_ERR_CAPACITY, "packed photons exceed 2^32 - 1");
  cudaStream_t s = ctx->stream;
  if (total + 1 > ctx->keep_cap) {
    FPPM_CUDA_OK(cudaStreamSynchronize(s));
    void *kp[] = {ctx->d_keep, ctx->d_keep_dst, ctx->d_keep_scan};
    for (void *p : kp)
      if (p) cudaFree(p);
    ctx->d_keep = ctx->d_keep_dst = ctx->d_keep_scan = nullptr;
    ctx->keep_cap = 0;
    const unsigned long long cap = std::max<unsigned long long>(total + 1, 4096);
    FPPM_CUDA_OK(dalloc(&ctx->d_keep, cap));
    FPPM_CUDA_OK(dalloc(&ctx->d_keep_dst, cap));
    FPPM_CUDA_OK(dalloc(&ctx->d_keep_scan, cap / 4096 + 8));
    ctx->keep_cap = cap;
  }
  if (!ctx->d_hpbox) FPPM_CUDA_OK(dalloc(&ctx->d_hpbox, 6));
  const double *box = nullptr;
  if (d_margin && ctx->H) {
    FPPM_CUDA_OK(launch_hp_box(s, reinterpret_cast<const double3 *>(ctx->d_pos), ctx->H, ctx->d_hpbox));
    box = ctx->d_hpbox;
  }
  // staging set 0 is rewritten (as by the light phase): wait for an upload into it
  if (ctx->ev_copied[0])  // any earlier upload into set 0 (a superseded one too)
    FPPM_CUDA_OK(cudaStreamWaitEvent(s, ctx->ev_copied[0], 0));
  ctx->stage_pending = -1;
  ctx->pf_set = -1;
  FPPM_CUDA_OK(launch_cull_packed(s, static_cast<const uint32_t *>(d_packed), part_stride, parts, part_n, box,
                                  d_margin, ctx->d_keep, ctx->d_keep_dst, ctx->d_keep_scan, ctx->d_ppos,
                                  ctx->d_pnrm, ctx->d_pwi, ctx->d_ppow, ctx->d_pdepth, ctx->sms));
  FPPM_CUDA_OK(cudaMemcpyAsync(ctx->h_total, ctx->d_keep_dst + total, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
  FPPM_CUDA_OK(cudaStreamSynchronize(s));
  const uint32_t kept = ctx->h_total[0];
  if (kept > ctx->cfg.max_photons) return fail(ctx, FPPM_ERR_CAPACITY, "photons exceed max_photons");
  ctx->N = kept;
  ctx->grid_valid = false;
  use_staging(ctx);
  if (n_kept) *n_kept = kept;
  return FPPM_OK;
}

int fppm_gpu_prefetch_photons(fppm_gpu_ctx *ctx, const fppm_photons *host, uint32_t n, uint64_t *token) {
  if (!ctx || !host || !token) return FPPM_ERR_INVALID_ARGUMENT;
  JOIN_RECS(ctx);
  if (n > ctx->cfg.max_photons) return fail(ctx, FPPM_ERR_CAPACITY, "photons exceed max_photons");
  if (n && (!host->pos || !host->normal || !host->wi || !host->power || !host->depth))
    return fail(ctx, FPPM_ERR_INVALID_ARGUMENT, "null photon array");
  const int set = ctx->stage_cur ^ 1;
  if (ctx->stage_pending == set) return fail(ctx, FPPM_ERR_STATE, "prefetch while the staged batch is unconsumed");
  ctx->pf_set = -1;
  const uint64_t digest = photon_digest(*host, n);
  int rc = upload_set(ctx, host, n, cudaMemcpyHostToDevice, set);
  if (rc) return rc;
  ctx->pf_set = set;
  ctx->pf_src = *host;
  ctx->pf_n = n;
  ctx->pf_digest = digest;
  ctx->pf_token = ++ctx->pf_counter;
  *token = ctx->pf_token;
  return FPPM_OK;
}

int fppm_gpu_adopt_photons(fppm_gpu_ctx *ctx, uint64_t token) {
  if (!ctx) return FPPM_ERR_INVALID_ARGUMENT;
  JOIN_RECS(ctx);
  if (ctx->pf_set < 0 || token == 0 || token != ctx->pf_token)
    return fail(ctx, FPPM_ERR_STATE, "no pending prefetch with this token (superseded or already adopted)");
  const int set = ctx->pf_set;
  ctx->pf_set = -1;
  if (photon_digest(ctx->pf_src, ctx->pf_n) != ctx->pf_digest)
    return fail(ctx, FPPM_ERR_STATE,
                "prefetched photon arrays changed after fppm_gpu_prefetch_photons; upload them with fppm_gpu_set_photons");
  ctx->stage_pending = set;
  ctx->N = ctx->pf_n;
  ctx->grid_valid = false;
  use_staging(ctx, set);
  return FPPM_OK;
}

static int upload_set(fppm_gpu_ctx *ctx, const fppm_photons *p, uint32_t n, cudaMemcpyKind kind, int set) {
  if (!ctx->cstream) {
    FPPM_CUDA_OK(cudaStreamCreateWithFlags(&ctx->cstream, cudaStreamNonBlocking));
    for (int i = 0; i < 2; ++i) {
      FPPM_CUDA_OK(cudaEventCreateWithFlags(&ctx->ev_copied[i], cudaEventDisableTiming));
      FPPM_CUDA_OK(cudaEventCreateWithFlags(&ctx->ev_free[i], cudaEventDisableTiming));
    }
  }
  cudaStream_t s = ctx->cstream;
  // the set must not be overwritten while an enqueued grid build still reads it,
  // nor while earlier work on the context stream (e.g. generation) writes it
  if (ctx->free_recorded[set]) FPPM_CUDA_OK(cudaStreamWaitEvent(s, ctx->ev_free[set], 0));
  else FPPM_CUDA_OK(cudaStreamSynchronize(ctx->stream));
  const size_t b3 = sizeof(float) * 3 * n;
  if (n) {
    FPPM_CUDA_OK(cudaMemcpyAsync(set ? ctx->d_ppos2 : ctx->d_ppos, p->pos, b3, kind, s));
    FPPM_CUDA_OK(cudaMemcpyAsync(set ? ctx->d_pnrm2 : ctx->d_pnrm, p->normal, b3, kind, s));
    FPPM_CUDA_OK(cudaMemcpyAsync(set ? ctx->d_pwi2 : ctx->d_pwi, p->wi, b3, kind, s));
    FPPM_CUDA_OK(cudaMemcpyAsync(set ? ctx->d_ppow2 : ctx->d_ppow, p->power, b3, kind, s));
    FPPM_CUDA_OK(cudaMemcpyAsync(set ? ctx->d_pdepth2 : ctx->d_pdepth, p->depth, sizeof(uint32_t) * n,
                                 kind, s));
  }
  FPPM_CUDA_OK(cudaEventRecord(ctx->ev_copied[set], s));
  return FPPM_OK;
}

int fppm_gpu_set_photons(fppm_gpu_ctx *ctx, const fppm_photons *host, uint32_t n) {
  return set_photons(ctx, host, n, cudaMemcpyHostToDevice);
}

// Zero copy: the grid build reads the caller's device arrays directly; they
// must stay valid and unchanged until the next build_grid has been issued.
int fppm_gpu_set_photons_device(fppm_gpu_ctx *ctx, const fppm_photons *dev, uint32_t n) {
  if (!ctx || !dev) return FPPM_ERR_INVALID_ARGUMENT;
  JOIN_RECS(ctx);
  if (n > ctx->cfg.max_photons) return fail(ctx, FPPM_ERR_CAPACITY, "photons exceed max_photons");
  if (n && (!dev->pos || !dev->normal || !dev->wi || !dev->power || !dev->depth))
    return fail(ctx, FPPM_ERR_INVALID_ARGUMENT, "null photon array");
  ctx->stage_pending = -1;  // an unconsumed upload is superseded
  ctx->pf_set = -1;
  ctx->in_pos = dev->pos;
  ctx->in_nrm = dev->normal;
  ctx->in_wi = dev->wi;
  ctx->in_pow = dev->power;
  ctx->in_depth = dev->depth;
  ctx->N = n;
  ctx->grid_valid = false;
  return FPPM_OK;
}

int fppm_gpu_generate_photons(fppm_gpu_ctx *ctx, int32_t workload, uint64_t seed, uint64_t iteration,
                              uint64_t begin, uint32_t n) {
  if (!ctx) return FPPM_ERR_INVALID_ARGUMENT;
  JOIN_RECS(ctx);
  if (workload != FPPM_WORKLOAD_C1 && workload != FPPM_WORKLOAD_C2 && workload != FPPM_WORKLOAD_C5)
    return fail(ctx, FPPM_ERR_INVALID_ARGUMENT, "unknown workload");
  if (workload == FPPM_WORKLOAD_C5 && !ctx->c5.pos) return fail(ctx, FPPM_ERR_STATE, "C5 photons before c5_setup");
  if (n > ctx->cfg.max_photons) return fail(ctx, FPPM_ERR_CAPACITY, "photons exceed max_photons");
  // a superseded upload into set 0 may still run on the copy stream: order
  // the generator after it (a no-op once the copy has finished)
  if (ctx->cstream) FPPM_CUDA_OK(cudaStreamWaitEvent(ctx->stream, ctx->ev_copied[0], 0));
  ctx->stage_pending = -1;
  ctx->pf_set = -1;  // set 0 is rewritten
  if (workload == FPPM_WORKLOAD_C5) {
    if (seed != ctx->c5.seed) return fail(ctx, FPPM_ERR_INVALID_ARGUMENT, "C5 seed differs from c5_setup");
    FPPM_CUDA_OK(launch_c5_photons(ctx->stream, ctx->c5, iteration, begin, n, ctx->d_ppos, ctx->d_pnrm, ctx->d_pwi,
                                   ctx->d_ppow, ctx->d_pdepth, ctx->sms));
  } else {
    launch_generate_photons(ctx->stream, workload, seed, iteration, begin, n, ctx->d_ppos, ctx->d_pnrm,
                            ctx->d_pwi, ctx->d_ppow, ctx->d_pdepth, ctx->sms);
  }
  FPPM_CUDA_OK(cudaGetLastError());
  ctx->N = n;
  ctx->grid_valid = false;
  use_staging(ctx);
  return FPPM_OK;
}

int fppm_gpu_generate_photons_to(fppm_gpu_ctx *ctx, int32_t workload, uint64_t seed,
                                 uint64_t iteration, uint64_t begin, uint32_t n,
                                 const fppm_photons *d) {
  if (!ctx || !d) return FPPM_ERR_INVALID_ARGUMENT;
  JOIN_RECS(ctx);
  if (workload != FPPM_WORKLOAD_C1 && workload != FPPM_WORKLOAD_C2 && workload != FPPM_WORKLOAD_C5)
    return fail(ctx, FPPM_ERR_INVALID_ARGUMENT, "unknown workload");
  if (n && (!d->pos || !d->normal || !d->wi || !d->power || !d->depth))
    return fail(ctx, FPPM_ERR_INVALID_ARGUMENT, "null photon array");
  if (workload == FPPM_WORKLOAD_C5) {
    if (!ctx->c5.pos) return fail(ctx, FPPM_ERR_STATE, "C5 photons before c5_setup");
    if (seed != ctx->c5.seed) return fail(ctx, FPPM_ERR_INVALID_ARGUMENT, "C5 seed differs from c5_setup");
    FPPM_CUDA_OK(launch_c5_photons(ctx->stream, ctx->c5, iteration, begin, n, const_cast<float *>(d->pos),
                                   const_cast<float *>(d->normal), const_cast<float *>(d->wi),
                                   const_cast<float *>(d->power), const_cast<uint32_t *>(d->depth), ctx->sms));
    return FPPM_OK;
  }
  launch_generate_photons(ctx->stream, workload, seed, iteration, begin, n,
                          const_cast<float *>(d->pos), const_cast<float *>(d->normal),
                          const_cast<float *>(d->wi), const_cast<float *>(d->power),
                          const_cast<uint32_t *>(d->depth), ctx->sms);
  FPPM_CUDA_OK(cudaGetLastError());
  return FPPM_OK;
}

int fppm_gpu_get_photons(fppm_gpu_ctx *ctx, float *pos, float *normal, float *wi, float *power,
                         uint32_t *depth) {
  if (!ctx) return FPPM_ERR_INVALID_ARGUMENT;
  JOIN_RECS(ctx);
  if (!ctx->in_pos) use_staging(ctx);
  if (ctx->stage_pending >= 0)
    FPPM_CUDA_OK(cudaStreamWaitEvent(ctx->stream, ctx->ev_copied[ctx->stage_pending], 0));
  const size_t b3 = sizeof(float) * 3 * ctx->N;
  int rc;
  if ((rc = copy_out(ctx, pos, ctx->in_pos, b3))) return rc;
  if ((rc = copy_out(ctx, normal, ctx->in_nrm, b3))) return rc;
  if ((rc = copy_out(ctx, wi, ctx->in_wi, b3))) return rc;
  if ((rc = copy_out(ctx, power, ctx->in_pow, b3))) return rc;
  if ((rc = copy_out(ctx, depth, ctx->in_depth, sizeof(uint32_t) * ctx->N))) return rc;
  FPPM_CUDA_OK(cudaStreamSynchronize(ctx->stream));
  return FPPM_OK;
}


// S_req > 1 asks for the fine (slab) table when the photon set allows it.
static int build_grid_impl(fppm_gpu_ctx *ctx, double cell_size, uint32_t S_req, const double *d_cell_in = nullptr) {
  if (!ctx) return FPPM_ERR_INVALID_ARGUMENT;
  JOIN_RECS(ctx);
  cudaStream_t s = ctx->stream;
  ctx->grid_valid = false;
  ctx->grid_explicit = cell_size > 0.0 || d_cell_in != nullptr;
  ctx->rcheck = ctx->grid_explicit;
  if (d_cell_in) {
    FPPM_CUDA_OK(cudaMemcpyAsync(ctx->d_cell, d_cell_in, sizeof(double), cudaMemcpyDeviceToDevice, s));
  } else if (cell_size > 0.0) {
    *ctx->h_cell = cell_size;
    FPPM_CUDA_OK(cudaMemcpyAsync(ctx->d_cell, ctx->h_cell, sizeof(double), cudaMemcpyHostToDevice, s));
  } else {
    int rc = device_max_radius(ctx, ctx->d_cell);  // integrator.cpp:159-161
    if (rc) return rc;
  }
  FPPM_CUDA_OK(cudaMemcpyAsync(ctx->d_bounds, ctx->h_bounds_init, sizeof(long long) * 8,
                               cudaMemcpyHostToDevice, s));
  if (!ctx->in_pos) use_staging(ctx);
  const int reading = ctx->stage_pending >= 0 ? ctx->stage_pending : -1;
  if (reading >= 0) {
    FPPM_CUDA_OK(cudaStreamWaitEvent(s, ctx->ev_copied[reading], 0));
    ctx->stage_pending = -1;
  }
  launch_cell_bounds(s, ctx->in_pos, ctx->N, ctx->d_cell, S_req, ctx->d_bounds, ctx->sms);
  launch_grid_header(s, ctx->d_bounds, ctx->d_cell, ctx->N, ctx->cfg.max_cells, S_req,
                     S_req > 1 ? ctx->d_lean_ok : nullptr, flat_records_enabled(), ctx->d_hdr);
  FPPM_CUDA_OK(cudaGetLastError());
  FPPM_CUDA_OK(cudaMemcpyAsync(ctx->h_hdr, ctx->d_hdr, sizeof(GridHeader), cudaMemcpyDeviceToHost, s));
  if (!ctx->ev_hdr) FPPM_CUDA_OK(cudaEventCreateWithFlags(&ctx->ev_hdr, cudaEventDisableTiming));
  FPPM_CUDA_OK(cudaEventRecord(ctx->ev_hdr, s));
  // Kernels that need only the device-side header are queued before the host
  // waits for its copy, so the device stays busy over the round trip: the
  // dense keys, and the record pack when the last build forked it (the
  // layout decision repeats from build to build).
  const bool spec = ctx->last_fork && ctx->recs.pack != nullptr && ctx->N > 0;
  if (spec) {
    if (!ctx->gstream) {
      FPPM_CUDA_OK(cudaStreamCreateWithFlags(&ctx->gstream, cudaStreamNonBlocking));
      FPPM_CUDA_OK(cudaEventCreateWithFlags(&ctx->ev_g_hdr, cudaEventDisableTiming));
      FPPM_CUDA_OK(cudaEventCreateWithFlags(&ctx->ev_g_sorted, cudaEventDisableTiming));
      FPPM_CUDA_OK(cudaEventCreateWithFlags(&ctx->ev_g_recs, cudaEventDisableTiming));
    }
    FPPM_CUDA_OK(cudaEventRecord(ctx->ev_g_hdr, s));
    FPPM_CUDA_OK(cudaStreamWaitEvent(ctx->gstream, ctx->ev_g_hdr, 0));
    launch_pack_fine(ctx->gstream, ctx->in_pos, ctx->in_nrm, ctx->in_wi, ctx->in_pow, ctx->in_depth, ctx->N,
                     ctx->d_hdr, ctx->cfg.normal_guard_cos, ctx->recs.pack, ctx->sms);
  }
  launch_dense_keys(s, ctx->in_pos, ctx->N, ctx->d_hdr, ctx->sort.keys_a, ctx->sort.vals_a, ctx->sms);
  FPPM_CUDA_OK(cudaEventSynchronize(ctx->ev_hdr));
  const GridHeader g = *ctx->h_hdr;
  if (!(g.cell > 0.0)) return fail(ctx, FPPM_ERR_INVALID_ARGUMENT, "PhotonGrid: cell size must be positive");
  if (!g.ok) return fail(ctx, FPPM_ERR_CAPACITY, "grid bounding box exceeds max_cells dense cells");
  if (g.ncells + 1 > ctx->cell_cap) {
    if (ctx->d_cell_start) cudaFree(ctx->d_cell_start);
    ctx->d_cell_start = nullptr;
    ctx->cell_cap = 0;
    const unsigned long long cap = std::max<unsigned long long>(2 * (g.ncells + 1), 1024);
    FPPM_CUDA_OK(cudaMalloc(&ctx->d_cell_start, sizeof(uint32_t) * cap));
    ctx->cell_cap = cap;
  }
  const bool fine_layout = effective_variant(ctx, g.S) == 4;
  // the fine layout's 48/64-B records (pack: needs only the header; permute:
  // needs the sort) are built on gstream, overlapping the key sort here and
  // the gather's scheduling kernels; the next consumer joins (join_recs)
  const bool fork = fine_layout && ctx->recs.pack != nullptr && ctx->N > 0;
  ctx->last_fork = fork;
  if (fork && !ctx->gstream) {
    FPPM_CUDA_OK(cudaStreamCreateWithFlags(&ctx->gstream, cudaStreamNonBlocking));
    FPPM_CUDA_OK(cudaEventCreateWithFlags(&ctx->ev_g_hdr, cudaEventDisableTiming));
    FPPM_CUDA_OK(cudaEventCreateWithFlags(&ctx->ev_g_sorted, cudaEventDisableTiming));
    FPPM_CUDA_OK(cudaEventCreateWithFlags(&ctx->ev_g_recs, cudaEventDisableTiming));
  }
  cudaStream_t rs = fork ? ctx->gstream : s;
  if (fork && !spec) {
    FPPM_CUDA_OK(cudaEventRecord(ctx->ev_g_hdr, s));
    FPPM_CUDA_OK(cudaStreamWaitEvent(rs, ctx->ev_g_hdr, 0));
    launch_pack_fine(rs, ctx->in_pos, ctx->in_nrm, ctx->in_wi, ctx->in_pow, ctx->in_depth, ctx->N, ctx->d_hdr,
                     ctx->cfg.normal_guard_cos, ctx->recs.pack, ctx->sms);
  } else if (spec && !fork) {
    // a speculative pack that this layout does not use: nothing else may
    // write the pack buffer before it has finished
    FPPM_CUDA_OK(cudaEventRecord(ctx->ev_g_recs, ctx->gstream));
    FPPM_CUDA_OK(cudaStreamWaitEvent(s, ctx->ev_g_recs, 0));
  }
  FPPM_CUDA_OK(radix_sort_pairs(s, ctx->sort, ctx->N, g.key_bits, &ctx->d_skeys, &ctx->d_order));
  if (fork) {
    FPPM_CUDA_OK(cudaEventRecord(ctx->ev_g_sorted, s));
    FPPM_CUDA_OK(cudaStreamWaitEvent(rs, ctx->ev_g_sorted, 0));
  }
  launch_cell_start(s, ctx->d_skeys, ctx->N, ctx->d_hdr, ctx->d_cell_start, g.ncells, ctx->sms);
  launch_permute(rs, ctx->d_order, ctx->N, ctx->in_pos, ctx->in_nrm, ctx->in_wi, ctx->in_pow,
                 ctx->in_depth, ctx->recs, fine_layout, ctx->d_hdr, ctx->sms);
  if (ctx->cfg.vcm_plus)
    launch_permute_f64x3(s, ctx->d_order, ctx->N, ctx->d_pmis_in[0], ctx->d_pmis_in[1], ctx->d_pmis_in[2],
                         ctx->d_pmis[0], ctx->d_pmis[1], ctx->d_pmis[2], ctx->sms);
  FPPM_CUDA_OK(cudaGetLastError());
  ctx->grid_set = -1;
  if (ctx->cstream && ctx->in_pos == (ctx->stage_cur ? ctx->d_ppos2 : ctx->d_ppos)) {
    // the staging set is consumed: a later upload may overwrite it -- after
    // the gather when the lean layout's exact path may still read it (the
    // stale event of an earlier iteration must not release it before that)
    if (fine_layout && (g.lean || lean_config(ctx))) {
      ctx->grid_set = ctx->stage_cur;
      ctx->free_recorded[ctx->stage_cur] = false;
    } else {
      FPPM_CUDA_OK(cudaEventRecord(ctx->ev_free[ctx->stage_cur], rs));  // after pack, dense_keys and the sort
      ctx->free_recorded[ctx->stage_cur] = true;
    }
  }
  if (fork) {
    FPPM_CUDA_OK(cudaEventRecord(ctx->ev_g_recs, rs));
    ctx->recs_pending = true;
  }
  ctx->grid_valid = true;
  return FPPM_OK;
}

// The fine gather uses the fine (slab) table; query_ball / export_grid switch
// back to reference cells on demand (ensure_reference_cells).
static uint32_t requested_S(const fppm_gpu_ctx *ctx) {
  const int v = gather_variant(ctx);
  uint32_t s3 = 2u;
  if (const char *e = std::getenv("FPPM_3D_S")) s3 = (uint32_t)std::atoi(e) == 1 ? 1u : 2u;  // measurement knob
  return v == 4 ? kFineS : (v == 5 ? s3 : 1u);
}

int fppm_gpu_build_grid_device(fppm_gpu_ctx *ctx, const double *d_cell) {
  if (!ctx || !d_cell) return FPPM_ERR_INVALID_ARGUMENT;
  return build_grid_impl(ctx, 0.0, requested_S(ctx), d_cell);
}

int fppm_gpu_build_grid(fppm_gpu_ctx *ctx, double cell_size) {
  if (!ctx) return FPPM_ERR_INVALID_ARGUMENT;
  // the fine kernel asks for slab fine cells (falling back to 3D fine cells
  // S = 2 or reference cells), the 3D kernel for S = 2 where the table fits
  const int v = gather_variant(ctx);
  (void)v;
  return build_grid_impl(ctx, cell_size, requested_S(ctx));
}

// query_ball / export need the reference-cell table
static int ensure_reference_cells(fppm_gpu_ctx *ctx) {
  if (!ctx->grid_valid || ctx->h_hdr->S == 1) return FPPM_OK;
  return build_grid_impl(ctx, ctx->h_hdr->cell, 1);
}

int fppm_gpu_export_grid(fppm_gpu_ctx *ctx, uint64_t *keys, uint32_t *begin, uint32_t *end,
                         uint32_t *order, uint64_t *ncells) {
  if (!ctx) return FPPM_ERR_INVALID_ARGUMENT;
  JOIN_RECS(ctx);
  if (!ctx->grid_valid) return fail(ctx, FPPM_ERR_STATE, "grid not built");
  if (int rc = ensure_reference_cells(ctx)) return rc;
  const uint32_t n = ctx->N;
  std::vector<uint32_t> sk(n), ord(n);
  if (n) {
    FPPM_CUDA_OK(cudaMemcpyAsync(sk.data(), ctx->d_skeys, 4ull * n, cudaMemcpyDeviceToHost, ctx->stream));
    FPPM_CUDA_OK(cudaMemcpyAsync(ord.data(), ctx->d_order, 4ull * n, cudaMemcpyDeviceToHost, ctx->stream));
  }
  FPPM_CUDA_OK(cudaStreamSynchronize(ctx->stream));
  const GridHeader g = *ctx->h_hdr;
  uint64_t nc = 0;
  const uint64_t bias = 1ull << 20;  // photon_map.cpp:11
  for (uint32_t i = 0; i < n; ++i) {
    if (i == 0 || sk[i] != sk[i - 1]) {
      const unsigned long long k = sk[i];
      const long long X = (long long)(k / ((unsigned long long)g.ny * g.nz));
      const long long Y = (long long)((k / (unsigned long long)g.nz) % (unsigned long long)g.ny);
      const long long Z = (long long)(k % (unsigned long long)g.nz);
      const uint64_t ix = (uint64_t)(X + g.ix0), iy = (uint64_t)(Y + g.iy0), iz = (uint64_t)(Z + g.iz0);
      if (keys) keys[nc] = ((ix + bias) << 42) | ((iy + bias) << 21) | (iz + bias);
      if (begin) begin[nc] = i;
      ++nc;
    }
    if (end) end[nc - 1] = i + 1;
  }
  if (order && n) std::memcpy(order, ord.data(), 4ull * n);
  if (ncells) *ncells = nc;
  return FPPM_OK;
}

int fppm_gpu_query_ball(fppm_gpu_ctx *ctx, const double *centers, const double *radii, uint32_t nq,
                        uint64_t *offsets, uint32_t *indices, uint64_t cap, uint64_t *total) {
  if (!ctx || (nq && (!centers || !radii || !offsets))) return FPPM_ERR_INVALID_ARGUMENT;
  JOIN_RECS(ctx);
  if (!ctx->grid_valid) return fail(ctx, FPPM_ERR_STATE, "grid not built");
  if (int rc = ensure_reference_cells(ctx)) return rc;
  const GridHeader g = *ctx->h_hdr;
  if (ctx->N > 0)
    for (uint32_t q = 0; q < nq; ++q)
      if (radii[q] > g.cell)  // photon_map.cpp:57-58
        return fail(ctx, FPPM_ERR_INVALID_ARGUMENT, "PhotonGrid: query radius exceeds cell size");
  const size_t need = sizeof(double) * 4 * nq + sizeof(unsigned long long) * 2 * (nq + 1) +
                      sizeof(uint32_t) * (cap + 1) + 256;
  FPPM_CUDA_OK(ensure_scratch(ctx, need));
  char *p = static_cast<char *>(ctx->d_scratch);
  double *d_c = reinterpret_cast<double *>(p);
  double *d_r = d_c + 3 * (size_t)nq;
  unsigned long long *d_cnt = reinterpret_cast<unsigned long long *>(d_r + nq);
  unsigned long long *d_off = d_cnt + nq + 1;
  uint32_t *d_out = reinterpret_cast<uint32_t *>(d_off + nq + 1);
  cudaStream_t s = ctx->stream;
  if (nq) {
    FPPM_CUDA_OK(cudaMemcpyAsync(d_c, centers, sizeof(double) * 3 * nq, cudaMemcpyHostToDevice, s));
    FPPM_CUDA_OK(cudaMemcpyAsync(d_r, radii, sizeof(double) * nq, cudaMemcpyHostToDevice, s));
  }
  launch_query_ball(s, d_c, d_r, nq, ctx->d_hdr, ctx->d_cell_start, ctx->recs.rec0, ctx->d_order,
                    d_cnt, nullptr, nullptr, 0);
  FPPM_CUDA_OK(cudaGetLastError());
  std::vector<unsigned long long> cnt(nq);
  if (nq) FPPM_CUDA_OK(cudaMemcpyAsync(cnt.data(), d_cnt, 8ull * nq, cudaMemcpyDeviceToHost, s));
  FPPM_CUDA_OK(cudaStreamSynchronize(s));
  uint64_t run = 0;
  for (uint32_t q = 0; q < nq; ++q) {
    offsets[q] = run;
    run += cnt[q];
  }
  offsets[nq] = run;
  if (total) *total = run;
  if (run <= cap && indices && run) {
    FPPM_CUDA_OK(cudaMemcpyAsync(d_off, offsets, 8ull * (nq + 1), cudaMemcpyHostToDevice, s));
    launch_query_ball(s, d_c, d_r, nq, ctx->d_hdr, ctx->d_cell_start, ctx->recs.rec0, ctx->d_order,
                      nullptr, d_off, d_out, 1);
    FPPM_CUDA_OK(cudaGetLastError());
    FPPM_CUDA_OK(cudaMemcpyAsync(indices, d_out, 4ull * run, cudaMemcpyDeviceToHost, s));
    FPPM_CUDA_OK(cudaStreamSynchronize(s));
  } else if (run > cap && indices) {
    return fail(ctx, FPPM_ERR_CAPACITY, "query result exceeds cap");
  }
  return FPPM_OK;
}

// ------------------------------------------------------------------ hot path
static int ensure_snapshots(fppm_gpu_ctx *ctx) {
  if (ctx->snap_cnt) return FPPM_OK;
  const size_t n = (size_t)std::max<uint32_t>(ctx->cfg.max_hitpoints, 1) * ctx->G * ctx->C;
  FPPM_CUDA_OK(dalloc(&ctx->snap_cnt, n));
  FPPM_CUDA_OK(dalloc(&ctx->snap_sum, n));
  FPPM_CUDA_OK(dalloc(&ctx->snap_sq, n));
  return FPPM_OK;
}

static int fill_summary(fppm_gpu_ctx *ctx, fppm_gpu_summary *sm) {
  cudaStream_t s = ctx->stream;
  FPPM_CUDA_OK(cudaMemcpyAsync(ctx->h_counters, ctx->d_counters, 32, cudaMemcpyDeviceToHost, s));
  FPPM_CUDA_OK(cudaMemcpyAsync(ctx->h_counters + 4, ctx->d_iter_tr, 8, cudaMemcpyDeviceToHost, s));
  FPPM_CUDA_OK(cudaMemcpyAsync(ctx->h_counters + 5, ctx->d_rmax_bits, 8, cudaMemcpyDeviceToHost, s));
  FPPM_CUDA_OK(cudaStreamSynchronize(s));
  const unsigned long long *c = ctx->h_counters;
  sm->accepted = c[0] - ctx->last_counters[0];
  sm->candidates = c[1] - ctx->last_counters[1];
  sm->exact_pairs = c[2] - ctx->last_counters[2];
  sm->ambiguous_pairs = c[3] - ctx->last_counters[3];
  for (int i = 0; i < 4; ++i) ctx->last_counters[i] = c[i];
  const unsigned int *tr = reinterpret_cast<const unsigned int *>(c + 4);
  sm->tested = tr[0];
  sm->rejected = tr[1];
  double rmax;
  std::memcpy(&rmax, c + 5, 8);
  sm->r_max_next = rmax;
  sm->cell_size = ctx->h_hdr->cell;
  sm->cells = ctx->h_hdr->ncells;
  return FPPM_OK;
}

// Bracket the dominant gather kernel with events (timed on its own stream).
static int kernel_event(fppm_gpu_ctx *ctx, int which) {
  const uint32_t slot = ctx->ev_head % fppm_gpu_ctx::kEvRing;
  cudaEvent_t &e = ctx->ev_k[slot][which];
  if (!e) FPPM_CUDA_OK(cudaEventCreate(&e));
  FPPM_CUDA_OK(cudaEventRecord(e, ctx->stream));
  if (which == 1) {
    ctx->ev_head++;
    if (ctx->ev_count < (uint32_t)fppm_gpu_ctx::kEvRing) ctx->ev_count++;
  }
  return FPPM_OK;
}

int fppm_gpu_record_bytes(const fppm_gpu_ctx *ctx) {
  if (!ctx || !ctx->grid_valid || !ctx->h_hdr) return 0;
  if (effective_variant(ctx, ctx->h_hdr->S) != 4) return 0;
  return ctx->h_hdr->lean == 2u ? 32 : ctx->h_hdr->lean == 1u ? 48 : 64;
}

int fppm_gpu_gather_kernel_ms(fppm_gpu_ctx *ctx, float *out, uint32_t max, uint32_t *n) {
  if (!ctx || (max && !out)) return FPPM_ERR_INVALID_ARGUMENT;
  const uint32_t cnt = std::min(ctx->ev_count, max);
  for (uint32_t i = 0; i < cnt; ++i) {
    const uint32_t slot =
        (ctx->ev_head + fppm_gpu_ctx::kEvRing - ctx->ev_count + i) % fppm_gpu_ctx::kEvRing;
    FPPM_CUDA_OK(cudaEventSynchronize(ctx->ev_k[slot][1]));
    FPPM_CUDA_OK(cudaEventElapsedTime(&out[i], ctx->ev_k[slot][0], ctx->ev_k[slot][1]));
  }
  if (n) *n = cnt;
  ctx->ev_count = 0;
  return FPPM_OK;
}

static void fill_gather_args(fppm_gpu_ctx *ctx, uint64_t iteration, GatherArgs &A) {
  std::memset(&A, 0, sizeof(A));
  A.pos = ctx->d_pos; A.nrm = ctx->d_nrm; A.K = ctx->d_K;
  A.eye_depth = ctx->d_eye; A.gathered = ctx->d_gathered;
  A.radius = ctx->d_radius; A.t = ctx->d_t;
  A.st_cnt = ctx->d_st_cnt; A.st_sum = ctx->d_st_sum; A.st_sq = ctx->d_st_sq;
  A.H = ctx->H;
  A.rec0 = ctx->recs.rec0; A.rec1 = ctx->recs.rec1; A.rec2 = ctx->recs.rec2; A.rec3 = ctx->recs.rec3;
  A.cell_start = ctx->d_cell_start; A.grid = ctx->d_hdr;
  A.order = ctx->d_order;
  A.in_pos = ctx->in_pos; A.in_nrm = ctx->in_nrm; A.in_wi = ctx->in_wi; A.in_pow = ctx->in_pow;
  A.in_depth = ctx->in_depth;
  A.na = ctx->cfg.n_annuli; A.ns = ctx->cfg.n_sectors;
  A.max_depth = ctx->cfg.max_depth; A.guard = ctx->cfg.normal_guard_cos;
  A.end = end_params(ctx, iteration);
  A.o_gather_r = ctx->o_gather_r; A.o_stat = ctx->o_stat; A.o_crit = ctx->o_crit;
  A.o_flux = ctx->o_flux; A.o_flags = ctx->o_flags; A.o_radiance = ctx->o_rad;
  A.o_accepted = ctx->o_acc;
  A.vcm = ctx->cfg.vcm_plus;
  A.mis_n_vm = ctx->cfg.mis_n_vm;
  A.mis_beta = ctx->cfg.mis_beta;
  A.eye_mis = ctx->d_eye_mis;
  A.p_vcm = ctx->d_pmis[0]; A.p_vm = ctx->d_pmis[1]; A.p_cont = ctx->d_pmis[2];
  A.wo = ctx->d_wo; A.alb = ctx->d_alb;
  A.counters = ctx->d_counters; A.iter_tr = ctx->d_iter_tr; A.work = ctx->d_work;
  A.rmax_bits = ctx->d_rmax_bits;
}

static int gather_impl(fppm_gpu_ctx *ctx, uint64_t iteration, fppm_gpu_iter_out *out,
                       fppm_gpu_summary *summary, double *delta);

int fppm_gpu_gather_test(fppm_gpu_ctx *ctx, uint64_t iteration, fppm_gpu_iter_out *out,
                         fppm_gpu_summary *summary) {
  return gather_impl(ctx, iteration, out, summary, nullptr);
}

uint32_t fppm_gpu_delta_stride(const fppm_gpu_ctx *ctx) {
  return ctx ? (uint32_t)(ctx->G + 2 * ctx->G * ctx->C + 3) : 0u;
}

int fppm_gpu_gather_deltas(fppm_gpu_ctx *ctx, uint64_t iteration, double *d_rows) {
  if (!ctx || (!d_rows && ctx->H)) return FPPM_ERR_INVALID_ARGUMENT;
  return gather_impl(ctx, iteration, nullptr, nullptr, d_rows);
}

int fppm_gpu_apply_deltas(fppm_gpu_ctx *ctx, uint64_t iteration, uint32_t h0, uint32_t n,
                          const double *d_rows, fppm_gpu_iter_out *out, fppm_gpu_summary *summary) {
  if (!ctx || (n && !d_rows)) return FPPM_ERR_INVALID_ARGUMENT;
  JOIN_RECS(ctx);
  if ((uint64_t)h0 + n > ctx->H) return fail(ctx, FPPM_ERR_INVALID_ARGUMENT, "apply range exceeds hit points");
  int rc = ensure_crit(ctx, ctx->end_calls + 2);
  if (rc) return rc;
  const bool snap = out && (out->stat_count || out->stat_sum || out->stat_sum_sq);
  if (snap && (rc = ensure_snapshots(ctx))) return rc;
  cudaStream_t s = ctx->stream;
  FPPM_CUDA_OK(cudaMemsetAsync(ctx->d_iter_tr, 0, 2 * sizeof(unsigned int), s));
  FPPM_CUDA_OK(cudaMemsetAsync(ctx->d_rmax_bits, 0, sizeof(unsigned long long), s));
  GatherArgs A;
  fill_gather_args(ctx, iteration, A);
  if (snap) { A.snap_cnt = ctx->snap_cnt; A.snap_sum = ctx->snap_sum; A.snap_sq = ctx->snap_sq; }
  FPPM_CUDA_OK(launch_apply_deltas(s, A, ctx->C, h0, n, d_rows));
  ctx->end_calls++;
  if (out && (rc = copy_iter_out(ctx, out, true, h0, n))) return rc;
  if (summary && (rc = fill_summary(ctx, summary))) return rc;
  return FPPM_OK;
}

static int gather_impl(fppm_gpu_ctx *ctx, uint64_t iteration, fppm_gpu_iter_out *out,
                       fppm_gpu_summary *summary, double *delta) {
  if (!ctx) return FPPM_ERR_INVALID_ARGUMENT;
  if (!ctx->grid_valid) return fail(ctx, FPPM_ERR_STATE, "gather before build_grid");
  if (ctx->rcheck && ctx->N > 0) {
    // photon_map.cpp:57-58: every gathered region's radius must fit the cell
    int rc0 = device_max_radius(ctx, ctx->d_cell_chk, ctx->d_gathered);
    if (rc0) return rc0;
    FPPM_CUDA_OK(cudaMemcpyAsync(ctx->h_cell, ctx->d_cell_chk, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    FPPM_CUDA_OK(cudaStreamSynchronize(ctx->stream));
    if (*ctx->h_cell > ctx->h_hdr->cell)
      return fail(ctx, FPPM_ERR_INVALID_ARGUMENT, "PhotonGrid: query radius exceeds cell size");
    ctx->rcheck = false;
  }
  const bool dbg = std::getenv("FPPM_DEBUG") != nullptr;
  auto now = [] { return std::chrono::steady_clock::now(); };
  auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
  const auto t0 = now();
  int rc = ensure_crit(ctx, ctx->end_calls + 2);
  if (rc) return rc;
  const auto t1 = now();
  const bool snap = out && (out->stat_count || out->stat_sum || out->stat_sum_sq);
  if (snap && (rc = ensure_snapshots(ctx))) return rc;
  cudaStream_t s = ctx->stream;
  FPPM_CUDA_OK(cudaMemsetAsync(ctx->d_work, 0, sizeof(unsigned int), s));
  FPPM_CUDA_OK(cudaMemsetAsync(ctx->d_iter_tr, 0, 2 * sizeof(unsigned int), s));
  FPPM_CUDA_OK(cudaMemsetAsync(ctx->d_rmax_bits, 0, sizeof(unsigned long long), s));
  GatherArgs A;
  fill_gather_args(ctx, iteration, A);
  if (snap) { A.snap_cnt = ctx->snap_cnt; A.snap_sum = ctx->snap_sum; A.snap_sq = ctx->snap_sq; }
  A.delta_out = delta;
  // auto: the fine kernel on slab (planar) grids, the thread-per-hit-point
  // kernel on 3D grids (S = 1: a few hit points per cell)
  const int var = effective_variant(ctx, ctx->h_hdr->S);
  if (var != 4 || !ctx->H) JOIN_RECS(ctx);
  if (ctx->H && (var == 1 || var == 5)) {
    if (var == 1) {
      if ((rc = kernel_event(ctx, 0))) return rc;
      FPPM_CUDA_OK(launch_gather_test(s, A, ctx->C, ctx->sms));
      if ((rc = kernel_event(ctx, 1))) return rc;
    } else {
      double *rows = delta;
      if (!rows) {
        const size_t need = (size_t)ctx->H * fppm_gpu_delta_stride(ctx);
        if (need > ctx->rows_cap) {
          if (ctx->d_rows) cudaFree(ctx->d_rows);
          ctx->d_rows = nullptr;
          ctx->rows_cap = 0;
          FPPM_CUDA_OK(dalloc(&ctx->d_rows, need));
          ctx->rows_cap = need;
        }
        rows = ctx->d_rows;
      }
      const uint32_t *order = nullptr;
      FPPM_CUDA_OK(hp_cell_order(s, A, ctx->tile, *ctx->h_hdr, ctx->sms, &order));
      if ((rc = kernel_event(ctx, 0))) return rc;
      void *hot3 = nullptr;
      if (dense_3d(*ctx->h_hdr) && (rc = ensure_hot3(ctx, ctx->H))) return rc;
      if (dense_3d(*ctx->h_hdr)) hot3 = ctx->hot3;
      FPPM_CUDA_OK(launch_gather_sparse(s, A, ctx->C, order, rows, ctx->sms, hot3, ctx->hot3_hits));
      if ((rc = kernel_event(ctx, 1))) return rc;
      if (!delta) {
        GatherArgs B = A;
        B.delta_out = nullptr;
        FPPM_CUDA_OK(launch_apply_deltas(s, B, ctx->C, 0, ctx->H, rows));
      }
    }
  } else if (ctx->H) {
    // ---- tiled path: bin hit points by home cell, build items, run
    TileSched &S = ctx->tile;
    const GridHeader g = *ctx->h_hdr;
    const unsigned long long n_ext =
        (unsigned long long)(g.nx + 2) * (unsigned long long)(g.ny + 2) * (unsigned long long)(g.nz + 2);
    if (n_ext + 2 > S.bucket_cap) {
      FPPM_CUDA_OK(cudaStreamSynchronize(s));
      void *old[] = {S.hp_start, S.items, S.chunks, S.item_base, S.scan_tmp, S.pbase};
      for (void *p : old)
        if (p) cudaFree(p);
      const unsigned long long cap = std::max<unsigned long long>(2 * (n_ext + 2), 4096);
      FPPM_CUDA_OK(dalloc(&S.hp_start, cap + 1));
      FPPM_CUDA_OK(dalloc(&S.items, cap + 1));
      FPPM_CUDA_OK(dalloc(&S.chunks, cap + 1));
      FPPM_CUDA_OK(dalloc(&S.item_base, cap + 1));
      FPPM_CUDA_OK(dalloc(&S.pbase, cap + 1));
      FPPM_CUDA_OK(dalloc(&S.scan_tmp, cap / 4096 + 8));
      S.bucket_cap = cap;
      S.bins_valid = false;
    }
    uint32_t nb = 0;
    // the fine-cell tiled kernel (slab grids, G * C <= 24)
    uint32_t cap64 = 0, cap48 = 0, fsub = 0;
    fine_caps(ctx->G, ctx->C, (int)g.lean, &cap64, &cap48, &fsub);
    FPPM_CUDA_OK(cudaMemsetAsync(S.nonempty, 0, sizeof(uint32_t), s));
    FPPM_CUDA_OK(fine_schedule_bins(s, A, S, g, ctx->sms, cap64, cap48, fsub, &nb, ctx->hp_version));
    FPPM_CUDA_OK(cudaMemcpyAsync(ctx->h_total, S.item_base + nb, sizeof(uint32_t),
                                 cudaMemcpyDeviceToHost, s));
    FPPM_CUDA_OK(cudaMemcpyAsync(ctx->h_total + 1, S.pbase + nb, sizeof(uint32_t),
                                 cudaMemcpyDeviceToHost, s));
    // the item descriptors are built speculatively into the current
    // capacity (k_fine_desc / k_fine_order skip items past it) while the
    // host waits for the totals; rebuilt below if the capacity was short
    if (!ctx->ev_sched) FPPM_CUDA_OK(cudaEventCreateWithFlags(&ctx->ev_sched, cudaEventDisableTiming));
    FPPM_CUDA_OK(cudaEventRecord(ctx->ev_sched, s));
    const bool spec_items = S.fdesc != nullptr && S.item_cap > 0;
    if (spec_items) FPPM_CUDA_OK(fine_schedule_items(s, A, S, nb, ctx->sms, cap64, cap48, fsub));
    const auto t2 = now();
    FPPM_CUDA_OK(cudaEventSynchronize(ctx->ev_sched));
    const auto t3 = now();
    const uint32_t total = ctx->h_total[0];
    const bool items_fit = total <= S.item_cap;
    if (dbg)
      std::fprintf(stderr, "[fppm] iteration %llu items %u rows %u (caps %llu %llu) crit %.3f sched-issue %.3f sync %.3f ms\n",
                   (unsigned long long)iteration, total, ctx->h_total[1], S.item_cap, S.row_cap, ms(t0, t1),
                   ms(t1, t2), ms(t2, t3));
    // partial rows: one per (hit point, item)
    const unsigned long long rows = (unsigned long long)ctx->h_total[1];
    if (total > S.item_cap) {
      if (S.fdesc) cudaFree(S.fdesc);
      S.fdesc = nullptr;
      // generous growth: reallocation inside a timed loop costs milliseconds
      const unsigned long long cap =
          std::max<unsigned long long>(2ull * total, (unsigned long long)ctx->H / 8 + 4096);
      FPPM_CUDA_OK(dalloc(&S.fdesc, cap));
      S.item_cap = cap;
    }
    if (rows > S.row_cap) {
      if (S.partials) cudaFree(S.partials);
      S.partials = nullptr;
      const unsigned long long cap =
          std::max<unsigned long long>(2ull * rows, 4ull * ctx->H + 4096);
      FPPM_CUDA_OK(dalloc(&S.partials, cap * (tile_partial_doubles(ctx->G, ctx->C) / 32)));
      S.row_cap = cap;
    }
    TileArgs T;
    T.hp_order = S.hp_order;
    T.partials = S.partials;
    T.hp_map = S.hp_map;
    T.total_items = S.item_base + nb;
    T.contig = fsub == 1;
    {
      if (!spec_items || !items_fit) FPPM_CUDA_OK(fine_schedule_items(s, A, S, nb, ctx->sms, cap64, cap48, fsub));
      FineArgs F;
      F.desc = S.fdesc;
      F.hot = static_cast<const FineHot *>(S.fhot);
      F.hits = static_cast<const Hit *>(S.fhit);
      F.hp_order = S.hp_order;
      F.partials = S.partials;
      F.hp_map = S.hp_map;
      F.total_items = S.item_base + nb;
      T.desc = nullptr;
      JOIN_RECS(ctx);  // the records built on gstream
      if ((rc = kernel_event(ctx, 0))) return rc;
      FPPM_CUDA_OK(launch_gather_fine(s, A, F, ctx->C, ctx->sms, (int)g.lean));
      if ((rc = kernel_event(ctx, 1))) return rc;
    }
    FPPM_CUDA_OK(launch_tile_finalize(s, A, T, ctx->C, ctx->sms));
  }
  if (ctx->grid_set >= 0) {  // the exact path read the staged input photons
    FPPM_CUDA_OK(cudaEventRecord(ctx->ev_free[ctx->grid_set], s));
    ctx->free_recorded[ctx->grid_set] = true;
    ctx->grid_set = -1;
  }
  if (delta) return FPPM_OK;  // option B: pooled and tested by the owner (apply_deltas)
  ctx->end_calls++;
  if (out && (rc = copy_iter_out(ctx, out, true))) return rc;
  if (summary && (rc = fill_summary(ctx, summary))) return rc;
  return FPPM_OK;
}

int fppm_gpu_iterate(fppm_gpu_ctx *ctx, uint64_t iteration, fppm_gpu_iter_out *out,
                     fppm_gpu_summary *summary) {
  int rc = fppm_gpu_build_grid(ctx, 0.0);
  if (rc) return rc;
  return fppm_gpu_gather_test(ctx, iteration, out, summary);
}

int fppm_gpu_accumulate(fppm_gpu_ctx *ctx, const uint32_t *region, const double *y,
                        const double *value, uint32_t n) {
  if (!ctx || (n && (!region || !y || !value))) return FPPM_ERR_INVALID_ARGUMENT;
  JOIN_RECS(ctx);
  if (n == 0) return FPPM_OK;
  const size_t need = (4 + 16 + 24 + 4) * (size_t)n + 64;
  FPPM_CUDA_OK(ensure_scratch(ctx, need));
  char *p = static_cast<char *>(ctx->d_scratch);
  double2 *d_y = reinterpret_cast<double2 *>(p);
  double *d_v = reinterpret_cast<double *>(d_y + n);
  uint32_t *d_reg = reinterpret_cast<uint32_t *>(d_v + 3 * (size_t)n);
  int *d_sec = reinterpret_cast<int *>(d_reg + n);
  int *d_err = d_sec + n;
  cudaStream_t s = ctx->stream;
  FPPM_CUDA_OK(cudaMemcpyAsync(d_y, y, 16ull * n, cudaMemcpyHostToDevice, s));
  FPPM_CUDA_OK(cudaMemcpyAsync(d_v, value, 24ull * n, cudaMemcpyHostToDevice, s));
  FPPM_CUDA_OK(cudaMemcpyAsync(d_reg, region, 4ull * n, cudaMemcpyHostToDevice, s));
  FPPM_CUDA_OK(cudaMemsetAsync(d_err, 0, sizeof(int), s));
  FPPM_CUDA_OK(launch_samples(s, d_reg, d_y, d_v, n, ctx->d_radius, ctx->H, ctx->cfg.n_annuli,
                              ctx->cfg.n_sectors, ctx->C, d_sec, d_err, nullptr, nullptr, nullptr, 0));
  int herr = 0;
  FPPM_CUDA_OK(cudaMemcpyAsync(&herr, d_err, sizeof(int), cudaMemcpyDeviceToHost, s));
  FPPM_CUDA_OK(cudaStreamSynchronize(s));
  if (herr == FPPM_ERR_DOMAIN) return fail(ctx, FPPM_ERR_DOMAIN, "sector_index: point outside the kernel disk");
  if (herr) return fail(ctx, herr, "region index out of range");
  FPPM_CUDA_OK(launch_samples(s, d_reg, d_y, d_v, n, ctx->d_radius, ctx->H, ctx->cfg.n_annuli,
                              ctx->cfg.n_sectors, ctx->C, d_sec, d_err, ctx->d_st_cnt, ctx->d_st_sum,
                              ctx->d_st_sq, 1));
  FPPM_CUDA_OK(cudaStreamSynchronize(s));
  return FPPM_OK;
}

int fppm_gpu_set_samples_per_iteration(fppm_gpu_ctx *ctx, uint64_t samples_per_iteration) {
  if (!ctx) return FPPM_ERR_INVALID_ARGUMENT;
  JOIN_RECS(ctx);
  if (samples_per_iteration == ctx->cfg.samples_per_iteration) return FPPM_OK;
  ctx->cfg.samples_per_iteration = samples_per_iteration;
  ctx->crit.clear();  // F_c depends on m = t * J
  return ensure_crit(ctx, ctx->end_calls + 2);
}

int fppm_gpu_end_iteration(fppm_gpu_ctx *ctx, uint64_t iteration, fppm_gpu_iter_out *out) {
  if (!ctx) return FPPM_ERR_INVALID_ARGUMENT;
  JOIN_RECS(ctx);
  int rc = ensure_crit(ctx, ctx->end_calls + 2);
  if (rc) return rc;
  const bool snap = out && (out->stat_count || out->stat_sum || out->stat_sum_sq);
  if (snap && (rc = ensure_snapshots(ctx))) return rc;
  EndArgs A;
  std::memset(&A, 0, sizeof(A));
  A.radius = ctx->d_radius; A.t = ctx->d_t;
  A.st_cnt = ctx->d_st_cnt; A.st_sum = ctx->d_st_sum; A.st_sq = ctx->d_st_sq;
  A.H = ctx->H; A.G = ctx->G; A.C = ctx->C;
  A.end = end_params(ctx, iteration);
  A.o_gather_r = ctx->o_gather_r; A.o_stat = ctx->o_stat; A.o_crit = ctx->o_crit;
  A.o_flags = ctx->o_flags;
  if (snap) { A.snap_cnt = ctx->snap_cnt; A.snap_sum = ctx->snap_sum; A.snap_sq = ctx->snap_sq; }
  FPPM_CUDA_OK(launch_end_iteration(ctx->stream, A));
  ctx->end_calls++;
  if (out) return copy_iter_out(ctx, out, false);
  return FPPM_OK;
}

int fppm_gpu_set_policy(fppm_gpu_ctx *ctx, int32_t policy) {
  if (!ctx) return FPPM_ERR_INVALID_ARGUMENT;
  JOIN_RECS(ctx);
  if (policy < FPPM_POLICY_FTEST || policy > FPPM_POLICY_SCHEDULE)
    return fail(ctx, FPPM_ERR_INVALID_ARGUMENT, "unknown end-of-iteration policy");
  if (policy == ctx->cfg.policy) return FPPM_OK;
  if (policy == FPPM_POLICY_CHI2 && !(ctx->chi2_crit > 0.0)) {
    int st = 0;  // gather.cpp:117-118: solved once per region
    const double v = host_chi2_quantile(1.0 - ctx->cfg.alpha_chi2, (double)(ctx->G - 1), &st);
    if (st) return fail(ctx, FPPM_ERR_INVALID_ARGUMENT, "chi2_quantile: bad alpha_chi2");
    ctx->chi2_crit = v;
  }
  ctx->cfg.policy = policy;
  ctx->crit.clear();  // the F table is only kept for the F policy
  return ensure_crit(ctx, ctx->end_calls + 2);
}

int fppm_gpu_sector_index(double u, double v, double radius, int32_t n_annuli, int32_t n_sectors,
                          int32_t *index) {
  if (!index) return FPPM_ERR_INVALID_ARGUMENT;
  int st = 0;
  *index = fppm_b200::host_sector_index(u, v, radius, n_annuli, n_sectors, &st);
  return st == 1 ? FPPM_ERR_INVALID_ARGUMENT : st == 2 ? FPPM_ERR_DOMAIN : FPPM_OK;
}

int fppm_gpu_build_frame(const double n[3], double u[3], double v[3]) {
  if (!n || !u || !v) return FPPM_ERR_INVALID_ARGUMENT;
  fppm_b200::host_build_frame(n, u, v);
  return FPPM_OK;
}

uint64_t fppm_gpu_kernel_launches(void) { return g_kernel_launches.load(); }

int fppm_gpu_set_scene(fppm_gpu_ctx *ctx, const fppm_scene *sc) {
  if (!ctx || !sc) return FPPM_ERR_INVALID_ARGUMENT;
  JOIN_RECS(ctx);
  const uint32_t nm = sc->n_materials, np = sc->n_primitives, ne = sc->n_emitters;
  if ((nm && (!sc->material_kind || !sc->material_rgb || !sc->material_ior)) ||
      (np && (!sc->shape_kind || !sc->shape || !sc->shape_material)) ||
      (ne && (!sc->emitter_shape || !sc->emitter_radiance)))
    return fail(ctx, FPPM_ERR_INVALID_ARGUMENT, "null scene array");
  for (uint32_t i = 0; i < nm; ++i)
    if (sc->material_kind[i] < 0 || sc->material_kind[i] > 2)
      return fail(ctx, FPPM_ERR_INVALID_ARGUMENT, "unsupported material kind");
  if (np > (uint32_t)fppm_b200::trace_max_prims())
    return fail(ctx, FPPM_ERR_INVALID_ARGUMENT, "scene has more primitives than the tracer supports");
  for (uint32_t i = 0; i < np; ++i)
    if (sc->shape_kind[i] < 0 || sc->shape_kind[i] > 1 || sc->shape_material[i] < 0 ||
        (uint32_t)sc->shape_material[i] >= nm)
      return fail(ctx, FPPM_ERR_INVALID_ARGUMENT, "bad primitive");
  for (uint32_t i = 0; i < ne; ++i)
    if (sc->emitter_shape[i] < 0 || (uint32_t)sc->emitter_shape[i] >= np)
      return fail(ctx, FPPM_ERR_INVALID_ARGUMENT, "bad emitter primitive");
  int rc;
  if ((rc = upload(ctx, ctx->scene_mem[0], sc->material_kind, nm)) ||
      (rc = upload(ctx, ctx->scene_mem[1], sc->material_rgb, 3 * (size_t)nm)) ||
      (rc = upload(ctx, ctx->scene_mem[2], sc->material_ior, nm)) ||
      (rc = upload(ctx, ctx->scene_mem[3], sc->shape_kind, np)) ||
      (rc = upload(ctx, ctx->scene_mem[4], sc->shape, 9 * (size_t)np)) ||
      (rc = upload(ctx, ctx->scene_mem[5], sc->shape_material, np)) ||
      (rc = upload(ctx, ctx->scene_mem[6], sc->emitter_shape, ne)) ||
      (rc = upload(ctx, ctx->scene_mem[7], sc->emitter_radiance, 3 * (size_t)ne)))
    return rc;
  fppm_b200::TraceScene &t = ctx->scene;
  t.n_mat = (int)nm;
  t.n_prim = (int)np;
  t.n_emit = (int)ne;
  t.mat_kind = static_cast<const int *>(ctx->scene_mem[0]);
  t.mat_rgb = static_cast<const double *>(ctx->scene_mem[1]);
  t.mat_ior = static_cast<const double *>(ctx->scene_mem[2]);
  t.prim_kind = static_cast<const int *>(ctx->scene_mem[3]);
  t.prim = static_cast<const double *>(ctx->scene_mem[4]);
  t.prim_mat = static_cast<const int *>(ctx->scene_mem[5]);
  t.emit_prim = static_cast<const int *>(ctx->scene_mem[6]);
  t.emit_rad = static_cast<const double *>(ctx->scene_mem[7]);
  if (ctx->scene_mem[8]) cudaFree(ctx->scene_mem[8]);
  ctx->scene_mem[8] = nullptr;
  FPPM_CUDA_OK(cudaMalloc(&ctx->scene_mem[8], fppm_b200::trace_prep_bytes((int)np)));
  FPPM_CUDA_OK(fppm_b200::launch_scene_prep(ctx->stream, t, ctx->scene_mem[8]));
  FPPM_CUDA_OK(cudaStreamSynchronize(ctx->stream));
  ctx->has_scene = true;
  return FPPM_OK;
}

int fppm_gpu_trace_photons(fppm_gpu_ctx *ctx, uint64_t seed, uint64_t iteration, uint32_t n_paths,
                           uint32_t max_depth, double mis_radius, uint32_t *n_photons) {
  return fppm_gpu_trace_photons_range(ctx, seed, iteration, 0, n_paths, max_depth, mis_radius, n_photons);
}

int fppm_gpu_trace_photons_range(fppm_gpu_ctx *ctx, uint64_t seed, uint64_t iteration, uint32_t path0,
                                 uint32_t n_paths, uint32_t max_depth, double mis_radius, uint32_t *n_photons) {
  if (!ctx) return FPPM_ERR_INVALID_ARGUMENT;
  if ((uint64_t)path0 + n_paths > 0xffffffffull) return fail(ctx, FPPM_ERR_INVALID_ARGUMENT, "path range overflows");
  JOIN_RECS(ctx);
  if (!ctx->has_scene) return fail(ctx, FPPM_ERR_STATE, "trace_photons before set_scene");
  cudaStream_t s = ctx->stream;
  const uint32_t depth = max_depth > 0 ? max_depth - 1 : 0;  // light_phase: max_depth - 1
  const unsigned long long slots = (unsigned long long)n_paths * depth;
  if (slots > ctx->t_slot_cap) {
    void *tp[] = {ctx->t_pos, ctx->t_nrm, ctx->t_wi, ctx->t_pow, ctx->t_depth, ctx->t_mis};
    FPPM_CUDA_OK(cudaStreamSynchronize(s));
    for (void *p : tp)
      if (p) cudaFree(p);
    const unsigned long long cap = std::max<unsigned long long>(slots, 1024);
    FPPM_CUDA_OK(dalloc(&ctx->t_pos, 3 * cap)); FPPM_CUDA_OK(dalloc(&ctx->t_nrm, 3 * cap));
    FPPM_CUDA_OK(dalloc(&ctx->t_wi, 3 * cap)); FPPM_CUDA_OK(dalloc(&ctx->t_pow, 3 * cap));
    FPPM_CUDA_OK(dalloc(&ctx->t_depth, cap));
    ctx->t_mis = nullptr;
    if (ctx->cfg.vcm_plus) FPPM_CUDA_OK(dalloc(&ctx->t_mis, 3 * cap));
    ctx->t_slot_cap = cap;
  }
  if ((unsigned long long)n_paths + 1 > ctx->t_path_cap) {
    void *tp[] = {ctx->t_count, ctx->t_base, ctx->t_scan};
    FPPM_CUDA_OK(cudaStreamSynchronize(s));
    for (void *p : tp)
      if (p) cudaFree(p);
    const unsigned long long cap = std::max<unsigned long long>(2ull * (n_paths + 1), 4096);
    FPPM_CUDA_OK(dalloc(&ctx->t_count, cap));
    FPPM_CUDA_OK(dalloc(&ctx->t_base, cap));
    FPPM_CUDA_OK(dalloc(&ctx->t_scan, cap / 4096 + 8));
    ctx->t_path_cap = cap;
  }
  double eta = 0.0;
  if (ctx->cfg.vcm_plus) {
    double r = mis_radius;
    if (!(r > 0.0)) {
      int rc = fppm_gpu_max_radius(ctx, &r);
      if (rc) return rc;
    }
    eta = (double)ctx->cfg.mis_n_vm * 3.141592653589793 * r * r;  // integrator.cpp:171-174
  }
  fppm_b200::TraceArgs T;
  T.sc = ctx->scene;
  T.seed = seed;
  T.iteration = iteration;
  T.n_paths = n_paths;
  T.light_depth = depth;
  T.path0 = path0;
  T.n_vm = ctx->cfg.mis_n_vm;
  T.beta = ctx->cfg.mis_beta > 0.0 ? ctx->cfg.mis_beta : 1.0;
  T.eta_vm = eta;
  T.v_pos = ctx->t_pos; T.v_nrm = ctx->t_nrm; T.v_wi = ctx->t_wi; T.v_pow = ctx->t_pow;
  T.v_depth = ctx->t_depth;
  T.v_mis = ctx->cfg.vcm_plus ? ctx->t_mis : nullptr;
  T.count = ctx->t_count;
  T.b_pos = T.b_sn = T.b_wi = T.b_thr = T.b_mis = nullptr;
  T.b_mat = nullptr;
  ctx->last_eta_light = eta;
  if (ctx->bidir_trace) {
    if (slots > ctx->b_slot_cap) {
      void *bp[] = {ctx->b_pos, ctx->b_sn, ctx->b_wi, ctx->b_thr, ctx->b_mis, ctx->b_mat};
      FPPM_CUDA_OK(cudaStreamSynchronize(s));
      for (void *p : bp)
        if (p) cudaFree(p);
      const unsigned long long cap = std::max<unsigned long long>(slots, 1024);
      FPPM_CUDA_OK(dalloc(&ctx->b_pos, 3 * cap)); FPPM_CUDA_OK(dalloc(&ctx->b_sn, 3 * cap));
      FPPM_CUDA_OK(dalloc(&ctx->b_wi, 3 * cap)); FPPM_CUDA_OK(dalloc(&ctx->b_thr, 3 * cap));
      FPPM_CUDA_OK(dalloc(&ctx->b_mis, 3 * cap)); FPPM_CUDA_OK(dalloc(&ctx->b_mat, cap));
      ctx->b_slot_cap = cap;
    }
    T.b_pos = ctx->b_pos; T.b_sn = ctx->b_sn; T.b_wi = ctx->b_wi; T.b_thr = ctx->b_thr;
    T.b_mis = ctx->b_mis; T.b_mat = ctx->b_mat;
  }
  FPPM_CUDA_OK(cudaMemsetAsync(ctx->t_count + n_paths, 0, sizeof(uint32_t), s));
  if (!ctx->t_ctr) FPPM_CUDA_OK(dalloc(&ctx->t_ctr, 1));
  T.path_counter = ctx->t_ctr;
  FPPM_CUDA_OK(launch_trace(s, T, ctx->scene_mem[8], ctx->sms));
  FPPM_CUDA_OK(launch_exclusive_scan(s, ctx->t_count, n_paths + 1, ctx->t_scan, ctx->t_base));
  FPPM_CUDA_OK(cudaMemcpyAsync(ctx->h_total, ctx->t_base + n_paths, sizeof(uint32_t), cudaMemcpyDeviceToHost,
                               s));
  FPPM_CUDA_OK(cudaStreamSynchronize(s));
  const uint32_t total = ctx->h_total[0];
  if (total > ctx->cfg.max_photons)
    return fail(ctx, FPPM_ERR_CAPACITY, "traced deposits exceed max_photons");
  // the deposits become the staged photons (set 0) of the next grid build
  if (ctx->ev_copied[0])  // any earlier upload into set 0 (a superseded one too)
    FPPM_CUDA_OK(cudaStreamWaitEvent(s, ctx->ev_copied[0], 0));
  ctx->stage_pending = -1;
  ctx->pf_set = -1;  // set 0 is rewritten
  FPPM_CUDA_OK(launch_trace_compact(s, T, ctx->t_base, ctx->d_ppos, ctx->d_pnrm, ctx->d_pwi, ctx->d_ppow,
                                    ctx->d_pdepth, ctx->cfg.vcm_plus ? ctx->d_pmis_in[0] : nullptr,
                                    ctx->d_pmis_in[1], ctx->d_pmis_in[2], ctx->sms));
  ctx->N = total;
  ctx->grid_valid = false;
  use_staging(ctx);
  if (n_photons) *n_photons = total;
  return FPPM_OK;
}

// make_camera_frame (path.cpp:122-133) on the host: glibc tan, no FMA, as
// the reference build.
static void vnorm(double v[3]) {
  const double l = std::sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
  v[0] = v[0] / l;
  v[1] = v[1] / l;
  v[2] = v[2] / l;
}
static void vcross(const double a[3], const double b[3], double o[3]) {
  o[0] = a[1] * b[2] - a[2] * b[1];
  o[1] = a[2] * b[0] - a[0] * b[2];
  o[2] = a[0] * b[1] - a[1] * b[0];
}

int fppm_gpu_set_camera(fppm_gpu_ctx *ctx, const fppm_camera *c) {
  if (!ctx || !c) return FPPM_ERR_INVALID_ARGUMENT;
  JOIN_RECS(ctx);
  if (c->width < 1 || c->height < 1) return fail(ctx, FPPM_ERR_INVALID_ARGUMENT, "camera resolution must be >= 1");
  const uint64_t npix = (uint64_t)c->width * (uint64_t)c->height;
  if (npix > ctx->cfg.max_hitpoints) return fail(ctx, FPPM_ERR_CAPACITY, "camera pixels exceed max_hitpoints");
  CamD &k = ctx->cam;
  for (int i = 0; i < 3; ++i) {
    k.pos[i] = c->position[i];
    k.fwd[i] = c->look_at[i] - c->position[i];
  }
  vnorm(k.fwd);
  vcross(k.fwd, c->up, k.right);
  vnorm(k.right);
  vcross(k.right, k.fwd, k.up);
  k.width = c->width;
  k.height = c->height;
  const double half_fov = 0.5 * c->vfov_deg * 3.141592653589793 / 180.0;
  k.plane_dist = (c->height * 0.5) / std::tan(half_fov);
  if (!ctx->d_emit) {
    const size_t n = std::max<uint32_t>(ctx->cfg.max_hitpoints, 1);
    FPPM_CUDA_OK(dalloc(&ctx->d_emit, n));
    FPPM_CUDA_OK(dalloc(&ctx->d_film, n));
    FPPM_CUDA_OK(dalloc(&ctx->d_vcvm, n));
  }
  FPPM_CUDA_OK(cudaMemsetAsync(ctx->d_film, 0, sizeof(double3) * npix, ctx->stream));
  FPPM_CUDA_OK(cudaMemsetAsync(ctx->d_vcvm, 0, sizeof(double2) * npix, ctx->stream));
  ctx->film_iters = 0;
  ctx->has_camera = true;
  return FPPM_OK;
}

int fppm_gpu_trace_eye(fppm_gpu_ctx *ctx, uint64_t seed, uint64_t iteration) {
  if (!ctx) return FPPM_ERR_INVALID_ARGUMENT;
  JOIN_RECS(ctx);
  if (!ctx->has_scene || !ctx->has_camera) return fail(ctx, FPPM_ERR_STATE, "trace_eye needs set_scene and set_camera");
  EyeArgs E;
  E.sc = ctx->scene;
  E.cam = ctx->cam;
  E.seed = seed;
  E.iteration = iteration;
  E.max_depth = ctx->cfg.max_depth;
  E.npix = (uint32_t)((uint64_t)ctx->cam.width * ctx->cam.height);
  E.pos = ctx->d_pos; E.nrm = ctx->d_nrm; E.wo = ctx->d_wo; E.thr = ctx->d_thr; E.alb = ctx->d_alb;
  E.emitted = ctx->d_emit;
  E.eye_depth = ctx->d_eye;
  E.gathered = ctx->d_gathered;
  FPPM_CUDA_OK(launch_trace_eye(ctx->stream, E, ctx->scene_mem[8], ctx->sms));
  return finish_hitpoints(ctx, E.npix, true);
}


// ------------------------------------------------------------------ VCM+ render
// One Renderer::step for vcm_plus (integrator.cpp:150-228, 492-653): light
// sub-paths with fp64 light vertices and their camera splats, eye sub-paths
// (emitter hits, next-event estimation, connections to light sub-path
// px % J), the primary rough vertex of every pixel gathered + tested as its
// region, the other rough vertices gathered as merge queries, film.
int fppm_gpu_render_vcm(fppm_gpu_ctx *ctx, uint64_t seed, uint64_t iteration, uint32_t light_paths,
                        uint32_t max_depth, uint32_t *n_photons) {
  if (!ctx) return FPPM_ERR_INVALID_ARGUMENT;
  JOIN_RECS(ctx);
  if (!ctx->cfg.vcm_plus) return fail(ctx, FPPM_ERR_STATE, "render_vcm needs a vcm_plus context");
  if (!ctx->has_scene || !ctx->has_camera) return fail(ctx, FPPM_ERR_STATE, "render_vcm needs set_scene and set_camera");
  if (max_depth < 1 || max_depth > kMaxBidirDepth)
    return fail(ctx, FPPM_ERR_INVALID_ARGUMENT, "render_vcm: max_depth must be in [1, 16]");
  if (light_paths == 0) return fail(ctx, FPPM_ERR_INVALID_ARGUMENT, "render_vcm: light_paths must be >= 1");
  if ((uint64_t)light_paths != ctx->cfg.samples_per_iteration)
    return fail(ctx, FPPM_ERR_INVALID_ARGUMENT, "render_vcm: light_paths must equal samples_per_iteration (J)");
  if (max_depth != ctx->cfg.max_depth)
    return fail(ctx, FPPM_ERR_INVALID_ARGUMENT, "render_vcm: max_depth must equal the context's max_depth");
  cudaStream_t s = ctx->stream;
  const uint32_t npix = (uint32_t)((uint64_t)ctx->cam.width * ctx->cam.height);
  const uint32_t nq = max_depth > 1 ? max_depth - 1 : 1;
  const unsigned long long nqt = (unsigned long long)npix * nq;
  const uint32_t stride = (uint32_t)(ctx->G + 2 * ctx->G * ctx->C + 3);
  if (nqt > 0xffffffffull) return fail(ctx, FPPM_ERR_CAPACITY, "render_vcm: too many merge vertices");
  if (nqt > ctx->q_cap) {
    void *qp[] = {ctx->q_pos, ctx->q_nrm, ctx->q_wo, ctx->q_thr, ctx->q_alb, ctx->q_K, ctx->q_eye,
                  ctx->q_gathered, ctx->q_radius, ctx->q_mis, ctx->d_splat, ctx->q_sort.keys_a,
                  ctx->q_sort.vals_a, ctx->q_sort.keys_b, ctx->q_sort.vals_b, ctx->q_sort.hist};
    FPPM_CUDA_OK(cudaStreamSynchronize(s));
    for (void *p : qp)
      if (p) cudaFree(p);
    FPPM_CUDA_OK(dalloc(&ctx->q_pos, nqt)); FPPM_CUDA_OK(dalloc(&ctx->q_nrm, nqt));
    FPPM_CUDA_OK(dalloc(&ctx->q_wo, nqt)); FPPM_CUDA_OK(dalloc(&ctx->q_thr, nqt));
    FPPM_CUDA_OK(dalloc(&ctx->q_alb, nqt)); FPPM_CUDA_OK(dalloc(&ctx->q_K, nqt));
    FPPM_CUDA_OK(dalloc(&ctx->q_eye, nqt)); FPPM_CUDA_OK(dalloc(&ctx->q_gathered, nqt));
    FPPM_CUDA_OK(dalloc(&ctx->q_radius, nqt)); FPPM_CUDA_OK(dalloc(&ctx->q_mis, nqt));
    FPPM_CUDA_OK(dalloc(&ctx->d_splat, std::max<uint32_t>(npix, 1)));
    FPPM_CUDA_OK(dalloc(&ctx->q_sort.keys_a, nqt)); FPPM_CUDA_OK(dalloc(&ctx->q_sort.vals_a, nqt));
    FPPM_CUDA_OK(dalloc(&ctx->q_sort.keys_b, nqt)); FPPM_CUDA_OK(dalloc(&ctx->q_sort.vals_b, nqt));
    FPPM_CUDA_OK(dalloc(&ctx->q_sort.hist, radix_hist_entries((uint32_t)nqt)));
    ctx->q_cap = nqt;
  }
  const unsigned long long nvt = (unsigned long long)npix * max_depth;  // eye vertices
  if (nvt > ctx->v_cap) {
    FPPM_CUDA_OK(cudaStreamSynchronize(s));
    void *vp[] = {ctx->v_d, ctx->v_i, ctx->v_n, ctx->v_rng};
    for (void *p : vp)
      if (p) cudaFree(p);
    ctx->v_d = nullptr; ctx->v_i = nullptr; ctx->v_n = nullptr; ctx->v_rng = nullptr;
    ctx->v_cap = 0;
    FPPM_CUDA_OK(dalloc(&ctx->v_d, 16 * nvt));
    FPPM_CUDA_OK(dalloc(&ctx->v_i, nvt));
    FPPM_CUDA_OK(dalloc(&ctx->v_n, std::max<uint32_t>(npix, 1)));
    FPPM_CUDA_OK(dalloc(&ctx->v_rng, std::max<uint32_t>(npix, 1)));
    ctx->v_cap = nvt;
  }
  if (nqt * stride > ctx->q_rows_cap) {
    if (ctx->q_rows) cudaFree(ctx->q_rows);
    ctx->q_rows = nullptr;
    FPPM_CUDA_OK(dalloc(&ctx->q_rows, nqt * stride));
    ctx->q_rows_cap = nqt * stride;
  }
  // the pixels are the regions (integrator.cpp:136-137): fresh regions on a new frame size
  if (ctx->H != npix) {
    ctx->H = npix;
    if (int rc0 = fppm_gpu_reset_regions(ctx)) return rc0;
  }
  // light phase with fp64 light vertices (r_max of the live radii, integrator.cpp:159-175)
  ctx->bidir_trace = true;
  int rc = fppm_gpu_trace_photons(ctx, seed, iteration, light_paths, max_depth, 0.0, n_photons);
  ctx->bidir_trace = false;
  if (rc) return rc;
  BidirArgs B;
  std::memset(&B, 0, sizeof(B));
  B.sc = ctx->scene;
  B.cam = ctx->cam;
  B.seed = seed;
  B.iteration = iteration;
  B.max_depth = max_depth;
  B.npix = npix;
  B.n_paths = light_paths;
  B.light_depth = max_depth - 1;
  B.n_vm = ctx->cfg.mis_n_vm;
  B.beta = ctx->cfg.mis_beta > 0.0 ? ctx->cfg.mis_beta : 1.0;
  B.eta_light = ctx->last_eta_light;
  B.radius = ctx->d_radius;
  B.l_pos = ctx->b_pos; B.l_sn = ctx->b_sn; B.l_wi = ctx->b_wi; B.l_thr = ctx->b_thr; B.l_mis = ctx->b_mis;
  B.l_mat = ctx->b_mat; B.l_depth = ctx->t_depth; B.l_count = ctx->t_count;
  B.direct = ctx->d_emit;
  B.pos = ctx->d_pos; B.nrm = ctx->d_nrm; B.wo = ctx->d_wo; B.thr = ctx->d_thr; B.alb = ctx->d_alb;
  B.eye_depth = ctx->d_eye; B.gathered = ctx->d_gathered; B.eye_mis = ctx->d_eye_mis;
  B.q_pos = ctx->q_pos; B.q_nrm = ctx->q_nrm; B.q_wo = ctx->q_wo; B.q_thr = ctx->q_thr; B.q_alb = ctx->q_alb;
  B.q_eye = ctx->q_eye; B.q_gathered = ctx->q_gathered; B.q_radius = ctx->q_radius; B.q_mis = ctx->q_mis;
  B.splat = ctx->d_splat;
  B.vtx_d = ctx->v_d; B.vtx_i = ctx->v_i; B.vtx_n = ctx->v_n; B.vtx_rng = ctx->v_rng;
  if (light_paths > 0 && B.light_depth > 0) {
    FPPM_CUDA_OK(cudaMemsetAsync(ctx->d_splat, 0, sizeof(double3) * npix, s));
    FPPM_CUDA_OK(launch_light_splat(s, B, ctx->scene_mem[8], ctx->sms));
  } else {
    FPPM_CUDA_OK(cudaMemsetAsync(ctx->d_splat, 0, sizeof(double3) * npix, s));
    B.l_count = ctx->t_count;
  }
  FPPM_CUDA_OK(launch_eye_bidir(s, B, ctx->scene_mem[8], ctx->sms));
  if ((rc = finish_hitpoints(ctx, npix, true))) return rc;
  FPPM_CUDA_OK(launch_hit_weights(s, ctx->q_nrm, ctx->q_wo, ctx->q_thr, ctx->q_alb, (uint32_t)nqt, ctx->q_K));
  // primary vertices: grid (cell = r_max) + VCM+ gather / F-test of the regions
  if ((rc = fppm_gpu_iterate(ctx, iteration, nullptr, nullptr))) return rc;
  // secondary vertices: merge queries with the pixel's radius, delta rows
  GatherArgs Q;
  fill_gather_args(ctx, iteration, Q);
  Q.pos = ctx->q_pos; Q.nrm = ctx->q_nrm; Q.K = ctx->q_K; Q.eye_depth = ctx->q_eye; Q.gathered = ctx->q_gathered;
  Q.radius = ctx->q_radius; Q.wo = ctx->q_wo; Q.alb = ctx->q_alb; Q.eye_mis = ctx->q_mis;
  Q.H = (uint32_t)nqt;
  Q.delta_out = ctx->q_rows;
  Q.o_gather_r = Q.o_stat = Q.o_crit = Q.o_flux = nullptr;
  Q.o_flags = nullptr;
  Q.o_radiance = nullptr;
  Q.o_accepted = nullptr;
  FPPM_CUDA_OK(cudaMemsetAsync(ctx->d_work, 0, sizeof(unsigned int), s));  // both kernels claim by counter
  if (gather_variant(ctx) == 1) {
    FPPM_CUDA_OK(launch_gather_test(s, Q, ctx->C, ctx->sms));
  } else {  // 3D kernel, merge vertices visited in home-cell order (neighbours share records in L1/L2)
    TileSched qs;
    qs.sort = ctx->q_sort;
    const uint32_t *order = nullptr;
    FPPM_CUDA_OK(hp_cell_order(s, Q, qs, *ctx->h_hdr, ctx->sms, &order));
    void *hot3 = nullptr, *qhits = nullptr;
    if (dense_3d(*ctx->h_hdr) && (rc = ensure_hot3(ctx, (uint32_t)nqt))) return rc;
    if (dense_3d(*ctx->h_hdr)) {
      hot3 = ctx->hot3;
      qhits = ctx->hot3_hits;
    }
    FPPM_CUDA_OK(launch_gather_sparse(s, Q, ctx->C, order, ctx->q_rows, ctx->sms, hot3, qhits));
  }
  FPPM_CUDA_OK(launch_film_vcm(s, npix, nq, ctx->d_emit, ctx->d_gathered, ctx->o_flux, ctx->o_gather_r,
                               ctx->q_rows, stride, ctx->q_gathered, ctx->q_radius, ctx->d_splat,
                               (double)light_paths, ctx->d_film, ctx->sms, ctx->d_vcvm));
  ctx->film_iters++;
  return FPPM_OK;
}

int fppm_gpu_get_hitpoints(fppm_gpu_ctx *ctx, fppm_hitpoints *o, double *emitted) {
  if (!ctx) return FPPM_ERR_INVALID_ARGUMENT;
  JOIN_RECS(ctx);
  const size_t H = ctx->H, b3 = sizeof(double3) * H;
  int rc;
  if (o) {
    if ((rc = copy_out(ctx, const_cast<double *>(o->pos), ctx->d_pos, b3))) return rc;
    if ((rc = copy_out(ctx, const_cast<double *>(o->normal), ctx->d_nrm, b3))) return rc;
    if ((rc = copy_out(ctx, const_cast<double *>(o->wo), ctx->d_wo, b3))) return rc;
    if ((rc = copy_out(ctx, const_cast<double *>(o->throughput), ctx->d_thr, b3))) return rc;
    if ((rc = copy_out(ctx, const_cast<double *>(o->albedo), ctx->d_alb, b3))) return rc;
    if ((rc = copy_out(ctx, const_cast<uint32_t *>(o->eye_depth), ctx->d_eye, sizeof(uint32_t) * H))) return rc;
    if ((rc = copy_out(ctx, const_cast<uint8_t *>(o->gathered), ctx->d_gathered, H))) return rc;
  }
  if (emitted) {
    if (!ctx->d_emit) return fail(ctx, FPPM_ERR_STATE, "no eye pass yet");
    if ((rc = copy_out(ctx, emitted, ctx->d_emit, b3))) return rc;
  }
  FPPM_CUDA_OK(cudaStreamSynchronize(ctx->stream));
  return FPPM_OK;
}

int fppm_gpu_film_add(fppm_gpu_ctx *ctx) {
  if (!ctx) return FPPM_ERR_INVALID_ARGUMENT;
  JOIN_RECS(ctx);
  if (!ctx->has_camera) return fail(ctx, FPPM_ERR_STATE, "film_add before set_camera");
  const uint32_t npix = (uint32_t)((uint64_t)ctx->cam.width * ctx->cam.height);
  if (npix != ctx->H) return fail(ctx, FPPM_ERR_STATE, "film_add: hit points are not the camera's pixels");
  FPPM_CUDA_OK(launch_film(ctx->stream, 0, npix, ctx->d_emit, ctx->d_gathered, ctx->o_flux, ctx->o_gather_r,
                           (double)ctx->cfg.samples_per_iteration, ctx->d_film, nullptr, ctx->sms, ctx->d_vcvm));
  ctx->film_iters++;
  return FPPM_OK;
}

int fppm_gpu_film_mean(fppm_gpu_ctx *ctx, double *rgb, uint64_t *iterations) {
  if (!ctx) return FPPM_ERR_INVALID_ARGUMENT;
  JOIN_RECS(ctx);
  if (!ctx->has_camera) return fail(ctx, FPPM_ERR_STATE, "film_mean before set_camera");
  const uint32_t npix = (uint32_t)((uint64_t)ctx->cam.width * ctx->cam.height);
  if (iterations) *iterations = ctx->film_iters;
  if (!rgb) return FPPM_OK;
  const size_t bytes = sizeof(double) * 3 * (size_t)npix;
  FPPM_CUDA_OK(ensure_scratch(ctx, bytes + 64));
  double *d = static_cast<double *>(ctx->d_scratch);
  FPPM_CUDA_OK(launch_film(ctx->stream, 1, npix, nullptr, nullptr, nullptr, nullptr, (double)ctx->film_iters,
                           ctx->d_film, d, ctx->sms));
  FPPM_CUDA_OK(cudaMemcpyAsync(rgb, d, bytes, cudaMemcpyDeviceToHost, ctx->stream));
  FPPM_CUDA_OK(cudaStreamSynchronize(ctx->stream));
  return FPPM_OK;
}

int fppm_gpu_film_splits(fppm_gpu_ctx *ctx, double *vc, double *vm) {
  if (!ctx) return FPPM_ERR_INVALID_ARGUMENT;
  JOIN_RECS(ctx);
  if (!ctx->has_camera) return fail(ctx, FPPM_ERR_STATE, "film_splits before set_camera");
  const size_t npix = (size_t)ctx->cam.width * ctx->cam.height;
  std::vector<double2> h(npix);
  if (npix) FPPM_CUDA_OK(cudaMemcpyAsync(h.data(), ctx->d_vcvm, sizeof(double2) * npix, cudaMemcpyDeviceToHost,
                                         ctx->stream));
  FPPM_CUDA_OK(cudaStreamSynchronize(ctx->stream));
  for (size_t i = 0; i < npix; ++i) {
    if (vc) vc[i] = h[i].x;
    if (vm) vm[i] = h[i].y;
  }
  return FPPM_OK;
}

int fppm_gpu_get_photon_mis(fppm_gpu_ctx *ctx, double *d_vcm, double *d_vm, double *cont) {
  if (!ctx) return FPPM_ERR_INVALID_ARGUMENT;
  JOIN_RECS(ctx);
  if (!ctx->cfg.vcm_plus || !ctx->d_pmis_in[0]) return fail(ctx, FPPM_ERR_STATE, "context is not vcm_plus");
  double *dst[3] = {d_vcm, d_vm, cont};
  for (int i = 0; i < 3; ++i)
    if (dst[i] && ctx->N)
      FPPM_CUDA_OK(cudaMemcpyAsync(dst[i], ctx->d_pmis_in[i], sizeof(double) * ctx->N, cudaMemcpyDeviceToHost,
                                   ctx->stream));
  FPPM_CUDA_OK(cudaStreamSynchronize(ctx->stream));
  return FPPM_OK;
}

int fppm_gpu_set_hitpoint_mis(fppm_gpu_ctx *ctx, const double *d_vcm, const double *d_vm, uint32_t n) {
  if (!ctx || (n && (!d_vcm || !d_vm))) return FPPM_ERR_INVALID_ARGUMENT;
  JOIN_RECS(ctx);
  if (!ctx->cfg.vcm_plus) return fail(ctx, FPPM_ERR_STATE, "MIS partials need vcm_plus");
  if (n != ctx->H) return fail(ctx, FPPM_ERR_INVALID_ARGUMENT, "one MIS pair per hit point");
  std::vector<double2> v(n);
  for (uint32_t h = 0; h < n; ++h) v[h] = make_double2(d_vcm[h], d_vm[h]);
  FPPM_CUDA_OK(cudaMemcpyAsync(ctx->d_eye_mis, v.data(), sizeof(double2) * n, cudaMemcpyHostToDevice,
                               ctx->stream));
  FPPM_CUDA_OK(cudaStreamSynchronize(ctx->stream));
  return FPPM_OK;
}

int fppm_gpu_set_photon_mis(fppm_gpu_ctx *ctx, const double *d_vcm, const double *d_vm, const double *cont,
                            uint32_t n) {
  if (!ctx || (n && (!d_vcm || !d_vm || !cont))) return FPPM_ERR_INVALID_ARGUMENT;
  JOIN_RECS(ctx);
  if (!ctx->cfg.vcm_plus) return fail(ctx, FPPM_ERR_STATE, "MIS partials need vcm_plus");
  if (n > ctx->cfg.max_photons) return fail(ctx, FPPM_ERR_CAPACITY, "photons exceed max_photons");
  const double *src[3] = {d_vcm, d_vm, cont};
  for (int i = 0; i < 3; ++i)
    if (n)
      FPPM_CUDA_OK(cudaMemcpyAsync(ctx->d_pmis_in[i], src[i], sizeof(double) * n, cudaMemcpyHostToDevice,
                                   ctx->stream));
  ctx->pmis_set = true;
  ctx->grid_valid = false;
  return FPPM_OK;
}

int fppm_gpu_counters(fppm_gpu_ctx *ctx, uint64_t out[4]) {
  if (!ctx || !out) return FPPM_ERR_INVALID_ARGUMENT;
  FPPM_CUDA_OK(cudaMemcpyAsync(ctx->h_counters, ctx->d_counters, 32, cudaMemcpyDeviceToHost,
                               ctx->stream));
  FPPM_CUDA_OK(cudaStreamSynchronize(ctx->stream));
  for (int i = 0; i < 4; ++i) out[i] = ctx->h_counters[i];
  return FPPM_OK;
}

double fppm_gpu_schedule_radius(double base, double alpha, uint64_t i) {
  return host_schedule_radius(base, alpha, i);
}

double fppm_gpu_f_quantile(double p, double d1, double d2, int *status) {
  if (status) *status = FPPM_OK;
  return host_f_quantile(p, d1, d2, status);
}

double fppm_gpu_chi2_quantile(double p, double df, int *status) {
  if (status) *status = FPPM_OK;
  return host_chi2_quantile(p, df, status);
}

}  // extern "C"
