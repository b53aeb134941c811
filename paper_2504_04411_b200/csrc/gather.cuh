// gather.cuh -- kernel argument blocks shared by gather.cu and context.cu.
#pragma once
#include <atomic>

#include "common.cuh"

namespace fppm_b200 {

// every kernel launch issued by this library (reported as gpu_launches)
extern std::atomic<unsigned long long> g_kernel_launches;
inline void note_launches(int n) { g_kernel_launches.fetch_add((unsigned long long)n); }

constexpr int kGatherThreads = 256;
constexpr int kMaxCG = 96;  // n_a * n_s <= 32, times up to 3 channels

// end-of-iteration policy parameters (gather.cpp:74-144)
struct EndParams {
  int policy;
  int override_decision;
  unsigned long long J;      // samples per iteration
  double k;                  // RadiusSchedule::k
  double floor_next;         // schedule_radius(r_min_base, alpha, i + 1)
  double sched_next;         // schedule_radius(r_1, alpha, i + 1)
  const double *crit;        // F_c by t (host-computed f_quantile table)
  uint32_t crit_len;
  double chi2_crit;
};

struct GatherArgs {
  // regions
  const double3 *pos, *nrm, *K;
  const uint32_t *eye_depth;
  const uint8_t *gathered;
  double *radius;
  uint32_t *t;
  unsigned long long *st_cnt;
  double *st_sum, *st_sq;
  uint32_t H;
  // grid
  const float4 *rec0, *rec1, *rec2, *rec3;
  const uint32_t *cell_start;
  const GridHeader *grid;
  // lean layout's exact path: sorted -> input order, and the input photons
  const uint32_t *order;
  const float *in_pos, *in_nrm, *in_wi, *in_pow;
  const uint32_t *in_depth;
  // config
  int na, ns;
  uint32_t max_depth;
  double guard;
  EndParams end;
  // outputs (device, nullable)
  double *o_gather_r, *o_stat, *o_crit, *o_flux;
  uint8_t *o_flags;
  float *o_radiance;
  uint32_t *o_accepted;
  unsigned long long *snap_cnt;
  double *snap_sum, *snap_sq;
  // VCM+ merge stage (warp kernel): MIS merge weight per pair
  int vcm;
  int mis_n_vm;
  double mis_beta;
  const double2 *eye_mis;                      // per hit point {d_vcm, d_vm}
  const double *p_vcm, *p_vm, *p_cont;         // per photon, sorted order
  const double3 *wo, *alb;                     // eye Bsdf (cos_o, continuation prob)
  // multi-GPU option B: per-hit-point partial sums of this launch's photons
  // (row [count G | sum C*G | sum_sq C*G | power 3], fp64) instead of the
  // end-of-iteration update; pooled on the owner by launch_apply_deltas
  double *delta_out;
  // counters
  unsigned long long *counters;  // cumulative [accepted, candidates, exact, ambiguous]
  unsigned int *iter_tr;         // this launch [tested, rejected]
  unsigned int *work;
  unsigned long long *rmax_bits;
};

struct EndArgs {
  double *radius;
  uint32_t *t;
  unsigned long long *st_cnt;
  double *st_sum, *st_sq;
  uint32_t H;
  int G, C;
  EndParams end;
  double *o_gather_r, *o_stat, *o_crit;
  uint8_t *o_flags;
  unsigned long long *snap_cnt;
  double *snap_sum, *snap_sq;
};

// ---- fine-kernel items (gather_fine.cu) and their pooling (sched.cu)
struct TileArgs {
  const void *desc;             // unused (fine items carry their own descriptors)
  const uint32_t *hp_order;     // cell-sorted hit point indices
  double *partials;             // [item][32][partial_size] per-item results
  const uint32_t *hp_map;       // per hit point: first item, chunks, wave slot
  const uint32_t *total_items;  // device scalar
  bool contig = false;          // ring schedule: each hit point's rows contiguous, in hit-point order
};

struct SortScratch {
  uint32_t *keys_a, *vals_a, *keys_b, *vals_b;
  uint32_t *hist;  // [digit][tile] + digit totals
};

// ---- fine-cell tiled gather (gather_fine.cu)
#ifndef FPPM_FINE_S
#define FPPM_FINE_S 4
#endif
constexpr uint32_t kFineS = FPPM_FINE_S;  // fine cells per reference cell and axis (slab layout)
constexpr int kFMaxPieces = 3 * (int)kFineS > 9 ? 3 * (int)kFineS : 9;  // slab rows / 3x3 columns
static_assert(kFMaxPieces <= 32, "one lane per run");
constexpr uint32_t kFSub = 16;   // windows per item (one CTA walks them in order)
struct alignas(16) FineDesc {  // one per (home cell, wave, run of <= kFSub windows)
  uint32_t hp_lo, hp_n, nwin, npieces;
  uint32_t c0, c1, pbase, pad0;     // windows [c0, c1) of the union; partial rows pbase + k
  int32_t ux0, ux1, uy0, uy1, uz0, uz1;  // union of the wave's fine boxes
  uint32_t src[kFMaxPieces];        // first sorted record of piece p
  uint32_t pre[kFMaxPieces + 1];    // flattened offset of piece p (pre[max] = union size)
  // ring schedule (one window per item): claim order of the wave's hit points,
  // largest fragment first; only the nclaim hit points whose window range
  // holds this window are claimed
  uint32_t nclaim;
  uint8_t order[32];
};
static_assert(sizeof(FineDesc) % 16 == 0 && sizeof(FineDesc) / 4 <= 256, "FineDesc layout");

struct FineHot;   // compact per hit point state staged per item
struct Hit;       // gather_dev.cuh
struct FineArgs {
  const FineDesc *desc;
  const FineHot *hot;
  const Hit *hits;  // full per-hit-point state (exact path), wave order
  const uint32_t *hp_order;
  double *partials;
  const uint32_t *hp_map;
  const uint32_t *total_items;
};

struct TileSched {
  FineDesc *fdesc = nullptr;
  unsigned long long fdesc_cap = 0;
  void *fhot = nullptr;   // FineHot[H]
  int4 *fbox = nullptr;   // [H] (bx1, bz0, bz1, -): the rest of a hit point's fine box (wave unions)
  void *fhit = nullptr;   // Hit[H]: full state for the exact path, wave order
  uint32_t *pbase = nullptr;  // [nb + 1] partial rows per bucket, scanned
  SortScratch sort;     // hit-point keys (capacity H)
  uint32_t *hp_order;   // alias of the sorted values
  uint32_t *hp_start;   // [nb + 1]
  uint32_t *items, *chunks, *item_base;  // [nb + 1]
  uint32_t *scan_tmp;
  double *partials;
  uint32_t *hp_map;     // [3 H]
  uint32_t *hp_nc = nullptr, *hp_rbase = nullptr, *hp_scan_tmp = nullptr;  // ring rows per hit point [H + 1]
  uint2 *hp_span = nullptr;  // ring: per wave position, the flattened span of the hit point's runs
  uint32_t *nonempty;   // device counter: buckets holding hit points
  unsigned long long bucket_cap, item_cap;
  unsigned long long row_cap = 0;  // partial rows allocated
  // hit-point bins of the last fine schedule (hp_order, hp_start): reused
  // while the hit points and the grid geometry they were binned on are
  // unchanged (a static frame whose r_max holds, e.g. C1 / C2)
  bool bins_valid = false;
  unsigned long long bins_version = 0;
  uint32_t bins_H = 0, bins_nb = 0;
  double bins_inv = 0.0;
  long long bins_dims[7] = {0, 0, 0, 0, 0, 0, 0};
};

// [count G | sum C G | sum_sq C G | power 3], padded to an even count (16-B rows)
__host__ __device__ constexpr int partial_size(int gmax, int ch) { return (gmax + 2 * ch * gmax + 3 + 1) & ~1; }

cudaError_t launch_tile_finalize(cudaStream_t s, const GatherArgs &A, const TileArgs &T, int C,
                                 int sms);
size_t tile_partial_doubles(int G, int C);

cudaError_t launch_bucket_start(cudaStream_t s, const uint32_t *skeys, uint32_t n, uint32_t nb,
                                uint32_t *start, int sms);
cudaError_t launch_exclusive_scan(cudaStream_t s, const uint32_t *in, uint32_t n, uint32_t *tmp,
                                  uint32_t *out);
// multi-GPU photon staging (shard.cu)
constexpr int kMaxPackedParts = 64;
cudaError_t launch_hp_box(cudaStream_t s, const double3 *pos, uint32_t n, double *box);
cudaError_t launch_cull_packed(cudaStream_t s, const uint32_t *data, unsigned long long stride, uint32_t parts,
                               const uint32_t *part_n, const double *box, const double *margin, uint32_t *keep,
                               uint32_t *dst, uint32_t *scan_tmp, float *pos, float *nrm, float *wi, float *pw,
                               uint32_t *depth, int sms);
bool fine_supported(int G, int C);
void fine_caps(int G, int C, int lean, uint32_t *cap64, uint32_t *cap48, uint32_t *fsub);  // lean: GridHeader::lean
bool flat_records_enabled();  // the 32-B flat lean layout may be chosen (ring kernel on, FPPM_FLAT != 0)
bool ring_enabled();
cudaError_t fine_schedule_bins(cudaStream_t s, const GatherArgs &A, TileSched &S, const GridHeader &g,
                               int sms, uint32_t cap64, uint32_t cap48, uint32_t fsub, uint32_t *nb_out,
                               unsigned long long hp_version);
cudaError_t fine_schedule_items(cudaStream_t s, const GatherArgs &A, TileSched &S, uint32_t nb, int sms,
                                uint32_t cap64, uint32_t cap48, uint32_t fsub);
size_t fine_acc_doubles(int G, int C);
cudaError_t launch_gather_fine(cudaStream_t s, const GatherArgs &A, const FineArgs &T, int C, int sms, int lean);
size_t fine_hot_bytes();
size_t fine_hit_bytes();

cudaError_t launch_gather_test(cudaStream_t s, const GatherArgs &A, int C, int sms);
cudaError_t launch_samples(cudaStream_t s, const uint32_t *region, const double2 *y,
                           const double *value, uint32_t n, const double *radius, uint32_t H,
                           int na, int ns, int C, int *sectors, int *err,
                           unsigned long long *st_cnt, double *st_sum, double *st_sq, int phase);
cudaError_t launch_end_iteration(cudaStream_t s, const EndArgs &A);
// thread-per-hit-point gather for sparse 3D frames (gather.cu)
// writes option-B rows [H][G + 2 G C + 3]; the caller pools them
// (launch_apply_deltas) unless they are the cross-rank partial sums
// hot3 != NULL: k_prep_3d + k_gather_3d, a warp per hit point (dense 3D
// frames, tens of candidates per hit point and more; hot3 holds
// hot3_bytes() and hits fine_hit_bytes() per hit point); else
// k_gather_sparse, one thread per hit point
cudaError_t launch_gather_sparse(cudaStream_t s, const GatherArgs &A, int C, const uint32_t *order,
                                 double *rows, int sms, void *hot3, void *hits);
size_t hot3_bytes();
cudaError_t hp_cell_order(cudaStream_t s, const GatherArgs &A, TileSched &S, const GridHeader &g, int sms,
                          const uint32_t **order);
size_t sparse_smem_bytes(int G, int C);
// pools summed option-B rows into regions [h0, h0 + n) and runs the
// end-of-iteration policy (finalize_hit)
cudaError_t launch_apply_deltas(cudaStream_t s, const GatherArgs &A, int C, uint32_t h0, uint32_t n,
                                const double *delta);
cudaError_t launch_hit_weights(cudaStream_t s, const double3 *nrm, const double3 *wo,
                               const double3 *thr, const double3 *alb, uint32_t H, double3 *K);
// *flag = 1 when every gathered hit point is planar (n = +z, fp32-exact
// centre) and gray (K0 = K1 = K2 finite): the lean record layout applies
cudaError_t launch_lean_check(cudaStream_t s, const double3 *pos, const double3 *nrm, const double3 *K,
                              const uint8_t *gathered, uint32_t H, uint32_t *flag);

// grid.cu
size_t radix_hist_entries(uint32_t n);
cudaError_t radix_sort_pairs(cudaStream_t s, SortScratch &sc, uint32_t n, uint32_t bits,
                             uint32_t **keys_sorted, uint32_t **vals_sorted);
void launch_cell_bounds(cudaStream_t s, const float *pos, uint32_t n, const double *cell,
                        uint32_t S, long long *bounds, int sms);
void launch_grid_header(cudaStream_t s, const long long *bounds, const double *cell, uint32_t n,
                        unsigned long long max_cells, uint32_t S, const uint32_t *lean_ok, bool allow_flat,
                        GridHeader *hdr);
void launch_dense_keys(cudaStream_t s, const float *pos, uint32_t n, const GridHeader *hdr,
                       uint32_t *keys, uint32_t *vals, int sms);
void launch_pack_fine(cudaStream_t s, const float *pos, const float *nrm, const float *wi, const float *pw,
                      const uint32_t *depth, uint32_t n, const GridHeader *hdr, double guard, float4 *pack,
                      int sms);
void launch_permute_f64x3(cudaStream_t s, const uint32_t *order, uint32_t n, const double *a,
                          const double *b, const double *c, double *oa, double *ob, double *oc, int sms);
void launch_cell_start(cudaStream_t s, const uint32_t *skeys, uint32_t n, const GridHeader *hdr,
                       uint32_t *start, unsigned long long ncells, int sms);
void launch_permute(cudaStream_t s, const uint32_t *order, uint32_t n, const float *pos,
                    const float *nrm, const float *wi, const float *pw, const uint32_t *depth,
                    const PhotonRecs &r, int fine_layout, const GridHeader *hdr, int sms);
void launch_query_ball(cudaStream_t s, const double *centers, const double *radii, uint32_t nq,
                       const GridHeader *hdr, const uint32_t *start, const float4 *rec0,
                       const uint32_t *order, unsigned long long *counts,
                       const unsigned long long *offsets, uint32_t *out, int fill);

// trace.cu (light phase on analytic geometry)
struct TraceScene {
  int n_mat, n_prim, n_emit;
  const int *mat_kind;      // FPPM_MATERIAL_*
  const double *mat_rgb;    // [n][3]
  const double *mat_ior;
  const int *prim_kind;     // FPPM_SHAPE_*
  const double *prim;       // [n][9]
  const int *prim_mat;
  const int *emit_prim;
  const double *emit_rad;   // [n][3]
};
struct TraceArgs {
  TraceScene sc;
  unsigned long long seed, iteration;
  uint32_t n_paths, light_depth;
  uint32_t path0;  // global index of path 0 (a rank's share of the light phase)
  int n_vm;
  double beta, eta_vm;
  float *v_pos, *v_nrm, *v_wi, *v_pow;  // per path slots [n_paths][light_depth][3]
  uint32_t *v_depth;
  double *v_mis;                        // [.][3] d_vcm, d_vm, cont (nullable)
  uint32_t *count;                      // [n_paths]
  uint32_t *path_counter;               // work queue (reset by launch_trace)
  // bidirectional (VCM+) light vertices in fp64, same slots (nullable):
  // LightVertex position, shading normal, wi, throughput, {d_vcm, d_vc, d_vm}
  double *b_pos, *b_sn, *b_wi, *b_thr, *b_mis;
  int *b_mat;
};
struct CamD {  // CameraFrame (path.hpp:93-98), built on the host (make_camera_frame)
  double pos[3], fwd[3], right[3], up[3];
  double plane_dist;
  int width, height;
};
struct EyeArgs {
  TraceScene sc;
  CamD cam;
  unsigned long long seed, iteration;
  uint32_t max_depth, npix;
  double3 *pos, *nrm, *wo, *thr, *alb, *emitted;
  uint32_t *eye_depth;
  uint8_t *gathered;
};
cudaError_t launch_trace_eye(cudaStream_t s, const EyeArgs &E, const void *prep, int sms);

// VCM+ bidirectional remainder (trace.cu): eye sub-paths with MIS partials,
// emitter hits, next-event estimation, connections to the pixel's light
// sub-path, merge vertices for the gathers; light-vertex splats to the camera.
constexpr uint32_t kMaxBidirDepth = 16;
struct BidirArgs {
  TraceScene sc;
  CamD cam;
  unsigned long long seed, iteration;
  uint32_t max_depth, npix, n_paths, light_depth;
  int n_vm;
  double beta, eta_light;          // light sub-paths' eta_vm (r_max; integrator.cpp:171-174)
  const double *radius;            // [npix] region radius before this iteration's update
  // light vertices (TraceArgs::b_*), per-path counts
  const double *l_pos, *l_sn, *l_wi, *l_thr, *l_mis;
  const int *l_mat;
  const uint32_t *l_depth;  // TraceArgs::v_depth slots (LightVertex::depth)
  const uint32_t *l_count;
  // outputs: direct estimate per pixel, primary merge vertex (the region's
  // hit point), secondary merge vertices [npix][max_depth - 1]
  double3 *direct;
  double3 *pos, *nrm, *wo, *thr, *alb;
  uint32_t *eye_depth;
  uint8_t *gathered;
  double2 *eye_mis;
  double3 *q_pos, *q_nrm, *q_wo, *q_thr, *q_alb;
  uint32_t *q_eye;
  uint8_t *q_gathered;
  double *q_radius;
  double2 *q_mis;
  double3 *splat;  // light-to-camera splats (atomic adds)
  // eye sub-paths between k_eye_walk and k_eye_bidir: [16][max_depth][npix]
  // fp64 fields, [max_depth][npix] int4, vertex counts, RNG states
  double *vtx_d;
  int4 *vtx_i;
  uint32_t *vtx_n;
  unsigned long long *vtx_rng;
};
cudaError_t launch_eye_bidir(cudaStream_t s, const BidirArgs &B, const void *prep, int sms);
cudaError_t launch_light_splat(cudaStream_t s, const BidirArgs &B, const void *prep, int sms);
// film for VCM+: est = direct + (flux + secondary merge sums) / (pi r^2 J) + splats
cudaError_t launch_film_vcm(cudaStream_t s, uint32_t npix, uint32_t nq_per_px, const double3 *direct,
                            const uint8_t *gathered, const double *flux, const double *gather_r,
                            const double *q_rows, uint32_t q_stride, const uint8_t *q_gathered,
                            const double *q_radius, const double3 *splat, double J, double3 *film, int sms,
                            double2 *vcvm);
// op 0: film += estimate (J = samples per iteration); op 1: mean_out = film / J (J = iterations)
cudaError_t launch_film(cudaStream_t s, int op, uint32_t npix, const double3 *emitted, const uint8_t *gathered,
                        const double *flux, const double *gather_r, double J, double3 *film, double *mean_out,
                        int sms, double2 *vcvm = nullptr);
size_t trace_prep_bytes(int n_prim);
int trace_max_prims();
cudaError_t launch_scene_prep(cudaStream_t s, const TraceScene &sc, void *prep);
cudaError_t launch_trace(cudaStream_t s, const TraceArgs &A, const void *prep, int sms);
cudaError_t launch_trace_compact(cudaStream_t s, const TraceArgs &A, const uint32_t *base, float *pos,
                                 float *nrm, float *wi, float *pw, uint32_t *depth, double *mv, double *mm,
                                 double *mc, int sms);

// generate.cu
// C5 workload (generate.cu)
constexpr int kC5Clusters = 64;
constexpr int kC5Attempts = 8;
struct C5Args {
  uint64_t seed;
  uint32_t H;
  int G;                       // NN grid: G^3 cells over the unit cube
  const double *clusters;      // [64][5] center xyz, sigma, cumulative weight
  const double3 *pos, *nrm;    // all H hit points
  const uint32_t *start, *items;
};
cudaError_t launch_c5_setup(cudaStream_t s, uint64_t seed, uint32_t H, int G, double *clusters, double3 *pos,
                            double3 *nrm, uint32_t *cnt, uint32_t *cell_of, uint32_t *start, uint32_t *fill,
                            uint32_t *items, uint32_t *scan_tmp, int sms);
cudaError_t launch_c5_photons(cudaStream_t s, const C5Args &C, uint64_t iteration, uint64_t begin, uint32_t n,
                              float *pos, float *nrm, float *wi, float *pw, uint32_t *depth, int sms);
cudaError_t launch_c5_set_hitpoints(cudaStream_t s, const C5Args &C, uint32_t h0, uint32_t n, double3 *pos,
                                    double3 *nrm, double3 *wo, double3 *thr, double3 *alb, uint32_t *eye_depth,
                                    uint8_t *gathered, int sms);
void launch_generate_photons(cudaStream_t s, int workload, uint64_t seed, uint64_t iteration,
                             uint64_t begin, uint32_t n, float *pos, float *nrm, float *wi,
                             float *pw, uint32_t *depth, int sms);
void launch_raster_hitpoints(cudaStream_t s, uint32_t W, double3 *pos, double3 *nrm,
                             double3 *wo, double3 *thr, double3 *alb, uint32_t *eye_depth,
                             uint8_t *gathered, int sms);

// host_stats.cpp
double host_f_quantile(double p, double d1, double d2, int *status);
double host_chi2_quantile(double p, double df, int *status);
int host_sector_index(double u, double v, double radius, int na, int ns, int *status);
void host_build_frame(const double n[3], double u[3], double v[3]);
double host_schedule_radius(double base, double alpha, uint64_t i);

}  // namespace fppm_b200
