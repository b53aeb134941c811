/*
 * fppm_gpu.h -- C ABI of the B200-native gather + F-test hot path.
 *
 * This is the drop-in boundary for the reference's in-process C++ interface
 * of the hot path (reference proj/core, installed headers fppm/*.hpp):
 *
 *   fppm::PhotonGrid(std::vector<LightVertex>, double cell)   photon_map.hpp:18
 *   fppm::PhotonGrid::query_ball(center, r, out)              photon_map.hpp:26-27
 *   fppm::GatherRegion(TestConfig, RadiusSchedule, r0)        gather.hpp:71-72
 *   fppm::GatherRegion::move_to / accumulate / end_iteration  gather.hpp:75-81
 *   fppm::GatherRegion::chi2_end_iteration / schedule_end_iteration  :84-87
 *   Renderer::gather_disk + pixel_pm gather block   integrator.cpp:388-402, :435-489
 *
 * The reference drives one GatherRegion per pixel from a host thread pool;
 * here one context owns all regions ("hit points") of a frame on one B200
 * and every call is a batched, stream-ordered operation over all of them.
 *
 * Conventions:
 *   - every entry point returns fppm_status (0 = ok); no exception crosses;
 *     the C++ wrapper fppm_gpu.hpp rethrows std::invalid_argument /
 *     std::domain_error for FPPM_ERR_INVALID_ARGUMENT / FPPM_ERR_DOMAIN;
 *   - the caller owns host buffers, the context owns device buffers;
 *   - calls are ordered on the context's CUDA stream and are not re-entrant
 *     (one host thread per context);
 *   - photons are canonical fp32 records (position, shading normal, incident
 *     direction wi, power/throughput RGB, depth); hit points are fp64 like the
 *     reference Point3/Normal3; accumulators and radii are fp64.
 */
#ifndef FPPM_GPU_H
#define FPPM_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FPPM_GPU_ABI_VERSION 1

typedef enum fppm_status {
  FPPM_OK = 0,
  FPPM_ERR_INVALID_ARGUMENT = 1, /* reference: std::invalid_argument */
  FPPM_ERR_DOMAIN = 2,           /* reference: std::domain_error */
  FPPM_ERR_CUDA = 3,             /* CUDA runtime failure (message in last_error) */
  FPPM_ERR_CAPACITY = 4,         /* a buffer bound in fppm_gpu_config exceeded */
  FPPM_ERR_STATE = 5,            /* call order violated (e.g. gather before grid) */
  FPPM_ERR_NO_DEVICE = 6         /* no sm_100 device: there is no CPU fallback */
} fppm_status;

/* gather.hpp:29 TestChannels (auto_detect is resolved by the caller) */
#define FPPM_CHANNELS_LUMINANCE 1
#define FPPM_CHANNELS_RGB 3
/* gather.hpp:32 TestOverride */
#define FPPM_OVERRIDE_NONE 0
#define FPPM_OVERRIDE_ALWAYS_REJECT 1
#define FPPM_OVERRIDE_NEVER_REJECT 2
/* end-of-iteration policy: gather.cpp:90 / :114 / :138 */
#define FPPM_POLICY_FTEST 0
#define FPPM_POLICY_CHI2 1
#define FPPM_POLICY_SCHEDULE 2
/* canonical synthetic workloads */
#define FPPM_WORKLOAD_C1 1
#define FPPM_WORKLOAD_C2 2
#define FPPM_WORKLOAD_C5 5  /* needs fppm_gpu_c5_setup (same seed) */

typedef struct fppm_gpu_config {
  /* TestConfig (gather.hpp:34-41).  Deliberate deviation: the reference
   * accepts any n_annuli * n_sectors >= 2 (gather.cpp:49-50); the device
   * keeps at most 32 sectors per region and fppm_gpu_create returns
   * FPPM_ERR_CAPACITY above that (the product is formed in 64 bits). */
  int32_t n_annuli;
  int32_t n_sectors;
  double alpha_f;
  double alpha_chi2;
  int32_t channels;          /* FPPM_CHANNELS_* */
  int32_t override_decision; /* FPPM_OVERRIDE_* */
  int32_t policy;            /* FPPM_POLICY_* */
  /* RadiusSchedule (gather.hpp:16-20) */
  double k;
  double alpha;
  double r_min_base;
  /* r_1 of every region (GatherRegion ctor, gather.cpp:35-52) */
  double initial_radius;
  /* J: nominal samples per iteration (end_iteration arg, integrator.cpp:480) */
  uint64_t samples_per_iteration;
  /* integrator.cpp:396-397 filters */
  uint32_t max_depth;
  double normal_guard_cos; /* 0.86602540378443865 in the reference */
  /* capacities (device buffers are sized once) */
  uint32_t max_hitpoints;
  uint32_t max_photons;
  uint32_t max_cells; /* 0 -> 1<<28 dense cells */
  int32_t device;     /* CUDA ordinal */
  void *stream;       /* cudaStream_t to order work on; NULL -> own stream */
  int32_t gather_kernel; /* 0 auto: 4 on slab (planar) grids when n_a*n_s*channels <= 24, else 5;
                            1 warp per hit point over reference cells (cross-check);
                            4 fine-cell tiled (slab grids; 3D grids use 5);
                            5 warp per hit point over 3D fine columns (S = 2 or 1) */
  /* VCM+ merge stage (integrator.cpp:595-627): every gathered photon value is
   * weighted by mis_weight_merge (path.cpp:103-111) with the tested radius;
   * needs fppm_gpu_set_hitpoint_mis / fppm_gpu_set_photon_mis; runs on the
   * 3D kernel (gather_kernel 0 or 5) or the warp kernel (1) */
  int32_t vcm_plus;
  int32_t mis_n_vm;   /* MisContext::n_vm (light paths per iteration, integrator.cpp:133) */
  double mis_beta;    /* MisContext::beta (MIS power) */
} fppm_gpu_config;

typedef struct fppm_gpu_ctx fppm_gpu_ctx;

/* Hit points (the GatherRegion centers of one iteration); all [n][3] fp64
 * except eye_depth (u32) and gathered (u8, NULL = every hit point gathers). */
typedef struct fppm_hitpoints {
  const double *pos;        /* gather point x (move_to center) */
  const double *normal;     /* shading normal (move_to normal, Bsdf frame) */
  const double *wo;         /* direction toward the eye (Bsdf cos_o) */
  const double *throughput; /* eye-path throughput (integrator.cpp:448) */
  const double *albedo;     /* Lambertian albedo (bsdf.cpp:63) */
  const uint32_t *eye_depth;/* depth of the gather vertex (integrator.cpp:444) */
  const uint8_t *gathered;  /* integrator.cpp:476-488 */
} fppm_hitpoints;

/* Photons = light vertices (LightVertex, path.hpp:76-89), canonical fp32.
 * The reference's LightVertex is fp64: a caller binding real LightVertex
 * data rounds position, normal and wi to fp32 here, and every predicate
 * (cell_coord, ball, guard, disk, sector) then runs on the rounded values
 * widened back to fp64.  Parity with the reference is bit-exact for
 * fp32-representable inputs (all synthetic workloads); for arbitrary fp64
 * positions a photon within ~2^-24 relative of a cell, ball, disk or sector
 * boundary may be classified differently. */
typedef struct fppm_photons {
  const float *pos;     /* [n][3] */
  const float *normal;  /* [n][3] shading normal at the deposit */
  const float *wi;      /* [n][3] unit, toward where the energy came from */
  const float *power;   /* [n][3] throughput RGB */
  const uint32_t *depth;/* [n] */
} fppm_photons;

/* Per-hit-point outputs of one iteration (host pointers; NULL skips).
 * Field meanings follow RadiusUpdate (gather.hpp:55-61) and pixel_pm. */
typedef struct fppm_gpu_iter_out {
  double *radius;        /* after the update */
  double *gather_radius; /* radius the gather used */
  uint64_t *t;           /* held_iterations() after the update */
  uint8_t *tested;
  uint8_t *rejected;
  double *statistic;
  double *critical;
  double *flux;          /* [n][3] sum of photon values (integrator.cpp:449) */
  float *radiance;       /* [n][3] flux / (pi r^2 J) (integrator.cpp:452-455) */
  uint32_t *accepted;    /* accepted photons this iteration */
  uint64_t *stat_count;  /* [n][C*G] pooled stats BEFORE end_iteration */
  double *stat_sum;
  double *stat_sum_sq;
} fppm_gpu_iter_out;

/* Whole-frame summary of one iteration (host). */
typedef struct fppm_gpu_summary {
  uint64_t accepted;       /* Q: accepted (hit point, photon) pairs */
  uint64_t candidates;     /* pairs ball-tested (27-cell neighbourhoods) */
  uint64_t exact_pairs;    /* pairs resolved on the fp64 exact path */
  uint64_t ambiguous_pairs;/* sector assignments within 1 ulp of a bin edge */
  uint32_t tested;
  uint32_t rejected;
  double cell_size;        /* grid cell (= max live radius before the update) */
  double r_max_next;       /* max radius after the update */
  uint64_t cells;          /* dense cells in the grid bounding box */
} fppm_gpu_summary;

/* Device pointers owned by the context (for zero-copy producers such as an
 * NCCL all-gather into the photon staging buffers). */
typedef struct fppm_gpu_device_view {
  float *photon_pos, *photon_normal, *photon_wi, *photon_power;
  uint32_t *photon_depth;
  double *radius;
  uint64_t *counters; /* [0]=accepted [1]=candidates [2]=exact [3]=ambiguous, cumulative */
} fppm_gpu_device_view;

int fppm_gpu_abi_version(void);
const char *fppm_gpu_status_string(int status);

int fppm_gpu_create(const fppm_gpu_config *config, fppm_gpu_ctx **out);
int fppm_gpu_destroy(fppm_gpu_ctx *ctx);
const char *fppm_gpu_last_error(const fppm_gpu_ctx *ctx);
int fppm_gpu_synchronize(fppm_gpu_ctx *ctx);
void *fppm_gpu_stream(fppm_gpu_ctx *ctx);
int fppm_gpu_device_view_get(fppm_gpu_ctx *ctx, fppm_gpu_device_view *view);

/* ---- hit points / regions (GatherRegion state) ---- */
int fppm_gpu_set_hitpoints(fppm_gpu_ctx *ctx, const fppm_hitpoints *host, uint32_t n);
int fppm_gpu_set_hitpoints_device(fppm_gpu_ctx *ctx, const fppm_hitpoints *dev, uint32_t n);
/* Canonical raster hit points ((i+1/2)/W, (j+1/2)/W, 0), n=+z. */
int fppm_gpu_generate_raster_hitpoints(fppm_gpu_ctx *ctx, uint32_t W);
/* Reset every region to r_1, t = 1, zero stats (GatherRegion ctor). */
int fppm_gpu_reset_regions(fppm_gpu_ctx *ctx);
/* Region state readback/overwrite (host arrays, NULL skips). */
int fppm_gpu_get_regions(fppm_gpu_ctx *ctx, double *radius, uint64_t *t,
                         uint64_t *stat_count, double *stat_sum, double *stat_sum_sq);
int fppm_gpu_set_regions(fppm_gpu_ctx *ctx, const double *radius, const uint64_t *t,
                         const uint64_t *stat_count, const double *stat_sum,
                         const double *stat_sum_sq);
int fppm_gpu_max_radius(fppm_gpu_ctx *ctx, double *r_max);
/* Multi-GPU plumbing (no host round trip): the max live radius written to
 * device memory d_r_max (asynchronous, context stream), and a grid build whose
 * cell is read on the device from d_cell -- e.g. the all-reduce(max) of every
 * rank's fppm_gpu_max_radius_device (integrator.cpp:159-161).  The cell must
 * be >= every gathered radius (the reference's r_max is); the next gather
 * checks it and fails with "query radius exceeds cell size" otherwise. */
int fppm_gpu_max_radius_device(fppm_gpu_ctx *ctx, double *d_r_max);
int fppm_gpu_build_grid_device(fppm_gpu_ctx *ctx, const double *d_cell);

/* ---- photons + grid (PhotonGrid) ---- */
int fppm_gpu_set_photons(fppm_gpu_ctx *ctx, const fppm_photons *host, uint32_t n);
/* Pipelining extension (no reference counterpart): uploads the NEXT batch
 * into the free staging set on the copy stream while the current iteration
 * runs, without changing the current photons, and returns a token.
 * fppm_gpu_adopt_photons(token) then makes that batch current without a copy.
 * Adoption is explicit: fppm_gpu_set_photons always copies (and discards a
 * pending prefetch).  The host arrays must stay unchanged until adoption;
 * adopt recomputes a sampled digest (every field of 4096 records spread over
 * the batch) and returns FPPM_ERR_STATE when they were rewritten, as it does
 * for a stale or superseded token -- the caller then uploads with
 * fppm_gpu_set_photons. */
int fppm_gpu_prefetch_photons(fppm_gpu_ctx *ctx, const fppm_photons *host, uint32_t n, uint64_t *token);
int fppm_gpu_adopt_photons(fppm_gpu_ctx *ctx, uint64_t token);
int fppm_gpu_set_photons_device(fppm_gpu_ctx *ctx, const fppm_photons *dev, uint32_t n);
/* Multi-GPU staging (DESIGN.md §7 option A): `parts` photon shares packed as
 * [part][13][part_stride] 32-bit words (pos xyz, shading normal xyz, wi xyz,
 * power rgb as fp32 bits, depth), e.g. the output of ONE all-gather of every
 * rank's packed share; part p holds part_n[p] photons (host array).  They
 * are staged in part order, and with d_margin (device double, e.g. the
 * all-reduced r_max the grid is then built with) only photons inside this
 * context's hit-point bounding box grown by *d_margin are kept -- no photon
 * beyond r_max of every local hit point can be gathered, so results are
 * unchanged while the grid build sorts only the band's photons.
 * *n_kept receives the staged count (the call synchronizes for it). */
int fppm_gpu_set_photons_packed(fppm_gpu_ctx *ctx, const void *d_packed, uint32_t parts, uint64_t part_stride,
                                const uint32_t *part_n, const double *d_margin, uint32_t *n_kept);
/* Canonical synthetic photons [begin, begin+n) of (seed, iteration). */
int fppm_gpu_generate_photons(fppm_gpu_ctx *ctx, int32_t workload, uint64_t seed,
                              uint64_t iteration, uint64_t begin, uint32_t n);
/* Same generator writing into caller-owned device arrays (no staging). */
int fppm_gpu_generate_photons_to(fppm_gpu_ctx *ctx, int32_t workload, uint64_t seed,
                                 uint64_t iteration, uint64_t begin, uint32_t n,
                                 const fppm_photons *dev_dst);
/* Copy the staged photons back to host arrays (NULL skips).
 * Host uploads (fppm_gpu_set_photons) alternate between two staging sets on a
 * copy stream, so uploading iteration i+1 overlaps the gather of iteration i. */
int fppm_gpu_get_photons(fppm_gpu_ctx *ctx, float *pos, float *normal, float *wi, float *power,
                         uint32_t *depth);
/* Build the uniform hash grid; cell_size <= 0 uses the max live radius
 * (integrator.cpp:159-161).  Throws invalid_argument when cell <= 0. */
int fppm_gpu_build_grid(fppm_gpu_ctx *ctx, double cell_size);
/* Reference-layout export (PhotonGrid keys_/cells_/order_, photon_map.cpp:26-51).
 * Pass NULL arrays to query *ncells first. */
int fppm_gpu_export_grid(fppm_gpu_ctx *ctx, uint64_t *keys, uint32_t *begin,
                         uint32_t *end, uint32_t *order, uint64_t *ncells);
/* Batched query_ball (photon_map.cpp:53-78): indices of stored photons with
 * |pos - c|^2 <= r^2 in reference visit order.  offsets has nq+1 entries;
 * indices holds cap entries; *total receives the full count. */
int fppm_gpu_query_ball(fppm_gpu_ctx *ctx, const double *centers, const double *radii,
                        uint32_t nq, uint64_t *offsets, uint32_t *indices,
                        uint64_t cap, uint64_t *total);

/* ---- the hot path ---- */
/* Gather + accumulate + end-of-iteration policy for every hit point against
 * the grid built last (pixel_pm, integrator.cpp:435-489).  `out` arrays are
 * filled by asynchronous copies on the context stream: call
 * fppm_gpu_synchronize() before reading them (use pinned host memory for a
 * non-blocking call).  A non-NULL summary synchronizes. */
int fppm_gpu_gather_test(fppm_gpu_ctx *ctx, uint64_t iteration,
                         fppm_gpu_iter_out *out, fppm_gpu_summary *summary);
/* One FPPM iteration: build_grid(max live radius) + gather_test. */
int fppm_gpu_iterate(fppm_gpu_ctx *ctx, uint64_t iteration,
                     fppm_gpu_iter_out *out, fppm_gpu_summary *summary);

/* ---- C5 synthetic workload (BASELINE configs[4]) ----
 * Generates the n_hitpoints hit points of the workload (uniform in the unit
 * cube, uniform random normals), their nearest-neighbour grid and the 64
 * photon clusters for `seed`; FPPM_WORKLOAD_C5 photons then come from
 * fppm_gpu_generate_photons(_to).  c5_hitpoints sets hit points
 * [h0, h0 + n) of that set as the context's hit points (a rank's share). */
int fppm_gpu_c5_setup(fppm_gpu_ctx *ctx, uint64_t seed, uint32_t n_hitpoints);
int fppm_gpu_c5_hitpoints(fppm_gpu_ctx *ctx, uint32_t h0, uint32_t n);

/* ---- multi-GPU, photon-sharded decomposition (SURVEY.md 8(e) option B) ----
 * Each rank builds the grid of its own photon share and gathers for ALL hit
 * points, producing per-hit-point partial sums instead of the end-of-iteration
 * update; the rows are summed across ranks (ncclReduceScatter) and each owner
 * pools its slice and runs the policy.  A row is fppm_gpu_delta_stride(ctx)
 * doubles: [count G | sum C*G | sum_sq C*G | power 3] (G = n_a*n_s, C =
 * channels; counts are exact integers in fp64).  Afterwards the owners'
 * radii are all-gathered into every rank's radius array
 * (fppm_gpu_device_view_get) so the next gather sees them. */
uint32_t fppm_gpu_delta_stride(const fppm_gpu_ctx *ctx);
/* Gather against the grid built last into d_rows (device, [H][stride]);
 * region state is unchanged. */
int fppm_gpu_gather_deltas(fppm_gpu_ctx *ctx, uint64_t iteration, double *d_rows);
/* Pools d_rows (device, [n][stride], summed over ranks) into regions
 * [h0, h0 + n) and runs the end-of-iteration policy; `out` arrays hold n
 * entries (the slice), asynchronous as for fppm_gpu_gather_test. */
int fppm_gpu_apply_deltas(fppm_gpu_ctx *ctx, uint64_t iteration, uint32_t h0, uint32_t n,
                          const double *d_rows, fppm_gpu_iter_out *out, fppm_gpu_summary *summary);

/* ---- GatherRegion primitives on explicit samples (gather.cpp:59-67, 90-144) ---- */
/* Adds samples (region index, plane coords y, RGB value) to pooled stats. */
int fppm_gpu_accumulate(fppm_gpu_ctx *ctx, const uint32_t *region, const double *y,
                        const double *value, uint32_t n);
/* J passed to end_iteration (gather.hpp:81 samples_per_iteration). */
int fppm_gpu_set_samples_per_iteration(fppm_gpu_ctx *ctx, uint64_t samples_per_iteration);
/* Runs the configured end-of-iteration policy on every region without a gather
 * (outputs asynchronous as for fppm_gpu_gather_test). */
int fppm_gpu_end_iteration(fppm_gpu_ctx *ctx, uint64_t iteration,
                           fppm_gpu_iter_out *out);

/* Switches the end-of-iteration policy of every region (gather.cpp:90 F-test,
 * :114 chi-squared, :138 fixed schedule), e.g. for a caller that drives one
 * region through different policies like the reference's GatherRegion. */
int fppm_gpu_set_policy(fppm_gpu_ctx *ctx, int32_t policy);
/* Host restatements of two reference free functions the C++ wrapper needs:
 * sector_index (gather.cpp:15-33; FPPM_ERR_INVALID_ARGUMENT for bin counts
 * < 1, FPPM_ERR_DOMAIN outside the disk) and build_tangent_frame
 * (frame.cpp:5-14).  The device kernels evaluate the same expressions. */
int fppm_gpu_sector_index(double u, double v, double radius, int32_t n_annuli, int32_t n_sectors,
                          int32_t *index);
int fppm_gpu_build_frame(const double n[3], double u[3], double v[3]);

/* ---- photon emission and tracing (integrator.cpp:230-265, path.cpp:388-449) ---- */
/* Analytic scene (Scene, scene.hpp): spheres and quads, Lambertian / mirror /
 * dielectric materials, area emitters on primitives.  Host arrays. */
#define FPPM_MATERIAL_LAMBERTIAN 0
#define FPPM_MATERIAL_MIRROR 1
#define FPPM_MATERIAL_DIELECTRIC 2
#define FPPM_SHAPE_SPHERE 0
#define FPPM_SHAPE_QUAD 1
typedef struct fppm_scene {
  uint32_t n_materials;
  const int32_t *material_kind;  /* FPPM_MATERIAL_* */
  const double *material_rgb;    /* [n][3] albedo / reflectance / tint */
  const double *material_ior;    /* [n] (dielectric) */
  uint32_t n_primitives;
  const int32_t *shape_kind;     /* FPPM_SHAPE_* */
  const double *shape;           /* [n][9] sphere: center xyz, radius; quad: corner, e1, e2 */
  const int32_t *shape_material; /* [n] */
  uint32_t n_emitters;           /* area emitters */
  const int32_t *emitter_shape;  /* [n] primitive the emitter lives on */
  const double *emitter_radiance;/* [n][3] */
} fppm_scene;
int fppm_gpu_set_scene(fppm_gpu_ctx *ctx, const fppm_scene *scene);
/* Light phase of one iteration: traces light paths j = 0..n_paths-1 with
 * RngStream(seed, iteration, j, kLightStream = 0) to light depth max_depth - 1
 * and stages every non-delta deposit, in path order, as the photons of the
 * next grid build (with VCM+ MIS partials when vcm_plus; eta_vm uses
 * mis_radius, or the max live radius when mis_radius <= 0).  *n_photons
 * receives the deposit count (synchronizes). */
int fppm_gpu_trace_photons(fppm_gpu_ctx *ctx, uint64_t seed, uint64_t iteration, uint32_t n_paths,
                           uint32_t max_depth, double mis_radius, uint32_t *n_photons);
/* A rank's share of the light phase: paths [path0, path0 + n_paths) of the
 * iteration (RngStream(seed, iteration, path0 + j, kLightStream)), deposits
 * in path order; concatenating the shares of all ranks in rank order gives
 * exactly the single-call photon array. */
int fppm_gpu_trace_photons_range(fppm_gpu_ctx *ctx, uint64_t seed, uint64_t iteration, uint32_t path0,
                                 uint32_t n_paths, uint32_t max_depth, double mis_radius, uint32_t *n_photons);
/* ---- eye pass and film (integrator.cpp:407-474, film.cpp:21-50) ---- */
typedef struct fppm_camera {   /* Camera (scene.hpp:75-82) */
  double position[3];
  double look_at[3];
  double up[3];
  double vfov_deg;
  int32_t width, height;
} fppm_camera;
/* Pinhole camera; width * height <= max_hitpoints.  Clears the film. */
int fppm_gpu_set_camera(fppm_gpu_ctx *ctx, const fppm_camera *camera);
/* Renderer::pixel_pm's camera walk for every pixel (RngStream(seed, iteration,
 * px, kEyeStream)): jittered ray, emitted radiance along the specular chain,
 * and the first non-delta hit as the pixel's hit point (move_to + eye Bsdf;
 * gathered = 0 when the walk ends without one).  Replaces set_hitpoints. */
int fppm_gpu_trace_eye(fppm_gpu_ctx *ctx, uint64_t seed, uint64_t iteration);
/* Copies the current hit points (fppm_hitpoints layout; any field may be
 * NULL) and, after trace_eye, the per-pixel emitted radiance [n][3]. */
int fppm_gpu_get_hitpoints(fppm_gpu_ctx *ctx, fppm_hitpoints *out, double *emitted);
/* Film::add_iteration of this iteration's estimate: emitted + flux / (pi r^2 J)
 * of the gather_test / iterate that followed trace_eye. */
int fppm_gpu_film_add(fppm_gpu_ctx *ctx);
/* One whole VCM+ iteration (Renderer::step with Algorithm::vcm_plus,
 * integrator.cpp:150-228, 236-301, 492-653) on the device: light sub-paths
 * (light_paths = J = samples_per_iteration, depth max_depth - 1, eta_vm of
 * the max live radius) and their camera splats; eye sub-paths with MIS
 * partials, emitter hits, next-event estimation and connections to light
 * sub-path px % J; kernel estimation at every rough eye vertex (the first one
 * accumulates into the pixel's region and is F-tested, the others only add
 * their merge sums); the estimate is added to the film.  Replaces the hit
 * points with the pixels' primary vertices.  Needs a vcm_plus context with
 * max_depth <= 16, set_scene and set_camera.  *n_photons (nullable) receives
 * the light-vertex count.
 * Replaces: Renderer::step for vcm_plus (integrator.cpp:150-228). */
int fppm_gpu_render_vcm(fppm_gpu_ctx *ctx, uint64_t seed, uint64_t iteration, uint32_t light_paths,
                        uint32_t max_depth, uint32_t *n_photons);
/* Film::image(): per-pixel mean over the added iterations ([npix][3] host). */
int fppm_gpu_film_mean(fppm_gpu_ctx *ctx, double *rgb, uint64_t *iterations);
/* Film::vc_total / vm_total (film.hpp:52-53, add_split film.cpp:28-31): the
 * per-pixel cumulative luminance delivered by merges (vm) and by everything
 * else (vc: emitted radiance, next-event estimation, connections, camera
 * splats) over the added iterations ([npix] host arrays, NULL skips). */
int fppm_gpu_film_splits(fppm_gpu_ctx *ctx, double *vc, double *vm);

/* Copies the staged photons' VCM partials (d_vcm, d_vm, cont; photon order)
 * to host arrays of n_photons doubles each (vcm_plus contexts only). */
int fppm_gpu_get_photon_mis(fppm_gpu_ctx *ctx, double *d_vcm, double *d_vm, double *cont);

/* ---- VCM+ merge stage inputs (host arrays) ---- */
/* Eye-vertex MIS partials per hit point (PathVertex::mis d_vcm, d_vm). */
int fppm_gpu_set_hitpoint_mis(fppm_gpu_ctx *ctx, const double *d_vcm, const double *d_vm, uint32_t n);
/* Light-vertex MIS partials and roulette survival per photon (LightVertex::mis
 * d_vcm, d_vm and ::cont, path.hpp:76-89), in the order of the photons passed
 * to fppm_gpu_set_photons; used by the next grid build. */
int fppm_gpu_set_photon_mis(fppm_gpu_ctx *ctx, const double *d_vcm, const double *d_vm,
                            const double *cont, uint32_t n);

/* Cumulative counters of this context: [accepted, candidates, exact, ambiguous]. */
int fppm_gpu_counters(fppm_gpu_ctx *ctx, uint64_t out[4]);
/* Durations (ms, CUDA events on the context stream) of the dominant gather
 * kernel of the gathers issued since the previous call (at most the last 64);
 * waits for them to finish. *n receives the count written to out. */
int fppm_gpu_gather_kernel_ms(fppm_gpu_ctx *ctx, float *out, uint32_t max, uint32_t *n);
/* Sorted-record layout of the current grid (bytes staged per photon by the
 * gather): 64 = general fine records, 48 = lean records (planar gray frames),
 * 32 = flat lean records (lean, and every photon shares one z), 0 = the grid
 * is not built or another gather kernel's layout is in use. Diagnostic. */
int fppm_gpu_record_bytes(const fppm_gpu_ctx *ctx);
/* Kernel launches issued by this library since load (all contexts). */
uint64_t fppm_gpu_kernel_launches(void);

/* ---- free functions (host-side numerics shared with the device tables) ---- */
double fppm_gpu_schedule_radius(double base, double alpha, uint64_t i);
double fppm_gpu_f_quantile(double p, double d1, double d2, int *status);
double fppm_gpu_chi2_quantile(double p, double df, int *status);

#ifdef __cplusplus
}
#endif
#endif /* FPPM_GPU_H */
