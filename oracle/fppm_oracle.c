/*
 * fppm_oracle.c -- TEST INFRASTRUCTURE ONLY (see fppm_oracle.h).
 *
 * Plain-C restatement of the reference hot path.  Compiled with
 * -O2 -ffp-contract=off on x86-64 (no FMA), matching the reference build
 * (0 vfmadd in gather.o/photon_map.o/stat_tests.o).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library, and only as the checker.
 */
#include "fppm_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

static const double kPi = 3.141592653589793;        /* std::numbers::pi */
static const double kInvPi = 0.3183098861837907;    /* std::numbers::inv_pi */
static const double kTwoPi = 2.0 * 3.141592653589793; /* sampling.hpp:11 */

static double dmax(double a, double b) { return (a < b) ? b : a; } /* std::max */
static double dmin(double a, double b) { return (b < a) ? b : a; } /* std::min */

/* ===================================================================== */
/* L0: frame.cpp:5-14 (branchless Duff basis), vec.hpp:79-81 luminance     */
/* ===================================================================== */
void orc_build_frame(const double n[3], double u[3], double v[3]) {
  const double sign = copysign(1.0, n[2]);
  const double a = -1.0 / (sign + n[2]);
  const double b = n[0] * n[1] * a;
  u[0] = 1.0 + sign * n[0] * n[0] * a;
  u[1] = sign * b;
  u[2] = -sign * n[0];
  v[0] = b;
  v[1] = sign + n[1] * n[1] * a;
  v[2] = -n[1];
}

double orc_luminance(double r, double g, double b) {
  return 0.2126 * r + 0.7152 * g + 0.0722 * b;
}

static double dot3(const double a[3], const double b[3]) { /* vec.hpp:463 */
  return a[0] * b[0] + a[1] * b[1] + a[2] * b[2];
}

/* ===================================================================== */
/* L1: special_functions.cpp                                             */
/* ===================================================================== */
#define K_MAX_ITER 500                               /* :7 */
static const double kEps = 2.220446049250313e-16;    /* :8 */
#define K_FPMIN (2.2250738585072014e-308 / 2.220446049250313e-16) /* :9 */

static double gamma_p_series(double a, double x) { /* :12-24 */
  double ap = a, sum = 1.0 / a, del = sum;
  for (int i = 0; i < K_MAX_ITER; ++i) {
    ap += 1.0;
    del *= x / ap;
    sum += del;
    if (fabs(del) < fabs(sum) * kEps) break;
  }
  return sum * exp(-x + a * log(x) - lgamma(a));
}

static double gamma_q_cf(double a, double x) { /* :27-49 */
  double b = x + 1.0 - a;
  double c = 1.0 / K_FPMIN;
  double d = 1.0 / b;
  double h = d;
  for (int i = 1; i <= K_MAX_ITER; ++i) {
    const double an = (double)(-i) * ((double)i - a);
    b += 2.0;
    d = an * d + b;
    if (fabs(d) < K_FPMIN) d = K_FPMIN;
    c = b + an / c;
    if (fabs(c) < K_FPMIN) c = K_FPMIN;
    d = 1.0 / d;
    const double del = d * c;
    h *= del;
    if (fabs(del - 1.0) < kEps) break;
  }
  return h * exp(-x + a * log(x) - lgamma(a));
}

static double beta_cf(double a, double b, double x) { /* :53-83 */
  const double qab = a + b, qap = a + 1.0, qam = a - 1.0;
  double c = 1.0;
  double d = 1.0 - qab * x / qap;
  if (fabs(d) < K_FPMIN) d = K_FPMIN;
  d = 1.0 / d;
  double h = d;
  for (int m = 1; m <= K_MAX_ITER; ++m) {
    const int m2 = 2 * m;
    double aa = (double)m * (b - (double)m) * x / ((qam + (double)m2) * (a + (double)m2));
    d = 1.0 + aa * d;
    if (fabs(d) < K_FPMIN) d = K_FPMIN;
    c = 1.0 + aa / c;
    if (fabs(c) < K_FPMIN) c = K_FPMIN;
    d = 1.0 / d;
    h *= d * c;
    aa = -(a + (double)m) * (qab + (double)m) * x / ((a + (double)m2) * (qap + (double)m2));
    d = 1.0 + aa * d;
    if (fabs(d) < K_FPMIN) d = K_FPMIN;
    c = 1.0 + aa / c;
    if (fabs(c) < K_FPMIN) c = K_FPMIN;
    d = 1.0 / d;
    const double del = d * c;
    h *= del;
    if (fabs(del - 1.0) < kEps) break;
  }
  return h;
}

typedef double (*cdf_fn)(double x, const double *par);

static double invert_cdf(cdf_fn cdf, const double *par, double p, double lo,
                         double hi) { /* :88-102 */
  for (int i = 0; i < 200; ++i) {
    const double mid = 0.5 * (lo + hi);
    if (mid == lo || mid == hi) break;
    if (cdf(mid, par) < p)
      lo = mid;
    else
      hi = mid;
    if (hi - lo <= 1e-15 * dmax(1.0, lo)) break;
  }
  return 0.5 * (lo + hi);
}

double orc_reg_lower_gamma(double a, double x, int *err) { /* :108-114 */
  if (!(a > 0.0) || x < 0.0) { if (err) *err = ORC_INVALID_ARGUMENT; return 0.0; }
  if (x == 0.0) return 0.0;
  return x < a + 1.0 ? gamma_p_series(a, x) : 1.0 - gamma_q_cf(a, x);
}

double orc_reg_inc_beta(double a, double b, double x, int *err) { /* :116-128 */
  if (!(a > 0.0) || !(b > 0.0)) { if (err) *err = ORC_INVALID_ARGUMENT; return 0.0; }
  if (x <= 0.0) return 0.0;
  if (x >= 1.0) return 1.0;
  const double front = exp(lgamma(a + b) - lgamma(a) - lgamma(b) + a * log(x) +
                           b * log1p(-x));
  if (x < (a + 1.0) / (a + b + 2.0)) return front * beta_cf(a, b, x) / a;
  return 1.0 - front * beta_cf(b, a, 1.0 - x) / b;
}

double orc_chi2_cdf(double x, double df, int *err) { /* :130-136 */
  if (!(df > 0.0)) { if (err) *err = ORC_INVALID_ARGUMENT; return 0.0; }
  if (x <= 0.0) return 0.0;
  return orc_reg_lower_gamma(0.5 * df, 0.5 * x, err);
}

static double chi2_cdf_cb(double x, const double *par) {
  return orc_chi2_cdf(x, par[0], NULL);
}

double orc_chi2_quantile(double p, double df, int *err) { /* :138-146 */
  if (!(p > 0.0 && p < 1.0)) { if (err) *err = ORC_INVALID_ARGUMENT; return 0.0; }
  if (!(df > 0.0)) { if (err) *err = ORC_INVALID_ARGUMENT; return 0.0; }
  double hi = df + 10.0 * sqrt(2.0 * df) + 10.0;
  while (orc_chi2_cdf(hi, df, NULL) < p) hi *= 2.0;
  return invert_cdf(chi2_cdf_cb, &df, p, 0.0, hi);
}

static const double kLargeD2 = 2e7; /* :150 */

double orc_f_cdf(double x, double d1, double d2, int *err) { /* :152-160 */
  if (!(d1 > 0.0) || !(d2 > 0.0)) { if (err) *err = ORC_INVALID_ARGUMENT; return 0.0; }
  if (x <= 0.0) return 0.0;
  if (d2 > kLargeD2) return orc_reg_lower_gamma(0.5 * d1, 0.5 * d1 * x, NULL);
  return orc_reg_inc_beta(0.5 * d1, 0.5 * d2, d1 * x / (d1 * x + d2), NULL);
}

static double f_cdf_cb(double x, const double *par) {
  return orc_f_cdf(x, par[0], par[1], NULL);
}

double orc_f_quantile(double p, double d1, double d2, int *err) { /* :162-170 */
  if (!(p > 0.0 && p < 1.0)) { if (err) *err = ORC_INVALID_ARGUMENT; return 0.0; }
  if (!(d1 > 0.0) || !(d2 > 0.0)) { if (err) *err = ORC_INVALID_ARGUMENT; return 0.0; }
  double hi = 16.0;
  while (orc_f_cdf(hi, d1, d2, NULL) < p) hi *= 4.0;
  const double par[2] = {d1, d2};
  return invert_cdf(f_cdf_cb, par, p, 0.0, hi);
}

/* ===================================================================== */
/* L1: stat_tests.cpp                                                    */
/* ===================================================================== */
double orc_f_statistic(const uint64_t *count, const double *sum,
                       const double *sum_sq, int n, uint64_t m, int *err) {
  (void)count; /* :12-44 reads sum/sum_sq only */
  if (n < 2 || m < 2) { if (err) *err = ORC_INVALID_ARGUMENT; return 0.0; }
  const double md = (double)m;
  double grand_sum = 0;
  for (int i = 0; i < n; ++i) grand_sum += sum[i];
  const double grand_mean = grand_sum / (md * (double)n);
  double between = 0, within = 0;
  for (int i = 0; i < n; ++i) {
    const double mean = sum[i] / md;
    const double dev = mean - grand_mean;
    between += md * dev * dev;
    within += sum_sq[i] - sum[i] * sum[i] / md;
  }
  between = dmax(between, 0.0);
  within = dmax(within, 0.0);
  if (between == 0.0) return 0.0;
  if (within == 0.0) return INFINITY;
  const double d1 = (double)(n - 1);
  const double d2 = (double)n * (md - 1.0);
  return (between / d1) / (within / d2);
}

/* Memo like stat_tests.cpp:72-82 (value-identical with or without it). */
#define CRIT_CACHE 256
static __thread struct { int64_t d1, d2; double alpha, value; int used; } crit_cache[CRIT_CACHE];

double orc_f_critical(int64_t d1, int64_t d2, double alpha) {
  uint64_t h = (uint64_t)d1 * 0x9e3779b97f4a7c15ull ^ (uint64_t)d2 * 0xbf58476d1ce4e5b9ull;
  for (int probe = 0; probe < CRIT_CACHE; ++probe) {
    const int slot = (int)((h + (uint64_t)probe) % CRIT_CACHE);
    if (crit_cache[slot].used && crit_cache[slot].d1 == d1 &&
        crit_cache[slot].d2 == d2 && crit_cache[slot].alpha == alpha)
      return crit_cache[slot].value;
    if (!crit_cache[slot].used) {
      const double v = orc_f_quantile(1.0 - alpha, (double)d1, (double)d2, NULL);
      crit_cache[slot].d1 = d1;
      crit_cache[slot].d2 = d2;
      crit_cache[slot].alpha = alpha;
      crit_cache[slot].value = v;
      crit_cache[slot].used = 1;
      return v;
    }
  }
  return orc_f_quantile(1.0 - alpha, (double)d1, (double)d2, NULL);
}

double orc_chi2_statistic(const uint64_t *counts, int n, int *err) { /* :100-116 */
  if (n < 2) { if (err) *err = ORC_INVALID_ARGUMENT; return 0.0; }
  uint64_t total = 0;
  for (int i = 0; i < n; ++i) total += counts[i];
  if (total == 0) { if (err) *err = ORC_INVALID_ARGUMENT; return 0.0; }
  const double expected = (double)total / (double)n;
  double chi2 = 0;
  for (int i = 0; i < n; ++i) {
    const double dev = (double)counts[i] - expected;
    chi2 += dev * dev / expected;
  }
  return chi2;
}

/* ===================================================================== */
/* L2a: gather.cpp                                                       */
/* ===================================================================== */
double orc_schedule_radius(double base, double alpha, uint64_t i) { /* :11-13 */
  return base * sqrt(pow((double)i, alpha - 1.0));
}

int orc_sector_index(double yu, double yv, double radius, int n_annuli,
                     int n_sectors, int *err) { /* :15-33 */
  if (n_annuli < 1 || n_sectors < 1) { if (err) *err = ORC_INVALID_ARGUMENT; return -1; }
  const double r2 = radius * radius;
  const double d2 = yu * yu + yv * yv;
  if (d2 > r2 * (1.0 + 1e-9)) { if (err) *err = ORC_DOMAIN_ERROR; return -1; }
  int a = (int)((double)n_annuli * d2 / r2);
  if (a > n_annuli - 1) a = n_annuli - 1;
  double theta = atan2(yv, yu);
  if (theta < 0.0) theta += kTwoPi;
  int s = (int)((double)n_sectors * theta / kTwoPi);
  if (s > n_sectors - 1) s = n_sectors - 1;
  return a * n_sectors + s;
}

/* ===================================================================== */
/* L2b: photon_map.cpp                                                   */
/* ===================================================================== */
static const int64_t kBias = (int64_t)1 << 20; /* :11 */

int64_t orc_cell_coord(double x, double inv_cell) { /* :13-15 */
  return (int64_t)floor(x * inv_cell);
}

uint64_t orc_cell_key(int64_t ix, int64_t iy, int64_t iz) { /* :19-24 */
  return ((uint64_t)(ix + kBias) << 42) | ((uint64_t)(iy + kBias) << 21) |
         (uint64_t)(iz + kBias);
}

struct orc_grid {
  size_t n;
  double *pos; /* n*3 */
  double cell;
  uint32_t *order;
  uint64_t *keys;
  uint32_t *begin, *end;
  size_t ncells;
};

typedef struct { uint64_t key; uint32_t idx; } keyed_t;

static int keyed_cmp(const void *a, const void *b) { /* std::pair operator< */
  const keyed_t *x = (const keyed_t *)a, *y = (const keyed_t *)b;
  if (x->key != y->key) return x->key < y->key ? -1 : 1;
  return x->idx < y->idx ? -1 : (x->idx > y->idx);
}

orc_grid *orc_grid_build(const double *pos, size_t n, double cell_size, int *err) {
  /* photon_map.cpp:26-51 */
  if (!(cell_size > 0.0)) { if (err) *err = ORC_INVALID_ARGUMENT; return NULL; }
  orc_grid *g = (orc_grid *)calloc(1, sizeof(orc_grid));
  g->n = n;
  g->cell = cell_size;
  g->pos = (double *)malloc(sizeof(double) * 3 * (n ? n : 1));
  if (n) memcpy(g->pos, pos, sizeof(double) * 3 * n);
  const double inv = 1.0 / cell_size;
  keyed_t *kd = (keyed_t *)malloc(sizeof(keyed_t) * (n ? n : 1));
  for (size_t i = 0; i < n; ++i) {
    kd[i].key = orc_cell_key(orc_cell_coord(pos[3 * i], inv),
                             orc_cell_coord(pos[3 * i + 1], inv),
                             orc_cell_coord(pos[3 * i + 2], inv));
    kd[i].idx = (uint32_t)i;
  }
  qsort(kd, n, sizeof(keyed_t), keyed_cmp);
  g->order = (uint32_t *)malloc(sizeof(uint32_t) * (n ? n : 1));
  g->keys = (uint64_t *)malloc(sizeof(uint64_t) * (n ? n : 1));
  g->begin = (uint32_t *)malloc(sizeof(uint32_t) * (n ? n : 1));
  g->end = (uint32_t *)malloc(sizeof(uint32_t) * (n ? n : 1));
  size_t nc = 0;
  for (size_t i = 0; i < n; ++i) {
    g->order[i] = kd[i].idx;
    if (i == 0 || kd[i].key != kd[i - 1].key) {
      g->keys[nc] = kd[i].key;
      g->begin[nc] = (uint32_t)i;
      ++nc;
    }
    g->end[nc - 1] = (uint32_t)(i + 1);
  }
  g->ncells = nc;
  free(kd);
  return g;
}

void orc_grid_free(orc_grid *g) {
  if (!g) return;
  free(g->pos); free(g->order); free(g->keys); free(g->begin); free(g->end);
  free(g);
}

size_t orc_grid_cell_count(const orc_grid *g) { return g->ncells; }

void orc_grid_export(const orc_grid *g, uint64_t *keys, uint32_t *begin,
                     uint32_t *end, uint32_t *order) {
  if (keys) memcpy(keys, g->keys, sizeof(uint64_t) * g->ncells);
  if (begin) memcpy(begin, g->begin, sizeof(uint32_t) * g->ncells);
  if (end) memcpy(end, g->end, sizeof(uint32_t) * g->ncells);
  if (order) memcpy(order, g->order, sizeof(uint32_t) * g->n);
}

static size_t lower_bound_u64(const uint64_t *a, size_t n, uint64_t key) {
  size_t lo = 0, hi = n;
  while (lo < hi) {
    const size_t mid = lo + (hi - lo) / 2;
    if (a[mid] < key) lo = mid + 1; else hi = mid;
  }
  return lo;
}

/* Visit callback form of query_ball (photon_map.cpp:53-78). */
typedef void (*visit_fn)(uint32_t idx, void *user);

static int grid_visit_ball(const orc_grid *g, const double c[3], double r,
                           visit_fn fn, void *user) {
  if (g->n == 0) return ORC_OK;
  if (r > g->cell) return ORC_INVALID_ARGUMENT;
  const double inv = 1.0 / g->cell;
  const double r2 = r * r;
  const int64_t cx = orc_cell_coord(c[0], inv);
  const int64_t cy = orc_cell_coord(c[1], inv);
  const int64_t cz = orc_cell_coord(c[2], inv);
  for (int64_t dx = -1; dx <= 1; ++dx)
    for (int64_t dy = -1; dy <= 1; ++dy)
      for (int64_t dz = -1; dz <= 1; ++dz) {
        const uint64_t key = orc_cell_key(cx + dx, cy + dy, cz + dz);
        const size_t it = lower_bound_u64(g->keys, g->ncells, key);
        if (it == g->ncells || g->keys[it] != key) continue;
        for (uint32_t i = g->begin[it]; i < g->end[it]; ++i) {
          const uint32_t v = g->order[i];
          const double *p = g->pos + 3 * (size_t)v;
          const double d[3] = {p[0] - c[0], p[1] - c[1], p[2] - c[2]};
          if (dot3(d, d) <= r2) fn(v, user);
        }
      }
  return ORC_OK;
}

typedef struct { uint32_t *out; size_t cap, n; } collect_t;
static void collect_cb(uint32_t idx, void *user) {
  collect_t *c = (collect_t *)user;
  if (c->n < c->cap) c->out[c->n] = idx;
  c->n++;
}

size_t orc_grid_query_ball(const orc_grid *g, const double c[3], double r,
                           uint32_t *out, size_t cap, int *err) {
  collect_t col = {out, cap, 0};
  const int rc = grid_visit_ball(g, c, r, collect_cb, &col);
  if (rc && err) *err = rc;
  return col.n;
}

/* ===================================================================== */
/* FPPM session: Renderer::step restricted to the gather path            */
/* ===================================================================== */
typedef struct {
  double radius, initial_radius;
  uint64_t t;
  double center[3], n[3], u[3], v[3]; /* TangentFrame (frame.hpp:8-19) */
  uint64_t *count;                    /* [C][G] */
  double *sum, *sum_sq;
} region_t;

struct orc_session {
  orc_config cfg;
  size_t H;
  int G, C;
  double *pos, *nrm, *wo, *thr, *alb;
  uint32_t *eye_depth;
  uint8_t *gathered;
  region_t *reg;
  uint64_t *stat_count;
  double *stat_sum, *stat_sum_sq;
  double *eye_d_vcm, *eye_d_vm;                           /* VCM+ (per hit point) */
  const double *ph_d_vcm, *ph_d_vm, *ph_cont;             /* VCM+ (per photon) */
};

/* path.cpp:11-13 */
static double mis_pow(double beta, double x) { return beta == 1.0 ? x : pow(x, beta); }

/* path.cpp:103-111 with vc_factor (path.cpp:22-24) of eta_vm = n_vm pi r^2
 * (integrator.cpp:503, evaluated left to right) */
double orc_mis_weight_merge(int n_vm, double beta, double r, double eye_d_vcm, double eye_d_vm,
                            double light_d_vcm, double light_d_vm, double bsdf_fwd_pdf_w,
                            double bsdf_rev_pdf_w) {
  const double eta_vm = (double)n_vm * kPi * r * r;
  const double vcf = eta_vm > 0.0 ? mis_pow(beta, 1.0 / eta_vm) : 0.0;
  const double w_light = light_d_vcm * vcf + light_d_vm * mis_pow(beta, bsdf_fwd_pdf_w);
  const double w_camera = eye_d_vcm * vcf + eye_d_vm * mis_pow(beta, bsdf_rev_pdf_w);
  return 1.0 / (w_light + 1.0 + w_camera);
}

void orc_session_set_eye_mis(orc_session *s, const double *d_vcm, const double *d_vm) {
  for (size_t h = 0; h < s->H; ++h) {
    s->eye_d_vcm[h] = d_vcm ? d_vcm[h] : 0.0;
    s->eye_d_vm[h] = d_vm ? d_vm[h] : 0.0;
  }
}

void orc_session_set_photon_mis(orc_session *s, const double *d_vcm, const double *d_vm,
                                const double *cont, size_t n) {
  (void)n;
  s->ph_d_vcm = d_vcm;
  s->ph_d_vm = d_vm;
  s->ph_cont = cont;
}

orc_session *orc_session_create(const orc_config *cfg, size_t H,
                                const double *pos, const double *nrm,
                                const double *wo, const double *thr,
                                const double *alb, const uint32_t *eye_depth,
                                const uint8_t *gathered, int *err) {
  /* GatherRegion ctor validation: gather.cpp:35-52 */
  const double r0 = cfg->initial_radius;
  if (!(r0 > 0) || !(cfg->k > 0 && cfg->k < 1) ||
      !(cfg->alpha >= 0.5 && cfg->alpha < 1) ||
      !(cfg->r_min_base > 0 && cfg->r_min_base <= r0) ||
      cfg->n_annuli * cfg->n_sectors < 2 || cfg->n_annuli < 1 || cfg->n_sectors < 1 ||
      !(cfg->channels == 1 || cfg->channels == 3)) {
    if (err) *err = ORC_INVALID_ARGUMENT;
    return NULL;
  }
  orc_session *s = (orc_session *)calloc(1, sizeof(orc_session));
  s->cfg = *cfg;
  s->H = H;
  s->G = cfg->n_annuli * cfg->n_sectors;
  s->C = cfg->channels;
  const size_t b3 = sizeof(double) * 3 * (H ? H : 1);
  s->pos = (double *)malloc(b3); s->nrm = (double *)malloc(b3);
  s->wo = (double *)malloc(b3); s->thr = (double *)malloc(b3);
  s->alb = (double *)malloc(b3);
  memcpy(s->pos, pos, sizeof(double) * 3 * H);
  memcpy(s->nrm, nrm, sizeof(double) * 3 * H);
  memcpy(s->wo, wo, sizeof(double) * 3 * H);
  memcpy(s->thr, thr, sizeof(double) * 3 * H);
  memcpy(s->alb, alb, sizeof(double) * 3 * H);
  s->eye_depth = (uint32_t *)malloc(sizeof(uint32_t) * (H ? H : 1));
  memcpy(s->eye_depth, eye_depth, sizeof(uint32_t) * H);
  s->gathered = (uint8_t *)malloc(H ? H : 1);
  if (gathered) memcpy(s->gathered, gathered, H); else memset(s->gathered, 1, H);
  const size_t cg = (size_t)s->G * (size_t)s->C;
  s->stat_count = (uint64_t *)calloc(cg * (H ? H : 1), sizeof(uint64_t));
  s->stat_sum = (double *)calloc(cg * (H ? H : 1), sizeof(double));
  s->stat_sum_sq = (double *)calloc(cg * (H ? H : 1), sizeof(double));
  s->reg = (region_t *)calloc(H ? H : 1, sizeof(region_t));
  s->eye_d_vcm = (double *)calloc(H ? H : 1, sizeof(double));
  s->eye_d_vm = (double *)calloc(H ? H : 1, sizeof(double));
  for (size_t h = 0; h < H; ++h) {
    s->reg[h].radius = r0;
    s->reg[h].initial_radius = r0;
    s->reg[h].t = 1;
    s->reg[h].count = s->stat_count + cg * h;
    s->reg[h].sum = s->stat_sum + cg * h;
    s->reg[h].sum_sq = s->stat_sum_sq + cg * h;
  }
  return s;
}

/* move_to with new hit points (integrator.cpp:433-440): the eye pass of every
 * iteration moves each region's center; radius, t and stats stay. */
void orc_session_set_hitpoints(orc_session *s, const double *pos, const double *nrm, const double *wo,
                               const double *thr, const double *alb, const uint32_t *eye_depth,
                               const uint8_t *gathered) {
  const size_t H = s->H;
  memcpy(s->pos, pos, sizeof(double) * 3 * H);
  memcpy(s->nrm, nrm, sizeof(double) * 3 * H);
  memcpy(s->wo, wo, sizeof(double) * 3 * H);
  memcpy(s->thr, thr, sizeof(double) * 3 * H);
  memcpy(s->alb, alb, sizeof(double) * 3 * H);
  memcpy(s->eye_depth, eye_depth, sizeof(uint32_t) * H);
  if (gathered) memcpy(s->gathered, gathered, H); else memset(s->gathered, 1, H);
}

void orc_session_free(orc_session *s) {
  if (!s) return;
  free(s->pos); free(s->nrm); free(s->wo); free(s->thr); free(s->alb);
  free(s->eye_depth); free(s->gathered);
  free(s->stat_count); free(s->stat_sum); free(s->stat_sum_sq); free(s->reg);
  free(s->eye_d_vcm); free(s->eye_d_vm);
  free(s);
}

double orc_session_max_radius(const orc_session *s) { /* integrator.cpp:159-161 */
  double r = 0.0;
  for (size_t h = 0; h < s->H; ++h) r = dmax(r, s->reg[h].radius);
  return r;
}

typedef struct {
  const orc_session *s;
  region_t *reg;
  size_t h;
  const float *ppos, *pnrm, *pwi, *ppow;
  const uint32_t *pdepth;
  double r, r2;
  double K[3];     /* throughput * albedo/pi (cos_o > 0), else throughput*0 */
  double Kzero[3]; /* throughput * 0 (bsdf.cpp:58: cos_i <= 0 -> Rgb()) */
  double sum[3];
  uint64_t accepted;
  int err;
  /* VCM+: eye cos_o, continuation probability and MIS partials */
  double cos_o, cont, e_vcm, e_vm;
} gather_ctx;

static void gather_cb(uint32_t id, void *user) {
  /* integrator.cpp:394-401 (gather_disk loop body) + :445-451 (callback) */
  gather_ctx *g = (gather_ctx *)user;
  const orc_config *cfg = &g->s->cfg;
  const double p[3] = {g->ppos[3 * id], g->ppos[3 * id + 1], g->ppos[3 * id + 2]};
  const double pn[3] = {g->pnrm[3 * id], g->pnrm[3 * id + 1], g->pnrm[3 * id + 2]};
  const uint32_t eye_depth = g->s->eye_depth[g->h];
  if (eye_depth + g->pdepth[id] > cfg->max_depth) return;          /* :396 */
  if (dot3(pn, g->reg->n) < cfg->normal_guard_cos) return;          /* :397 */
  const double d[3] = {p[0] - g->reg->center[0], p[1] - g->reg->center[1],
                       p[2] - g->reg->center[2]};                    /* frame.hpp:32-36 */
  const double yu = dot3(d, g->reg->u), yv = dot3(d, g->reg->v);
  if (yu * yu + yv * yv > g->r2) return;                            /* :399 */
  /* Bsdf::eval Lambertian (bsdf.cpp:53-63) with frame_.n = shading normal */
  const double wi[3] = {g->pwi[3 * id], g->pwi[3 * id + 1], g->pwi[3 * id + 2]};
  const double cos_i = dot3(wi, g->reg->n);
  const double *k = cos_i <= 0.0 ? g->Kzero : g->K;
  double val[3] = {k[0] * (double)g->ppow[3 * id], k[1] * (double)g->ppow[3 * id + 1],
                   k[2] * (double)g->ppow[3 * id + 2]};
  if (cfg->vcm_plus) {
    /* integrator.cpp:612-616: f, pf, pr of Bsdf::eval (bsdf.cpp:53-63, pdfs
     * zero when the value is black), merge weight, val = thr * f * p.thr * w */
    const int black = g->cos_o <= 0.0 || cos_i <= 0.0;
    const double pf = black ? 0.0 : (cos_i > 0 ? cos_i * kInvPi : 0.0);
    const double pr = black ? 0.0 : (g->cos_o > 0 ? g->cos_o * kInvPi : 0.0);
    const double w = orc_mis_weight_merge(cfg->mis_n_vm, cfg->mis_beta, g->r, g->e_vcm, g->e_vm,
                                          g->s->ph_d_vcm[id], g->s->ph_d_vm[id], pf * g->cont,
                                          pr * g->s->ph_cont[id]);
    val[0] = val[0] * w;
    val[1] = val[1] * w;
    val[2] = val[2] * w;
  }
  g->sum[0] += val[0]; g->sum[1] += val[1]; g->sum[2] += val[2];
  g->accepted++;
  /* GatherRegion::accumulate (gather.cpp:59-67) */
  int err = 0;
  const int sector = orc_sector_index(yu, yv, g->reg->radius, cfg->n_annuli,
                                      cfg->n_sectors, &err);
  if (err) { g->err = err; return; }
  const int G = g->s->G;
  if (g->s->C == 1) {
    const double v = orc_luminance(val[0], val[1], val[2]);
    g->reg->count[sector]++;            /* SectorStats::add stat_tests.hpp:18-22 */
    g->reg->sum[sector] += v;
    g->reg->sum_sq[sector] += v * v;
  } else {
    for (int c = 0; c < 3; ++c) {
      g->reg->count[c * G + sector]++;
      g->reg->sum[c * G + sector] += val[c];
      g->reg->sum_sq[c * G + sector] += val[c] * val[c];
    }
  }
}

typedef struct {
  orc_session *s;
  const orc_grid *grid;
  uint64_t iteration;
  const float *ppos, *pnrm, *pwi, *ppow;
  const uint32_t *pdepth;
  const uint32_t *subset;
  size_t begin, end;
  orc_iter_out *out;
  int err;
} worker_t;

static void process_hit(worker_t *w, size_t slot) {
  orc_session *s = w->s;
  const orc_config *cfg = &s->cfg;
  const size_t h = w->subset ? w->subset[slot] : slot;
  region_t *reg = &s->reg[h];
  const int CG = s->G * s->C;
  orc_iter_out *o = w->out;
  const double r = reg->radius; /* integrator.cpp:411 */
  if (o && o->gather_r) o->gather_r[slot] = r;
  double flux[3] = {0, 0, 0};
  uint64_t accepted = 0;
  int gathered = s->gathered[h];
  if (gathered) {
    /* region->move_to (gather.cpp:54-57) */
    memcpy(reg->center, s->pos + 3 * h, sizeof(double) * 3);
    memcpy(reg->n, s->nrm + 3 * h, sizeof(double) * 3);
    orc_build_frame(reg->n, reg->u, reg->v);
    gather_ctx g;
    memset(&g, 0, sizeof(g));
    g.s = s; g.reg = reg; g.h = h;
    g.ppos = w->ppos; g.pnrm = w->pnrm; g.pwi = w->pwi; g.ppow = w->ppow; g.pdepth = w->pdepth;
    g.r = r; g.r2 = r * r;
    const double *thr = s->thr + 3 * h, *alb = s->alb + 3 * h;
    const double cos_o = dot3(s->wo + 3 * h, reg->n); /* bsdf.cpp:34 */
    g.cos_o = cos_o;
    {
      /* bsdf.cpp:42-51 (Lambertian): min(1, albedo.max_component()),
       * std::max / std::min semantics (vec.hpp:73) */
      const double *a = s->alb + 3 * h;
      const double m1 = a[1] < a[2] ? a[2] : a[1];
      const double amax = a[0] < m1 ? m1 : a[0];
      g.cont = amax < 1.0 ? amax : 1.0;
    }
    g.e_vcm = s->eye_d_vcm[h];
    g.e_vm = s->eye_d_vm[h];
    for (int c = 0; c < 3; ++c) {
      const double f = cos_o <= 0.0 ? 0.0 : alb[c] * kInvPi; /* bsdf.cpp:58,63 */
      g.K[c] = thr[c] * f;                                  /* integrator.cpp:448 */
      g.Kzero[c] = thr[c] * 0.0;
    }
    const int rc = grid_visit_ball(w->grid, reg->center, r, gather_cb, &g);
    if (rc) { w->err = rc; return; }
    if (g.err) { w->err = g.err; return; }
    flux[0] = g.sum[0]; flux[1] = g.sum[1]; flux[2] = g.sum[2];
    accepted = g.accepted;
  }
  if (o && o->flux) { o->flux[3 * slot] = flux[0]; o->flux[3 * slot + 1] = flux[1]; o->flux[3 * slot + 2] = flux[2]; }
  if (o && o->radiance) {
    const double denom = kPi * r * r * (double)cfg->samples_per_iteration; /* :452-453 */
    for (int c = 0; c < 3; ++c) o->radiance[3 * slot + c] = gathered ? flux[c] / denom : 0.0;
  }
  if (o && o->accepted) o->accepted[slot] = accepted;
  if (o && o->stat_count) memcpy(o->stat_count + (size_t)CG * slot, reg->count, sizeof(uint64_t) * CG);
  if (o && o->stat_sum) memcpy(o->stat_sum + (size_t)CG * slot, reg->sum, sizeof(double) * CG);
  if (o && o->stat_sum_sq) memcpy(o->stat_sum_sq + (size_t)CG * slot, reg->sum_sq, sizeof(double) * CG);

  /* end_iteration (gather.cpp:90-112) + apply_decision (:74-88), or hold
   * without observation (integrator.cpp:483-488). */
  int tested = 0, rejected = 0;
  double stat = 0, critical = 0;
  if (cfg->policy == 2) {
    /* schedule_end_iteration (gather.cpp:138-144) for every region, gathered
     * or not: the global SPPM / VCM radius (integrator.cpp:159-164, 213-217) */
    reg->radius = orc_schedule_radius(reg->initial_radius, cfg->alpha, w->iteration + 1);
    ++reg->t;
  } else if (gathered) {
    int decide = 0;
    if (cfg->override_decision != 0) {
      rejected = cfg->override_decision == 1;
      decide = 1;
    } else if (cfg->policy == 1) {
      /* chi2_end_iteration (gather.cpp:114-136): channel-0 counts only */
      uint64_t total = 0;
      for (int g = 0; g < s->G; ++g) total += reg->count[g];
      if (total == 0) {
        rejected = 0;
      } else {
        critical = orc_chi2_quantile(1.0 - cfg->alpha_chi2, (double)(s->G - 1), NULL);
        stat = orc_chi2_statistic(reg->count, s->G, NULL);
        rejected = stat > critical;
        tested = 1;
      }
      decide = 1;
    } else {
      const uint64_t m = reg->t * cfg->samples_per_iteration;
      if (m < 2) {
        rejected = 0;
        decide = 1;
      } else {
        int reject = 0;
        for (int c = 0; c < s->C; ++c) {
          const double f = orc_f_statistic(reg->count + c * s->G, reg->sum + c * s->G,
                                           reg->sum_sq + c * s->G, s->G, m, NULL);
          const int64_t d1 = (int64_t)s->G - 1;
          const int64_t d2 = (int64_t)s->G * (int64_t)(m - 1);
          const double crit = orc_f_critical(d1, d2, cfg->alpha_f);
          reject = reject || (f > crit);
          stat = dmax(stat, f);
          critical = crit;
        }
        rejected = reject;
        tested = 1;
        decide = 1;
      }
    }
    if (decide) {
      if (rejected) {
        reg->radius = dmax(cfg->k * reg->radius,
                           orc_schedule_radius(cfg->r_min_base, cfg->alpha, w->iteration + 1));
        memset(reg->count, 0, sizeof(uint64_t) * CG);
        memset(reg->sum, 0, sizeof(double) * CG);
        memset(reg->sum_sq, 0, sizeof(double) * CG);
        reg->t = 1;
      } else {
        ++reg->t;
      }
    }
  }
  if (o && o->radius) o->radius[slot] = reg->radius;
  if (o && o->t) o->t[slot] = reg->t;
  if (o && o->tested) o->tested[slot] = (uint8_t)tested;
  if (o && o->rejected) o->rejected[slot] = (uint8_t)rejected;
  if (o && o->statistic) o->statistic[slot] = stat;
  if (o && o->critical) o->critical[slot] = critical;
}

static void *worker_main(void *arg) {
  worker_t *w = (worker_t *)arg;
  for (size_t i = w->begin; i < w->end && !w->err; ++i) process_hit(w, i);
  return NULL;
}

int orc_session_iterate(orc_session *s, uint64_t iteration,
                        const float *ppos, const float *pnrm, const float *pwi,
                        const float *ppow, const uint32_t *pdepth, size_t N,
                        double cell_size, const uint32_t *subset, size_t nsub,
                        orc_iter_out *out) {
  const double cell = cell_size > 0 ? cell_size : orc_session_max_radius(s);
  double *pd = (double *)malloc(sizeof(double) * 3 * (N ? N : 1));
  for (size_t i = 0; i < 3 * N; ++i) pd[i] = (double)ppos[i];
  int err = 0;
  orc_grid *grid = orc_grid_build(pd, N, cell, &err); /* integrator.cpp:262-264 */
  free(pd);
  if (!grid) return err;
  const size_t count = subset ? nsub : s->H;
  /* parallel_ranges static split (integrator.cpp:55-70) */
  int T = s->cfg.threads > 0 ? s->cfg.threads : 1;
  if ((size_t)T > count) T = count ? (int)count : 1;
  worker_t *ws = (worker_t *)calloc((size_t)T, sizeof(worker_t));
  pthread_t *th = (pthread_t *)calloc((size_t)T, sizeof(pthread_t));
  for (int t = 0; t < T; ++t) {
    ws[t].s = s; ws[t].grid = grid; ws[t].iteration = iteration;
    ws[t].ppos = ppos; ws[t].pnrm = pnrm; ws[t].pwi = pwi; ws[t].ppow = ppow;
    ws[t].pdepth = pdepth; ws[t].subset = subset; ws[t].out = out;
    ws[t].begin = count * (size_t)t / (size_t)T;
    ws[t].end = count * (size_t)(t + 1) / (size_t)T;
  }
  for (int t = 1; t < T; ++t) pthread_create(&th[t], NULL, worker_main, &ws[t]);
  worker_main(&ws[0]);
  for (int t = 1; t < T; ++t) pthread_join(th[t], NULL);
  int rc = 0;
  for (int t = 0; t < T; ++t) if (ws[t].err) rc = ws[t].err;
  free(ws); free(th);
  orc_grid_free(grid);
  return rc;
}

/* ===================================================================== */
/* Canonical synthetic inputs -- oracle copy.             */
/* Only IEEE-exact operations (+,-,*,/,sqrt, integer) so that the GPU     */
/* generator and this one agree bit for bit.                             */
/* ===================================================================== */
static uint64_t mix64(uint64_t z) { /* splitmix64 finaliser */
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

#define PCG_MULT 6364136223846793005ull

static uint64_t pcg_advance(uint64_t state, uint64_t delta, uint64_t inc) {
  uint64_t cur_mult = PCG_MULT, cur_plus = inc, acc_mult = 1, acc_plus = 0;
  while (delta > 0) {
    if (delta & 1) {
      acc_mult *= cur_mult;
      acc_plus = acc_plus * cur_mult + cur_plus;
    }
    cur_plus = (cur_mult + 1) * cur_plus;
    cur_mult *= cur_mult;
    delta >>= 1;
  }
  return acc_mult * state + acc_plus;
}

static uint32_t pcg_output(uint64_t old) {
  const uint32_t xorshifted = (uint32_t)(((old >> 18) ^ old) >> 27);
  const uint32_t rot = (uint32_t)(old >> 59);
  return (xorshifted >> rot) | (xorshifted << ((32u - rot) & 31u));
}

static uint64_t pcg_seed_state(uint64_t seed, uint64_t inc) { /* pcg32_srandom */
  uint64_t st = 0;
  st = st * PCG_MULT + inc;
  st += seed;
  st = st * PCG_MULT + inc;
  return st;
}

uint32_t orc_pcg32_at(uint64_t seed, uint64_t stream, uint64_t offset) {
  const uint64_t inc = (stream << 1) | 1u;
  return pcg_output(pcg_advance(pcg_seed_state(seed, inc), offset, inc));
}

static uint64_t stream_id(uint64_t iteration, uint64_t kind) {
  return mix64(iteration + 0x9e3779b97f4a7c15ull * (kind + 1));
}

static float u24(uint32_t x) { return (float)(x >> 8) * 0x1p-24f; }
static double uopen(uint32_t x) { return ((double)x + 0.5) * 0x1p-32; }

void orc_dm_sincos2pi(double u, double *sn, double *cs) {
  const double q = floor(u * 4.0 + 0.5);
  const double x = u - q * 0.25;
  const double t = x * 0x1.921fb54442d18p+2;
  const double z = t * t;
  const double sp =
      -0x1.5555555555555p-3 + z * (0x1.1111111111111p-7 + z * (-0x1.a01a01a01a01ap-13 +
      z * (0x1.71de3a556c734p-19 + z * (-0x1.ae64567f544e4p-26 + z * (0x1.6124613a86d09p-33 +
      z * (-0x1.ae7f3e733b81fp-41 + z * 0x1.952c77030ad4ap-49))))));
  const double s = t + t * (z * sp);
  const double cp =
      0x1.5555555555555p-5 + z * (-0x1.6c16c16c16c17p-10 + z * (0x1.a01a01a01a01ap-16 +
      z * (-0x1.27e4fb7789f5cp-22 + z * (0x1.1eed8eff8d898p-29 + z * (-0x1.93974a8c07c9dp-37 +
      z * (0x1.ae7f3e733b81fp-45 + z * -0x1.6827863b97d97p-53))))));
  const double c = 1.0 + (z * -0.5 + z * (z * cp));
  const int qi = ((int)q) & 3;
  switch (qi) {
    case 0: *sn = s; *cs = c; break;
    case 1: *sn = c; *cs = -s; break;
    case 2: *sn = -s; *cs = -c; break;
    default: *sn = -c; *cs = s; break;
  }
}

double orc_dm_log(double x) {
  uint64_t bits;
  memcpy(&bits, &x, 8);
  int e = (int)((bits >> 52) & 0x7ff) - 1023;
  const uint64_t mb = (bits & 0x000fffffffffffffull) | 0x3ff0000000000000ull;
  double m;
  memcpy(&m, &mb, 8);
  if (m > 0x1.6a09e667f3bcdp+0) { m = m * 0.5; e += 1; }
  const double f = (m - 1.0) / (m + 1.0);
  const double s = f * f;
  const double p =
      0x1.5555555555555p-1 + s * (0x1.999999999999ap-2 + s * (0x1.2492492492492p-2 +
      s * (0x1.c71c71c71c71cp-3 + s * (0x1.745d1745d1746p-3 + s * (0x1.3b13b13b13b14p-3 +
      s * (0x1.1111111111111p-3 + s * (0x1.e1e1e1e1e1e1ep-4 + s * (0x1.af286bca1af28p-4 +
      s * (0x1.8618618618618p-4 + s * (0x1.642c8590b2164p-4 + s * (0x1.47ae147ae147bp-4 +
      s * 0x1.2f684bda12f68p-4)))))))))));
  const double lm = (f + f) + f * (s * p);
  const double ed = (double)e;
  return ed * 0x1.62e42fee00000p-1 + (ed * 0x1.a39ef35793c76p-33 + lm);
}

double orc_dm_exp(double x) {
  const double k = floor(x * 0x1.71547652b82fep+0 + 0.5);
  const double r = (x - k * 0x1.62e42fee00000p-1) - k * 0x1.a39ef35793c76p-33;
  const double p =
      0x1.0000000000000p-1 + r * (0x1.5555555555555p-3 + r * (0x1.5555555555555p-5 +
      r * (0x1.1111111111111p-7 + r * (0x1.6c16c16c16c17p-10 + r * (0x1.a01a01a01a01ap-13 +
      r * (0x1.a01a01a01a01ap-16 + r * (0x1.71de3a556c734p-19 + r * (0x1.27e4fb7789f5cp-22 +
      r * (0x1.ae64567f544e4p-26 + r * (0x1.1eed8eff8d898p-29 + r * (0x1.6124613a86d09p-33 +
      r * 0x1.93974a8c07c9dp-37)))))))))));
  const double er = 1.0 + (r + r * (r * p));
  const uint64_t sb = (uint64_t)((int64_t)k + 1023) << 52;
  double scale;
  memcpy(&scale, &sb, 8);
  return er * scale;
}

#define DRAWS_PER_PHOTON 16u
#define SEED_KIND_PHOTON 0u

void orc_gen_photons(int workload, uint64_t seed, uint64_t iteration,
                     uint64_t begin, uint64_t count, float *pos, float *nrm,
                     float *wi, float *pow_, uint32_t *depth) {
  const uint64_t stream = stream_id(iteration, SEED_KIND_PHOTON);
  const uint64_t inc = (stream << 1) | 1u;
  const uint64_t st0 = pcg_seed_state(seed, inc);
  for (uint64_t k = 0; k < count; ++k) {
    const uint64_t j = begin + k;
    uint64_t st = pcg_advance(st0, j * DRAWS_PER_PHOTON, inc);
    uint32_t d[DRAWS_PER_PHOTON];
    for (unsigned i = 0; i < DRAWS_PER_PHOTON; ++i) {
      d[i] = pcg_output(st);
      st = st * PCG_MULT + inc;
    }
    double x, y;
    unsigned wdraw, pdraw;
    if (workload == ORC_WL_C1) {
      x = (double)u24(d[0]);
      y = (double)u24(d[1]);
      pdraw = 2; wdraw = 5;
    } else { /* ORC_WL_C2 */
      if (u24(d[0]) < 0.7f) {
        const double xs = (double)u24(d[2]);
        x = u24(d[1]) < (float)(10.0 / 11.0) ? 0.5 + 0.5 * xs : 0.5 * xs;
        y = (double)u24(d[3]);
      } else {
        const double rad = sqrt(-2.0 * orc_dm_log(uopen(d[4])));
        double sn, cs;
        orc_dm_sincos2pi((double)u24(d[5]), &sn, &cs);
        x = 0.3 + 0.03 * (rad * cs);
        y = 0.7 + 0.03 * (rad * sn);
      }
      pdraw = 6; wdraw = 9;
    }
    pos[3 * k] = (float)x;
    pos[3 * k + 1] = (float)y;
    pos[3 * k + 2] = 0.0f;
    nrm[3 * k] = 0.0f; nrm[3 * k + 1] = 0.0f; nrm[3 * k + 2] = 1.0f;
    pow_[3 * k] = u24(d[pdraw]);
    pow_[3 * k + 1] = u24(d[pdraw + 1]);
    pow_[3 * k + 2] = u24(d[pdraw + 2]);
    /* cosine-distributed about +z (sampling.hpp:15-19 convention) */
    const double u1 = (double)u24(d[wdraw]);
    double sn, cs;
    orc_dm_sincos2pi((double)u24(d[wdraw + 1]), &sn, &cs);
    const double r = sqrt(u1);
    wi[3 * k] = (float)(r * cs);
    wi[3 * k + 1] = (float)(r * sn);
    wi[3 * k + 2] = (float)sqrt(dmax(0.0, 1.0 - u1));
    depth[k] = 1;
  }
}

void orc_gen_raster_hitpoints(uint32_t W, double *pos, double *nrm, double *wo,
                              double *thr, double *alb, uint32_t *eye_depth) {
  for (uint32_t j = 0; j < W; ++j)
    for (uint32_t i = 0; i < W; ++i) {
      const size_t h = (size_t)j * W + i;
      pos[3 * h] = (double)(float)(((double)i + 0.5) / (double)W);
      pos[3 * h + 1] = (double)(float)(((double)j + 0.5) / (double)W);
      pos[3 * h + 2] = 0.0;
      nrm[3 * h] = 0.0; nrm[3 * h + 1] = 0.0; nrm[3 * h + 2] = 1.0;
      wo[3 * h] = 0.0; wo[3 * h + 1] = 0.0; wo[3 * h + 2] = 1.0;
      thr[3 * h] = thr[3 * h + 1] = thr[3 * h + 2] = 1.0;
      alb[3 * h] = alb[3 * h + 1] = alb[3 * h + 2] = 1.0;
      eye_depth[h] = 1;
    }
}


/* ---------------------------------------------------------------- C5
 * BASELINE configs[4] workload generator (same draws and operation order as
 * generate.cu's C5 kernels): hit points uniform in the unit cube with uniform
 * random normals; photons from 64 Gaussian clusters (sigma 0.01 * 5^u,
 * Dirichlet(1) weights) + 20 % uniform, rejected (up to 8 attempts) unless
 * within 0.05 of the tangent plane of the nearest hit point, whose normal is
 * the deposit normal; wi cosine-distributed about it. */
#define C5_CLUSTERS 64
#define C5_ATTEMPTS 8

struct orc_c5 {
  uint64_t seed;
  uint32_t H;
  int G;
  double cl[5 * C5_CLUSTERS];
  double *pos, *nrm;
  uint32_t *start, *items;
};

static void c5_draws(uint64_t seed, uint64_t iteration, uint64_t kind, uint64_t idx, uint32_t *d, int n) {
  const uint64_t stream = stream_id(iteration, kind);
  const uint64_t inc = (stream << 1) | 1u;
  uint64_t st = pcg_advance(pcg_seed_state(seed, inc), idx * DRAWS_PER_PHOTON, inc);
  for (int i = 0; i < n; ++i) {
    d[i] = pcg_output(st);
    st = st * PCG_MULT + inc;
  }
}

static int c5_cell(double x, int G) {
  const double f = floor(x * (double)G);
  return f < 0.0 ? 0 : (f > (double)(G - 1) ? G - 1 : (int)f);
}

orc_c5 *orc_c5_create(uint64_t seed, uint32_t H) {
  orc_c5 *c = (orc_c5 *)calloc(1, sizeof(orc_c5));
  c->seed = seed;
  c->H = H;
  int G = 1;
  while ((uint64_t)(G + 1) * (G + 1) * (G + 1) * 2u <= H) ++G;
  c->G = G;
  double w[C5_CLUSTERS], total = 0.0;
  for (int k = 0; k < C5_CLUSTERS; ++k) {
    uint32_t d[5];
    c5_draws(seed, 0, 3, (uint64_t)k, d, 5);
    c->cl[5 * k] = (double)u24(d[0]);
    c->cl[5 * k + 1] = (double)u24(d[1]);
    c->cl[5 * k + 2] = (double)u24(d[2]);
    c->cl[5 * k + 3] = 0.01 * orc_dm_exp((double)u24(d[3]) * 0x1.9c041f7ed8d33p+0);
    w[k] = -orc_dm_log(uopen(d[4]));
    total = total + w[k];
  }
  double run = 0.0;
  for (int k = 0; k < C5_CLUSTERS; ++k) {
    run = run + w[k];
    c->cl[5 * k + 4] = run / total;
  }
  c->pos = (double *)malloc(sizeof(double) * 3 * (H ? H : 1));
  c->nrm = (double *)malloc(sizeof(double) * 3 * (H ? H : 1));
  for (uint32_t h = 0; h < H; ++h) {
    uint32_t d[5];
    c5_draws(seed, 0, 2, h, d, 5);
    c->pos[3 * h] = (double)u24(d[0]);
    c->pos[3 * h + 1] = (double)u24(d[1]);
    c->pos[3 * h + 2] = (double)u24(d[2]);
    const double z = 1.0 - 2.0 * (double)u24(d[3]);
    const double q = 1.0 - z * z;
    const double r = sqrt(q > 0.0 ? q : 0.0);
    double sn, cs;
    orc_dm_sincos2pi((double)u24(d[4]), &sn, &cs);
    c->nrm[3 * h] = r * cs;
    c->nrm[3 * h + 1] = r * sn;
    c->nrm[3 * h + 2] = z;
  }
  const size_t nc = (size_t)G * G * G;
  c->start = (uint32_t *)calloc(nc + 1, sizeof(uint32_t));
  c->items = (uint32_t *)malloc(sizeof(uint32_t) * (H ? H : 1));
  uint32_t *cell = (uint32_t *)malloc(sizeof(uint32_t) * (H ? H : 1));
  for (uint32_t h = 0; h < H; ++h) {
    cell[h] = ((uint32_t)c5_cell(c->pos[3 * h + 2], G) * (uint32_t)G + (uint32_t)c5_cell(c->pos[3 * h + 1], G)) *
                  (uint32_t)G + (uint32_t)c5_cell(c->pos[3 * h], G);
    c->start[cell[h] + 1]++;
  }
  for (size_t i = 0; i < nc; ++i) c->start[i + 1] += c->start[i];
  uint32_t *fill = (uint32_t *)calloc(nc ? nc : 1, sizeof(uint32_t));
  for (uint32_t h = 0; h < H; ++h) c->items[c->start[cell[h]] + fill[cell[h]]++] = h;
  free(fill);
  free(cell);
  return c;
}

void orc_c5_free(orc_c5 *c) {
  if (!c) return;
  free(c->pos); free(c->nrm); free(c->start); free(c->items);
  free(c);
}

static uint32_t c5_nearest(const orc_c5 *C, double px, double py, double pz) {
  const int G = C->G;
  const int cx = c5_cell(px, G), cy = c5_cell(py, G), cz = c5_cell(pz, G);
  const double cs = 1.0 / (double)G;
  double best = 1e300;
  uint32_t bi = 0xffffffffu;
  for (int k = 0; k <= G; ++k) {
    for (int z = cz - k; z <= cz + k; ++z) {
      if (z < 0 || z >= G) continue;
      for (int y = cy - k; y <= cy + k; ++y) {
        if (y < 0 || y >= G) continue;
        for (int x = cx - k; x <= cx + k; ++x) {
          if (x < 0 || x >= G) continue;
          if (z != cz - k && z != cz + k && y != cy - k && y != cy + k && x != cx - k && x != cx + k) continue;
          const uint32_t c = ((uint32_t)z * (uint32_t)G + (uint32_t)y) * (uint32_t)G + (uint32_t)x;
          for (uint32_t e = C->start[c]; e < C->start[c + 1]; ++e) {
            const uint32_t h = C->items[e];
            const double dx = px - C->pos[3 * h], dy = py - C->pos[3 * h + 1], dz = pz - C->pos[3 * h + 2];
            const double d2 = dx * dx + dy * dy + dz * dz;
            if (d2 < best || (d2 == best && h < bi)) {
              best = d2;
              bi = h;
            }
          }
        }
      }
    }
    const double b = (double)k * cs;
    if (bi != 0xffffffffu && best <= b * b) break;
  }
  return bi;
}

void orc_c5_hitpoints(const orc_c5 *C, uint32_t h0, uint32_t n, double *pos, double *nrm, double *wo, double *thr,
                      double *alb, uint32_t *eye_depth) {
  for (uint32_t i = 0; i < n; ++i) {
    for (int k = 0; k < 3; ++k) {
      pos[3 * i + k] = C->pos[3 * (h0 + i) + k];
      nrm[3 * i + k] = C->nrm[3 * (h0 + i) + k];
      wo[3 * i + k] = C->nrm[3 * (h0 + i) + k];
      thr[3 * i + k] = 1.0;
      alb[3 * i + k] = 1.0;
    }
    eye_depth[i] = 1;
  }
}

void orc_c5_photons(const orc_c5 *C, uint64_t iteration, uint64_t begin, uint64_t count, float *pos, float *nrm,
                    float *wi, float *pow_, uint32_t *depth) {
  for (uint64_t k = 0; k < count; ++k) {
    const uint64_t j = begin + k;
    uint32_t d[11];
    float fx = 0.f, fy = 0.f, fz = 0.f;
    uint32_t hn = 0;
    for (int a = 0; a < C5_ATTEMPTS; ++a) {
      c5_draws(C->seed, iteration, a == 0 ? 0u : (uint64_t)(7 + a), j, d, 11);
      double x, y, z;
      if (u24(d[0]) < 0.2f) {
        x = (double)u24(d[2]);
        y = (double)u24(d[3]);
        z = (double)u24(d[4]);
      } else {
        const double u = (double)u24(d[1]);
        int c = 0;
        while (c < C5_CLUSTERS - 1 && !(u < C->cl[5 * c + 4])) ++c;
        const double *q = C->cl + 5 * c;
        const double r1 = sqrt(-2.0 * orc_dm_log(uopen(d[2])));
        const double r2 = sqrt(-2.0 * orc_dm_log(uopen(d[4])));
        double s1, c1, s2, c2;
        orc_dm_sincos2pi((double)u24(d[3]), &s1, &c1);
        orc_dm_sincos2pi((double)u24(d[5]), &s2, &c2);
        x = q[0] + q[3] * (r1 * c1);
        y = q[1] + q[3] * (r1 * s1);
        z = q[2] + q[3] * (r2 * c2);
      }
      fx = (float)x;
      fy = (float)y;
      fz = (float)z;
      hn = c5_nearest(C, (double)fx, (double)fy, (double)fz);
      const double *hp = C->pos + 3 * (size_t)hn, *hv = C->nrm + 3 * (size_t)hn;
      const double off = ((double)fx - hp[0]) * hv[0] + ((double)fy - hp[1]) * hv[1] + ((double)fz - hp[2]) * hv[2];
      if (fabs(off) <= 0.05) break;
    }
    const double *nv = C->nrm + 3 * (size_t)hn;
    pos[3 * k] = fx;
    pos[3 * k + 1] = fy;
    pos[3 * k + 2] = fz;
    nrm[3 * k] = (float)nv[0];
    nrm[3 * k + 1] = (float)nv[1];
    nrm[3 * k + 2] = (float)nv[2];
    pow_[3 * k] = u24(d[6]);
    pow_[3 * k + 1] = u24(d[7]);
    pow_[3 * k + 2] = u24(d[8]);
    const double u1 = (double)u24(d[9]);
    double sn, cs;
    orc_dm_sincos2pi((double)u24(d[10]), &sn, &cs);
    const double r = sqrt(u1);
    const double zz = 1.0 - u1;
    const double lx = r * cs, ly = r * sn, lz = sqrt(zz < 0.0 ? 0.0 : zz);
    double fu[3], fv[3];
    orc_build_frame(nv, fu, fv);
    for (int i = 0; i < 3; ++i) wi[3 * k + i] = (float)(fu[i] * lx + fv[i] * ly + nv[i] * lz);
    depth[k] = 1;
  }
}
