/* SPDX-License-Identifier: Apache-2.0
 *
 * vest_oracle.c -- TEST INFRASTRUCTURE: CPU restatement of the VeST CD hot
 * path (see vest_oracle.h).  Every function cites the reference function it
 * restates; loop nests and accumulation orders follow the reference so the
 * results are bit-identical (build with -ffp-contract=off, see Makefile).
 */
#include "vest_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define VO_MAXN 32

struct vo_session {
  int n;
  uint64_t dims[VO_MAXN];
  uint64_t ranks[VO_MAXN];
  uint64_t nnz;
  uint32_t* coords; /* nnz * n, entry-major */
  double* values;
  /* ModeIndex */
  uint64_t* offsets[VO_MAXN];
  uint32_t* ids[VO_MAXN];
  /* TuckerModel */
  uint64_t core_size;
  double* core;
  uint8_t* core_mask;
  double* factors[VO_MAXN];
  uint8_t* fmasks[VO_MAXN];
  /* Residuals */
  double* r;
  int have_res;
  double sum_sq, x_norm, re;
  /* ResponsibilityTable */
  double* resp_core;
  double* resp_f[VO_MAXN];
  int have_table;
};

static char g_err[256];
static int fail(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}
const char* vo_last_error(void) { return g_err; }

/* ------------------------------------------------------------------ RNG --
 * std::mt19937_64 and libstdc++'s generate_canonical<double, 53> as used by
 * std::uniform_real_distribution<double>(0, 1) in init_random
 * (tucker_model.hpp:96-107). */
typedef struct {
  uint64_t mt[312];
  int i;
} mt64;

static void mt64_seed(mt64* s, uint64_t seed) {
  s->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
  s->i = 312;
}

static uint64_t mt64_next(mt64* s) {
  if (s->i >= 312) {
    for (int k = 0; k < 312; ++k) {
      uint64_t y = (s->mt[k] & 0xFFFFFFFF80000000ULL) | (s->mt[(k + 1) % 312] & 0x7FFFFFFFULL);
      uint64_t v = y >> 1;
      if (y & 1ULL) v ^= 0xB5026F5AA96619E9ULL;
      s->mt[k] = s->mt[(k + 156) % 312] ^ v;
    }
    s->i = 0;
  }
  uint64_t x = s->mt[s->i++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= (x >> 43);
  return x;
}

static double mt64_unit(mt64* s) {
  double u = (double)mt64_next(s) / 18446744073709551616.0;
  if (u >= 1.0) u = nextafter(1.0, 0.0);
  return u;
}

/* ------------------------------------------------------------- helpers -- */
/* detail::advance_multi_index (tucker_model.hpp:58-65) */
static int advance(uint64_t* idx, const uint64_t* shape, int n) {
  for (int k = n; k-- > 0;) {
    if (++idx[k] < shape[k]) return 1;
    idx[k] = 0;
  }
  return 0;
}

static const uint32_t* entry(const vo_session* s, uint64_t e) { return s->coords + e * s->n; }

/* ModeIndex::slice (sparse_tensor.hpp:113-116) */
static void slice(const vo_session* s, int mode, uint64_t i, const uint32_t** ids, uint64_t* len) {
  *ids = s->ids[mode] + s->offsets[mode][i];
  *len = s->offsets[mode][i + 1] - s->offsets[mode][i];
}

static int lex_n;
static const uint32_t* lex_coords;
static int cmp_lex(const void* a, const void* b) {
  const uint32_t* ca = lex_coords + (*(const uint64_t*)a) * lex_n;
  const uint32_t* cb = lex_coords + (*(const uint64_t*)b) * lex_n;
  for (int k = 0; k < lex_n; ++k) {
    if (ca[k] < cb[k]) return -1;
    if (ca[k] > cb[k]) return 1;
  }
  return 0;
}

/* --------------------------------------------------------- construction -- */
void vo_destroy(vo_session* s) {
  if (!s) return;
  free(s->coords);
  free(s->values);
  for (int k = 0; k < s->n; ++k) {
    free(s->offsets[k]);
    free(s->ids[k]);
    free(s->factors[k]);
    free(s->fmasks[k]);
    free(s->resp_f[k]);
  }
  free(s->core);
  free(s->core_mask);
  free(s->r);
  free(s->resp_core);
  free(s);
}

/* make_tensor/check_tensor (sparse_tensor.hpp:68-105), build_mode_index
 * (:119-137) and a zero model of the given ranks. */
int vo_create(int order, const uint64_t* dims, uint64_t nnz, const uint32_t* coords,
              const double* values, const uint64_t* ranks, vo_session** out) {
  *out = NULL;
  if (order <= 0) return fail(1, "tensor order must be at least 1");
  if (order > VO_MAXN) return fail(1, "order too large for the oracle");
  for (int k = 0; k < order; ++k) {
    if (dims[k] == 0) return fail(1, "tensor dimensions must be positive");
    if (ranks[k] == 0) return fail(1, "dims and ranks must be positive");
  }
  for (uint64_t e = 0; e < nnz; ++e)
    for (int k = 0; k < order; ++k)
      if (coords[e * order + k] >= dims[k]) return fail(1, "coordinate out of bounds");
  if (nnz > 1) {
    uint64_t* ids = (uint64_t*)malloc(nnz * sizeof(uint64_t));
    for (uint64_t e = 0; e < nnz; ++e) ids[e] = e;
    lex_n = order;
    lex_coords = coords;
    qsort(ids, nnz, sizeof(uint64_t), cmp_lex);
    for (uint64_t e = 1; e < nnz; ++e)
      if (cmp_lex(&ids[e - 1], &ids[e]) == 0) {
        free(ids);
        return fail(1, "duplicate coordinate in tensor");
      }
    free(ids);
  }
  vo_session* s = (vo_session*)calloc(1, sizeof(vo_session));
  s->n = order;
  s->nnz = nnz;
  memcpy(s->dims, dims, order * sizeof(uint64_t));
  memcpy(s->ranks, ranks, order * sizeof(uint64_t));
  s->coords = (uint32_t*)malloc((nnz * order + 1) * sizeof(uint32_t));
  s->values = (double*)malloc((nnz + 1) * sizeof(double));
  memcpy(s->coords, coords, nnz * order * sizeof(uint32_t));
  memcpy(s->values, values, nnz * sizeof(double));
  for (int m = 0; m < order; ++m) {
    uint64_t* count = (uint64_t*)calloc(dims[m] + 1, sizeof(uint64_t));
    for (uint64_t e = 0; e < nnz; ++e) ++count[entry(s, e)[m] + 1];
    for (uint64_t i = 1; i < dims[m] + 1; ++i) count[i] += count[i - 1];
    s->offsets[m] = count;
    s->ids[m] = (uint32_t*)malloc((nnz + 1) * sizeof(uint32_t));
    uint64_t* cursor = (uint64_t*)malloc((dims[m] + 1) * sizeof(uint64_t));
    memcpy(cursor, count, dims[m] * sizeof(uint64_t));
    for (uint64_t e = 0; e < nnz; ++e) {
      uint32_t i = entry(s, e)[m];
      s->ids[m][cursor[i]++] = (uint32_t)e;
    }
    free(cursor);
  }
  s->core_size = 1;
  for (int k = 0; k < order; ++k) s->core_size *= ranks[k];
  s->core = (double*)calloc(s->core_size, sizeof(double));
  s->core_mask = (uint8_t*)calloc(s->core_size, 1);
  for (int k = 0; k < order; ++k) {
    s->factors[k] = (double*)calloc(dims[k] * ranks[k], sizeof(double));
    s->fmasks[k] = (uint8_t*)calloc(dims[k] * ranks[k], 1);
  }
  s->r = (double*)calloc(nnz + 1, sizeof(double));
  *out = s;
  return 0;
}

/* init_random (tucker_model.hpp:88-108) */
int vo_init_random(vo_session* s, uint64_t seed) {
  mt64 g;
  mt64_seed(&g, seed);
  for (int n = 0; n < s->n; ++n) {
    uint64_t sz = s->dims[n] * s->ranks[n];
    memset(s->fmasks[n], 0, sz);
    for (uint64_t k = 0; k < sz; ++k) s->factors[n][k] = mt64_unit(&g);
  }
  memset(s->core_mask, 0, s->core_size);
  for (uint64_t k = 0; k < s->core_size; ++k) s->core[k] = mt64_unit(&g);
  s->have_res = s->have_table = 0;
  return 0;
}

int vo_set_model(vo_session* s, const double* core, const uint8_t* core_mask,
                 const double* const* factors, const uint8_t* const* factor_masks) {
  memcpy(s->core, core, s->core_size * sizeof(double));
  memcpy(s->core_mask, core_mask, s->core_size);
  for (int n = 0; n < s->n; ++n) {
    uint64_t sz = s->dims[n] * s->ranks[n];
    memcpy(s->factors[n], factors[n], sz * sizeof(double));
    memcpy(s->fmasks[n], factor_masks[n], sz);
  }
  s->have_res = s->have_table = 0;
  return 0;
}

int vo_get_model(const vo_session* s, double* core, uint8_t* core_mask, double* const* factors,
                 uint8_t* const* factor_masks) {
  if (core) memcpy(core, s->core, s->core_size * sizeof(double));
  if (core_mask) memcpy(core_mask, s->core_mask, s->core_size);
  for (int n = 0; n < s->n; ++n) {
    uint64_t sz = s->dims[n] * s->ranks[n];
    if (factors && factors[n]) memcpy(factors[n], s->factors[n], sz * sizeof(double));
    if (factor_masks && factor_masks[n]) memcpy(factor_masks[n], s->fmasks[n], sz);
  }
  return 0;
}

int vo_get_index(const vo_session* s, int mode, uint64_t* offsets, uint32_t* ids) {
  if (mode < 0 || mode >= s->n) return fail(1, "mode out of range");
  memcpy(offsets, s->offsets[mode], (s->dims[mode] + 1) * sizeof(uint64_t));
  memcpy(ids, s->ids[mode], s->nnz * sizeof(uint32_t));
  return 0;
}

/* ------------------------------------------------------------ kernels -- */
/* SparseTensor::frobenius_norm (sparse_tensor.hpp:45-49) */
double vo_frobenius_norm(const vo_session* s) {
  double acc = 0.0;
  for (uint64_t e = 0; e < s->nnz; ++e) acc += s->values[e] * s->values[e];
  return sqrt(acc);
}

/* reconstruct_entry (tucker_model.hpp:112-131) */
static double reconstruct_entry(const vo_session* s, const uint32_t* at) {
  const int n = s->n;
  uint64_t beta[VO_MAXN] = {0};
  double acc = 0.0;
  uint64_t lin = 0;
  do {
    const double g = s->core[lin];
    if (g != 0.0) {
      double p = g;
      for (int k = 0; k < n; ++k) p *= s->factors[k][at[k] * s->ranks[k] + beta[k]];
      acc += p;
    }
    ++lin;
  } while (advance(beta, s->ranks, n));
  return acc;
}

int vo_reconstruct(const vo_session* s, const uint32_t* at, uint64_t nq, double* out) {
  for (uint64_t q = 0; q < nq; ++q) {
    for (int k = 0; k < s->n; ++k)
      if (at[q * s->n + k] >= s->dims[k]) return fail(1, "query coordinate out of bounds");
    out[q] = reconstruct_entry(s, at + q * s->n);
  }
  return 0;
}

/* compute_delta (updates.hpp:35-52) */
static void compute_delta(const vo_session* s, const uint32_t* at, int mode, double* out) {
  const int n = s->n;
  const uint64_t J = s->ranks[mode];
  for (uint64_t j = 0; j < J; ++j) out[j] = 0.0;
  uint64_t beta[VO_MAXN] = {0};
  uint64_t lin = 0;
  do {
    const double g = s->core[lin];
    if (g != 0.0) {
      double p = g;
      for (int k = 0; k < n; ++k)
        if (k != mode) p *= s->factors[k][at[k] * s->ranks[k] + beta[k]];
      out[beta[mode]] += p;
    }
    ++lin;
  } while (advance(beta, s->ranks, n));
}

/* The nonzero core cells in row-major order with their multi-indices: the
 * cells compute_delta / reconstruct_entry do not skip (updates.hpp:44,
 * tucker_model.hpp:121).  Iterating this list instead of the odometer visits
 * the same cells in the same order with the same arithmetic (bit-identical);
 * it only saves the skipped iterations at BASELINE sizes (config 4: 411 of
 * 4096 cells). */
typedef struct {
  uint64_t n;
  double* g;
  uint16_t* beta; /* n * order */
} cell_list;

static cell_list nonzero_cells(const vo_session* s) {
  cell_list c;
  c.n = 0;
  c.g = (double*)malloc((s->core_size + 1) * sizeof(double));
  c.beta = (uint16_t*)malloc((s->core_size + 1) * s->n * sizeof(uint16_t));
  uint64_t beta[VO_MAXN] = {0};
  uint64_t lin = 0;
  do {
    if (s->core[lin] != 0.0) {
      c.g[c.n] = s->core[lin];
      for (int k = 0; k < s->n; ++k) c.beta[c.n * s->n + k] = (uint16_t)beta[k];
      ++c.n;
    }
    ++lin;
  } while (advance(beta, s->ranks, s->n));
  return c;
}

static void free_cells(cell_list* c) {
  free(c->g);
  free(c->beta);
}

static void compute_delta_cells(const vo_session* s, const cell_list* c, const uint32_t* at, int mode, double* out) {
  const int n = s->n;
  const uint64_t J = s->ranks[mode];
  for (uint64_t j = 0; j < J; ++j) out[j] = 0.0;
  for (uint64_t q = 0; q < c->n; ++q) {
    const uint16_t* b = c->beta + q * n;
    double p = c->g[q];
    for (int k = 0; k < n; ++k)
      if (k != mode) p *= s->factors[k][at[k] * s->ranks[k] + b[k]];
    out[b[mode]] += p;
  }
}

static double reconstruct_cells(const vo_session* s, const cell_list* c, const uint32_t* at) {
  const int n = s->n;
  double acc = 0.0;
  for (uint64_t q = 0; q < c->n; ++q) {
    const uint16_t* b = c->beta + q * n;
    double p = c->g[q];
    for (int k = 0; k < n; ++k) p *= s->factors[k][at[k] * s->ranks[k] + b[k]];
    acc += p;
  }
  return acc;
}

/* partial_reconstruct (tucker_model.hpp:136-154) */
int vo_partial_reconstruct(const vo_session* s, const uint32_t* at, uint64_t nq, int mode, uint64_t j,
                           double* out) {
  if (mode < 0 || mode >= s->n) return fail(1, "mode out of range");
  const int n = s->n;
  for (uint64_t q = 0; q < nq; ++q) {
    const uint32_t* a = at + q * n;
    uint64_t beta[VO_MAXN] = {0};
    double acc = 0.0;
    uint64_t lin = 0;
    do {
      if (beta[mode] == j) {
        const double g = s->core[lin];
        if (g != 0.0) {
          double p = g;
          for (int k = 0; k < n; ++k) p *= s->factors[k][a[k] * s->ranks[k] + beta[k]];
          acc += p;
        }
      }
      ++lin;
    } while (advance(beta, s->ranks, n));
    out[q] = acc;
  }
  return 0;
}

int vo_compute_delta(const vo_session* s, const uint32_t* at, int mode, double* out) {
  if (mode < 0 || mode >= s->n) return fail(1, "mode out of range");
  compute_delta(s, at, mode, out);
  return 0;
}

/* compute_row_stats (updates.hpp:64-79); delta/gram/xdelta are the
 * RowUpdateScratch buffers (:20-30). */
static void row_stats(const vo_session* s, const cell_list* cl, int mode, uint64_t i, double* delta, double* gram,
                      double* xdelta) {
  const uint64_t J = s->ranks[mode];
  for (uint64_t t = 0; t < J; ++t) delta[t] = 0.0, xdelta[t] = 0.0;
  for (uint64_t t = 0; t < J * J; ++t) gram[t] = 0.0;
  const uint32_t* ids;
  uint64_t len;
  slice(s, mode, i, &ids, &len);
  for (uint64_t q = 0; q < len; ++q) {
    const uint32_t e = ids[q];
    compute_delta_cells(s, cl, entry(s, e), mode, delta);
    const double xv = s->values[e];
    for (uint64_t t = 0; t < J; ++t) {
      const double dt = delta[t];
      if (dt == 0.0) continue;
      xdelta[t] += xv * dt;
      double* row = gram + t * J;
      for (uint64_t j = 0; j < J; ++j) row[j] += dt * delta[j];
    }
  }
}

/* update_factor_row_lf (updates.hpp:88-106) / update_factor_row_l1 (:113-139) */
static void update_row(vo_session* s, const cell_list* cl, int reg, int mode, uint64_t i, double lambda,
                       double* delta, double* gram, double* xdelta) {
  const uint64_t J = s->ranks[mode];
  if (reg == 0 && s->offsets[mode][i + 1] == s->offsets[mode][i]) return;
  row_stats(s, cl, mode, i, delta, gram, xdelta);
  double* row = s->factors[mode] + i * J;
  const uint8_t* mask = s->fmasks[mode] + i * J;
  for (uint64_t j = 0; j < J; ++j) {
    if (mask[j]) continue;
    const double* gj = gram + j * J;
    if (reg == 0) {
      double num = xdelta[j];
      for (uint64_t t = 0; t < J; ++t)
        if (t != j) num -= gj[t] * row[t];
      const double den = gj[j] + lambda;
      if (den == 0.0) continue;
      row[j] = num / den;
    } else {
      double lin = xdelta[j];
      for (uint64_t t = 0; t < J; ++t)
        if (t != j) lin -= gj[t] * row[t];
      const double g = -2.0 * lin;
      const double d = 2.0 * gj[j];
      if (d == 0.0) {
        if (fabs(g) <= lambda) row[j] = 0.0;
        continue;
      }
      if (g > lambda)
        row[j] = (lambda - g) / d;
      else if (g < -lambda)
        row[j] = -(lambda + g) / d;
      else
        row[j] = 0.0;
    }
  }
}

int vo_update_factor_row(vo_session* s, int reg, int mode, uint64_t row, double lambda) {
  if (mode < 0 || mode >= s->n || row >= s->dims[mode]) return fail(1, "row out of range");
  const uint64_t J = s->ranks[mode];
  double* buf = (double*)malloc((J * J + 2 * J) * sizeof(double));
  cell_list cl = nonzero_cells(s);
  update_row(s, &cl, reg, mode, row, lambda, buf, buf + J, buf + J + J * J);
  free_cells(&cl);
  free(buf);
  s->have_res = s->have_table = 0;
  return 0;
}

/* compute_row_stats (updates.hpp:64-79) into RowUpdateScratch-shaped buffers */
int vo_row_stats(vo_session* s, int mode, uint64_t row, double* delta, double* gram, double* xdelta) {
  if (mode < 0 || mode >= s->n || row >= s->dims[mode]) return fail(1, "row out of range");
  cell_list cl = nonzero_cells(s);
  row_stats(s, &cl, mode, row, delta, gram, xdelta);
  free_cells(&cl);
  return 0;
}

/* One mode of update_all_factors (updates.hpp:162-173): the rows of `mode`
 * in parallel (independent within a mode). */
int vo_update_factor_mode(vo_session* s, int reg, int mode, double lambda, int threads) {
  if (mode < 0 || mode >= s->n) return fail(1, "mode out of range");
  const int T = threads > 0 ? threads : 1;
  const long rows = (long)s->dims[mode];
  const uint64_t J = s->ranks[mode];
  cell_list cl = nonzero_cells(s);
#pragma omp parallel num_threads(T)
  {
    double* buf = (double*)malloc((J * J + 2 * J) * sizeof(double));
#pragma omp for schedule(dynamic, 8)
    for (long i = 0; i < rows; ++i)
      update_row(s, &cl, reg, mode, (uint64_t)i, lambda, buf, buf + J, buf + J + J * J);
    free(buf);
  }
  free_cells(&cl);
  s->have_res = s->have_table = 0;
  return 0;
}

/* update_all_factors (updates.hpp:157-175) */
int vo_update_all_factors(vo_session* s, int reg, double lambda, int threads) {
  for (int mode = 0; mode < s->n; ++mode) vo_update_factor_mode(s, reg, mode, lambda, threads);
  return 0;
}

/* detail::core_sweep (updates.hpp:185-245) */
int vo_update_core(vo_session* s, int reg, double lambda, int threads) {
  const int T = threads > 0 ? threads : 1;
  const long nnz = (long)s->nnz;
  const int n = s->n;
  double* recon = (double*)malloc((s->nnz + 1) * sizeof(double));
  {
    cell_list cl = nonzero_cells(s);
#pragma omp parallel for schedule(static) num_threads(T)
    for (long e = 0; e < nnz; ++e) recon[e] = reconstruct_cells(s, &cl, entry(s, e));
    free_cells(&cl);
  }
  double* prod = (double*)malloc((s->nnz + 1) * sizeof(double));
  uint64_t beta[VO_MAXN] = {0};
  uint64_t lin = 0;
  do {
    if (s->core_mask[lin]) {
      ++lin;
      continue;
    }
    const double g_old = s->core[lin];
#pragma omp parallel for schedule(static) num_threads(T)
    for (long e = 0; e < nnz; ++e) {
      const uint32_t* at = entry(s, e);
      double p = 1.0;
      for (int k = 0; k < n; ++k) p *= s->factors[k][at[k] * s->ranks[k] + beta[k]];
      prod[e] = p;
    }
    double num = 0.0;
    double den = 0.0;
    for (long e = 0; e < nnz; ++e) {
      const double p = prod[e];
      num += (s->values[e] - recon[e] + g_old * p) * p;
      den += p * p;
    }
    double g_new = g_old;
    if (reg == 0) {
      if (den + lambda != 0.0) g_new = num / (den + lambda);
    } else {
      const double g = -2.0 * num;
      const double d = 2.0 * den;
      if (d != 0.0) {
        if (g > lambda)
          g_new = (lambda - g) / d;
        else if (g < -lambda)
          g_new = -(lambda + g) / d;
        else
          g_new = 0.0;
      }
    }
    if (g_new != g_old) {
      s->core[lin] = g_new;
      const double dg = g_new - g_old;
#pragma omp parallel for schedule(static) num_threads(T)
      for (long e = 0; e < nnz; ++e) recon[e] += dg * prod[e];
    }
    ++lin;
  } while (advance(beta, s->ranks, n));
  free(recon);
  free(prod);
  s->have_res = s->have_table = 0;
  return 0;
}

/* compute_residuals (tucker_model.hpp:168-183) */
int vo_compute_residuals(vo_session* s, int threads, double* r_out, double* sum_sq,
                         double* x_norm, double* re) {
  const int T = threads > 0 ? threads : 1;
  const double xn = vo_frobenius_norm(s);
  if (xn == 0.0) return fail(1, "zero-norm tensor");
  const long nnz = (long)s->nnz;
  cell_list cl = nonzero_cells(s);
#pragma omp parallel for schedule(static) num_threads(T)
  for (long e = 0; e < nnz; ++e) s->r[e] = s->values[e] - reconstruct_cells(s, &cl, entry(s, e));
  free_cells(&cl);
  double acc = 0.0;
  for (long e = 0; e < nnz; ++e) acc += s->r[e] * s->r[e];
  s->sum_sq = acc;
  s->x_norm = xn;
  s->re = sqrt(acc) / xn;
  s->have_res = 1;
  if (r_out) memcpy(r_out, s->r, s->nnz * sizeof(double));
  if (sum_sq) *sum_sq = s->sum_sq;
  if (x_norm) *x_norm = s->x_norm;
  if (re) *re = s->re;
  return 0;
}

/* compute_core_responsibilities (pruning.hpp:98-134) */
static void core_resp(vo_session* s, int T, double* resp) {
  const double inf = INFINITY;
  const uint64_t cs = s->core_size;
  const int n = s->n;
  for (uint64_t c = 0; c < cs; ++c) resp[c] = inf;
  if (s->re == 0.0) return;
  uint64_t* multi = (uint64_t*)malloc(cs * n * sizeof(uint64_t));
  uint64_t beta[VO_MAXN] = {0};
  uint64_t lin = 0;
  do {
    for (int k = 0; k < n; ++k) multi[lin * n + k] = beta[k];
    ++lin;
  } while (advance(beta, s->ranks, n));
#pragma omp parallel for schedule(dynamic, 1) num_threads(T)
  for (long c = 0; c < (long)cs; ++c) {
    if (s->core_mask[c]) continue;
    const uint64_t* b = multi + (uint64_t)c * n;
    const double g = s->core[c];
    double acc = 0.0;
    for (uint64_t e = 0; e < s->nnz; ++e) {
      const uint32_t* at = entry(s, e);
      double p = 1.0;
      for (int k = 0; k < n; ++k) p *= s->factors[k][at[k] * s->ranks[k] + b[k]];
      const double t = s->r[e] + g * p;
      acc += t * t;
    }
    const double re_without = sqrt(acc) / s->x_norm;
    resp[c] = (re_without - s->re) / s->re;
  }
  free(multi);
}

/* compute_factor_responsibilities (pruning.hpp:141-179) */
static void factor_resp(vo_session* s, int mode, int T, double* resp) {
  const double inf = INFINITY;
  const uint64_t J = s->ranks[mode];
  const uint64_t I = s->dims[mode];
  for (uint64_t k = 0; k < I * J; ++k) resp[k] = inf;
  if (s->re == 0.0) return;
  const double x2 = s->x_norm * s->x_norm;
  const double re2 = s->re * s->re;
  cell_list cl = nonzero_cells(s);
#pragma omp parallel num_threads(T)
  {
    double* delta = (double*)malloc(J * sizeof(double));
    double* acc = (double*)malloc(J * sizeof(double));
#pragma omp for schedule(dynamic, 4)
    for (long i = 0; i < (long)I; ++i) {
      for (uint64_t j = 0; j < J; ++j) acc[j] = 0.0;
      const uint32_t* ids;
      uint64_t len;
      slice(s, mode, (uint64_t)i, &ids, &len);
      for (uint64_t q = 0; q < len; ++q) {
        const uint32_t e = ids[q];
        compute_delta_cells(s, &cl, entry(s, e), mode, delta);
        const double r = s->r[e];
        for (uint64_t j = 0; j < J; ++j) {
          const double p = delta[j] * s->factors[mode][(uint64_t)i * J + j];
          acc[j] += (2.0 * r + p) * p;
        }
      }
      for (uint64_t j = 0; j < J; ++j) {
        if (s->fmasks[mode][(uint64_t)i * J + j]) continue;
        double err2 = re2 + acc[j] / x2;
        if (err2 < 0.0) err2 = 0.0;
        resp[(uint64_t)i * J + j] = (sqrt(err2) - s->re) / s->re;
      }
    }
    free(delta);
    free(acc);
  }
  free_cells(&cl);
}

/* compute_responsibilities (pruning.hpp:181-191) */
int vo_compute_responsibilities(vo_session* s, int threads, double* core_out,
                                double* const* factor_outs) {
  if (!s->have_res) return fail(1, "compute_residuals must run first");
  const int T = threads > 0 ? threads : 1;
  if (!s->resp_core) {
    s->resp_core = (double*)malloc(s->core_size * sizeof(double));
    for (int n = 0; n < s->n; ++n)
      s->resp_f[n] = (double*)malloc(s->dims[n] * s->ranks[n] * sizeof(double));
  }
  core_resp(s, T, s->resp_core);
  for (int n = 0; n < s->n; ++n) factor_resp(s, n, T, s->resp_f[n]);
  s->have_table = 1;
  if (core_out) memcpy(core_out, s->resp_core, s->core_size * sizeof(double));
  for (int n = 0; n < s->n; ++n)
    if (factor_outs && factor_outs[n])
      memcpy(factor_outs[n], s->resp_f[n], s->dims[n] * s->ranks[n] * sizeof(double));
  return 0;
}

/* detail::prune_lowest (pruning.hpp:206-222): candidates are the unmasked
 * positions, ordered by (resp ascending, index ascending). */
typedef struct {
  double r;
  uint64_t i;
} cand_t;
static int cmp_cand(const void* a, const void* b) {
  const cand_t* x = (const cand_t*)a;
  const cand_t* y = (const cand_t*)b;
  if (x->r != y->r) return x->r < y->r ? -1 : 1;
  return x->i < y->i ? -1 : (x->i > y->i ? 1 : 0);
}

static uint64_t prune_lowest(const double* resp, uint64_t size, uint64_t want, double* values,
                             uint8_t* mask) {
  cand_t* cand = (cand_t*)malloc((size + 1) * sizeof(cand_t));
  uint64_t nc = 0;
  for (uint64_t i = 0; i < size; ++i)
    if (!mask[i]) cand[nc].r = resp[i], cand[nc].i = i, ++nc;
  const uint64_t take = want < nc ? want : nc;
  if (take == 0) {
    free(cand);
    return 0;
  }
  qsort(cand, nc, sizeof(cand_t), cmp_cand);
  for (uint64_t k = 0; k < take; ++k) {
    values[cand[k].i] = 0.0;
    mask[cand[k].i] = 1;
  }
  free(cand);
  return take;
}

/* prune_step (pruning.hpp:234-247) */
int vo_prune_step(vo_session* s, double pr, const double* core_resp,
                  const double* const* factor_resp, uint64_t* counts) {
  if (!(pr >= 0.0 && pr < 1.0)) return fail(1, "prune rate must be in [0, 1)");
  if (!core_resp && !s->have_table) return fail(1, "no responsibility table");
  const double* rc = core_resp ? core_resp : s->resp_core;
  counts[0] = prune_lowest(rc, s->core_size, (uint64_t)(pr * (double)s->core_size), s->core,
                           s->core_mask);
  for (int n = 0; n < s->n; ++n) {
    const uint64_t size = s->dims[n] * s->ranks[n];
    const double* rf = core_resp ? factor_resp[n] : s->resp_f[n];
    counts[1 + n] = prune_lowest(rf, size, (uint64_t)(pr * (double)size), s->factors[n], s->fmasks[n]);
  }
  s->have_res = s->have_table = 0;
  return 0;
}

static uint64_t num_elements(const vo_session* s) {
  uint64_t t = s->core_size;
  for (int n = 0; n < s->n; ++n) t += s->dims[n] * s->ranks[n];
  return t;
}

/* sparsity (tucker_model.hpp:192-198) */
double vo_sparsity(const vo_session* s) {
  uint64_t zeros = 0;
  for (uint64_t k = 0; k < s->core_size; ++k) zeros += (s->core[k] == 0.0);
  for (int n = 0; n < s->n; ++n)
    for (uint64_t k = 0; k < s->dims[n] * s->ranks[n]; ++k) zeros += (s->factors[n][k] == 0.0);
  return (double)zeros / (double)num_elements(s);
}

/* masked_fraction (tucker_model.hpp:201-207) */
double vo_masked_fraction(const vo_session* s) {
  uint64_t m = 0;
  for (uint64_t k = 0; k < s->core_size; ++k) m += s->core_mask[k];
  for (int n = 0; n < s->n; ++n)
    for (uint64_t k = 0; k < s->dims[n] * s->ranks[n]; ++k) m += s->fmasks[n][k];
  return (double)m / (double)num_elements(s);
}

/* normalize_columns (tucker_model.hpp:212-236) */
int vo_normalize_columns(vo_session* s) {
  const int n = s->n;
  for (int mode = 0; mode < n; ++mode) {
    const uint64_t J = s->ranks[mode];
    const uint64_t I = s->dims[mode];
    for (uint64_t j = 0; j < J; ++j) {
      double acc = 0.0;
      for (uint64_t i = 0; i < I; ++i) {
        const double v = s->factors[mode][i * J + j];
        acc += v * v;
      }
      if (acc == 0.0) continue;
      const double norm = sqrt(acc);
      for (uint64_t i = 0; i < I; ++i) s->factors[mode][i * J + j] /= norm;
      uint64_t beta[VO_MAXN] = {0};
      uint64_t lin = 0;
      do {
        if (beta[mode] == j) s->core[lin] *= norm;
        ++lin;
      } while (advance(beta, s->ranks, n));
    }
  }
  s->have_res = s->have_table = 0;
  return 0;
}

/* fit() loop body up to the residuals (trainer.hpp:121-127) */
int vo_cd_iteration(vo_session* s, int reg, double lambda, int threads, double* re) {
  int rc = vo_update_all_factors(s, reg, lambda, threads);
  if (rc) return rc;
  rc = vo_update_core(s, reg, lambda, threads);
  if (rc) return rc;
  return vo_compute_residuals(s, threads, NULL, NULL, NULL, re);
}
