// SPDX-License-Identifier: Apache-2.0
//
// ref_shim.cpp -- TEST INFRASTRUCTURE.  A C-ABI wrapper around the UNMODIFIED
// reference library (the header-only sparsetuck:: API under
// /root/reference/proj/include, included -- never copied).  oracle/Makefile
// compiles it with the reference's Release flags (-O3 -DNDEBUG -fopenmp,
// proj/CMakeLists.txt:7-9) into oracle/_ref/libsparsetuck_ref.so.
//
// Used for: (1) generating tests/golden fixtures (tests/golden/make_golden.py),
// (2) pinning the C restatement (vest_oracle.c), (3) bench.py's CPU baseline
// ("kind": "reference") and --impl reference arm, (4) the byte-level parity of
// the I/O row (load_coo / save_coo / save_model / load_model).  The exported
// names mirror vest_oracle.h with a vr_ prefix so both oracles share one
// Python binding.
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "sparsetuck/model_io.hpp"
#include "sparsetuck/pruning.hpp"
#include "sparsetuck/sparse_tensor.hpp"
#include "sparsetuck/synthetic.hpp"
#include "sparsetuck/trainer.hpp"
#include "sparsetuck/tucker_model.hpp"
#include "sparsetuck/updates.hpp"

using namespace sparsetuck;

namespace {
thread_local std::string g_err;

struct Session {
  SparseTensor x;
  ModeIndex idx;
  TuckerModel m;
  Residuals res;
  bool have_res = false;
  ResponsibilityTable table;
  bool have_table = false;
};

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

Regularizer to_reg(int r) { return r == 0 ? Regularizer::LF : Regularizer::L1; }
}  // namespace

extern "C" {

const char* vr_last_error(void) { return g_err.c_str(); }

int vr_create(int order, const uint64_t* dims, uint64_t nnz, const uint32_t* coords,
              const double* values, const uint64_t* ranks, void** out) {
  *out = nullptr;
  return guard([&] {
    auto s = std::make_unique<Session>();
    std::vector<std::size_t> d(dims, dims + order), r(ranks, ranks + order);
    s->x = make_tensor(d, std::vector<Coord>(coords, coords + nnz * order),
                       std::vector<double>(values, values + nnz));
    s->idx = build_mode_index(s->x);
    s->m = init_random(d, r, 0);
    *out = s.release();
  });
}

void vr_destroy(void* p) { delete static_cast<Session*>(p); }

int vr_init_random(void* p, uint64_t seed) {
  auto* s = static_cast<Session*>(p);
  return guard([&] {
    s->m = init_random(s->m.dims, s->m.ranks, seed);
    s->have_res = s->have_table = false;
  });
}

int vr_set_model(void* p, const double* core, const uint8_t* core_mask,
                 const double* const* factors, const uint8_t* const* factor_masks) {
  auto* s = static_cast<Session*>(p);
  return guard([&] {
    auto& m = s->m;
    std::memcpy(m.core.data(), core, m.core.size() * sizeof(double));
    std::memcpy(m.core_mask.data(), core_mask, m.core_mask.size());
    for (std::size_t n = 0; n < m.order(); ++n) {
      std::memcpy(m.factors[n].data(), factors[n], m.factors[n].size() * sizeof(double));
      std::memcpy(m.factor_masks[n].data(), factor_masks[n], m.factor_masks[n].size());
    }
    s->have_res = s->have_table = false;
  });
}

int vr_get_model(const void* p, double* core, uint8_t* core_mask, double* const* factors,
                 uint8_t* const* factor_masks) {
  const auto* s = static_cast<const Session*>(p);
  return guard([&] {
    const auto& m = s->m;
    if (core) std::memcpy(core, m.core.data(), m.core.size() * sizeof(double));
    if (core_mask) std::memcpy(core_mask, m.core_mask.data(), m.core_mask.size());
    for (std::size_t n = 0; n < m.order(); ++n) {
      if (factors && factors[n])
        std::memcpy(factors[n], m.factors[n].data(), m.factors[n].size() * sizeof(double));
      if (factor_masks && factor_masks[n])
        std::memcpy(factor_masks[n], m.factor_masks[n].data(), m.factor_masks[n].size());
    }
  });
}

int vr_get_index(const void* p, int mode, uint64_t* offsets, uint32_t* ids) {
  const auto* s = static_cast<const Session*>(p);
  return guard([&] {
    const auto& off = s->idx.offsets.at(mode);
    for (std::size_t i = 0; i < off.size(); ++i) offsets[i] = off[i];
    std::memcpy(ids, s->idx.ids[mode].data(), s->idx.ids[mode].size() * sizeof(uint32_t));
  });
}

int vr_compute_delta(const void* p, const uint32_t* at, int mode, double* out) {
  const auto* s = static_cast<const Session*>(p);
  return guard([&] {
    std::span<double> o(out, s->m.ranks.at(mode));
    compute_delta(s->m, at, mode, o);
  });
}

int vr_reconstruct(const void* p, const uint32_t* at, uint64_t nq, double* out) {
  const auto* s = static_cast<const Session*>(p);
  return guard([&] {
    auto v = predict(s->m, std::span<const Coord>(at, nq * s->m.order()));
    std::memcpy(out, v.data(), v.size() * sizeof(double));
  });
}

int vr_update_factor_row(void* p, int reg, int mode, uint64_t row, double lambda) {
  auto* s = static_cast<Session*>(p);
  return guard([&] {
    if (reg == 0)
      update_factor_row_lf(s->m, s->x, s->idx, mode, row, lambda);
    else
      update_factor_row_l1(s->m, s->x, s->idx, mode, row, lambda);
    s->have_res = s->have_table = false;
  });
}

int vr_row_stats(void* p, int mode, uint64_t row, double* delta, double* gram, double* xdelta) {
  auto* s = static_cast<Session*>(p);
  return guard([&] {
    RowUpdateScratch sc;
    compute_row_stats(s->m, s->x, s->idx, mode, row, sc);
    std::memcpy(delta, sc.delta.data(), sc.delta.size() * sizeof(double));
    std::memcpy(gram, sc.gram.data(), sc.gram.size() * sizeof(double));
    std::memcpy(xdelta, sc.xdelta.data(), sc.xdelta.size() * sizeof(double));
  });
}

int vr_partial_reconstruct(const void* p, const uint32_t* at, uint64_t nq, int mode, uint64_t j, double* out) {
  const auto* s = static_cast<const Session*>(p);
  return guard([&] {
    for (uint64_t q = 0; q < nq; ++q) out[q] = partial_reconstruct(s->m, at + q * s->m.order(), mode, j);
  });
}

int vr_update_all_factors(void* p, int reg, double lambda, int threads) {
  auto* s = static_cast<Session*>(p);
  return guard([&] {
    update_all_factors(s->m, s->x, s->idx, to_reg(reg), lambda, threads);
    s->have_res = s->have_table = false;
  });
}

int vr_update_core(void* p, int reg, double lambda, int threads) {
  auto* s = static_cast<Session*>(p);
  return guard([&] {
    if (reg == 0)
      update_core_lf(s->m, s->x, lambda, threads);
    else
      update_core_l1(s->m, s->x, lambda, threads);
    s->have_res = s->have_table = false;
  });
}

int vr_compute_residuals(void* p, int threads, double* r_out, double* sum_sq, double* x_norm,
                         double* re) {
  auto* s = static_cast<Session*>(p);
  return guard([&] {
    s->res = compute_residuals(s->m, s->x, threads);
    s->have_res = true;
    if (r_out) std::memcpy(r_out, s->res.r.data(), s->res.r.size() * sizeof(double));
    if (sum_sq) *sum_sq = s->res.sum_sq;
    if (x_norm) *x_norm = s->res.x_norm;
    if (re) *re = s->res.re;
  });
}

int vr_compute_responsibilities(void* p, int threads, double* core_out,
                                double* const* factor_outs) {
  auto* s = static_cast<Session*>(p);
  return guard([&] {
    if (!s->have_res) throw std::invalid_argument("compute_residuals must run first");
    s->table = compute_responsibilities(s->m, s->x, s->idx, s->res, threads);
    s->have_table = true;
    if (core_out)
      std::memcpy(core_out, s->table.core.data(), s->table.core.size() * sizeof(double));
    for (std::size_t n = 0; n < s->m.order(); ++n)
      if (factor_outs && factor_outs[n])
        std::memcpy(factor_outs[n], s->table.factors[n].data(),
                    s->table.factors[n].size() * sizeof(double));
  });
}

int vr_prune_step(void* p, double pr, const double* core_resp, const double* const* factor_resp,
                  uint64_t* counts) {
  auto* s = static_cast<Session*>(p);
  return guard([&] {
    ResponsibilityTable t;
    if (core_resp) {
      t.core.assign(core_resp, core_resp + s->m.core_size());
      t.factors.resize(s->m.order());
      for (std::size_t n = 0; n < s->m.order(); ++n)
        t.factors[n].assign(factor_resp[n], factor_resp[n] + s->m.factors[n].size());
    } else {
      if (!s->have_table) throw std::invalid_argument("no responsibility table");
      t = s->table;
    }
    const PruneCounts c = prune_step(s->m, t, pr);
    counts[0] = c.core;
    for (std::size_t n = 0; n < c.factors.size(); ++n) counts[1 + n] = c.factors[n];
    s->have_res = s->have_table = false;
  });
}

double vr_sparsity(const void* p) { return sparsity(static_cast<const Session*>(p)->m); }
double vr_masked_fraction(const void* p) {
  return masked_fraction(static_cast<const Session*>(p)->m);
}
int vr_normalize_columns(void* p) {
  auto* s = static_cast<Session*>(p);
  return guard([&] {
    normalize_columns(s->m);
    s->have_res = s->have_table = false;
  });
}
double vr_frobenius_norm(const void* p) {
  return static_cast<const Session*>(p)->x.frobenius_norm();
}

int vr_cd_iteration(void* p, int reg, double lambda, int threads, double* re) {
  auto* s = static_cast<Session*>(p);
  return guard([&] {
    update_all_factors(s->m, s->x, s->idx, to_reg(reg), lambda, threads);
    if (reg == 0)
      update_core_lf(s->m, s->x, lambda, threads);
    else
      update_core_l1(s->m, s->x, lambda, threads);
    s->res = compute_residuals(s->m, s->x, threads);
    s->have_res = true;
    s->have_table = false;
    if (re) *re = s->res.re;
  });
}

// split_train_test (sparse_tensor.hpp:232-260): returns the entry ids of the
// train and test parts (ascending) for fixtures of the ingest "next" row.
int vr_split_ids(uint64_t nnz, double test_fraction, uint64_t seed, uint64_t* test_ids,
                 uint64_t* n_test, uint64_t* train_ids, uint64_t* n_train) {
  return guard([&] {
    SparseTensor x;
    x.dims = {std::size_t(nnz > 0 ? nnz : 1)};
    for (uint64_t e = 0; e < nnz; ++e) {
      x.coords.push_back(Coord(e));
      x.values.push_back(double(e));
    }
    auto [tr, te] = split_train_test(x, test_fraction, seed);
    *n_test = te.nnz();
    *n_train = tr.nnz();
    for (std::size_t k = 0; k < te.nnz(); ++k) test_ids[k] = te.coords[k];
    for (std::size_t k = 0; k < tr.nnz(); ++k) train_ids[k] = tr.coords[k];
  });
}

// fit() (trainer.hpp:103-168) for the trace fixtures.  Writes per-iteration
// re / pruned flag / sparsity into the caller's arrays (max_iters long).
int vr_fit(void* p, int reg, double lambda, int auto_mode, double target_sparsity,
           double elbow_threshold, double init_pr, double max_pr, uint64_t max_iters, double tol,
           uint64_t seed, int normalize, int threads, double* re_trace, uint8_t* pruned_trace,
           double* sparsity_trace, uint64_t* iters, double* final_re) {
  auto* s = static_cast<Session*>(p);
  return guard([&] {
    TrainConfig cfg;
    cfg.ranks = s->m.ranks;
    cfg.reg = to_reg(reg);
    cfg.lambda = lambda;
    cfg.mode = auto_mode ? StopMode::Auto : StopMode::Manual;
    cfg.target_sparsity = target_sparsity;
    cfg.elbow_threshold = elbow_threshold;
    cfg.schedule.init_pr = init_pr;
    cfg.schedule.max_pr = max_pr;
    cfg.max_iters = max_iters;
    cfg.tol = tol;
    cfg.threads = threads;
    cfg.seed = seed;
    cfg.normalize_output = normalize != 0;
    FitResult r = fit(s->x, cfg);
    *iters = r.report.iters;
    for (std::size_t t = 0; t < r.report.iterations.size(); ++t) {
      re_trace[t] = r.report.iterations[t].re;
      pruned_trace[t] = r.report.iterations[t].pruned ? 1 : 0;
      sparsity_trace[t] = r.report.iterations[t].sparsity;
    }
    *final_re = r.report.final_re;
    s->m = std::move(r.model);
    s->have_res = s->have_table = false;
  });
}

// ------------------------------------------------------------------- I/O --
// load_coo (sparse_tensor.hpp:143-209): two calls -- sizes (coords/values NULL),
// then the data.
int vr_load_coo(const char* path, int one_based, int* order, uint64_t* nnz, uint64_t* dims,
                uint32_t* coords, double* values) {
  return guard([&] {
    const SparseTensor x = load_coo(path, one_based != 0);
    *order = (int)x.order();
    *nnz = x.nnz();
    if (dims)
      for (std::size_t k = 0; k < x.order(); ++k) dims[k] = x.dims[k];
    if (coords) std::memcpy(coords, x.coords.data(), x.coords.size() * sizeof(Coord));
    if (values) std::memcpy(values, x.values.data(), x.values.size() * sizeof(double));
  });
}

// save_coo (sparse_tensor.hpp:211-228)
int vr_save_coo(const char* path, int order, const uint64_t* dims, uint64_t nnz, const uint32_t* coords,
                const double* values) {
  return guard([&] {
    SparseTensor x;
    x.dims.assign(dims, dims + order);
    x.coords.assign(coords, coords + nnz * order);
    x.values.assign(values, values + nnz);
    save_coo(x, path);
  });
}

// save_model (model_io.hpp:22-51)
int vr_save_model(const char* dir, int order, const uint64_t* dims, const uint64_t* ranks, const double* core,
                  const double* const* factors) {
  return guard([&] {
    TuckerModel m;
    m.dims.assign(dims, dims + order);
    m.ranks.assign(ranks, ranks + order);
    m.core.assign(core, core + m.core_size());
    m.core_mask.assign(m.core.size(), 0);
    m.factors.resize(order);
    m.factor_masks.resize(order);
    for (int n = 0; n < order; ++n) {
      m.factors[n].assign(factors[n], factors[n] + dims[n] * ranks[n]);
      m.factor_masks[n].assign(m.factors[n].size(), 0);
    }
    save_model(m, dir);
  });
}

// load_model (model_io.hpp:53-104): sizes first (core/factors NULL), then data
int vr_load_model(const char* dir, int* order, uint64_t* dims, uint64_t* ranks, double* core,
                  uint8_t* core_mask, double* const* factors, uint8_t* const* factor_masks) {
  return guard([&] {
    const TuckerModel m = load_model(dir);
    *order = (int)m.order();
    for (std::size_t n = 0; n < m.order(); ++n) {
      if (dims) dims[n] = m.dims[n];
      if (ranks) ranks[n] = m.ranks[n];
    }
    if (core) std::memcpy(core, m.core.data(), m.core.size() * sizeof(double));
    if (core_mask) std::memcpy(core_mask, m.core_mask.data(), m.core_mask.size());
    for (std::size_t n = 0; n < m.order(); ++n) {
      if (factors && factors[n]) std::memcpy(factors[n], m.factors[n].data(), m.factors[n].size() * sizeof(double));
      if (factor_masks && factor_masks[n]) std::memcpy(factor_masks[n], m.factor_masks[n].data(), m.factor_masks[n].size());
    }
  });
}

// gen_synthetic (synthetic.hpp:105-155): planted model + observations
int vr_gen_synthetic(int order, const uint64_t* dims, const uint64_t* ranks, uint64_t nnz, double density,
                     double noise, uint64_t seed, uint32_t* coords, double* values, double* core, uint8_t* core_mask,
                     double* const* factors, uint8_t* const* factor_masks) {
  return guard([&] {
    SyntheticSpec spec;
    spec.dims.assign(dims, dims + order);
    spec.ranks.assign(ranks, ranks + order);
    spec.nnz = nnz;
    spec.factor_density = density;
    spec.noise_std = noise;
    spec.seed = seed;
    const SyntheticData d = gen_synthetic(spec);
    std::memcpy(coords, d.tensor.coords.data(), d.tensor.coords.size() * sizeof(Coord));
    std::memcpy(values, d.tensor.values.data(), d.tensor.values.size() * sizeof(double));
    std::memcpy(core, d.truth.core.data(), d.truth.core.size() * sizeof(double));
    std::memcpy(core_mask, d.truth.core_mask.data(), d.truth.core_mask.size());
    for (int n = 0; n < order; ++n) {
      std::memcpy(factors[n], d.truth.factors[n].data(), d.truth.factors[n].size() * sizeof(double));
      std::memcpy(factor_masks[n], d.truth.factor_masks[n].data(), d.truth.factor_masks[n].size());
    }
  });
}

}  // extern "C"
