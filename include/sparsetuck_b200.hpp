// SPDX-License-Identifier: Apache-2.0
//
// sparsetuck_b200.hpp -- drop-in C++ surface of the reference library
// (namespace sparsetuck::, /root/reference/proj/include/sparsetuck/*.hpp) on
// the B200 path.  Replace
//     #include "sparsetuck/sparsetuck.hpp"
// with
//     #include "sparsetuck_b200.hpp"        // and link -lvest_cuda
// and the hot path (CD updates, residuals, responsibilities, pruning) runs in
// libvest_cuda.so through the C-ABI of vest.h.  Types, member names,
// signatures, defaults and exception messages follow the reference; each
// function cites the reference declaration it replaces.
//
// Buffers stay caller-owned std::vectors, mutated in place like the reference.
// The tensor's device context (per-mode CSF in HBM) is cached per
// (tensor buffers, ranks) and reused across calls, the role the reference's
// ModeIndex plays; each call syncs the model host<->device (the "slow path").
// fit() keeps the model resident for the whole loop (the fast path).
// The `threads` arguments are accepted for source compatibility and ignored.
#pragma once

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <map>
#include <memory>
#include <mutex>
#include <span>
#include <stdexcept>
#include <string>
#include <thread>
#include <tuple>
#include <utility>
#include <vector>

#include "vest.h"

namespace sparsetuck {

using Coord = std::uint32_t;    // sparse_tensor.hpp:22
using EntryId = std::uint32_t;  // sparse_tensor.hpp:23

namespace b200_detail {
inline void check(int rc) {
  if (rc == VEST_OK) return;
  const std::string msg = vest_last_error();
  if (rc == VEST_EINVAL) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}
}  // namespace b200_detail

// ------------------------------------------------------------------ tensor --
// sparse_tensor.hpp:29-50
struct SparseTensor {
  std::vector<std::size_t> dims;
  std::vector<Coord> coords;  // nnz() * order(), entry-major
  std::vector<double> values;

  std::size_t order() const { return dims.size(); }
  std::size_t nnz() const { return values.size(); }
  const Coord* entry(std::size_t e) const { return coords.data() + e * dims.size(); }
  std::span<const Coord> entry_span(std::size_t e) const {
    return {coords.data() + e * dims.size(), dims.size()};
  }
  double frobenius_norm() const {
    double acc = 0.0;
    for (double v : values) acc += v * v;
    return std::sqrt(acc);
  }
};

// make_tensor (sparse_tensor.hpp:100-105): validated on the device (bounds
// and duplicate coordinates, the reference's messages) by a probe context.
inline SparseTensor make_tensor(std::vector<std::size_t> dims, std::vector<Coord> coords,
                                std::vector<double> values) {
  SparseTensor x{std::move(dims), std::move(coords), std::move(values)};
  if (x.order() == 0) throw std::invalid_argument("tensor order must be at least 1");
  for (std::size_t d : x.dims)
    if (d == 0) throw std::invalid_argument("tensor dimensions must be positive");
  if (x.coords.size() != x.nnz() * x.order())
    throw std::invalid_argument("coordinate buffer size does not match nnz * order");
  std::vector<std::uint64_t> d(x.dims.begin(), x.dims.end()), r(x.order(), 1);
  vest_ctx* h = nullptr;
  b200_detail::check(vest_ctx_create((int)x.order(), d.data(), x.nnz(), x.coords.data(), x.values.data(),
                                     r.data(), 0, &h));
  vest_ctx_destroy(h);
  return x;
}

// --------------------------------------------------------------- model ------
// tucker_model.hpp:21-47
struct TuckerModel {
  std::vector<std::size_t> dims;
  std::vector<std::size_t> ranks;
  std::vector<double> core;
  std::vector<std::uint8_t> core_mask;
  std::vector<std::vector<double>> factors;
  std::vector<std::vector<std::uint8_t>> factor_masks;

  std::size_t order() const { return dims.size(); }
  std::size_t core_size() const {
    std::size_t s = 1;
    for (std::size_t r : ranks) s *= r;
    return s;
  }
  double factor_at(std::size_t n, std::size_t i, std::size_t j) const { return factors[n][i * ranks[n] + j]; }
  std::size_t num_elements() const {
    std::size_t s = core_size();
    for (std::size_t n = 0; n < order(); ++n) s += dims[n] * ranks[n];
    return s;
  }
};

enum class Regularizer { LF, L1 };  // updates.hpp:15

// --------------------------------------------------------- device contexts --
namespace b200_detail {

struct Ctx {
  vest_ctx* h = nullptr;
  std::uint64_t fingerprint = 0;  // content of the tensor the CSF was built from
  std::uint64_t last_use = 0;
  ~Ctx() {
    if (h) vest_ctx_destroy(h);
  }
};

using Key = std::tuple<const void*, const void*, std::size_t, std::vector<std::size_t>, std::vector<std::size_t>>;

inline std::map<Key, std::shared_ptr<Ctx>>& registry() {
  static std::map<Key, std::shared_ptr<Ctx>> r;
  return r;
}
inline std::mutex& registry_mutex() {
  static std::mutex m;
  return m;
}

// 64-bit content hash of a byte range (8-byte words, multiply-rotate mixing;
// split across threads, partial hashes combined in order).
inline std::uint64_t hash_bytes(const void* p, std::size_t bytes) {
  const unsigned char* b = static_cast<const unsigned char*>(p);
  auto mix = [](std::uint64_t h, std::uint64_t w) {
    h ^= w * 0x9E3779B97F4A7C15ull;
    h = (h << 27) | (h >> 37);
    return h * 0xBF58476D1CE4E5B9ull + 0x94D049BB133111EBull;
  };
  auto range = [&](std::size_t lo, std::size_t hi) {
    std::uint64_t h = 0x2545F4914F6CDD1Dull ^ (hi - lo);
    std::size_t i = lo;
    for (; i + 8 <= hi; i += 8) {
      std::uint64_t w;
      std::memcpy(&w, b + i, 8);
      h = mix(h, w);
    }
    std::uint64_t t = 0;
    if (i < hi) std::memcpy(&t, b + i, hi - i);
    return mix(h, t);
  };
  const std::size_t kPart = std::size_t(1) << 24;  // 16 MB per task
  const std::size_t parts = (bytes + kPart - 1) / kPart;
  if (parts <= 1) return range(0, bytes);
  std::vector<std::uint64_t> ph(parts);
  const unsigned nt = std::max(1u, std::min<unsigned>(std::thread::hardware_concurrency(), (unsigned)parts));
  std::vector<std::thread> pool;
  for (unsigned t = 0; t < nt; ++t)
    pool.emplace_back([&, t] {
      for (std::size_t q = t; q < parts; q += nt) ph[q] = range(q * kPart, std::min(bytes, (q + 1) * kPart));
    });
  for (auto& th : pool) th.join();
  std::uint64_t h = 0;
  for (std::uint64_t v : ph) h = mix(h, v);
  return h;
}

inline std::uint64_t fingerprint(const SparseTensor& x) {
  return hash_bytes(x.coords.data(), x.coords.size() * sizeof(Coord)) * 31 +
         hash_bytes(x.values.data(), x.values.size() * sizeof(double));
}

// Device contexts kept at once (least recently used evicted first);
// SPARSETUCK_B200_MAX_CONTEXTS overrides.
inline std::size_t max_contexts() {
  if (const char* env = std::getenv("SPARSETUCK_B200_MAX_CONTEXTS")) {
    const long v = std::strtol(env, nullptr, 10);
    if (v > 0) return (std::size_t)v;
  }
  return 4;
}

// Context for (tensor, ranks); created (CSF built on the device) on first
// use.  The cache is keyed on the buffers AND verified against a content
// fingerprint on every lookup: a tensor edited in place, or a new tensor whose
// buffers reuse a freed address, gets a fresh context instead of a stale CSF.
// An empty tensor gives a model-only context.
inline std::shared_ptr<Ctx> context(const SparseTensor& x, const std::vector<std::size_t>& ranks) {
  std::lock_guard<std::mutex> g(registry_mutex());
  static std::uint64_t clock = 0;
  auto& reg = registry();
  Key k{x.coords.data(), x.values.data(), x.nnz(), x.dims, ranks};
  const std::uint64_t fp = fingerprint(x);
  auto it = reg.find(k);
  if (it != reg.end() && it->second->fingerprint != fp) {
    reg.erase(it);  // stale: the buffers at this address hold different data now
    it = reg.end();
  }
  if (it == reg.end()) {
    while (!reg.empty() && reg.size() >= max_contexts()) {
      auto lru = reg.begin();
      for (auto q = reg.begin(); q != reg.end(); ++q)
        if (q->second->last_use < lru->second->last_use) lru = q;
      reg.erase(lru);
    }
    auto c = std::make_shared<Ctx>();
    std::vector<std::uint64_t> d(x.dims.begin(), x.dims.end()), r(ranks.begin(), ranks.end());
    check(vest_ctx_create((int)x.order(), d.data(), x.nnz(), x.coords.data(), x.values.data(), r.data(), 0, &c->h));
    c->fingerprint = fp;
    it = reg.emplace(k, c).first;
  }
  it->second->last_use = ++clock;
  return it->second;  // the caller's reference keeps it alive across an eviction
}

// Number of cached device contexts (tests / diagnostics).
inline std::size_t cached_contexts() {
  std::lock_guard<std::mutex> g(registry_mutex());
  return registry().size();
}

}  // namespace b200_detail

// Frees every cached device context (their HBM); later calls rebuild them.
inline void release_device_contexts() {
  std::lock_guard<std::mutex> g(b200_detail::registry_mutex());
  b200_detail::registry().clear();
}

namespace b200_detail {

inline std::shared_ptr<Ctx> model_context(const TuckerModel& m) {
  static std::map<std::pair<std::vector<std::size_t>, std::vector<std::size_t>>, SparseTensor> empties;
  static std::mutex mu;
  const SparseTensor* x;
  {
    std::lock_guard<std::mutex> g(mu);
    auto& t = empties[{m.dims, m.ranks}];
    t.dims = m.dims;
    x = &t;
  }
  return context(*x, m.ranks);
}

inline void push(vest_ctx* h, const TuckerModel& m) {
  std::vector<const double*> f(m.order());
  std::vector<const std::uint8_t*> k(m.order());
  for (std::size_t n = 0; n < m.order(); ++n) f[n] = m.factors[n].data(), k[n] = m.factor_masks[n].data();
  check(vest_set_model(h, m.core.data(), m.core_mask.data(), f.data(), k.data()));
}

inline void pull(vest_ctx* h, TuckerModel& m) {
  std::vector<double*> f(m.order());
  std::vector<std::uint8_t*> k(m.order());
  for (std::size_t n = 0; n < m.order(); ++n) f[n] = m.factors[n].data(), k[n] = m.factor_masks[n].data();
  check(vest_get_model(h, m.core.data(), m.core_mask.data(), f.data(), k.data()));
}

inline std::shared_ptr<Ctx> bind(const TuckerModel& m, const SparseTensor& x) {
  if (m.dims != x.dims) throw std::invalid_argument("model/tensor shape mismatch");
  auto c = context(x, m.ranks);
  push(c->h, m);
  return c;
}

}  // namespace b200_detail

// ModeIndex / build_mode_index (sparse_tensor.hpp:109-137): the device CSF
// read back (same order: ids ascending within each slice).
struct ModeIndex {
  std::vector<std::vector<std::size_t>> offsets;
  std::vector<std::vector<EntryId>> ids;
  std::span<const EntryId> slice(std::size_t mode, Coord i) const {
    const auto& off = offsets[mode];
    return {ids[mode].data() + off[i], off[i + 1] - off[i]};
  }
};

inline ModeIndex build_mode_index(const SparseTensor& x) {
  const auto hold = b200_detail::context(x, std::vector<std::size_t>(x.order(), 1));
  vest_ctx* h = hold->h;
  ModeIndex idx;
  idx.offsets.resize(x.order());
  idx.ids.resize(x.order());
  for (std::size_t n = 0; n < x.order(); ++n) {
    std::vector<std::uint64_t> off(x.dims[n] + 1);
    idx.ids[n].resize(x.nnz());
    b200_detail::check(vest_get_mode_index(h, (int)n, off.data(), idx.ids[n].data()));
    idx.offsets[n].assign(off.begin(), off.end());
  }
  return idx;
}

// split_train_test (sparse_tensor.hpp:232-260)
inline std::pair<SparseTensor, SparseTensor> split_train_test(const SparseTensor& x, double test_fraction,
                                                              std::uint64_t seed) {
  if (!(test_fraction >= 0.0 && test_fraction <= 1.0)) throw std::invalid_argument("test_fraction must be in [0, 1]");
  std::vector<std::uint64_t> te(x.nnz() + 1), tr(x.nnz() + 1);
  std::uint64_t nte = 0, ntr = 0;
  b200_detail::check(vest_split_ids(x.nnz(), test_fraction, seed, te.data(), &nte, tr.data(), &ntr));
  auto take = [&](const std::vector<std::uint64_t>& ids, std::uint64_t n) {
    SparseTensor t;
    t.dims = x.dims;
    for (std::uint64_t q = 0; q < n; ++q) {
      const Coord* c = x.entry(ids[q]);
      t.coords.insert(t.coords.end(), c, c + x.order());
      t.values.push_back(x.values[ids[q]]);
    }
    return t;
  };
  return {take(tr, ntr), take(te, nte)};
}

// init_random (tucker_model.hpp:88-108): identical draws (same engine and
// distribution, same order).
inline TuckerModel init_random(const std::vector<std::size_t>& dims, const std::vector<std::size_t>& ranks,
                               std::uint64_t seed) {
  if (dims.size() != ranks.size()) throw std::invalid_argument("ranks/dims order mismatch");
  TuckerModel m;
  m.dims = dims;
  m.ranks = ranks;
  m.factors.resize(dims.size());
  m.factor_masks.resize(dims.size());
  std::vector<double*> f(dims.size());
  for (std::size_t n = 0; n < dims.size(); ++n) {
    m.factors[n].resize(dims[n] * ranks[n]);
    m.factor_masks[n].assign(m.factors[n].size(), 0);
    f[n] = m.factors[n].data();
  }
  m.core.resize(m.core_size());
  m.core_mask.assign(m.core.size(), 0);
  std::vector<std::uint64_t> d(dims.begin(), dims.end()), r(ranks.begin(), ranks.end());
  b200_detail::check(vest_init_random_host((int)dims.size(), d.data(), r.data(), seed, m.core.data(), f.data()));
  return m;
}

// reconstruct_entry (tucker_model.hpp:112-131) and predict (trainer.hpp:172-185)
inline std::vector<double> predict(const TuckerModel& m, std::span<const Coord> flat_coords) {
  const std::size_t n = m.order();
  if (n == 0 || flat_coords.size() % n != 0)
    throw std::invalid_argument("coordinate buffer must hold order() values per query");
  const auto hold = b200_detail::model_context(m);
  vest_ctx* h = hold->h;
  b200_detail::push(h, m);
  std::vector<double> out(flat_coords.size() / n);
  b200_detail::check(vest_predict(h, flat_coords.data(), out.size(), out.data()));
  return out;
}

inline double reconstruct_entry(const TuckerModel& m, const Coord* at) {
  return predict(m, std::span<const Coord>(at, m.order()))[0];
}
inline double reconstruct_entry(const TuckerModel& m, std::span<const Coord> at) {
  return reconstruct_entry(m, at.data());
}

// partial_reconstruct (tucker_model.hpp:136-154): the reconstruction restricted
// to the core cells whose mode-`mode` index is j (bit-identical).
inline double partial_reconstruct(const TuckerModel& m, const Coord* at, std::size_t mode, std::size_t j) {
  const auto hold = b200_detail::model_context(m);
  vest_ctx* h = hold->h;
  b200_detail::push(h, m);
  double out = 0.0;
  b200_detail::check(vest_partial_reconstruct(h, at, 1, (int)mode, j, &out));
  return out;
}

// Residuals / compute_residuals / reconstruction_error (tucker_model.hpp:161-188)
struct Residuals {
  std::vector<double> r;
  double sum_sq = 0.0;
  double x_norm = 0.0;
  double re = 0.0;
};

inline Residuals compute_residuals(const TuckerModel& m, const SparseTensor& x, int /*threads*/ = 1) {
  const auto hold = b200_detail::bind(m, x);
  vest_ctx* h = hold->h;
  Residuals res;
  res.r.resize(x.nnz());
  b200_detail::check(vest_compute_residuals(h, res.r.data(), &res.sum_sq, &res.x_norm, &res.re));
  return res;
}

inline double reconstruction_error(const TuckerModel& m, const SparseTensor& x) {
  const auto hold = b200_detail::bind(m, x);
  vest_ctx* h = hold->h;
  double re = 0.0;
  b200_detail::check(vest_compute_residuals(h, nullptr, nullptr, nullptr, &re));
  return re;
}

// sparsity / masked_fraction (tucker_model.hpp:192-207)
inline double sparsity(const TuckerModel& m) {
  const auto hold = b200_detail::model_context(m);
  vest_ctx* h = hold->h;
  b200_detail::push(h, m);
  double z = 0, k = 0;
  b200_detail::check(vest_sparsity(h, &z, &k));
  return z;
}
inline double masked_fraction(const TuckerModel& m) {
  const auto hold = b200_detail::model_context(m);
  vest_ctx* h = hold->h;
  b200_detail::push(h, m);
  double z = 0, k = 0;
  b200_detail::check(vest_sparsity(h, &z, &k));
  return k;
}

// normalize_columns (tucker_model.hpp:212-236)
inline void normalize_columns(TuckerModel& m) {
  const auto hold = b200_detail::model_context(m);
  vest_ctx* h = hold->h;
  b200_detail::push(h, m);
  b200_detail::check(vest_normalize_columns(h));
  b200_detail::pull(h, m);
}

// ------------------------------------------------------------- updates -------
// compute_delta (updates.hpp:35-59)
inline void compute_delta(const TuckerModel& m, const Coord* at, std::size_t mode, std::span<double> out) {
  const auto hold = b200_detail::model_context(m);
  vest_ctx* h = hold->h;
  b200_detail::push(h, m);
  b200_detail::check(vest_compute_delta(h, at, (int)mode, out.data()));
}
inline std::vector<double> compute_delta(const TuckerModel& m, const Coord* at, std::size_t mode) {
  std::vector<double> out(m.ranks[mode]);
  compute_delta(m, at, mode, out);
  return out;
}

// RowUpdateScratch (updates.hpp:17-30): per-call workspace of one row update.
struct RowUpdateScratch {
  std::vector<double> delta;   // J (the slice's last entry, as the reference leaves it)
  std::vector<double> gram;    // J x J, gram[t*J+j] = sum_e delta(t)*delta(j)
  std::vector<double> xdelta;  // J, sum_e x[e]*delta(j)

  void reset(std::size_t J) {
    delta.assign(J, 0.0);
    gram.assign(J * J, 0.0);
    xdelta.assign(J, 0.0);
  }
};

namespace b200_detail {
inline void row_stats(vest_ctx* h, std::size_t mode, std::size_t i, std::size_t J, RowUpdateScratch& s) {
  s.reset(J);
  check(vest_compute_row_stats(h, (int)mode, i, s.gram.data(), s.xdelta.data(), s.delta.data()));
}
// only row i of factor `mode` changes in a row update: read back just that row
inline void pull_row(vest_ctx* h, TuckerModel& m, std::size_t mode, std::size_t i) {
  check(vest_get_factor_rows(h, (int)mode, i, 1, m.factors[mode].data() + i * m.ranks[mode]));
}
inline void check_row(const TuckerModel& m, std::size_t mode, std::size_t i) {
  if (mode >= m.order() || i >= m.dims[mode]) throw std::invalid_argument("row out of range");
}
}  // namespace b200_detail

// compute_row_stats (updates.hpp:64-79): gram and xdelta over the row's
// observed entries, bit-identical to the reference (device, reference order).
inline void compute_row_stats(const TuckerModel& m, const SparseTensor& x, const ModeIndex&, std::size_t mode,
                              std::size_t i, RowUpdateScratch& s) {
  b200_detail::check_row(m, mode, i);
  const auto hold = b200_detail::bind(m, x);
  b200_detail::row_stats(hold->h, mode, i, m.ranks[mode], s);
}

// update_factor_row_lf / _l1 (updates.hpp:88-151); the scratch overloads
// leave the row's statistics in `s` as the reference does.
inline void update_factor_row_lf(TuckerModel& m, const SparseTensor& x, const ModeIndex& idx, std::size_t mode,
                                 std::size_t i, double lambda, RowUpdateScratch& s) {
  b200_detail::check_row(m, mode, i);
  if (!idx.offsets.empty() && idx.slice(mode, static_cast<Coord>(i)).empty()) return;  // updates.hpp:91
  const auto hold = b200_detail::bind(m, x);
  vest_ctx* h = hold->h;
  b200_detail::row_stats(h, mode, i, m.ranks[mode], s);
  b200_detail::check(vest_update_factor_row(h, VEST_LF, (int)mode, i, lambda));
  b200_detail::pull_row(h, m, mode, i);
}
inline void update_factor_row_l1(TuckerModel& m, const SparseTensor& x, const ModeIndex&, std::size_t mode,
                                 std::size_t i, double lambda, RowUpdateScratch& s) {
  b200_detail::check_row(m, mode, i);
  const auto hold = b200_detail::bind(m, x);
  vest_ctx* h = hold->h;
  b200_detail::row_stats(h, mode, i, m.ranks[mode], s);
  b200_detail::check(vest_update_factor_row(h, VEST_L1, (int)mode, i, lambda));
  b200_detail::pull_row(h, m, mode, i);
}
inline void update_factor_row_lf(TuckerModel& m, const SparseTensor& x, const ModeIndex&, std::size_t mode,
                                 std::size_t i, double lambda) {
  b200_detail::check_row(m, mode, i);
  const auto hold = b200_detail::bind(m, x);
  vest_ctx* h = hold->h;
  b200_detail::check(vest_update_factor_row(h, VEST_LF, (int)mode, i, lambda));
  b200_detail::pull_row(h, m, mode, i);
}
inline void update_factor_row_l1(TuckerModel& m, const SparseTensor& x, const ModeIndex&, std::size_t mode,
                                 std::size_t i, double lambda) {
  b200_detail::check_row(m, mode, i);
  const auto hold = b200_detail::bind(m, x);
  vest_ctx* h = hold->h;
  b200_detail::check(vest_update_factor_row(h, VEST_L1, (int)mode, i, lambda));
  b200_detail::pull_row(h, m, mode, i);
}

// update_all_factors (updates.hpp:157-175)
inline void update_all_factors(TuckerModel& m, const SparseTensor& x, const ModeIndex&, Regularizer reg,
                               double lambda, int /*threads*/ = 1) {
  const auto hold = b200_detail::bind(m, x);
  vest_ctx* h = hold->h;
  b200_detail::check(vest_update_all_factors(h, reg == Regularizer::LF ? VEST_LF : VEST_L1, lambda));
  b200_detail::pull(h, m);
}

// update_core_lf / _l1 (updates.hpp:253-262)
inline void update_core_lf(TuckerModel& m, const SparseTensor& x, double lambda, int /*threads*/ = 1) {
  const auto hold = b200_detail::bind(m, x);
  vest_ctx* h = hold->h;
  b200_detail::check(vest_update_core(h, VEST_LF, lambda));
  b200_detail::pull(h, m);
}
inline void update_core_l1(TuckerModel& m, const SparseTensor& x, double lambda, int /*threads*/ = 1) {
  const auto hold = b200_detail::bind(m, x);
  vest_ctx* h = hold->h;
  b200_detail::check(vest_update_core(h, VEST_L1, lambda));
  b200_detail::pull(h, m);
}

// ------------------------------------------------------------- pruning -------
// PruneSchedule (pruning.hpp:20-33)
struct PruneSchedule {
  double init_pr = 0.01;
  double max_pr = 0.1;
  void validate() const {
    if (!(init_pr > 0.0 && init_pr <= max_pr && max_pr < 1.0))
      throw std::invalid_argument("require 0 < init_pr <= max_pr < 1");
  }
  double rate(std::size_t iter) const {
    if (iter == 0) throw std::invalid_argument("iterations are 1-based");
    return std::min(init_pr * double(iter), max_pr);
  }
};

enum class StopMode { Manual, Auto };  // pruning.hpp:35

// StopController (pruning.hpp:45-81)
struct StopController {
  StopMode mode = StopMode::Manual;
  double target_sparsity = 0.0;
  double elbow_threshold = 0.05;

  bool should_prune(double current_sparsity, double re, double pr) {
    if (stopped_) return false;
    if (re == 0.0) return false;
    if (mode == StopMode::Manual) {
      if (current_sparsity >= target_sparsity) {
        stopped_ = true;
        return false;
      }
      return true;
    }
    if (history_.size() >= 2) {
      const double prev = history_[history_.size() - 1];
      const double prev2 = history_[history_.size() - 2];
      if ((re + prev2 - 2.0 * prev) / pr > elbow_threshold) {
        stopped_ = true;
        return false;
      }
    }
    return true;
  }
  void record_prune_event(double re) { history_.push_back(re); }
  bool stopped() const { return stopped_; }

 private:
  bool stopped_ = false;
  std::vector<double> history_;
};

// ResponsibilityTable / compute_*_responsibilities (pruning.hpp:83-191).
// The residual used is the device residual of m on x -- what the reference
// is always handed (trainer.hpp:127,136).
struct ResponsibilityTable {
  std::vector<double> core;
  std::vector<std::vector<double>> factors;
  double base_re = 0.0;
};

inline ResponsibilityTable compute_responsibilities(const TuckerModel& m, const SparseTensor& x, const ModeIndex&,
                                                    const Residuals&, int /*threads*/ = 1) {
  const auto hold = b200_detail::bind(m, x);
  vest_ctx* h = hold->h;
  ResponsibilityTable t;
  t.core.resize(m.core_size());
  t.factors.resize(m.order());
  std::vector<double*> f(m.order());
  for (std::size_t n = 0; n < m.order(); ++n) {
    t.factors[n].resize(m.dims[n] * m.ranks[n]);
    f[n] = t.factors[n].data();
  }
  b200_detail::check(vest_compute_responsibilities(h, t.core.data(), f.data(), &t.base_re));
  return t;
}

inline std::vector<double> compute_core_responsibilities(const TuckerModel& m, const SparseTensor& x,
                                                         const Residuals& res, int threads = 1) {
  return compute_responsibilities(m, x, ModeIndex{}, res, threads).core;
}

inline std::vector<double> compute_factor_responsibilities(const TuckerModel& m, const SparseTensor& x,
                                                           const ModeIndex& idx, std::size_t mode,
                                                           const Residuals& res, int threads = 1) {
  return compute_responsibilities(m, x, idx, res, threads).factors[mode];
}

// PruneCounts / prune_step (pruning.hpp:193-247): device radix select
struct PruneCounts {
  std::size_t core = 0;
  std::vector<std::size_t> factors;
  std::size_t total() const {
    std::size_t s = core;
    for (std::size_t f : factors) s += f;
    return s;
  }
};

inline PruneCounts prune_step(TuckerModel& m, const ResponsibilityTable& t, double pr) {
  if (!(pr >= 0.0 && pr < 1.0)) throw std::invalid_argument("prune rate must be in [0, 1)");
  const auto hold = b200_detail::model_context(m);
  vest_ctx* h = hold->h;
  b200_detail::push(h, m);
  std::vector<const double*> f(m.order());
  for (std::size_t n = 0; n < m.order(); ++n) f[n] = t.factors[n].data();
  std::vector<std::uint64_t> c(1 + m.order());
  b200_detail::check(vest_prune_step(h, pr, t.core.data(), f.data(), c.data()));
  b200_detail::pull(h, m);
  PruneCounts out;
  out.core = c[0];
  for (std::size_t n = 0; n < m.order(); ++n) out.factors.push_back(c[1 + n]);
  return out;
}

// -------------------------------------------------------------- trainer ------
// resolve_threads / TrainConfig / reports / fit (trainer.hpp:20-190)
inline int resolve_threads(int requested) {
  if (requested > 0) return requested;
  if (const char* env = std::getenv("SPARSETUCK_THREADS")) {
    char* end = nullptr;
    const long v = std::strtol(env, &end, 10);
    if (end != env && *end == '\0' && v > 0) return static_cast<int>(v);
  }
  const unsigned hc = std::thread::hardware_concurrency();
  return hc > 0 ? static_cast<int>(hc) : 1;
}

struct TrainConfig {
  std::vector<std::size_t> ranks;
  Regularizer reg = Regularizer::LF;
  double lambda = 0.01;
  StopMode mode = StopMode::Manual;
  double target_sparsity = 0.0;
  double elbow_threshold = 0.05;
  PruneSchedule schedule{};
  std::size_t max_iters = 100;
  double tol = 1e-4;
  int threads = 0;
  std::uint64_t seed = 0;
  bool normalize_output = true;
};

struct IterationReport {
  std::size_t iter = 0;
  double re = 0.0;
  double prune_rate = 0.0;
  bool pruned = false;
  std::size_t pruned_core = 0;
  std::vector<std::size_t> pruned_factors;
  double sparsity = 0.0;
  double masked = 0.0;
  double wall_ms = 0.0;
};

struct TrainReport {
  std::vector<IterationReport> iterations;
  bool converged = false;
  std::size_t iters = 0;
  double final_re = 0.0;
  double final_sparsity = 0.0;
  double final_masked = 0.0;
  double elapsed_sec = 0.0;
};

struct FitResult {
  TuckerModel model;
  TrainReport report;
};

namespace b200_detail {
inline void check_config(const SparseTensor& x, const TrainConfig& cfg) {  // trainer.hpp:80-93
  if (cfg.ranks.size() != x.order()) throw std::invalid_argument("ranks order mismatch");
  for (std::size_t r : cfg.ranks)
    if (r == 0) throw std::invalid_argument("ranks must be positive");
  if (!(cfg.lambda >= 0.0)) throw std::invalid_argument("lambda must be nonnegative");
  if (!(cfg.tol >= 0.0)) throw std::invalid_argument("tol must be nonnegative");
  if (cfg.max_iters == 0) throw std::invalid_argument("max_iters must be positive");
  if (!(cfg.target_sparsity >= 0.0 && cfg.target_sparsity < 1.0))
    throw std::invalid_argument("target sparsity must be in [0, 1)");
  cfg.schedule.validate();
  if (x.nnz() == 0) throw std::invalid_argument("empty tensor");
  if (x.frobenius_norm() == 0.0) throw std::invalid_argument("tensor values are all zero; nothing to fit");
}
}  // namespace b200_detail

// fit (trainer.hpp:103-168): the model stays in HBM for the whole loop; the
// host reads back re, sparsity and prune counts per iteration for the
// schedule / stop controller (host control, as in the reference).
inline FitResult fit(const SparseTensor& x, const TrainConfig& cfg) {
  b200_detail::check_config(x, cfg);
  const auto t_start = std::chrono::steady_clock::now();
  std::vector<std::uint64_t> d(x.dims.begin(), x.dims.end()), r(cfg.ranks.begin(), cfg.ranks.end());
  b200_detail::Ctx ctx;
  b200_detail::check(vest_ctx_create((int)x.order(), d.data(), x.nnz(), x.coords.data(), x.values.data(), r.data(),
                                     0, &ctx.h));
  b200_detail::check(vest_init_random(ctx.h, cfg.seed));
  const int reg = cfg.reg == Regularizer::LF ? VEST_LF : VEST_L1;
  StopController ctrl;
  ctrl.mode = cfg.mode;
  ctrl.target_sparsity = cfg.target_sparsity;
  ctrl.elbow_threshold = cfg.elbow_threshold;
  FitResult out;
  double prev_re = std::numeric_limits<double>::infinity();
  for (std::size_t t = 1; t <= cfg.max_iters; ++t) {
    const auto it_start = std::chrono::steady_clock::now();
    double re = 0.0;
    b200_detail::check(vest_cd_iteration(ctx.h, reg, cfg.lambda, &re));
    const double pr = cfg.schedule.rate(t);
    IterationReport rec;
    rec.iter = t;
    rec.re = re;
    rec.prune_rate = pr;
    rec.pruned_factors.assign(x.order(), 0);
    double zero = 0.0, masked = 0.0;
    b200_detail::check(vest_sparsity(ctx.h, &zero, &masked));
    if (ctrl.should_prune(zero, re, pr)) {
      double base = 0.0;
      b200_detail::check(vest_compute_responsibilities(ctx.h, nullptr, nullptr, &base));
      std::vector<std::uint64_t> c(1 + x.order());
      b200_detail::check(vest_prune_step(ctx.h, pr, nullptr, nullptr, c.data()));
      std::size_t total = 0;
      for (auto v : c) total += v;
      if (total > 0) {
        ctrl.record_prune_event(re);
        rec.pruned = true;
        rec.pruned_core = c[0];
        for (std::size_t n = 0; n < x.order(); ++n) rec.pruned_factors[n] = c[1 + n];
      }
    }
    b200_detail::check(vest_sparsity(ctx.h, &rec.sparsity, &rec.masked));
    rec.wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - it_start).count();
    out.report.iterations.push_back(std::move(rec));
    if (std::abs(prev_re - re) < cfg.tol) {
      out.report.converged = true;
      break;
    }
    prev_re = re;
  }
  if (cfg.normalize_output) b200_detail::check(vest_normalize_columns(ctx.h));
  out.report.iters = out.report.iterations.size();
  b200_detail::check(vest_compute_residuals(ctx.h, nullptr, nullptr, nullptr, &out.report.final_re));
  b200_detail::check(vest_sparsity(ctx.h, &out.report.final_sparsity, &out.report.final_masked));
  TuckerModel& m = out.model;
  m.dims = x.dims;
  m.ranks = cfg.ranks;
  m.core.resize(m.core_size());
  m.core_mask.resize(m.core_size());
  m.factors.resize(x.order());
  m.factor_masks.resize(x.order());
  for (std::size_t n = 0; n < x.order(); ++n) {
    m.factors[n].resize(x.dims[n] * cfg.ranks[n]);
    m.factor_masks[n].resize(x.dims[n] * cfg.ranks[n]);
  }
  b200_detail::pull(ctx.h, m);
  out.report.elapsed_sec = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
  return out;
}

// evaluate_test (trainer.hpp:188-190)
inline double evaluate_test(const TuckerModel& m, const SparseTensor& test) {
  if (m.dims != test.dims) throw std::invalid_argument("model/tensor shape mismatch");
  const auto hold = b200_detail::model_context(m);
  vest_ctx* h = hold->h;
  b200_detail::push(h, m);
  double re = 0.0;
  b200_detail::check(vest_evaluate(h, test.coords.data(), test.values.data(), test.nnz(), &re));
  return re;
}

// Prune-rate sweep (BASELINE config 5's protocol: rates 0.1..0.9 on a train /
// test split; the manual counterpart of the auto mode's elbow search,
// pruning.hpp:45-81).  For each rate, from the SAME trained model: score
// responsibilities on the training entries (pruning.hpp:181-191),
// prune_step(rate) (pruning.hpp:234-247), then the relative error on the
// training entries (tucker_model.hpp:186-188) and on the held-out entries
// (trainer.hpp:188-190).  Every rate starts from the same model, so the
// responsibility table is scored once and reused by each rate's prune_step; the evaluations are the inner loop.  The caller's model is not
// modified.
struct RateResult {
  double rate = 0.0;
  PruneCounts pruned;
  double sparsity = 0.0;
  double train_re = 0.0;
  double test_re = 0.0;
};

inline std::vector<RateResult> prune_rate_sweep(const TuckerModel& m, const SparseTensor& train,
                                                const SparseTensor& test, std::span<const double> rates) {
  if (m.dims != train.dims || m.dims != test.dims) throw std::invalid_argument("model/tensor shape mismatch");
  for (double pr : rates)
    if (!(pr >= 0.0 && pr < 1.0)) throw std::invalid_argument("prune rate must be in [0, 1)");
  const ResponsibilityTable t = compute_responsibilities(m, train, ModeIndex{}, Residuals{});
  const auto hold = b200_detail::bind(m, train);  // the same cached context
  vest_ctx* h = hold->h;
  std::vector<const double*> f(m.order());
  for (std::size_t n = 0; n < m.order(); ++n) f[n] = t.factors[n].data();
  std::vector<RateResult> out;
  for (double pr : rates) {
    b200_detail::push(h, m);
    std::vector<std::uint64_t> c(1 + m.order());
    b200_detail::check(vest_prune_step(h, pr, t.core.data(), f.data(), c.data()));
    RateResult r;
    r.rate = pr;
    r.pruned.core = c[0];
    for (std::size_t n = 0; n < m.order(); ++n) r.pruned.factors.push_back(c[1 + n]);
    double masked = 0.0;
    b200_detail::check(vest_sparsity(h, &r.sparsity, &masked));
    b200_detail::check(vest_compute_residuals(h, nullptr, nullptr, nullptr, &r.train_re));
    b200_detail::check(vest_evaluate(h, test.coords.data(), test.values.data(), test.nnz(), &r.test_re));
    out.push_back(std::move(r));
  }
  return out;
}

// ------------------------------------------------------------ data formats --
// load_coo / save_coo (sparse_tensor.hpp:139-228), save_model / load_model
// (model_io.hpp:22-104): vest_io.cpp, parallel, byte-compatible files and the
// reference's exceptions and messages.
namespace b200_detail {
inline void io_check(int rc) {
  if (rc == VEST_OK) return;
  const std::string msg = vest_io_last_error();
  if (rc == VEST_EINVAL) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}
inline SparseTensor coo_take(vest_coo* h) {
  std::unique_ptr<vest_coo, void (*)(vest_coo*)> g(h, vest_coo_free);
  int order = 0;
  std::uint64_t nnz = 0;
  io_check(vest_coo_info(h, &order, &nnz, nullptr, nullptr, nullptr));
  std::vector<std::uint64_t> d(order);
  const std::uint32_t* c = nullptr;
  const double* v = nullptr;
  io_check(vest_coo_info(h, nullptr, nullptr, d.data(), &c, &v));
  SparseTensor x;
  x.dims.assign(d.begin(), d.end());
  x.coords.assign(c, c + nnz * order);
  x.values.assign(v, v + nnz);
  return x;
}
}  // namespace b200_detail

inline SparseTensor load_coo(const std::string& path, bool one_based = false) {
  vest_coo* h = nullptr;
  b200_detail::io_check(vest_coo_load(path.c_str(), one_based ? 1 : 0, 0, &h));
  return b200_detail::coo_take(h);
}

inline void save_coo(const SparseTensor& x, const std::string& path) {
  std::vector<std::uint64_t> d(x.dims.begin(), x.dims.end());
  b200_detail::io_check(vest_coo_save(path.c_str(), (int)x.order(), d.data(), x.nnz(), x.coords.data(),
                                      x.values.data()));
}

inline void save_model(const TuckerModel& m, const std::string& dir) {
  std::vector<std::uint64_t> d(m.dims.begin(), m.dims.end()), r(m.ranks.begin(), m.ranks.end());
  std::vector<const double*> f(m.order());
  for (std::size_t n = 0; n < m.order(); ++n) f[n] = m.factors[n].data();
  b200_detail::io_check(vest_model_save(dir.c_str(), (int)m.order(), d.data(), r.data(), m.core.data(), f.data()));
}

inline TuckerModel load_model(const std::string& dir) {
  vest_model_file* h = nullptr;
  b200_detail::io_check(vest_model_load(dir.c_str(), &h));
  std::unique_ptr<vest_model_file, void (*)(vest_model_file*)> g(h, vest_model_file_free);
  int order = 0;
  b200_detail::io_check(vest_model_file_info(h, &order, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr));
  std::vector<std::uint64_t> d(order), r(order);
  const double* core = nullptr;
  const std::uint8_t* cm = nullptr;
  std::vector<const double*> f(order);
  std::vector<const std::uint8_t*> k(order);
  b200_detail::io_check(vest_model_file_info(h, nullptr, d.data(), r.data(), &core, &cm, f.data(), k.data()));
  TuckerModel m;
  m.dims.assign(d.begin(), d.end());
  m.ranks.assign(r.begin(), r.end());
  m.core.assign(core, core + m.core_size());
  m.core_mask.assign(cm, cm + m.core_size());
  m.factors.resize(order);
  m.factor_masks.resize(order);
  for (int n = 0; n < order; ++n) {
    m.factors[n].assign(f[n], f[n] + m.dims[n] * m.ranks[n]);
    m.factor_masks[n].assign(k[n], k[n] + m.dims[n] * m.ranks[n]);
  }
  return m;
}

}  // namespace sparsetuck
