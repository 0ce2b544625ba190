// SPDX-License-Identifier: Apache-2.0
// C++ drop-in check: code written against the reference's sparsetuck:: API
// compiled against include/sparsetuck_b200.hpp (the B200 path), with the
// reference suite's own known answers (tests/test_updates.cpp:186-220,
// tests/test_pruning.cpp:179-231, tests/test_sparse_tensor.cpp:173-211) and a
// fit() trajectory checked against the C restatement oracle (test infra).
// Built and run by tests/test_gpu_cpp.py.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <random>
#include <stdexcept>
#include <string>

#include "../../oracle/vest_oracle.h"
#include "sparsetuck_b200.hpp"

using namespace sparsetuck;

static int failures = 0;
#define CHECK(cond)                                                      \
  do {                                                                   \
    if (!(cond)) {                                                       \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);        \
      ++failures;                                                        \
    }                                                                    \
  } while (0)

static TuckerModel one_cell() {
  TuckerModel b;
  b.dims = {1, 1};
  b.ranks = {1, 1};
  b.core = {1.0};
  b.core_mask = {0};
  b.factors = {{1.0}, {1.0}};
  b.factor_masks = {{0}, {0}};
  return b;
}

int main() {
  // known closed-form updates on a one-cell problem
  {
    const auto x = make_tensor({1, 1}, {0, 0}, {2.0});
    const ModeIndex idx = build_mode_index(x);
    auto m = one_cell();
    update_factor_row_lf(m, x, idx, 0, 0, 1.0);
    CHECK(std::abs(m.factors[0][0] - 1.0) <= 1e-15);
    m = one_cell();
    update_factor_row_l1(m, x, idx, 0, 0, 1.0);
    CHECK(std::abs(m.factors[0][0] - 1.5) <= 1e-15);
    const auto x3 = make_tensor({1, 1}, {0, 0}, {3.0});
    m = one_cell();
    update_core_l1(m, x3, 1.0, 1);
    CHECK(std::abs(m.core[0] - 2.5) <= 1e-15);
    m = one_cell();
    update_core_lf(m, x3, 1.0, 1);
    CHECK(std::abs(m.core[0] - 1.5) <= 1e-15);
  }
  // prune ties / floor / saturation
  {
    auto m = init_random({2, 2}, {2, 2}, 3);
    ResponsibilityTable t;
    t.core = {0.5, 0.2, 0.2, 0.9};
    t.factors = {{0.1, 0.4, 0.4, 0.4}, {0.7, 0.6, 0.5, 0.4}};
    const PruneCounts c = prune_step(m, t, 0.5);
    CHECK(c.core == 2 && c.total() == 6);
    CHECK((m.core_mask == std::vector<std::uint8_t>{0, 1, 1, 0}));
    CHECK((m.factor_masks[0] == std::vector<std::uint8_t>{1, 1, 0, 0}));
    CHECK((m.factor_masks[1] == std::vector<std::uint8_t>{0, 0, 1, 1}));
    bool threw = false;
    try {
      prune_step(m, t, 1.0);
    } catch (const std::invalid_argument&) {
      threw = true;
    }
    CHECK(threw);
  }
  // validation messages
  {
    bool dup = false;
    try {
      make_tensor({3, 3}, {1, 2, 0, 0, 1, 2}, {1.0, 2.0, 3.0});
    } catch (const std::invalid_argument& e) {
      dup = std::string(e.what()).find("duplicate") != std::string::npos;
    }
    CHECK(dup);
  }
  // split sizes (test_sparse_tensor.cpp:173-211 uses 1200 entries, 10%)
  {
    SparseTensor x;
    x.dims = {1200};
    for (Coord e = 0; e < 1200; ++e) x.coords.push_back(e), x.values.push_back(1.0 + e);
    auto [tr, te] = split_train_test(x, 0.1, 5);
    CHECK(tr.nnz() == 1080 && te.nnz() == 120);
  }
  // fit(): device-resident loop vs the oracle's CD iterations (no pruning)
  {
    std::mt19937_64 rng(11);
    std::vector<Coord> coords;
    std::vector<double> values;
    std::uniform_int_distribution<int> pi(0, 39), pj(0, 29), pk(0, 19);
    std::uniform_real_distribution<double> u(0.0, 1.0);
    std::vector<char> seen(40 * 30 * 20, 0);
    while (values.size() < 3000) {
      const int i = pi(rng), j = pj(rng), k = pk(rng);
      if (seen[(i * 30 + j) * 20 + k]) continue;
      seen[(i * 30 + j) * 20 + k] = 1;
      coords.insert(coords.end(), {Coord(i), Coord(j), Coord(k)});
      values.push_back(u(rng));
    }
    const auto x = make_tensor({40, 30, 20}, coords, values);
    TrainConfig cfg;
    cfg.ranks = {5, 5, 5};
    cfg.max_iters = 6;
    cfg.tol = 0.0;
    cfg.seed = 9;
    cfg.mode = StopMode::Manual;
    cfg.target_sparsity = 0.0;  // stop controller latches at once: no pruning
    cfg.normalize_output = false;
    const FitResult r = fit(x, cfg);
    CHECK(r.report.iters == 6);
    vo_session* s = nullptr;
    const std::uint64_t d[3] = {40, 30, 20}, rk[3] = {5, 5, 5};
    CHECK(vo_create(3, d, x.nnz(), x.coords.data(), x.values.data(), rk, &s) == 0);
    vo_init_random(s, 9);
    for (std::size_t t = 0; t < 6; ++t) {
      double re = 0.0;
      vo_cd_iteration(s, 0, cfg.lambda, 1, &re);
      const double got = r.report.iterations[t].re;
      CHECK(std::abs(got - re) <= 1e-6 * re);
    }
    std::vector<double> core(125);
    vo_get_model(s, core.data(), nullptr, nullptr, nullptr);
    double num = 0, den = 0;
    for (std::size_t q = 0; q < 125; ++q) num += (core[q] - r.model.core[q]) * (core[q] - r.model.core[q]), den += core[q] * core[q];
    CHECK(std::sqrt(num / den) <= 1e-6);
    vo_destroy(s);
    // the slow path (per-call model sync) agrees with fit's resident loop
    TuckerModel m = init_random(x.dims, cfg.ranks, 9);
    const ModeIndex idx = build_mode_index(x);
    for (int t = 0; t < 6; ++t) {
      update_all_factors(m, x, idx, Regularizer::LF, cfg.lambda, 8);
      update_core_lf(m, x, cfg.lambda, 8);
    }
    CHECK(std::abs(reconstruction_error(m, x) - r.report.iterations[5].re) <= 1e-9 * r.report.iterations[5].re);
  }
  // prune_rate_sweep (BASELINE config 5's protocol): per rate, prune the same
  // trained model and report train / held-out error -- against the oracle's
  // compute_responsibilities + prune_step + residuals on the same split
  {
    std::mt19937_64 rng(23);
    std::vector<Coord> coords;
    std::vector<double> values;
    std::uniform_int_distribution<int> pi(0, 29), pj(0, 24), pk(0, 19);
    std::uniform_real_distribution<double> u(0.0, 1.0);
    std::vector<char> seen(30 * 25 * 20, 0);
    while (values.size() < 4000) {
      const int i = pi(rng), j = pj(rng), k = pk(rng);
      if (seen[(i * 25 + j) * 20 + k]) continue;
      seen[(i * 25 + j) * 20 + k] = 1;
      coords.insert(coords.end(), {Coord(i), Coord(j), Coord(k)});
      values.push_back(u(rng));
    }
    const auto x = make_tensor({30, 25, 20}, coords, values);
    const auto [tr, te] = split_train_test(x, 0.1, 3);
    TuckerModel m = init_random(x.dims, {4, 3, 5}, 2);
    const ModeIndex idx = build_mode_index(tr);
    for (int t = 0; t < 3; ++t) {
      update_all_factors(m, tr, idx, Regularizer::LF, 0.01, 1);
      update_core_lf(m, tr, 0.01, 1);
    }
    const TuckerModel keep = m;
    const std::vector<double> rates = {0.1, 0.5, 0.9};
    const auto sweep = prune_rate_sweep(m, tr, te, rates);
    CHECK(sweep.size() == 3);
    CHECK(m.core == keep.core && m.factors == keep.factors && m.core_mask == keep.core_mask);
    vo_session* s = nullptr;
    const std::uint64_t d[3] = {30, 25, 20}, rk[3] = {4, 3, 5};
    CHECK(vo_create(3, d, tr.nnz(), tr.coords.data(), tr.values.data(), rk, &s) == 0);
    double te_norm = 0.0;
    for (double v : te.values) te_norm += v * v;
    te_norm = std::sqrt(te_norm);
    double last_sparsity = -1.0;
    for (std::size_t i = 0; i < sweep.size(); ++i) {
      const double* f[3] = {keep.factors[0].data(), keep.factors[1].data(), keep.factors[2].data()};
      const std::uint8_t* fm[3] = {keep.factor_masks[0].data(), keep.factor_masks[1].data(), keep.factor_masks[2].data()};
      CHECK(vo_set_model(s, keep.core.data(), keep.core_mask.data(), f, fm) == 0);
      double ss = 0, xn = 0, re = 0;
      vo_compute_residuals(s, 1, nullptr, &ss, &xn, &re);
      vo_compute_responsibilities(s, 1, nullptr, nullptr);
      std::uint64_t cnt[4] = {};
      vo_prune_step(s, rates[i], nullptr, nullptr, cnt);
      vo_compute_residuals(s, 1, nullptr, &ss, &xn, &re);
      std::vector<double> pred(te.nnz());
      vo_reconstruct(s, te.coords.data(), te.nnz(), pred.data());
      double err = 0.0;
      for (std::size_t e = 0; e < te.nnz(); ++e) err += (te.values[e] - pred[e]) * (te.values[e] - pred[e]);
      const double test_re = std::sqrt(err) / te_norm;
      const RateResult& g = sweep[i];
      CHECK(g.rate == rates[i]);
      CHECK(g.pruned.core == cnt[0] && g.pruned.factors[0] == cnt[1] && g.pruned.factors[1] == cnt[2] &&
            g.pruned.factors[2] == cnt[3]);
      CHECK(std::abs(g.train_re - re) <= 1e-6 * re);
      CHECK(std::abs(g.test_re - test_re) <= 1e-6 * test_re);
      CHECK(std::abs(g.sparsity - vo_sparsity(s)) <= 1e-15);
      CHECK(g.sparsity > last_sparsity);
      last_sparsity = g.sparsity;
    }
    vo_destroy(s);
  }
  {  // data formats: model directory and COO text round trips (vest_io.cpp)
    TuckerModel m = init_random({40, 30, 20}, {3, 2, 4}, 9);
    m.core[1] = 0.0;
    const std::string dir = "/tmp/vest_mirror_model";
    save_model(m, dir);
    const TuckerModel back = load_model(dir);
    CHECK(back.dims == m.dims && back.ranks == m.ranks && back.core == m.core && back.factors == m.factors);
    CHECK(back.core_mask[1] == 1 && back.core_mask[0] == 0);
    SparseTensor x = make_tensor({5, 6}, {0, 1, 4, 5, 2, 2}, {0.25, -1e-300, 3.0});
    save_coo(x, "/tmp/vest_mirror.coo");
    const SparseTensor y = load_coo("/tmp/vest_mirror.coo");
    CHECK(y.dims == x.dims && y.coords == x.coords && y.values == x.values);
    bool threw = false;
    try {
      load_coo("/tmp/vest_mirror_absent.coo");
    } catch (const std::runtime_error& e) {
      threw = std::string(e.what()).find("cannot open") != std::string::npos;
    }
    CHECK(threw);
  }
  // RowUpdateScratch / compute_row_stats / scratch overloads / partial_reconstruct
  // (updates.hpp:17-30,64-139; tucker_model.hpp:136-154) vs the C restatement,
  // bit for bit
  {
    std::mt19937_64 rng(5);
    std::vector<Coord> coords;
    std::vector<double> values;
    std::uniform_int_distribution<int> pi(0, 24), pj(0, 7), pk(0, 6);
    std::uniform_real_distribution<double> u(-1.0, 2.0);
    std::vector<char> seen(25 * 8 * 7, 0);
    while (values.size() < 500) {
      const int i = pi(rng) % 20, j = pj(rng), k = pk(rng);  // rows 20..24 of mode 0 stay empty
      if (seen[(i * 8 + j) * 7 + k]) continue;
      seen[(i * 8 + j) * 7 + k] = 1;
      coords.insert(coords.end(), {Coord(i), Coord(j), Coord(k)});
      values.push_back(u(rng));
    }
    const auto x = make_tensor({25, 8, 7}, coords, values);
    const ModeIndex idx = build_mode_index(x);
    TuckerModel m = init_random(x.dims, {4, 3, 2}, 21);
    m.core[5] = 0.0, m.core_mask[5] = 1;
    m.core[11] = 0.0;  // an incidental zero: skipped like a masked one
    vo_session* s = nullptr;
    const std::uint64_t d[3] = {25, 8, 7}, rk[3] = {4, 3, 2};
    CHECK(vo_create(3, d, x.nnz(), x.coords.data(), x.values.data(), rk, &s) == 0);
    std::vector<const double*> fp(3);
    std::vector<const std::uint8_t*> mp(3);
    for (int n = 0; n < 3; ++n) fp[n] = m.factors[n].data(), mp[n] = m.factor_masks[n].data();
    CHECK(vo_set_model(s, m.core.data(), m.core_mask.data(), fp.data(), mp.data()) == 0);
    for (std::size_t n = 0; n < 3; ++n) {
      for (std::size_t i : {std::size_t(0), std::size_t(3), std::size_t(6)}) {
        RowUpdateScratch sc;
        compute_row_stats(m, x, idx, n, i, sc);
        const std::size_t J = m.ranks[n];
        std::vector<double> dd(J), gg(J * J), xx(J);
        CHECK(vo_row_stats(s, (int)n, i, dd.data(), gg.data(), xx.data()) == 0);
        CHECK(sc.delta == dd && sc.gram == gg && sc.xdelta == xx);
      }
      for (std::size_t j = 0; j < m.ranks[n]; ++j) {
        for (std::size_t e : {std::size_t(0), std::size_t(17), std::size_t(499)}) {
          double want = 0.0;
          CHECK(vo_partial_reconstruct(s, x.entry(e), 1, (int)n, j, &want) == 0);
          CHECK(partial_reconstruct(m, x.entry(e), n, j) == want);
        }
      }
    }
    // LF on an empty row: returns before touching the scratch (updates.hpp:91)
    RowUpdateScratch sc;
    sc.reset(4);
    sc.gram.assign(16, 7.0);
    const auto before = m.factors[0];
    update_factor_row_lf(m, x, idx, 0, 22, 0.05, sc);
    CHECK(sc.gram == std::vector<double>(16, 7.0) && m.factors[0] == before);
    // L1 on an empty row: statistics are zero, unmasked elements become 0
    update_factor_row_l1(m, x, idx, 0, 22, 0.05, sc);
    CHECK(sc.gram == std::vector<double>(16, 0.0));
    CHECK(vo_update_factor_row(s, 1, 0, 22, 0.05) == 0);
    // a busy row through the scratch overload == the oracle's row update
    update_factor_row_lf(m, x, idx, 0, 3, 0.05, sc);
    CHECK(vo_update_factor_row(s, 0, 0, 3, 0.05) == 0);
    std::vector<double> f0(25 * 4), f1(8 * 3), f2(7 * 2);
    double* fo[3] = {f0.data(), f1.data(), f2.data()};
    CHECK(vo_get_model(s, nullptr, nullptr, fo, nullptr) == 0);
    CHECK(m.factors[1] == f1 && m.factors[2] == f2);  // untouched modes: identical
    for (std::size_t q = 0; q < f0.size(); ++q)  // the row solves: same result up to summation order
      CHECK(std::abs(m.factors[0][q] - f0[q]) <= 1e-9 * std::max(1.0, std::abs(f0[q])));
    vo_destroy(s);
  }
  // the tensor-context cache is verified against the tensor's contents:
  // an in-place edit, or new contents in the same buffers (address reuse),
  // gets a fresh device CSF; at most a few contexts stay cached (LRU)
  {
    auto x = make_tensor({6, 5, 4}, {0, 0, 0, 1, 2, 3, 5, 4, 3, 2, 2, 2}, {1.0, 2.0, 3.0, 4.0});
    TuckerModel m = init_random(x.dims, {2, 2, 2}, 4);
    auto oracle_re = [&](const SparseTensor& t) {
      vo_session* s = nullptr;
      const std::uint64_t d[3] = {6, 5, 4}, rk[3] = {2, 2, 2};
      vo_create(3, d, t.nnz(), t.coords.data(), t.values.data(), rk, &s);
      std::vector<const double*> fp(3);
      std::vector<const std::uint8_t*> mp(3);
      for (int n = 0; n < 3; ++n) fp[n] = m.factors[n].data(), mp[n] = m.factor_masks[n].data();
      vo_set_model(s, m.core.data(), m.core_mask.data(), fp.data(), mp.data());
      double ss, xn, re;
      vo_compute_residuals(s, 1, nullptr, &ss, &xn, &re);
      vo_destroy(s);
      return re;
    };
    const double re1 = reconstruction_error(m, x);
    CHECK(std::abs(re1 - oracle_re(x)) <= 1e-12 * re1);
    x.values[2] = -7.5;  // in place
    const double re2 = reconstruction_error(m, x);
    CHECK(re2 != re1 && std::abs(re2 - oracle_re(x)) <= 1e-12 * re2);
    const Coord* addr = x.coords.data();
    x.coords = {0, 1, 0, 1, 2, 1, 5, 4, 0, 3, 2, 2};  // same size: the same buffer, new tensor
    CHECK(x.coords.data() == addr);
    const double re3 = reconstruction_error(m, x);
    CHECK(std::abs(re3 - oracle_re(x)) <= 1e-12 * re3);
    for (int t = 0; t < 7; ++t) {
      auto y = make_tensor({6, 5, 4}, {Coord(t % 6), 0, 0, 1, 2, 3}, {1.0 + t, 2.0});
      reconstruction_error(m, y);
    }
    CHECK(b200_detail::cached_contexts() <= b200_detail::max_contexts());
    release_device_contexts();
    CHECK(b200_detail::cached_contexts() == 0);
    CHECK(std::abs(reconstruction_error(m, x) - re3) <= 1e-15 * re3);
  }
  if (failures == 0) std::printf("ALL OK\n");
  return failures == 0 ? 0 : 1;
}
