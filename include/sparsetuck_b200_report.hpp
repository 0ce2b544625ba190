// SPDX-License-Identifier: Apache-2.0
// sparsetuck_b200_report.hpp -- the data formats and generators either side of
// the B200 path that the reference's CLI uses, on top of
// sparsetuck_b200.hpp:
//   * write_report_jsonl / write_bench_csv: the reference's report lines
//     (report.hpp:130-175), same keys, order and "%.17g" numbers;
//   * SyntheticSpec / gen_synthetic: the planted-model generator
//     (synthetic.hpp:17-155) -- the same seeded engine and draw order (truth
//     values and masks, coordinate sample, noise), so model, coordinates and
//     noise are the reference's; the noise-free values are reconstructed on the
//     device (vest_predict), i.e. equal to the reference's up to fp64 rounding;
//   * scaling_benchmark (report.hpp:70-127): per-iteration fit time per config;
//     the "threads" column is kept for the format and does not change the
//     device run;
//   * row_density_report (report.hpp:24-45).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <limits>
#include <new>
#include <ostream>
#include <random>
#include <set>
#include <string>
#include <unordered_set>
#include <vector>

#include "sparsetuck_b200.hpp"

namespace sparsetuck {

struct RowDensity {
  std::size_t row = 0;
  std::size_t nonzeros = 0;
  double norm = 0.0;
};

inline std::vector<RowDensity> row_density_report(const TuckerModel& m, std::size_t mode) {
  const std::size_t J = m.ranks[mode];
  std::vector<RowDensity> rows(m.dims[mode]);
  for (std::size_t i = 0; i < m.dims[mode]; ++i) {
    double s = 0.0;
    std::size_t nz = 0;
    for (std::size_t j = 0; j < J; ++j) {
      const double v = m.factors[mode][i * J + j];
      nz += v != 0.0;
      s += v * v;
    }
    rows[i] = {i, nz, std::sqrt(s)};
  }
  std::sort(rows.begin(), rows.end(), [](const RowDensity& a, const RowDensity& b) {
    return a.nonzeros != b.nonzeros ? a.nonzeros > b.nonzeros : a.row < b.row;
  });
  return rows;
}

struct SyntheticSpec {
  std::vector<std::size_t> dims;
  std::vector<std::size_t> ranks;
  std::size_t nnz = 0;
  double factor_density = 1.0;
  double noise_std = 0.0;
  std::uint64_t seed = 0;
};

struct SyntheticData {
  SparseTensor tensor;
  TuckerModel truth;
};

namespace b200_detail {

// distinct coordinates in canonical (row-major) order, the reference's two
// regimes and draw sequence (synthetic.hpp:37-103)
inline std::vector<Coord> sample_coords(const std::vector<std::size_t>& dims, std::size_t nnz,
                                        std::mt19937_64& rng) {
  const std::size_t n = dims.size();
  std::uint64_t total = 1;
  bool wide = false;
  for (std::size_t d : dims) {
    if (total > std::numeric_limits<std::uint64_t>::max() / d) {
      wide = true;
      break;
    }
    total *= d;
  }
  std::vector<Coord> flat;
  flat.reserve(nnz * n);
  auto emit = [&](std::uint64_t key) {
    std::vector<Coord> c(n);
    for (std::size_t k = n; k-- > 0;) {
      c[k] = static_cast<Coord>(key % dims[k]);
      key /= dims[k];
    }
    flat.insert(flat.end(), c.begin(), c.end());
  };
  if (!wide) {
    if (nnz > total) throw std::invalid_argument("nnz exceeds tensor cell count");
    std::vector<std::uint64_t> keys;
    keys.reserve(nnz);
    if (nnz * 2 >= total) {  // dense: partial Fisher-Yates over all positions
      std::vector<std::uint64_t> all(total);
      for (std::uint64_t i = 0; i < total; ++i) all[i] = i;
      for (std::size_t k = 0; k < nnz; ++k) {
        std::uniform_int_distribution<std::uint64_t> pick(k, total - 1);
        std::swap(all[k], all[pick(rng)]);
      }
      keys.assign(all.begin(), all.begin() + nnz);
    } else {  // sparse: rejection against the keys drawn so far
      std::unordered_set<std::uint64_t> seen;
      std::uniform_int_distribution<std::uint64_t> pick(0, total - 1);
      while (keys.size() < nnz) {
        const std::uint64_t k = pick(rng);
        if (seen.insert(k).second) keys.push_back(k);
      }
    }
    std::sort(keys.begin(), keys.end());
    for (std::uint64_t key : keys) emit(key);
  } else {  // > 2^64 cells: coordinate tuples, ordered-set dedup
    std::set<std::vector<Coord>> seen;
    while (seen.size() < nnz) {
      std::vector<Coord> c(n);
      for (std::size_t k = 0; k < n; ++k) {
        std::uniform_int_distribution<std::uint64_t> pick(0, dims[k] - 1);
        c[k] = static_cast<Coord>(pick(rng));
      }
      seen.insert(std::move(c));
    }
    for (const auto& c : seen) flat.insert(flat.end(), c.begin(), c.end());
  }
  return flat;
}

inline std::string num17(double v) {
  char buf[64];
  std::snprintf(buf, sizeof buf, "%.17g", v);
  std::string s(buf);
  if (s.find("inf") != std::string::npos || s.find("nan") != std::string::npos) s = "null";
  return s;
}

}  // namespace b200_detail

inline SyntheticData gen_synthetic(const SyntheticSpec& spec) {
  if (spec.dims.size() != spec.ranks.size()) throw std::invalid_argument("ranks order mismatch");
  if (spec.dims.empty()) throw std::invalid_argument("order must be at least 1");
  if (!(spec.factor_density > 0.0 && spec.factor_density <= 1.0))
    throw std::invalid_argument("factor_density must be in (0, 1]");
  if (!(spec.noise_std >= 0.0)) throw std::invalid_argument("noise_std must be nonnegative");
  if (spec.nnz == 0) throw std::invalid_argument("nnz must be positive");
  std::mt19937_64 rng(spec.seed);
  std::uniform_real_distribution<double> unif(0.0, 1.0);
  SyntheticData out;
  TuckerModel& t = out.truth;
  t.dims = spec.dims;
  t.ranks = spec.ranks;
  t.factors.resize(spec.dims.size());
  t.factor_masks.resize(spec.dims.size());
  auto draw = [&](double& v, std::uint8_t& mask) {  // value first, then the keep test
    const double value = unif(rng);
    const bool drop = spec.factor_density < 1.0 && unif(rng) >= spec.factor_density;
    v = drop ? 0.0 : value;
    mask = drop ? 1 : 0;
  };
  for (std::size_t n = 0; n < spec.dims.size(); ++n) {
    t.factors[n].resize(spec.dims[n] * spec.ranks[n]);
    t.factor_masks[n].resize(t.factors[n].size());
    for (std::size_t k = 0; k < t.factors[n].size(); ++k) draw(t.factors[n][k], t.factor_masks[n][k]);
  }
  t.core.resize(t.core_size());
  t.core_mask.resize(t.core.size());
  for (std::size_t k = 0; k < t.core.size(); ++k) draw(t.core[k], t.core_mask[k]);
  SparseTensor& x = out.tensor;
  x.dims = spec.dims;
  x.coords = b200_detail::sample_coords(spec.dims, spec.nnz, rng);
  x.values = predict(t, std::span<const Coord>(x.coords));  // on the device
  if (spec.noise_std > 0.0) {
    std::normal_distribution<double> noise(0.0, 1.0);
    for (double& v : x.values) v += spec.noise_std * noise(rng);
  }
  return out;
}

inline void write_report_jsonl(const TrainReport& report, std::ostream& out) {
  using b200_detail::num17;
  for (const IterationReport& it : report.iterations) {
    out << "{\"iter\":" << it.iter << ",\"re\":" << num17(it.re) << ",\"prune_rate\":" << num17(it.prune_rate)
        << ",\"pruned\":" << (it.pruned ? "true" : "false") << ",\"pruned_core\":" << it.pruned_core
        << ",\"pruned_factors\":[";
    for (std::size_t n = 0; n < it.pruned_factors.size(); ++n) out << (n ? "," : "") << it.pruned_factors[n];
    out << "],\"sparsity\":" << num17(it.sparsity) << ",\"masked\":" << num17(it.masked)
        << ",\"wall_ms\":" << num17(it.wall_ms) << "}\n";
  }
}

struct BenchConfig {
  std::vector<std::size_t> dims;
  std::vector<std::size_t> ranks;
  std::size_t nnz = 0;
};

struct BenchOptions {
  std::size_t iters = 3;
  std::size_t reps = 5;
  Regularizer reg = Regularizer::LF;
  double lambda = 0.01;
  std::uint64_t seed = 0;
};

struct BenchResult {
  BenchConfig config;
  int threads = 1;
  double sec_per_iter = 0.0;
  double speedup = 1.0;
  bool skipped = false;
  std::string note;
};

inline std::vector<BenchResult> scaling_benchmark(const std::vector<BenchConfig>& configs,
                                                  const std::vector<int>& thread_counts,
                                                  const BenchOptions& opt = {}) {
  std::vector<BenchResult> out;
  for (const BenchConfig& bc : configs) {
    SyntheticData data;
    bool failed = false;
    try {
      SyntheticSpec spec;
      spec.dims = bc.dims;
      spec.ranks = bc.ranks;
      spec.nnz = bc.nnz;
      spec.seed = opt.seed;
      data = gen_synthetic(spec);
    } catch (const std::bad_alloc&) {
      failed = true;
    }
    double base = 0.0;
    for (std::size_t ti = 0; ti < thread_counts.size(); ++ti) {
      BenchResult cell;
      cell.config = bc;
      cell.threads = thread_counts[ti];
      if (failed) {
        cell.skipped = true;
        cell.note = "allocation failed";
        out.push_back(cell);
        continue;
      }
      TrainConfig cfg;
      cfg.ranks = bc.ranks;
      cfg.reg = opt.reg;
      cfg.lambda = opt.lambda;
      cfg.max_iters = opt.iters;
      cfg.tol = 0.0;
      cfg.threads = cell.threads;
      cfg.seed = opt.seed;
      cfg.normalize_output = false;
      std::vector<double> times;
      for (std::size_t rep = 0; rep < opt.reps; ++rep)
        times.push_back(fit(data.tensor, cfg).report.elapsed_sec / double(opt.iters));
      std::sort(times.begin(), times.end());
      cell.sec_per_iter = times[times.size() / 2];
      if (ti == 0) base = cell.sec_per_iter;
      cell.speedup = cell.sec_per_iter > 0.0 ? base / cell.sec_per_iter : 0.0;
      cell.note = "b200";
      out.push_back(cell);
    }
  }
  return out;
}

inline void write_bench_csv(const std::vector<BenchResult>& cells, std::ostream& out) {
  using b200_detail::num17;
  out << "order,dims,ranks,nnz,threads,sec_per_iter,speedup,skipped,note\n";
  auto join = [](const std::vector<std::size_t>& v) {
    std::string s;
    for (std::size_t k = 0; k < v.size(); ++k) s += (k ? "x" : "") + std::to_string(v[k]);
    return s;
  };
  for (const BenchResult& c : cells)
    out << c.config.dims.size() << ',' << join(c.config.dims) << ',' << join(c.config.ranks) << ','
        << c.config.nnz << ',' << c.threads << ',' << num17(c.sec_per_iter) << ',' << num17(c.speedup) << ','
        << (c.skipped ? 1 : 0) << ',' << c.note << '\n';
}

}  // namespace sparsetuck
