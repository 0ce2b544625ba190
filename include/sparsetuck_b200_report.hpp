// SPDX-License-Identifier: Apache-2.0
// sparsetuck_b200_report.hpp -- the data formats and generators either side of
// the B200 path that the reference's CLI uses, on top of
// sparsetuck_b200.hpp:
//   * write_report_jsonl / write_bench_csv: the reference's report lines
//     (report.hpp:130-175): same keys, key order and "%.17g" numbers;
//   * SyntheticSpec / gen_synthetic: the planted-model generator
//     (synthetic.hpp:17-155) -- the same seeded engine consumed in the same
//     order (truth values with their keep draws, coordinate sample, noise), so
//     the planted model, coordinates and noise equal the reference's; the
//     noise-free values are reconstructed on the device (vest_predict), i.e.
//     equal to the reference's up to fp64 rounding;
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
#include <numeric>
#include <optional>
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

// rows of factor `mode` by nonzero count (descending), ties by row index
inline std::vector<RowDensity> row_density_report(const TuckerModel& m, std::size_t mode) {
  const std::size_t width = m.ranks[mode];
  const std::vector<double>& f = m.factors[mode];
  std::vector<RowDensity> table;
  table.reserve(m.dims[mode]);
  for (std::size_t i = 0; i < m.dims[mode]; ++i) {
    const double* row = f.data() + i * width;
    const auto nz = static_cast<std::size_t>(std::count_if(row, row + width, [](double v) { return v != 0.0; }));
    const double sq = std::inner_product(row, row + width, row, 0.0);
    table.push_back(RowDensity{i, nz, std::sqrt(sq)});
  }
  std::stable_sort(table.begin(), table.end(),
                   [](const RowDensity& l, const RowDensity& r) { return l.nonzeros > r.nonzeros; });
  return table;
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

using Engine = std::mt19937_64;

// cells = prod(dims), or 0 when it does not fit 64 bits
inline std::uint64_t cell_count(const std::vector<std::size_t>& dims) {
  std::uint64_t cells = 1;
  for (std::size_t d : dims) {
    if (cells > std::numeric_limits<std::uint64_t>::max() / d) return 0;
    cells *= d;
  }
  return cells;
}

// nnz distinct linear cell ids: a partial Fisher-Yates shuffle of all ids when
// at least half the cells are drawn, rejection against the ids so far otherwise
// (the reference's regimes and draw sequence, synthetic.hpp:56-74)
inline std::vector<std::uint64_t> draw_cells(std::uint64_t cells, std::size_t nnz, Engine& eng) {
  std::vector<std::uint64_t> ids;
  if (2 * nnz >= cells) {
    std::vector<std::uint64_t> perm(cells);
    std::iota(perm.begin(), perm.end(), std::uint64_t{0});
    for (std::size_t slot = 0; slot < nnz; ++slot) {
      const std::uint64_t j = std::uniform_int_distribution<std::uint64_t>(slot, cells - 1)(eng);
      std::swap(perm[slot], perm[j]);
    }
    perm.resize(nnz);
    ids = std::move(perm);
  } else {
    std::uniform_int_distribution<std::uint64_t> any(0, cells - 1);
    std::unordered_set<std::uint64_t> taken;
    ids.reserve(nnz);
    while (ids.size() < nnz) {
      const std::uint64_t id = any(eng);
      if (taken.insert(id).second) ids.push_back(id);
    }
  }
  std::sort(ids.begin(), ids.end());
  return ids;
}

// distinct coordinates in canonical (row-major) order
inline std::vector<Coord> sample_coords(const std::vector<std::size_t>& dims, std::size_t nnz, Engine& eng) {
  const std::size_t order = dims.size();
  std::vector<Coord> flat(nnz * order);
  const std::uint64_t cells = cell_count(dims);
  if (cells != 0) {
    if (nnz > cells) throw std::invalid_argument("nnz exceeds tensor cell count");
    const std::vector<std::uint64_t> ids = draw_cells(cells, nnz, eng);
    for (std::size_t e = 0; e < nnz; ++e) {
      std::uint64_t id = ids[e];
      for (std::size_t k = order; k-- > 0;) {
        flat[e * order + k] = static_cast<Coord>(id % dims[k]);
        id /= dims[k];
      }
    }
    return flat;
  }
  // more than 2^64 cells: whole tuples, mode by mode, ordered-set dedup
  std::set<std::vector<Coord>> tuples;
  std::vector<Coord> t(order);
  while (tuples.size() < nnz) {
    for (std::size_t k = 0; k < order; ++k)
      t[k] = static_cast<Coord>(std::uniform_int_distribution<std::uint64_t>(0, dims[k] - 1)(eng));
    tuples.insert(t);
  }
  std::size_t at = 0;
  for (const auto& tup : tuples) std::copy(tup.begin(), tup.end(), flat.begin() + static_cast<long>(at++ * order));
  return flat;
}

inline std::string num17(double v) {
  if (!std::isfinite(v)) return "null";  // JSON has no inf/nan literals
  char buf[40];
  std::snprintf(buf, sizeof buf, "%.17g", v);
  return buf;
}

inline void check_spec(const SyntheticSpec& s) {
  if (s.dims.size() != s.ranks.size()) throw std::invalid_argument("ranks order mismatch");
  if (s.dims.empty()) throw std::invalid_argument("order must be at least 1");
  if (!(s.factor_density > 0.0 && s.factor_density <= 1.0))
    throw std::invalid_argument("factor_density must be in (0, 1]");
  if (!(s.noise_std >= 0.0)) throw std::invalid_argument("noise_std must be nonnegative");
  if (s.nnz == 0) throw std::invalid_argument("nnz must be positive");
}

}  // namespace b200_detail

inline SyntheticData gen_synthetic(const SyntheticSpec& spec) {
  b200_detail::check_spec(spec);
  b200_detail::Engine eng(spec.seed);
  std::uniform_real_distribution<double> u01(0.0, 1.0);
  const bool thin = spec.factor_density < 1.0;
  // one planted element: its value is drawn first, then (density < 1) its keep draw
  auto plant = [&](std::vector<double>& vals, std::vector<std::uint8_t>& mask, std::size_t count) {
    vals.assign(count, 0.0);
    mask.assign(count, 0);
    for (std::size_t q = 0; q < count; ++q) {
      const double v = u01(eng);
      const bool dropped = thin && !(u01(eng) < spec.factor_density);
      vals[q] = dropped ? 0.0 : v;
      mask[q] = dropped ? 1 : 0;
    }
  };
  SyntheticData out;
  TuckerModel& truth = out.truth;
  truth.dims = spec.dims;
  truth.ranks = spec.ranks;
  truth.factors.resize(spec.dims.size());
  truth.factor_masks.resize(spec.dims.size());
  for (std::size_t n = 0; n < spec.dims.size(); ++n)
    plant(truth.factors[n], truth.factor_masks[n], spec.dims[n] * spec.ranks[n]);
  plant(truth.core, truth.core_mask, truth.core_size());
  SparseTensor& obs = out.tensor;
  obs.dims = spec.dims;
  obs.coords = b200_detail::sample_coords(spec.dims, spec.nnz, eng);
  obs.values = predict(truth, std::span<const Coord>(obs.coords));  // on the device
  if (spec.noise_std > 0.0) {
    std::normal_distribution<double> gauss(0.0, 1.0);
    for (double& v : obs.values) v += spec.noise_std * gauss(eng);
  }
  return out;
}

// one JSON object per iteration (report.hpp:140-156 keys and order)
inline void write_report_jsonl(const TrainReport& report, std::ostream& out) {
  using b200_detail::num17;
  for (const IterationReport& it : report.iterations) {
    std::string facs;
    for (std::size_t n = 0; n < it.pruned_factors.size(); ++n)
      facs += (n ? "," : "") + std::to_string(it.pruned_factors[n]);
    out << "{\"iter\":" + std::to_string(it.iter) + ",\"re\":" + num17(it.re) +
               ",\"prune_rate\":" + num17(it.prune_rate) + ",\"pruned\":" + (it.pruned ? "true" : "false") +
               ",\"pruned_core\":" + std::to_string(it.pruned_core) + ",\"pruned_factors\":[" + facs +
               "],\"sparsity\":" + num17(it.sparsity) + ",\"masked\":" + num17(it.masked) +
               ",\"wall_ms\":" + num17(it.wall_ms) + "}\n";
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

// median seconds per sweep of plain descent (no pruning, no early stop) for
// every (config, thread count) cell
inline std::vector<BenchResult> scaling_benchmark(const std::vector<BenchConfig>& configs,
                                                  const std::vector<int>& thread_counts,
                                                  const BenchOptions& opt = {}) {
  std::vector<BenchResult> cells;
  for (const BenchConfig& bc : configs) {
    std::optional<SyntheticData> data;
    try {
      SyntheticSpec spec;
      spec.dims = bc.dims;
      spec.ranks = bc.ranks;
      spec.nnz = bc.nnz;
      spec.seed = opt.seed;
      data = gen_synthetic(spec);
    } catch (const std::bad_alloc&) {
      data.reset();
    }
    double first = 0.0;
    for (std::size_t ti = 0; ti < thread_counts.size(); ++ti) {
      BenchResult cell{bc, thread_counts[ti]};
      if (!data) {
        cell.skipped = true;
        cell.note = "allocation failed";
        cells.push_back(cell);
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
      std::vector<double> per_iter(opt.reps);
      for (double& t : per_iter) t = fit(data->tensor, cfg).report.elapsed_sec / static_cast<double>(opt.iters);
      std::nth_element(per_iter.begin(), per_iter.begin() + per_iter.size() / 2, per_iter.end());
      cell.sec_per_iter = per_iter[per_iter.size() / 2];
      if (ti == 0) first = cell.sec_per_iter;
      cell.speedup = cell.sec_per_iter > 0.0 ? first / cell.sec_per_iter : 0.0;
      cell.note = "b200";
      cells.push_back(cell);
    }
  }
  return cells;
}

inline void write_bench_csv(const std::vector<BenchResult>& cells, std::ostream& out) {
  using b200_detail::num17;
  auto dimstr = [](const std::vector<std::size_t>& v) {
    std::string s;
    for (std::size_t v_i : v) s += (s.empty() ? "" : "x") + std::to_string(v_i);
    return s;
  };
  out << "order,dims,ranks,nnz,threads,sec_per_iter,speedup,skipped,note\n";
  for (const BenchResult& c : cells) {
    const std::string fields[] = {std::to_string(c.config.dims.size()), dimstr(c.config.dims),
                                  dimstr(c.config.ranks),             std::to_string(c.config.nnz),
                                  std::to_string(c.threads),          num17(c.sec_per_iter),
                                  num17(c.speedup),                   c.skipped ? "1" : "0",
                                  c.note};
    std::string line;
    for (const std::string& f : fields) line += (line.empty() ? "" : ",") + f;
    out << line << '\n';
  }
}

}  // namespace sparsetuck
