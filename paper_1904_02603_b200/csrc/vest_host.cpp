// SPDX-License-Identifier: Apache-2.0
// vest_host.cpp -- host-side utilities of libvest_cuda.so that sit next to the
// hot path: seeded synthetic inputs for the BASELINE configs, the reference's
// train/test split, and the nnz-balanced row partition used for multi-GPU
// sharding.
#include <algorithm>
#include <cmath>
#include <parallel/algorithm>
#include <cstdint>
#include <cstring>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/vest.h"

namespace {
thread_local std::string g_herr;

int bits_for(uint64_t d) {
  int b = 1;
  while (b < 63 && (1ull << b) < d) ++b;
  return b;
}

using u128 = unsigned __int128;

// Zipf(s) over {0..I-1}: P(i) proportional to (i+1)^-s (rank 1 -> index 0),
// sampled by inverse CDF.
struct Zipf {
  std::vector<double> cdf;
  explicit Zipf(uint64_t I, double s) : cdf(I) {
    double acc = 0.0;
    for (uint64_t i = 0; i < I; ++i) {
      acc += std::pow(double(i + 1), -s);
      cdf[i] = acc;
    }
    for (auto& v : cdf) v /= acc;
  }
  uint64_t draw(double u) const {
    auto it = std::lower_bound(cdf.begin(), cdf.end(), u);
    if (it == cdf.end()) --it;
    return uint64_t(it - cdf.begin());
  }
};
}  // namespace

// Deterministic and thread-count independent: draws come in chunks of
// kSynthChunk, each from its own engine seeded by (seed, round, chunk); the
// keys are sorted and deduplicated (parallel sort), and the shortfall redrawn.
constexpr uint64_t kSynthChunk = 1u << 20;

static uint64_t chunk_seed(uint64_t seed, uint64_t round, uint64_t chunk) {
  uint64_t z = seed + 0x9E3779B97F4A7C15ull * (round * 1000003ull + chunk + 1);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

extern "C" int vest_synth(int order, const uint64_t* dims, uint64_t nnz, const double* zipf_s, int values_kind,
                          uint64_t seed, uint32_t* coords_out, double* values_out) {
  try {
    if (order <= 0 || order > 8) throw std::invalid_argument("order must be in [1, 8]");
    int tot = 0;
    std::vector<int> bits(order), shift(order);
    for (int k = order - 1; k >= 0; --k) {
      bits[k] = bits_for(dims[k]);
      shift[k] = tot;
      tot += bits[k];
    }
    if (tot > 128) throw std::invalid_argument("coordinate tuple does not fit 128 bits");
    long double cells = 1;
    for (int k = 0; k < order; ++k) cells *= (long double)dims[k];
    if ((long double)nnz > cells) throw std::invalid_argument("nnz exceeds tensor cell count");
    std::vector<Zipf> z;
    z.reserve(order);
    std::vector<int> use_z(order, 0);
    for (int k = 0; k < order; ++k) {
      use_z[k] = zipf_s && zipf_s[k] > 0.0;
      z.emplace_back(use_z[k] ? dims[k] : 1, use_z[k] ? zipf_s[k] : 1.0);
    }
    std::vector<u128> keys;
    keys.reserve(nnz);
    for (uint64_t round = 0; keys.size() < nnz; ++round) {
      if (round > 10000) throw std::runtime_error("could not draw enough distinct coordinates");
      const uint64_t have = keys.size(), need = nnz - have;
      keys.resize(nnz);
      const uint64_t nch = (need + kSynthChunk - 1) / kSynthChunk;
#pragma omp parallel for schedule(dynamic, 1)
      for (int64_t ch = 0; ch < (int64_t)nch; ++ch) {
        std::mt19937_64 rng(chunk_seed(seed, round, (uint64_t)ch));
        std::uniform_real_distribution<double> unif(0.0, 1.0);
        const uint64_t b = have + (uint64_t)ch * kSynthChunk, e = std::min<uint64_t>(nnz, b + kSynthChunk);
        for (uint64_t q = b; q < e; ++q) {
          u128 key = 0;
          for (int k = 0; k < order; ++k) {
            uint64_t c;
            if (use_z[k]) {
              c = z[k].draw(unif(rng));
            } else {
              std::uniform_int_distribution<uint64_t> pick(0, dims[k] - 1);
              c = pick(rng);
            }
            key |= (u128)c << shift[k];
          }
          keys[q] = key;
        }
      }
      __gnu_parallel::sort(keys.begin(), keys.end());
      keys.erase(std::unique(keys.begin(), keys.end()), keys.end());
    }
    // canonical entry order: row-major over the coordinate tuple
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < (int64_t)nnz; ++e)
      for (int k = 0; k < order; ++k)
        coords_out[e * order + k] = (uint32_t)((keys[e] >> shift[k]) & (((u128)1 << bits[k]) - 1));
    const uint64_t nch = (nnz + kSynthChunk - 1) / kSynthChunk;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t ch = 0; ch < (int64_t)nch; ++ch) {
      std::mt19937_64 rng(chunk_seed(seed ^ 0x5EED5EEDull, 0, (uint64_t)ch));
      const uint64_t b = (uint64_t)ch * kSynthChunk, e = std::min<uint64_t>(nnz, b + kSynthChunk);
      if (values_kind == 0) {
        std::uniform_real_distribution<double> d(0.0, 1.0);
        for (uint64_t q = b; q < e; ++q) values_out[q] = d(rng);
      } else if (values_kind == 1) {
        std::uniform_int_distribution<int> d(1, 5);
        for (uint64_t q = b; q < e; ++q) values_out[q] = double(d(rng));
      } else {
        std::normal_distribution<double> d(0.0, 1.0);
        for (uint64_t q = b; q < e; ++q) values_out[q] = double(float(d(rng)));
      }
    }
    return 0;
  } catch (const std::invalid_argument& e) {
    g_herr = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_herr = e.what();
    return 2;
  }
}

// split_train_test (sparse_tensor.hpp:232-260): same engine, same shuffle,
// same rounding of the test count; returns the entry ids of both parts.
extern "C" int vest_split_ids(uint64_t nnz, double test_fraction, uint64_t seed, uint64_t* test_ids,
                              uint64_t* n_test, uint64_t* train_ids, uint64_t* n_train) {
  if (!(test_fraction >= 0.0 && test_fraction <= 1.0)) return 1;
  std::vector<std::size_t> ids(nnz);
  for (std::size_t e = 0; e < nnz; ++e) ids[e] = e;
  std::mt19937_64 rng(seed);
  std::shuffle(ids.begin(), ids.end(), rng);
  const auto ntest = static_cast<std::size_t>(std::llround(test_fraction * double(nnz)));
  std::vector<std::size_t> te(ids.begin(), ids.begin() + ntest), tr(ids.begin() + ntest, ids.end());
  std::sort(te.begin(), te.end());
  std::sort(tr.begin(), tr.end());
  for (std::size_t k = 0; k < te.size(); ++k) test_ids[k] = te[k];
  for (std::size_t k = 0; k < tr.size(); ++k) train_ids[k] = tr[k];
  *n_test = te.size();
  *n_train = tr.size();
  return 0;
}

// Multi-GPU sharding plan: contiguous row ranges,
// balanced by observed entries.  bounds[r] = first row whose prefix count
// reaches r * nnz / world; ranges are monotone and cover all rows.
extern "C" int vest_partition_rows(const uint64_t* off, uint64_t rows, int world, uint64_t* bounds) {
  if (world <= 0) return 1;
  const uint64_t nnz = off[rows];
  bounds[0] = 0;
  for (int r = 1; r < world; ++r) {
    const uint64_t target = (uint64_t)((u128)nnz * (u128)r / (u128)world);
    // first row i with off[i] >= target
    uint64_t lo = 0, hi = rows;
    while (lo < hi) {
      const uint64_t mid = (lo + hi) / 2;
      if (off[mid] < target) lo = mid + 1; else hi = mid;
    }
    bounds[r] = std::max(bounds[r - 1], lo);
  }
  bounds[world] = rows;
  return 0;
}

// init_random (tucker_model.hpp:88-108) on the host: mt19937_64(seed),
// uniform_real_distribution<double>(0, 1), factor 0 row-major, ..., then core.
extern "C" int vest_init_random_host(int order, const uint64_t* dims, const uint64_t* ranks, uint64_t seed,
                                     double* core, double* const* factors) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> unif(0.0, 1.0);
  uint64_t g = 1;
  for (int n = 0; n < order; ++n) {
    for (uint64_t k = 0; k < dims[n] * ranks[n]; ++k) factors[n][k] = unif(rng);
    g *= ranks[n];
  }
  for (uint64_t k = 0; k < g; ++k) core[k] = unif(rng);
  return 0;
}
