// SPDX-License-Identifier: Apache-2.0
// vest_io.cpp -- the data formats either side of the hot path (SURVEY.md 8(f)
// f3/f4), host side, OpenMP-parallel:
//   * COO text read (load_coo, sparse_tensor.hpp:139-209): the file is read
//     whole and split at line boundaries across threads; every thread parses
//     its lines with the reference's rules (whitespace tokens, "# dims:"
//     headers, std::stoll coordinates, strict strtod values, first-error-by-
//     line precedence with the same messages);
//   * COO text write (save_coo, :211-228) and the model directory
//     (save_model / load_model, model_io.hpp:22-104): threads format ranges
//     of lines with the reference's printf conversions ("%.17g", tabs), the
//     buffers are written in order -- byte-identical files;
//   * a binary cache of a tensor (magic, order, nnz, dims, coords, values) so
//     a large input is parsed once.
// Tensor validation (check_tensor, :68-95: bounds, duplicates) is applied
// where the reference applies it (load_coo's make_tensor, load_model).
#include <omp.h>
#include <parallel/algorithm>

#include <algorithm>
#include <cerrno>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <filesystem>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/vest.h"

namespace {

thread_local std::string g_io_err;

struct ArgErr : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};

template <class F>
int io_guard(F&& f) {
  try {
    f();
    return VEST_OK;
  } catch (const std::invalid_argument& e) {
    g_io_err = e.what();
    return VEST_EINVAL;
  } catch (const std::exception& e) {
    g_io_err = e.what();
    return VEST_ERUNTIME;
  }
}

inline bool is_ws(char c) { return c == ' ' || c == '\t' || c == '\n' || c == '\v' || c == '\f' || c == '\r'; }

// detail::parse_double (sparse_tensor.hpp:57-66): the whole token, finite
bool parse_double(const std::string& tok, double& out) {
  const char* s = tok.c_str();
  char* end = nullptr;
  errno = 0;
  const double v = std::strtod(s, &end);
  if (end == s || *end != '\0') return false;
  if (std::isinf(v) || std::isnan(v)) return false;
  out = v;
  return true;
}

// std::stoll semantics on a whitespace-free token: optional sign, base-10
// digits up to the first other character; no digits or overflow -> failure
bool parse_stoll(const std::string& tok, long long& out) {
  const char* s = tok.c_str();
  char* end = nullptr;
  errno = 0;
  const long long v = std::strtoll(s, &end, 10);
  if (end == s || errno == ERANGE) return false;
  out = v;
  return true;
}

// istream >> size_t on a token stream: the numeric prefix of the token; a
// partial token ends the extraction after it, an empty one before it
// (returns 0: stop, 1: value and continue, 2: value and stop)
int extract_size(const std::string& tok, uint64_t& out) {
  const char* s = tok.c_str();
  char* end = nullptr;
  errno = 0;
  const unsigned long long v = std::strtoull(s, &end, 10);
  if (end == s || errno == ERANGE) return 0;
  out = v;
  return *end == '\0' ? 1 : 2;
}

void tokens_of(const char* b, const char* e, std::vector<std::string>& toks) {
  toks.clear();
  const char* p = b;
  while (p < e) {
    while (p < e && is_ws(*p)) ++p;
    if (p >= e) break;
    const char* q = p;
    while (q < e && !is_ws(*q)) ++q;
    toks.emplace_back(p, q);
    p = q;
  }
}

std::string read_file(const std::string& path) {
  FILE* f = std::fopen(path.c_str(), "rb");
  if (!f) throw std::runtime_error("cannot open " + path);
  std::string buf;
  if (std::fseek(f, 0, SEEK_END) == 0) {
    const long n = std::ftell(f);
    if (n > 0) {
      buf.resize((size_t)n);
      std::fseek(f, 0, SEEK_SET);
      const size_t got = std::fread(buf.data(), 1, buf.size(), f);
      buf.resize(got);
    }
  }
  std::fclose(f);
  return buf;
}

struct Coo {
  int order = 0;
  std::vector<uint64_t> dims;
  std::vector<uint32_t> coords;
  std::vector<double> values;
};

// check_tensor (sparse_tensor.hpp:68-95): bounds, then duplicates by sorting
// entry ids by coordinate tuple
void check_tensor(const Coo& x) {
  const size_t n = x.order;
  if (n == 0) throw ArgErr("tensor order must be at least 1");
  for (uint64_t d : x.dims)
    if (d == 0) throw ArgErr("tensor dimensions must be positive");
  const size_t nnz = x.values.size();
  if (x.coords.size() != nnz * n) throw ArgErr("coordinate buffer size does not match nnz * order");
  bool oob = false;
#pragma omp parallel for reduction(|| : oob)
  for (size_t e = 0; e < nnz; ++e)
    for (size_t k = 0; k < n; ++k) oob = oob || x.coords[e * n + k] >= x.dims[k];
  if (oob) throw ArgErr("coordinate out of bounds");
  std::vector<uint64_t> ids(nnz);
  for (size_t e = 0; e < nnz; ++e) ids[e] = e;
  const uint32_t* c = x.coords.data();
  __gnu_parallel::sort(ids.begin(), ids.end(), [&](uint64_t a, uint64_t b) {
    return std::lexicographical_compare(c + a * n, c + a * n + n, c + b * n, c + b * n + n);
  });
  bool dup = false;
#pragma omp parallel for reduction(|| : dup)
  for (size_t e = 1; e < nnz; ++e) dup = dup || std::equal(c + ids[e - 1] * n, c + ids[e - 1] * n + n, c + ids[e] * n);
  if (dup) throw ArgErr("duplicate coordinate in tensor");
}

// -------------------------------------------------------------- COO read --
struct ChunkParse {
  uint64_t nlines = 0;
  std::vector<uint64_t> dims;       // "# dims:" values, in order
  std::vector<uint32_t> coords;
  std::vector<double> values;
  int64_t first_data = -1;          // local line index of the first data line
  size_t first_cols = 0;            // its token count
  int64_t err_line = -1;            // first local error (with this chunk's order)
  std::string err_msg;              // message without the "path:line" prefix
};

void parse_chunk(const char* b, const char* e, bool one_based, ChunkParse& out) {
  std::vector<std::string> toks;
  size_t order = 0;
  uint64_t line = 0;
  const char* p = b;
  while (p < e) {
    const char* q = static_cast<const char*>(std::memchr(p, '\n', (size_t)(e - p)));
    const char* le = q ? q : e;
    tokens_of(p, le, toks);
    const uint64_t li = line++;
    p = q ? q + 1 : e;
    if (toks.empty()) continue;  // blank
    if (toks[0][0] == '#') {
      if (toks.size() >= 2 && toks[1] == "dims:") {
        for (size_t t = 2; t < toks.size(); ++t) {
          uint64_t d;
          const int r = extract_size(toks[t], d);
          if (r == 0) break;
          out.dims.push_back(d);
          if (r == 2) break;
        }
      }
      continue;
    }
    if (out.err_line >= 0) continue;  // only lines before the first error matter
    if (order == 0) {
      out.first_data = (int64_t)li;
      out.first_cols = toks.size();
      if (toks.size() < 2) {
        out.err_line = (int64_t)li;
        out.err_msg = "need at least one coordinate and a value";
        continue;
      }
      order = toks.size() - 1;
    } else if (toks.size() != order + 1) {
      out.err_line = (int64_t)li;
      out.err_msg = "inconsistent column count";
      continue;
    }
    for (size_t k = 0; k < order; ++k) {
      long long c;
      if (!parse_stoll(toks[k], c)) {
        out.err_line = (int64_t)li;
        out.err_msg = "bad coordinate '" + toks[k] + "'";
        break;
      }
      if (one_based) c -= 1;
      if (c < 0) {
        out.err_line = (int64_t)li;
        out.err_msg = "negative coordinate";
        break;
      }
      out.coords.push_back(static_cast<uint32_t>(c));
    }
    if (out.err_line >= 0) continue;
    double v;
    if (!parse_double(toks[order], v)) {
      out.err_line = (int64_t)li;
      out.err_msg = "bad value '" + toks[order] + "'";
      continue;
    }
    out.values.push_back(v);
  }
  out.nlines = line;
}

Coo load_coo_impl(const std::string& path, bool one_based, int threads) {
  const std::string buf = read_file(path);
  const char* b = buf.data();
  const char* e = b + buf.size();
  const int T = std::max(1, std::min<int>(threads > 0 ? threads : omp_get_max_threads(),
                                          (int)(buf.size() / (1 << 16)) + 1));
  // chunk boundaries at line starts
  std::vector<const char*> cut(T + 1);
  cut[0] = b;
  cut[T] = e;
  for (int t = 1; t < T; ++t) {
    const char* q = b + buf.size() * t / T;
    if (q < cut[t - 1]) q = cut[t - 1];
    const char* nl = static_cast<const char*>(std::memchr(q, '\n', (size_t)(e - q)));
    cut[t] = nl ? nl + 1 : e;
  }
  std::vector<ChunkParse> cp(T);
#pragma omp parallel for num_threads(T) schedule(static, 1)
  for (int t = 0; t < T; ++t) parse_chunk(cut[t], cut[t + 1], one_based, cp[t]);
  // global line numbers (1-based) and the order fixed by the first data line
  std::vector<uint64_t> base(T + 1, 0);
  for (int t = 0; t < T; ++t) base[t + 1] = base[t] + cp[t].nlines;
  size_t order = 0;
  for (int t = 0; t < T && order == 0; ++t)
    if (cp[t].first_data >= 0 && cp[t].first_cols >= 2) order = cp[t].first_cols - 1;
  // the first error in file order
  uint64_t err_line = UINT64_MAX;
  std::string err_msg;
  bool seen_data = false;
  for (int t = 0; t < T; ++t) {
    const ChunkParse& c = cp[t];
    if (c.first_data < 0) continue;
    const uint64_t fd = base[t] + (uint64_t)c.first_data;
    uint64_t el = UINT64_MAX;
    std::string em;
    if (!seen_data) {
      // the global first data line: this chunk parsed with the right order
      if (c.err_line >= 0) {
        el = base[t] + (uint64_t)c.err_line;
        em = c.err_msg;
      }
    } else if (c.first_cols != order + 1) {
      el = fd;
      em = "inconsistent column count";
    } else if (c.err_line >= 0) {
      el = base[t] + (uint64_t)c.err_line;
      em = c.err_msg;
    }
    seen_data = true;
    if (el < err_line) {
      err_line = el;
      err_msg = em;
    }
  }
  if (err_line != UINT64_MAX)
    throw std::runtime_error(path + ":" + std::to_string(err_line + 1) + ": " + err_msg);
  Coo x;
  for (int t = 0; t < T; ++t) x.dims.insert(x.dims.end(), cp[t].dims.begin(), cp[t].dims.end());
  uint64_t nnz = 0;
  std::vector<uint64_t> voff(T + 1, 0);
  for (int t = 0; t < T; ++t) voff[t + 1] = voff[t] + cp[t].values.size();
  nnz = voff[T];
  if (order == 0 && x.dims.empty()) throw std::runtime_error(path + ": no entries");
  if (order == 0) order = x.dims.size();  // header-only file: an empty tensor
  x.order = (int)order;
  x.values.resize(nnz);
  x.coords.resize(nnz * order);
#pragma omp parallel for num_threads(T) schedule(static, 1)
  for (int t = 0; t < T; ++t) {
    std::copy(cp[t].values.begin(), cp[t].values.end(), x.values.begin() + voff[t]);
    std::copy(cp[t].coords.begin(), cp[t].coords.end(), x.coords.begin() + voff[t] * order);
  }
  if (x.dims.empty()) {
    x.dims.assign(order, 0);
    for (uint64_t q = 0; q < nnz; ++q)
      for (size_t k = 0; k < order; ++k) x.dims[k] = std::max<uint64_t>(x.dims[k], (uint64_t)x.coords[q * order + k] + 1);
  } else if (x.dims.size() != order) {
    throw std::runtime_error(path + ": dims header order does not match data");
  }
  check_tensor(x);  // make_tensor
  return x;
}

// ------------------------------------------------------------- COO write --
void append_uint(std::string& s, uint64_t v) {
  char b[24];
  const int n = std::snprintf(b, sizeof b, "%llu", (unsigned long long)v);
  s.append(b, (size_t)n);
}
void append_g17(std::string& s, double v) {
  char b[64];
  const int n = std::snprintf(b, sizeof b, "%.17g", v);
  s.append(b, (size_t)n);
}

// the lines of [e0, e1): "c0\tc1\t...\t%.17g\n"
void format_entries(std::string& s, int order, const uint32_t* coords, const double* values, uint64_t e0,
                    uint64_t e1) {
  s.reserve((size_t)(e1 - e0) * (size_t)(order * 8 + 24));
  for (uint64_t q = e0; q < e1; ++q) {
    for (int k = 0; k < order; ++k) {
      append_uint(s, coords[q * order + k]);
      s.push_back('\t');
    }
    append_g17(s, values[q]);
    s.push_back('\n');
  }
}

template <class Fmt>
void write_parallel(const std::string& path, const std::string& head, uint64_t nitems, Fmt fmt,
                    const std::string& err_open, const std::string& err_write) {
  const int T = std::max(1, std::min<int>(omp_get_max_threads(), (int)(nitems / 4096) + 1));
  std::vector<std::string> parts(T);
#pragma omp parallel for num_threads(T) schedule(static, 1)
  for (int t = 0; t < T; ++t) fmt(parts[t], nitems * t / T, nitems * (t + 1) / T);
  FILE* f = std::fopen(path.c_str(), "wb");
  if (!f) throw std::runtime_error(err_open);
  bool ok = std::fwrite(head.data(), 1, head.size(), f) == head.size();
  for (const auto& p : parts) ok = ok && std::fwrite(p.data(), 1, p.size(), f) == p.size();
  ok = (std::fclose(f) == 0) && ok;
  if (!ok) throw std::runtime_error(err_write);
}

void save_coo_impl(const std::string& path, int order, const uint64_t* dims, uint64_t nnz, const uint32_t* coords,
                   const double* values) {
  std::string head = "# dims:";
  for (int k = 0; k < order; ++k) {
    head.push_back(' ');
    append_uint(head, dims[k]);
  }
  head.push_back('\n');
  write_parallel(
      path, head, nnz,
      [&](std::string& s, uint64_t a, uint64_t b) { format_entries(s, order, coords, values, a, b); },
      "cannot write " + path, "write failed: " + path);
}

// -------------------------------------------------------------- model I/O --
void save_model_impl(const std::string& dir, int order, const uint64_t* dims, const uint64_t* ranks,
                     const double* core, const double* const* factors) {
  std::filesystem::create_directories(dir);
  const std::filesystem::path d(dir);
  for (int n = 0; n < order; ++n) {
    const uint64_t J = ranks[n];
    const double* F = factors[n];
    const std::string p = (d / ("factor_" + std::to_string(n) + ".tsv")).string();
    write_parallel(
        p, std::string(), dims[n],
        [&](std::string& s, uint64_t a, uint64_t b) {
          s.reserve((size_t)(b - a) * (size_t)J * 24);
          for (uint64_t i = a; i < b; ++i) {
            for (uint64_t j = 0; j < J; ++j) {
              if (j) s.push_back('\t');
              append_g17(s, F[i * J + j]);
            }
            s.push_back('\n');
          }
        },
        "cannot write factor file in " + d.string(), "write failed in " + d.string());
  }
  // core.coo: the nonzero cells in row-major order, ranks as dims
  uint64_t G = 1;
  for (int n = 0; n < order; ++n) G *= ranks[n];
  std::vector<uint32_t> cc;
  std::vector<double> cv;
  std::vector<uint64_t> beta(order, 0);
  for (uint64_t lin = 0; lin < G; ++lin) {
    if (core[lin] != 0.0) {
      for (int k = 0; k < order; ++k) cc.push_back((uint32_t)beta[k]);
      cv.push_back(core[lin]);
    }
    for (int k = order - 1; k >= 0; --k) {  // row-major odometer
      if (++beta[k] < ranks[k]) break;
      beta[k] = 0;
    }
  }
  save_coo_impl((d / "core.coo").string(), order, ranks, cv.size(), cc.data(), cv.data());
}

struct ModelFile {
  int order = 0;
  std::vector<uint64_t> dims, ranks;
  std::vector<double> core;
  std::vector<uint8_t> core_mask;
  std::vector<std::vector<double>> factors;
  std::vector<std::vector<uint8_t>> masks;
};

ModelFile load_model_impl(const std::string& dir) {
  const std::filesystem::path d(dir);
  const Coo core = load_coo_impl((d / "core.coo").string(), false, 0);
  ModelFile m;
  m.order = core.order;
  m.ranks = core.dims;
  const int n = m.order;
  uint64_t G = 1;
  for (uint64_t r : m.ranks) G *= r;
  m.core.assign(G, 0.0);
  std::vector<uint64_t> strides(n, 1);
  for (int k = n - 2; k >= 0; --k) strides[k] = strides[k + 1] * m.ranks[k + 1];
  for (uint64_t e = 0; e < core.values.size(); ++e) {
    uint64_t lin = 0;
    for (int k = 0; k < n; ++k) lin += core.coords[e * n + k] * strides[k];
    m.core[lin] = core.values[e];
  }
  m.core_mask.resize(G);
  for (uint64_t k = 0; k < G; ++k) m.core_mask[k] = m.core[k] == 0.0;
  m.dims.resize(n);
  m.factors.resize(n);
  m.masks.resize(n);
  std::vector<std::string> toks;
  for (int mode = 0; mode < n; ++mode) {
    const std::string path = (d / ("factor_" + std::to_string(mode) + ".tsv")).string();
    FILE* probe = std::fopen(path.c_str(), "rb");
    if (!probe) throw std::runtime_error("cannot open " + path);
    std::fclose(probe);
    const std::string buf = read_file(path);
    const char* p = buf.data();
    const char* e = p + buf.size();
    uint64_t rows = 0;
    auto& F = m.factors[mode];
    while (p < e) {
      const char* q = static_cast<const char*>(std::memchr(p, '\n', (size_t)(e - p)));
      const char* le = q ? q : e;
      tokens_of(p, le, toks);
      p = q ? q + 1 : e;
      for (const auto& tok : toks) {
        double v;
        if (!parse_double(tok, v)) throw std::runtime_error(path + ": bad value '" + tok + "'");
        F.push_back(v);
      }
      if (toks.empty()) continue;  // trailing blank lines
      if (toks.size() != m.ranks[mode])
        throw std::runtime_error(path + ": expected " + std::to_string(m.ranks[mode]) + " columns");
      ++rows;
    }
    if (rows == 0) throw std::runtime_error(path + ": empty factor");
    m.dims[mode] = rows;
    m.masks[mode].resize(F.size());
    for (size_t k = 0; k < F.size(); ++k) m.masks[mode][k] = F[k] == 0.0;
  }
  // check_model (tucker_model.hpp:67-80)
  if (n == 0) throw ArgErr("model order must be at least 1");
  for (int k = 0; k < n; ++k) {
    if (m.dims[k] == 0 || m.ranks[k] == 0) throw ArgErr("dims and ranks must be positive");
    if (m.factors[k].size() != m.dims[k] * m.ranks[k]) throw ArgErr("factor buffer size mismatch");
  }
  return m;
}

// ----------------------------------------------------------- binary cache --
constexpr char kMagic[8] = {'V', 'E', 'S', 'T', 'C', 'O', 'O', '1'};

}  // namespace

struct vest_coo {
  Coo x;
};
struct vest_model_file {
  ModelFile m;
};

extern "C" {

const char* vest_io_last_error(void) { return g_io_err.c_str(); }

int vest_coo_load(const char* path, int one_based, int threads, vest_coo** out) {
  return io_guard([&] {
    auto h = std::make_unique<vest_coo>();
    h->x = load_coo_impl(path, one_based != 0, threads);
    *out = h.release();
  });
}

int vest_coo_info(const vest_coo* h, int* order, uint64_t* nnz, uint64_t* dims, const uint32_t** coords,
                  const double** values) {
  return io_guard([&] {
    if (order) *order = h->x.order;
    if (nnz) *nnz = h->x.values.size();
    if (dims) std::copy(h->x.dims.begin(), h->x.dims.end(), dims);
    if (coords) *coords = h->x.coords.data();
    if (values) *values = h->x.values.data();
  });
}

void vest_coo_free(vest_coo* h) { delete h; }

int vest_coo_save(const char* path, int order, const uint64_t* dims, uint64_t nnz, const uint32_t* coords,
                  const double* values) {
  return io_guard([&] { save_coo_impl(path, order, dims, nnz, coords, values); });
}

int vest_coo_cache_save(const char* path, int order, const uint64_t* dims, uint64_t nnz, const uint32_t* coords,
                        const double* values) {
  return io_guard([&] {
    FILE* f = std::fopen(path, "wb");
    if (!f) throw std::runtime_error(std::string("cannot write ") + path);
    const uint64_t hdr[2] = {(uint64_t)order, nnz};
    bool ok = std::fwrite(kMagic, 1, 8, f) == 8 && std::fwrite(hdr, 8, 2, f) == 2 &&
              std::fwrite(dims, 8, order, f) == (size_t)order &&
              std::fwrite(coords, 4, nnz * order, f) == nnz * order && std::fwrite(values, 8, nnz, f) == nnz;
    ok = (std::fclose(f) == 0) && ok;
    if (!ok) throw std::runtime_error(std::string("write failed: ") + path);
  });
}

int vest_coo_cache_load(const char* path, vest_coo** out) {
  return io_guard([&] {
    FILE* f = std::fopen(path, "rb");
    if (!f) throw std::runtime_error(std::string("cannot open ") + path);
    std::unique_ptr<FILE, int (*)(FILE*)> guard(f, std::fclose);
    char magic[8];
    uint64_t hdr[2];
    if (std::fread(magic, 1, 8, f) != 8 || std::memcmp(magic, kMagic, 8) != 0 || std::fread(hdr, 8, 2, f) != 2 ||
        hdr[0] == 0 || hdr[0] > 8)
      throw std::runtime_error(std::string(path) + ": not a vest COO cache");
    auto h = std::make_unique<vest_coo>();
    Coo& x = h->x;
    x.order = (int)hdr[0];
    x.dims.resize(x.order);
    x.coords.resize(hdr[1] * x.order);
    x.values.resize(hdr[1]);
    if (std::fread(x.dims.data(), 8, x.order, f) != (size_t)x.order ||
        std::fread(x.coords.data(), 4, x.coords.size(), f) != x.coords.size() ||
        std::fread(x.values.data(), 8, x.values.size(), f) != x.values.size())
      throw std::runtime_error(std::string(path) + ": truncated cache");
    *out = h.release();
  });
}

int vest_model_save(const char* dir, int order, const uint64_t* dims, const uint64_t* ranks, const double* core,
                    const double* const* factors) {
  return io_guard([&] { save_model_impl(dir, order, dims, ranks, core, factors); });
}

int vest_model_load(const char* dir, vest_model_file** out) {
  return io_guard([&] {
    auto h = std::make_unique<vest_model_file>();
    h->m = load_model_impl(dir);
    *out = h.release();
  });
}

int vest_model_file_info(const vest_model_file* h, int* order, uint64_t* dims, uint64_t* ranks, const double** core,
                         const uint8_t** core_mask, const double** factors, const uint8_t** factor_masks) {
  return io_guard([&] {
    const ModelFile& m = h->m;
    if (order) *order = m.order;
    for (int n = 0; n < m.order; ++n) {
      if (dims) dims[n] = m.dims[n];
      if (ranks) ranks[n] = m.ranks[n];
      if (factors) factors[n] = m.factors[n].data();
      if (factor_masks) factor_masks[n] = m.masks[n].data();
    }
    if (core) *core = m.core.data();
    if (core_mask) *core_mask = m.core_mask.data();
  });
}

void vest_model_file_free(vest_model_file* h) { delete h; }

}  // extern "C"
