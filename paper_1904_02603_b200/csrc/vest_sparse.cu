// SPDX-License-Identifier: Apache-2.0
// vest_sparse.cu -- delta contraction specialised to the core's sparsity
// pattern (compute_delta, updates.hpp:35-52, which skips zero cells).
//
// A pruned core (BASELINE config 4: 8^4 cells, 90 % masked) makes the dense
// factorised contraction of the row-pass kernels do mostly multiplications by
// zero.  The unmasked cells change only at prune events, so the contraction is
// generated as straight-line CUDA for the current mask -- every core offset an
// immediate (constant-bank operand), every factor value a register -- and
// compiled at run time with NVRTC for sm_100a:
//   * cells are ordered by (beta of the other modes but the last, beta_n,
//     beta of the last other mode); each prefix product w = prod u_k[beta_k]
//     is formed once, each (prefix, beta_n) group sums
//     t = sum_cells G[beta] u_last[beta_last] and adds w * t to delta[beta_n]:
//     about 2 FMA per unmasked cell instead of |G| + |G|/J + ... per entry;
//   * masked cells are exactly 0 (tucker_model.hpp:15-20) and skipped; unmasked
//     cells that happen to be 0 are kept (adding 0 * p changes nothing), so
//     the code depends on the mask only and is recompiled only after a prune;
//   * the kernel writes delta SoA (delta[j][pos]) for the mode's CSF
//     positions; k_rowpass_delta (vest_rowpass.cu) then accumulates the row
//     statistics on DMMA, solves the rows and emits the fused residual.
// NVRTC is dlopen'ed (no link-time dependency); the module is loaded with the
// runtime's library API and its constant-bank core refreshed from d_core
// before each use.
#include <dlfcn.h>

#include <algorithm>
#include <chrono>
#include <exception>
#include <future>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <sstream>
#include <string>
#include <system_error>
#include <vector>

#include "vest_internal.h"

namespace vest {

struct SparseDeltaArgs {
  const uint32_t* oc[VEST_MAXN];
  const double* f[VEST_MAXN];
  const float* g[VEST_MAXN];  // fp32 factor copies (gather_f32)
  double* out;
  unsigned long long p0, n, stride;
};

namespace {

// ------------------------------------------------------------------ NVRTC --
typedef int (*nvrtcCreateProgram_t)(void**, const char*, const char*, int, const char* const*, const char* const*);
typedef int (*nvrtcCompileProgram_t)(void*, int, const char* const*);
typedef int (*nvrtcGetProgramLogSize_t)(void*, size_t*);
typedef int (*nvrtcGetProgramLog_t)(void*, char*);
typedef int (*nvrtcGetCUBINSize_t)(void*, size_t*);
typedef int (*nvrtcGetCUBIN_t)(void*, char*);
typedef int (*nvrtcDestroyProgram_t)(void**);

struct Nvrtc {
  void* h = nullptr;
  nvrtcCreateProgram_t create = nullptr;
  nvrtcCompileProgram_t compile = nullptr;
  nvrtcGetProgramLogSize_t log_size = nullptr;
  nvrtcGetProgramLog_t log = nullptr;
  nvrtcGetCUBINSize_t cubin_size = nullptr;
  nvrtcGetCUBIN_t cubin = nullptr;
  nvrtcDestroyProgram_t destroy = nullptr;
};

const Nvrtc& nvrtc() {
  static Nvrtc n = [] {
    Nvrtc r;
    const char* names[] = {"libnvrtc.so.12", "libnvrtc.so", "/usr/local/cuda/lib64/libnvrtc.so.12"};
    for (const char* nm : names)
      if ((r.h = dlopen(nm, RTLD_NOW | RTLD_LOCAL))) break;
    if (!r.h) return r;
    r.create = (nvrtcCreateProgram_t)dlsym(r.h, "nvrtcCreateProgram");
    r.compile = (nvrtcCompileProgram_t)dlsym(r.h, "nvrtcCompileProgram");
    r.log_size = (nvrtcGetProgramLogSize_t)dlsym(r.h, "nvrtcGetProgramLogSize");
    r.log = (nvrtcGetProgramLog_t)dlsym(r.h, "nvrtcGetProgramLog");
    r.cubin_size = (nvrtcGetCUBINSize_t)dlsym(r.h, "nvrtcGetCUBINSize");
    r.cubin = (nvrtcGetCUBIN_t)dlsym(r.h, "nvrtcGetCUBIN");
    r.destroy = (nvrtcDestroyProgram_t)dlsym(r.h, "nvrtcDestroyProgram");
    return r;
  }();
  return n;
}

// ------------------------------------------------------- source generation --
struct Cell {
  int lin;
  int beta[VEST_MAXN];
};

// u<k>_<b>: mode k's factor value beta = b of the entry (registers)
std::string u(int k, int b) { return "u" + std::to_string(k) + "_" + std::to_string(b); }

// the unmasked cells in contraction order for mode n: other modes but the
// last (prefix), then beta_n, then the last other mode
std::vector<Cell> ordered_cells(const Ctx& c, int n, std::vector<int>& oth) {
  const int N = c.N;
  oth.clear();
  for (int k = 0; k < N; ++k)
    if (k != n) oth.push_back(k);
  const int L = (int)oth.size();
  std::vector<Cell> cells;
  for (int lin = 0; lin < c.G; ++lin) {
    if (c.h_core_mask[lin]) continue;
    Cell cl{lin, {}};
    int rem = lin;
    for (int k = N - 1; k >= 0; --k) {
      cl.beta[k] = rem % c.ranks[k];
      rem /= c.ranks[k];
    }
    cells.push_back(cl);
  }
  auto key = [&](const Cell& a, const Cell& b) {
    for (int q = 0; q + 1 < L; ++q)
      if (a.beta[oth[q]] != b.beta[oth[q]]) return a.beta[oth[q]] < b.beta[oth[q]];
    if (a.beta[n] != b.beta[n]) return a.beta[n] < b.beta[n];
    return a.beta[oth[L - 1]] < b.beta[oth[L - 1]];
  };
  std::sort(cells.begin(), cells.end(), key);
  return cells;
}

// Loads of entry E's other-mode factor rows into registers u<k>_<b>e<E>;
// pos is the expression of the entry's CSF position.
// Cache hints of the delta kernel (VEST_SD_HINT=0/1, A/B): the CSF coordinate
// stream is read once (ld.global.cs, evict-first) and delta is written once
// for the next kernel (st.global.cs), so the gathered factor rows -- the only
// data with reuse -- keep the L2.
bool sd_hint() {
  static const bool v = [] {
    const char* e = getenv("VEST_SD_HINT");
    return e ? e[0] == '1' : true;
  }();
  return v;
}

// VEST_SD_LPF=1 (A/B; off): L1 prefetch of the lazily read rows at the top of
// the iteration, next to the other rows' loads -- measured slower (config 4
// factor modes 55.8 -> 58.8 ms per iteration).
bool sd_lazy_prefetch() {
  static const bool v = [] {
    const char* e = getenv("VEST_SD_LPF");
    return e && e[0] == '1';
  }();
  return v;
}

void emit_row_loads(std::ostringstream& o, const Ctx& c, const std::vector<int>& oth, int e, const std::string& pos,
                    int lazy = 0, bool f32 = false) {
  const std::string E = std::to_string(e);
  for (int k : oth) {
    const int ld = c.ld[k];
    const std::string rk = "r" + std::to_string(k) + "e" + E;
    const int lvl = (int)(std::find(oth.begin(), oth.end(), k) - oth.begin());
    if (lvl < lazy && lvl + 1 < (int)oth.size()) {  // read where the prefix opens (emit_cells), not held in registers
      o << "    const " << (c.gather_f32 ? "float" : "double") << "* " << rk << " = a." << (c.gather_f32 ? "g" : "f")
        << "[" << k << "] + (unsigned long long)" << (sd_hint() ? "__ldcs" : "__ldg") << "(a.oc[" << k << "] + " << pos << ") * " << ld << "ull;\n";
      if (sd_lazy_prefetch())  // the row's first lazy read would otherwise miss to DRAM inside the contraction
        o << "    asm volatile(\"prefetch.global.L1 [%0];\" ::\"l\"(" << rk << "));\n";
      continue;
    }
    if (c.gather_f32) {  // fp32 copy of the row, widened to fp64 in registers (kept fp32 in the fp32 contraction)
      const bool v4 = ld % 4 == 0;
      o << "    const float* " << rk << " = a.g[" << k << "] + (unsigned long long)" << (sd_hint() ? "__ldcs" : "__ldg") << "(a.oc[" << k << "] + " << pos
        << ") * " << ld << "ull;\n";
      for (int b = 0; b < c.ranks[k]; b += (v4 ? 4 : 2)) {
        const std::string v = "v" + std::to_string(k) + "_" + std::to_string(b) + "e" + E;
        o << "    const " << (v4 ? "float4 " : "float2 ") << v << " = __ldg(reinterpret_cast<const "
          << (v4 ? "float4" : "float2") << "*>(" << rk << " + " << b << "));\n";
        const char* comp[4] = {"x", "y", "z", "w"};
        for (int q = 0; q < (v4 ? 4 : 2) && b + q < c.ranks[k]; ++q)
          o << "    const " << (f32 ? "float " : "double ") << u(k, b + q) << "e" << E << " = " << (f32 ? "" : "(double)")
            << v << "." << comp[q] << ";\n";
      }
      continue;
    }
    o << "    const double* " << rk << " = a.f[" << k << "] + (unsigned long long)" << (sd_hint() ? "__ldcs" : "__ldg") << "(a.oc[" << k << "] + " << pos
      << ") * " << ld << "ull;\n";
    for (int b = 0; b < c.ranks[k]; b += 2) {
      const std::string ua = u(k, b) + "e" + E;
      if (b + 1 < c.ranks[k]) {
        const std::string v = "v" + std::to_string(k) + "_" + std::to_string(b) + "e" + E;
        o << "    const double2 " << v << " = __ldg(reinterpret_cast<const double2*>(" << rk << " + " << b << "));\n"
          << "    const double " << ua << " = " << v << ".x, " << u(k, b + 1) << "e" << E << " = " << v << ".y;\n";
      } else {
        o << "    const double " << ua << " = __ldg(" << rk << " + " << b << ");\n";
      }
    }
  }
}

// d<j>e<E> = delta_j of entries E < ne (updates.hpp:35-52 restricted to the
// unmasked cells): each prefix product formed once, each (prefix, beta_n)
// group t = sum G u_last, then d[beta_n] += w t.  Every core value G[lin] is a
// constant-bank operand shared by the ne entries.
void emit_cells(std::ostringstream& o, const Ctx& c, int n, const std::vector<int>& oth, const std::vector<Cell>& cells,
                int ne, int lazy = 0, bool f32 = false, const std::string& mid = std::string()) {
  const int L = (int)oth.size();
  bool mid_done = mid.empty();
  const std::string T = f32 ? "float" : "double", Gs = f32 ? "Gf[" : "G[", fma_ = f32 ? "fmaf(" : "fma(";
  for (int e = 0; e < ne; ++e)
    for (int j = 0; j < c.ranks[n]; ++j) o << "    " << T << " d" << j << "e" << e << " = " << (f32 ? "0.0f" : "0.0") << ";\n";
  auto same_prefix = [&](const Cell& a, const Cell& b, int upto) {
    for (int q = 0; q <= upto; ++q)
      if (a.beta[oth[q]] != b.beta[oth[q]]) return false;
    return true;
  };
  size_t i = 0;
  while (i < cells.size()) {
    for (int q = 0; q + 1 < L; ++q) {  // open the prefix levels of cells[i]
      const int k = oth[q], b = cells[i].beta[k];
      o << "    {";
      for (int e = 0; e < ne; ++e) {
        const std::string E = std::to_string(e);
        const std::string val = q < lazy ? "(" + T + ")__ldg(r" + std::to_string(k) + "e" + E + " + " + std::to_string(b) + ")"
                                         : u(k, b) + "e" + E;
        if (q == 0) o << " const " << T << " w0e" << E << " = " << val << ";";
        else o << " const " << T << " w" << q << "e" << E << " = w" << (q - 1) << "e" << E << " * " << val << ";";
      }
      o << "\n";
    }
    size_t e_end = i;
    while (e_end < cells.size() && (L < 2 || same_prefix(cells[i], cells[e_end], L - 2))) ++e_end;
    const int kl = oth[L - 1];
    for (size_t g = i; g < e_end;) {
      const int bn = cells[g].beta[n];
      size_t h = g;
      o << "      { " << T << " g = " << Gs << cells[h].lin << "];";
      for (int e = 0; e < ne; ++e) o << " " << T << " t" << e << " = g * " << u(kl, cells[h].beta[kl]) << "e" << e << ";";
      for (++h; h < e_end && cells[h].beta[n] == bn; ++h) {
        o << " g = " << Gs << cells[h].lin << "];";
        for (int e = 0; e < ne; ++e)
          o << " t" << e << " = " << fma_ << "g, " << u(kl, cells[h].beta[kl]) << "e" << e << ", t" << e << ");";
      }
      for (int e = 0; e < ne; ++e) {
        if (L >= 2) o << " d" << bn << "e" << e << " = " << fma_ << "w" << (L - 2) << "e" << e << ", t" << e << ", d" << bn << "e" << e << ");";
        else o << " d" << bn << "e" << e << " += t" << e << ";";
      }
      o << " }\n";
      g = h;
    }
    for (int q = 0; q + 1 < L; ++q) o << "    }\n";
    i = e_end;
    if (!mid_done && 4 * i >= cells.size()) {  // a quarter into the contraction
      o << mid;
      mid_done = true;
    }
  }
}

// VEST_SD_LAZY (A/B): the outermost prefix mode's factor values are read
// (L1 hits) where their prefix opens instead of held in registers
// (default: 1 with fp32 gathers -- fewer live registers, less spill traffic
// at 2 entries per thread; config 4: 270.0 / 267.5 / 272.1 ms per iteration at
// 0 / 1 / 2 -- and 0 with fp64 gathers, where the lazy reads cost more: factor
// modes 83.5 -> 95.6 ms)
int sd_lazy(const Ctx& c) {  // prefix levels read lazily: 0, 1 (outermost) or 2 (the two outer levels)
  static const int env = [] {
    const char* e = getenv("VEST_SD_LAZY");
    return e ? std::max(0, std::min(2, atoi(e))) : -1;
  }();
  return env >= 0 ? env : (c.gather_f32 ? 1 : 0);
}

// CTAs per SM the delta kernel is register-budgeted for (VEST_SD_MINB: A/B;
// 2 = 128 registers with some stack, 1 = up to 255 registers at half the warps)
int sd_min_blocks() {
  static const int v = [] {
    const char* e = getenv("VEST_SD_MINB");
    return e ? std::max(1, std::min(4, atoi(e))) : 2;
  }();
  return v;
}

// The contraction in fp32 arithmetic (fp32 mode only, VEST_SD_F32=0 for the
// fp64 one): the fp32 copies of the factor rows, the core rounded to fp32
// (constant bank Gf) and FFMA -- twice the FP64 rate and half the registers
// per value.  delta is written as fp32 in the fp32 mode either way; the
// statistics, solves and residuals after it stay fp64 (k_rowpass_delta).
bool sd_f32(const Ctx& c) {
  static const int env = [] {
    const char* e = getenv("VEST_SD_F32");
    return e && (e[0] == '0' || e[0] == '1') ? e[0] - '0' : -1;
  }();
  return c.gather_f32 && env != 0;
}

// Next-iteration row prefetch (VEST_SD_PF=1, A/B; off): the thread reads the
// coordinates of its next grid-stride entries at the top of the iteration and,
// a quarter into the contraction, prefetches their factor rows into the L2
// (prefetch.global.L2).  Measured slower (config 4 factor modes 41.4 -> 50.6
// ms per iteration): the prefetches wait on their coordinate loads inside the
// contraction and double the gather requests.
bool sd_prefetch() {
  static const bool v = [] {
    const char* e = getenv("VEST_SD_PF");
    return e && e[0] == '1';
  }();
  return v;
}

// entries per thread of the delta kernel (VEST_SD_NE: A/B; 2 in fp64, 3 in fp32 --
// config 4 fp32 mode, ms per iteration at 2 / 3 / 4: 190.2 / 186.8 / 193.4)
int sd_entries(const Ctx& c) {
  static const int env = [] {
    const char* e = getenv("VEST_SD_NE");
    return e ? std::max(1, std::min(8, atoi(e))) : 0;
  }();
  return env > 0 ? env : (sd_f32(c) ? 3 : 2);
}

void emit_mode(std::ostringstream& o, const Ctx& c, int n) {
  std::vector<int> oth;
  const std::vector<Cell> cells = ordered_cells(c, n, oth);
  const bool f32 = sd_f32(c);
  const int ne = sd_entries(c);
  const std::string NB = std::to_string(256 * ne);
  // ne entries per thread (e: t0 + 256 e of the block's stride window): every
  // core value is loaded once (uniform constant load) and feeds all ne
  // entries' FMAs
  o << "extern \"C\" __global__ void __launch_bounds__(256, " << sd_min_blocks() << ") vest_sd_" << n
    << "(const SparseDeltaArgs a) {\n"
    << "  for (unsigned long long t0 = blockIdx.x * " << NB << "ull + threadIdx.x; t0 < a.n; t0 += gridDim.x * " << NB
    << "ull) {\n";
  for (int e = 1; e < ne; ++e)
    o << "    const unsigned long long t" << e << " = t0 + " << 256 * e << "ull < a.n ? t0 + " << 256 * e << "ull : t0;\n";
  const int lazy = oth.size() >= 2 ? std::min<int>(sd_lazy(c), (int)oth.size() - 1) : 0;
  for (int e = 0; e < ne; ++e) emit_row_loads(o, c, oth, e, "a.p0 + t" + std::to_string(e), lazy, f32);
  std::ostringstream mid;
  if (sd_prefetch() && c.gather_f32) {
    o << "    const unsigned long long tn = t0 + gridDim.x * " << NB << "ull;\n";
    for (int e = 0; e < ne; ++e)
      for (int k : oth) {
        const std::string nm = "n" + std::to_string(k) + "e" + std::to_string(e);
        o << "    const unsigned " << nm << " = tn + " << 256 * e << "ull < a.n ? __ldcs(a.oc[" << k << "] + a.p0 + tn + "
          << 256 * e << "ull) : 0xffffffffu;\n";
        mid << "    if (" << nm << " != 0xffffffffu) asm volatile(\"prefetch.global.L2 [%0];\" ::\"l\"(a.g[" << k
            << "] + (unsigned long long)" << nm << " * " << c.ld[k] << "ull));\n";
      }
  }
  emit_cells(o, c, n, oth, cells, ne, lazy, f32, mid.str());
  // delta SoA for k_rowpass_delta: fp64, or fp32 in the fp32 mode (gather_f32)
  const std::string dst = c.gather_f32 ? "reinterpret_cast<float*>(a.out)" : "a.out";
  const std::string cv = c.gather_f32 && !f32 ? "(float)" : "";
  for (int e = 0; e < ne; ++e) {
    const std::string E = std::to_string(e);
    if (e > 0) o << "    if (t" << E << " != t0) {\n";
    for (int j = 0; j < c.ranks[n]; ++j)
      if (sd_hint())
        o << "      __stcs(" << dst << " + " << j << "ull * a.stride + t" << E << ", " << cv << "d" << j << "e" << E << ");\n";
      else
        o << "      " << dst << "[" << j << "ull * a.stride + t" << E << "] = " << cv << "d" << j << "e" << E << ";\n";
    if (e > 0) o << "    }\n";
  }
  o << "  }\n}\n";
}

// The fused factor-mode update (modes without the fused residual): one warp
// per chunk of a row, one entry per lane per 32-entry round -- the
// contraction above in registers, then (delta, x) staged transposed in shared
// memory and the row's Gram accumulated on DMMA, the light row solved in the
// kernel (heavy rows: partials for k_heavy).  The same arithmetic as
// vest_sd_<n> + k_rowpass_delta (bit-identical) without the delta round trip
// through HBM.
const char* kFusedPrelude = R"CUDA(
struct Chunk { unsigned row, beg, end, slot; };
struct SparseFusedArgs {
  const unsigned* oc[8]; const double* f[8]; const float* g[8];
  const double* val; const Chunk* chunks; unsigned nchunks;
  double* row_base; int ld_n; const unsigned char* fmask;
  double* heavy_out; int stride_na; int reg; double lambda;
};
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
constexpr int kXld = 36;
// Gram of the staged columns (delta_0..delta_{J-1}, x): tile (1,1) only when
// delta has rows >= 8 (J > 8); for J == 8 it would hold x.x, which no one reads
template <int NC, bool T11>
__device__ __forceinline__ void gram_dmma(const double* X, double (&d)[3][2], int lane) {
  const int g = lane >> 2, tq = lane & 3;
#pragma unroll
  for (int kk = 0; kk < 8; ++kk) {
    const int e = 4 * kk + tq;
    const double f0 = X[g * kXld + e];
    dmma884(d[0][0], d[0][1], f0, f0);
    if constexpr (NC > 8) {
      const double f1 = X[(8 + g) * kXld + e];
      dmma884(d[1][0], d[1][1], f0, f1);
      if constexpr (T11) dmma884(d[2][0], d[2][1], f1, f1);
    }
  }
}

__device__ __forceinline__ void gram_coord(int t, int i, int lane, int& row, int& col) {
  const int I = t == 2 ? 1 : 0, J = t == 0 ? 0 : 1;
  row = 8 * I + (lane >> 2);
  col = 8 * J + 2 * (lane & 3) + i;
}
__device__ __forceinline__ void solve_row(int J, int reg, double lambda, const double* G, const double* xd,
                                          double* row, const unsigned char* mask, int lane) {
  double v = lane < J ? row[lane] : 0.0;
  for (int j = 0; j < J; ++j) {
    if (mask[j]) continue;
    const double prod = (lane < J && lane != j) ? G[j * J + lane] * v : 0.0;
    const double s = warp_sum(prod);
    const double lin = xd[j] - s;
    const double gjj = G[j * J + j];
    double nv = 0.0;
    bool upd;
    if (reg == 0) {
      const double den = gjj + lambda;
      upd = den != 0.0;
      nv = lin / den;
    } else {
      const double g = -2.0 * lin;
      const double d = 2.0 * gjj;
      if (d == 0.0) {
        upd = fabs(g) <= lambda;
        nv = 0.0;
      } else {
        upd = true;
        nv = g > lambda ? (lambda - g) / d : (g < -lambda ? -(lambda + g) / d : 0.0);
      }
    }
    if (upd && lane == j) v = nv;
  }
  if (lane < J) row[lane] = v;
}
)CUDA";

void emit_fused(std::ostringstream& o, const Ctx& c, int n) {
  std::vector<int> oth;
  const std::vector<Cell> cells = ordered_cells(c, n, oth);
  const int J = c.ranks[n];
  o << "extern \"C\" __global__ void __launch_bounds__(256, 2) vest_sf_" << n << "(const SparseFusedArgs a) {\n"
    << "  constexpr int J = " << J << ", NG = J * (J + 1) / 2;\n"
    << "  __shared__ double smem_d[8][16 * kXld];\n"
    << "  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;\n"
    << "  const unsigned ci = blockIdx.x * 8 + warp;\n"
    << "  if (ci >= a.nchunks) return;\n"
    << "  const Chunk ch = a.chunks[ci];\n"
    << "  double* wsm = smem_d[warp];\n"
    << "  for (int t = lane; t < 16 * kXld; t += 32) wsm[t] = 0.0;\n"
    << "  __syncwarp();\n"
    << "  double tc[3][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};\n"
    << "  for (unsigned base = ch.beg; base < ch.end; base += 32) {\n"
    << "    const bool valid = base + lane < ch.end;\n"
    << "    const unsigned pos = valid ? base + lane : ch.beg;\n";
  emit_row_loads(o, c, oth, 0, "pos");
  emit_cells(o, c, n, oth, cells, 1);
  for (int j = 0; j < J; ++j) o << "    wsm[" << j << " * kXld + lane] = valid ? d" << j << "e0 : 0.0;\n";
  o << "    wsm[J * kXld + lane] = valid ? __ldg(a.val + pos) : 0.0;\n"
    << "    __syncwarp();\n"
    << "    gram_dmma<J + 1, (J > 8)>(wsm, tc, lane);\n"
    << "    __syncwarp();\n"
    << "  }\n"
    << "  double* Gs = wsm;\n"
    << "  double* xd = wsm + J * J;\n"
    << "#pragma unroll\n"
    << "  for (int t = 0; t < (J + 1 > 8 ? 3 : 1); ++t) {\n"
    << "#pragma unroll\n"
    << "    for (int i = 0; i < 2; ++i) {\n"
    << "      int row, col;\n"
    << "      gram_coord(t, i, lane, row, col);\n"
    << "      const double v = tc[t][i];\n"
    << "      int slot = -1;\n"
    << "      if (row <= col && col < J) slot = row * J - row * (row - 1) / 2 + (col - row);\n"
    << "      else if (col == J && row < J) slot = NG + row;\n"
    << "      if (slot < 0) continue;\n"
    << "      if (ch.slot != 0xFFFFFFFFu) {\n"
    << "        a.heavy_out[(unsigned long long)ch.slot * a.stride_na + slot] = v;\n"
    << "      } else if (col == J) {\n"
    << "        xd[row] = v;\n"
    << "      } else {\n"
    << "        Gs[row * J + col] = v;\n"
    << "        Gs[col * J + row] = v;\n"
    << "      }\n"
    << "    }\n"
    << "  }\n"
    << "  if (ch.slot != 0xFFFFFFFFu) return;\n"
    << "  __syncwarp();\n"
    << "  solve_row(J, a.reg, a.lambda, Gs, xd, a.row_base + (unsigned long long)ch.row * a.ld_n,\n"
    << "            a.fmask + (unsigned long long)ch.row * J, lane);\n"
    << "}\n";
}

// the fused kernel's DMMA tile holds (delta, x): J + 1 <= 16
bool fused_ok(const Ctx& c) {
  for (int k = 0; k < c.N; ++k)
    if (c.ranks[k] + 1 > 16) return false;
  return true;
}

const char* kModeMark = "//@@MODE\n";

std::string gen_source(const Ctx& c) {
  std::ostringstream o;
  o << "struct SparseDeltaArgs { const unsigned* oc[" << VEST_MAXN << "]; const double* f[" << VEST_MAXN
    << "]; const float* g[" << VEST_MAXN << "]; double* out; unsigned long long p0, n, stride; };\n"
    << "extern \"C\" __constant__ double G[" << c.G << "];\n";
  if (sd_f32(c))  // the core rounded to fp32 for the fp32 contraction (staged in Gf_src, copied to the bank)
    o << "extern \"C\" __constant__ float Gf[" << c.G << "];\n"
      << "extern \"C\" __device__ float Gf_src[" << c.G << "];\n"
      << "extern \"C\" __global__ void vest_core_f32(const double* s) {\n"
      << "  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < " << c.G << "; i += gridDim.x * blockDim.x) Gf_src[i] = (float)s[i];\n"
      << "}\n";
  const bool fused = sparse_fused_enabled(c);  // off by default: not worth half the compile time
  if (fused) o << kFusedPrelude;
  for (int n = 0; n < c.N; ++n) {  // one program per mode (sparse_compile cuts here)
    o << kModeMark;
    emit_mode(o, c, n);
    if (fused) emit_fused(o, c, n);
  }
  return o.str();
}

uint64_t mask_key(const Ctx& c) {
  uint64_t h = 1469598103934665603ull;  // FNV-1a over shape and mask
  auto mix = [&](uint64_t v) {
    h ^= v;
    h *= 1099511628211ull;
  };
  mix((uint64_t)c.N);
  for (int k = 0; k < c.N; ++k) mix((uint64_t)c.ranks[k] << 8 | (uint64_t)c.ld[k]);
  for (uint8_t m : c.h_core_mask) mix(m);
  mix(0xF32u + (uint64_t)c.gather_f32);
  mix(0x5DF32u + (uint64_t)sd_f32(c) * 16 + (uint64_t)sd_entries(c));
  mix(0xF05Du + (uint64_t)sparse_fused_enabled(c));
  return h;
}

}  // namespace

// One module per mode (compiled in parallel, sparse_compile): each carries its
// own copy of the core constant bank(s), loaded before its kernel runs.
struct SparseState {
  uint64_t key = 0;
  cudaLibrary_t lib[VEST_MAXN] = {};
  cudaKernel_t k[VEST_MAXN] = {};
  cudaKernel_t kf[VEST_MAXN] = {};  // fused factor-mode updates (vest_sf_<n>)
  double* G[VEST_MAXN] = {};
  float* Gf[VEST_MAXN] = {};  // fp32 contraction: the bank copy and its staging buffer
  float* Gf_src[VEST_MAXN] = {};
  cudaKernel_t core_f32[VEST_MAXN] = {};
  double compile_s = 0.0;
};

void sparse_free(Ctx& c) {
  if (!c.sparse) return;
  for (cudaLibrary_t l : c.sparse->lib)
    if (l) cudaLibraryUnload(l);
  delete c.sparse;
  c.sparse = nullptr;
}

bool nvrtc_available() {
  const Nvrtc& nv = nvrtc();
  return nv.h && nv.create && nv.compile && nv.cubin;
}

// Live-cell threshold: the generated contraction costs ~2 FMA per unmasked
// cell against >= |G| for the dense factorised one.
static int sparse_mode(const Ctx& c) {
  static const int env = [] {  // VEST_SPARSE_DELTA=0/1 overrides "auto" (A/B timing)
    const char* e = getenv("VEST_SPARSE_DELTA");
    return e && (e[0] == '0' || e[0] == '1') ? e[0] - '0' : -1;
  }();
  return c.sparse_delta >= 0 ? c.sparse_delta : env;
}

// The mask qualifies (or the path is forced on).
bool sparse_delta_eligible(const Ctx& c) {
  const int mode = sparse_mode(c);
  if (mode == 0 || c.N < 2) return false;
  for (int k = 0; k < c.N; ++k)
    if (c.ranks[k] > 15) return false;  // the statistics kernel's DMMA tile
  if (mode == 1) return true;
  if (!c.ops || c.force_generic || !nvrtc_available()) return false;
  long live = 0;
  for (uint8_t m : c.h_core_mask) live += !m;
  return 4 * live < c.G;
}

// ... and, in auto mode, the mask has outlived one sweep.
bool sparse_delta_enabled(const Ctx& c) {
  if (!sparse_delta_eligible(c)) return false;
  return sparse_mode(c) == 1 || c.mask_sweeps >= 2;
}

uint64_t core_mask_hash(const Ctx& c) { return mask_key(c); }

// VEST_NVRTC_ASYNC=0: compile the mask's kernels where they are first used (A/B)
static bool nvrtc_async() {
  static const bool v = [] {
    const char* e = getenv("VEST_NVRTC_ASYNC");
    return !(e && e[0] == '0');
  }();
  return v;
}

std::vector<char> nvrtc_compile(const std::string& src, const char* name);
std::vector<char> sparse_compile(const std::string& src, const char* name);

// Start compiling `src` on a host thread unless that key is already in the
// slot.  A superseded compile that is still running is parked (its future's
// destructor would block); while one is parked no new compile is started -- a
// schedule that prunes every iteration must not pile up compiler threads.
void prefetch_cubin(Ctx& c, Ctx::AsyncCubin& slot, uint64_t key, std::string src, const char* name, CompileFn fn) {
  if (!fn) fn = nvrtc_compile;
  if (!nvrtc_async()) return;
  if (slot.valid && slot.key == key) return;
  auto running = [](const std::shared_future<std::vector<char>>& f) {
    return f.valid() && f.wait_for(std::chrono::seconds(0)) != std::future_status::ready;
  };
  if (slot.valid && running(slot.fut)) c.pre_stale.push_back(slot.fut);
  slot.valid = false;
  for (size_t i = 0; i < c.pre_stale.size();)
    if (running(c.pre_stale[i])) ++i;
    else c.pre_stale.erase(c.pre_stale.begin() + (long)i);
  if (!c.pre_stale.empty()) return;
  slot.key = key;
  try {
    slot.fut = std::async(std::launch::async, [s = std::move(src), name, fn]() { return fn(s, name); }).share();
    slot.valid = true;
  } catch (const std::system_error&) {  // no thread to be had: the kernels are compiled where first used
    slot.valid = false;
  }
}

// The slot's cubin when it was compiled for `key` (waits for the compile).
bool take_cubin(Ctx::AsyncCubin& slot, uint64_t key, std::vector<char>& out) {
  if (!slot.valid || slot.key != key) return false;
  slot.valid = false;
  out = slot.fut.get();  // rethrows a compile error
  return true;
}

void note_sweep(Ctx& c) {
  const uint64_t key = mask_key(c);
  if (key == c.mask_key && c.mask_sweeps > 0) {
    ++c.mask_sweeps;
  } else {
    c.mask_key = key;
    c.mask_sweeps = 1;
    // auto mode switches the mask's kernels in from the next sweep: compile them now, off-thread
    if (sparse_mode(c) < 0 && sparse_delta_eligible(c) && !(c.sparse && c.sparse->key == key))
      prefetch_cubin(c, c.pre_sparse, key, gen_source(c), "vest_sparse_delta.cu", sparse_compile);
    core_gen_prefetch(c);
  }
}

std::vector<char> nvrtc_compile(const std::string& src, const char* name) {
  const Nvrtc& nv = nvrtc();
  if (!nv.h || !nv.create || !nv.compile || !nv.cubin) throw RtError{"libnvrtc not found (mask-specialised kernels)"};
  void* prog = nullptr;
  if (nv.create(&prog, src.c_str(), name, 0, nullptr, nullptr) != 0)
    throw RtError{"nvrtcCreateProgram failed"};
  const char* opts[] = {"--gpu-architecture=sm_100a", "--std=c++17", "-default-device"};
  const int rc = nv.compile(prog, 3, opts);
  if (rc != 0) {
    size_t ls = 0;
    nv.log_size(prog, &ls);
    std::string log(ls, '\0');
    nv.log(prog, &log[0]);
    nv.destroy(&prog);
    throw RtError{std::string("NVRTC compile failed (") + name + "): " + log.substr(0, 2000)};
  }
  size_t sz = 0;
  nv.cubin_size(prog, &sz);
  std::vector<char> cubin(sz);
  nv.cubin(prog, cubin.data());
  nv.destroy(&prog);
  if (const char* dir = getenv("VEST_NVRTC_DUMP")) {  // inspection: source + cubin (cuobjdump -sass)
    const std::string base = std::string(dir) + "/" + name;
    if (FILE* f = fopen((base + ".src").c_str(), "w")) {
      fwrite(src.data(), 1, src.size(), f);
      fclose(f);
    }
    if (FILE* f = fopen((base + ".cubin").c_str(), "wb")) {
      fwrite(cubin.data(), 1, cubin.size(), f);
      fclose(f);
    }
  }
  return cubin;
}

// The common head (argument struct, constant banks, fused prelude) plus one
// mode's kernels per program, compiled on parallel host threads; one blob
// [count | sizes | cubins], program n = mode n.
std::vector<char> sparse_compile(const std::string& src, const char* name) {
  std::vector<size_t> cut;
  for (size_t p = src.find(kModeMark); p != std::string::npos; p = src.find(kModeMark, p + 1)) cut.push_back(p);
  const int np = (int)cut.size();
  if (np == 0) throw RtError{"sparse delta source without mode marks"};
  std::vector<std::string> part(np), pname(np);
  for (int q = 0; q < np; ++q) {
    part[q] = src.substr(0, cut[0]) + src.substr(cut[q], (q + 1 < np ? cut[q + 1] : src.size()) - cut[q]);
    pname[q] = std::string(name) + (q ? ".m" + std::to_string(q) : "");
  }
  std::vector<std::future<std::vector<char>>> fut;
  for (int q = 1; q < np; ++q)  // deferred (= compiled in get() below) when no thread can be started
    fut.push_back(std::async(std::launch::async | std::launch::deferred,
                             [&part, &pname, q]() { return nvrtc_compile(part[q], pname[q].c_str()); }));
  std::vector<std::vector<char>> bin(np);
  std::exception_ptr err;
  try {
    bin[0] = nvrtc_compile(part[0], pname[0].c_str());
  } catch (...) {
    err = std::current_exception();
  }
  for (int q = 1; q < np; ++q) {
    try {
      bin[q] = fut[q - 1].get();
    } catch (...) {
      if (!err) err = std::current_exception();
    }
  }
  if (err) std::rethrow_exception(err);
  std::vector<char> blob((size_t)(1 + np) * sizeof(uint64_t));
  uint64_t* hdr = reinterpret_cast<uint64_t*>(blob.data());
  hdr[0] = (uint64_t)np;
  for (int q = 0; q < np; ++q) hdr[1 + q] = bin[q].size();
  for (int q = 0; q < np; ++q) blob.insert(blob.end(), bin[q].begin(), bin[q].end());
  return blob;
}

static void ensure_module(Ctx& c) {
  const uint64_t key = mask_key(c);
  if (c.sparse && c.sparse->key == key) return;
  sparse_free(c);
  std::vector<char> cubin;
  if (!take_cubin(c.pre_sparse, key, cubin)) cubin = sparse_compile(gen_source(c), "vest_sparse_delta.cu");
  auto* s = new SparseState;
  s->key = key;
  uint64_t nparts = 0;
  memcpy(&nparts, cubin.data(), sizeof(uint64_t));
  if ((int)nparts != c.N) throw RtError{"sparse delta: one program per mode expected"};
  std::vector<uint64_t> sz(nparts);
  memcpy(sz.data(), cubin.data() + sizeof(uint64_t), nparts * sizeof(uint64_t));
  size_t off = (size_t)(1 + nparts) * sizeof(uint64_t);
  for (int n = 0; n < c.N; ++n) {
    check(cudaLibraryLoadData(&s->lib[n], cubin.data() + off, nullptr, nullptr, 0, nullptr, nullptr, 0),
          "sparse delta load");
    off += sz[n];
    const std::string nm = "vest_sd_" + std::to_string(n);
    check(cudaLibraryGetKernel(&s->k[n], s->lib[n], nm.c_str()), "sparse delta kernel");
    if (sparse_fused_enabled(c)) {
      const std::string nf = "vest_sf_" + std::to_string(n);
      check(cudaLibraryGetKernel(&s->kf[n], s->lib[n], nf.c_str()), "fused factor kernel");
    }
    size_t gb = 0;
    check(cudaLibraryGetGlobal(reinterpret_cast<void**>(&s->G[n]), &gb, s->lib[n], "G"), "sparse delta core symbol");
    if (sd_f32(c)) {
      check(cudaLibraryGetGlobal(reinterpret_cast<void**>(&s->Gf[n]), &gb, s->lib[n], "Gf"), "sparse delta core symbol");
      check(cudaLibraryGetGlobal(reinterpret_cast<void**>(&s->Gf_src[n]), &gb, s->lib[n], "Gf_src"),
            "sparse delta core symbol");
      check(cudaLibraryGetKernel(&s->core_f32[n], s->lib[n], "vest_core_f32"), "sparse delta core kernel");
    }
  }
  c.sparse = s;
}

// delta[j][pos - p0] for the positions [p0, p0 + n) of mode `mode`'s CSF
void sparse_delta(Ctx& c, int mode, uint64_t p0, uint64_t n, double* out) {
  ensure_module(c);
  if (n == 0) return;
  if (c.sparse->Gf[mode]) {  // fp32 contraction: the core rounded to fp32 into its constant bank
    const double* src = c.d_core;
    void* cargs[] = {&src};
    check(cudaLaunchKernel(reinterpret_cast<const void*>(c.sparse->core_f32[mode]), dim3((c.G + 255) / 256), dim3(256), cargs,
                           0, c.stream),
          "sparse delta core (fp32)");
    count_launch();
    check(cudaMemcpyAsync(c.sparse->Gf[mode], c.sparse->Gf_src[mode], sizeof(float) * c.G, cudaMemcpyDeviceToDevice,
                          c.stream),
          "sparse delta core (fp32)");
  } else {
    check(cudaMemcpyAsync(c.sparse->G[mode], c.d_core, sizeof(double) * c.G, cudaMemcpyDeviceToDevice, c.stream),
          "sparse delta core");
  }
  SparseDeltaArgs a{};
  const DevCSF csf = c.csf_view(mode);
  if (c.gather_f32) refresh_factor_shadows(c, mode);
  for (int k = 0; k < c.N; ++k) {
    a.oc[k] = csf.oc[k];
    a.f[k] = c.d_factor[k];
    a.g[k] = c.d_factor32[k];
  }
  a.out = out;
  a.p0 = p0;
  a.n = n;
  a.stride = n;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c.device);
  const uint64_t per_cta = 256ull * sd_entries(c);
  const unsigned grid = (unsigned)std::min<uint64_t>((n + per_cta - 1) / per_cta, (uint64_t)sms * 2 * sd_min_blocks());
  void* args[] = {&a};
  check(cudaLaunchKernel(reinterpret_cast<const void*>(c.sparse->k[mode]), dim3(grid), dim3(256), args, 0, c.stream),
        "sparse delta launch");
  count_launch();
}

struct SparseFusedArgs {
  const uint32_t* oc[VEST_MAXN];
  const double* f[VEST_MAXN];
  const float* g[VEST_MAXN];
  const double* val;
  const Chunk* chunks;
  uint32_t nchunks;
  double* row_base;
  int ld_n;
  const uint8_t* fmask;
  double* heavy_out;
  int stride_na;
  int reg;
  double lambda;
};

bool sparse_fused_enabled(const Ctx& c) {
  static const int env = [] {  // VEST_SPARSE_FUSED=0 selects vest_sd + k_rowpass_delta (A/B timing)
    const char* e = getenv("VEST_SPARSE_FUSED");
    return e && (e[0] == '0' || e[0] == '1') ? e[0] - '0' : -1;
  }();
  const int mode = c.sparse_fused >= 0 ? c.sparse_fused : env;
  return mode == 1 && fused_ok(c);  // auto = off: measured slower than vest_sd + k_rowpass_delta
}

// One factor mode through the fused kernel (statistics + light-row solves),
// then k_heavy for rows split over several chunks.
void sparse_fused(Ctx& c, int mode, const RowPassArgs& ra) {
  ensure_module(c);
  if (c.gather_f32) refresh_factor_shadows(c, mode);
  if (ra.csf.nchunks > 0) {
    SparseFusedArgs a{};
    for (int k = 0; k < c.N; ++k) {
      a.oc[k] = ra.csf.oc[k];
      a.f[k] = c.d_factor[k];
      a.g[k] = c.d_factor32[k];
    }
    a.val = ra.csf.val;
    a.chunks = ra.csf.chunks;
    a.nchunks = ra.csf.nchunks;
    a.row_base = ra.m.factor[mode];
    a.ld_n = ra.m.ld[mode];
    a.fmask = ra.m.fmask[mode];
    a.heavy_out = ra.heavy_out;
    a.stride_na = ra.stride_na;
    a.reg = ra.reg;
    a.lambda = ra.lambda;
    check(cudaMemcpyAsync(c.sparse->G[mode], c.d_core, sizeof(double) * c.G, cudaMemcpyDeviceToDevice, c.stream),
          "sparse delta core");
    void* args[] = {&a};
    check(cudaLaunchKernel(reinterpret_cast<const void*>(c.sparse->kf[mode]), dim3((ra.csf.nchunks + 7) / 8),
                           dim3(256), args, 0, c.stream),
          "fused factor launch");
    count_launch();
  }
  check(launch_heavy_stats(ra, c.stream), "heavy rows");
}

// Host-only check (no GPU needed): generate and NVRTC-compile the
// contraction for a shape and core mask; returns the cubin size in *bytes.
int sparse_compile_check(int N, const int* ranks, const uint8_t* core_mask, uint64_t* bytes, std::string* err) {
  try {
    Ctx c;
    c.N = N;
    c.G = 1;
    for (int k = 0; k < N; ++k) {
      c.ranks[k] = ranks[k];
      c.ld[k] = (ranks[k] + 1) & ~1;
      c.G *= ranks[k];
    }
    c.h_core_mask.assign(core_mask, core_mask + c.G);
    if (const char* e = getenv("VEST_GATHER_F32")) c.gather_f32 = e[0] == '1';
    c.stats_f32 = c.gather_f32;  // the fp32-statistics form of the passes too
    *bytes = nvrtc_compile(gen_source(c), "vest_sparse_delta.cu").size();
    if (N >= 2) {  // the plan-specialised core passes of the same mask
      std::vector<int> nts;
      int ldr = 0;
      *bytes += nvrtc_compile(core_gen_source(c, core_gen_plan(c), nts, ldr), "vest_core_gen.cu").size();
    }
    return 0;
  } catch (const RtError& e) {
    *err = e.msg;
    return 1;
  }
}

}  // namespace vest
