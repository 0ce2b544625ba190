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
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <sstream>
#include <string>
#include <vector>

#include "vest_internal.h"

namespace vest {

struct SparseDeltaArgs {
  const uint32_t* oc[VEST_MAXN];
  const double* f[VEST_MAXN];
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

void emit_mode(std::ostringstream& o, const Ctx& c, int n) {
  const int N = c.N;
  std::vector<int> oth;
  for (int k = 0; k < N; ++k)
    if (k != n) oth.push_back(k);
  const int L = (int)oth.size();  // other modes; the last one is contracted innermost
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
  // order: other modes but the last (prefix), then beta_n, then the last other mode
  auto key = [&](const Cell& a, const Cell& b) {
    for (int q = 0; q + 1 < L; ++q)
      if (a.beta[oth[q]] != b.beta[oth[q]]) return a.beta[oth[q]] < b.beta[oth[q]];
    if (a.beta[n] != b.beta[n]) return a.beta[n] < b.beta[n];
    return a.beta[oth[L - 1]] < b.beta[oth[L - 1]];
  };
  std::sort(cells.begin(), cells.end(), key);

  // two entries per thread (E = 0, 1: t and t + 256 of the block's stride
  // window): every core value is loaded once (uniform constant load) and
  // feeds both entries' FMAs
  o << "extern \"C\" __global__ void __launch_bounds__(256, 2) vest_sd_" << n << "(const SparseDeltaArgs a) {\n"
    << "  for (unsigned long long t0 = blockIdx.x * 512ull + threadIdx.x; t0 < a.n; t0 += gridDim.x * 512ull) {\n"
    << "    const unsigned long long t1 = t0 + 256ull < a.n ? t0 + 256ull : t0;\n";
  for (int e = 0; e < 2; ++e) {
    const std::string E = std::to_string(e);
    for (int k : oth) {
      const int ld = c.ld[k];
      const std::string rk = "r" + std::to_string(k) + "e" + E;
      o << "    const double* " << rk << " = a.f[" << k << "] + (unsigned long long)__ldg(a.oc[" << k << "] + a.p0 + t"
        << E << ") * " << ld << "ull;\n";
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
    for (int j = 0; j < c.ranks[n]; ++j) o << "    double d" << j << "e" << E << " = 0.0;\n";
  }
  auto same_prefix = [&](const Cell& a, const Cell& b, int upto) {
    for (int q = 0; q <= upto; ++q)
      if (a.beta[oth[q]] != b.beta[oth[q]]) return false;
    return true;
  };
  size_t i = 0;
  while (i < cells.size()) {
    // open the prefix levels of cells[i] (both entries)
    for (int q = 0; q + 1 < L; ++q) {
      const int k = oth[q], b = cells[i].beta[k];
      o << "    {";
      for (int e = 0; e < 2; ++e) {
        const std::string E = std::to_string(e);
        if (q == 0) o << " const double w0e" << E << " = " << u(k, b) << "e" << E << ";";
        else o << " const double w" << q << "e" << E << " = w" << (q - 1) << "e" << E << " * " << u(k, b) << "e" << E << ";";
      }
      o << "\n";
    }
    size_t e_end = i;
    while (e_end < cells.size() && (L < 2 || same_prefix(cells[i], cells[e_end], L - 2))) ++e_end;
    const int kl = oth[L - 1];
    for (size_t g = i; g < e_end;) {
      const int bn = cells[g].beta[n];
      size_t h = g;
      o << "      { double g = G[" << cells[h].lin << "]; double t0 = g * " << u(kl, cells[h].beta[kl]) << "e0, t1 = g * "
        << u(kl, cells[h].beta[kl]) << "e1;";
      for (++h; h < e_end && cells[h].beta[n] == bn; ++h)
        o << " g = G[" << cells[h].lin << "]; t0 = fma(g, " << u(kl, cells[h].beta[kl]) << "e0, t0); t1 = fma(g, "
          << u(kl, cells[h].beta[kl]) << "e1, t1);";
      if (L >= 2)
        o << " d" << bn << "e0 = fma(w" << (L - 2) << "e0, t0, d" << bn << "e0); d" << bn << "e1 = fma(w" << (L - 2)
          << "e1, t1, d" << bn << "e1); }\n";
      else
        o << " d" << bn << "e0 += t0; d" << bn << "e1 += t1; }\n";
      g = h;
    }
    for (int q = 0; q + 1 < L; ++q) o << "    }\n";
    i = e_end;
  }
  for (int j = 0; j < c.ranks[n]; ++j) o << "    a.out[" << j << "ull * a.stride + t0] = d" << j << "e0;\n";
  o << "    if (t1 != t0) {\n";
  for (int j = 0; j < c.ranks[n]; ++j) o << "      a.out[" << j << "ull * a.stride + t1] = d" << j << "e1;\n";
  o << "    }\n  }\n}\n";
}

std::string gen_source(const Ctx& c) {
  std::ostringstream o;
  o << "struct SparseDeltaArgs { const unsigned* oc[" << VEST_MAXN << "]; const double* f[" << VEST_MAXN
    << "]; double* out; unsigned long long p0, n, stride; };\n"
    << "extern \"C\" __constant__ double G[" << c.G << "];\n";
  for (int n = 0; n < c.N; ++n) emit_mode(o, c, n);
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
  return h;
}

}  // namespace

struct SparseState {
  uint64_t key = 0;
  cudaLibrary_t lib = nullptr;
  cudaKernel_t k[VEST_MAXN] = {};
  double* G = nullptr;
  double compile_s = 0.0;
};

void sparse_free(Ctx& c) {
  if (!c.sparse) return;
  if (c.sparse->lib) cudaLibraryUnload(c.sparse->lib);
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

void note_sweep(Ctx& c) {
  const uint64_t key = mask_key(c);
  if (key == c.mask_key && c.mask_sweeps > 0) {
    ++c.mask_sweeps;
  } else {
    c.mask_key = key;
    c.mask_sweeps = 1;
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

static void ensure_module(Ctx& c) {
  const uint64_t key = mask_key(c);
  if (c.sparse && c.sparse->key == key) return;
  sparse_free(c);
  const std::vector<char> cubin = nvrtc_compile(gen_source(c), "vest_sparse_delta.cu");
  auto* s = new SparseState;
  s->key = key;
  check(cudaLibraryLoadData(&s->lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0), "sparse delta load");
  for (int n = 0; n < c.N; ++n) {
    const std::string nm = "vest_sd_" + std::to_string(n);
    check(cudaLibraryGetKernel(&s->k[n], s->lib, nm.c_str()), "sparse delta kernel");
  }
  size_t gb = 0;
  check(cudaLibraryGetGlobal(reinterpret_cast<void**>(&s->G), &gb, s->lib, "G"), "sparse delta core symbol");
  c.sparse = s;
}

// delta[j][pos - p0] for the positions [p0, p0 + n) of mode `mode`'s CSF
void sparse_delta(Ctx& c, int mode, uint64_t p0, uint64_t n, double* out) {
  ensure_module(c);
  if (n == 0) return;
  check(cudaMemcpyAsync(c.sparse->G, c.d_core, sizeof(double) * c.G, cudaMemcpyDeviceToDevice, c.stream),
        "sparse delta core");
  SparseDeltaArgs a{};
  const DevCSF csf = c.csf_view(mode);
  for (int k = 0; k < c.N; ++k) {
    a.oc[k] = csf.oc[k];
    a.f[k] = c.d_factor[k];
  }
  a.out = out;
  a.p0 = p0;
  a.n = n;
  a.stride = n;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c.device);
  const unsigned grid = (unsigned)std::min<uint64_t>((n + 511) / 512, (uint64_t)sms * 4);
  void* args[] = {&a};
  check(cudaLaunchKernel(reinterpret_cast<const void*>(c.sparse->k[mode]), dim3(grid), dim3(256), args, 0, c.stream),
        "sparse delta launch");
  count_launch();
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
