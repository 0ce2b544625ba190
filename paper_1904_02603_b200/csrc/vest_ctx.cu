// SPDX-License-Identifier: Apache-2.0
// vest_ctx.cu -- device context: tensor validation and the per-mode CSF build
// (make_tensor / build_mode_index, sparse_tensor.hpp:68-137), model storage,
// the orchestration of the hot path (update_all_factors, core sweep,
// residuals, responsibilities, prune), and the C-ABI of include/vest.h.

#include <algorithm>
#include <cmath>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "../../include/vest.h"
#include "vest_common.cuh"

namespace vest {

void core_responsibilities(Ctx& c);
void fill_factor_resp(Ctx& c, int n, double unmasked);
void l1_empty_rows(Ctx& c, int n, double lambda);

uint64_t& launch_counter() {
  static uint64_t n = 0;
  return n;
}

void check(cudaError_t e, const char* where) {
  if (e != cudaSuccess) throw CudaError{e, where};
}

void comm_allreduce(Ctx& c, double* p, uint64_t n) {
  if (!c.comm.allreduce_sum) return;
  if (c.comm.allreduce_sum(c.comm.user, p, n, (void*)c.stream) != 0) throw RtError{"allreduce_sum hook failed"};
}

void comm_allgather_rows(Ctx& c, int mode, double* base, uint64_t ld) {
  if (!c.comm.allgather_rows) return;
  if (c.comm.allgather_rows(c.comm.user, mode, base, ld, (void*)c.stream) != 0)
    throw RtError{"allgather_rows hook failed"};
}

void* dalloc(Ctx& c, size_t bytes) {
  void* p = nullptr;
  if (bytes == 0) bytes = 16;
  check(cudaMalloc(&p, bytes), "cudaMalloc");
  c.device_bytes += bytes;
  ++c.alloc_epoch;
  return p;
}

void ensure(Ctx& c, double** p, size_t* cap, size_t n) {
  if (*cap >= n && *p) return;
  if (*p) {
    check(cudaStreamSynchronize(c.stream), "ensure sync");
    cudaFree(*p);
    c.device_bytes -= *cap * sizeof(double);
  }
  n = std::max<size_t>(n, 16);
  *p = static_cast<double*>(dalloc(c, n * sizeof(double)));
  *cap = n;
}

DevModel Ctx::model_view() const {
  DevModel m{};
  for (int k = 0; k < N; ++k) {
    m.factor[k] = d_factor[k];
    m.fmask[k] = d_fmask[k];
    m.ld[k] = ld[k];
    m.J[k] = ranks[k];
    m.I[k] = dims[k];
  }
  int s = 1;
  for (int k = N - 1; k >= 0; --k) {
    m.stride[k] = s;
    s *= ranks[k];
  }
  m.core = d_core;
  m.core_mask = d_core_mask;
  m.cellbeta = d_cellbeta;
  m.N = N;
  m.G = G;
  return m;
}

DevCSF Ctx::csf_view(int mode) const {
  const ModeData& md = modes[mode];
  DevCSF v{};
  for (int k = 0; k < N; ++k) v.oc[k] = md.d_oc[k];
  v.val = md.d_val;
  v.eid = md.d_eid;
  v.offsets = md.d_offsets;
  v.chunks = md.d_chunks;
  v.heavy = md.d_heavy;
  v.nchunks = md.nchunks;
  v.nheavy = md.nheavy;
  v.nslots = md.nslots;
  v.mode = mode;
  return v;
}

// ------------------------------------------------------------------ build --
__global__ void k_bounds(const uint32_t* coords, uint64_t nnz, int N, DevModel m, int* flag) {
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < nnz * N; t += (uint64_t)gridDim.x * blockDim.x)
    if (coords[t] >= m.I[t % N]) atomicExch(flag, 1);
}

__global__ void k_gather_key(const uint32_t* coords, const uint32_t* perm, uint64_t nnz, int N, int k,
                             uint32_t* keys) {
  for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < nnz; p += (uint64_t)gridDim.x * blockDim.x)
    keys[p] = coords[(uint64_t)(perm ? perm[p] : p) * N + k];
}

__global__ void k_iota(uint32_t* v, uint64_t n) {
  for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < n; p += (uint64_t)gridDim.x * blockDim.x)
    v[p] = (uint32_t)p;
}

__global__ void k_dups(const uint32_t* coords, const uint32_t* perm, uint64_t nnz, int N, int* flag) {
  for (uint64_t p = 1 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < nnz; p += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t* a = coords + (uint64_t)perm[p - 1] * N;
    const uint32_t* b = coords + (uint64_t)perm[p] * N;
    bool eq = true;
    for (int k = 0; k < N; ++k) eq = eq && a[k] == b[k];
    if (eq) atomicExch(flag, 1);
  }
}

__global__ void k_offsets(const uint32_t* sorted_keys, uint64_t nnz, uint64_t I, uint64_t* off) {
  // off[i] = lower_bound(keys, i)
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i <= I; i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t lo = 0, hi = nnz;
    while (lo < hi) {
      const uint64_t mid = (lo + hi) / 2;
      if (sorted_keys[mid] < i) lo = mid + 1; else hi = mid;
    }
    off[i] = lo;
  }
}

__global__ void k_csf_fill(const uint32_t* coords, const double* values, const uint32_t* eid, uint64_t nnz,
                           int N, int k, uint32_t* oc, double* val) {
  for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < nnz; p += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t e = eid[p];
    if (oc) oc[p] = coords[e * N + k];
    if (val) val[p] = values[e];
  }
}

__global__ void k_cellbeta(uint32_t* cb, int G, int N, DevModel m) {
  const int lin = blockIdx.x * blockDim.x + threadIdx.x;
  if (lin >= G) return;
  uint32_t packed = 0;
  int rest = lin;
  for (int k = N - 1; k >= 0; --k) {
    packed |= (uint32_t)(rest % m.J[k]) << (4 * k);
    rest /= m.J[k];
  }
  cb[lin] = packed;
}

// stable sort of (key, value) pairs by the key's low end_bit bits (vest_sort.cu)
static void sort_pairs(Ctx& c, const uint32_t* kin, uint32_t* kout, const uint32_t* vin, uint32_t* vout, uint64_t n,
                       int end_bit, void*& tmp, size_t& tmp_bytes) {
  const size_t need = radix_sort_tmp_bytes(n);
  if (need > tmp_bytes) {
    if (tmp) {
      check(cudaStreamSynchronize(c.stream), "sync");
      cudaFree(tmp);
    }
    check(cudaMalloc(&tmp, need), "sort tmp");
    tmp_bytes = need;
  }
  count_launch(radix_sort_pairs(kin, kout, vin, vout, n, end_bit, tmp, c.stream));
  check(cudaGetLastError(), "radix sort");
}

static int bits_for(uint64_t d) {
  int b = 1;
  while (b < 32 && (1ull << b) < d) ++b;
  return b;
}

// rows up to this length run lane-per-row (VEST_TINY_MAX overrides kTinyRow: A/B timing)
static uint32_t tiny_max() {
  static const uint32_t v = [] {
    const char* e = getenv("VEST_TINY_MAX");
    return e ? (uint32_t)std::max(0, atoi(e)) : kTinyRow;
  }();
  return v;
}

// Keep only positions [p0, p1) of mode n's entry arrays (a shard's own rows;
// each GPU stores the mode-n CSF only for its row range), stored
// shifted by -p0 so that absolute CSF positions still index them.
static void compact_owned(Ctx& c, int n) {
  ModeData& md = c.modes[n];
  const uint64_t p0 = md.h_offsets[c.row_lo[n]], p1 = md.h_offsets[c.row_hi[n]];
  if (p0 == 0 && p1 == c.nnz) return;
  const uint64_t keep = std::max<uint64_t>(p1 - p0, 1), full = std::max<uint64_t>(c.nnz, 1);
  auto shrink = [&](auto*& ptr, size_t elem) {
    using T = std::remove_reference_t<decltype(*ptr)>;
    T* fresh = static_cast<T*>(dalloc(c, keep * elem));
    if (p1 > p0) check(cudaMemcpyAsync(fresh, ptr + p0, (p1 - p0) * elem, cudaMemcpyDeviceToDevice, c.stream), "compact");
    check(cudaStreamSynchronize(c.stream), "compact");
    cudaFree(ptr);
    c.device_bytes -= full * elem;
    ptr = fresh - p0;
  };
  shrink(md.d_eid, sizeof(uint32_t));
  shrink(md.d_val, sizeof(double));
  for (int k = 0; k < c.N; ++k)
    if (k != n) shrink(md.d_oc[k], sizeof(uint32_t));
  md.pos0 = p0;
}

void build_csf(Ctx& c, const uint32_t* h_coords, const double* h_values) {
  const uint64_t nnz = c.nnz;
  const int N = c.N;
  uint32_t* d_coords = static_cast<uint32_t*>(nullptr);
  double* d_values = nullptr;
  uint32_t *keys = nullptr, *keys2 = nullptr, *perm = nullptr, *perm2 = nullptr;
  int* d_flag = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  const size_t cb = std::max<uint64_t>(nnz, 1);
  check(cudaMalloc(&d_coords, cb * N * sizeof(uint32_t)), "coords");
  check(cudaMalloc(&d_values, cb * sizeof(double)), "values");
  check(cudaMalloc(&keys, cb * 4), "keys");
  check(cudaMalloc(&keys2, cb * 4), "keys2");
  check(cudaMalloc(&perm, cb * 4), "perm");
  check(cudaMalloc(&perm2, cb * 4), "perm2");
  check(cudaMalloc(&d_flag, 2 * sizeof(int)), "flag");
  check(cudaMemsetAsync(d_flag, 0, 2 * sizeof(int), c.stream), "flag0");
  if (nnz) {
    check(cudaMemcpyAsync(d_coords, h_coords, nnz * N * sizeof(uint32_t), cudaMemcpyHostToDevice, c.stream), "h2d coords");
    check(cudaMemcpyAsync(d_values, h_values, nnz * sizeof(double), cudaMemcpyHostToDevice, c.stream), "h2d values");
  }
  const DevModel mv = c.model_view();
  const int grid = 1184;
  int flags[2] = {0, 0};
  if (nnz) {
    k_bounds<<<grid, 256, 0, c.stream>>>(d_coords, nnz, N, mv, d_flag);
    count_launch();
    check(cudaMemcpyAsync(flags, d_flag, sizeof(int), cudaMemcpyDeviceToHost, c.stream), "flag");
    check(cudaStreamSynchronize(c.stream), "bounds");
  }
  auto cleanup = [&]() {
    cudaFree(d_coords);
    cudaFree(d_values);
    cudaFree(keys);
    cudaFree(keys2);
    cudaFree(perm);
    cudaFree(perm2);
    cudaFree(d_flag);
    if (tmp) cudaFree(tmp);
  };
  if (flags[0]) {
    cleanup();
    throw ArgError{"coordinate out of bounds"};
  }
  // duplicates: stable LSD sort over the modes gives lexicographic order
  // (sparse_tensor.hpp:80-94 sorts by coordinate tuple and scans neighbours)
  if (nnz > 1) {
    k_iota<<<grid, 256, 0, c.stream>>>(perm, nnz);
    for (int k = N - 1; k >= 0; --k) {
      k_gather_key<<<grid, 256, 0, c.stream>>>(d_coords, perm, nnz, N, k, keys);
      sort_pairs(c, keys, keys2, perm, perm2, nnz, bits_for(c.dims[k]), tmp, tmp_bytes);
      std::swap(perm, perm2);
    }
    k_dups<<<grid, 256, 0, c.stream>>>(d_coords, perm, nnz, N, d_flag + 1);
    count_launch(2 + N);
    check(cudaMemcpyAsync(flags + 1, d_flag + 1, sizeof(int), cudaMemcpyDeviceToHost, c.stream), "dupflag");
    check(cudaStreamSynchronize(c.stream), "dups");
    if (flags[1]) {
      cleanup();
      throw ArgError{"duplicate coordinate in tensor"};
    }
  }
  // per-mode CSF: stable sort of entry ids by coordinate n -> ids ascending
  // within each slice, exactly the ModeIndex order (sparse_tensor.hpp:107-137)
  for (int n = 0; n < N; ++n) {
    ModeData& md = c.modes[n];
    md.d_offsets = static_cast<uint64_t*>(dalloc(c, (c.dims[n] + 1) * sizeof(uint64_t)));
    md.d_eid = static_cast<uint32_t*>(dalloc(c, cb * 4));
    md.d_val = static_cast<double*>(dalloc(c, cb * 8));
    for (int k = 0; k < N; ++k)
      if (k != n) md.d_oc[k] = static_cast<uint32_t*>(dalloc(c, cb * 4));
    if (nnz) {
      k_gather_key<<<grid, 256, 0, c.stream>>>(d_coords, nullptr, nnz, N, n, keys);
      k_iota<<<grid, 256, 0, c.stream>>>(perm, nnz);
      sort_pairs(c, keys, keys2, perm, md.d_eid, nnz, bits_for(c.dims[n]), tmp, tmp_bytes);
      k_offsets<<<grid, 256, 0, c.stream>>>(keys2, nnz, c.dims[n], md.d_offsets);
      for (int k = 0; k < N; ++k)
        if (k != n) k_csf_fill<<<grid, 256, 0, c.stream>>>(d_coords, d_values, md.d_eid, nnz, N, k, md.d_oc[k], nullptr);
      k_csf_fill<<<grid, 256, 0, c.stream>>>(d_coords, d_values, md.d_eid, nnz, N, 0, nullptr, md.d_val);
      count_launch(3 + N);
    } else {
      check(cudaMemsetAsync(md.d_offsets, 0, (c.dims[n] + 1) * sizeof(uint64_t), c.stream), "off0");
    }
    md.h_offsets.resize(c.dims[n] + 1);
    check(cudaMemcpyAsync(md.h_offsets.data(), md.d_offsets, (c.dims[n] + 1) * sizeof(uint64_t),
                          cudaMemcpyDeviceToHost, c.stream),
          "offsets");
    check(cudaStreamSynchronize(c.stream), "csf");
    // work list: chunks of <= kChunk entries of one row
    std::vector<Chunk> chunks;
    std::vector<Heavy> heavy;
    std::vector<uint32_t> empty;
    uint32_t slot = 0;
    c.local_nnz[n] = md.h_offsets[c.row_hi[n]] - md.h_offsets[c.row_lo[n]];
    compact_owned(c, n);  // a shard keeps only the CSF positions of its own rows
    {
      uint64_t mx = 0;
      for (uint64_t i = 0; i < c.dims[n]; ++i) mx = std::max(mx, md.h_offsets[i + 1] - md.h_offsets[i]);
      c.skewed[n] = c.nnz > 0 && mx * 1000 > c.nnz;
    }
    for (uint64_t i = c.row_lo[n]; i < c.row_hi[n]; ++i) {  // this context's rows
      const uint64_t b = md.h_offsets[i], e = md.h_offsets[i + 1], len = e - b;
      if (len == 0) {
        empty.push_back((uint32_t)i);
        continue;
      }
      if (len <= kChunk) {
        chunks.push_back({(uint32_t)i, (uint32_t)b, (uint32_t)e, kLight});
        continue;
      }
      const uint32_t nch = (uint32_t)((len + kChunk - 1) / kChunk);
      heavy.push_back({(uint32_t)i, slot, nch, 0});
      for (uint32_t q = 0; q < nch; ++q) {
        const uint64_t cb0 = b + len * q / nch, cb1 = b + len * (q + 1) / nch;
        chunks.push_back({(uint32_t)i, (uint32_t)cb0, (uint32_t)cb1, slot + q});
      }
      slot += nch;
    }
    std::vector<Chunk> hchunks;
    for (const Chunk& ch : chunks)
      if (ch.slot != kLight) hchunks.push_back(ch);
    md.nheavy_chunks = (uint32_t)hchunks.size();
    md.d_heavy_chunks = static_cast<Chunk*>(dalloc(c, std::max<size_t>(1, hchunks.size()) * sizeof(Chunk)));
    if (!hchunks.empty())
      check(cudaMemcpy(md.d_heavy_chunks, hchunks.data(), hchunks.size() * sizeof(Chunk), cudaMemcpyHostToDevice),
            "heavy chunks");
    {  // tiny rows (light, <= kTinyRow entries) sorted by length; the rest of the chunks
      std::vector<std::pair<uint32_t, uint32_t>> tiny;
      std::vector<Chunk> big;
      for (const Chunk& ch : chunks) {
        if (ch.slot == kLight && ch.end - ch.beg <= tiny_max()) tiny.push_back({ch.end - ch.beg, ch.row});
        else big.push_back(ch);
      }
      std::stable_sort(tiny.begin(), tiny.end(),
                       [](const std::pair<uint32_t, uint32_t>& x, const std::pair<uint32_t, uint32_t>& y) {
                         return x.first < y.first;
                       });
      std::vector<uint32_t> trows(tiny.size());
      for (size_t q = 0; q < tiny.size(); ++q) trows[q] = tiny[q].second;
      md.ntiny = (uint32_t)trows.size();
      md.nchunks_big = (uint32_t)big.size();
      md.d_tiny = static_cast<uint32_t*>(dalloc(c, std::max<size_t>(1, trows.size()) * 4));
      md.d_chunks_big = static_cast<Chunk*>(dalloc(c, std::max<size_t>(1, big.size()) * sizeof(Chunk)));
      if (!trows.empty())
        check(cudaMemcpy(md.d_tiny, trows.data(), trows.size() * 4, cudaMemcpyHostToDevice), "tiny rows");
      if (!big.empty())
        check(cudaMemcpy(md.d_chunks_big, big.data(), big.size() * sizeof(Chunk), cudaMemcpyHostToDevice), "big");
    }
    md.nchunks = (uint32_t)chunks.size();
    md.nheavy = (uint32_t)heavy.size();
    md.nslots = slot;
    md.nempty = (uint32_t)empty.size();
    md.d_chunks = static_cast<Chunk*>(dalloc(c, std::max<size_t>(1, chunks.size()) * sizeof(Chunk)));
    md.d_heavy = static_cast<Heavy*>(dalloc(c, std::max<size_t>(1, heavy.size()) * sizeof(Heavy)));
    md.d_empty = static_cast<uint32_t*>(dalloc(c, std::max<size_t>(1, empty.size()) * 4));
    if (!chunks.empty())
      check(cudaMemcpy(md.d_chunks, chunks.data(), chunks.size() * sizeof(Chunk), cudaMemcpyHostToDevice), "chunks");
    if (!heavy.empty())
      check(cudaMemcpy(md.d_heavy, heavy.data(), heavy.size() * sizeof(Heavy), cudaMemcpyHostToDevice), "heavy");
    if (!empty.empty())
      check(cudaMemcpy(md.d_empty, empty.data(), empty.size() * 4, cudaMemcpyHostToDevice), "empty");
  }
  cleanup();
}

// --------------------------------------------------------------- hot path --
// VEST_TINY_ROWS=0: short rows through the warp-per-chunk kernel (A/B timing)
static bool tiny_rows_off() {
  static const bool v = [] {
    const char* e = getenv("VEST_TINY_ROWS");
    return e && e[0] == '0';
  }();
  return v;
}

__global__ void k_factor_f32(const double* __restrict__ src, float* __restrict__ dst, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    dst[i] = (float)src[i];  // round to nearest; same (row, ld) layout as d_factor
}

void refresh_factor_shadows(Ctx& c, int skip_mode) {
  if (!c.d_factor32[0]) {  // one contiguous buffer, modes in order (one L2 access-policy window covers them)
    uint64_t off[VEST_MAXN + 1] = {};
    for (int k = 0; k < c.N; ++k) off[k + 1] = off[k] + ((c.dims[k] * (uint64_t)c.ld[k] + 63) & ~63ull);
    float* base = static_cast<float*>(dalloc(c, std::max<uint64_t>(off[c.N], 1) * sizeof(float)));
    for (int k = 0; k < c.N; ++k) c.d_factor32[k] = base + off[k];
  }
  for (int k = 0; k < c.N; ++k) {
    if (k == skip_mode) continue;
    const uint64_t n = c.dims[k] * (uint64_t)c.ld[k];
    k_factor_f32<<<592, 256, 0, c.stream>>>(c.d_factor[k], c.d_factor32[k], n);
    count_launch();
  }
  check(cudaGetLastError(), "factor shadows");
}

static RowPassArgs row_args(Ctx& c, int mode) {
  RowPassArgs a{};
  a.m = c.model_view();
  a.csf = c.csf_view(mode);
  a.mode = mode;
  return a;
}

static cudaError_t run_rows(Ctx& c, const RowPassArgs& a, int kind, uint32_t nchunks) {
  if (c.ops && !c.force_generic) {
    ConstBankLease lease(c);
    return c.ops->rowpass(a, kind, nchunks, c.stream);
  }
  return launch_rowpass_generic(a, kind, nchunks, c.stream);
}

void update_factor_mode(Ctx& c, int mode, int reg, double lambda, bool fuse_resid) {
  if (mode == 0) note_sweep(c);
  RowPassArgs a = row_args(c, mode);
  const int J = c.ranks[mode];
  a.reg = reg;
  a.lambda = lambda;
  a.stride_na = J * (J + 1) / 2 + J;
  ensure(c, &c.d_heavy_part, &c.heavy_part_cap, (size_t)c.modes[mode].nslots * a.stride_na + 1);
  a.heavy_out = c.d_heavy_part;
  // the last mode's update can emit the residual of the updated model for the
  // core sweep (rank-specialised kernels only; see fused_residual)
  const bool fuse = fuse_resid && mode == c.N - 1 && c.ops && !c.force_generic;
  a.fuse_resid = fuse ? 1 : 0;
  a.r_out = c.d_r;
  const ModeData& mdd = c.modes[mode];
  const uint64_t p0 = mdd.h_offsets[c.row_lo[mode]], p1 = mdd.h_offsets[c.row_hi[mode]];
  if (sparse_delta_enabled(c)) {
    // mask-specialised contraction (vest_sparse.cu), then the statistics,
    // solves and fused residual from the materialised delta
    const bool fuse_d = fuse_resid && mode == c.N - 1;
    a.fuse_resid = fuse_d ? 1 : 0;
    if (!fuse_d && sparse_fused_enabled(c)) {
      // contraction, statistics and solves in one kernel (no delta in HBM)
      ProfScope ps(c, kProfFactor);
      sparse_fused(c, mode, a);
      if (reg == 1) l1_empty_rows(c, mode, lambda);
    } else {
      ensure(c, &c.d_delta, &c.delta_cap, (size_t)J * (p1 - p0) + 1);
      ProfScope ps(c, fuse_d ? kProfFactorFused : kProfFactor);
      sparse_delta(c, mode, p0, p1 - p0, c.d_delta);
      check(launch_rowpass_delta(a, kStats, a.csf.nchunks, c.d_delta, p1 - p0, p0, c.stream, c.gather_f32 != 0),
            "factor update (delta)");
      if (reg == 1) l1_empty_rows(c, mode, lambda);
    }
    c.r_valid = false;
    c.r_pending[0] = c.r_pending[1] = -1;
    c.r_fresh = false;
    c.table_valid = false;
    if (fuse_d) {
      if (mdd.nheavy_chunks > 0) {
        RowPassArgs b = row_args(c, mode);
        b.csf.chunks = mdd.d_heavy_chunks;
        b.csf.nchunks = mdd.nheavy_chunks;
        b.csf.nheavy = 0;
        b.r_out = c.d_r;
        ensure(c, &c.d_chunk_sum, &c.chunk_sum_cap, mdd.nchunks + 1);
        b.chunk_out = c.d_chunk_sum;
        ProfScope ps(c, kProfResid);
        check(launch_rowpass_delta(b, kResid, b.csf.nchunks, c.d_delta, p1 - p0, p0, c.stream, c.gather_f32 != 0),
              "heavy-row residual");
      }
      c.r_fresh = true;
    }
    comm_allgather_rows(c, mode, c.d_factor[mode], (uint64_t)c.ld[mode]);
    return;
  }
  {
    ProfScope ps(c, fuse ? kProfFactorFused : kProfFactor);
    // short rows of skewed modes lane-per-row (the fused mode keeps them in
    // the chunk kernel, which also writes their residuals)
    const bool tiny = !fuse && c.ops && !c.force_generic && c.ops->rowtiny && mdd.ntiny > 0 && !tiny_rows_off();
    if (tiny) {
      RowPassArgs bg = a;
      bg.csf.chunks = mdd.d_chunks_big;
      bg.csf.nchunks = mdd.nchunks_big;
      check(run_rows(c, bg, kStats, bg.csf.nchunks), "factor update");
      ConstBankLease lease(c);
      check(c.ops->rowtiny(a, mdd.d_tiny, mdd.ntiny, c.stream), "factor update (short rows)");
    } else {
      check(run_rows(c, a, kStats, a.csf.nchunks), "factor update");
    }
    if (reg == 1) l1_empty_rows(c, mode, lambda);
  }
  c.r_valid = false;
  c.r_pending[0] = c.r_pending[1] = -1;
  c.r_fresh = false;
  c.table_valid = false;
  if (fuse) {
    const ModeData& md = c.modes[mode];
    if (md.nheavy_chunks > 0) {
      // heavy rows were solved by k_heavy: their residual needs a second pass
      RowPassArgs b = row_args(c, mode);
      b.csf.chunks = md.d_heavy_chunks;
      b.csf.nchunks = md.nheavy_chunks;
      b.r_out = c.d_r;
      ensure(c, &c.d_chunk_sum, &c.chunk_sum_cap, md.nchunks + 1);
      b.chunk_out = c.d_chunk_sum;
      ProfScope ps(c, kProfResid);
      check(run_rows(c, b, kResid, b.csf.nchunks), "heavy-row residual");
    }
    c.r_fresh = true;
  }
  comm_allgather_rows(c, mode, c.d_factor[mode], (uint64_t)c.ld[mode]);
}

void update_factor_rows(Ctx& c, int mode, const uint32_t* rows, uint32_t nrows, int reg, double lambda) {
  // work list restricted to the given rows (update_factor_row_*)
  const ModeData& md = c.modes[mode];
  std::vector<Chunk> chunks;
  std::vector<Heavy> heavy;
  std::vector<uint32_t> empty;
  uint32_t slot = 0;
  for (uint32_t q = 0; q < nrows; ++q) {
    const uint32_t i = rows[q];
    const uint64_t b = md.h_offsets[i], e = md.h_offsets[i + 1], len = e - b;
    if (len == 0) {
      empty.push_back(i);
      continue;
    }
    if (len <= kChunk) {
      chunks.push_back({i, (uint32_t)b, (uint32_t)e, kLight});
      continue;
    }
    const uint32_t nch = (uint32_t)((len + kChunk - 1) / kChunk);
    heavy.push_back({i, slot, nch, 0});
    for (uint32_t k = 0; k < nch; ++k)
      chunks.push_back({i, (uint32_t)(b + len * k / nch), (uint32_t)(b + len * (k + 1) / nch), slot + k});
    slot += nch;
  }
  RowPassArgs a = row_args(c, mode);
  const int J = c.ranks[mode];
  a.reg = reg;
  a.lambda = lambda;
  a.stride_na = J * (J + 1) / 2 + J;
  ensure(c, &c.d_heavy_part, &c.heavy_part_cap, (size_t)slot * a.stride_na + 1);
  a.heavy_out = c.d_heavy_part;
  Chunk* dch = nullptr;
  Heavy* dhv = nullptr;
  uint32_t* dem = nullptr;
  check(cudaMalloc(&dch, std::max<size_t>(1, chunks.size()) * sizeof(Chunk)), "tmp");
  check(cudaMalloc(&dhv, std::max<size_t>(1, heavy.size()) * sizeof(Heavy)), "tmp");
  check(cudaMalloc(&dem, std::max<size_t>(1, empty.size()) * 4), "tmp");
  if (!chunks.empty()) check(cudaMemcpy(dch, chunks.data(), chunks.size() * sizeof(Chunk), cudaMemcpyHostToDevice), "h2d");
  if (!heavy.empty()) check(cudaMemcpy(dhv, heavy.data(), heavy.size() * sizeof(Heavy), cudaMemcpyHostToDevice), "h2d");
  if (!empty.empty()) check(cudaMemcpy(dem, empty.data(), empty.size() * 4, cudaMemcpyHostToDevice), "h2d");
  a.csf.chunks = dch;
  a.csf.nchunks = (uint32_t)chunks.size();
  a.csf.heavy = dhv;
  a.csf.nheavy = (uint32_t)heavy.size();
  sync_const_core(c);
  check(run_rows(c, a, kStats, a.csf.nchunks), "row update");
  if (reg == 1 && !empty.empty()) {
    ModeData tmp;
    ModeData& m2 = c.modes[mode];
    std::swap(tmp.d_empty, m2.d_empty);
    std::swap(tmp.nempty, m2.nempty);
    m2.d_empty = dem;
    m2.nempty = (uint32_t)empty.size();
    l1_empty_rows(c, mode, lambda);
    m2.d_empty = tmp.d_empty;
    m2.nempty = tmp.nempty;
  }
  check(cudaStreamSynchronize(c.stream), "row sync");
  cudaFree(dch);
  cudaFree(dhv);
  cudaFree(dem);
  c.r_valid = false;
  c.r_pending[0] = c.r_pending[1] = -1;
    c.r_fresh = false;
  c.table_valid = false;
}

bool core_apply_pending(Ctx& c);

void compute_residual(Ctx& c) {
  if (core_apply_pending(c)) return;  // r lacks only the last core block's update
  const int m = c.N - 1;
  RowPassArgs a = row_args(c, m);
  ensure(c, &c.d_chunk_sum, &c.chunk_sum_cap, c.modes[m].nchunks + 1);
  a.r_out = c.d_r;
  a.chunk_out = c.d_chunk_sum;
  sync_const_core(c);
  {
    ProfScope ps(c, kProfResid);
    check(run_rows(c, a, kResid, a.csf.nchunks), "residual");
  }
  c.sum_sq = reduce_chunk_sums(c, c.d_chunk_sum, c.modes[m].nchunks);
  c.re = std::sqrt(c.sum_sq) / c.x_norm;
  c.r_valid = true;
  c.r_fresh = true;
}

void responsibilities(Ctx& c) {
  if (!c.r_valid) compute_residual(c);
  ProfScope ps(c, kProfResp);
  core_responsibilities(c);
  const double re = c.re, re2 = re * re, x2 = c.x_norm * c.x_norm;
  for (int n = 0; n < c.N; ++n) {
    if (re == 0.0) {
      fill_factor_resp(c, n, INFINITY);
      continue;
    }
    // rows without entries: acc = 0 -> err2 = re^2 (pruning.hpp:170-175)
    double err2 = re2;
    fill_factor_resp(c, n, (std::sqrt(err2) - re) / re);
    RowPassArgs a = row_args(c, n);
    a.re = re;
    a.re2 = re2;
    a.x2 = x2;
    a.resp_out = c.d_resp_f[n];
    a.stride_na = c.ranks[n];
    ensure(c, &c.d_heavy_part, &c.heavy_part_cap, (size_t)c.modes[n].nslots * a.stride_na + 1);
    a.heavy_out = c.d_heavy_part;
    check(run_rows(c, a, kResp, a.csf.nchunks), "factor resp");
    comm_allgather_rows(c, n, c.d_resp_f[n], (uint64_t)c.ranks[n]);
  }
  check(cudaStreamSynchronize(c.stream), "resp sync");
  c.table_valid = true;
  c.table_re = re;
}

}  // namespace vest

// ===================================================================== C-ABI
using namespace vest;

struct vest_ctx {
  Ctx c;
};

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    g_err.clear();
    return VEST_OK;
  } catch (const ArgError& e) {
    g_err = e.msg;
    return VEST_EINVAL;
  } catch (const RtError& e) {
    g_err = e.msg;
    return VEST_ERUNTIME;
  } catch (const CudaError& e) {
    g_err = std::string("CUDA error in ") + e.where + ": " + cudaGetErrorString(e.err);
    return VEST_ECUDA;
  } catch (const std::bad_alloc&) {
    g_err = "host allocation failed";
    return VEST_ERUNTIME;
  } catch (const std::exception& e) {  // e.g. std::system_error from a host thread
    g_err = e.what();
    return VEST_ERUNTIME;
  }
}

void set_dev(const Ctx& c) { check(cudaSetDevice(c.device), "cudaSetDevice"); }

// packed [rows][J] <-> strided [rows][ld] on the device (ld = J rounded up to
// even): host transfers stay single contiguous DMAs
__global__ void k_restride(const double* src, int sld, double* dst, int dld, int J, uint64_t rows) {
  const uint64_t n = rows * (uint64_t)J;
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < n; t += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t r = t / J;
    const int j = (int)(t - r * J);
    dst[r * dld + j] = src[r * sld + j];
  }
}

void copy_factor_h2d(Ctx& c, int n, const double* host) {
  const int J = c.ranks[n];
  const size_t bytes = c.dims[n] * J * sizeof(double);
  if (c.ld[n] == J) {
    check(cudaMemcpyAsync(c.d_factor[n], host, bytes, cudaMemcpyHostToDevice, c.stream), "factor");
    return;
  }
  ensure(c, &c.d_xfer, &c.xfer_cap, c.dims[n] * J);
  check(cudaMemcpyAsync(c.d_xfer, host, bytes, cudaMemcpyHostToDevice, c.stream), "factor");
  k_restride<<<592, 256, 0, c.stream>>>(c.d_xfer, J, c.d_factor[n], c.ld[n], J, c.dims[n]);
  count_launch();
  check(cudaGetLastError(), "factor restride");
}

void copy_factor_d2h(Ctx& c, int n, double* host) {
  const int J = c.ranks[n];
  const size_t bytes = c.dims[n] * J * sizeof(double);
  if (c.ld[n] == J) {
    check(cudaMemcpyAsync(host, c.d_factor[n], bytes, cudaMemcpyDeviceToHost, c.stream), "factor");
    return;
  }
  ensure(c, &c.d_xfer, &c.xfer_cap, c.dims[n] * J);
  k_restride<<<592, 256, 0, c.stream>>>(c.d_factor[n], c.ld[n], c.d_xfer, J, J, c.dims[n]);
  count_launch();
  check(cudaGetLastError(), "factor restride");
  check(cudaMemcpyAsync(host, c.d_xfer, bytes, cudaMemcpyDeviceToHost, c.stream), "factor");
  // (the staging buffer is reused by the next factor: keep the copies ordered)
  check(cudaStreamSynchronize(c.stream), "factor d2h");
}

void upload_model(Ctx& c, const double* core, const uint8_t* core_mask, const double* const* factors,
                  const uint8_t* const* fmasks) {
  sync_const_core(c);  // the core changes: the constant-bank copy is stale
  if (core) check(cudaMemcpyAsync(c.d_core, core, c.G * sizeof(double), cudaMemcpyHostToDevice, c.stream), "core");
  if (core_mask) {
    check(cudaMemcpyAsync(c.d_core_mask, core_mask, c.G, cudaMemcpyHostToDevice, c.stream), "core mask");
    std::memcpy(c.h_core_mask.data(), core_mask, c.G);
  }
  for (int n = 0; n < c.N; ++n) {
    const int J = c.ranks[n];
    if (factors && factors[n]) {
      copy_factor_h2d(c, n, factors[n]);
      if (c.ld[n] != J) check(cudaStreamSynchronize(c.stream), "factor h2d");  // staging reuse
    }
    if (fmasks && fmasks[n])
      check(cudaMemcpyAsync(c.d_fmask[n], fmasks[n], c.dims[n] * J, cudaMemcpyHostToDevice, c.stream), "fmask");
  }
  check(cudaStreamSynchronize(c.stream), "set_model");
  c.r_valid = false;
  c.r_pending[0] = c.r_pending[1] = -1;
    c.r_fresh = false;
  c.table_valid = false;
}

__global__ void k_scatter_r(const double* r, const uint32_t* eid, uint64_t p0, uint64_t n, double* out) {
  for (uint64_t p = p0 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < p0 + n; p += (uint64_t)gridDim.x * blockDim.x)
    out[eid[p]] = r[p];
}

__global__ void k_delta_one(DevModel m, const uint32_t* at, int mode, double* out) {
  // compute_delta (updates.hpp:35-52), reference cell order
  if (threadIdx.x != 0) return;
  const int J = m.J[mode];
  for (int j = 0; j < J; ++j) out[j] = 0.0;
  for (int lin = 0; lin < m.G; ++lin) {
    const double g = m.core[lin];
    if (g == 0.0) continue;
    const uint32_t b = m.cellbeta[lin];
    double p = g;  // __dmul_rn/__dadd_rn: no FMA contraction, reference rounding
    for (int k = 0; k < m.N; ++k)
      if (k != mode) p = __dmul_rn(p, m.factor[k][(size_t)at[k] * m.ld[k] + ((b >> (4 * k)) & 15u)]);
    out[(b >> (4 * mode)) & 15u] = __dadd_rn(out[(b >> (4 * mode)) & 15u], p);
  }
}

__global__ void k_partial_recon(DevModel m, const uint32_t* coords, uint64_t nq, int mode, uint32_t j, double* out) {
  // partial_reconstruct (tucker_model.hpp:136-154): cells with beta_mode == j
  // in row-major order, zeros skipped, p = g * a_0 * ... * a_{N-1}
  for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < nq; q += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t* at = coords + q * m.N;
    double acc = 0.0;
    for (int lin = 0; lin < m.G; ++lin) {
      const uint32_t b = m.cellbeta[lin];
      if (((b >> (4 * mode)) & 15u) != j) continue;
      const double g = m.core[lin];
      if (g == 0.0) continue;
      double p = g;
      for (int k = 0; k < m.N; ++k) p = __dmul_rn(p, m.factor[k][(size_t)at[k] * m.ld[k] + ((b >> (4 * k)) & 15u)]);
      acc = __dadd_rn(acc, p);
    }
    out[q] = acc;
  }
}

__global__ void k_row_stats_ref(DevModel m, DevCSF csf, int mode, uint32_t row, uint64_t p0, uint64_t p1,
                                double* gram, double* xdelta, double* last_delta) {
  // compute_row_stats (updates.hpp:64-79): one block; thread j < J forms
  // delta_j of each entry (compute_delta's cell order for that j), thread
  // (t, j) accumulates gram[t*J+j] serially over the slice in ascending entry
  // id, thread t also xdelta[t]; reference rounding (no contraction)
  __shared__ double dsh[VEST_MAXJ];
  __shared__ double xv_sh;
  const int J = m.J[mode], tid = threadIdx.x;
  const int t = tid / J, jj = tid % J;
  double g_acc = 0.0, x_acc = 0.0;
  if (tid < J) dsh[tid] = 0.0;
  __syncthreads();
  for (uint64_t p = p0; p < p1; ++p) {
    if (tid < J) {
      double d = 0.0;
      for (int lin = 0; lin < m.G; ++lin) {
        const uint32_t b = m.cellbeta[lin];
        if ((int)((b >> (4 * mode)) & 15u) != tid) continue;
        const double g = m.core[lin];
        if (g == 0.0) continue;
        double pr = g;
        for (int k = 0; k < m.N; ++k) {
          if (k == mode) continue;
          const uint32_t ik = csf.oc[k][p];
          pr = __dmul_rn(pr, m.factor[k][(size_t)ik * m.ld[k] + ((b >> (4 * k)) & 15u)]);
        }
        d = __dadd_rn(d, pr);
      }
      dsh[tid] = d;
    }
    if (tid == 0) xv_sh = csf.val[p];
    __syncthreads();
    if (tid < J * J) {
      const double dt = dsh[t];
      if (dt != 0.0) {
        if (jj == 0) x_acc = __dadd_rn(x_acc, __dmul_rn(xv_sh, dt));
        g_acc = __dadd_rn(g_acc, __dmul_rn(dt, dsh[jj]));
      }
    }
    __syncthreads();
  }
  if (tid < J * J) gram[tid] = g_acc;
  if (tid < J * J && jj == 0) xdelta[t] = x_acc;
  if (tid < J) last_delta[tid] = dsh[tid];
}

int coo_recon(Ctx& c, const uint32_t* coords, const double* values, uint64_t n, double* out, double* sums) {
  for (uint64_t q = 0; q < n; ++q)
    for (int k = 0; k < c.N; ++k)
      if (coords[q * c.N + k] >= c.dims[k]) throw ArgError{"query coordinate out of bounds"};
  uint32_t* dc = nullptr;
  double *dv = nullptr, *dout = nullptr, *dpart = nullptr;
  const int nblocks = 592;
  check(cudaMalloc(&dc, std::max<uint64_t>(n, 1) * c.N * 4), "coo");
  check(cudaMalloc(&dpart, 2 * nblocks * sizeof(double)), "coo");
  if (values) check(cudaMalloc(&dv, std::max<uint64_t>(n, 1) * 8), "coo");
  else check(cudaMalloc(&dout, std::max<uint64_t>(n, 1) * 8), "coo");
  if (n) {
    check(cudaMemcpyAsync(dc, coords, n * c.N * 4, cudaMemcpyHostToDevice, c.stream), "coo h2d");
    if (values) check(cudaMemcpyAsync(dv, values, n * 8, cudaMemcpyHostToDevice, c.stream), "coo h2d");
    const DevModel m = c.model_view();
    if (c.ops && !c.force_generic) {
      ConstBankLease lease(c);
      check(c.ops->coo_recon(m, dc, dv, n, dout, dpart, nblocks, c.stream), "coo recon");
    } else {
      check(launch_coo_recon_generic(m, dc, dv, n, dout, dpart, nblocks, c.stream), "coo recon");
    }
    if (values) {
      std::vector<double> part(2 * nblocks);
      check(cudaMemcpyAsync(part.data(), dpart, part.size() * 8, cudaMemcpyDeviceToHost, c.stream), "d2h");
      check(cudaStreamSynchronize(c.stream), "coo sync");
      double a = 0, b = 0;
      for (int i = 0; i < nblocks; ++i) a += part[2 * i], b += part[2 * i + 1];
      sums[0] = a;
      sums[1] = b;
    } else {
      check(cudaMemcpyAsync(out, dout, n * 8, cudaMemcpyDeviceToHost, c.stream), "d2h");
    }
  }
  check(cudaStreamSynchronize(c.stream), "coo sync");
  cudaFree(dc);
  cudaFree(dv);
  cudaFree(dout);
  cudaFree(dpart);
  return 0;
}

}  // namespace

extern "C" {

const char* vest_last_error(void) { return g_err.c_str(); }
const char* vest_version(void) { return "vest-b200 0.1 (sm_100a)"; }
uint64_t vest_launch_count(void) { return launch_counter(); }

static int create_impl(int order, const uint64_t* dims, uint64_t nnz, const uint32_t* coords, const double* values,
                       const uint64_t* ranks, int device, const uint64_t* row_lo, const uint64_t* row_hi,
                       vest_ctx** out);

int vest_ctx_create(int order, const uint64_t* dims, uint64_t nnz, const uint32_t* coords, const double* values,
                    const uint64_t* ranks, int device, vest_ctx** out) {
  return create_impl(order, dims, nnz, coords, values, ranks, device, nullptr, nullptr, out);
}

int vest_ctx_create_shard(int order, const uint64_t* dims, uint64_t nnz, const uint32_t* coords,
                          const double* values, const uint64_t* ranks, int device, const uint64_t* row_lo,
                          const uint64_t* row_hi, vest_ctx** out) {
  return create_impl(order, dims, nnz, coords, values, ranks, device, row_lo, row_hi, out);
}

int vest_ctx_set_comm(vest_ctx* h, const vest_comm* comm) {
  Ctx& c = h->c;
  if (c.comm_free) {
    c.comm_free(c.comm.user);
    c.comm_free = nullptr;
  }
  c.comm = CommHooks{};
  c.comm_capturable = false;  // host callbacks block: never inside a graph
  if (comm) {
    c.comm.user = comm->user;
    c.comm.allreduce_sum = comm->allreduce_sum;
    c.comm.allgather_rows = comm->allgather_rows;
  }
  return VEST_OK;
}

uint64_t vest_ctx_local_nnz(vest_ctx* h, int mode) {
  return (mode >= 0 && mode < h->c.N) ? h->c.local_nnz[mode] : 0;
}

static int create_impl(int order, const uint64_t* dims, uint64_t nnz, const uint32_t* coords, const double* values,
                       const uint64_t* ranks, int device, const uint64_t* row_lo, const uint64_t* row_hi,
                       vest_ctx** out) {
  *out = nullptr;
  auto* h = new vest_ctx();
  Ctx& c = h->c;
  if (const char* e = getenv("VEST_GATHER_F32")) c.gather_f32 = e[0] == '1';  // A/B default
  const int rc = guard([&] {
    if (order <= 0) throw ArgError{"tensor order must be at least 1"};
    if (order > VEST_MAXN) throw ArgError{"tensor order exceeds the device kernels' limit (8)"};
    for (int k = 0; k < order; ++k)
      if (dims[k] == 0) throw ArgError{"tensor dimensions must be positive"};
    for (int k = 0; k < order; ++k) {
      if (ranks[k] == 0) throw ArgError{"dims and ranks must be positive"};
      if (ranks[k] > VEST_MAXJ) throw ArgError{"rank exceeds the device kernels' limit (16)"};
      if (dims[k] > 0xFFFFFFFFull) throw ArgError{"dimension exceeds the uint32 coordinate range"};
    }
    if (nnz >= 0xFFFFFFFFull) throw ArgError{"nnz exceeds the uint32 entry-id range"};
    c.device = device;
    c.N = order;
    c.nnz = nnz;
    c.G = 1;
    for (int k = 0; k < order; ++k) {
      c.row_lo[k] = row_lo ? row_lo[k] : 0;
      c.row_hi[k] = row_hi ? row_hi[k] : dims[k];
      if (c.row_lo[k] > c.row_hi[k] || c.row_hi[k] > dims[k]) throw ArgError{"shard row range out of bounds"};
      c.dims[k] = dims[k];
      c.ranks[k] = (int)ranks[k];
      c.G *= (int)ranks[k];
      c.ld[k] = ((int)ranks[k] + 1) & ~1;
    }
    set_dev(c);
    check(cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking), "stream");
    // frobenius_norm (sparse_tensor.hpp:45-49): serial, entry order
    double acc = 0.0;
    for (uint64_t e = 0; e < nnz; ++e) acc += values[e] * values[e];
    c.x_norm = std::sqrt(acc);
    for (int n = 0; n < order; ++n) {
      c.d_factor[n] = static_cast<double*>(dalloc(c, c.dims[n] * c.ld[n] * sizeof(double)));
      c.d_fmask[n] = static_cast<uint8_t*>(dalloc(c, c.dims[n] * c.ranks[n]));
      c.d_resp_f[n] = static_cast<double*>(dalloc(c, c.dims[n] * c.ranks[n] * sizeof(double)));
      check(cudaMemsetAsync(c.d_factor[n], 0, c.dims[n] * c.ld[n] * sizeof(double), c.stream), "zero");
      check(cudaMemsetAsync(c.d_fmask[n], 0, c.dims[n] * c.ranks[n], c.stream), "zero");
    }
    c.d_core = static_cast<double*>(dalloc(c, c.G * sizeof(double)));
    c.d_core_mask = static_cast<uint8_t*>(dalloc(c, c.G));
    c.d_resp_core = static_cast<double*>(dalloc(c, c.G * sizeof(double)));
    c.d_cellbeta = static_cast<uint32_t*>(dalloc(c, c.G * sizeof(uint32_t)));
    check(cudaMemsetAsync(c.d_core, 0, c.G * sizeof(double), c.stream), "zero");
    check(cudaMemsetAsync(c.d_core_mask, 0, c.G, c.stream), "zero");
    c.h_core_mask.assign(c.G, 0);
    c.d_counts = static_cast<unsigned long long*>(dalloc(c, 4096 * sizeof(unsigned long long)));
    c.d_sel = dalloc(c, 4096);
    c.d_small = static_cast<double*>(dalloc(c, 64));
    check(cudaMallocHost(&c.h_small, 64), "pinned");
    const DevModel mv = c.model_view();
    k_cellbeta<<<(c.G + 255) / 256, 256, 0, c.stream>>>(c.d_cellbeta, c.G, c.N, mv);
    count_launch();
    build_csf(c, coords, values);
    {  // residual, CSF order of the last mode: this context's positions only
      const ModeData& ml = c.modes[c.N - 1];
      c.d_r = static_cast<double*>(dalloc(c, std::max<uint64_t>(c.local_nnz[c.N - 1], 1) * sizeof(double))) - ml.pos0;
    }
    c.ops = find_shape_ops(c.N, c.ranks);
    if (c.ops && c.G > VEST_CONST_CORE_MAX) c.ops = nullptr;
    check(cudaStreamSynchronize(c.stream), "create");
  });
  if (rc != VEST_OK) {
    vest_ctx_destroy(h);
    return rc;
  }
  *out = h;
  return VEST_OK;
}

int vest_nccl_unique_id(void* id_out) {
  return guard([&] { nccl_unique_id(id_out); });
}

int vest_ctx_set_nccl(vest_ctx* h, int rank, int world, const void* id, const uint64_t* bounds) {
  Ctx& c = h->c;
  return guard([&] {
    set_dev(c);
    ctx_set_nccl(c, rank, world, id, bounds);
  });
}

int vest_ctx_destroy(vest_ctx* h) {
  if (!h) return VEST_OK;
  Ctx& c = h->c;
  cudaSetDevice(c.device);
  if (c.stream) cudaStreamSynchronize(c.stream);
  const_bank_forget(c);  // a later context at this address must reload the bank
  if (c.comm_free) {
    c.comm_free(c.comm.user);
    c.comm_free = nullptr;
  }
  for (int n = 0; n < VEST_MAXN; ++n) {
    ModeData& md = c.modes[n];
    cudaFree(md.d_offsets);
    for (int k = 0; k < VEST_MAXN; ++k)
      if (md.d_oc[k]) cudaFree(md.d_oc[k] + md.pos0);
    if (md.d_val) cudaFree(md.d_val + md.pos0);
    if (md.d_eid) cudaFree(md.d_eid + md.pos0);
    cudaFree(md.d_chunks);
    cudaFree(md.d_heavy);
    cudaFree(md.d_empty);
    cudaFree(md.d_heavy_chunks);
    cudaFree(c.d_factor[n]);
    cudaFree(c.d_fmask[n]);
    cudaFree(c.d_resp_f[n]);
  }
  cudaFree(c.d_factor32[0]);  // one buffer for every mode's shadow
  cudaFree(c.d_core);
  cudaFree(c.d_core_mask);
  cudaFree(c.d_cellbeta);
  if (c.d_r) cudaFree(c.d_r + c.modes[c.N > 0 ? c.N - 1 : 0].pos0);
  cudaFree(c.d_resp_core);
  cudaFree(c.d_heavy_part);
  cudaFree(c.d_chunk_stats);
  cudaFree(c.d_gemm_part);
  cudaFree(c.d_gemm_out);
  cudaFree(c.d_chunk_sum);
  cudaFree(c.d_small);
  cudaFree(c.d_fibers);
  cudaFree(c.d_dg);
  if (c.graph_exec) cudaGraphExecDestroy(c.graph_exec);
  cudaFree(c.d_delta);
  cudaFree(c.d_hstab);
  sparse_free(c);
  core_gen_free(c);
  cudaFree(c.d_pack_u);
  cudaFree(c.d_pack_w);
  cudaFree(c.d_counter);
  cudaFree(c.d_xfer);
  cudaFree(c.d_counts);
  cudaFree(c.d_sel);
  if (c.h_small) cudaFreeHost(c.h_small);
  if (c.stream) cudaStreamDestroy(c.stream);
  if (c.copy_stream) cudaStreamDestroy(c.copy_stream);
  for (auto& e : c.ev_copy)
    if (e) cudaEventDestroy(e);
  delete h;
  return VEST_OK;
}

void* vest_ctx_stream(vest_ctx* h) { return h ? (void*)h->c.stream : nullptr; }
uint64_t vest_ctx_device_bytes(const vest_ctx* h) { return h ? h->c.device_bytes : 0; }
int vest_ctx_specialised(const vest_ctx* h) { return h && h->c.ops && !h->c.force_generic ? 1 : 0; }
int vest_ctx_force_generic(vest_ctx* h, int on) {
  h->c.force_generic = on != 0;
  return VEST_OK;
}
int vest_ctx_set_core_block(vest_ctx* h, int fibers) {
  h->c.core_block = fibers;
  return VEST_OK;
}
int vest_ctx_set_sparse_delta(vest_ctx* h, int mode) {
  h->c.sparse_delta = mode < 0 ? -1 : (mode ? 1 : 0);
  return VEST_OK;
}
int vest_ctx_set_sparse_fused(vest_ctx* h, int mode) {
  if (!h) return VEST_EINVAL;
  h->c.sparse_fused = mode < 0 ? -1 : (mode ? 1 : 0);
  return VEST_OK;
}

int vest_ctx_set_gather_f32(vest_ctx* h, int on) {
  if (!h) return VEST_EINVAL;
  h->c.gather_f32 = on ? 1 : 0;
  return VEST_OK;
}

int vest_ctx_set_core_gen(vest_ctx* h, int mode) {
  h->c.core_gen_mode = mode < 0 ? -1 : (mode ? 1 : 0);
  return VEST_OK;
}
int vest_ctx_sparse_delta_active(const vest_ctx* h) { return h && sparse_delta_eligible(h->c) ? 1 : 0; }
int vest_sparse_compile_check(int order, const uint64_t* ranks, const uint8_t* core_mask, uint64_t* cubin_bytes) {
  return guard([&] {
    if (order < 2 || order > VEST_MAXN) throw ArgError{"order must be in [2, 8]"};
    int r[VEST_MAXN];
    for (int k = 0; k < order; ++k) r[k] = (int)ranks[k];
    std::string err;
    if (sparse_compile_check(order, r, core_mask, cubin_bytes, &err)) throw RtError{err};
  });
}

int vest_init_random(vest_ctx* h, uint64_t seed) {
  Ctx& c = h->c;
  return guard([&] {
    sync_const_core(c);  // the core changes here: the constant-bank copy is stale
    // init_random (tucker_model.hpp:88-108): same engine, distribution and
    // draw order, so the host-side model is identical to the reference's.
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> unif(0.0, 1.0);
    std::vector<std::vector<double>> f(c.N);
    std::vector<const double*> fp(c.N);
    std::vector<std::vector<uint8_t>> m(c.N);
    std::vector<const uint8_t*> mp(c.N);
    for (int n = 0; n < c.N; ++n) {
      f[n].resize(c.dims[n] * c.ranks[n]);
      for (double& v : f[n]) v = unif(rng);
      fp[n] = f[n].data();
      m[n].assign(c.dims[n] * c.ranks[n], 0);
      mp[n] = m[n].data();
    }
    std::vector<double> core(c.G);
    for (double& v : core) v = unif(rng);
    std::vector<uint8_t> cm(c.G, 0);
    set_dev(c);
    upload_model(c, core.data(), cm.data(), fp.data(), mp.data());
  });
}

int vest_set_model(vest_ctx* h, const double* core, const uint8_t* core_mask, const double* const* factors,
                   const uint8_t* const* factor_masks) {
  Ctx& c = h->c;
  return guard([&] {
    set_dev(c);
    upload_model(c, core, core_mask, factors, factor_masks);
  });
}

int vest_get_model(vest_ctx* h, double* core, uint8_t* core_mask, double* const* factors,
                   uint8_t* const* factor_masks) {
  Ctx& c = h->c;
  return guard([&] {
    set_dev(c);
    if (core) check(cudaMemcpyAsync(core, c.d_core, c.G * sizeof(double), cudaMemcpyDeviceToHost, c.stream), "core");
    if (core_mask) check(cudaMemcpyAsync(core_mask, c.d_core_mask, c.G, cudaMemcpyDeviceToHost, c.stream), "mask");
    for (int n = 0; n < c.N; ++n) {
      const int J = c.ranks[n];
      if (factors && factors[n]) copy_factor_d2h(c, n, factors[n]);
      if (factor_masks && factor_masks[n])
        check(cudaMemcpyAsync(factor_masks[n], c.d_fmask[n], c.dims[n] * J, cudaMemcpyDeviceToHost, c.stream),
              "fmask");
    }
    check(cudaStreamSynchronize(c.stream), "get_model");
  });
}

static void check_reg(int reg) {
  if (reg != VEST_LF && reg != VEST_L1) throw ArgError{"unknown regularizer"};
}

int vest_update_all_factors(vest_ctx* h, int reg, double lambda) {
  Ctx& c = h->c;
  return guard([&] {
    check_reg(reg);
    set_dev(c);
    sync_const_core(c);
    for (int n = 0; n < c.N; ++n) update_factor_mode(c, n, reg, lambda, false);
    check(cudaStreamSynchronize(c.stream), "factors");
  });
}

int vest_update_factor_mode(vest_ctx* h, int mode, int reg, double lambda) {
  Ctx& c = h->c;
  return guard([&] {
    check_reg(reg);
    if (mode < 0 || mode >= c.N) throw ArgError{"mode out of range"};
    set_dev(c);
    sync_const_core(c);
    update_factor_mode(c, mode, reg, lambda, false);
    check(cudaStreamSynchronize(c.stream), "factor mode");
  });
}

int vest_update_factor_row(vest_ctx* h, int reg, int mode, uint64_t row, double lambda) {
  Ctx& c = h->c;
  return guard([&] {
    check_reg(reg);
    if (mode < 0 || mode >= c.N || row >= c.dims[mode]) throw ArgError{"row out of range"};
    if (row < c.row_lo[mode] || row >= c.row_hi[mode]) throw ArgError{"row not owned by this shard context"};
    set_dev(c);
    const uint32_t r = (uint32_t)row;
    update_factor_rows(c, mode, &r, 1, reg, lambda);
  });
}

int vest_update_core(vest_ctx* h, int reg, double lambda) {
  Ctx& c = h->c;
  return guard([&] {
    check_reg(reg);
    set_dev(c);
    core_sweep(c, reg, lambda);
    c.table_valid = false;
    check(cudaStreamSynchronize(c.stream), "core");
  });
}

int vest_compute_residuals(vest_ctx* h, double* r_out, double* sum_sq, double* x_norm, double* re) {
  Ctx& c = h->c;
  return guard([&] {
    if (c.x_norm == 0.0) throw ArgError{"zero-norm tensor"};
    set_dev(c);
    if (!c.r_valid) compute_residual(c);
    if (r_out && c.nnz) {
      double* tmp = nullptr;
      check(cudaMalloc(&tmp, c.nnz * sizeof(double)), "r tmp");
      const ModeData& md = c.modes[c.N - 1];
      // a shard holds the residuals of its own last-mode rows; the rest are 0
      check(cudaMemsetAsync(tmp, 0, c.nnz * sizeof(double), c.stream), "r tmp");
      k_scatter_r<<<592, 256, 0, c.stream>>>(c.d_r, md.d_eid, md.pos0, c.local_nnz[c.N - 1], tmp);
      count_launch();
      check(cudaMemcpyAsync(r_out, tmp, c.nnz * sizeof(double), cudaMemcpyDeviceToHost, c.stream), "r d2h");
      check(cudaStreamSynchronize(c.stream), "r sync");
      cudaFree(tmp);
    }
    if (sum_sq) *sum_sq = c.sum_sq;
    if (x_norm) *x_norm = c.x_norm;
    if (re) *re = c.re;
  });
}

// ------------------------------------------------------- iteration graphs --
// One CD iteration of the 3-mode all-prefix path is ~20 launches with no host
// synchronisation except the final sum read-back, and its host logic depends
// only on (core mask, regulariser, lambda, kernel choice).  Once the same key
// has run twice, the iteration is captured into a CUDA graph (relaxed capture
// mode; the read-back is a captured D2H copy into pinned memory) and replayed:
// one launch per iteration instead of ~20 (config 1 is launch-bound).  Same
// kernels in the same order: bit-identical to the stream path.
// VEST_GRAPH=0 disables it.
static bool graph_off() {
  static const bool v = [] {
    const char* e = getenv("VEST_GRAPH");
    return e && e[0] == '0';
  }();
  return v;
}

static bool graph_eligible(const Ctx& c) {
  const bool hooks_ok = (!c.comm.allreduce_sum && !c.comm.allgather_rows) || c.comm_capturable;
  return !graph_off() && !c.prof_on && hooks_ok && core_sweep_capturable(c) && c.mask_sweeps >= 3;
}

static uint64_t graph_key_of(const Ctx& c, int reg, double lambda) {
  uint64_t h = core_mask_hash(c) ^ 0x9E3779B97F4A7C15ull;
  auto mix = [&](uint64_t v) {
    h ^= v + 0x9E3779B97F4A7C15ull + (h << 6) + (h >> 2);
  };
  uint64_t lb;
  std::memcpy(&lb, &lambda, 8);
  mix((uint64_t)reg);
  mix(lb);
  mix(sparse_delta_enabled(c) ? 1 : 0);
  mix(c.alloc_epoch);  // any (re)allocation since the capture invalidates the graph
  return h;
}

static void graph_free(Ctx& c) {
  if (c.graph_exec) cudaGraphExecDestroy(c.graph_exec);
  c.graph_exec = nullptr;
  c.graph_key = 0;
}

static void iteration_body(Ctx& c, int reg, double lambda) {
  sync_const_core(c);
  for (int n = 0; n < c.N; ++n) update_factor_mode(c, n, reg, lambda, true);
  core_sweep(c, reg, lambda);
  c.table_valid = false;
}

// replay the captured iteration and restore the host state it leaves
static void graph_replay(Ctx& c) {
  {
    ConstBankLease lease(c, true);
    check(cudaGraphLaunch(c.graph_exec, c.stream), "graph launch");
  }
  launch_counter() += c.graph_launches;
  note_sweep(c);
  check(cudaStreamSynchronize(c.stream), "graph sync");
  c.table_valid = false;
  if (c.graph_general && !c.graph_pending_general) {  // a general sweep that ended with r current
    c.r_valid = true;
    c.r_fresh = true;
    c.r_pending[0] = c.r_pending[1] = -1;
    c.sum_sq = c.h_small[0];
    c.re = std::sqrt(c.sum_sq) / c.x_norm;
    return;
  }
  // r lacks the sweep's last block (3-mode group or general block): the sums
  // read back are [s', s] of the quadratic form
  c.r_valid = false;
  c.r_fresh = false;
  c.r_pending[0] = c.graph_pending[0];
  c.r_pending[1] = c.graph_pending[1];
  c.r_pending_ops = c.graph_pending_ops;
  c.r_pending_general = c.graph_pending_general;
  sum_from_quadratic_form(c);
}

int vest_cd_iteration(vest_ctx* h, int reg, double lambda, double* re) {
  Ctx& c = h->c;
  return guard([&] {
    check_reg(reg);
    if (c.x_norm == 0.0) throw ArgError{"zero-norm tensor"};
    set_dev(c);
    if (graph_eligible(c)) {
      const uint64_t key = graph_key_of(c, reg, lambda);
      if (c.graph_exec && c.graph_key == key) {
        graph_replay(c);
        if (re) *re = c.re;
        return;
      }
      if (c.graph_seen_key == key && c.graph_seen >= 1) {
        graph_free(c);
        const uint64_t l0 = launch_counter();
        check(cudaStreamBeginCapture(c.stream, cudaStreamCaptureModeRelaxed), "begin capture");
        c.capturing = true;
        try {
          iteration_body(c, reg, lambda);
        } catch (...) {
          cudaGraph_t g = nullptr;
          cudaStreamEndCapture(c.stream, &g);
          if (g) cudaGraphDestroy(g);
          c.capturing = false;
          const_bank_forget(c);
          throw;
        }
        c.capturing = false;
        cudaGraph_t g = nullptr;
        const_bank_forget(c);
        check(cudaStreamEndCapture(c.stream, &g), "end capture");
        const cudaError_t ie = cudaGraphInstantiate(&c.graph_exec, g, 0);
        cudaGraphDestroy(g);
        check(ie, "graph instantiate");
        c.graph_key = key;
        c.graph_launches = launch_counter() - l0;
        launch_counter() = l0;  // counted when replayed
        c.graph_general = core_sweep_general(c);
        c.graph_pending_general = c.r_pending_general && c.r_pending[0] >= 0;
        c.graph_pending[0] = c.r_pending[0];
        c.graph_pending[1] = c.r_pending[1];
        c.graph_pending_ops = c.r_pending_ops;
        c.mask_sweeps -= 1;  // the capture ran no sweep; the replay counts it
        graph_replay(c);
        if (re) *re = c.re;
        return;
      }
      c.graph_seen_key = key;
      c.graph_seen = 1;
    }
    iteration_body(c, reg, lambda);
    if (re) *re = c.re;
  });
}

int vest_cd_iteration_host(vest_ctx* h, double* core, const uint8_t* core_mask, double* const* factors,
                           const uint8_t* const* factor_masks, int reg, double lambda, double* re) {
  Ctx& c = h->c;
  return guard([&] {
    check_reg(reg);
    if (c.x_norm == 0.0) throw ArgError{"zero-norm tensor"};
    set_dev(c);
    if (!c.copy_stream) {
      check(cudaStreamCreateWithFlags(&c.copy_stream, cudaStreamNonBlocking), "copy stream");
      for (auto& e : c.ev_copy) check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "copy event");
    }
    upload_model(c, core, core_mask, const_cast<const double* const*>(factors), factor_masks);
    // read-back staging for factors whose device rows are padded (ld != J)
    uint64_t stage = 0;
    for (int n = 0; n < c.N; ++n)
      if (c.ld[n] != c.ranks[n]) stage += c.dims[n] * c.ranks[n];
    if (stage) ensure(c, &c.d_xfer, &c.xfer_cap, stage);
    sync_const_core(c);
    uint64_t off = 0;
    for (int n = 0; n < c.N; ++n) {
      update_factor_mode(c, n, reg, lambda, true);
      // factor n is final for this iteration: copy it out behind the next modes
      const int J = c.ranks[n];
      const size_t bytes = c.dims[n] * J * sizeof(double);
      const double* src = c.d_factor[n];
      if (c.ld[n] != J) {
        k_restride<<<592, 256, 0, c.stream>>>(c.d_factor[n], c.ld[n], c.d_xfer + off, J, J, c.dims[n]);
        count_launch();
        check(cudaGetLastError(), "factor restride");
        src = c.d_xfer + off;
        off += c.dims[n] * J;
      }
      if (factors && factors[n]) {
        check(cudaEventRecord(c.ev_copy[n], c.stream), "copy event");
        check(cudaStreamWaitEvent(c.copy_stream, c.ev_copy[n], 0), "copy wait");
        check(cudaMemcpyAsync(factors[n], src, bytes, cudaMemcpyDeviceToHost, c.copy_stream), "factor d2h");
      }
    }
    core_sweep(c, reg, lambda);
    c.table_valid = false;
    if (core) check(cudaMemcpyAsync(core, c.d_core, c.G * sizeof(double), cudaMemcpyDeviceToHost, c.stream), "core");
    check(cudaStreamSynchronize(c.stream), "iteration");
    check(cudaStreamSynchronize(c.copy_stream), "factor read-back");
    if (re) *re = c.re;
  });
}

int vest_compute_delta(vest_ctx* h, const uint32_t* at, int mode, double* out) {
  Ctx& c = h->c;
  return guard([&] {
    if (mode < 0 || mode >= c.N) throw ArgError{"mode out of range"};
    for (int k = 0; k < c.N; ++k)
      if (at[k] >= c.dims[k]) throw ArgError{"query coordinate out of bounds"};
    set_dev(c);
    uint32_t* da = nullptr;
    double* dout = nullptr;
    check(cudaMalloc(&da, c.N * 4), "tmp");
    check(cudaMalloc(&dout, VEST_MAXJ * 8), "tmp");
    check(cudaMemcpyAsync(da, at, c.N * 4, cudaMemcpyHostToDevice, c.stream), "h2d");
    k_delta_one<<<1, 32, 0, c.stream>>>(c.model_view(), da, mode, dout);
    count_launch();
    check(cudaMemcpyAsync(out, dout, c.ranks[mode] * 8, cudaMemcpyDeviceToHost, c.stream), "d2h");
    check(cudaStreamSynchronize(c.stream), "delta");
    cudaFree(da);
    cudaFree(dout);
  });
}

int vest_compute_row_stats(vest_ctx* h, int mode, uint64_t row, double* gram, double* xdelta, double* last_delta) {
  Ctx& c = h->c;
  return guard([&] {
    if (mode < 0 || mode >= c.N || row >= c.dims[mode]) throw ArgError{"row out of range"};
    if (row < c.row_lo[mode] || row >= c.row_hi[mode]) throw ArgError{"row not owned by this shard context"};
    if (!gram || !xdelta) throw ArgError{"null output buffer"};
    set_dev(c);
    const int J = c.ranks[mode];
    const ModeData& md = c.modes[mode];
    const uint64_t p0 = md.h_offsets[row], p1 = md.h_offsets[row + 1];
    double* d = nullptr;
    check(cudaMalloc(&d, (J * J + 2 * J) * sizeof(double)), "tmp");
    k_row_stats_ref<<<1, std::max(J * J, 32), 0, c.stream>>>(c.model_view(), c.csf_view(mode), mode, (uint32_t)row,
                                                            p0, p1, d, d + J * J, d + J * J + J);
    count_launch();
    check(cudaGetLastError(), "row stats");
    std::vector<double> h_out(J * J + 2 * J);
    check(cudaMemcpyAsync(h_out.data(), d, h_out.size() * 8, cudaMemcpyDeviceToHost, c.stream), "d2h");
    check(cudaStreamSynchronize(c.stream), "row stats");
    cudaFree(d);
    std::copy(h_out.begin(), h_out.begin() + J * J, gram);
    std::copy(h_out.begin() + J * J, h_out.begin() + J * J + J, xdelta);
    if (last_delta) std::copy(h_out.begin() + J * J + J, h_out.end(), last_delta);
  });
}

int vest_partial_reconstruct(vest_ctx* h, const uint32_t* coords, uint64_t nq, int mode, uint64_t j, double* out) {
  Ctx& c = h->c;
  return guard([&] {
    if (mode < 0 || mode >= c.N) throw ArgError{"mode out of range"};
    if (j >= (uint64_t)c.ranks[mode]) throw ArgError{"rank index out of range"};
    for (uint64_t q = 0; q < nq; ++q)
      for (int k = 0; k < c.N; ++k)
        if (coords[q * c.N + k] >= c.dims[k]) throw ArgError{"query coordinate out of bounds"};
    if (nq == 0) return;
    set_dev(c);
    uint32_t* dc = nullptr;
    double* dout = nullptr;
    check(cudaMalloc(&dc, nq * c.N * 4), "tmp");
    check(cudaMalloc(&dout, nq * 8), "tmp");
    check(cudaMemcpyAsync(dc, coords, nq * c.N * 4, cudaMemcpyHostToDevice, c.stream), "h2d");
    const int blocks = (int)std::min<uint64_t>((nq + 255) / 256, 4096);
    k_partial_recon<<<blocks, 256, 0, c.stream>>>(c.model_view(), dc, nq, mode, (uint32_t)j, dout);
    count_launch();
    check(cudaGetLastError(), "partial reconstruct");
    check(cudaMemcpyAsync(out, dout, nq * 8, cudaMemcpyDeviceToHost, c.stream), "d2h");
    check(cudaStreamSynchronize(c.stream), "partial reconstruct");
    cudaFree(dc);
    cudaFree(dout);
  });
}

int vest_get_factor_rows(vest_ctx* h, int mode, uint64_t row_lo, uint64_t nrows, double* out) {
  Ctx& c = h->c;
  return guard([&] {
    if (mode < 0 || mode >= c.N || row_lo > c.dims[mode] || nrows > c.dims[mode] - row_lo)
      throw ArgError{"row out of range"};
    if (nrows == 0) return;
    set_dev(c);
    const int J = c.ranks[mode];
    check(cudaMemcpy2DAsync(out, J * sizeof(double), c.d_factor[mode] + row_lo * c.ld[mode], c.ld[mode] * sizeof(double),
                            J * sizeof(double), nrows, cudaMemcpyDeviceToHost, c.stream),
          "factor rows d2h");
    check(cudaStreamSynchronize(c.stream), "factor rows");
  });
}

int vest_predict(vest_ctx* h, const uint32_t* coords, uint64_t nq, double* out) {
  Ctx& c = h->c;
  return guard([&] {
    set_dev(c);
    coo_recon(c, coords, nullptr, nq, out, nullptr);
  });
}

int vest_evaluate(vest_ctx* h, const uint32_t* coords, const double* values, uint64_t n, double* re) {
  Ctx& c = h->c;
  return guard([&] {
    set_dev(c);
    double acc = 0.0;  // frobenius_norm of the test tensor, serial like the reference
    for (uint64_t e = 0; e < n; ++e) acc += values[e] * values[e];
    const double xn = std::sqrt(acc);
    if (xn == 0.0) throw ArgError{"zero-norm tensor"};
    double sums[2] = {0, 0};
    coo_recon(c, coords, values, n, nullptr, sums);
    *re = std::sqrt(sums[0]) / xn;
  });
}

int vest_compute_responsibilities(vest_ctx* h, double* core_out, double* const* factor_outs, double* base_re) {
  Ctx& c = h->c;
  return guard([&] {
    if (c.x_norm == 0.0) throw ArgError{"zero-norm tensor"};
    set_dev(c);
    responsibilities(c);
    if (core_out)
      check(cudaMemcpyAsync(core_out, c.d_resp_core, c.G * sizeof(double), cudaMemcpyDeviceToHost, c.stream), "d2h");
    for (int n = 0; n < c.N; ++n)
      if (factor_outs && factor_outs[n])
        check(cudaMemcpyAsync(factor_outs[n], c.d_resp_f[n], c.dims[n] * c.ranks[n] * sizeof(double),
                              cudaMemcpyDeviceToHost, c.stream),
              "d2h");
    check(cudaStreamSynchronize(c.stream), "resp d2h");
    if (base_re) *base_re = c.table_re;
  });
}

int vest_prune_step(vest_ctx* h, double pr, const double* core_resp, const double* const* factor_resp,
                    uint64_t* counts) {
  Ctx& c = h->c;
  return guard([&] {
    sync_const_core(c);  // the core changes here: the constant-bank copy is stale
    if (!(pr >= 0.0 && pr < 1.0)) throw ArgError{"prune rate must be in [0, 1)"};
    set_dev(c);
    if (core_resp) {
      check(cudaMemcpyAsync(c.d_resp_core, core_resp, c.G * sizeof(double), cudaMemcpyHostToDevice, c.stream), "h2d");
      for (int n = 0; n < c.N; ++n)
        check(cudaMemcpyAsync(c.d_resp_f[n], factor_resp[n], c.dims[n] * c.ranks[n] * sizeof(double),
                              cudaMemcpyHostToDevice, c.stream),
              "h2d");
    } else if (!c.table_valid) {
      throw ArgError{"no responsibility table: call compute_responsibilities first"};
    }
    prune(c, pr, counts);
    c.r_valid = false;
    c.r_pending[0] = c.r_pending[1] = -1;
    c.r_fresh = false;
    c.table_valid = false;
    sync_const_core(c);
  });
}

int vest_sparsity(vest_ctx* h, double* zero_fraction, double* masked_fraction) {
  Ctx& c = h->c;
  return guard([&] {
    set_dev(c);
    sparsity(c, zero_fraction, masked_fraction);
  });
}

int vest_normalize_columns(vest_ctx* h) {
  Ctx& c = h->c;
  return guard([&] {
    sync_const_core(c);  // the core changes here: the constant-bank copy is stale
    set_dev(c);
    normalize_columns(c);
    c.r_valid = false;
    c.r_pending[0] = c.r_pending[1] = -1;
    c.r_fresh = false;
    c.table_valid = false;
    sync_const_core(c);
  });
}

int vest_get_mode_index(vest_ctx* h, int mode, uint64_t* offsets, uint32_t* ids) {
  Ctx& c = h->c;
  return guard([&] {
    if (mode < 0 || mode >= c.N) throw ArgError{"mode out of range"};
    set_dev(c);
    const ModeData& md = c.modes[mode];
    if (c.local_nnz[mode] != c.nnz) throw ArgError{"a shard context holds the index of its own rows only"};
    std::memcpy(offsets, md.h_offsets.data(), (c.dims[mode] + 1) * sizeof(uint64_t));
    if (c.nnz) check(cudaMemcpy(ids, md.d_eid, c.nnz * sizeof(uint32_t), cudaMemcpyDeviceToHost), "ids");
  });
}

int vest_ctx_profile(vest_ctx* h, int on) {
  h->c.prof_on = on != 0;
  return VEST_OK;
}

int vest_ctx_profile_read(vest_ctx* h, double* ms, uint64_t* launches, int reset) {
  Ctx& c = h->c;
  return guard([&] {
    set_dev(c);
    check(cudaStreamSynchronize(c.stream), "profile sync");
    for (auto& e : c.prof_events) {
      float t = 0.f;
      check(cudaEventElapsedTime(&t, e.a, e.b), "event time");
      c.prof_ms[e.fam] += t;
      c.prof_n[e.fam] += 1;
      cudaEventDestroy(e.a);
      cudaEventDestroy(e.b);
    }
    c.prof_events.clear();
    for (int f = 0; f < VEST_PROF_FAMILIES; ++f) {
      if (ms) ms[f] = c.prof_ms[f];
      if (launches) launches[f] = c.prof_n[f];
      if (reset) c.prof_ms[f] = 0.0, c.prof_n[f] = 0;
    }
  });
}

int vest_frobenius_norm(vest_ctx* h, double* out) {
  *out = h->c.x_norm;
  return VEST_OK;
}

}  // extern "C"
