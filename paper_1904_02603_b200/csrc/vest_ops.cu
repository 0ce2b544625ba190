// SPDX-License-Identifier: Apache-2.0
// vest_ops.cu -- prune_step (pruning.hpp:193-247) as a device radix select,
// sparsity / masked_fraction (tucker_model.hpp:190-207), normalize_columns
// (tucker_model.hpp:212-236), and small reductions / fills.
#include <algorithm>
#include <cmath>
#include <vector>

#include "../../include/vest.h"
#include "vest_common.cuh"

namespace vest {

// --------------------------------------------------------------- reductions --
// Deterministic sum of n doubles: one CTA, fixed per-thread strides and a
// fixed tree (run-to-run bit-identical).
__global__ void __launch_bounds__(1024) k_sum(const double* in, uint64_t n, double* out) {
  __shared__ double red[32];
  double s = 0.0;
  for (uint64_t i = threadIdx.x; i < n; i += blockDim.x) s += in[i];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    v = warp_sum(v);
    if (threadIdx.x == 0) *out = v;
  }
}

// the sum into a device slot (global over the shards), no host read-back
void sum_chunks_device(Ctx& c, const double* d_in, uint64_t n, double* out) {
  k_sum<<<1, 1024, 0, c.stream>>>(d_in, n, out);
  count_launch();
  comm_allreduce(c, out, 1);
}

double reduce_chunk_sums(Ctx& c, const double* d_in, uint64_t n) {
  k_sum<<<1, 1024, 0, c.stream>>>(d_in, n, c.d_small);
  count_launch();
  comm_allreduce(c, c.d_small, 1);  // residual sums are global over the shards
  check(cudaMemcpyAsync(c.h_small, c.d_small, sizeof(double), cudaMemcpyDeviceToHost, c.stream),
        "sum readback");
  if (c.capturing) return 0.0;  // a captured read-back: the replay's caller reads h_small[0]
  check(cudaStreamSynchronize(c.stream), "sum sync");
  return c.h_small[0];
}

__global__ void k_fill_resp(double* resp, const uint8_t* mask, uint64_t n, double unmasked) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    resp[i] = mask[i] ? INFINITY : unmasked;
}

// L1 rows without observations (updates.hpp:113-139 with empty statistics):
// lin = 0, g = 0, d = 0 -> |g| <= lambda sets every unmasked element to 0.
__global__ void k_l1_empty(const uint32_t* rows, uint32_t n, double* factor, int ld, const uint8_t* mask,
                           int J, double lambda) {
  const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (t >= (uint64_t)n * J) return;
  const uint32_t row = rows[t / J];
  const int j = t % J;
  if (!mask[(size_t)row * J + j] && 0.0 <= lambda) factor[(size_t)row * ld + j] = 0.0;
}

void fill_factor_resp(Ctx& c, int n, double unmasked) {
  const uint64_t cnt = c.dims[n] * c.ranks[n];
  k_fill_resp<<<296, 256, 0, c.stream>>>(c.d_resp_f[n], c.d_fmask[n], cnt, unmasked);
  count_launch();
}

void l1_empty_rows(Ctx& c, int n, double lambda) {
  const ModeData& md = c.modes[n];
  if (md.nempty == 0) return;
  const uint64_t t = (uint64_t)md.nempty * c.ranks[n];
  k_l1_empty<<<(unsigned)((t + 255) / 256), 256, 0, c.stream>>>(md.d_empty, md.nempty, c.d_factor[n], c.ld[n],
                                                             c.d_fmask[n], c.ranks[n], lambda);
  count_launch();
}

// ------------------------------------------------------------------- prune --
// Keys: doubles mapped to an unsigned order-preserving 64-bit key, with -0.0
// canonicalised to +0.0 (the reference comparator treats them as equal,
// pruning.hpp:215-218).  Masked positions are not candidates.
__device__ __forceinline__ unsigned long long okey(double v) {
  if (v == 0.0) v = 0.0;
  const long long b = __double_as_longlong(v);
  return b >= 0 ? (unsigned long long)b ^ 0x8000000000000000ull : ~(unsigned long long)b;
}

struct SelState {
  unsigned long long prefix, pmask, krem;
  unsigned long long hist[256];
};

__global__ void k_count_cand(const uint8_t* mask, uint64_t n, unsigned long long* out) {
  unsigned long long c = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    c += mask[i] ? 0 : 1;
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

__global__ void k_sel_init(SelState* s, unsigned long long k) {
  s->prefix = 0;
  s->pmask = 0;
  s->krem = k;
  for (int i = 0; i < 256; ++i) s->hist[i] = 0;
}

__global__ void k_sel_hist(const double* resp, const uint8_t* mask, uint64_t n, SelState* s, int shift) {
  __shared__ unsigned int h[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) h[i] = 0;
  __syncthreads();
  const unsigned long long prefix = s->prefix, pmask = s->pmask;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    if (mask[i]) continue;
    const unsigned long long key = okey(resp[i]);
    if ((key & pmask) != prefix) continue;
    atomicAdd(&h[(key >> shift) & 255u], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 256; i += blockDim.x)
    if (h[i]) atomicAdd(&s->hist[i], (unsigned long long)h[i]);
}

__global__ void k_sel_pick(SelState* s, int shift) {
  unsigned long long cum = 0;
  int d = 0;
  for (; d < 256; ++d) {
    if (cum + s->hist[d] >= s->krem) break;
    cum += s->hist[d];
  }
  if (d > 255) d = 255;
  s->prefix |= (unsigned long long)d << shift;
  s->pmask |= 255ull << shift;
  s->krem -= cum;
  for (int i = 0; i < 256; ++i) s->hist[i] = 0;
}

// Ties at the threshold key are taken in ascending index order: per-CTA tie
// counts first, then each CTA ranks its own (contiguous) range.
constexpr int kApplyThreads = 256;

__global__ void k_tie_count(const double* resp, const uint8_t* mask, uint64_t n, const SelState* s,
                            uint64_t per, unsigned long long* cta_ties) {
  const uint64_t lo = blockIdx.x * per, hi = min(n, lo + per);
  unsigned long long c = 0;
  for (uint64_t i = lo + threadIdx.x; i < hi; i += blockDim.x)
    if (!mask[i] && okey(resp[i]) == s->prefix) ++c;
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  __shared__ unsigned long long red[kApplyThreads / 32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (int w = 0; w < kApplyThreads / 32; ++w) t += red[w];
    cta_ties[blockIdx.x] = t;
  }
}

__global__ void k_prune_apply(const double* resp, uint8_t* mask, uint64_t n, const SelState* s,
                              uint64_t per, const unsigned long long* cta_ties, double* values,
                              int J, int ld, int take_all) {
  __shared__ unsigned long long base;
  __shared__ unsigned int wsum[kApplyThreads / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    unsigned long long b = 0;
    for (unsigned i = 0; i < blockIdx.x; ++i) b += cta_ties[i];
    base = b;
  }
  __syncthreads();
  const uint64_t lo = blockIdx.x * per, hi = min(n, lo + per);
  const unsigned long long thr = take_all ? 0 : s->prefix;
  const unsigned long long krem = take_all ? 0 : s->krem;
  for (uint64_t t0 = lo; t0 < hi; t0 += blockDim.x) {
    const uint64_t i = t0 + threadIdx.x;
    bool cand = false, tie = false;
    unsigned long long key = 0;
    if (i < hi && !mask[i]) {
      cand = true;
      key = okey(resp[i]);
      tie = !take_all && key == thr;
    }
    const unsigned bal = __ballot_sync(0xffffffffu, tie);
    if (lane == 0) wsum[warp] = __popc(bal);
    __syncthreads();
    unsigned before = 0;
    for (int w = 0; w < warp; ++w) before += wsum[w];
    unsigned tot = 0;
    for (int w = 0; w < kApplyThreads / 32; ++w) tot += wsum[w];
    const unsigned long long rank = base + before + __popc(bal & ((1u << lane) - 1u));
    bool take = false;
    if (cand) take = take_all || key < thr || (tie && rank < krem);
    if (take) {
      mask[i] = 1;
      values[(i / J) * ld + (i % J)] = 0.0;
    }
    __syncthreads();
    if (threadIdx.x == 0) base += tot;
    __syncthreads();
  }
}

// detail::prune_lowest (pruning.hpp:206-222) on one block of n elements.
static uint64_t prune_block(Ctx& c, const double* resp, uint8_t* mask, double* values, uint64_t n,
                            int J, int ld, uint64_t want) {
  if (want == 0 || n == 0) return 0;
  unsigned long long* cnt = c.d_counts;
  check(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long), c.stream), "memset");
  k_count_cand<<<296, 256, 0, c.stream>>>(mask, n, cnt);
  unsigned long long ncand = 0;
  check(cudaMemcpyAsync(&ncand, cnt, sizeof(ncand), cudaMemcpyDeviceToHost, c.stream), "ncand");
  check(cudaStreamSynchronize(c.stream), "ncand sync");
  count_launch();
  const uint64_t take = std::min<uint64_t>(want, ncand);
  if (take == 0) return 0;
  SelState* s = static_cast<SelState*>(c.d_sel);
  const int grid = (int)std::min<uint64_t>(592, (n + 255) / 256);
  const bool all = take == ncand;
  if (!all) {
    k_sel_init<<<1, 1, 0, c.stream>>>(s, take);
    for (int d = 0; d < 8; ++d) {
      const int shift = 56 - 8 * d;
      k_sel_hist<<<grid, 256, 0, c.stream>>>(resp, mask, n, s, shift);
      k_sel_pick<<<1, 1, 0, c.stream>>>(s, shift);
    }
    count_launch(17);
  }
  const int napply = (int)std::min<uint64_t>(592, (n + kApplyThreads - 1) / kApplyThreads);
  const uint64_t per = (n + napply - 1) / napply;
  unsigned long long* ties = cnt + 1;
  if (!all) {
    k_tie_count<<<napply, kApplyThreads, 0, c.stream>>>(resp, mask, n, s, per, ties);
    count_launch();
  }
  k_prune_apply<<<napply, kApplyThreads, 0, c.stream>>>(resp, mask, n, s, per, ties, values, J, ld, all ? 1 : 0);
  count_launch();
  check(cudaGetLastError(), "prune");
  return take;
}

void prune(Ctx& c, double pr, uint64_t* counts) {
  ProfScope ps(c, kProfPrune);
  // k = floor(pr * size) with size the block's full element count
  // (pruning.hpp:237-245), computed exactly as the reference does.
  counts[0] = prune_block(c, c.d_resp_core, c.d_core_mask, c.d_core, (uint64_t)c.G, c.G, c.G,
                          static_cast<uint64_t>(pr * double(c.G)));
  for (int n = 0; n < c.N; ++n) {
    const uint64_t size = c.dims[n] * c.ranks[n];
    counts[1 + n] = prune_block(c, c.d_resp_f[n], c.d_fmask[n], c.d_factor[n], size, c.ranks[n], c.ld[n],
                                static_cast<uint64_t>(pr * double(size)));
  }
  check(cudaMemcpyAsync(c.h_core_mask.data(), c.d_core_mask, c.G, cudaMemcpyDeviceToHost, c.stream), "mask");
  check(cudaStreamSynchronize(c.stream), "prune sync");
}

// ---------------------------------------------------------------- sparsity --
__global__ void k_count_zero(const double* v, const uint8_t* mask, uint64_t n, int J, int ld,
                             unsigned long long* out) {
  unsigned long long z = 0, m = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    z += v[(i / J) * ld + (i % J)] == 0.0;
    m += mask[i];
  }
  for (int o = 16; o > 0; o >>= 1) {
    z += __shfl_xor_sync(0xffffffffu, z, o);
    m += __shfl_xor_sync(0xffffffffu, m, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (z) atomicAdd(out, z);
    if (m) atomicAdd(out + 1, m);
  }
}

void sparsity(Ctx& c, double* zero_frac, double* masked_frac) {
  unsigned long long* cnt = c.d_counts;
  check(cudaMemsetAsync(cnt, 0, 2 * sizeof(unsigned long long), c.stream), "memset");
  k_count_zero<<<64, 256, 0, c.stream>>>(c.d_core, c.d_core_mask, c.G, c.G, c.G, cnt);
  uint64_t total = c.G;
  for (int n = 0; n < c.N; ++n) {
    const uint64_t sz = c.dims[n] * c.ranks[n];
    k_count_zero<<<296, 256, 0, c.stream>>>(c.d_factor[n], c.d_fmask[n], sz, c.ranks[n], c.ld[n], cnt);
    total += sz;
  }
  count_launch(1 + c.N);
  unsigned long long h[2];
  check(cudaMemcpyAsync(h, cnt, sizeof h, cudaMemcpyDeviceToHost, c.stream), "count readback");
  check(cudaStreamSynchronize(c.stream), "count sync");
  if (zero_frac) *zero_frac = double(h[0]) / double(total);
  if (masked_frac) *masked_frac = double(h[1]) / double(total);
}

// ----------------------------------------------------------- normalisation --
__global__ void k_colsq(const double* a, uint64_t I, int J, int ld, double* partial) {
  // partial[block][j] = sum over this block's rows of a[i][j]^2
  extern __shared__ double sh[];
  const uint64_t per = (I + gridDim.x - 1) / gridDim.x;
  const uint64_t lo = blockIdx.x * per, hi = min(I, lo + per);
  for (int j = 0; j < J; ++j) {
    double s = 0.0;
    for (uint64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
      const double v = a[i * ld + j];
      s = fma(v, v, s);
    }
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sh[w];
      partial[(size_t)blockIdx.x * J + j] = t;
    }
    __syncthreads();
  }
}

__global__ void k_colnorm(const double* partial, int nparts, int J, double* norms) {
  const int j = threadIdx.x;
  if (j >= J) return;
  double s = 0.0;
  for (int p = 0; p < nparts; ++p) s += partial[(size_t)p * J + j];
  norms[j] = s;  // squared; 0 -> column skipped
}

__global__ void k_colscale(double* a, uint64_t I, int J, int ld, const double* norms2) {
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < I * J; t += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t i = t / J;
    const int j = t % J;
    const double n2 = norms2[j];
    if (n2 != 0.0) a[i * ld + j] /= sqrt(n2);
  }
}

__global__ void k_corescale(double* core, int G, int N, const uint32_t* cellbeta, const double* norms2,
                            const int* noff) {
  const int lin = blockIdx.x * blockDim.x + threadIdx.x;
  if (lin >= G) return;
  const uint32_t b = cellbeta[lin];
  double v = core[lin];
  for (int k = 0; k < N; ++k) {
    const double n2 = norms2[noff[k] + ((b >> (4 * k)) & 15u)];
    if (n2 != 0.0) v *= sqrt(n2);
  }
  core[lin] = v;
}

void normalize_columns(Ctx& c) {
  std::vector<int> noff(c.N + 1, 0);
  for (int k = 0; k < c.N; ++k) noff[k + 1] = noff[k] + c.ranks[k];
  const int nparts = 148;
  ensure(c, &c.d_gemm_part, &c.gemm_part_cap, (size_t)nparts * VEST_MAXJ);
  ensure(c, &c.d_gemm_out, &c.gemm_out_cap, (size_t)noff[c.N] + 8);
  for (int k = 0; k < c.N; ++k) {
    k_colsq<<<nparts, 256, 8 * sizeof(double), c.stream>>>(c.d_factor[k], c.dims[k], c.ranks[k], c.ld[k], c.d_gemm_part);
    k_colnorm<<<1, 32, 0, c.stream>>>(c.d_gemm_part, nparts, c.ranks[k], c.d_gemm_out + noff[k]);
    k_colscale<<<296, 256, 0, c.stream>>>(c.d_factor[k], c.dims[k], c.ranks[k], c.ld[k], c.d_gemm_out + noff[k]);
    count_launch(3);
  }
  int* d_noff = reinterpret_cast<int*>(c.d_gemm_part);
  check(cudaMemcpyAsync(d_noff, noff.data(), noff.size() * sizeof(int), cudaMemcpyHostToDevice, c.stream), "noff");
  k_corescale<<<(c.G + 255) / 256, 256, 0, c.stream>>>(c.d_core, c.G, c.N, c.d_cellbeta, c.d_gemm_out, d_noff);
  count_launch();
  check(cudaStreamSynchronize(c.stream), "normalize");
}

// ----------------------------------------------------- FP64 peak benchmark --
// 8 independent DFMA chains per thread, enough warps to fill every SMSP; the
// result is the FP64 FMA roof the bench divides by (2 flops per DFMA).
__global__ void __launch_bounds__(256) k_dfma_peak(double* out, int iters, double a, double b) {
  double v[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = threadIdx.x * 1e-9 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = fma(v[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += v[i];
  if (s == 12345.678) out[0] = s;
}

}  // namespace vest

extern "C" int vest_measure_fp64_peak(int device, double* tflops) {
  using namespace vest;
  if (cudaSetDevice(device) != cudaSuccess) return VEST_ECUDA;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  double* out = nullptr;
  cudaMalloc(&out, 64);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  // ~4 ms per launch (short launches under-report the pipe by their ramp/tail)
  const int blocks = sms * 8, threads = 256, iters = 32768;
  k_dfma_peak<<<blocks, threads>>>(out, 256, 0.999999, 1e-7);  // warm up clocks
  double best = 0.0;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    k_dfma_peak<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 2.0 * 8.0 * iters * (double)blocks * threads;
    best = std::max(best, flops / (ms * 1e-3) / 1e12);
  }
  count_launch(6);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  *tflops = best;
  return cudaGetLastError() == cudaSuccess ? VEST_OK : VEST_ECUDA;
}
