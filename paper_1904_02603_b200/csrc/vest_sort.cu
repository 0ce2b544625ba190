// SPDX-License-Identifier: Apache-2.0
// vest_sort.cu -- stable LSD radix sort of (uint32 key, uint32 value) pairs on
// the device: the K1 step of the CSF build (sparse_tensor.hpp:119-137 sorts
// entry ids by one coordinate, ids ascending within a slice) and of the
// duplicate check (sparse_tensor.hpp:80-94).
//
// 8 bits per pass.  A pass is three steps over warp tiles (kRsTile consecutive
// elements owned by one warp):
//   1. k_rs_hist     per-tile digit counts -> hist[digit][tile]
//   2. scan          exclusive prefix over hist in (digit, tile) order: the
//                    global position of each tile's first element per digit
//   3. k_rs_scatter  the warp walks its tile 32 elements at a time, in order;
//                    lanes with equal digits find each other with eight
//                    ballots (one per digit bit), a lane's rank among them is the popcount
//                    of the lower lanes -- stable without any atomics -- and
//                    the tile's running per-digit position lives in shared
//                    memory.
// Everything is deterministic; no block-wide synchronisation in steps 1 and 3.
#include <algorithm>

#include "vest_internal.h"

namespace vest {

namespace {

constexpr int kRsTile = 8192;  // elements per warp tile
constexpr int kRsWarps = 8;    // warps per CTA
constexpr int kScanItems = 16, kScanThreads = 256, kScanChunk = kScanItems * kScanThreads;

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Lanes holding the same 8-bit digit as this one (valid lanes only): eight
// ballots, one per digit bit -- a fixed cost, where match.any iterates once per
// distinct value in the warp (~32 for random digits).
__device__ __forceinline__ uint32_t same_digit(uint32_t d, bool valid) {
  uint32_t m = __ballot_sync(0xffffffffu, valid);
#pragma unroll
  for (int b = 0; b < 8; ++b) {
    const bool bit = (d >> b) & 1u;
    const uint32_t bal = __ballot_sync(0xffffffffu, bit);
    m &= bit ? bal : ~bal;
  }
  return m;
}

__global__ void __launch_bounds__(kRsWarps * 32) k_rs_hist(const uint32_t* __restrict__ keys, uint64_t n, int shift,
                                                           uint32_t mask, uint32_t ntiles,
                                                           uint32_t* __restrict__ hist) {
  __shared__ uint32_t h[kRsWarps][256];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (uint32_t tile = blockIdx.x * kRsWarps + warp; tile < ntiles; tile += gridDim.x * kRsWarps) {
#pragma unroll
    for (int j = 0; j < 8; ++j) h[warp][lane + 32 * j] = 0;
    __syncwarp();
    const uint64_t beg = (uint64_t)tile * kRsTile, end = min(n, beg + kRsTile);
    for (uint64_t i0 = beg; i0 < end; i0 += 32) {
      const uint64_t i = i0 + lane;
      const bool valid = i < end;
      const uint32_t d = valid ? (__ldg(keys + i) >> shift) & mask : 0u;
      const uint32_t m = same_digit(d, valid);
      if (valid && (m & lanemask_lt()) == 0) h[warp][d] += __popc(m);  // one leader per digit
      __syncwarp();
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) hist[(uint64_t)(lane + 32 * j) * ntiles + tile] = h[warp][lane + 32 * j];
    __syncwarp();
  }
}

__global__ void __launch_bounds__(kRsWarps * 32) k_rs_scatter(const uint32_t* __restrict__ kin,
                                                              const uint32_t* __restrict__ vin,
                                                              uint32_t* __restrict__ kout, uint32_t* __restrict__ vout,
                                                              uint64_t n, int shift, uint32_t mask, uint32_t ntiles,
                                                              const uint32_t* __restrict__ offs) {
  __shared__ uint32_t base[kRsWarps][256];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (uint32_t tile = blockIdx.x * kRsWarps + warp; tile < ntiles; tile += gridDim.x * kRsWarps) {
#pragma unroll
    for (int j = 0; j < 8; ++j) base[warp][lane + 32 * j] = offs[(uint64_t)(lane + 32 * j) * ntiles + tile];
    __syncwarp();
    const uint64_t beg = (uint64_t)tile * kRsTile, end = min(n, beg + kRsTile);
    uint32_t nkey = beg + lane < end ? __ldg(kin + beg + lane) : 0u;  // one step ahead
    uint32_t nval = beg + lane < end ? __ldg(vin + beg + lane) : 0u;
    for (uint64_t i0 = beg; i0 < end; i0 += 32) {
      const uint64_t i = i0 + lane;
      const bool valid = i < end;
      const uint32_t key = nkey, val = nval;
      if (i + 32 < end) {
        nkey = __ldg(kin + i + 32);
        nval = __ldg(vin + i + 32);
      }
      const uint32_t d = valid ? (key >> shift) & mask : 0u;
      const uint32_t m = same_digit(d, valid);
      const uint32_t rank = __popc(m & lanemask_lt());
      if (valid) {
        const uint32_t pos = base[warp][d] + rank;
        kout[pos] = key;
        vout[pos] = val;
      }
      __syncwarp();
      if (valid && rank == 0) base[warp][d] += __popc(m);
      __syncwarp();
    }
  }
}

// ---- exclusive scan of a uint32 array, in place ---------------------------
__device__ __forceinline__ uint32_t block_exclusive(uint32_t v, uint32_t* total) {
  __shared__ uint32_t ws[kScanThreads / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += t;
  }
  if (lane == 31) ws[warp] = inc;
  __syncthreads();
  uint32_t before = 0, all = 0;
#pragma unroll
  for (int w = 0; w < kScanThreads / 32; ++w) {
    const uint32_t s = ws[w];
    if (w < warp) before += s;
    all += s;
  }
  __syncthreads();
  *total = all;
  return before + inc - v;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_sums(const uint32_t* __restrict__ data, uint64_t len,
                                                            uint32_t* __restrict__ sums) {
  const uint64_t beg = (uint64_t)blockIdx.x * kScanChunk + (uint64_t)threadIdx.x * kScanItems;
  uint32_t s = 0;
#pragma unroll
  for (int j = 0; j < kScanItems; ++j)
    if (beg + j < len) s += data[beg + j];
  uint32_t total;
  block_exclusive(s, &total);
  if (threadIdx.x == 0) sums[blockIdx.x] = total;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_top(uint32_t* sums, uint32_t nb) {
  uint32_t carry = 0;
  for (uint32_t off = 0; off < nb; off += kScanThreads) {
    const uint32_t i = off + threadIdx.x;
    const uint32_t v = i < nb ? sums[i] : 0;
    uint32_t total;
    const uint32_t ex = block_exclusive(v, &total);
    if (i < nb) sums[i] = carry + ex;
    carry += total;
  }
}

__global__ void __launch_bounds__(kScanThreads) k_scan_apply(uint32_t* __restrict__ data, uint64_t len,
                                                             const uint32_t* __restrict__ sums) {
  const uint64_t beg = (uint64_t)blockIdx.x * kScanChunk + (uint64_t)threadIdx.x * kScanItems;
  uint32_t v[kScanItems], s = 0;
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    v[j] = beg + j < len ? data[beg + j] : 0;
    s += v[j];
  }
  uint32_t total;
  uint32_t run = sums[blockIdx.x] + block_exclusive(s, &total);
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    if (beg + j < len) data[beg + j] = run;
    run += v[j];
  }
}

}  // namespace

// Temporary storage of radix_sort_pairs for n elements: the alternate key and
// value buffers of the ping-pong, the tile histogram and the scan's block sums.
size_t radix_sort_tmp_bytes(uint64_t n) {
  const uint64_t ntiles = (n + kRsTile - 1) / kRsTile;
  const uint64_t len = 256 * ntiles, nb = (len + kScanChunk - 1) / kScanChunk;
  return (size_t)(2 * n + len + nb + 64) * sizeof(uint32_t);
}

// Stable sort of (kin, vin) by bits [0, end_bit) of the key into (kout, vout);
// the inputs are left intact, outputs must not alias them.  Returns the number
// of kernels launched.
int radix_sort_pairs(const uint32_t* kin, uint32_t* kout, const uint32_t* vin, uint32_t* vout, uint64_t n, int end_bit,
                     void* tmp, cudaStream_t stream) {
  if (n == 0) return 0;
  const int passes = std::max(1, (end_bit + 7) / 8);
  const uint32_t ntiles = (uint32_t)((n + kRsTile - 1) / kRsTile);
  const uint64_t len = 256ull * ntiles;
  const uint32_t nb = (uint32_t)((len + kScanChunk - 1) / kScanChunk);
  uint32_t* alt_k = static_cast<uint32_t*>(tmp);
  uint32_t* alt_v = alt_k + n;
  uint32_t* hist = alt_v + n;
  uint32_t* sums = hist + len;
  int sms = 148;
  {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const unsigned grid = (unsigned)std::min<uint64_t>((ntiles + kRsWarps - 1) / kRsWarps, (uint64_t)sms * 8);
  // the scatter's write frontier is (resident warps) x 256 bins x 2 arrays x one
  // 32-byte sector: 2 CTAs per SM keep it (~39 MB) inside the L2, so sectors
  // fill there before they are written back
  const unsigned sgrid = (unsigned)std::min<uint64_t>((ntiles + kRsWarps - 1) / kRsWarps, (uint64_t)sms * 2);
  const uint32_t* sk = kin;
  const uint32_t* sv = vin;
  int launches = 0;
  for (int p = 1; p <= passes; ++p) {
    const int shift = 8 * (p - 1);
    const int bits = std::min(8, std::max(1, end_bit - shift));
    const uint32_t mask = (1u << bits) - 1u;
    const bool to_out = (passes - p) % 2 == 0;
    uint32_t* dk = to_out ? kout : alt_k;
    uint32_t* dv = to_out ? vout : alt_v;
    k_rs_hist<<<grid, kRsWarps * 32, 0, stream>>>(sk, n, shift, mask, ntiles, hist);
    k_scan_sums<<<nb, kScanThreads, 0, stream>>>(hist, len, sums);
    k_scan_top<<<1, kScanThreads, 0, stream>>>(sums, nb);
    k_scan_apply<<<nb, kScanThreads, 0, stream>>>(hist, len, sums);
    k_rs_scatter<<<sgrid, kRsWarps * 32, 0, stream>>>(sk, sv, dk, dv, n, shift, mask, ntiles, hist);
    launches += 5;
    sk = dk;
    sv = dv;
  }
  return launches;
}

}  // namespace vest
