// SPDX-License-Identifier: Apache-2.0
// vest_core.cu -- the core update (updates.hpp:177-262) and the core
// responsibilities (pruning.hpp:93-134).
//
// Exact Gauss-Seidel over the core cells in row-major order, blocked by
// FIBERS along the last mode m = N-1 (a fiber = the J_m consecutive cells that
// share the prefix beta_0..beta_{m-1}).  For a block of F fibers, with
//   s_ef = prod_{k<m} A_k[i_k, beta_k(f)]    (per entry)
//   p_e(f,c) = s_ef * A_m[i_m, c]
// every block statistic factorises over the slices i_m of the last mode:
//   c_(f,c)            = sum_e r_e p_e(f,c)  = sum_slices A_m[s,c]       * R^s_f
//   H_(f,c),(f',c')    = sum_e p p           = sum_slices A_m[s,c]A_m[s,c'] * S^s_ff'
// with R^s_f = sum_{e in s} s_ef r_e and S^s_ff' = sum_{e in s} s_ef s_ef'.
// One pass over the entries (k_core_pass) produces (S, R) per slice chunk,
// a small GEMM over the slices (k_core_gemm + k_colsum) produces (T, C), and one
// warp solves the block's cells sequentially (k_core_solve):
//   num_q = c_q - sum_{q' < q} dg_q' H_q'q + g_old H_qq ,  den_q = H_qq
// which is exactly the reference's num/den (updates.hpp:211-217) for the
// state after the earlier cells' updates; only the summation order differs.
// The next pass applies r -= sum dg p for the finished block before it
// accumulates the next block, and a final pass applies the last block and sums
// r^2 (the residual/RE of compute_residuals, tucker_model.hpp:168-183).
#include <algorithm>
#include <cstdlib>
#include <vector>

#include "vest_common.cuh"

namespace vest {

constexpr int kFMax = 15;  // fibers per block (general pass: 15 s-columns + r on DMMA)
constexpr int kPassWarps = 8;

struct CorePassArgs {
  DevModel m;
  DevCSF csf;  // mode N-1
  double* r;
  // block fibers: prefix lin index over modes 0..m-1
  const uint32_t* prev_fib;
  int prev_nf;
  const double* prev_dg;  // [prev_nf][Jm]
  const uint32_t* cur_fib;
  int cur_nf;
  int kind;  // 0 sweep (S, R), 1 responsibility (R, D), 2 final (apply prev, sum r^2)
  double* stats;
  int stride;
  double* chunk_sq;
};

template <int B, int E, class F>
__device__ __forceinline__ void sfor(F&& f) {
  if constexpr (B < E) {
    f(std::integral_constant<int, B>{});
    sfor<B + 1, E>(f);
  }
}

template <int V>
__device__ __forceinline__ void treduce(double (&v)[V], int lane) {
  sfor<0, 5>([&](auto sc) {
    constexpr int s = decltype(sc)::value;
    constexpr int H = (V >> s) / 2;
    constexpr int off = 16 >> s;
    const bool up = (lane & off) != 0;
#pragma unroll
    for (int i = 0; i < H; ++i) {
      const double keep = up ? v[i + H] : v[i];
      const double send = up ? v[i] : v[i + H];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
    }
  });
}

// One warp per chunk of a last-mode slice (runtime ranks / sparse fiber
// lists).  Per entry: the rows of modes < m are gathered once (vector loads,
// all issued before use) into a lane-major shared-memory stage; the previous
// block's residual update and the current block's fiber products
// s_f = prod_k row_k[beta_k(f)] read it; the (s_0..s_{nf-1}, r) vectors are
// staged transposed (r in column 15) and S = sum s s^T, R = sum s r are
// accumulated on the FP64 tensor cores (DMMA), as in the structured pass.
template <int M>
__global__ void __launch_bounds__(kPassWarps * 32) k_core_pass(CorePassArgs a) {
  extern __shared__ double smem[];
  __shared__ int sb[2][kFMax][M > 0 ? M : 1];  // beta of each fiber (prev, cur)
  __shared__ double sdg[kFMax * VEST_MAXJ];
  __shared__ double sq_q[kPassWarps][kFMax];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int Jm = a.m.J[M];
  for (int t = threadIdx.x; t < 2 * kFMax * M; t += blockDim.x) {
    const int which = t / (kFMax * M), rest = t % (kFMax * M), f = rest / M, k = rest % M;
    const uint32_t* fl = which ? a.cur_fib : a.prev_fib;
    const int nf = which ? a.cur_nf : a.prev_nf;
    int b = 0;
    if (f < nf) b = (a.m.cellbeta[fl[f] * Jm] >> (4 * k)) & 15u;
    sb[which][f][k] = b;
  }
  for (int t = threadIdx.x; t < kFMax * Jm; t += blockDim.x)
    sdg[t] = (a.prev_nf > 0 && t < a.prev_nf * Jm) ? a.prev_dg[t] : 0.0;
  int offs[M > 0 ? M : 1];
  int tot = 0;
#pragma unroll
  for (int k = 0; k < M; ++k) {
    offs[k] = tot;
    tot += a.m.J[k];
  }
  double* st = smem + (size_t)warp * (tot * 32 + 16 * kXld);
  double* X = st + tot * 32;
  for (int t = lane; t < 16 * kXld; t += 32) X[t] = 0.0;
  __syncthreads();
  const uint32_t ci = blockIdx.x * kPassWarps + warp;
  if (ci >= a.csf.nchunks) return;
  const Chunk ch = a.csf.chunks[ci];

  // q_f = sum_c A_m[s, c] dg_prev[f][c]
  const double* arow = a.m.factor[M] + (size_t)ch.row * a.m.ld[M];
  if (lane < kFMax) {
    double t = 0.0;
    if (lane < a.prev_nf)
      for (int c = 0; c < Jm; ++c) t = fma(__ldg(arow + c), sdg[lane * Jm + c], t);
    sq_q[warp][lane] = t;
  }
  __syncwarp();

  double d[3][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
  double sq = 0.0;
  const int nf = a.cur_nf;
  const bool acc = a.kind != 2 && nf > 0;

  for (uint32_t base = ch.beg; base < ch.end; base += 32) {
    const uint32_t pos = base + lane;
    const bool valid = pos < ch.end;
    double r = 0.0;
    if (valid) {
      uint32_t idx[M > 0 ? M : 1];
#pragma unroll
      for (int k = 0; k < M; ++k) idx[k] = __ldg(a.csf.oc[k] + pos);
      r = a.r[pos];
#pragma unroll
      for (int k = 0; k < M; ++k) {
        const double* row = a.m.factor[k] + (size_t)idx[k] * a.m.ld[k];
        const int Jk = a.m.J[k];
#pragma unroll
        for (int b = 0; b < VEST_MAXJ; b += 2) {
          if (b < Jk) {
            const double2 v = __ldg(reinterpret_cast<const double2*>(row + b));
            st[(offs[k] + b) * 32 + lane] = v.x;
            if (b + 1 < Jk) st[(offs[k] + b + 1) * 32 + lane] = v.y;
          }
        }
      }
    }
    __syncwarp();
    if (valid && a.prev_nf > 0) {
      double t = 0.0;
#pragma unroll
      for (int f = 0; f < kFMax; ++f) {
        if (f < a.prev_nf) {
          double s = 1.0;
#pragma unroll
          for (int k = 0; k < M; ++k) s *= st[(offs[k] + sb[0][f][k]) * 32 + lane];
          t = fma(s, sq_q[warp][f], t);
        }
      }
      r -= t;
      if (a.kind != 1) a.r[pos] = r;
    }
    if (a.kind == 2) {
      sq = fma(r, r, sq);
      __syncwarp();
      continue;
    }
    if (acc) {
#pragma unroll
      for (int f = 0; f < kFMax; ++f) {
        if (f < nf) {
          double v = 0.0;
          if (valid) {
            v = 1.0;
#pragma unroll
            for (int k = 0; k < M; ++k) v *= st[(offs[k] + sb[1][f][k]) * 32 + lane];
          }
          X[f * kXld + lane] = v;
        }
      }
      X[15 * kXld + lane] = valid ? r : 0.0;
      __syncwarp();
      gram_dmma<16>(X, d, lane);
    }
    __syncwarp();
  }

  if (a.kind == 2) {
    sq = warp_sum(sq);
    if (lane == 0) a.chunk_sq[ci] = sq;
    return;
  }
  if (!acc) return;
  double* out = a.stats + (size_t)ci * a.stride;
  const int NS = nf * (nf + 1) / 2;
#pragma unroll
  for (int t = 0; t < 3; ++t) {
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      int row, col;
      gram_coord(t, i, lane, row, col);
      const double v = d[t][i];
      if (a.kind == 0) {
        if (row <= col && col < nf) out[row * nf - row * (row - 1) / 2 + (col - row)] = v;
        else if (col == 15 && row < nf) out[NS + row] = v;
      } else {
        if (col == 15 && row < nf) out[row] = v;
        else if (row == col && row < nf) out[nf + row] = v;
      }
    }
  }
}

// T[pS][pA] = sum_chunks S[pS] * (a_c a_c')[pA], C[f][c] = sum R[f] a_c
// (kind 0), or C = sum R a_c, D = sum D a_c^2 (kind 1).  Each CTA covers a
// contiguous range of chunks and writes its partial sums; k_colsum adds the
// partials in CTA order (deterministic).
struct CoreGemmArgs {
  const double* stats;
  int stride;
  const Chunk* chunks;
  uint32_t nchunks;
  const double* A;  // factor of the last mode
  int ld, Jm, nf, kind;
  int NS, NAm, nT, nout;
  double* partial;
};

constexpr int kGemmThreads = 256;
constexpr int kGemmBatch = 16;
constexpr int kTileMax = 2;  // 4x4 tiles per thread

__global__ void __launch_bounds__(kGemmThreads) k_core_gemm(CoreGemmArgs a) {
  extern __shared__ double sm[];
  const int NSp = (a.NS + 3) & ~3, NAp = (a.NAm + 3) & ~3;
  double* sS = sm;                                  // [batch][NSp]
  double* sA = sS + kGemmBatch * NSp;               // [batch][NAp]
  double* sR = sA + kGemmBatch * NAp;               // [batch][nf] (R) and [batch][nf] (D)
  double* sa = sR + kGemmBatch * 2 * kFMax;         // [batch][Jm]
  const uint32_t per = (a.nchunks + gridDim.x - 1) / gridDim.x;
  const uint32_t c0 = blockIdx.x * per;
  const uint32_t c1 = min(a.nchunks, c0 + per);
  const int tilesS = NSp / 4, tilesA = NAp / 4;
  const int ntiles = a.kind == 0 ? tilesS * tilesA : 0;
  double acc[kTileMax][16];
#pragma unroll
  for (int k = 0; k < kTileMax; ++k)
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[k][i] = 0.0;
  double accC = 0.0, accD = 0.0;
  const int nfj = a.nf * a.Jm;
  for (uint32_t cb = c0; cb < c1; cb += kGemmBatch) {
    const int nb = min((uint32_t)kGemmBatch, c1 - cb);
    __syncthreads();
    // stage the batch
    for (int t = threadIdx.x; t < kGemmBatch * NSp; t += blockDim.x) {
      const int b = t / NSp, p = t % NSp;
      double v = 0.0;
      if (b < nb && a.kind == 0 && p < a.NS) v = a.stats[(size_t)(cb + b) * a.stride + p];
      sS[t] = v;
    }
    for (int t = threadIdx.x; t < kGemmBatch * 2 * kFMax; t += blockDim.x) {
      const int b = t / (2 * kFMax), p = t % (2 * kFMax);
      double v = 0.0;
      if (b < nb) {
        if (a.kind == 0) {
          if (p < a.nf) v = a.stats[(size_t)(cb + b) * a.stride + a.NS + p];
        } else if (p < 2 * a.nf) {
          v = a.stats[(size_t)(cb + b) * a.stride + p];
        }
      }
      sR[t] = v;
    }
    for (int t = threadIdx.x; t < kGemmBatch * a.Jm; t += blockDim.x) {
      const int b = t / a.Jm, c = t % a.Jm;
      sa[t] = b < nb ? __ldg(a.A + (size_t)a.chunks[cb + b].row * a.ld + c) : 0.0;
    }
    __syncthreads();
    for (int t = threadIdx.x; t < kGemmBatch * NAp; t += blockDim.x) {
      const int b = t / NAp, p = t % NAp;
      double v = 0.0;
      if (p < a.NAm) {
        int c = 0, rem = p;
        while (rem >= a.Jm - c) {
          rem -= a.Jm - c;
          ++c;
        }
        v = sa[b * a.Jm + c] * sa[b * a.Jm + c + rem];
      }
      sA[t] = v;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kTileMax; ++k) {
      const int tile = threadIdx.x + k * blockDim.x;
      if (tile < ntiles) {
        const int ts = tile / tilesA, ta = tile % tilesA;
        for (int b = 0; b < kGemmBatch; ++b) {
          const double4 sv = *reinterpret_cast<const double4*>(sS + b * NSp + 4 * ts);
          const double4 av = *reinterpret_cast<const double4*>(sA + b * NAp + 4 * ta);
          const double s4[4] = {sv.x, sv.y, sv.z, sv.w};
          const double a4[4] = {av.x, av.y, av.z, av.w};
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[k][i * 4 + j] = fma(s4[i], a4[j], acc[k][i * 4 + j]);
        }
      }
    }
    if (threadIdx.x < nfj) {
      const int f = threadIdx.x / a.Jm, c = threadIdx.x % a.Jm;
      for (int b = 0; b < kGemmBatch; ++b) {
        const double av = sa[b * a.Jm + c];
        if (a.kind == 0) {
          accC = fma(sR[b * 2 * kFMax + f], av, accC);
        } else {
          accC = fma(sR[b * 2 * kFMax + f], av, accC);
          accD = fma(sR[b * 2 * kFMax + a.nf + f], av * av, accD);
        }
      }
    }
  }
  double* out = a.partial + (size_t)blockIdx.x * a.nout;
#pragma unroll
  for (int k = 0; k < kTileMax; ++k) {
    const int tile = threadIdx.x + k * blockDim.x;
    if (tile < ntiles) {
      const int ts = tile / tilesA, ta = tile % tilesA;
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int ps = 4 * ts + i, pa = 4 * ta + j;
          if (ps < a.NS && pa < a.NAm) out[ps * a.NAm + pa] = acc[k][i * 4 + j];
        }
    }
  }
  if (threadIdx.x < nfj) {
    out[a.nT + threadIdx.x] = accC;
    if (a.kind == 1) out[a.nT + nfj + threadIdx.x] = accD;
  }
}

__global__ void k_colsum(const double* partial, int nparts, int n, double* out) {
  const int o = blockIdx.x * blockDim.x + threadIdx.x;
  if (o >= n) return;
  double s = 0.0;
  for (int p = 0; p < nparts; ++p) s += partial[(size_t)p * n + o];
  out[o] = s;
}

__device__ __forceinline__ int tri(int i, int j, int n) {  // i <= j
  return i * n - i * (i - 1) / 2 + (j - i);
}

// The same block GEMM on the FP64 tensor cores.  With L = the chunk
// statistics row ([S | R] or [R | D], K = chunks) and Rt = the chunk's
// last-mode products ([a a^T (packed) | a] or [a | a o a]), the CTA computes
// its slice of L^T Rt with DMMA m8n8k4 (8x8 output tiles, 4 chunks per
// k-step); k_gemm_reduce then sums the CTA partials in fixed order and maps
// the needed blocks to [T | C] or [C | D].  Cross blocks (S^T a, R^T a a^T)
// are computed and discarded -- cheaper than splitting the operand staging.
struct GemmTcArgs {
  const double* stats;
  int stride;
  const Chunk* chunks;
  uint32_t nchunks;
  const double* A;
  int ld, Jm, nf, kind;
  int LW, RW, MT, NT;
  double* partial;  // [gridDim.x][MT*NT][64]
};

constexpr int kTcWarps = 8;
constexpr int kTcTilesPerWarp = 14;
constexpr int kTcLPer = 18;
constexpr int kTcLd = 36;  // == 4 mod 16: conflict-free fragment loads

__global__ void __launch_bounds__(kTcWarps * 32) k_core_gemm_tc(GemmTcArgs a) {
  extern __shared__ double sm[];
  double* Lt = sm;                           // [MT*8][kTcLd]
  double* Rt = Lt + a.MT * 8 * kTcLd;        // [NT*8][kTcLd]
  double* sa = Rt + a.NT * 8 * kTcLd;        // [32][Jm]
  int* rmap = reinterpret_cast<int*>(sa + 32 * a.Jm);  // Rt column -> (c, c') packed
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int col = threadIdx.x; col < a.NT * 8; col += blockDim.x) {
    int v = -1;
    if (col < a.RW) {
      const int NAm0 = a.Jm * (a.Jm + 1) / 2;
      if (a.kind == 0 && col < NAm0) {
        int c = 0, rem = col;
        while (rem >= a.Jm - c) {
          rem -= a.Jm - c;
          ++c;
        }
        v = (c << 8) | (c + rem);
      } else if (a.kind == 0) {
        v = (1 << 16) | (col - NAm0);  // plain a_c
      } else {
        v = col < a.Jm ? ((1 << 16) | col) : ((2 << 16) | (col - a.Jm));  // a_c or a_c^2
      }
    }
    rmap[col] = v;
  }
  const int g = lane >> 2, tq = lane & 3;
  const int ntiles = a.MT * a.NT;
  const uint32_t per = ((a.nchunks + gridDim.x - 1) / gridDim.x + 31) & ~31u;
  const uint32_t c0 = blockIdx.x * per;
  const uint32_t c1 = min(a.nchunks, c0 + per);
  double acc[kTcTilesPerWarp][2];
#pragma unroll
  for (int i = 0; i < kTcTilesPerWarp; ++i) acc[i][0] = acc[i][1] = 0.0;
  const int Jm = a.Jm;
  const int LWp = a.MT * 8;
  // software pipeline: the next batch's statistics rows and last-mode factor
  // rows are loaded into registers while the current batch runs on DMMA
  constexpr int kLPer = kTcLPer, kAPer = 2;  // per-thread staging share (LWp*32 <= kTcLPer*256, 32*Jm <= 512)
  double lv[kLPer], av[kAPer];
  auto prefetch = [&](uint32_t cb) {
    const int nb = (int)min(32u, c1 - cb);
#pragma unroll
    for (int i = 0; i < kLPer; ++i) {
      const int t = threadIdx.x + i * blockDim.x;
      const int k = t / LWp, col = t - k * LWp;
      lv[i] = (t < LWp * 32 && k < nb && col < a.LW) ? a.stats[(size_t)(cb + k) * a.stride + col] : 0.0;
    }
#pragma unroll
    for (int i = 0; i < kAPer; ++i) {
      const int t = threadIdx.x + i * blockDim.x;
      const int k = t / Jm, c = t - (t / Jm) * Jm;
      av[i] = (t < 32 * Jm && k < nb) ? __ldg(a.A + (size_t)a.chunks[cb + k].row * a.ld + c) : 0.0;
    }
  };
  if (c0 < c1) prefetch(c0);
  for (uint32_t cb = c0; cb < c1; cb += 32) {
    __syncthreads();
#pragma unroll
    for (int i = 0; i < kLPer; ++i) {
      const int t = threadIdx.x + i * blockDim.x;
      if (t < LWp * 32) {
        const int k = t / LWp, col = t - k * LWp;
        Lt[col * kTcLd + k] = lv[i];
      }
    }
#pragma unroll
    for (int i = 0; i < kAPer; ++i) {
      const int t = threadIdx.x + i * blockDim.x;
      if (t < 32 * Jm) sa[t] = av[i];
    }
    __syncthreads();
    for (int t = threadIdx.x; t < a.NT * 8 * 32; t += blockDim.x) {
      const int col = t >> 5, k = t & 31;
      const int mp = rmap[col];
      double v = 0.0;
      if (mp >= 0) {
        const double* ak = sa + k * Jm;
        const int kind = mp >> 16;
        if (kind == 0) v = ak[(mp >> 8) & 255] * ak[mp & 255];
        else if (kind == 1) v = ak[mp & 255];
        else v = ak[mp & 255] * ak[mp & 255];
      }
      Rt[col * kTcLd + k] = v;
    }
    __syncthreads();
    if (cb + 32 < c1) prefetch(cb + 32);
#pragma unroll
    for (int i = 0; i < kTcTilesPerWarp; ++i) {
      const int tile = warp + kTcWarps * i;
      if (tile < ntiles) {
        const int mt = tile / a.NT, nt = tile % a.NT;
        const double* la = Lt + (8 * mt + g) * kTcLd + tq;
        const double* rb = Rt + (8 * nt + g) * kTcLd + tq;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) dmma884(acc[i][0], acc[i][1], la[4 * kk], rb[4 * kk]);
      }
    }
  }
  double* out = a.partial + (size_t)blockIdx.x * ntiles * 64;
#pragma unroll
  for (int i = 0; i < kTcTilesPerWarp; ++i) {
    const int tile = warp + kTcWarps * i;
    if (tile < ntiles) {
      out[tile * 64 + lane * 2] = acc[i][0];
      out[tile * 64 + lane * 2 + 1] = acc[i][1];
    }
  }
}

// raw[j] = sum over a group of CTA partials (fixed order); grid.y = groups
__global__ void k_gemm_reduce1(const double* partial, int nparts, int n, int groups, double* raw) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int per = (nparts + groups - 1) / groups;
  const int p0 = blockIdx.y * per, p1 = min(nparts, p0 + per);
  double s = 0.0;
  for (int p = p0; p < p1; ++p) s += partial[(size_t)p * n + j];
  raw[(size_t)blockIdx.y * n + j] = s;
}

// out = [T | C] (kind 0) or [C | D] (kind 1) from the group sums of the tile layout
__global__ void k_gemm_reduce2(const double* raw, int n, int groups, int kind, int nf, int Jm, int NT,
                               double* out) {
  const int o = blockIdx.x * blockDim.x + threadIdx.x;
  const int NAm = Jm * (Jm + 1) / 2;
  const int NS = nf * (nf + 1) / 2;
  int row, col, nout;
  if (kind == 0) {
    nout = NS * NAm + nf * Jm;
    if (o >= nout) return;
    if (o < NS * NAm) {
      row = o / NAm;
      col = o % NAm;
    } else {
      row = NS + (o - NS * NAm) / Jm;
      col = NAm + (o - NS * NAm) % Jm;
    }
  } else {
    nout = 2 * nf * Jm;
    if (o >= nout) return;
    const int q = o % (nf * Jm);
    const int hi = o / (nf * Jm);
    row = hi * nf + q / Jm;
    col = hi * Jm + q % Jm;
  }
  const int j = ((row >> 3) * NT + (col >> 3)) * 64 + (row & 7) * 8 + (col & 7);
  double s = 0.0;
  for (int gq = 0; gq < groups; ++gq) s += raw[(size_t)gq * n + j];
  out[o] = s;
}

// Sequential Gauss-Seidel over the block's cells.  The CTA loads [T | C],
// the block's core values and masks into shared memory and expands the dense
// cell Gram H (nq x nq, H_qq' = T[{f,f'}][{c,c'}]); then one warp runs the
// nq sequential steps, each a handful of shared-memory reads plus one
// coalesced row update of the remaining cells' c.
__global__ void __launch_bounds__(256) k_core_solve(const double* tc, int nf, int Jm, const uint32_t* fib,
                                                    double* core, const uint8_t* core_mask, int reg,
                                                    double lambda, double* dg_out) {
  extern __shared__ double sm[];
  const int NAm = Jm * (Jm + 1) / 2;
  const int nT = nf * (nf + 1) / 2 * NAm;
  const int nq = nf * Jm;
  double* H = sm;             // nq x nq
  double* cc = H + nq * nq;   // nq
  double* gv = cc + nq;       // nq
  double* mk = gv + nq;       // nq
  double* rd = mk + nq;       // nq: 1 / (H_qq + lambda) (LF) or 1 / (2 H_qq) (L1)
  for (int t = threadIdx.x; t < nq * nq; t += blockDim.x) {
    const int q = t / nq, q2 = t % nq;
    const int f = q / Jm, c = q % Jm, f2 = q2 / Jm, c2 = q2 % Jm;
    const int ps = f <= f2 ? tri(f, f2, nf) : tri(f2, f, nf);
    const int pa = c <= c2 ? tri(c, c2, Jm) : tri(c2, c, Jm);
    H[t] = tc[ps * NAm + pa];
  }
  for (int q = threadIdx.x; q < nq; q += blockDim.x) {
    cc[q] = tc[nT + q];
    const int lin = (int)fib[q / Jm] * Jm + q % Jm;
    gv[q] = core[lin];
    mk[q] = core_mask[lin] ? 1.0 : 0.0;
    // the denominators do not depend on the sweep state: invert them in
    // parallel, off the sequential critical path
    const int f = q / Jm, c = q % Jm;
    const double hqq = tc[tri(f, f, nf) * NAm + tri(c, c, Jm)];
    const double den = reg == 0 ? hqq + lambda : 2.0 * hqq;
    rd[q] = den != 0.0 ? 1.0 / den : 0.0;
  }
  __syncthreads();
  if (threadIdx.x >= 32) return;
  const int lane = threadIdx.x;
  for (int q = 0; q < nq; ++q) {
    double dg = 0.0;
    if (mk[q] == 0.0) {
      const double hqq = H[q * nq + q];
      const double g_old = gv[q];
      const double num = cc[q] + g_old * hqq;
      const double den = hqq;
      double g_new = g_old;
      const double r = rd[q];
      if (reg == 0) {
        if (den + lambda != 0.0) g_new = num * r;
      } else {
        const double g = -2.0 * num;
        if (2.0 * den != 0.0) g_new = g > lambda ? (lambda - g) * r : (g < -lambda ? -(lambda + g) * r : 0.0);
      }
      if (g_new != g_old) dg = g_new - g_old;
      if (lane == 0) gv[q] = g_new;
    }
    if (lane == 0) dg_out[q] = dg;
    if (dg != 0.0) {
      const double* hr = H + q * nq;
      for (int q2 = q + 1 + lane; q2 < nq; q2 += 32) cc[q2] = fma(-dg, hr[q2], cc[q2]);
    }
    __syncwarp();
  }
  for (int q = lane; q < nq; q += 32)
    if (mk[q] == 0.0) core[(int)fib[q / Jm] * Jm + q % Jm] = gv[q];
}

// Closed-form core responsibility (pruning.hpp:98-134): zeroing cell beta
// shifts every residual by g p_beta, so
//   acc = sum (r + g p)^2 = S + g (2 c + g d),  c = sum r p, d = sum p^2
// resp = (sqrt(acc)/||x|| - re)/re; masked cells keep +inf.
__global__ void k_core_resp_final(const double* cd, int nf, int Jm, const uint32_t* fib,
                                  const double* core, const uint8_t* core_mask, double S,
                                  double x_norm, double re, double* resp) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nf * Jm) return;
  const int f = q / Jm, c = q % Jm;
  const int lin = (int)fib[f] * Jm + c;
  if (core_mask[lin]) return;
  const double g = core[lin];
  const double cq = cd[q], dq = cd[nf * Jm + q];
  double acc = S + g * (2.0 * cq + g * dq);
  if (acc < 0.0) acc = 0.0;
  resp[lin] = (sqrt(acc) / x_norm - re) / re;
}

__global__ void k_fill(double* p, size_t n, double v) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    p[i] = v;
}

// ---------------------------------------------------------------- host side --
const void* find_core_ops(int N, const int* J);
cudaError_t core_pass_structured(const void* ops, const DevModel& m, const DevCSF& csf, double* r, int prev_p,
                                 const double* prev_dg, int cur_p, int kind, double* stats, int stride,
                                 double* chunk_sq, const double* U, const double* W, uint64_t wstride,
                                 cudaStream_t s);
cudaError_t core_pack_structured(const void* ops, const DevModel& m, const DevCSF& csf, uint64_t p0, uint64_t p1,
                                 double* U, double* W, uint64_t wstride, cudaStream_t s);

void core_sweep_sall(Ctx& c, const void* ops, int reg, double lambda, const std::vector<int>& prefixes,
                     const std::vector<int>& starts);
const void* find_core_all_ops(int N, const int* J);

namespace {

// VEST_CORE_BLOCK_PASSES=1: the per-block statistics passes (packed operands,
// one GEMM per block) instead of the all-prefix sweep -- kept for A/B timing.
bool legacy_block_passes() {
  static const bool v = [] {
    const char* e = getenv("VEST_CORE_BLOCK_PASSES");
    return e && e[0] == '1';
  }();
  return v;
}

struct Blocks {
  std::vector<uint32_t> fib;    // fibers of all blocks, row-major order
  std::vector<int> start, len;  // block ranges into fib
  std::vector<int> prefix;      // structured plan: the block's prefix p
};

// General plan: runs of F consecutive live fibers.
Blocks plan_blocks(const Ctx& c, int F) {
  Blocks b;
  const int Jm = c.ranks[c.N - 1];
  const int P = c.G / Jm;
  for (int p = 0; p < P; ++p) {
    bool live = false;
    for (int q = 0; q < Jm && !live; ++q) live = !c.h_core_mask[(size_t)p * Jm + q];
    if (live) b.fib.push_back(p);
  }
  for (int s = 0; s < (int)b.fib.size(); s += F) {
    b.start.push_back(s);
    b.len.push_back(std::min(F, (int)b.fib.size() - s));
  }
  return b;
}

// Structured plan (compile-time ranks): one block per prefix over modes
// 0..N-3 that has an unmasked cell; all J_{N-2} fibers of the prefix.
Blocks plan_structured(const Ctx& c) {
  Blocks b;
  const int Jm = c.ranks[c.N - 1], F = c.ranks[c.N - 2];
  const int P = c.G / (F * Jm);
  for (int p = 0; p < P; ++p) {
    bool live = false;
    for (int q = 0; q < F * Jm && !live; ++q) live = !c.h_core_mask[(size_t)p * F * Jm + q];
    if (!live) continue;
    b.start.push_back((int)b.fib.size());
    b.len.push_back(F);
    b.prefix.push_back(p);
    for (int f = 0; f < F; ++f) b.fib.push_back(p * F + f);
  }
  return b;
}

int pick_block(const Ctx& c) {
  const int Jm = c.ranks[c.N - 1];
  int F = c.core_block > 0 ? std::min(c.core_block, kFMax) : kFMax;
  // keep the block within the solve's shared memory (dense H of (F*Jm)^2) and
  // the tensor-core gemm's staging / tile capacity
  while (F > 1) {
    const int NS = F * (F + 1) / 2, NAm = Jm * (Jm + 1) / 2;
    const int nq = F * Jm;
    const int MT = (NS + F + 7) / 8, NT = (NAm + Jm + 7) / 8;
    const bool solve_ok = (size_t)(nq * nq + 4 * nq) * 8 <= 200 * 1024;
    const bool tc_ok = MT * NT <= kTcWarps * kTcTilesPerWarp && MT * 8 * 32 <= kTcLPer * 256 && 32 * Jm <= 512;
    if (solve_ok && tc_ok) break;
    --F;
  }
  return F;
}

const void* structured_ops(const Ctx& c) {
  if (c.force_generic || c.N < 3 || c.core_block > 0) return nullptr;
  return find_core_ops(c.N, c.ranks);
}

void launch_pass(Ctx& c, const CorePassArgs& a) {
  ProfScope ps(c, kProfCorePass);
  const int M = c.N - 1;
  int tot = 0;
  for (int k = 0; k < M; ++k) tot += c.ranks[k];
  const size_t sm = (size_t)kPassWarps * (tot * 32 + 16 * kXld) * sizeof(double);
  const dim3 grid((a.csf.nchunks + kPassWarps - 1) / kPassWarps);
  if (a.csf.nchunks == 0) return;
#define VEST_PASS(MM)                                                                       \
  case MM:                                                                                  \
    check(cudaFuncSetAttribute(k_core_pass<MM>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                               (int)sm),                                                    \
          "pass smem");                                                                     \
    k_core_pass<MM><<<grid, kPassWarps * 32, sm, c.stream>>>(a);                            \
    break;
  switch (M) {
    VEST_PASS(1)
    VEST_PASS(2)
    VEST_PASS(3)
    VEST_PASS(4)
    VEST_PASS(5)
    VEST_PASS(6)
    VEST_PASS(7)
    default:
      throw ArgError{"unsupported order"};
  }
#undef VEST_PASS
  count_launch();
  check(cudaGetLastError(), "core pass");
}

// One pass of the block schedule: previous block's residual update, then
// the current block's statistics (kind 0/1) or the sum of r^2 (kind 2).
void run_pass(Ctx& c, const void* sops, const Blocks& b, int prev, int cur, int kind, int stride) {
  const int m = c.N - 1;
  if (sops) {
    ProfScope ps(c, kProfCorePass);
    check(core_pass_structured(sops, c.model_view(), c.csf_view(m), c.d_r, prev >= 0 ? b.prefix[prev] : -1,
                               c.d_dg, cur >= 0 ? b.prefix[cur] : -1, kind, c.d_chunk_stats, stride,
                               c.d_chunk_sum, c.d_pack_u, c.d_pack_w, c.nnz, c.stream),
          "core pass (structured)");
    return;
  }
  CorePassArgs a{};
  a.m = c.model_view();
  a.csf = c.csf_view(m);
  a.r = c.d_r;
  a.stats = c.d_chunk_stats;
  a.stride = stride;
  a.chunk_sq = c.d_chunk_sum;
  a.prev_dg = c.d_dg;
  a.kind = kind;
  a.cur_fib = cur >= 0 ? c.d_fibers + b.start[cur] : c.d_fibers;
  a.cur_nf = cur >= 0 ? b.len[cur] : 0;
  a.prev_fib = prev >= 0 ? c.d_fibers + b.start[prev] : c.d_fibers;
  a.prev_nf = prev >= 0 ? b.len[prev] : 0;
  launch_pass(c, a);
}

// (T, C) or (C, D) for one block into c.d_gemm_out; returns nout.
int block_gemm(Ctx& c, int nf, int kind, int stride) {
  const int m = c.N - 1, Jm = c.ranks[m];
  CoreGemmArgs g{};
  g.stats = c.d_chunk_stats;
  g.stride = stride;
  g.chunks = c.modes[m].d_chunks;
  g.nchunks = c.modes[m].nchunks;
  g.A = c.d_factor[m];
  g.ld = c.ld[m];
  g.Jm = Jm;
  g.nf = nf;
  g.kind = kind;
  g.NS = kind == 0 ? nf * (nf + 1) / 2 : 0;
  g.NAm = Jm * (Jm + 1) / 2;
  g.nT = kind == 0 ? g.NS * g.NAm : 0;
  g.nout = g.nT + (kind == 0 ? 1 : 2) * nf * Jm;
  int nblocks = 0;
  cudaDeviceGetAttribute(&nblocks, cudaDevAttrMultiProcessorCount, c.device);
  nblocks = std::max(1, std::min<int>(2 * nblocks, (g.nchunks + kGemmBatch - 1) / kGemmBatch));
  ensure(c, &c.d_gemm_part, &c.gemm_part_cap, (size_t)nblocks * g.nout);
  ensure(c, &c.d_gemm_out, &c.gemm_out_cap, (size_t)g.nout);
  g.partial = c.d_gemm_part;
  ProfScope ps(c, kProfCoreGemm);
  GemmTcArgs t{};
  t.stats = g.stats;
  t.stride = stride;
  t.chunks = g.chunks;
  t.nchunks = g.nchunks;
  t.A = g.A;
  t.ld = g.ld;
  t.Jm = Jm;
  t.nf = nf;
  t.kind = kind;
  t.LW = kind == 0 ? g.NS + nf : 2 * nf;
  t.RW = kind == 0 ? g.NAm + Jm : 2 * Jm;
  t.MT = (t.LW + 7) / 8;
  t.NT = (t.RW + 7) / 8;
  const int ntiles = t.MT * t.NT;
  if (ntiles <= kTcWarps * kTcTilesPerWarp && t.MT * 8 * 32 <= kTcLPer * 256 && 32 * Jm <= 2 * 256) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c.device);
    const int nparts = std::max(1, std::min<int>(2 * sms, (g.nchunks + 31) / 32));
    const int n = ntiles * 64;
    const int groups = 16;
    ensure(c, &c.d_gemm_part, &c.gemm_part_cap, (size_t)nparts * n + (size_t)groups * n);
    t.partial = c.d_gemm_part;
    double* raw = c.d_gemm_part + (size_t)nparts * n;
    const size_t sm = ((size_t)(t.MT + t.NT) * 8 * kTcLd + 32 * Jm) * sizeof(double) + (size_t)t.NT * 8 * sizeof(int);
    check(cudaFuncSetAttribute(k_core_gemm_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm), "gemm smem");
    k_core_gemm_tc<<<nparts, kTcWarps * 32, sm, c.stream>>>(t);
    k_gemm_reduce1<<<dim3((n + 255) / 256, groups), 256, 0, c.stream>>>(t.partial, nparts, n, groups, raw);
    k_gemm_reduce2<<<(g.nout + 255) / 256, 256, 0, c.stream>>>(raw, n, groups, kind, nf, Jm, t.NT, c.d_gemm_out);
    count_launch(3);
    check(cudaGetLastError(), "core gemm (tensor cores)");
    return g.nout;
  }
  const int NSp = (g.NS + 3) & ~3, NAp = (g.NAm + 3) & ~3;
  const size_t sm = (size_t)kGemmBatch * (NSp + NAp + 2 * kFMax + Jm) * sizeof(double);
  check(cudaFuncSetAttribute(k_core_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm), "gemm smem");
  k_core_gemm<<<nblocks, kGemmThreads, sm, c.stream>>>(g);
  k_colsum<<<(g.nout + 255) / 256, 256, 0, c.stream>>>(c.d_gemm_part, nblocks, g.nout, c.d_gemm_out);
  count_launch(2);
  check(cudaGetLastError(), "core gemm");
  return g.nout;
}

void upload_fibers(Ctx& c, const Blocks& b) {
  ensure(c, reinterpret_cast<double**>(&c.d_fibers), &c.fibers_cap, (b.fib.size() + 1) / 2 + 1);
  check(cudaMemcpyAsync(c.d_fibers, b.fib.data(), b.fib.size() * sizeof(uint32_t), cudaMemcpyHostToDevice,
                        c.stream),
        "fibers");
}

// Pack the structured pass operands (U, W) for this context's positions of the
// last mode's CSF (the factors are fixed during the sweep / responsibilities).
void pack_operands(Ctx& c, const void* sops) {
  const int m = c.N - 1, F = c.ranks[c.N - 2];
  const int P = c.G / (F * c.ranks[m]);
  ensure(c, &c.d_pack_u, &c.pack_u_cap, (size_t)c.nnz * F + 1);
  ensure(c, &c.d_pack_w, &c.pack_w_cap, (size_t)c.nnz * P + 1);
  const ModeData& md = c.modes[m];
  const uint64_t p0 = md.h_offsets[c.row_lo[m]], p1 = md.h_offsets[c.row_hi[m]];
  ProfScope ps(c, kProfCorePass);
  check(core_pack_structured(sops, c.model_view(), c.csf_view(m), p0, p1, c.d_pack_u, c.d_pack_w, c.nnz,
                             c.stream),
        "pack operands");
}

}  // namespace

void core_sweep(Ctx& c, int reg, double lambda) {
  const int m = c.N - 1, Jm = c.ranks[m];
  // r = x - B(alpha) for the model after the factor updates
  // (the reference rebuilds its reconstruction cache here, updates.hpp:190-192);
  // already fresh when the last factor mode emitted it
  if (!c.r_fresh) compute_residual(c);
  const void* sops = structured_ops(c);
  const int F = sops ? c.ranks[c.N - 2] : pick_block(c);
  const Blocks b = sops ? plan_structured(c) : plan_blocks(c, F);
  if (b.fib.empty()) return;  // fully pruned core: nothing to update
  upload_fibers(c, b);
  if (sops && !legacy_block_passes()) {
    if (const void* aops = find_core_all_ops(c.N, c.ranks)) {
      core_sweep_sall(c, aops, reg, lambda, b.prefix, b.start);
      return;
    }
  }
  if (sops) pack_operands(c, sops);
  const int stride = F * (F + 1) / 2 + F;
  ensure(c, &c.d_chunk_stats, &c.chunk_stats_cap, (size_t)c.modes[m].nchunks * stride);
  ensure(c, &c.d_dg, &c.dg_cap, (size_t)16 * VEST_MAXJ);
  ensure(c, &c.d_chunk_sum, &c.chunk_sum_cap, c.modes[m].nchunks + 1);
  const int nb = (int)b.start.size();
  for (int bi = 0; bi <= nb; ++bi) {
    const bool last = bi == nb;
    run_pass(c, sops, b, bi - 1, last ? -1 : bi, last ? 2 : 0, stride);
    if (last) break;
    const int nf = b.len[bi];
    const int nout = block_gemm(c, nf, 0, stride);
    comm_allreduce(c, c.d_gemm_out, (uint64_t)nout);  // block statistics over the shards
    ProfScope ps(c, kProfCoreSolve);
    const size_t nq = (size_t)nf * Jm;
    const size_t sm = (nq * nq + 4 * nq) * sizeof(double);
    check(cudaFuncSetAttribute(k_core_solve, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm), "solve smem");
    k_core_solve<<<1, 256, sm, c.stream>>>(c.d_gemm_out, nf, Jm, c.d_fibers + b.start[bi], c.d_core,
                                           c.d_core_mask, reg, lambda, c.d_dg);
    count_launch();
    check(cudaGetLastError(), "core solve");
  }
  c.sum_sq = reduce_chunk_sums(c, c.d_chunk_sum, c.modes[m].nchunks);
  c.re = std::sqrt(c.sum_sq) / c.x_norm;
  c.r_valid = true;
  c.r_fresh = true;
}

void core_responsibilities(Ctx& c) {
  const int m = c.N - 1, Jm = c.ranks[m];
  const size_t G = c.G;
  k_fill<<<64, 256, 0, c.stream>>>(c.d_resp_core, G, INFINITY);
  count_launch();
  if (c.re == 0.0) return;  // perfect fit: everything +inf (pruning.hpp:102-103)
  const void* sops = structured_ops(c);
  const int F = sops ? c.ranks[c.N - 2] : pick_block(c);
  const Blocks b = sops ? plan_structured(c) : plan_blocks(c, F);
  if (b.fib.empty()) return;
  upload_fibers(c, b);
  if (sops) pack_operands(c, sops);
  const int stride = 2 * F;
  ensure(c, &c.d_chunk_stats, &c.chunk_stats_cap, (size_t)c.modes[m].nchunks * stride);
  ensure(c, &c.d_dg, &c.dg_cap, (size_t)16 * VEST_MAXJ);
  for (int bi = 0; bi < (int)b.start.size(); ++bi) {
    run_pass(c, sops, b, -1, bi, 1, stride);
    const int nf = b.len[bi];
    const int nout = block_gemm(c, nf, 1, stride);
    comm_allreduce(c, c.d_gemm_out, (uint64_t)nout);
    k_core_resp_final<<<(nf * Jm + 127) / 128, 128, 0, c.stream>>>(
        c.d_gemm_out, nf, Jm, c.d_fibers + b.start[bi], c.d_core, c.d_core_mask, c.sum_sq, c.x_norm, c.re,
        c.d_resp_core);
    count_launch();
    check(cudaGetLastError(), "core resp");
  }
}

}  // namespace vest
