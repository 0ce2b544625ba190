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
// a small GEMM over the slices (k_core_gemm_tc) produces (T, C), and one
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

constexpr int kFMax = 31;       // fibers per block (31 s-columns + r: a 32-column DMMA Gram)
constexpr int kSolveCells = 160;  // live cells per block (dense Gram of the block in shared memory)
#ifndef VEST_PASS_WARPS
#define VEST_PASS_WARPS 4
#endif
constexpr int kPassWarps = VEST_PASS_WARPS;

// A block's fibers as the pass kernel reads them: the shared-memory stage row
// of each fiber's factor values (compile-time fiber index in the unrolled
// loops -> constant-bank operands).  Fibers are in row-major order, so
// consecutive fibers usually share the prefix beta_0..beta_{m-2}; its product
// w is recomputed only where the prefix changes (newp).
struct FibTab {
  int nf;
  int last[kFMax];                 // stage row of beta_{m-1}(f)
  int pre[kFMax][VEST_MAXN - 2];   // stage rows of beta_k(f), k < m-1
  int newp[kFMax];
};

// Prefix blocks for a compile-time last-fiber rank JL: the block is np <=
// 31 / JL whole prefixes (beta_0..beta_{m-2}) -- all JL fibers of each, the
// masked cells included (the solve skips them) -- so fiber (slot p, b) is
// Gram column p * JL + b at compile time; the lane's A_{m-1} row sits in
// registers and each prefix's product w is formed once.
constexpr int kPreMax = 8;
struct PreTab {
  int nf;
  int np;
  int pre[kPreMax][VEST_MAXN - 2];  // stage offsets of beta_k(p), k < m-1
};
union BlockTab {
  FibTab fib;
  PreTab pre;  // nf is the common first member
};

struct CorePassArgs {
  DevModel m;
  DevCSF csf;  // mode N-1
  double* r;
  const double* prev_dg;  // [prev.nf][Jm]
  BlockTab prev, cur;
  int kind;  // 0 sweep (S, R), 1 responsibility (R, D), 2 final (apply prev, sum r^2)
  int soff[VEST_MAXN];  // per-lane stage offset of mode k's factor row (k < m, even)
  int rslot;            // per-lane stage slot of r
  int prefix_plan;      // blocks are whole prefixes (PreTab)
  int ldr;              // per-lane stage stride (== 2 mod 4: 16-byte copies, 2-way read conflicts)
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

// Gram of the NT*8 staged columns of 32 entries on DMMA: upper tiles (I <= J)
// of X^T X, tile t in row-major order over I <= J.
template <int NT>
__device__ __forceinline__ void gram_nt(const double* X, double (&d)[NT * (NT + 1) / 2][2], int lane) {
  const int g = lane >> 2, tq = lane & 3;
#pragma unroll
  for (int kk = 0; kk < 8; ++kk) {
    const int e = 4 * kk + tq;
    double f[NT];
#pragma unroll
    for (int i = 0; i < NT; ++i) f[i] = X[(8 * i + g) * kXld + e];
    int t = 0;
#pragma unroll
    for (int I = 0; I < NT; ++I)
#pragma unroll
      for (int J = I; J < NT; ++J) {
        dmma884(d[t][0], d[t][1], f[I], f[J]);
        ++t;
      }
  }
}

// fiber product s_f = prod_{k<m} A_k[i_k, beta_k(f)] from the lane's staged
// rows (st = the lane's stage row), reusing the running prefix product w
template <int M>
__device__ __forceinline__ double fiber_product(const FibTab& T, int f, const double* st, double& w) {
  if constexpr (M > 1) {
    if (T.newp[f]) {
      w = st[T.pre[f][0]];
#pragma unroll
      for (int k = 1; k < M - 1; ++k) w *= st[T.pre[f][k]];
    }
    return w * st[T.last[f]];
  } else {
    return st[T.last[f]];
  }
}

// prefix product w_p = prod_{k<m-1} A_k[i_k, beta_k(p)] (1 for m = 1)
template <int M>
__device__ __forceinline__ double prefix_weight(const PreTab& T, int pi, const double* st) {
  double w = 1.0;
  if constexpr (M > 1) {
    w = st[T.pre[pi][0]];
#pragma unroll
    for (int k = 1; k < M - 1; ++k) w *= st[T.pre[pi][k]];
  }
  return w;
}

__device__ __forceinline__ uint32_t cp_smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async8_s(uint32_t smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async16_s(uint32_t smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(smem), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int K>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(K) : "memory"); }

// Persistent, one warp per chunk of a last-mode slice at a time (runtime
// ranks / sparse fiber lists).  Rounds of 32 entries (one per lane): the rows
// of modes < m and r are copied global -> shared by cp.async one round ahead
// (coordinates two rounds ahead) into a per-lane, odd-strided stage, so the
// gathers of the next round overlap this round's arithmetic.  Per entry: the
// previous block's residual update and the current block's fiber products
// read the stage; the (s_0..s_{nf-1}, r) vectors are staged transposed (r in
// the last column) and S = sum s s^T, R = sum s r are accumulated on the FP64
// tensor cores (DMMA).  NT = 2/3/4 column tiles (<= 15/23/31 fibers).
template <int M, int NT, int JL, int JALL>
__global__ void __launch_bounds__(kPassWarps * 32) k_core_pass(const __grid_constant__ CorePassArgs a) {
  extern __shared__ __align__(16) double smem[];
  __shared__ double sq_q[kPassWarps][kFMax];
  constexpr int NC = NT * 8;
  constexpr int NTT = NT * (NT + 1) / 2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int Jm = a.m.J[M];
  const int ldr = a.ldr;
  double* const stage = smem + (size_t)warp * (2 * 32 * ldr + NC * kXld);  // [2][32][ldr]
  double* const X = stage + 2 * 32 * ldr;
  for (int t = lane; t < NC * kXld; t += 32) X[t] = 0.0;  // columns >= nf stay zero
  const int nf = a.cur.fib.nf;
  const int pnf = a.prev.fib.nf;
  const bool acc = a.kind != 2 && nf > 0;
  const uint32_t wstride = gridDim.x * kPassWarps;

  struct Cur {
    uint32_t ci, beg, end, base, row;
  };
  auto first = [&](uint32_t ci) {
    Cur c{ci, 0, 0, 0, 0};
    if (ci < a.csf.nchunks) {
      const Chunk ch = a.csf.chunks[ci];
      c.beg = ch.beg;
      c.end = ch.end;
      c.base = ch.beg;
      c.row = ch.row;
    }
    return c;
  };
  auto next = [&](const Cur& c) {
    if (c.base + 32 < c.end) return Cur{c.ci, c.beg, c.end, c.base + 32, c.row};
    return first(c.ci + wstride);
  };
  auto coords = [&](const Cur& c, uint32_t (&idx)[M]) {
    const bool v = c.ci < a.csf.nchunks && c.base + lane < c.end;
#pragma unroll
    for (int k = 0; k < M; ++k) idx[k] = v ? __ldg(a.csf.oc[k] + c.base + lane) : 0u;
  };
  const uint32_t sbase = cp_smem_u32(stage);
  auto issue = [&](const Cur& c, int b, const uint32_t (&idx)[M]) {
    if (c.ci < a.csf.nchunks && c.base + lane < c.end) {
      const uint32_t st = sbase + (uint32_t)((b * 32 + lane) * ldr) * 8u;
#pragma unroll
      for (int k = 0; k < M; ++k) {
        // rows are ld_k (even) doubles: 16-byte copies, the padding included
        const int ldk = JALL > 0 ? ((JALL + 1) & ~1) : a.m.ld[k];
        const double* row = a.m.factor[k] + (size_t)idx[k] * ldk;
#pragma unroll
        for (int t = 0; t < (JALL > 0 ? (JALL + 1) / 2 : VEST_MAXJ / 2); ++t)
          if (JALL > 0 || 2 * t < ldk) cp_async16_s(st + (uint32_t)(a.soff[k] + 2 * t) * 8u, row + 2 * t);
      }
      cp_async8_s(st + (uint32_t)a.rslot * 8u, a.r + c.base + lane);
    }
    cp_async_commit();
  };
  // chunk prologue: q_f = sum_c A_m[s, c] dg_prev[f][c]
  auto prologue = [&](const Cur& c) {
    if (lane < kFMax) {
      double t = 0.0;
      if (lane < pnf) {
        const double* arow = a.m.factor[M] + (size_t)c.row * a.m.ld[M];
        for (int q = 0; q < Jm; ++q) t = fma(__ldg(arow + q), __ldg(a.prev_dg + lane * Jm + q), t);
      }
      sq_q[warp][lane] = t;
    }
    __syncwarp();
  };

  Cur cur = first(blockIdx.x * kPassWarps + warp);
  if (cur.ci >= a.csf.nchunks) return;
  {
    uint32_t i0[M];
    coords(cur, i0);
    issue(cur, 0, i0);
  }
  Cur nxt = next(cur);
  uint32_t inx[M];
  coords(nxt, inx);
  prologue(cur);

  double d[NTT][2];
#pragma unroll
  for (int t = 0; t < NTT; ++t) d[t][0] = d[t][1] = 0.0;
  double sq = 0.0;
  int buf = 0;
  while (true) {
    // next round's gathers into the other buffer, the round after's coordinates
    issue(nxt, buf ^ 1, inx);
    const Cur nn = next(nxt);
    coords(nn, inx);
    cp_async_wait<1>();
    __syncwarp();
    const double* st = stage + (size_t)(buf * 32 + lane) * ldr;
    const uint32_t pos = cur.base + lane;
    const bool valid = pos < cur.end;
    double r = valid ? st[a.rslot] : 0.0;
    double ul[JL > 0 ? JL : 1];
    if constexpr (JL > 0) {
#pragma unroll
      for (int b = 0; b < JL; ++b) ul[b] = valid ? st[a.soff[M - 1] + b] : 0.0;  // stale stage: no NaN
    }
    if (valid && pnf > 0) {
      double t = 0.0;
      if constexpr (JL > 0) {
#pragma unroll
        for (int pi = 0; pi < kFMax / JL; ++pi) {
          if (pi < a.prev.pre.np) {
            const double w = prefix_weight<M>(a.prev.pre, pi, st);
            double s = ul[0] * sq_q[warp][pi * JL];
#pragma unroll
            for (int b = 1; b < JL; ++b) s = fma(ul[b], sq_q[warp][pi * JL + b], s);
            t = fma(w, s, t);
          }
        }
      } else {
        double w = 1.0;
#pragma unroll
        for (int f = 0; f < kFMax; ++f) {
          if (f < pnf) t = fma(fiber_product<M>(a.prev.fib, f, st, w), sq_q[warp][f], t);
        }
      }
      r -= t;
      if (a.kind != 1) a.r[pos] = r;
    }
    if (a.kind == 2) {
      sq = fma(r, r, sq);
    } else if (acc) {
      if constexpr (JL > 0) {
#pragma unroll
        for (int pi = 0; pi < kFMax / JL; ++pi) {
          if (pi < a.cur.pre.np) {
            const double w = valid ? prefix_weight<M>(a.cur.pre, pi, st) : 0.0;
#pragma unroll
            for (int b = 0; b < JL; ++b) X[(pi * JL + b) * kXld + lane] = w * ul[b];
          }
        }
      } else {
        double w = 1.0;
#pragma unroll
        for (int f = 0; f < NC - 1 && f < kFMax; ++f) {
          if (f < nf) {
            const double v = fiber_product<M>(a.cur.fib, f, st, w);
            X[f * kXld + lane] = valid ? v : 0.0;
          }
        }
      }
      X[(NC - 1) * kXld + lane] = valid ? r : 0.0;
      __syncwarp();
      gram_nt<NT>(X, d, lane);
    }
    __syncwarp();

    if (nxt.ci != cur.ci) {  // chunk epilogue
      const uint32_t ci = cur.ci;
      if (a.kind == 2) {
        sq = warp_sum(sq);
        if (lane == 0) a.chunk_sq[ci] = sq;
        sq = 0.0;
      } else if (acc) {
        double* out = a.stats + (size_t)ci * a.stride;
        const int NS = nf * (nf + 1) / 2;
        const int g = lane >> 2, tq = lane & 3;
        int t = 0;
#pragma unroll
        for (int I = 0; I < NT; ++I) {
#pragma unroll
          for (int J = I; J < NT; ++J) {
#pragma unroll
            for (int i = 0; i < 2; ++i) {
              const int row = 8 * I + g, col = 8 * J + 2 * tq + i;
              const double v = d[t][i];
              if (a.kind == 0) {
                if (row <= col && col < nf) out[row * nf - row * (row - 1) / 2 + (col - row)] = v;
                else if (col == NC - 1 && row < nf) out[NS + row] = v;
              } else {
                if (col == NC - 1 && row < nf) out[row] = v;
                else if (row == col && row < nf) out[nf + row] = v;
              }
              d[t][i] = 0.0;
            }
            ++t;
          }
        }
      }
      if (nxt.ci >= a.csf.nchunks) break;
      prologue(nxt);
    }
    cur = nxt;
    nxt = nn;
    buf ^= 1;
  }
  cp_async_wait<0>();
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
  int MTy;          // row tiles per CTA row (blockIdx.y): large blocks split the L rows
  double* partial;  // [gridDim.x][MT*NT][64]
};

constexpr int kTcWarps = 8;
constexpr int kTcTilesPerWarp = 14;
constexpr int kTcLPer = 18;
constexpr int kTcLd = 36;  // == 4 mod 16: conflict-free fragment loads

__global__ void __launch_bounds__(kTcWarps * 32) k_core_gemm_tc(GemmTcArgs a) {
  extern __shared__ double sm[];
  double* Lt = sm;                           // [MT*8][kTcLd]
  double* Rt = Lt + a.MTy * 8 * kTcLd;       // [NT*8][kTcLd]
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
  const int mt0 = blockIdx.y * a.MTy;
  const int MTl = min(a.MTy, a.MT - mt0);
  const int ntiles = MTl * a.NT;
  const uint32_t per = ((a.nchunks + gridDim.x - 1) / gridDim.x + 31) & ~31u;
  const uint32_t c0 = blockIdx.x * per;
  const uint32_t c1 = min(a.nchunks, c0 + per);
  double acc[kTcTilesPerWarp][2];
#pragma unroll
  for (int i = 0; i < kTcTilesPerWarp; ++i) acc[i][0] = acc[i][1] = 0.0;
  const int Jm = a.Jm;
  const int LWp = MTl * 8;
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
      lv[i] = (t < LWp * 32 && k < nb && mt0 * 8 + col < a.LW)
                  ? a.stats[(size_t)(cb + k) * a.stride + mt0 * 8 + col]
                  : 0.0;
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
  double* out = a.partial + (size_t)blockIdx.x * a.MT * a.NT * 64 + (size_t)mt0 * a.NT * 64;
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

// Live-cell block Gram without the dense GEMM: for a sparse block (config 4:
// ~43 live cells of 31 fibers x 8) the GEMM over [S | R] x [a a^T | a] forms
// every (fiber pair, c pair) -- ~20x the entries the solve reads.  Each thread
// owns up to kHsPer entries of H (upper triangle over the live cells) or C,
// tab[e] = s-index | a-index << 16, the a-index naming one of the chunk's
// weights aa = [a_c a_c' (c <= c', row-major triangle) | a_c] (the C entries,
// R x a_c) that the CTA forms once per staged chunk, and accumulates s * aa
// over its CTA's chunks in order (batches of chunk statistics rows staged in
// shared memory); CTA partials are summed in a fixed order afterwards
// (deterministic).
constexpr int kHsBatch = 8, kHsPer = 8, kHsThreads = 256;
// shared-memory row pitches are compile-time (the widest block, the largest
// rank), so the accumulation loop's addresses are register + immediate
constexpr int kHsWP = (kFMax * (kFMax + 1) / 2 + kFMax + 3) & ~3;
constexpr int kHsAWP = VEST_MAXJ * (VEST_MAXJ + 1) / 2 + VEST_MAXJ;
__device__ __forceinline__ void hs_cp8(double* dst, const double* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void hs_cp16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}

template <class T>
__global__ void __launch_bounds__(kHsThreads) k_core_hsample(const T* __restrict__ stats, int stride, int width,
                                                             const Chunk* __restrict__ chunks, uint32_t nchunks,
                                                             const double* __restrict__ A, int ld, int Jm,
                                                             const uint32_t* __restrict__ tab, int E,
                                                             double* __restrict__ partial) {
  extern __shared__ double hs_raw[];
  // two batch buffers [kHsBatch][width] (T) + [kHsBatch][Jm] (double): the next
  // batch's rows are copied by cp.async while this batch is accumulated;
  // statistics rows are staged in 16-byte pieces (stride and the smem row
  // width are multiples of 16 bytes)
  constexpr int V = 16 / sizeof(T);
  constexpr int wpad = kHsWP;
  constexpr int bufw = kHsBatch * wpad;  // T elements per statistics buffer
  const uint32_t per = (nchunks + gridDim.x - 1) / gridDim.x;
  const uint32_t c0 = blockIdx.x * per, c1 = min(nchunks, c0 + per);
  uint32_t my[kHsPer];
  double acc[kHsPer];
#pragma unroll
  for (int j = 0; j < kHsPer; ++j) {
    const int e = threadIdx.x + kHsThreads * j;
    my[j] = e < E ? __ldg(tab + e) : 0xffffffffu;
    acc[j] = 0.0;
  }
  T* const sstat = reinterpret_cast<T*>(hs_raw);                     // [2][kHsBatch][wpad]
  double* const sarow = reinterpret_cast<double*>(sstat + 2 * bufw);  // [2][kHsBatch][Jm]
  const int AW = Jm * (Jm + 1) / 2 + Jm;
  double* const saa = sarow + 2 * kHsBatch * Jm;                       // [kHsBatch][kHsAWP]
  auto stage = [&](uint32_t cb, int buf) {
    const int nb = (int)min((uint32_t)kHsBatch, c1 - cb);
    T* ss = sstat + buf * bufw;
    double* sa = sarow + buf * kHsBatch * Jm;
    const int pieces = (width + V - 1) / V;
    for (int t = threadIdx.x; t < nb * pieces; t += kHsThreads) {
      const int b = t / pieces, w = V * (t - b * pieces);
      hs_cp16(ss + b * wpad + w, stats + (size_t)(cb + b) * stride + w);
    }
    for (int t = threadIdx.x; t < nb * Jm; t += kHsThreads) {
      const int b = t / Jm, q = t - b * Jm;
      hs_cp8(sa + t, A + (size_t)chunks[cb + b].row * ld + q);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  // weight slot p of a chunk -> (c, c') (c' < 0: the single a_c of a C entry)
  __shared__ int hs_pc[VEST_MAXJ * (VEST_MAXJ + 1) / 2 + VEST_MAXJ];
  for (int p = threadIdx.x; p < AW; p += kHsThreads) {
    int c = 0, q = p, c2 = -1;
    if (p >= AW - Jm) {
      c = p - (AW - Jm);
    } else {
      while (q >= Jm - c) q -= Jm - c, ++c;
      c2 = c + q;
    }
    hs_pc[p] = c | c2 << 8;
  }
  if (c0 < c1) stage(c0, 0);
  int buf = 0;
  for (uint32_t cb = c0; cb < c1; cb += kHsBatch) {
    const int nb = (int)min((uint32_t)kHsBatch, c1 - cb);
    if (cb + kHsBatch < c1) {
      stage(cb + kHsBatch, buf ^ 1);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    const T* ss = sstat + buf * bufw;
    const double* sa = sarow + buf * kHsBatch * Jm;
    for (int t = threadIdx.x; t < nb * AW; t += kHsThreads) {
      const int b = t / AW, pc = hs_pc[t - b * AW];
      const double a0 = sa[b * Jm + (pc & 255)];
      saa[b * kHsAWP + (t - b * AW)] = pc >= 0 ? a0 * sa[b * Jm + (pc >> 8)] : a0;
    }
    __syncthreads();
    if (nb == kHsBatch) {
#pragma unroll
      for (int j = 0; j < kHsPer; ++j) {
        if (my[j] == 0xffffffffu) continue;
        const T* pj = ss + (my[j] & 0xffffu);
        const double* qj = saa + (my[j] >> 16);
#pragma unroll
        for (int b = 0; b < kHsBatch; ++b) acc[j] = fma((double)pj[b * wpad], qj[b * kHsAWP], acc[j]);
      }
    } else {
      for (int b = 0; b < nb; ++b) {
#pragma unroll
        for (int j = 0; j < kHsPer; ++j) {
          if (my[j] == 0xffffffffu) continue;
          acc[j] = fma((double)ss[b * wpad + (my[j] & 0xffffu)], saa[b * kHsAWP + (my[j] >> 16)], acc[j]);
        }
      }
    }
    __syncthreads();  // the buffers are re-staged / rewritten from the next batch on
    buf ^= 1;
  }
#pragma unroll
  for (int j = 0; j < kHsPer; ++j) {
    const int e = threadIdx.x + kHsThreads * j;
    if (e < E) partial[(size_t)blockIdx.x * E + e] = acc[j];
  }
}

__global__ void k_sum_groups(const double* raw, int n, int groups, double* out) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  double s = 0.0;
  for (int g = 0; g < groups; ++g) s += raw[(size_t)g * n + j];
  out[j] = s;
}

// Sequential Gauss-Seidel over the block's live cells.  The CTA compacts the
// block's unmasked cells (ballot scan, row-major order), loads [T | C], their
// core values into shared memory and expands the dense live-cell Gram H
// (nl x nl, H_qq' = T[{f,f'}][{c,c'}]); then one warp runs the nl sequential
// steps, each a handful of shared-memory reads plus one coalesced row update
// of the remaining cells' c.  Masked cells keep dg = 0 (updates.hpp:199-202).
// With s_out (packed statistics only): the sum of squared residuals after this
// block's update from the statistics, s' = s - 2 dg.C + dg^T H dg (s = *s_in,
// the sum before it; C the block's right-hand side before the Gauss-Seidel
// corrections): s_out[0] = s', s_out[1] = s (the deferred last pass,
// sum_from_quadratic_form).
__global__ void __launch_bounds__(256) k_core_solve(const double* tc, int nf, int Jm, int nl, const uint32_t* fib,
                                                    double* core, const uint8_t* core_mask, int reg,
                                                    double lambda, double* dg_out, int packed,
                                                    const double* s_in = nullptr, double* s_out = nullptr) {
  extern __shared__ double sm[];
  const int NAm = Jm * (Jm + 1) / 2;
  const int nT = nf * (nf + 1) / 2 * NAm;
  const int nq = nf * Jm;
  double* H = sm;             // nl x nl
  double* cc = H + nl * nl;   // nl
  double* gv = cc + nl;       // nl
  double* rd = gv + nl;       // nl: 1 / (H_qq + lambda) (LF) or 1 / (2 H_qq) (L1)
  int* lq = reinterpret_cast<int*>(rd + nl);  // live cell -> q
  for (int q = threadIdx.x; q < nq; q += blockDim.x) dg_out[q] = 0.0;
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    int n = 0;
    for (int base = 0; base < nq; base += 32) {
      const int q = base + lane;
      const bool live = q < nq && !core_mask[(int)fib[q / Jm] * Jm + q % Jm];
      const unsigned bal = __ballot_sync(0xffffffffu, live);
      if (live) lq[n + __popc(bal & ((1u << lane) - 1u))] = q;
      n += __popc(bal);
    }
  }
  __syncthreads();
  // packed: tc = [H (upper triangle over the live cells, row-major) | C (live)]
  // (k_core_hsample); else [T | C] of the block GEMM
  const int nh = nl * (nl + 1) / 2;
  for (int t = threadIdx.x; t < nl * nl; t += blockDim.x) {
    if (packed) {
      const int i = t / nl, j = t % nl;
      H[t] = tc[i <= j ? tri(i, j, nl) : tri(j, i, nl)];
      continue;
    }
    const int q = lq[t / nl], q2 = lq[t % nl];
    const int f = q / Jm, c = q % Jm, f2 = q2 / Jm, c2 = q2 % Jm;
    const int ps = f <= f2 ? tri(f, f2, nf) : tri(f2, f, nf);
    const int pa = c <= c2 ? tri(c, c2, Jm) : tri(c2, c, Jm);
    H[t] = tc[ps * NAm + pa];
  }
  for (int l = threadIdx.x; l < nl; l += blockDim.x) {
    const int q = lq[l];
    cc[l] = packed ? tc[nh + l] : tc[nT + q];
    gv[l] = core[(int)fib[q / Jm] * Jm + q % Jm];
    // the denominators do not depend on the sweep state: invert them in
    // parallel, off the sequential critical path
    const int f = q / Jm, c = q % Jm;
    const double hqq = packed ? tc[tri(l, l, nl)] : tc[tri(f, f, nf) * NAm + tri(c, c, Jm)];
    const double den = reg == 0 ? hqq + lambda : 2.0 * hqq;
    rd[l] = den != 0.0 ? 1.0 / den : 0.0;
  }
  __syncthreads();
  if (threadIdx.x >= 32) return;
  const int lane = threadIdx.x;
  for (int l = 0; l < nl; ++l) {
    double dg = 0.0;
    const double hqq = H[l * nl + l];
    const double g_old = gv[l];
    const double num = cc[l] + g_old * hqq;
    const double den = hqq;
    double g_new = g_old;
    const double r = rd[l];
    if (reg == 0) {
      if (den + lambda != 0.0) g_new = num * r;
    } else {
      const double g = -2.0 * num;
      if (2.0 * den != 0.0) g_new = g > lambda ? (lambda - g) * r : (g < -lambda ? -(lambda + g) * r : 0.0);
    }
    if (g_new != g_old) dg = g_new - g_old;
    if (lane == 0) {
      gv[l] = g_new;
      dg_out[lq[l]] = dg;
    }
    if (dg != 0.0) {
      const double* hr = H + l * nl;
      for (int l2 = l + 1 + lane; l2 < nl; l2 += 32) cc[l2] = fma(-dg, hr[l2], cc[l2]);
    }
    __syncwarp();
  }
  if (s_out && packed) {
    __syncwarp();  // dg_out (lane 0's writes) visible to the warp
    double lin = 0.0, quad = 0.0;
    for (int l = lane; l < nl; l += 32) {
      const double dl = dg_out[lq[l]];
      if (dl == 0.0) continue;
      lin = fma(dl, tc[nh + l], lin);
      double hd = 0.0;
      for (int l2 = 0; l2 < nl; ++l2) hd = fma(H[l * nl + l2], dg_out[lq[l2]], hd);
      quad = fma(dl, hd, quad);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      lin += __shfl_xor_sync(0xffffffffu, lin, o);
      quad += __shfl_xor_sync(0xffffffffu, quad, o);
    }
    if (lane == 0) {
      s_out[0] = *s_in - 2.0 * lin + quad;
      s_out[1] = *s_in;
    }
  }
  for (int l = lane; l < nl; l += 32) {
    const int q = lq[l];
    core[(int)fib[q / Jm] * Jm + q % Jm] = gv[l];
  }
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
  std::vector<int> nlive;       // general plan: unmasked cells of the block
  std::vector<int> prefix;      // structured plan: the block's prefix p
  bool pre = false;             // prefix plan (whole prefixes, PreTab)
};

// General plan: runs of <= F consecutive live fibers (a fiber is live when
// one of its cells is unmasked) holding <= kSolveCells unmasked cells.
Blocks plan_blocks(const Ctx& c, int F) {
  Blocks b;
  const int Jm = c.ranks[c.N - 1];
  const int P = c.G / Jm;
  std::vector<int> nl;
  for (int p = 0; p < P; ++p) {
    int n = 0;
    for (int q = 0; q < Jm; ++q) n += !c.h_core_mask[(size_t)p * Jm + q];
    if (n > 0) {
      b.fib.push_back(p);
      nl.push_back(n);
    }
  }
  for (int s = 0; s < (int)b.fib.size();) {
    int len = 0, cells = 0;
    while (s + len < (int)b.fib.size() && len < F && cells + nl[s + len] <= kSolveCells) cells += nl[s + len++];
    b.start.push_back(s);
    b.len.push_back(len);
    b.nlive.push_back(cells);
    s += len;
  }
  return b;
}

// Per-lane stage row of the pass kernel: mode k's factor row (ld_k values,
// even) at offs[k], then r; stride == 2 mod 4 doubles (16-byte aligned rows,
// at most 2-way bank conflicts on the 64-bit reads).  16-byte cp.async
// halves the L1 wavefronts of the random-row gathers against 8-byte copies.
void stage_layout(const Ctx& c, int* offs, int* rslot, int* ldr) {
  const int m = c.N - 1;
  int o = 0;
  for (int k = 0; k < m; ++k) {
    offs[k] = o;
    o += c.ld[k];
  }
  if (rslot) *rslot = o;
  ++o;
  while (o % 4 != 2) ++o;
  if (ldr) *ldr = o;
}

// compile-time last-fiber rank of the prefix-grouped pass kernel (0: per-fiber kernel)
int pass_jl(const Ctx& c) {
  if (c.force_generic || c.core_block > 0) return 0;
  const int M = c.N - 1, JL = c.ranks[c.N - 2];
  if ((M == 2 && (JL == 5 || JL == 10)) || (M == 3 && (JL == 5 || JL == 8)) || (M == 4 && JL == 5)) return JL;
  return 0;
}

// The pass kernel's view of a block's fibers grouped by prefix (see PreTab).
PreTab make_pretab(const Ctx& c, const Blocks& b, int bi) {
  PreTab t{};
  if (bi < 0) return t;
  const int m = c.N - 1, JL = c.ranks[m - 1];
  int offs[VEST_MAXN] = {};
  stage_layout(c, offs, nullptr, nullptr);
  t.nf = b.len[bi];
  int64_t last_p = -1;
  for (int f = 0; f < t.nf; ++f) {
    const uint32_t fib = b.fib[b.start[bi] + f];
    const uint32_t pfx = fib / (uint32_t)JL;
    if ((int64_t)pfx != last_p) {
      if (t.np == kPreMax) throw RtError{"core block spans too many prefixes"};
      uint32_t p = pfx;
      for (int k = m - 2; k >= 0; --k) {
        t.pre[t.np][k] = offs[k] + (int)(p % (uint32_t)c.ranks[k]);
        p /= (uint32_t)c.ranks[k];
      }
      ++t.np;
      last_p = pfx;
    }
  }
  return t;
}

BlockTab block_tab(const Ctx& c, const Blocks& b, int bi);

// The pass kernel's view of a block's fibers (see FibTab).
FibTab make_tab(const Ctx& c, const Blocks& b, int bi) {
  FibTab t{};
  if (bi < 0) return t;
  const int m = c.N - 1;
  int offs[VEST_MAXN] = {};
  stage_layout(c, offs, nullptr, nullptr);
  t.nf = b.len[bi];
  int prevb[VEST_MAXN] = {};
  for (int f = 0; f < t.nf; ++f) {
    uint32_t p = b.fib[b.start[bi] + f];  // row-major index over modes 0..m-1
    int beta[VEST_MAXN] = {};
    for (int k = m - 1; k >= 0; --k) {
      beta[k] = (int)(p % (uint32_t)c.ranks[k]);
      p /= (uint32_t)c.ranks[k];
    }
    t.last[f] = offs[m - 1] + beta[m - 1];
    bool same = f > 0;
    for (int k = 0; k < m - 1; ++k) {
      t.pre[f][k] = offs[k] + beta[k];
      same = same && beta[k] == prevb[k];
      prevb[k] = beta[k];
    }
    t.newp[f] = same ? 0 : 1;
  }
  return t;
}

BlockTab block_tab(const Ctx& c, const Blocks& b, int bi) {
  BlockTab t{};
  if (b.pre) t.pre = make_pretab(c, b, bi);
  else t.fib = make_tab(c, b, bi);
  return t;
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

// Fibers per block: up to kFMax (the live-cell cap of the solve is applied by
// plan_blocks); the block GEMM splits its rows over CTA rows, so it imposes no
// limit.
int pass_jl(const Ctx& c);

// Prefix plan (pass_jl > 0): runs of <= 31 / JL consecutive prefixes
// (beta_0..beta_{m-2}) with an unmasked cell, all JL fibers of each, holding
// <= kSolveCells unmasked cells.
Blocks plan_prefix_blocks(const Ctx& c) {
  Blocks b;
  const int Jm = c.ranks[c.N - 1], JL = c.ranks[c.N - 2];
  const int P = c.G / (JL * Jm), per = kFMax / JL;
  std::vector<int> live;
  std::vector<int> pf;
  for (int p = 0; p < P; ++p) {
    int n = 0;
    for (int q = 0; q < JL * Jm; ++q) n += !c.h_core_mask[(size_t)p * JL * Jm + q];
    if (n > 0) {
      pf.push_back(p);
      live.push_back(n);
    }
  }
  for (int s = 0; s < (int)pf.size();) {
    int np = 0, cells = 0;
    while (s + np < (int)pf.size() && np < per && (np == 0 || cells + live[s + np] <= kSolveCells))
      cells += live[s + np++];
    b.pre = true;
    b.start.push_back((int)b.fib.size());
    b.len.push_back(np * JL);
    b.nlive.push_back(cells);
    for (int i = 0; i < np; ++i)
      for (int f = 0; f < JL; ++f) b.fib.push_back((uint32_t)pf[s + i] * JL + f);
    s += np;
  }
  return b;
}

// Prefix blocks carry their prefixes' masked fibers as Gram columns; use them
// while most fibers of the live prefixes are live (dense cores), runs of live
// fibers otherwise (e.g. config 4's 10 %-dense core: 11 passes instead of 23).
Blocks plan_general(const Ctx& c, int F) {
  if (pass_jl(c) > 0) {
    const int Jm = c.ranks[c.N - 1], JL = c.ranks[c.N - 2];
    const int P = c.G / (JL * Jm);
    long live_f = 0, tot_f = 0;
    for (int p = 0; p < P; ++p) {
      int lf = 0;
      for (int f = 0; f < JL; ++f) {
        bool live = false;
        for (int q = 0; q < Jm && !live; ++q) live = !c.h_core_mask[((size_t)p * JL + f) * Jm + q];
        lf += live;
      }
      if (lf > 0) live_f += lf, tot_f += JL;
    }
    if (tot_f > 0 && 4 * live_f >= 3 * tot_f) return plan_prefix_blocks(c);
  }
  return plan_blocks(c, F);
}

bool use_core_gen(const Ctx& c) {
  if (c.core_gen_mode >= 0) return c.core_gen_mode == 1;
  return c.ops && !c.force_generic && c.core_block == 0 && nvrtc_available() && c.mask_sweeps >= 2;
}

std::vector<std::vector<uint32_t>> block_lists(const Blocks& b) {
  std::vector<std::vector<uint32_t>> out(b.start.size());
  for (size_t i = 0; i < b.start.size(); ++i)
    out[i].assign(b.fib.begin() + b.start[i], b.fib.begin() + b.start[i] + b.len[i]);
  return out;
}

uint64_t plan_key(const Ctx& c, const Blocks& b, int F) {
  uint64_t h = 1469598103934665603ull;
  auto mix = [&](uint64_t v) {
    h ^= v;
    h *= 1099511628211ull;
  };
  mix((uint64_t)c.N);
  for (int k = 0; k < c.N; ++k) mix((uint64_t)c.ranks[k] << 8 | (uint64_t)c.ld[k]);
  mix((uint64_t)F);
  mix(b.pre ? 1 : 0);
  mix(0xF32u + (uint64_t)c.gather_f32);
  for (size_t i = 0; i < b.start.size(); ++i) mix((uint64_t)b.start[i] << 20 | (uint64_t)b.len[i]);
  for (uint32_t f : b.fib) mix(f);
  return h;
}

int pick_block(const Ctx& c) {
  static const int env = [] {  // VEST_CORE_FMAX: fibers per general block (A/B timing)
    const char* e = getenv("VEST_CORE_FMAX");
    return e ? std::max(1, std::min(kFMax, atoi(e))) : kFMax;
  }();
  return c.core_block > 0 ? std::min(c.core_block, kFMax) : env;
}

const void* structured_ops(const Ctx& c) {
  if (c.force_generic || c.N < 3 || c.core_block > 0) return nullptr;
  return find_core_ops(c.N, c.ranks);
}

template <int MM, int NT, int JL, int JALL>
void launch_pass_nt(Ctx& c, const CorePassArgs& a) {
  const size_t sm = (size_t)kPassWarps * (2 * 32 * a.ldr + NT * 8 * kXld) * sizeof(double);
  check(cudaFuncSetAttribute(k_core_pass<MM, NT, JL, JALL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm),
        "pass smem");
  // persistent: as many CTAs as are resident, each warp strides over the chunks
  int per_sm = 0, sms = 0;
  check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_core_pass<MM, NT, JL, JALL>, kPassWarps * 32, sm),
        "pass occupancy");
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c.device);
  const uint32_t need = (a.csf.nchunks + kPassWarps - 1) / kPassWarps;
  const dim3 grid(std::max(1u, std::min<uint32_t>(need, (uint32_t)std::max(1, per_sm) * sms)));
  k_core_pass<MM, NT, JL, JALL><<<grid, kPassWarps * 32, sm, c.stream>>>(a);
}

template <int MM, int JL, int JALL = 0>
void launch_pass_j(Ctx& c, const CorePassArgs& a, int NT) {
  if (NT == 2) launch_pass_nt<MM, 2, JL, JALL>(c, a);
  else if (NT == 3) launch_pass_nt<MM, 3, JL, JALL>(c, a);
  else launch_pass_nt<MM, 4, JL, JALL>(c, a);
}

template <int MM>
void launch_pass_m(Ctx& c, const CorePassArgs& a, int NT) {
  const int jl = a.prefix_plan ? pass_jl(c) : 0;
  // uniform ranks over the staged modes: compile-time row copies
  bool uni = true;
  for (int k = 0; k < MM; ++k) uni = uni && c.ranks[k] == c.ranks[0];
  const int ja = uni ? c.ranks[0] : 0;
  if constexpr (MM == 2) {
    if (jl == 5) return ja == 5 ? launch_pass_j<2, 5, 5>(c, a, NT) : launch_pass_j<2, 5>(c, a, NT);
    if (jl == 10) return ja == 10 ? launch_pass_j<2, 10, 10>(c, a, NT) : launch_pass_j<2, 10>(c, a, NT);
  } else if constexpr (MM == 3) {
    if (jl == 5) return ja == 5 ? launch_pass_j<3, 5, 5>(c, a, NT) : launch_pass_j<3, 5>(c, a, NT);
    if (jl == 8) return ja == 8 ? launch_pass_j<3, 8, 8>(c, a, NT) : launch_pass_j<3, 8>(c, a, NT);
    if (ja == 8) return launch_pass_j<3, 0, 8>(c, a, NT);
  } else if constexpr (MM == 4) {
    if (jl == 5) return ja == 5 ? launch_pass_j<4, 5, 5>(c, a, NT) : launch_pass_j<4, 5>(c, a, NT);
    if (ja == 5) return launch_pass_j<4, 0, 5>(c, a, NT);
  }
  launch_pass_j<MM, 0>(c, a, NT);
}

void launch_pass(Ctx& c, const CorePassArgs& a) {
  ProfScope ps(c, kProfCorePass);
  const int M = c.N - 1;
  if (a.csf.nchunks == 0) return;
  // column tiles: the block's fibers + the residual column
  const int nf = a.kind == 2 ? 0 : a.cur.fib.nf;
  const int NT = nf <= 15 ? 2 : (nf <= 23 ? 3 : 4);
  switch (M) {
    case 1: launch_pass_m<1>(c, a, NT); break;
    case 2: launch_pass_m<2>(c, a, NT); break;
    case 3: launch_pass_m<3>(c, a, NT); break;
    case 4: launch_pass_m<4>(c, a, NT); break;
    case 5: launch_pass_m<5>(c, a, NT); break;
    case 6: launch_pass_m<6>(c, a, NT); break;
    case 7: launch_pass_m<7>(c, a, NT); break;
    default:
      throw ArgError{"unsupported order"};
  }
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
  a.prefix_plan = b.pre ? 1 : 0;
  a.cur = block_tab(c, b, cur);
  a.prev = block_tab(c, b, prev);
  stage_layout(c, a.soff, &a.rslot, &a.ldr);
  launch_pass(c, a);
}

// (T, C) or (C, D) for one block into c.d_gemm_out; returns nout.
int block_gemm(Ctx& c, int nf, int kind, int stride) {
  const int m = c.N - 1, Jm = c.ranks[m];
  const int NS = kind == 0 ? nf * (nf + 1) / 2 : 0;
  const int NAm = Jm * (Jm + 1) / 2;
  const int nout = (kind == 0 ? NS * NAm : 0) + (kind == 0 ? 1 : 2) * nf * Jm;
  ensure(c, &c.d_gemm_out, &c.gemm_out_cap, (size_t)nout);
  ProfScope ps(c, kProfCoreGemm);
  GemmTcArgs t{};
  t.stats = c.d_chunk_stats;
  t.stride = stride;
  t.chunks = c.modes[m].d_chunks;
  t.nchunks = c.modes[m].nchunks;
  t.A = c.d_factor[m];
  t.ld = c.ld[m];
  t.Jm = Jm;
  t.nf = nf;
  t.kind = kind;
  t.LW = kind == 0 ? NS + nf : 2 * nf;
  t.RW = kind == 0 ? NAm + Jm : 2 * Jm;
  t.MT = (t.LW + 7) / 8;
  t.NT = (t.RW + 7) / 8;
  // row tiles per CTA row: the staging (kTcLPer per thread) and the warps'
  // tile slots bound it
  t.MTy = std::min({t.MT, kTcLPer * 256 / 256, kTcWarps * kTcTilesPerWarp / t.NT});
  const int ysplit = (t.MT + t.MTy - 1) / t.MTy;
  const int ntiles = t.MT * t.NT;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c.device);
  const int nparts = std::max(1, std::min<int>(2 * sms, (t.nchunks + 31) / 32));
  const int n = ntiles * 64;
  const int groups = 16;
  ensure(c, &c.d_gemm_part, &c.gemm_part_cap, (size_t)nparts * n + (size_t)groups * n);
  t.partial = c.d_gemm_part;
  double* raw = c.d_gemm_part + (size_t)nparts * n;
  const size_t sm =
      ((size_t)(t.MTy + t.NT) * 8 * kTcLd + 32 * Jm) * sizeof(double) + (size_t)t.NT * 8 * sizeof(int);
  check(cudaFuncSetAttribute(k_core_gemm_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm), "gemm smem");
  k_core_gemm_tc<<<dim3(nparts, ysplit), kTcWarps * 32, sm, c.stream>>>(t);
  k_gemm_reduce1<<<dim3((n + 255) / 256, groups), 256, 0, c.stream>>>(t.partial, nparts, n, groups, raw);
  k_gemm_reduce2<<<(nout + 255) / 256, 256, 0, c.stream>>>(raw, n, groups, kind, nf, Jm, t.NT, c.d_gemm_out);
  count_launch(3);
  check(cudaGetLastError(), "core gemm (tensor cores)");
  return nout;
}

// The sampled live-cell Gram (k_core_hsample) for block bi of a general plan,
// into c.d_gemm_out as [H packed | C]; returns its length, or -1 when the
// dense block GEMM is cheaper (dense blocks) or the block is too wide.
// The sampled live-cell Gram's entry table of block bi (H[q,q'] / C[q] of the
// block's live cells -> statistics row | c | c'), or empty when the dense block
// GEMM is the cheaper path.
static bool hsample_eligible(const Ctx& c, int nf, int nl) {
  const int Jm = c.ranks[c.N - 1];
  const int E = nl * (nl + 1) / 2 + nl;
  const int NS = nf * (nf + 1) / 2, NAm = Jm * (Jm + 1) / 2;
  return E <= kHsPer * kHsThreads && 4 * E < (NS + nf) * (NAm + Jm);
}

static std::vector<uint32_t> hsample_table(const Ctx& c, const Blocks& b, int bi) {
  const int m = c.N - 1, Jm = c.ranks[m];
  const int nf = b.len[bi], nl = b.nlive[bi];
  const int E = nl * (nl + 1) / 2 + nl;
  const int NS = nf * (nf + 1) / 2;
  if (!hsample_eligible(c, nf, nl)) return {};
  std::vector<int> lq;
  for (int f = 0; f < nf; ++f)
    for (int q = 0; q < Jm; ++q)
      if (!c.h_core_mask[(size_t)b.fib[b.start[bi] + f] * Jm + q]) lq.push_back(f * Jm + q);
  std::vector<uint32_t> tab(E);
  auto tri_h = [](int i, int j, int n) { return i * n - i * (i - 1) / 2 + (j - i); };
  for (int i = 0; i < nl; ++i) {
    const int fi = lq[i] / Jm, ci = lq[i] % Jm;
    for (int j = i; j < nl; ++j) {
      const int fj = lq[j] / Jm, cj = lq[j] % Jm;  // fi <= fj (row-major live order)
      tab[tri_h(i, j, nl)] =
          (uint32_t)tri_h(fi, fj, nf) | (uint32_t)tri_h(std::min(ci, cj), std::max(ci, cj), Jm) << 16;
    }
    tab[nl * (nl + 1) / 2 + i] = (uint32_t)(NS + fi) | (uint32_t)(Jm * (Jm + 1) / 2 + ci) << 16;
  }
  return tab;
}

// Every block's table in one device buffer, uploaded only when the plan
// changes (a copy from a host buffer must not be recorded into an iteration
// graph; the tables depend on the core mask only).
static void upload_hsample_tables(Ctx& c, const Blocks& b) {
  std::vector<uint32_t> all;
  std::vector<int64_t> off(b.start.size(), -1);
  for (size_t bi = 0; bi < b.start.size(); ++bi) {
    const std::vector<uint32_t> t = hsample_table(c, b, (int)bi);
    if (t.empty()) continue;
    off[bi] = (int64_t)all.size();
    all.insert(all.end(), t.begin(), t.end());
  }
  c.hstab_off = off;
  if (c.d_hstab && c.h_hstab == all) return;
  ensure(c, reinterpret_cast<double**>(&c.d_hstab), &c.hstab_cap, (all.size() + 1) / 2 + 1);
  if (!all.empty())
    check(cudaMemcpyAsync(c.d_hstab, all.data(), all.size() * 4, cudaMemcpyHostToDevice, c.stream), "hsample tables");
  check(cudaStreamSynchronize(c.stream), "hsample tables");
  c.h_hstab = all;
}

int block_hsample(Ctx& c, const Blocks& b, int bi, int stride) {
  const int m = c.N - 1, Jm = c.ranks[m];
  const int nf = b.len[bi], nl = b.nlive[bi];
  const int E = nl * (nl + 1) / 2 + nl;
  const int NS = nf * (nf + 1) / 2;
  if (bi >= (int)c.hstab_off.size() || c.hstab_off[bi] < 0) return -1;
  const uint32_t* tab = c.d_hstab + c.hstab_off[bi];
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c.device);
  const ModeData& md = c.modes[m];
  const int nparts = std::max(1, std::min<int>(4 * sms, (int)((md.nchunks + kHsBatch - 1) / kHsBatch)));
  const int groups = 16;
  ensure(c, &c.d_gemm_part, &c.gemm_part_cap, (size_t)nparts * E + (size_t)groups * E);
  ensure(c, &c.d_gemm_out, &c.gemm_out_cap, (size_t)E);
  double* raw = c.d_gemm_part + (size_t)nparts * E;
  const int width = NS + nf;
  ProfScope ps(c, kProfCoreGemm);
  if (c.stats_f32) {
    const size_t sm = (size_t)2 * kHsBatch * (kHsWP * sizeof(float) + Jm * sizeof(double)) +
                      (size_t)kHsBatch * kHsAWP * sizeof(double);
    check(cudaFuncSetAttribute(k_core_hsample<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm),
          "hsample smem");
    k_core_hsample<float><<<nparts, kHsThreads, sm, c.stream>>>(reinterpret_cast<const float*>(c.d_chunk_stats), stride,
                                                                 width, md.d_chunks, md.nchunks, c.d_factor[m], c.ld[m],
                                                                 Jm, tab, E, c.d_gemm_part);
  } else {
    const size_t sm = (size_t)2 * kHsBatch * (kHsWP + Jm) * sizeof(double) +
                      (size_t)kHsBatch * kHsAWP * sizeof(double);
    check(cudaFuncSetAttribute(k_core_hsample<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm),
          "hsample smem");
    k_core_hsample<double><<<nparts, kHsThreads, sm, c.stream>>>(c.d_chunk_stats, stride, width, md.d_chunks,
                                                                  md.nchunks, c.d_factor[m], c.ld[m], Jm, tab, E,
                                                                  c.d_gemm_part);
  }
  k_gemm_reduce1<<<dim3((E + 255) / 256, groups), 256, 0, c.stream>>>(c.d_gemm_part, nparts, E, groups, raw);
  k_sum_groups<<<(E + 255) / 256, 256, 0, c.stream>>>(raw, E, groups, c.d_gemm_out);
  count_launch(3);
  check(cudaGetLastError(), "hsample");
  return E;
}

void upload_fibers(Ctx& c, const Blocks& b) {
  // the plan changes only with the mask: skip identical uploads (a copy from a
  // temporary host buffer must not be recorded into an iteration graph)
  if (c.d_fibers && c.h_fibers == b.fib) return;
  ensure(c, reinterpret_cast<double**>(&c.d_fibers), &c.fibers_cap, (b.fib.size() + 1) / 2 + 1);
  check(cudaMemcpyAsync(c.d_fibers, b.fib.data(), b.fib.size() * sizeof(uint32_t), cudaMemcpyHostToDevice,
                        c.stream),
        "fibers");
  c.h_fibers = b.fib;
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

// 3-mode all-prefix sweep, or the general sweep through the plan-specialised
// passes (their modules are built by the time the key has repeated)
bool core_sweep_capturable(const Ctx& c) {
  const void* sops = structured_ops(c);
  if (sops) return !legacy_block_passes() && find_core_all_ops(c.N, c.ranks);
  return use_core_gen(c);
}

bool core_sweep_general(const Ctx& c) { return structured_ops(c) == nullptr; }

// VEST_DEFER_LAST=0: run the general sweep's final residual pass eagerly (A/B)
bool defer_last_enabled() {
  static const bool v = [] {
    const char* e = getenv("VEST_DEFER_LAST");
    return !(e && e[0] == '0');
  }();
  return v;
}

// Apply the general sweep's deferred last block to r (its final pass: previous
// block's update + per-chunk r^2) and sum r^2 exactly.
void core_apply_pending_general(Ctx& c) {
  const int m = c.N - 1;
  {
    ProfScope ps(c, kProfResid);
    core_gen_pass(c, c.r_pending[0], c.d_dg, c.d_chunk_stats, c.pending_stride, c.d_chunk_sum);
  }
  c.sum_sq = reduce_chunk_sums(c, c.d_chunk_sum, c.modes[m].nchunks);
  c.re = std::sqrt(c.sum_sq) / c.x_norm;
  c.r_valid = true;
  c.r_fresh = true;
  c.r_pending[0] = c.r_pending[1] = -1;
  c.r_pending_general = false;
}

// Key of a plan's generated module: the plan, plus the two sweep-level choices
// the source depends on (fp32 chunk statistics, deferred last pass).
static uint64_t gen_module_key(uint64_t pk, bool stats_f32, bool defer_last) {
  return pk * 1099511628211ull ^ (0x9E3779B97F4A7C15ull + (stats_f32 ? 2u : 0u) + (defer_last ? 1u : 0u));
}

// Start compiling the plan-specialised passes of the current mask on a host
// thread (note_sweep: the first sweep with a new mask; auto mode switches them
// in from the second).  The source is generated here, with the sweep-level
// flags the second sweep will use.
void core_gen_prefetch(Ctx& c) {
  if (c.core_gen_mode >= 0) return;  // forced on: compiled where first used; off: never
  if (!(c.ops && !c.force_generic && c.core_block == 0 && nvrtc_available()) || structured_ops(c)) return;
  const int F = pick_block(c);
  const Blocks b = plan_general(c, F);
  if (b.fib.empty()) return;
  bool elig = true;
  for (size_t bi = 0; bi < b.start.size(); ++bi) elig = elig && hsample_eligible(c, b.len[bi], b.nlive[bi]);
  const bool sf = c.gather_f32 && elig, dl = defer_last_enabled() && elig;
  const uint64_t key = gen_module_key(plan_key(c, b, F), sf, dl);
  if (c.pre_gen.valid && c.pre_gen.key == key) return;
  const bool sf0 = c.stats_f32, dl0 = c.defer_last;
  c.stats_f32 = sf;
  c.defer_last = dl;
  std::vector<int> nts;
  int ldr = 0;
  std::string src = core_gen_source(c, block_lists(b), nts, ldr);
  c.stats_f32 = sf0;
  c.defer_last = dl0;
  prefetch_cubin(c, c.pre_gen, key, std::move(src), "vest_core_gen.cu", core_gen_compile);
}

// the general plan's blocks (host-only compile check of the generated passes)
std::vector<std::vector<uint32_t>> core_gen_plan(const Ctx& c) { return block_lists(plan_general(c, pick_block(c))); }

static void core_sweep_impl(Ctx& c, int reg, double lambda);

// The sweep rewrites d_core: the constant-bank copy is stale after it (and a
// ConstCore kernel inside it -- the residual it may recompute first -- must not
// leave the pre-sweep core marked current).
void core_sweep(Ctx& c, int reg, double lambda) {
  sync_const_core(c);
  core_sweep_impl(c, reg, lambda);
  sync_const_core(c);
}

static void core_sweep_impl(Ctx& c, int reg, double lambda) {
  const int m = c.N - 1, Jm = c.ranks[m];
  // r = x - B(alpha) for the model after the factor updates
  // (the reference rebuilds its reconstruction cache here, updates.hpp:190-192);
  // already fresh when the last factor mode emitted it
  if (!c.r_fresh) compute_residual(c);
  const void* sops = structured_ops(c);
  const int F = sops ? c.ranks[c.N - 2] : pick_block(c);
  const Blocks b = sops ? plan_structured(c) : plan_general(c, F);
  if (b.fib.empty()) {  // fully pruned core: nothing to update, but the RE of
    // the updated factors is still due (a residual emitted by the last factor
    // mode carries no sum of squares yet)
    c.r_fresh = false;
    compute_residual(c);
    return;
  }
  upload_fibers(c, b);
  if (sops && !legacy_block_passes()) {
    if (const void* aops = find_core_all_ops(c.N, c.ranks)) {
      core_sweep_sall(c, aops, reg, lambda, b.prefix, b.start);
      return;
    }
  }
  if (sops) pack_operands(c, sops);
  // fp32 mode with every block on the sampled Gram: the passes write fp32 chunk
  // statistics (half the traffic to k_core_hsample); rows 16-byte aligned
  c.stats_f32 = false;
  if (!sops && c.gather_f32 && use_core_gen(c)) {
    c.stats_f32 = true;
    for (size_t bi = 0; bi < b.start.size(); ++bi) c.stats_f32 = c.stats_f32 && hsample_eligible(c, b.len[bi], b.nlive[bi]);
  }
  const int stride = c.stats_f32 ? (F * (F + 1) / 2 + F + 3) & ~3 : (F * (F + 1) / 2 + F + 1) & ~1;
  ensure(c, &c.d_chunk_stats, &c.chunk_stats_cap, (size_t)c.modes[m].nchunks * stride);
  ensure(c, &c.d_dg, &c.dg_cap, (size_t)kFMax * VEST_MAXJ);
  ensure(c, &c.d_chunk_sum, &c.chunk_sum_cap, c.modes[m].nchunks + 1);
  const int nb = (int)b.start.size();
  // plan-specialised passes (vest_core_gen.cu) for the general plans
  const bool gen = !sops && use_core_gen(c);
  // every block on the sampled Gram (packed statistics): the last block's
  // residual update is deferred -- the sum of squares after it follows from its
  // statistics, and r is brought up to date only if something reads it (the
  // next iteration's last factor mode rewrites it anyway)
  c.defer_last = gen && defer_last_enabled();
  for (size_t bi = 0; c.defer_last && bi < b.start.size(); ++bi)
    c.defer_last = hsample_eligible(c, b.len[bi], b.nlive[bi]);
  if (gen) core_gen_prepare(c, block_lists(b), gen_module_key(plan_key(c, b, F), c.stats_f32, c.defer_last));
  if (!sops) upload_hsample_tables(c, b);
  for (int bi = 0; bi <= nb; ++bi) {
    const bool last = bi == nb;
    if (last && c.defer_last) break;
    if (gen) {
      ProfScope ps(c, kProfCorePass);
      core_gen_pass(c, bi, c.d_dg, c.d_chunk_stats, stride, c.d_chunk_sum);
    } else {
      run_pass(c, sops, b, bi - 1, last ? -1 : bi, last ? 2 : 0, stride);
    }
    if (last) break;
    const int nf = b.len[bi];
    int nout = sops ? -1 : block_hsample(c, b, bi, stride);
    const int packed = nout >= 0 ? 1 : 0;
    if (nout < 0) nout = block_gemm(c, nf, 0, stride);
    comm_allreduce(c, c.d_gemm_out, (uint64_t)nout);  // block statistics over the shards
    ProfScope ps(c, kProfCoreSolve);
    const size_t nq = (size_t)nf * Jm, nl = (size_t)b.nlive[bi];
    const size_t sm = (nl * nl + 3 * nl) * sizeof(double) + nq * sizeof(int);
    check(cudaFuncSetAttribute(k_core_solve, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm), "solve smem");
    const bool quad = c.defer_last && bi == nb - 1;
    if (quad) sum_chunks_device(c, c.d_chunk_sum, c.modes[m].nchunks, c.d_small + 2);  // s before the last block
    k_core_solve<<<1, 256, sm, c.stream>>>(c.d_gemm_out, nf, Jm, (int)nl, c.d_fibers + b.start[bi], c.d_core,
                                           c.d_core_mask, reg, lambda, c.d_dg, packed, quad ? c.d_small + 2 : nullptr,
                                           quad ? c.d_small : nullptr);
    count_launch();
    check(cudaGetLastError(), "core solve");
  }
  if (c.defer_last) {
    check(cudaMemcpyAsync(c.h_small, c.d_small, 2 * sizeof(double), cudaMemcpyDeviceToHost, c.stream), "sum readback");
    c.r_valid = false;
    c.r_fresh = false;
    c.r_pending[0] = nb;  // the skipped final pass
    c.r_pending[1] = -1;
    c.r_pending_ops = nullptr;
    c.r_pending_general = true;
    c.pending_stride = stride;
    if (!c.capturing) {  // a captured iteration reads the sums after the graph launch
      check(cudaStreamSynchronize(c.stream), "sum sync");
      sum_from_quadratic_form(c);
    }
    return;
  }
  const double ss = reduce_chunk_sums(c, c.d_chunk_sum, c.modes[m].nchunks);  // captured: read after the replay
  if (!c.capturing) {
    c.sum_sq = ss;
    c.re = std::sqrt(c.sum_sq) / c.x_norm;
  }
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
  const Blocks b = sops ? plan_structured(c) : plan_general(c, F);
  if (b.fib.empty()) return;
  upload_fibers(c, b);
  if (sops) pack_operands(c, sops);
  const int stride = 2 * F;
  ensure(c, &c.d_chunk_stats, &c.chunk_stats_cap, (size_t)c.modes[m].nchunks * stride);
  ensure(c, &c.d_dg, &c.dg_cap, (size_t)kFMax * VEST_MAXJ);
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
