// SPDX-License-Identifier: Apache-2.0
// vest_core_s.cu -- core-sweep pass for compile-time ranks ("structured"
// blocks).  A block is every fiber that shares the prefix p = (beta_0 ..
// beta_{m-2}) (m = N-1, the last mode): F = J_{m-1} fibers, F * J_m
// consecutive core cells in row-major order.  For an entry e
//   s_f(e) = w_p(e) * A_{m-1}[i_{m-1}, f],  w_p(e) = prod_{k<m-1} A_k[i_k, beta_k(p)]
// so one vectorised factor-row gather plus (m-1) scalar gathers give all F
// fiber products.  The per-slice statistics S_ff' = sum s_f s_f' and
// R_f = sum s_f r are accumulated on the FP64 tensor cores: the 32 lanes'
// vectors x = (s_0..s_{F-1}, r) are staged (transposed) in shared memory and
// X^T X is accumulated with mma.sync m8n8k4 f64 (DMMA) per 4-entry k-step;
// the accumulator tiles hold the whole chunk's sums, so no cross-lane
// reduction is needed.  See vest_core.cu for the block algebra.
#include <algorithm>
#include <type_traits>
#include <vector>

#include "vest_common.cuh"

namespace vest {

struct CorePassSArgs {
  DevModel m;
  DevCSF csf;  // mode N-1
  double* r;
  int prev_p;             // prefix of the previous block (-1: none)
  const double* prev_dg;  // [F][Jm]
  int cur_p;              // prefix of the current block (-1: none)
  int kind;               // 0 sweep (S, R), 1 responsibility (R, D), 2 final (apply prev, sum r^2)
  double* stats;
  int stride;
  double* chunk_sq;
  // packed per-entry operands (CSF order of the last mode, SoA), built once per
  // sweep: U[f][pos] = A_{m-1}[i_{m-1}, f], W[p][pos] = prod_{k<m-1} A_k[i_k, beta_k(p)]
  const double* U;
  const double* W;
  uint64_t wstride;
};

// Pack U and W for positions [p0, p1) of the last mode's CSF.  The factors do
// not change during the core sweep, so the passes stream these coalesced
// instead of re-gathering factor rows and coordinates every pass.
template <class S>
__global__ void __launch_bounds__(256) k_pack_uw(DevModel m, DevCSF csf, uint64_t p0, uint64_t p1, double* U,
                                                 double* W, uint64_t wstride) {
  constexpr int N = S::N;
  constexpr int mm = N - 2;
  constexpr int F = S::J(mm);
  constexpr int P = S::G() / (F * S::J(N - 1));
  for (uint64_t pos = p0 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; pos < p1;
       pos += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t idx[N - 1];
#pragma unroll
    for (int k = 0; k < N - 1; ++k) idx[k] = __ldg(csf.oc[k] + pos);
    constexpr int ldu = (F + 1) & ~1;
    const double* urow = m.factor[mm] + (size_t)idx[mm] * ldu;
    double u[F];
#pragma unroll
    for (int f = 0; f + 1 < F; f += 2) {
      const double2 v = __ldg(reinterpret_cast<const double2*>(urow + f));
      u[f] = v.x;
      u[f + 1] = v.y;
    }
    if constexpr (F & 1) u[F - 1] = __ldg(urow + F - 1);
    if constexpr (N == 3) {
      // W[p][pos] = A_0[i_0, p]: one vectorised row gather
      constexpr int J0 = S::J(0);
      constexpr int ld0 = (J0 + 1) & ~1;
      const double* row0 = m.factor[0] + (size_t)idx[0] * ld0;
      double w[J0];
#pragma unroll
      for (int p = 0; p + 1 < J0; p += 2) {
        const double2 v = __ldg(reinterpret_cast<const double2*>(row0 + p));
        w[p] = v.x;
        w[p + 1] = v.y;
      }
      if constexpr (J0 & 1) w[J0 - 1] = __ldg(row0 + J0 - 1);
#pragma unroll
      for (int p = 0; p < J0; ++p) __stcs(W + (uint64_t)p * wstride + pos, w[p]);
    } else {
#pragma unroll 1
      for (int p = 0; p < P; ++p) {
        int rest = p;
        double w = 1.0;
#pragma unroll
        for (int k = mm - 1; k >= 0; --k) {
          const int b = rest % S::J(k);
          rest /= S::J(k);
          w *= __ldg(m.factor[k] + (size_t)idx[k] * m.ld[k] + b);
        }
        __stcs(W + (uint64_t)p * wstride + pos, w);
      }
    }
#pragma unroll
    for (int f = 0; f < F; ++f) __stcs(U + (uint64_t)f * wstride + pos, u[f]);  // SoA: coalesced
  }
}

template <int B, int E, class Fn>
__device__ __forceinline__ void sfor_s(Fn&& f) {
  if constexpr (B < E) {
    f(std::integral_constant<int, B>{});
    sfor_s<B + 1, E>(f);
  }
}

constexpr int kSWarps = 8;

template <class S>
__global__ void __launch_bounds__(kSWarps * 32) k_core_pass_s(CorePassSArgs a) {
  constexpr int N = S::N;
  constexpr int m = N - 1;
  constexpr int mm = m - 1;  // mode whose row gives the fiber index
  constexpr int F = S::J(mm);
  constexpr int Jm = S::J(m);
  constexpr int NC = F + 1;            // columns: s_0..s_{F-1}, r
  constexpr int NT = NC > 8 ? 2 : 1;   // 8-wide column tiles
  static_assert(NC <= 16, "structured pass supports F <= 15");
  __shared__ double xs[kSWarps][16 * kXld];
  __shared__ double qs[kSWarps][F];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* X = xs[warp];
  for (int t = lane; t < 16 * kXld; t += 32) X[t] = 0.0;
  const uint32_t ci = blockIdx.x * kSWarps + warp;
  if (ci >= a.csf.nchunks) return;
  const Chunk ch = a.csf.chunks[ci];

  // prefix multi-indices (modes 0..mm-1) of the previous / current block
  int bp[mm > 0 ? mm : 1], bc[mm > 0 ? mm : 1];
  {
    int rp = a.prev_p, rc = a.cur_p;
#pragma unroll
    for (int k = mm - 1; k >= 0; --k) {
      bp[k] = rp >= 0 ? rp % S::J(k) : 0;
      bc[k] = rc >= 0 ? rc % S::J(k) : 0;
      rp = rp >= 0 ? rp / S::J(k) : -1;
      rc = rc >= 0 ? rc / S::J(k) : -1;
    }
  }
  // q_f = sum_c A_m[s, c] dg_prev[f][c]
  const bool has_prev = a.prev_p >= 0;
  if (has_prev && lane < F) {
    constexpr int ldm = (Jm + 1) & ~1;
    const double* arow = a.m.factor[m] + (size_t)ch.row * ldm;
    double t = 0.0;
#pragma unroll
    for (int c = 0; c < Jm; ++c) t = fma(__ldg(arow + c), a.prev_dg[lane * Jm + c], t);
    qs[warp][lane] = t;
  }
  __syncwarp();

  double d[3][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
  double sq = 0.0;
  const bool acc = a.kind != 2 && a.cur_p >= 0;
  const int g = lane >> 2, tq = lane & 3;

  for (uint32_t base = ch.beg; base < ch.end; base += 32) {
    const uint32_t pos = base + lane;
    const bool valid = pos < ch.end;
    double u[F];
    double wp = 1.0, wc = 1.0, r = 0.0;
    if (valid) {
      r = a.r[pos];
      if (a.U) {
        // packed operands, SoA [F][nnz]: every load coalesced across the warp
#pragma unroll
        for (int f = 0; f < F; ++f) u[f] = __ldcs(a.U + (uint64_t)f * a.wstride + pos);
        if (has_prev) wp = __ldcs(a.W + (uint64_t)a.prev_p * a.wstride + pos);
        if (acc) wc = __ldcs(a.W + (uint64_t)a.cur_p * a.wstride + pos);
      } else {
        uint32_t idx[m];
#pragma unroll
        for (int k = 0; k < m; ++k) idx[k] = __ldg(a.csf.oc[k] + pos);
        constexpr int ldu = (F + 1) & ~1;
        const double* urow = a.m.factor[mm] + (size_t)idx[mm] * ldu;
#pragma unroll
        for (int f = 0; f + 1 < F; f += 2) {
          const double2 v = __ldg(reinterpret_cast<const double2*>(urow + f));
          u[f] = v.x;
          u[f + 1] = v.y;
        }
        if constexpr (F & 1) u[F - 1] = __ldg(urow + F - 1);
        sfor_s<0, mm>([&](auto kc) {
          constexpr int k = decltype(kc)::value;
          constexpr int ld = (S::J(k) + 1) & ~1;
          const double* row = a.m.factor[k] + (size_t)idx[k] * ld;
          if (has_prev) wp *= __ldg(row + bp[k]);
          if (acc) wc *= __ldg(row + bc[k]);
        });
      }
      if (has_prev) {
        double t = 0.0;
#pragma unroll
        for (int f = 0; f < F; ++f) t = fma(u[f], qs[warp][f], t);
        r = fma(-wp, t, r);
        if (a.kind != 1) a.r[pos] = r;
      }
    } else {
#pragma unroll
      for (int f = 0; f < F; ++f) u[f] = 0.0;
      wc = 0.0;
    }
    if (a.kind == 2) {
      sq = fma(r, r, sq);
      continue;
    }
    if (!acc) continue;
    // stage x = (wc * u, r) transposed: X[col][lane]
#pragma unroll
    for (int f = 0; f < F; ++f) X[f * kXld + lane] = wc * u[f];
    X[F * kXld + lane] = valid ? r : 0.0;
    __syncwarp();
    gram_dmma<NC>(X, d, lane);
    __syncwarp();
  }

  if (a.kind == 2) {
    sq = warp_sum(sq);
    if (lane == 0) a.chunk_sq[ci] = sq;
    return;
  }
  if (!acc) return;
  // tile t: (I, J) = (0,0), (0,1), (1,1); lane holds (8I + g, 8J + 2tq + i)
  double* out = a.stats + (size_t)ci * a.stride;
  constexpr int NS = F * (F + 1) / 2;
#pragma unroll
  for (int t = 0; t < (NT == 1 ? 1 : 3); ++t) {
    const int I = t == 2 ? 1 : 0, J = t == 0 ? 0 : 1;
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int row = 8 * I + g, col = 8 * J + 2 * tq + i;
      const double v = d[t][i];
      if (a.kind == 0) {
        if (row <= col && col < F) out[row * F - row * (row - 1) / 2 + (col - row)] = v;
        else if (col == F && row < F) out[NS + row] = v;
      } else {
        if (col == F && row < F) out[row] = v;
        else if (row == col && row < F) out[F + row] = v;
      }
    }
  }
}

// ======================================================= all-prefix sweep --
// The exact block Gauss-Seidel needs, per block p, only its diagonal Gram
// T_p = sum_slices S_p,slice (x) a a^T: the coupling between blocks is carried
// by the residual, which is updated between blocks.  For N == 3 the S_p depend
// only on the (fixed) factors, so ONE pass produces all of them,
//   S_p,slice[(f,f')] = sum_{e in chunk} A_0[i_0,p]^2 u_f u_f',  u = A_1[i_1,:],
// and ONE tensor-core GEMM produces every T_p.  Per block what remains is a
// light pass (previous block's residual update, R_p = sum w_p r u, folded into
// C_p = sum_slices R_p (x) a) and the solve.
constexpr int kAllWarps = 8;    // k_core_sall warps per CTA
constexpr int kRWarps = 8;      // k_core_rpass warps per CTA

// pair index p of the row-major upper triangle of an n x n matrix -> (i, j)
__device__ __forceinline__ void tri_pair(int p, int n, int& i, int& j) {
  int r = p;
  i = 0;
  while (r >= n - i) {
    r -= n - i;
    ++i;
  }
  j = i + r;
}

// S_p for every prefix p of one chunk per warp (persistent over chunks).
// FP64 pipe, lane-owned outputs: lane l owns the pairs l, l+32, ... for every
// p, so the chunk's sums need no cross-lane reduction.  Rounds of 32 entries
// are staged in shared memory by cp.async one round ahead (double buffer;
// the coordinates two rounds ahead), so the FMA loop never waits on the L2
// gathers; a per-round fix-up pass squares the weights in place and writes
// the raw ones (W, SoA) for the block passes.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(smem))),
               "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// staged row stride: [w | u] padded to == 4 (mod 16) doubles, so the DMMA
// fragment loads (4 rows x 4..8 columns per half-warp) are conflict-free
__host__ __device__ constexpr int sall_ldr(int P, int F) {
  return (((P + 1) & ~1) + ((F + 1) & ~1)) + ((4 - (((P + 1) & ~1) + ((F + 1) & ~1)) % 16) + 16) % 16;
}

template <class S>
__global__ void __launch_bounds__(kAllWarps * 32, 2) k_core_sall(DevModel m, DevCSF csf, double* stats, double* W,
                                                                 uint64_t wstride) {
  static_assert(S::N == 3, "all-prefix statistics: 3-mode shapes");
  constexpr int P = S::J(0), F = S::J(1), NV = F * (F + 1) / 2;
  constexpr int ld0 = (P + 1) & ~1, ld1 = (F + 1) & ~1;
  constexpr int LDR = sall_ldr(P, F);  // staged row: [w (ld0) | u (ld1) | pad]
  extern __shared__ __align__(16) double sall_smem[];  // [warp][2][32 * LDR]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* const stage0 = sall_smem + (size_t)warp * 2 * 32 * LDR;
  // DMMA tiling: A = w^2 (rows = prefixes, MT tiles), B = u_i u_j (cols =
  // pairs, NT tiles); fragments A[g][t], B[t][g], D[g][2t + i]
  constexpr int MT = (P + 7) / 8, NT = (NV + 7) / 8;
  const int g = lane >> 2, tq = lane & 3;
  int bi[NT], bj[NT];  // this lane's B-fragment pair (u offsets), per column tile
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    bi[nt] = bj[nt] = -1;
    if (8 * nt + g < NV) tri_pair(8 * nt + g, F, bi[nt], bj[nt]);
  }
  const uint32_t stride = gridDim.x * kAllWarps;
  // round cursor: (chunk, base); advance = next 32 entries of the chunk, else
  // the warp's next chunk
  struct Cur {
    uint32_t ci, beg, end, base;
  };
  auto first = [&](uint32_t ci) {
    Cur c{ci, 0, 0, 0};
    if (ci < csf.nchunks) {
      const Chunk ch = csf.chunks[ci];
      c.beg = ch.beg;
      c.end = ch.end;
      c.base = ch.beg;
    }
    return c;
  };
  auto next = [&](const Cur& c) {
    if (c.base + 32 < c.end) return Cur{c.ci, c.beg, c.end, c.base + 32};
    return first(c.ci + stride);
  };
  // issue round c's row copies into buffer b (coordinates already loaded)
  auto issue = [&](const Cur& c, int b, uint32_t i0, uint32_t i1) {
    double* row = stage0 + b * 32 * LDR + lane * LDR;
    if (c.ci < csf.nchunks && c.base + lane < c.end) {
      const double* r0 = m.factor[0] + (size_t)i0 * ld0;
      const double* r1 = m.factor[1] + (size_t)i1 * ld1;
#pragma unroll
      for (int t = 0; t < ld0 / 2; ++t) cp_async16(row + 2 * t, r0 + 2 * t);
#pragma unroll
      for (int t = 0; t < ld1 / 2; ++t) cp_async16(row + ld0 + 2 * t, r1 + 2 * t);
    } else {
      // zero weight: padded entries contribute nothing
#pragma unroll
      for (int t = 0; t < LDR; ++t) row[t] = 0.0;
    }
  };
  auto coords = [&](const Cur& c, uint32_t& i0, uint32_t& i1) {
    i0 = i1 = 0;
    if (c.ci < csf.nchunks && c.base + lane < c.end) {
      i0 = __ldg(csf.oc[0] + c.base + lane);
      i1 = __ldg(csf.oc[1] + c.base + lane);
    }
  };

  Cur cur = first(blockIdx.x * kAllWarps + warp);
  if (cur.ci >= csf.nchunks) return;
  uint32_t a0, a1;
  coords(cur, a0, a1);
  issue(cur, 0, a0, a1);
  Cur nxt = next(cur);
  uint32_t n0, n1;
  coords(nxt, n0, n1);
  double acc[MT][NT][2];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
  int buf = 0;
  while (true) {
    // this round's rows have landed: square the weights (and emit the raw ones)
    cp_async_wait_all();
    __syncwarp();
    {
      double* row = stage0 + buf * 32 * LDR + lane * LDR;
      const uint32_t pos = cur.base + lane;
      if (pos < cur.end) {
#pragma unroll
        for (int t = 0; t < ld0 / 2; ++t) {
          const double2 v = reinterpret_cast<const double2*>(row)[t];
          __stcs(W + (uint64_t)(2 * t) * wstride + pos, v.x);
          if (2 * t + 1 < P) __stcs(W + (uint64_t)(2 * t + 1) * wstride + pos, v.y);
          reinterpret_cast<double2*>(row)[t] = make_double2(v.x * v.x, v.y * v.y);
        }
      }
    }
    __syncwarp();
    // next round's copies go out now (their coordinates arrived a round ago)
    const bool more = nxt.ci < csf.nchunks;
    if (more) issue(nxt, buf ^ 1, n0, n1);
    const Cur nn = more ? next(nxt) : nxt;
    uint32_t m0 = 0, m1 = 0;
    if (more) coords(nn, m0, m1);
    // X^T-style product over this round on the FP64 tensor cores: 8 k-steps
    // of 4 entries (rows past the chunk end were zeroed at staging)
    {
      const double* st = stage0 + buf * 32 * LDR;
      const int nk = (int)(min(32u, cur.end - cur.base) + 3) >> 2;
#pragma unroll 2
      for (int kk = 0; kk < nk; ++kk) {
        const double* row = st + (4 * kk + tq) * LDR;
        double a[MT];
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) a[mt] = (8 * mt + g < P) ? row[8 * mt + g] : 0.0;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const double b = bi[nt] >= 0 ? row[ld0 + bi[nt]] * row[ld0 + bj[nt]] : 0.0;
#pragma unroll
          for (int mt = 0; mt < MT; ++mt) dmma884(acc[mt][nt][0], acc[mt][nt][1], a[mt], b);
        }
      }
    }
    // chunk finished: write its statistics
    if (!more || nxt.ci != cur.ci) {
      double* out = stats + (size_t)cur.ci * (P * NV);
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const int b = 8 * mt + g, pr = 8 * nt + 2 * tq + i;
            if (b < P && pr < NV) out[b * NV + pr] = acc[mt][nt][i];
            acc[mt][nt][i] = 0.0;
          }
    }
    if (!more) break;
    __syncwarp();
    cur = nxt;
    nxt = nn;
    n0 = m0;
    n1 = m1;
    buf ^= 1;
  }
}

struct RPassArgs {
  DevModel m;
  DevCSF csf;          // mode N-1
  double* r;
  int prev_p;          // previous block's prefix (-1: none)
  const double* prev_dg;  // [F][Jm]
  int cur_p;           // current block's prefix (-1: final pass)
  double* chunk_sq;    // final pass: per-chunk sum of r^2
  double* part;        // [gridDim.x][F*Jm] CTA partials of C
  double* cout;        // C_p = sum_slices R_p (x) a   [F*Jm]
  unsigned* counter;   // CTA arrival counter (self-resetting)
  const double* W;     // [P][wstride] block weights A_0[i_0, p] (k_core_sall)
  uint64_t wstride;
  int want_sq;         // also sum r^2 (after the previous block's update) into cout[F*Jm]
};

// Per block: r -= w_prev (u . q_prev) (q_prev = dg_prev a, per slice), then
// R_f = sum w_cur r u_f per chunk and C[f][c] += R_f a_c (lane-owned).  The
// CTAs' partial C are summed in a fixed order by the last CTA to arrive, so
// the result is deterministic and ready without another launch.  Gather-bound
// (L2): the next round's coordinates and residuals are prefetched while the
// current round's factor rows are in flight; <= 64 registers for 32 warps/SM.
template <class S>
#ifndef VEST_RPASS_MINB
#define VEST_RPASS_MINB 4
#endif
__global__ void __launch_bounds__(kRWarps * 32, VEST_RPASS_MINB) k_core_rpass(RPassArgs a) {
  static_assert(S::N == 3, "block pass: 3-mode shapes");
  constexpr int F = S::J(1), Jm = S::J(2), NQ = F * Jm, KQ = (NQ + 31) / 32;
  static_assert(NQ < 128, "block pass: F * J_m < 128");
  constexpr int ld1 = (F + 1) & ~1, ld2 = (Jm + 1) & ~1;
  __shared__ double dgs[NQ];
  __shared__ __align__(16) double qs[kRWarps][ld1];
  __shared__ double rs[kRWarps][F];
  __shared__ double cs[kRWarps][KQ * 32];
  __shared__ double sqs[kRWarps];
  __shared__ bool last_cta;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool has_prev = a.prev_p >= 0, fin = a.cur_p < 0;
  if (threadIdx.x < kRWarps) sqs[threadIdx.x] = 0.0;
  if (has_prev)
    for (int t = threadIdx.x; t < NQ; t += blockDim.x) dgs[t] = a.prev_dg[t];
  if (threadIdx.x < kRWarps * ld1) (&qs[0][0])[threadIdx.x] = 0.0;
  __syncthreads();
  double cacc[KQ];
#pragma unroll
  for (int k = 0; k < KQ; ++k) cacc[k] = 0.0;
  const uint32_t stride = gridDim.x * kRWarps;
  for (uint32_t ci = blockIdx.x * kRWarps + warp; ci < a.csf.nchunks; ci += stride) {
    const Chunk ch = a.csf.chunks[ci];
    const double* arow = a.m.factor[2] + (size_t)ch.row * ld2;
    // first round's coordinates / residual in flight during the prologue
    uint32_t pos = ch.beg + lane;
    bool valid = pos < ch.end;
    uint32_t i1 = 0;
    double r = 0.0;
    if (valid) {
      i1 = __ldg(a.csf.oc[1] + pos);
      r = a.r[pos];
    }
    if (has_prev) {
      if (lane < F) {
        double t = 0.0;
#pragma unroll
        for (int c = 0; c < Jm; ++c) t = fma(__ldg(arow + c), dgs[lane * Jm + c], t);
        qs[warp][lane] = t;
      }
      __syncwarp();
    }
    double R[F];
#pragma unroll
    for (int f = 0; f < F; ++f) R[f] = 0.0;
    double sq = 0.0;
    for (uint32_t base = ch.beg; base < ch.end; base += 32) {
      // prefetch the next round
      const uint32_t npos = base + 32 + lane;
      const bool nvalid = npos < ch.end;
      uint32_t n1 = 0;
      double nr = 0.0;
      if (nvalid) {
        n1 = __ldg(a.csf.oc[1] + npos);
        nr = a.r[npos];
      }
      if (valid) {
        const double2* r1 = reinterpret_cast<const double2*>(a.m.factor[1] + (size_t)i1 * ld1);
        double u[ld1];
#pragma unroll
        for (int t = 0; t < ld1 / 2; ++t) {
          const double2 v = __ldg(r1 + t);
          u[2 * t] = v.x;
          u[2 * t + 1] = v.y;
        }
        if (has_prev) {
          const double wp = __ldcs(a.W + (uint64_t)a.prev_p * a.wstride + pos);
          const double2* q2 = reinterpret_cast<const double2*>(qs[warp]);
          double t = 0.0;
#pragma unroll
          for (int f2 = 0; f2 < ld1 / 2; ++f2) {
            const double2 q = q2[f2];
            t = fma(u[2 * f2], q.x, t);
            if (2 * f2 + 1 < F) t = fma(u[2 * f2 + 1], q.y, t);
          }
          r = fma(-wp, t, r);
          a.r[pos] = r;
        }
        if (fin || a.want_sq) sq = fma(r, r, sq);
        if (!fin) {
          const double wr = __ldcs(a.W + (uint64_t)a.cur_p * a.wstride + pos) * r;
#pragma unroll
          for (int f = 0; f < F; ++f) R[f] = fma(wr, u[f], R[f]);
        }
      }
      pos = npos;
      valid = nvalid;
      i1 = n1;
      r = nr;
    }
    if (fin) {
      sq = warp_sum(sq);
      if (lane == 0) a.chunk_sq[ci] = sq;
      continue;
    }
#pragma unroll
    for (int f = 0; f < F; ++f) {
      const double v = warp_sum(R[f]);
      if (lane == 0) rs[warp][f] = v;
    }
    if (a.want_sq) {
      sq = warp_sum(sq);
      if (lane == 0) sqs[warp] += sq;
    }
    __syncwarp();
#pragma unroll
    for (int k = 0; k < KQ; ++k) {
      const int q = lane + 32 * k;
      if (q < NQ) cacc[k] = fma(rs[warp][q / Jm], __ldg(arow + q % Jm), cacc[k]);
    }
    __syncwarp();
  }
  if (fin) return;
  // CTA partial: warps summed in order
#pragma unroll
  for (int k = 0; k < KQ; ++k) cs[warp][lane + 32 * k] = cacc[k];
  __syncthreads();
  constexpr int NP = NQ + 1;  // partial row: C, then sum r^2
  if (threadIdx.x < NQ) {
    double t = 0.0;
    for (int w = 0; w < kRWarps; ++w) t += cs[w][threadIdx.x];
    a.part[(size_t)blockIdx.x * NP + threadIdx.x] = t;
  } else if (threadIdx.x == NQ) {
    double t = 0.0;
    for (int w = 0; w < kRWarps; ++w) t += sqs[w];
    a.part[(size_t)blockIdx.x * NP + NQ] = t;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last_cta = atomicAdd(a.counter, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last_cta) return;
  __threadfence();
  // the last CTA: G groups of 128 threads each sum every G-th partial, then
  // the group sums are added in group order
  constexpr int G = kRWarps * 32 / 128;
  const int grp = threadIdx.x >> 7, q = threadIdx.x & 127;
  double t = 0.0;
  if (q < NP) {
    // four independent chains (fixed assignment): the loads overlap
    double t4[4] = {0.0, 0.0, 0.0, 0.0};
    uint32_t b = grp;
    for (; b + 3 * G < gridDim.x; b += 4 * G)
#pragma unroll
      for (int j = 0; j < 4; ++j) t4[j] += __ldcg(a.part + (size_t)(b + j * G) * NP + q);
    for (; b < gridDim.x; b += G) t4[0] += __ldcg(a.part + (size_t)b * NP + q);
    t = (t4[0] + t4[1]) + (t4[2] + t4[3]);
  }
  double* gs = &cs[0][0];  // reuse: [G][128]
  __syncthreads();
  gs[grp * 128 + q] = t;
  __syncthreads();
  if (threadIdx.x < NP) {
    double s2 = 0.0;
    for (int g2 = 0; g2 < G; ++g2) s2 += gs[g2 * 128 + threadIdx.x];
    a.cout[threadIdx.x] = s2;
  }
  if (threadIdx.x == 0) *a.counter = 0u;
}

// T_p for every prefix at once: out[(p, ff'), cc'] = sum_chunks S[chunk][(p, ff')]
// a_c a_c' on the FP64 tensor cores.  grid = (K splits, 64-row groups of the
// left operand); warp w owns the 8-row tile w of its group against all column
// tiles; per 32-chunk batch the statistics rows and the chunks' last-mode
// factor rows are prefetched into registers while the previous batch runs.
constexpr int kSgLd = 36;  // == 4 mod 16 doubles: conflict-free fragment loads
template <class S>
__global__ void __launch_bounds__(256) k_sall_gemm(const double* stats, int LW, const Chunk* chunks,
                                                   uint32_t nchunks, const double* A, double* partial) {
  constexpr int Jm = S::J(2), NAm = Jm * (Jm + 1) / 2, NT = (NAm + 7) / 8;
  constexpr int ld2 = (Jm + 1) & ~1;
  __shared__ double Lt[64 * kSgLd];
  __shared__ double Rt[NT * 8 * kSgLd];
  __shared__ double sa[32 * Jm];
  __shared__ int rmap[NT * 8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, tq = lane & 3;
  const int row0 = blockIdx.y * 64;
  for (int col = threadIdx.x; col < NT * 8; col += blockDim.x) {
    int v = -1;
    if (col < NAm) {
      int i, j;
      tri_pair(col, Jm, i, j);
      v = (i << 8) | j;
    }
    rmap[col] = v;
  }
  const uint32_t per = ((nchunks + gridDim.x - 1) / gridDim.x + 31) & ~31u;
  const uint32_t c0 = blockIdx.x * per;
  const uint32_t c1 = min(nchunks, c0 + per);
  double acc[NT][2];
#pragma unroll
  for (int t = 0; t < NT; ++t) acc[t][0] = acc[t][1] = 0.0;
  constexpr int kL = 64 * 32 / 256, kA = (32 * Jm + 255) / 256;
  double lv[kL], av[kA];
  auto prefetch = [&](uint32_t cb) {
    const int nb = (int)min(32u, c1 - cb);
#pragma unroll
    for (int i = 0; i < kL; ++i) {
      const int t = threadIdx.x + 256 * i;
      const int k = t >> 6, r = t & 63;
      lv[i] = (k < nb && row0 + r < LW) ? __ldcs(stats + (size_t)(cb + k) * LW + row0 + r) : 0.0;
    }
#pragma unroll
    for (int i = 0; i < kA; ++i) {
      const int t = threadIdx.x + 256 * i;
      const int k = t / Jm, c = t - k * Jm;
      av[i] = (t < 32 * Jm && k < nb) ? __ldg(A + (size_t)chunks[cb + k].row * ld2 + c) : 0.0;
    }
  };
  if (c0 < c1) prefetch(c0);
  for (uint32_t cb = c0; cb < c1; cb += 32) {
    __syncthreads();
#pragma unroll
    for (int i = 0; i < kL; ++i) {
      const int t = threadIdx.x + 256 * i;
      Lt[(t & 63) * kSgLd + (t >> 6)] = lv[i];
    }
#pragma unroll
    for (int i = 0; i < kA; ++i) {
      const int t = threadIdx.x + 256 * i;
      if (t < 32 * Jm) sa[t] = av[i];
    }
    __syncthreads();
    for (int t = threadIdx.x; t < NT * 8 * 32; t += 256) {
      const int col = t >> 5, k = t & 31;
      const int mp = rmap[col];
      Rt[col * kSgLd + k] = mp >= 0 ? sa[k * Jm + (mp >> 8)] * sa[k * Jm + (mp & 255)] : 0.0;
    }
    __syncthreads();
    if (cb + 32 < c1) prefetch(cb + 32);
    const double* la = Lt + (8 * warp + g) * kSgLd + tq;
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      const double av2 = la[4 * kk];
#pragma unroll
      for (int t = 0; t < NT; ++t) dmma884(acc[t][0], acc[t][1], av2, Rt[(8 * t + g) * kSgLd + tq + 4 * kk]);
    }
  }
  const int row = row0 + 8 * warp + g;
  if (row >= LW) return;
  double* out = partial + (size_t)blockIdx.x * LW * NAm + (size_t)row * NAm;
#pragma unroll
  for (int t = 0; t < NT; ++t)
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int col = 8 * t + 2 * tq + i;
      if (col < NAm) out[col] = acc[t][i];
    }
}

__global__ void k_colsum_s(const double* partial, int nparts, int n, double* out) {
  const int o = blockIdx.x * blockDim.x + threadIdx.x;
  if (o >= n) return;
  double t = 0.0;
  for (int p = 0; p < nparts; ++p) t += partial[(size_t)p * n + o];
  out[o] = t;
}

__host__ __device__ __forceinline__ int tri_s_host(int i, int j, int n) { return i * n - i * (i - 1) / 2 + (j - i); }
__device__ __forceinline__ int tri_s(int i, int j, int n) {  // i <= j
  return i * n - i * (i - 1) / 2 + (j - i);
}

// Block solve (updates.hpp:171-188 restricted to the block's cells, in
// ascending order): H_p expanded densely from T_p in shared memory by the
// whole CTA, then one warp runs the sequential Gauss-Seidel with the cells'
// state in registers (lane l holds cells l, l+32, ...): the owner lane solves
// its cell, the step broadcasts dg and every lane folds -dg H[q][q2] into the
// later cells' right-hand sides.  With s_out: the sum of squared residuals
// after this block's update, from the statistics alone,
//   sum (r - P dg)^2 = s_in - 2 dg.C + dg^T H dg   (C, s_in before the update),
// so the last block's residual pass can be deferred (Ctx::r_pending).
// Dense H_p[q][q2] (q = f*Jm + c) of every block from T_p's Kronecker-packed
// pairs, once per sweep (the solves then stream their block coalesced).
// Block p starts at H + p * hstride (hstride = nq^2 rounded up to even: every
// block 16-byte aligned for the solve's bulk copy).
__host__ __device__ constexpr size_t h_stride(int nq) { return ((size_t)nq * nq + 1) & ~(size_t)1; }
__global__ void k_expand_h(const double* T, int P, int nf, int Jm, double* H) {
  const int NAm = Jm * (Jm + 1) / 2, NS = nf * (nf + 1) / 2, nq = nf * Jm;
  const size_t n = (size_t)P * nq * nq;
  for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < n; t += (size_t)gridDim.x * blockDim.x) {
    const int p = (int)(t / ((size_t)nq * nq));
    const int r = (int)(t - (size_t)p * nq * nq);
    double* Hp = H + p * h_stride(nq);
    const int q = r / nq, q2 = r - q * nq;
    const int f = q / Jm, c = q - f * Jm, f2 = q2 / Jm, c2 = q2 - f2 * Jm;
    const int ps = f <= f2 ? tri_s(f, f2, nf) : tri_s(f2, f, nf);
    const int pa = c <= c2 ? tri_s(c, c2, Jm) : tri_s(c2, c, Jm);
    Hp[r] = T[((size_t)p * NS + ps) * NAm + pa];
  }
}

constexpr int kSolveK = 4;  // cells per lane: F * J_m <= 128
#ifdef VEST_SOLVE_CLOCKS
__device__ long long vest_solve_clocks[4];
#endif
constexpr int kSolveSlack = 128;  // doubles after H: unconditional row reads stay in bounds
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int REG>
__global__ void __launch_bounds__(32) k_core_solve_s(const double* Hg, const double* C, int nf, int Jm,
                                                     const uint32_t* fib, double* core,
                                                     const uint8_t* core_mask, double lambda,
                                                     double* dg_out, double* s_out) {
  constexpr int reg = REG;
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) uint64_t bar;
#ifdef VEST_SOLVE_CLOCKS
  long long tclk[6];
  tclk[0] = clock64();
#define VEST_TCLK(i) tclk[i] = clock64()
#else
#define VEST_TCLK(i)
#endif
  const int nq = nf * Jm;
  double* H = sm;                           // nq x nq (+ slack)
  double* dgs = H + nq * nq + kSolveSlack;  // nq (s_out only)
  // the block's dense H arrives by one bulk (TMA) copy while the lanes load
  // the cells' state
  const uint32_t bytes = ((uint32_t)(nq * nq) * 8u + 15u) & ~15u;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(H)),
        "l"(Hg), "r"(bytes), "r"(smem_u32(&bar))
        : "memory");
  }
  for (int t = (int)(bytes / 8) + threadIdx.x; t < nq * nq + kSolveSlack; t += 32) H[t] = 0.0;
  VEST_TCLK(1);
  VEST_TCLK(2);
  const int lane = threadIdx.x;
  double cc[kSolveK], c0[kSolveK], gv[kSolveK], hd[kSolveK], rd[kSolveK], dgl[kSolveK];
  bool mk[kSolveK], upd[kSolveK];
  int lin[kSolveK];
#pragma unroll
  for (int k = 0; k < kSolveK; ++k) {
    const int q = lane + 32 * k;
    cc[k] = gv[k] = hd[k] = rd[k] = dgl[k] = 0.0;
    mk[k] = true;
    lin[k] = 0;
    if (q < nq) {
      lin[k] = (int)fib[q / Jm] * Jm + q % Jm;
      cc[k] = C[q];
      gv[k] = core[lin[k]];
      mk[k] = core_mask[lin[k]] != 0;
    }
    c0[k] = cc[k];
  }
  VEST_TCLK(3);
  {
    uint32_t done = 0;
    while (!done)
      asm volatile(
          "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
          : "=r"(done)
          : "r"(smem_u32(&bar))
          : "memory");
  }
#pragma unroll
  for (int k = 0; k < kSolveK; ++k) {
    const int q = lane + 32 * k;
    if (q < nq) {
      hd[k] = H[q * nq + q];
      const double den = reg == 0 ? hd[k] + lambda : 2.0 * hd[k];
      rd[k] = den != 0.0 ? 1.0 / den : 0.0;
    }
    // a cell is updated unless masked or its denominator vanishes (then it keeps its value)
    upd[k] = !mk[k] && (reg == 0 ? hd[k] + lambda != 0.0 : 2.0 * hd[k] != 0.0);
  }
  const double* hrow = H + lane;  // row q of H, advanced by nq per step
  double hcur[kSolveK];
#pragma unroll
  for (int k2 = 0; k2 < kSolveK; ++k2) hcur[k2] = hrow[32 * k2];

  // Sequential over the cells, branch-free per step: every lane evaluates its
  // own slot-k cell, the owner's (lane lo) dg is broadcast, all lanes fold it
  // into the later cells (dg == 0 folds to a no-op).
#pragma unroll
  for (int k = 0; k < kSolveK; ++k) {
    if (32 * k >= nq) break;
#pragma unroll
    for (int lo = 0; lo < 32; ++lo) {
      const int q = 32 * k + lo;
      if (q >= nq) break;
      const double g_old = gv[k];
      const double num = cc[k] + g_old * hd[k];
      double g_new;
      if (reg == 0) {
        g_new = num * rd[k];
      } else {
        const double gg = -2.0 * num;
        g_new = gg > lambda ? (lambda - gg) * rd[k] : (gg < -lambda ? -(lambda + gg) * rd[k] : 0.0);
      }
      if (!upd[k]) g_new = g_old;
      const double dg = __shfl_sync(0xffffffffu, g_new - g_old, lo);  // (x - x == +0: no-op fold)
      if (lane == lo) {
        gv[k] = g_new;
        dgl[k] = dg;
        dg_out[q] = dg;
      }
      // cells q2 <= q (and past nq) are finished / absent: folding into
      // their right-hand sides is harmless, so no predicate on the chain
#pragma unroll
      for (int k2 = k; k2 < kSolveK; ++k2) cc[k2] = fma(-dg, hcur[k2], cc[k2]);
      hrow += nq;
#pragma unroll
      for (int k2 = 0; k2 < kSolveK; ++k2) hcur[k2] = hrow[32 * k2];  // next row, off the chain
    }
  }
  VEST_TCLK(4);
#pragma unroll
  for (int k = 0; k < kSolveK; ++k)
    if (lane + 32 * k < nq && !mk[k]) core[lin[k]] = gv[k];
#ifdef VEST_SOLVE_CLOCKS
  if (lane == 0)
    for (int i = 1; i < 5; ++i) vest_solve_clocks[i - 1] = tclk[i] - tclk[i - 1];
#endif
  if (!s_out) return;
  // s_in - 2 dg.C + dg^T H dg
#pragma unroll
  for (int k = 0; k < kSolveK; ++k)
    if (lane + 32 * k < nq) dgs[lane + 32 * k] = dgl[k];
  __syncwarp();
  double acc = 0.0;
#pragma unroll
  for (int k = 0; k < kSolveK; ++k) {
    const int q = lane + 32 * k;
    if (q < nq && dgl[k] != 0.0) {
      const double* hr = H + q * nq;
      double hv = 0.0;
      for (int q2 = 0; q2 < nq; ++q2) hv = fma(hr[q2], dgs[q2], hv);
      acc = fma(dgl[k], hv - 2.0 * c0[k], acc);
    }
  }
  acc = warp_sum(acc);
  if (lane == 0) *s_out = C[nq] + acc;
}

// ---------------------------------------------------------------- dispatch --
template <class S>
cudaError_t run_core_pass_s(const CorePassSArgs& a, cudaStream_t s) {
  if (a.csf.nchunks == 0) return cudaSuccess;
  const dim3 grid((a.csf.nchunks + kSWarps - 1) / kSWarps);
  k_core_pass_s<S><<<grid, kSWarps * 32, 0, s>>>(a);
  count_launch();
  return cudaGetLastError();
}

template <class S>
cudaError_t run_pack_uw(const DevModel& m, const DevCSF& csf, uint64_t p0, uint64_t p1, double* U, double* W,
                        uint64_t wstride, cudaStream_t s) {
  if (p1 > p0) {
    k_pack_uw<S><<<1184, 256, 0, s>>>(m, csf, p0, p1, U, W, wstride);
    count_launch();
  }
  return cudaGetLastError();
}

template <class S>
cudaError_t run_core_sall(const DevModel& m, const DevCSF& csf, double* stats, double* W, uint64_t wstride,
                          int grid, cudaStream_t s) {
  if (csf.nchunks == 0) return cudaSuccess;
  constexpr int LDR = sall_ldr(S::J(0), S::J(1));
  const int smem = kAllWarps * 2 * 32 * LDR * (int)sizeof(double);
  cudaFuncSetAttribute(k_core_sall<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k_core_sall<S><<<grid, kAllWarps * 32, smem, s>>>(m, csf, stats, W, wstride);
  count_launch();
  return cudaGetLastError();
}

template <class S>
cudaError_t run_core_rpass(const RPassArgs& a, int grid, cudaStream_t s) {
  k_core_rpass<S><<<grid, kRWarps * 32, 0, s>>>(a);
  count_launch();
  return cudaGetLastError();
}

template <class S>
cudaError_t run_sall_gemm(const double* stats, int LW, const Chunk* chunks, uint32_t nchunks, const double* A,
                          double* partial, int ksplit, cudaStream_t s) {
  const dim3 grid(ksplit, (LW + 63) / 64);
  k_sall_gemm<S><<<grid, 256, 0, s>>>(stats, LW, chunks, nchunks, A, partial);
  count_launch();
  return cudaGetLastError();
}

struct CoreSOps {
  int N;
  int J[VEST_MAXN];
  cudaError_t (*pass)(const CorePassSArgs& a, cudaStream_t s);
  cudaError_t (*pack)(const DevModel& m, const DevCSF& csf, uint64_t p0, uint64_t p1, double* U, double* W,
                      uint64_t wstride, cudaStream_t s);
  cudaError_t (*sall)(const DevModel& m, const DevCSF& csf, double* stats, double* W, uint64_t wstride, int grid,
                      cudaStream_t s);
  cudaError_t (*rpass)(const RPassArgs& a, int grid, cudaStream_t s);
  cudaError_t (*sgemm)(const double* stats, int LW, const Chunk* chunks, uint32_t nchunks, const double* A,
                       double* partial, int ksplit, cudaStream_t s);
};

template <int... Js>
constexpr CoreSOps make_core_ops() {
  CoreSOps o{};
  o.N = sizeof...(Js);
  const int js[] = {Js...};
  for (int k = 0; k < (int)sizeof...(Js); ++k) o.J[k] = js[k];
  o.pass = &run_core_pass_s<SShape<Js...>>;
  o.pack = &run_pack_uw<SShape<Js...>>;
  o.sall = &run_core_sall<SShape<Js...>>;
  o.rpass = &run_core_rpass<SShape<Js...>>;
  o.sgemm = &run_sall_gemm<SShape<Js...>>;
  return o;
}

static const CoreSOps kCoreOps[] = {
    make_core_ops<5, 5, 5>(),
    make_core_ops<10, 10, 10>(),
    make_core_ops<10, 10, 5>(),
};

const void* find_core_ops(int N, const int* J) {
  for (const auto& o : kCoreOps) {
    if (o.N != N) continue;
    bool eq = true;
    for (int k = 0; k < N; ++k) eq = eq && o.J[k] == J[k];
    if (eq) return &o;
  }
  return nullptr;
}

cudaError_t core_pack_structured(const void* ops, const DevModel& m, const DevCSF& csf, uint64_t p0, uint64_t p1,
                                 double* U, double* W, uint64_t wstride, cudaStream_t s) {
  return static_cast<const CoreSOps*>(ops)->pack(m, csf, p0, p1, U, W, wstride, s);
}

cudaError_t core_pass_structured(const void* ops, const DevModel& m, const DevCSF& csf, double* r, int prev_p,
                                 const double* prev_dg, int cur_p, int kind, double* stats, int stride,
                                 double* chunk_sq, const double* U, const double* W, uint64_t wstride,
                                 cudaStream_t s) {
  CorePassSArgs a{};
  a.U = U;
  a.W = W;
  a.wstride = wstride;
  a.m = m;
  a.csf = csf;
  a.r = r;
  a.prev_p = prev_p;
  a.prev_dg = prev_dg;
  a.cur_p = cur_p;
  a.kind = kind;
  a.stats = stats;
  a.stride = stride;
  a.chunk_sq = chunk_sq;
  return static_cast<const CoreSOps*>(ops)->pass(a, s);
}

}  // namespace vest

namespace vest {

// ------------------------------------------------- all-prefix sweep (host) --
// Structured core sweep for 3-mode static shapes (see k_core_sall): one
// all-prefix statistics pass, one GEMM for every block Gram, then per live
// block a residual/R pass and the register Gauss-Seidel solve.
static int rpass_grid(Ctx& c) {
  int sms = 0, occ = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c.device);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_core_rpass<SShape<10, 10, 10>>, kRWarps * 32, 0);
  return std::max(1, std::min(occ, VEST_RPASS_MINB)) * sms;  // (the last CTA sums grid partials)
}

static RPassArgs rpass_args(Ctx& c, int prev_p, int cur_p, double* part, double* cout, int want_sq) {
  RPassArgs a{};
  a.m = c.model_view();
  a.csf = c.csf_view(c.N - 1);
  a.r = c.d_r;
  a.prev_p = prev_p;
  a.prev_dg = c.d_dg;
  a.cur_p = cur_p;
  a.chunk_sq = c.d_chunk_sum;
  a.part = part;
  a.cout = cout;
  a.counter = c.d_counter;
  a.W = c.d_pack_w;
  a.wstride = c.nnz;
  a.want_sq = want_sq;
  return a;
}

void core_sweep_sall(Ctx& c, const void* ops_, int reg, double lambda, const std::vector<int>& prefixes,
                     const std::vector<int>& starts) {
  const CoreSOps* ops = static_cast<const CoreSOps*>(ops_);
  const int m = c.N - 1;
  const int P = c.ranks[0], F = c.ranks[1], Jm = c.ranks[2];
  const int NV = F * (F + 1) / 2, NAm = Jm * (Jm + 1) / 2, LW = P * NV, nq = F * Jm;
  const DevCSF csf = c.csf_view(m);
  const DevModel mv = c.model_view();
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c.device);
  const size_t nT = (size_t)LW * NAm;
  const int ksplit = std::max(1, std::min<int>(64, (int)((csf.nchunks + 1023) / 1024)));
  const int rgrid = rpass_grid(c);
  ensure(c, &c.d_chunk_stats, &c.chunk_stats_cap, (size_t)csf.nchunks * LW + 1);
  ensure(c, &c.d_pack_w, &c.pack_w_cap, (size_t)c.nnz * P + 1);
  ensure(c, &c.d_gemm_part, &c.gemm_part_cap, std::max((size_t)ksplit * nT, (size_t)rgrid * (nq + 1)) + 1);
  const size_t nH = (size_t)P * h_stride(nq) + 2;  // (+2: the bulk copy rounds up to 16 bytes)
  ensure(c, &c.d_gemm_out, &c.gemm_out_cap, nT + 1 + nH + nq + 2);
  ensure(c, &c.d_dg, &c.dg_cap, (size_t)16 * VEST_MAXJ);
  ensure(c, &c.d_chunk_sum, &c.chunk_sum_cap, c.modes[m].nchunks + 1);
  if (!c.d_counter) {
    check(cudaMalloc(&c.d_counter, sizeof(unsigned)), "sweep counter");
    check(cudaMemsetAsync(c.d_counter, 0, sizeof(unsigned), c.stream), "sweep counter");
  }
  double* T = c.d_gemm_out;
  double* Hd = c.d_gemm_out + ((nT + 1) & ~(size_t)1);  // dense H_p of every block (16-byte aligned)
  double* Cb = Hd + nH;                                    // [C (nq) | sum r^2]
  {
    ProfScope ps(c, kProfCorePass);
    check(ops->sall(mv, csf, c.d_chunk_stats, c.d_pack_w, c.nnz, 2 * sms, c.stream),
          "core all-prefix statistics");
  }
  {
    ProfScope ps(c, kProfCoreGemm);
    if (csf.nchunks > 0) {
      check(ops->sgemm(c.d_chunk_stats, LW, csf.chunks, csf.nchunks, mv.factor[m], c.d_gemm_part, ksplit,
                       c.stream),
            "core all-prefix gemm");
      k_colsum_s<<<(unsigned)((nT + 255) / 256), 256, 0, c.stream>>>(c.d_gemm_part, ksplit, (int)nT, T);
      count_launch();
    } else {
      check(cudaMemsetAsync(T, 0, nT * sizeof(double), c.stream), "core gemm (empty)");
    }
    check(cudaGetLastError(), "core all-prefix gemm");
  }
  comm_allreduce(c, T, (uint64_t)nT);
  {
    ProfScope ps(c, kProfCoreGemm);
    k_expand_h<<<(unsigned)std::min<size_t>(4096, (nH + 255) / 256), 256, 0, c.stream>>>(T, P, F, Jm, Hd);
    count_launch();
    check(cudaGetLastError(), "core expand H");
  }
  const size_t smem = ((size_t)nq * nq + kSolveSlack + nq) * sizeof(double);
  auto solve = reg == 0 ? k_core_solve_s<0> : k_core_solve_s<1>;
  check(cudaFuncSetAttribute(solve, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "solve smem");
  const int nb = (int)prefixes.size();
  for (int bi = 0; bi < nb; ++bi) {
    const bool last = bi == nb - 1;
    {
      ProfScope ps(c, kProfCorePass);
      if (csf.nchunks > 0) {
        const RPassArgs a = rpass_args(c, bi > 0 ? prefixes[bi - 1] : -1, prefixes[bi], c.d_gemm_part, Cb, last);
        check(ops->rpass(a, rgrid, c.stream), "core block pass");
      } else {
        check(cudaMemsetAsync(Cb, 0, (nq + 1) * sizeof(double), c.stream), "core block pass (empty)");
      }
    }
    comm_allreduce(c, Cb, (uint64_t)nq + 1);  // C and (last block) sum r^2 over the shards
    ProfScope ps(c, kProfCoreSolve);
    solve<<<1, 32, smem, c.stream>>>(Hd + (size_t)prefixes[bi] * h_stride(nq), Cb, F, Jm, c.d_fibers + starts[bi],
                                      c.d_core, c.d_core_mask, lambda, c.d_dg, last ? c.d_small : nullptr);
    count_launch();
    check(cudaGetLastError(), "core solve");
  }
  // sum r^2 after the last block from its statistics; r itself lacks that
  // block's update until someone reads it (core_apply_pending)
  check(cudaMemcpyAsync(c.h_small, c.d_small, sizeof(double), cudaMemcpyDeviceToHost, c.stream), "sum readback");
  check(cudaStreamSynchronize(c.stream), "sum sync");
  c.sum_sq = std::max(0.0, c.h_small[0]);
  c.re = std::sqrt(c.sum_sq) / c.x_norm;
  c.r_valid = false;
  c.r_fresh = false;
  c.r_pending = prefixes[nb - 1];
  c.r_pending_ops = ops_;
}

// Apply the deferred last-block update to r (and recompute sum r^2 exactly).
bool core_apply_pending(Ctx& c) {
  if (c.r_pending < 0) return false;
  const CoreSOps* ops = static_cast<const CoreSOps*>(c.r_pending_ops);
  const DevCSF csf = c.csf_view(c.N - 1);
  if (csf.nchunks > 0) {
    ProfScope ps(c, kProfResid);
    const RPassArgs a = rpass_args(c, c.r_pending, -1, c.d_gemm_part, nullptr, 0);
    check(ops->rpass(a, rpass_grid(c), c.stream), "core pending update");
  }
  c.sum_sq = reduce_chunk_sums(c, c.d_chunk_sum, c.modes[c.N - 1].nchunks);
  c.re = std::sqrt(c.sum_sq) / c.x_norm;
  c.r_valid = true;
  c.r_fresh = true;
  c.r_pending = -1;
  return true;
}

}  // namespace vest
