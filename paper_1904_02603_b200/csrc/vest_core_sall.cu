// SPDX-License-Identifier: Apache-2.0
// vest_core_sall.cu -- the exact core sweep (updates.hpp:159-195: cells in
// ascending order, each solved with the fresh values of all earlier cells)
// for 3-mode compile-time ranks, organised around the FP64 tensor cores.
//
// Blocks: block p = the F * J_2 cells with beta_0 = p (consecutive in the
// reference's row-major order).  Exact Gauss-Seidel over the blocks needs,
// per block, its Gram H_p = sum_e P_p(e) P_p(e)^T and C_p = sum_e P_p(e) r(e)
// with r already carrying every earlier block's update.  With
//   P_{p,(f,c)}(e) = w_p(e) u_f(e) a_c(e),  w_p = A_0[i_0,p], u = A_1[i_1,:],
//   a = A_2[i_2,:]   (i_2 = the slice = the chunk's row),
// the Grams factor through per-slice statistics
//   H_p = sum_slices S_p (x) a a^T,  S_p[(f,f')] = sum_{e in slice} w_p^2 u_f u_f',
// which depend only on the (fixed) factors: ONE pass (k_core_sall) computes
// them for every block at once and ONE GEMM (k_sall_gemm) turns them into
// every H_p.  The DMMA tiles of that pass have 16 rows for the P = 10 block
// weights; the spare rows carry the cross weights w_{2x} w_{2x+1}, whose
// Grams H_{2x,2x+1} couple the two blocks of a pair group.  A group (one or
// two consecutive live blocks) then costs one residual pass (k_core_rpass:
// apply the previous group's updates to r, accumulate C for both blocks) and
// one solve (k_core_solve_g: block a; C_b -= H_ba dg_a; block b).  The last
// group's residual update is deferred (Ctx::r_pending): the sum of squared
// residuals follows from the statistics (s - 2 dg.C + dg^T H dg).
#include <algorithm>
#include <vector>

#include "vest_common.cuh"

namespace vest {

namespace {

// ----------------------------------------------------------------- helpers --
// pair index p of the row-major upper triangle of an n x n matrix -> (i, j)
__host__ __device__ inline void tri_pair(int p, int n, int& i, int& j) {
  int r = p;
  i = 0;
  while (r >= n - i) {
    r -= n - i;
    ++i;
  }
  j = i + r;
}
__host__ __device__ constexpr int tri_idx(int i, int j, int n) {  // i <= j
  return i * n - i * (i - 1) / 2 + (j - i);
}
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}
// factor-row gathers: through L1 (.ca) -- under skewed coordinates (Zipf) a
// few hot rows take a large share of the gathers, which L2-only copies would
// funnel into the same L2 slices
__device__ __forceinline__ void cp_async16_ca(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async16_row(void* smem, const void* gmem, bool via_l1) {
  if (via_l1) cp_async16_ca(smem, gmem);
  else cp_async16(smem, gmem);
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

__device__ __forceinline__ void mbar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// one bulk (TMA) global -> shared copy completing on `bar`
__device__ __forceinline__ void bulk_copy(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done)
                 : "r"(smem_u32(bar)), "r"(parity)
                 : "memory");
}

// A rows of the statistics: w_p^2 (P), then w_{2x} w_{2x+1} (X = P / 2)
__host__ __device__ constexpr int sall_rows(int P) { return P + P / 2; }
__host__ __device__ constexpr int sall_arow(int P) { return (sall_rows(P) + 7) / 8 * 8; }
// staged row [A (arow) | u (ld1) | pad], stride == 4 (mod 8) doubles: the DMMA
// fragment loads (4 rows x 4 consecutive doubles per quarter) are conflict-free
__host__ __device__ constexpr int sall_ldr(int P, int F) {
  return sall_arow(P) + ((F + 1) & ~1) + ((4 - (sall_arow(P) + ((F + 1) & ~1)) % 8) + 8) % 8;
}
// dense H blocks are 16-byte aligned (bulk copies)
__host__ __device__ constexpr size_t h_stride(int nq) { return ((size_t)nq * nq + 1) & ~(size_t)1; }

constexpr int kAllWarps = 4;    // k_core_sall warps per CTA
#ifndef VEST_RPASS_RE
#define VEST_RPASS_RE 1  // RE=2: 14% fewer instructions but lower occupancy, measured no faster
#endif
constexpr int kRE = VEST_RPASS_RE;  // k_core_rpass entries per lane per round
constexpr int kRRound = 32 * kRE;
constexpr int kRWarps = kRE > 1 ? 4 : 8;  // k_core_rpass warps per CTA (staging smem)
constexpr int kSgLd = 36;       // k_sall_gemm staging stride (== 4 mod 16)
constexpr int kSolveK = 4;      // solve: cells per lane, F * J_m <= 128
constexpr int kSolveSlack = 128;  // doubles after each H buffer (unconditional row reads)

// ------------------------------------------------------------ statistics --
// S_r[(f,f')] for every A row r of one chunk (slice) per warp, persistent
// over chunks.  Rounds of 32 entries: the raw factor rows are staged into a
// double buffer by cp.async one round ahead (coordinates two rounds ahead),
// a fix-up turns the raw w into the A rows (and emits W, SoA, for the
// residual passes), then X_A^T X_B over the round's 4-entry k-steps runs on
// DMMA with B = u_i u_j formed from the staged u at fragment load.
template <class S>
__global__ void __launch_bounds__(kAllWarps * 32) k_core_sall(DevModel m, DevCSF csf, double* stats, double* W,
                                                              uint64_t wstride, int hot) {
  static_assert(S::N == 3, "all-prefix statistics: 3-mode shapes");
  constexpr int P = S::J(0), F = S::J(1), NV = F * (F + 1) / 2;
  constexpr int X = P / 2, R = sall_rows(P), AR = sall_arow(P);
  constexpr int ld0 = (P + 1) & ~1, ld1 = (F + 1) & ~1;
  constexpr int LDR = sall_ldr(P, F);
  constexpr int MT = AR / 8, NT = (NV + 7) / 8;
  static_assert(ld0 <= AR, "raw weights land in the A region");
  extern __shared__ __align__(16) double sall_smem[];  // [warp][2][32 * LDR]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* const stage0 = sall_smem + (size_t)warp * 2 * 32 * LDR;
  const int g = lane >> 2, tq = lane & 3;
  int bi[NT], bj[NT];  // this lane's B-fragment pair (u offsets), per column tile
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    bi[nt] = bj[nt] = -1;
    if (8 * nt + g < NV) tri_pair(8 * nt + g, F, bi[nt], bj[nt]);
  }
  const uint32_t stride = gridDim.x * kAllWarps;
  struct Cur {
    uint32_t ci, end, base;
  };
  auto first = [&](uint32_t ci) {
    Cur c{ci, 0, 0};
    if (ci < csf.nchunks) {
      const Chunk ch = csf.chunks[ci];
      c.end = ch.end;
      c.base = ch.beg;
    }
    return c;
  };
  auto next = [&](const Cur& c) {
    if (c.base + 32 < c.end) return Cur{c.ci, c.end, c.base + 32};
    return first(c.ci + stride);
  };
  auto coords = [&](const Cur& c, uint32_t& i0, uint32_t& i1) {
    i0 = i1 = 0;
    if (c.ci < csf.nchunks && c.base + lane < c.end) {
      i0 = __ldg(csf.oc[0] + c.base + lane);
      i1 = __ldg(csf.oc[1] + c.base + lane);
    }
  };
  auto issue = [&](const Cur& c, int b, uint32_t i0, uint32_t i1) {
    double* row = stage0 + b * 32 * LDR + lane * LDR;
    if (c.ci < csf.nchunks && c.base + lane < c.end) {
      const double* r0 = m.factor[0] + (size_t)i0 * ld0;
      const double* r1 = m.factor[1] + (size_t)i1 * ld1;
#pragma unroll
      for (int t = 0; t < ld0 / 2; ++t) cp_async16_row(row + 2 * t, r0 + 2 * t, hot & 1);
#pragma unroll
      for (int t = 0; t < ld1 / 2; ++t) cp_async16_row(row + AR + 2 * t, r1 + 2 * t, hot & 2);
    } else {
#pragma unroll
      for (int t = 0; t < LDR; ++t) row[t] = 0.0;  // zero weights: no contribution
    }
  };

  Cur cur = first(blockIdx.x * kAllWarps + warp);
  if (cur.ci >= csf.nchunks) return;
  {
    uint32_t a0, a1;
    coords(cur, a0, a1);
    issue(cur, 0, a0, a1);
  }
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
    cp_async_wait_all();
    __syncwarp();
    {  // fix-up: raw w -> W (SoA) and the A rows
      double* row = stage0 + buf * 32 * LDR + lane * LDR;
      const uint32_t pos = cur.base + lane;
      if (pos < cur.end) {
        double w[ld0];
#pragma unroll
        for (int t = 0; t < ld0 / 2; ++t) {
          const double2 v = reinterpret_cast<const double2*>(row)[t];
          w[2 * t] = v.x;
          w[2 * t + 1] = v.y;
        }
#pragma unroll
        for (int p = 0; p < P; ++p) __stcs(W + (uint64_t)p * wstride + pos, w[p]);
        double av[AR];
#pragma unroll
        for (int p = 0; p < AR; ++p) av[p] = 0.0;
#pragma unroll
        for (int p = 0; p < P; ++p) av[p] = w[p] * w[p];
#pragma unroll
        for (int x = 0; x < X; ++x) av[P + x] = w[2 * x] * w[2 * x + 1];
#pragma unroll
        for (int t = 0; t < AR / 2; ++t) reinterpret_cast<double2*>(row)[t] = make_double2(av[2 * t], av[2 * t + 1]);
      }
    }
    __syncwarp();
    const bool more = nxt.ci < csf.nchunks;
    if (more) issue(nxt, buf ^ 1, n0, n1);
    const Cur nn = more ? next(nxt) : nxt;
    uint32_t m0 = 0, m1 = 0;
    if (more) coords(nn, m0, m1);
    {
      const double* st = stage0 + buf * 32 * LDR;
      const int nk = (int)(min(32u, cur.end - cur.base) + 3) >> 2;
#pragma unroll 2
      for (int kk = 0; kk < nk; ++kk) {
        const double* row = st + (4 * kk + tq) * LDR;
        double a[MT];
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) a[mt] = row[8 * mt + g];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const double b = bi[nt] >= 0 ? row[AR + bi[nt]] * row[AR + bj[nt]] : 0.0;
#pragma unroll
          for (int mt = 0; mt < MT; ++mt) dmma884(acc[mt][nt][0], acc[mt][nt][1], a[mt], b);
        }
      }
    }
    if (!more || nxt.ci != cur.ci) {  // chunk finished: its statistics
      double* out = stats + (size_t)cur.ci * (R * NV);
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const int rr = 8 * mt + g, pr = 8 * nt + 2 * tq + i;
            if (rr < R && pr < NV) out[rr * NV + pr] = acc[mt][nt][i];
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

// ------------------------------------------------------------------ GEMM --
// Every block Gram at once: out[(r, ff'), cc'] = sum_chunks S[chunk][(r, ff')]
// a_c a_c' on DMMA.  grid = (K splits, 128-row groups); warp w owns the 8-row
// tiles w and w + 8 of its group against all column tiles (each B fragment
// feeds two MMAs); the next 32-chunk batch is prefetched into registers while
// the current one runs.
constexpr int kSgRows = 128;
// staging element t -> (row r, chunk k): each warp access covers 8 rows x 4
// chunks, i.e. 4 runs of 8 consecutive doubles in global memory and 2-way
// (minimal) bank use in the transposed tile (row stride kSgLd == 4 mod 16)
__device__ __forceinline__ void lt_coord(int t, int& r, int& k) {
  const int lane = t & 31, wi = t >> 5;
  r = (wi % (kSgRows / 8)) * 8 + (lane & 7);
  k = (wi / (kSgRows / 8)) * 4 + (lane >> 3);
}
template <class S>
__global__ void __launch_bounds__(256) k_sall_gemm(const double* stats, int LW, const Chunk* chunks,
                                                   uint32_t nchunks, const double* A, double* partial) {
  constexpr int Jm = S::J(2), NAm = Jm * (Jm + 1) / 2, NT = (NAm + 7) / 8;
  constexpr int ld2 = (Jm + 1) & ~1;
  extern __shared__ __align__(16) double sg_smem[];
  double* Lt = sg_smem;                    // [kSgRows][kSgLd]
  double* Rt = Lt + kSgRows * kSgLd;       // [NT * 8][kSgLd]
  double* sa = Rt + NT * 8 * kSgLd;        // [32][Jm]
  __shared__ int rmap[NT * 8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, tq = lane & 3;
  const int row0 = blockIdx.y * kSgRows;
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
  double acc[2][NT][2];
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int t = 0; t < NT; ++t) acc[h][t][0] = acc[h][t][1] = 0.0;
  constexpr int kL = kSgRows * 32 / 256, kA = (32 * Jm + 255) / 256;
  double lv[kL], av[kA];
  auto prefetch = [&](uint32_t cb) {
    const int nb = (int)min(32u, c1 - cb);
#pragma unroll
    for (int i = 0; i < kL; ++i) {
      int r, k;
      lt_coord(threadIdx.x + 256 * i, r, k);
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
      int r, k;
      lt_coord(threadIdx.x + 256 * i, r, k);
      Lt[r * kSgLd + k] = lv[i];
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
    const double* la0 = Lt + (8 * warp + g) * kSgLd + tq;
    const double* la1 = Lt + (8 * (warp + 8) + g) * kSgLd + tq;
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      const double a0 = la0[4 * kk], a1 = la1[4 * kk];
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        const double b = Rt[(8 * t + g) * kSgLd + tq + 4 * kk];
        dmma884(acc[0][t][0], acc[0][t][1], a0, b);
        dmma884(acc[1][t][0], acc[1][t][1], a1, b);
      }
    }
  }
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int row = row0 + 8 * (warp + 8 * h) + g;
    if (row >= LW) continue;
    double* out = partial + (size_t)blockIdx.x * LW * NAm + (size_t)row * NAm;
#pragma unroll
    for (int t = 0; t < NT; ++t)
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int col = 8 * t + 2 * tq + i;
        if (col < NAm) out[col] = acc[h][t][i];
      }
  }
}

template <class S>
constexpr int sgemm_smem() {
  constexpr int NT = (S::J(2) * (S::J(2) + 1) / 2 + 7) / 8;
  return (kSgRows * kSgLd + NT * 8 * kSgLd + 32 * S::J(2)) * (int)sizeof(double);
}

__global__ void k_colsum_s(const double* partial, int nparts, int n, double* out) {
  const int o = blockIdx.x * blockDim.x + threadIdx.x;
  if (o >= n) return;
  double t = 0.0;
  for (int p = 0; p < nparts; ++p) t += partial[(size_t)p * n + o];
  out[o] = t;
}

// Dense H[q][q2] (q = f*Jm + c) of every A row's block from its Kronecker-
// packed pairs, once per sweep: rows p < P are the diagonal blocks H_pp,
// rows P + x the cross blocks H_{2x,2x+1} (symmetric in q <-> q2).
__global__ void k_expand_h(const double* T, int nblk, int nf, int Jm, double* H) {
  const int NAm = Jm * (Jm + 1) / 2, NS = nf * (nf + 1) / 2, nq = nf * Jm;
  const size_t n = (size_t)nblk * nq * nq;
  for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < n; t += (size_t)gridDim.x * blockDim.x) {
    const int p = (int)(t / ((size_t)nq * nq));
    const int r = (int)(t - (size_t)p * nq * nq);
    const int q = r / nq, q2 = r - q * nq;
    const int f = q / Jm, c = q - f * Jm, f2 = q2 / Jm, c2 = q2 - f2 * Jm;
    const int ps = f <= f2 ? tri_idx(f, f2, nf) : tri_idx(f2, f, nf);
    const int pa = c <= c2 ? tri_idx(c, c2, Jm) : tri_idx(c2, c, Jm);
    H[p * h_stride(nq) + r] = T[((size_t)p * NS + ps) * NAm + pa];
  }
}

// -------------------------------------------------------- residual pass --
struct RPassArgs {
  DevModel m;
  DevCSF csf;             // mode N-1
  double* r;
  int prev_p[2];          // previous group's prefixes (-1: none)
  const double* prev_dg;  // [2][F*Jm]
  int cur_p[2];           // current group's prefixes (cur_p[0] < 0: final pass)
  double* chunk_sq;       // final pass: per-chunk sum of r^2
  double* part;           // [gridDim.x][2*F*Jm + 1] CTA partials
  double* cout;           // [C_a (F*Jm) | C_b (F*Jm) | sum r^2]
  unsigned* counter;      // CTA arrival counter (self-resetting)
  const double* W;        // [P][wstride] block weights A_0[i_0, p] (k_core_sall)
  uint64_t wstride;
  int want_sq;            // also sum r^2 (after the previous group's update)
  int hot;                // bit k: mode k is skewed (its row gathers go through L1)
};

// One pair group: r -= sum_prev w_p (u . q_p) (q_p = dg_p a per slice), then
// R_j = sum w_{cur j} r u per chunk and C_j[f][c] += R_j[f] a_c.  Rounds of 32
// entries, flattened over the warp's chunks, are staged into a double buffer
// by cp.async one round ahead (u rows gathered from L2; the weights and the
// residual streamed; the slice's A_2 row), coordinates two rounds ahead, so
// the FMAs never wait on memory.  The CTAs' partials are summed in a fixed
// order by the last CTA to arrive (deterministic, no extra launch).
#ifndef VEST_RPASS_MINB
#define VEST_RPASS_MINB 2
#endif
template <int F, int Jm>
struct RStage {  // one round's staged operands (kRRound entries), per warp (doubles)
  static constexpr int ld1 = (F + 1) & ~1, ld2 = (Jm + 1) & ~1;
  static constexpr int U = 0;                   // [kRRound][ld1]
  static constexpr int Wv = U + kRRound * ld1;  // [4][kRRound]: prev_a, prev_b, cur_a, cur_b
  static constexpr int Rr = Wv + 4 * kRRound;   // [kRRound]
  static constexpr int A2 = Rr + kRRound;       // [ld2]
  static constexpr int size = (A2 + ld2 + 1) & ~1;
};
// v[i] summed over the warp, scattered: lane l returns with v[0] = sum of v[l]
// (5 butterfly rounds exchanging 16, 8, 4, 2, 1 values)
__device__ __forceinline__ void transpose_reduce(double (&v)[32], int lane) {
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) {
    const bool hi = lane & s;
#pragma unroll
    for (int i = 0; i < s; ++i) {
      const double send = hi ? v[i] : v[i + s];
      const double keep = hi ? v[i + s] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, s);
    }
  }
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}

template <class S>
__global__ void __launch_bounds__(kRWarps * 32, VEST_RPASS_MINB) k_core_rpass(RPassArgs a) {
  static_assert(S::N == 3, "block pass: 3-mode shapes");
  constexpr int F = S::J(1), Jm = S::J(2), NQ = F * Jm;
  constexpr int NC = 2 * NQ, NP = NC + 1, KC = (NC + 31) / 32;
  static_assert(2 * F + 1 <= 32, "chunk sums fit one reduce-scatter");
  using RS = RStage<F, Jm>;
  constexpr int ld1 = RS::ld1, ld2 = RS::ld2;
  extern __shared__ __align__(16) double rp_smem[];  // [warp][2][RS::size]
  __shared__ double dgs[2][NQ];
  __shared__ __align__(16) double qs[kRWarps][2][ld1];
  __shared__ double as[kRWarps][ld2];  // the current chunk's A_2 row
  __shared__ double rs[kRWarps][2][F];
  constexpr int KS = (NP + 31) / 32;  // >= KC: the final reduction reuses cs
  __shared__ double cs[kRWarps][KS * 32];
  __shared__ double sqs[kRWarps];
  __shared__ bool last_cta;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* const st0 = rp_smem + (size_t)warp * 2 * RS::size;
  const int np = (a.prev_p[0] >= 0) + (a.prev_p[1] >= 0);
  const int nc = (a.cur_p[0] >= 0) + (a.cur_p[1] >= 0);
  const bool fin = nc == 0;
  const int wrow[4] = {a.prev_p[0], a.prev_p[1], a.cur_p[0], a.cur_p[1]};
  for (int t = threadIdx.x; t < 2 * NQ; t += blockDim.x) (&dgs[0][0])[t] = t < np * NQ ? a.prev_dg[t] : 0.0;
  for (int t = threadIdx.x; t < kRWarps * 2 * ld1; t += blockDim.x) (&qs[0][0][0])[t] = 0.0;
  for (int t = threadIdx.x; t < kRWarps * KS * 32; t += blockDim.x) (&cs[0][0])[t] = 0.0;
  if (threadIdx.x < kRWarps) sqs[threadIdx.x] = 0.0;
  __syncthreads();
  const uint32_t stride = gridDim.x * kRWarps;
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
    if (c.base + kRRound < c.end) return Cur{c.ci, c.beg, c.end, c.base + kRRound, c.row};
    return first(c.ci + stride);
  };
  struct Co {
    uint32_t i[kRE];
  };
  auto coord = [&](const Cur& c) {
    Co o;
#pragma unroll
    for (int e = 0; e < kRE; ++e) {
      const uint32_t pos = c.base + 32 * e + lane;
      o.i[e] = (c.ci < a.csf.nchunks && pos < c.end) ? __ldg(a.csf.oc[1] + pos) : 0u;
    }
    return o;
  };
  auto issue = [&](const Cur& c, int b, const Co& co) {
    double* st = st0 + b * RS::size;
#pragma unroll
    for (int e = 0; e < kRE; ++e) {
      const uint32_t pos = c.base + 32 * e + lane;
      const int sl = 32 * e + lane;  // staged slot
      if (c.ci < a.csf.nchunks && pos < c.end) {
        const double* r1 = a.m.factor[1] + (size_t)co.i[e] * ld1;
#pragma unroll
        for (int t = 0; t < ld1 / 2; ++t) cp_async16_row(st + RS::U + sl * ld1 + 2 * t, r1 + 2 * t, a.hot & 2);
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (wrow[j] >= 0) cp_async8(st + RS::Wv + kRRound * j + sl, a.W + (uint64_t)wrow[j] * a.wstride + pos);
        cp_async8(st + RS::Rr + sl, a.r + pos);
      }
    }
    if (c.ci < a.csf.nchunks && c.base == c.beg && 2 * lane < ld2)
      cp_async16(st + RS::A2 + 2 * lane, a.m.factor[2] + (size_t)c.row * ld2 + 2 * lane);
  };

  Cur cur = first(blockIdx.x * kRWarps + warp);
  if (cur.ci < a.csf.nchunks) {
    issue(cur, 0, coord(cur));
    Cur nxt = next(cur);
    Co n1 = coord(nxt);
    double R0[F], R1[F];
#pragma unroll
    for (int f = 0; f < F; ++f) R0[f] = R1[f] = 0.0;
    double sq = 0.0;
    int buf = 0;
    while (true) {
      cp_async_wait_all();
      __syncwarp();
      const double* st = st0 + buf * RS::size;
      if (cur.base == cur.beg) {  // new chunk: keep its A_2 row; q_j = dg_j a
        if (lane < ld2) as[warp][lane] = st[RS::A2 + lane];
        if (np > 0 && lane < np * F) {
          const int j = lane / F, f = lane - j * F;
          double t = 0.0;
#pragma unroll
          for (int c = 0; c < Jm; ++c) t = fma(st[RS::A2 + c], dgs[j][f * Jm + c], t);
          qs[warp][j][f] = t;
        }
        __syncwarp();
      }
      const bool more = nxt.ci < a.csf.nchunks;
      if (more) issue(nxt, buf ^ 1, n1);
      const Cur nn = more ? next(nxt) : nxt;
      Co m1;
      if (more) m1 = coord(nn);
#pragma unroll
      for (int e = 0; e < kRE; ++e) {
      const uint32_t pos = cur.base + 32 * e + lane;
      const int sl = 32 * e + lane;
      if (pos < cur.end) {
        double u[ld1];
#pragma unroll
        for (int t = 0; t < ld1 / 2; ++t) {
          const double2 v = reinterpret_cast<const double2*>(st + RS::U + sl * ld1)[t];
          u[2 * t] = v.x;
          u[2 * t + 1] = v.y;
        }
        double r = st[RS::Rr + sl];
        if (np > 0) {
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            if (j < np) {
              const double2* q2 = reinterpret_cast<const double2*>(qs[warp][j]);
              double t = 0.0;
#pragma unroll
              for (int f2 = 0; f2 < ld1 / 2; ++f2) {
                const double2 q = q2[f2];
                t = fma(u[2 * f2], q.x, t);
                if (2 * f2 + 1 < F) t = fma(u[2 * f2 + 1], q.y, t);
              }
              r = fma(-st[RS::Wv + kRRound * j + sl], t, r);
            }
          }
          a.r[pos] = r;
        }
        if (fin || a.want_sq) sq = fma(r, r, sq);
        if (nc > 0) {
          const double w0 = st[RS::Wv + 2 * kRRound + sl] * r;
#pragma unroll
          for (int f = 0; f < F; ++f) R0[f] = fma(w0, u[f], R0[f]);
          if (nc > 1) {
            const double w1 = st[RS::Wv + 3 * kRRound + sl] * r;
#pragma unroll
            for (int f = 0; f < F; ++f) R1[f] = fma(w1, u[f], R1[f]);
          }
        }
      }
      }
      if (!more || nxt.ci != cur.ci) {  // chunk finished
        if (fin) {
          sq = warp_sum(sq);
          if (lane == 0) a.chunk_sq[cur.ci] = sq;
        } else {
          {
            // all 2F (+ sum r^2) chunk sums at once: butterfly reduce-scatter,
            // lane l ends with sum l (31 exchanges instead of 5 per value)
            double v[32];
#pragma unroll
            for (int f = 0; f < 32; ++f) v[f] = 0.0;
#pragma unroll
            for (int f = 0; f < F; ++f) {
              v[f] = R0[f];
              v[F + f] = R1[f];
            }
            v[2 * F] = sq;
            transpose_reduce(v, lane);
            if (lane < F) rs[warp][0][lane] = v[0];
            else if (lane < 2 * F) rs[warp][1][lane - F] = v[0];
            else if (lane == 2 * F && a.want_sq) sqs[warp] += v[0];
          }
          __syncwarp();
          // C_j[f][c] += R_j[f] a_c (lane-owned, in shared memory)
#pragma unroll
          for (int k = 0; k < KC; ++k) {
            const int q = lane + 32 * k;
            if (q < nc * NQ) {
              const int j = q / NQ, qq = q - j * NQ;
              cs[warp][q] = fma(rs[warp][j][qq / Jm], as[warp][qq % Jm], cs[warp][q]);
            }
          }
        }
#pragma unroll
        for (int f = 0; f < F; ++f) R0[f] = R1[f] = 0.0;
        sq = 0.0;
      }
      if (!more) break;
      __syncwarp();
      cur = nxt;
      nxt = nn;
      n1 = m1;
      buf ^= 1;
    }
  }
  if (fin) return;
  __syncthreads();
  for (int q = threadIdx.x; q < NP; q += blockDim.x) {
    double t = 0.0;
    if (q < NC) {
      for (int w = 0; w < kRWarps; ++w) t += cs[w][q];
    } else {
      for (int w = 0; w < kRWarps; ++w) t += sqs[w];
    }
    a.part[(size_t)blockIdx.x * NP + q] = t;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last_cta = atomicAdd(a.counter, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last_cta) return;
  __threadfence();
  // last CTA: warp w sums partial rows w, w + 8, ... (coalesced, many loads in
  // flight), then the warps' sums are added in warp order
  constexpr int KP = (NP + 31) / 32;
  double t[KP];
#pragma unroll
  for (int k = 0; k < KP; ++k) t[k] = 0.0;
  for (uint32_t b = warp; b < gridDim.x; b += kRWarps) {
    const double* prow = a.part + (size_t)b * NP;
#pragma unroll
    for (int k = 0; k < KP; ++k)
      if (lane + 32 * k < NP) t[k] += __ldcg(prow + lane + 32 * k);
  }
  __syncthreads();
  double* gs = &cs[0][0];  // reuse: [kRWarps][KP * 32]
#pragma unroll
  for (int k = 0; k < KP; ++k) gs[warp * KP * 32 + lane + 32 * k] = t[k];
  __syncthreads();
  for (int q = threadIdx.x; q < NP; q += blockDim.x) {
    double s2 = 0.0;
    for (int w = 0; w < kRWarps; ++w) s2 += gs[w * KP * 32 + q];
    a.cout[q] = s2;
  }
  if (threadIdx.x == 0) *a.counter = 0u;
}

// ----------------------------------------------------------------- solve --
// Sequential Gauss-Seidel over one block's cells (updates.hpp:171-188): one
// warp, the cells' state in registers (lane l holds cells l, l+32, ...);
// branch-free steps: every lane evaluates its slot-k cell, the owner's dg is
// broadcast, every lane folds -dg H[q][.] into its later cells (finished
// cells' right-hand sides are never read again).  H is dense in shared memory.
template <int REG>
__device__ __forceinline__ void gs_block(const double* H, int nq, int Jm, const uint32_t* fib, double* core,
                                         const uint8_t* core_mask, double lambda, double (&cc)[kSolveK],
                                         double (&dgl)[kSolveK], double* dg_out) {
  const int lane = threadIdx.x;
  double gv[kSolveK], hd[kSolveK], rd[kSolveK];
  bool upd[kSolveK];
  int lin[kSolveK];
#pragma unroll
  for (int k = 0; k < kSolveK; ++k) {
    const int q = lane + 32 * k;
    gv[k] = hd[k] = rd[k] = dgl[k] = 0.0;
    upd[k] = false;
    lin[k] = 0;
    if (q < nq) {
      lin[k] = (int)fib[q / Jm] * Jm + q % Jm;
      gv[k] = core[lin[k]];
      hd[k] = H[q * nq + q];
      const double den = REG == 0 ? hd[k] + lambda : 2.0 * hd[k];
      rd[k] = den != 0.0 ? 1.0 / den : 0.0;
      // a cell is updated unless masked or its denominator vanishes
      upd[k] = !core_mask[lin[k]] && den != 0.0;
    }
  }
  const double* hrow = H + lane;
  double hcur[kSolveK];
#pragma unroll
  for (int k2 = 0; k2 < kSolveK; ++k2) hcur[k2] = hrow[32 * k2];
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
      if (REG == 0) {
        g_new = num * rd[k];
      } else {
        const double gg = -2.0 * num;
        g_new = gg > lambda ? (lambda - gg) * rd[k] : (gg < -lambda ? -(lambda + gg) * rd[k] : 0.0);
      }
      if (!upd[k]) g_new = g_old;
      const double dg = __shfl_sync(0xffffffffu, g_new - g_old, lo);  // (x - x == +0: a no-op fold)
      if (lane == lo) {
        gv[k] = g_new;
        dgl[k] = dg;
        dg_out[q] = dg;
      }
#pragma unroll
      for (int k2 = k; k2 < kSolveK; ++k2) cc[k2] = fma(-dg, hcur[k2], cc[k2]);
      hrow += nq;
#pragma unroll
      for (int k2 = 0; k2 < kSolveK; ++k2) hcur[k2] = hrow[32 * k2];  // next row, off the chain
    }
  }
#pragma unroll
  for (int k = 0; k < kSolveK; ++k)
    if (lane + 32 * k < nq && upd[k]) core[lin[k]] = gv[k];
}

// x^T M y for lane-distributed x, y (slots) with M dense in shared memory
__device__ __forceinline__ double quad(const double* M, int nq, const double (&x)[kSolveK], const double* ys) {
  const int lane = threadIdx.x;
  double acc = 0.0;
#pragma unroll
  for (int k = 0; k < kSolveK; ++k) {
    const int q = lane + 32 * k;
    if (q < nq && x[k] != 0.0) {
      const double* mr = M + q * nq;
      double hv = 0.0;
      for (int q2 = 0; q2 < nq; ++q2) hv = fma(mr[q2], ys[q2], hv);
      acc = fma(x[k], hv, acc);
    }
  }
  return warp_sum(acc);
}

// One pair group (or a single block): block a; C_b -= H_ba dg_a; block b.
// H_aa / H_bb arrive by bulk copies at launch, H_ab replaces H_aa once block a
// is done.  With s_out: the sum of squared residuals after the group,
//   s - 2 (dg_a.C_a + dg_b.C_b) + dg_a^T H_aa dg_a + 2 dg_a^T H_ab dg_b + dg_b^T H_bb dg_b.
template <int REG>
__global__ void __launch_bounds__(32) k_core_solve_g(const double* Ha, const double* Hb, const double* Hx,
                                                     const double* C, int nf, int Jm, const uint32_t* fib_a,
                                                     const uint32_t* fib_b, double* core, const uint8_t* core_mask,
                                                     double lambda, double* dg_out, double* s_out) {
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) uint64_t bar[3];
  const int nq = nf * Jm, lane = threadIdx.x;
  const bool two = Hb != nullptr;
  const size_t hs = h_stride(nq) + kSolveSlack;
  double* bufA = sm;
  double* bufB = sm + hs;
  double* dga = sm + 2 * hs;  // nq
  double* dgb = dga + nq;     // nq
  const uint32_t bytes = ((uint32_t)(nq * nq) * 8u + 15u) & ~15u;
  if (lane == 0) {
    mbar_init(&bar[0]);
    mbar_init(&bar[1]);
    mbar_init(&bar[2]);
    bulk_copy(bufA, Ha, bytes, &bar[0]);
    if (two) bulk_copy(bufB, Hb, bytes, &bar[1]);
  }
  for (int t = (int)(bytes / 8) + lane; t < (int)hs; t += 32) {
    bufA[t] = 0.0;
    bufB[t] = 0.0;
  }
  double cca[kSolveK], ccb[kSolveK], c0a[kSolveK], c0b[kSolveK], dla[kSolveK], dlb[kSolveK];
#pragma unroll
  for (int k = 0; k < kSolveK; ++k) {
    const int q = lane + 32 * k;
    cca[k] = q < nq ? C[q] : 0.0;
    ccb[k] = (two && q < nq) ? C[nq + q] : 0.0;
    c0a[k] = cca[k];
    c0b[k] = ccb[k];
    dlb[k] = 0.0;
  }
  __syncwarp();
  mbar_wait(&bar[0], 0);
  gs_block<REG>(bufA, nq, Jm, fib_a, core, core_mask, lambda, cca, dla, dg_out);
#pragma unroll
  for (int k = 0; k < kSolveK; ++k)
    if (lane + 32 * k < nq) dga[lane + 32 * k] = dla[k];
  __syncwarp();
  double s = 0.0;
  if (s_out) {
    double d = 0.0;
#pragma unroll
    for (int k = 0; k < kSolveK; ++k) d = fma(dla[k], c0a[k], d);
    s = C[2 * nq] - 2.0 * warp_sum(d) + quad(bufA, nq, dla, dga);
  }
  if (two) {
    __syncwarp();
    if (lane == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic reads of bufA before the async write
      bulk_copy(bufA, Hx, bytes, &bar[2]);
    }
    mbar_wait(&bar[2], 0);
    // C_b -= H_ba dg_a (H_ab symmetric in q <-> q2)
#pragma unroll
    for (int k = 0; k < kSolveK; ++k) {
      const int q2 = lane + 32 * k;
      if (q2 < nq) {
        double t = 0.0;
        for (int q = 0; q < nq; ++q) t = fma(bufA[q * nq + q2], dga[q], t);
        ccb[k] -= t;
      }
    }
    mbar_wait(&bar[1], 0);
    gs_block<REG>(bufB, nq, Jm, fib_b, core, core_mask, lambda, ccb, dlb, dg_out + nq);
#pragma unroll
    for (int k = 0; k < kSolveK; ++k)
      if (lane + 32 * k < nq) dgb[lane + 32 * k] = dlb[k];
    __syncwarp();
    if (s_out) {
      double d = 0.0;
#pragma unroll
      for (int k = 0; k < kSolveK; ++k) d = fma(dlb[k], c0b[k], d);
      s += -2.0 * warp_sum(d) + 2.0 * quad(bufA, nq, dla, dgb) + quad(bufB, nq, dlb, dgb);
    }
  }
  if (s_out && lane == 0) {
    s_out[0] = s;
    s_out[1] = C[2 * nq];  // the sum before the group's update (cancellation check, sum_from_quadratic_form)
  }
}

// --------------------------------------------------------------- dispatch --
struct CoreAllOps {
  int J[3];
  cudaError_t (*sall)(const DevModel& m, const DevCSF& csf, double* stats, double* W, uint64_t wstride, int hot,
                      int grid, cudaStream_t s);
  cudaError_t (*rpass)(const RPassArgs& a, int grid, cudaStream_t s);
  cudaError_t (*sgemm)(const double* stats, int LW, const Chunk* chunks, uint32_t nchunks, const double* A,
                       double* partial, int ksplit, cudaStream_t s);
  int (*rpass_occupancy)();
};

template <class S>
cudaError_t run_core_sall(const DevModel& m, const DevCSF& csf, double* stats, double* W, uint64_t wstride,
                          int hot, int grid, cudaStream_t s) {
  if (csf.nchunks == 0) return cudaSuccess;
  const int smem = kAllWarps * 2 * 32 * sall_ldr(S::J(0), S::J(1)) * (int)sizeof(double);
  cudaFuncSetAttribute(k_core_sall<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k_core_sall<S><<<grid, kAllWarps * 32, smem, s>>>(m, csf, stats, W, wstride, hot);
  count_launch();
  return cudaGetLastError();
}

template <class S>
constexpr int rpass_smem() {
  return kRWarps * 2 * RStage<S::J(1), S::J(2)>::size * (int)sizeof(double);
}

template <class S>
cudaError_t run_core_rpass(const RPassArgs& a, int grid, cudaStream_t s) {
  cudaFuncSetAttribute(k_core_rpass<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, rpass_smem<S>());
  k_core_rpass<S><<<grid, kRWarps * 32, rpass_smem<S>(), s>>>(a);
  count_launch();
  return cudaGetLastError();
}

template <class S>
int rpass_occupancy() {
  int occ = 0;
  cudaFuncSetAttribute(k_core_rpass<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, rpass_smem<S>());
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_core_rpass<S>, kRWarps * 32, rpass_smem<S>());
  return occ;
}

template <class S>
cudaError_t run_sall_gemm(const double* stats, int LW, const Chunk* chunks, uint32_t nchunks, const double* A,
                          double* partial, int ksplit, cudaStream_t s) {
  const dim3 grid(ksplit, (LW + kSgRows - 1) / kSgRows);
  cudaFuncSetAttribute(k_sall_gemm<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, sgemm_smem<S>());
  k_sall_gemm<S><<<grid, 256, sgemm_smem<S>(), s>>>(stats, LW, chunks, nchunks, A, partial);
  count_launch();
  return cudaGetLastError();
}

template <int J0, int J1, int J2>
constexpr CoreAllOps make_all_ops() {
  using S = SShape<J0, J1, J2>;
  static_assert(J1 * J2 <= 128, "pair solve: F * J_2 <= 128");
  CoreAllOps o{};
  o.J[0] = J0;
  o.J[1] = J1;
  o.J[2] = J2;
  o.sall = &run_core_sall<S>;
  o.rpass = &run_core_rpass<S>;
  o.sgemm = &run_sall_gemm<S>;
  o.rpass_occupancy = &rpass_occupancy<S>;
  return o;
}

const CoreAllOps kAllOps[] = {
    make_all_ops<5, 5, 5>(),
    make_all_ops<10, 10, 10>(),
    make_all_ops<10, 10, 5>(),
};

int hot_modes(const Ctx& c) { return (c.skewed[0] ? 1 : 0) | (c.skewed[1] ? 2 : 0); }

int rpass_grid(Ctx& c, const CoreAllOps* ops) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c.device);
  return std::max(1, std::min(ops->rpass_occupancy(), 4)) * sms;  // one resident wave (the last CTA sums the partials)
}

RPassArgs rpass_args(Ctx& c, const int (&prev)[2], const int (&cur)[2], double* cout, int want_sq) {
  RPassArgs a{};
  a.m = c.model_view();
  a.csf = c.csf_view(c.N - 1);
  a.r = c.d_r;
  a.prev_p[0] = prev[0];
  a.prev_p[1] = prev[1];
  a.prev_dg = c.d_dg;
  a.cur_p[0] = cur[0];
  a.cur_p[1] = cur[1];
  a.chunk_sq = c.d_chunk_sum;
  a.part = c.d_gemm_part;
  a.cout = cout;
  a.counter = c.d_counter;
  a.W = c.d_pack_w - c.modes[c.N - 1].pos0;  // [P][local nnz], absolute positions
  a.wstride = c.local_nnz[c.N - 1];
  a.want_sq = want_sq;
  a.hot = hot_modes(c);
  return a;
}

}  // namespace

const void* find_core_all_ops(int N, const int* J) {
  if (N != 3) return nullptr;
  for (const auto& o : kAllOps)
    if (o.J[0] == J[0] && o.J[1] == J[1] && o.J[2] == J[2]) return &o;
  return nullptr;
}

// The sweep over the live blocks (prefixes, ascending), grouped in pairs
// (2x, 2x+1) where both are live.
void core_sweep_sall(Ctx& c, const void* ops_, int reg, double lambda, const std::vector<int>& prefixes,
                     const std::vector<int>& starts) {
  const CoreAllOps* ops = static_cast<const CoreAllOps*>(ops_);
  const int m = c.N - 1;
  const int P = c.ranks[0], F = c.ranks[1], Jm = c.ranks[2];
  const int X = P / 2, RW = P + X;
  const int NV = F * (F + 1) / 2, NAm = Jm * (Jm + 1) / 2, LW = RW * NV, nq = F * Jm;
  const DevCSF csf = c.csf_view(m);
  const DevModel mv = c.model_view();
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c.device);
  const size_t nT = (size_t)LW * NAm;
  // one wave: (K splits) x (row groups) == 2 CTAs per SM
  const int gy = (LW + kSgRows - 1) / kSgRows;
  const int ksplit = std::max(1, std::min<int>((2 * sms) / gy, (int)((csf.nchunks + 255) / 256)));
  const int rgrid = rpass_grid(c, ops);
  const size_t hs = h_stride(nq);
  const size_t nH = (size_t)RW * hs + 2;  // (+2: bulk copies round up to 16 bytes)
  ensure(c, &c.d_chunk_stats, &c.chunk_stats_cap, (size_t)csf.nchunks * LW + 1);
  ensure(c, &c.d_pack_w, &c.pack_w_cap, (size_t)c.local_nnz[m] * P + 1);
  ensure(c, &c.d_gemm_part, &c.gemm_part_cap, std::max((size_t)ksplit * nT, (size_t)rgrid * (2 * nq + 1)) + 1);
  ensure(c, &c.d_gemm_out, &c.gemm_out_cap, nT + 1 + nH + 2 * nq + 2);
  ensure(c, &c.d_dg, &c.dg_cap, (size_t)2 * nq + 1);
  ensure(c, &c.d_chunk_sum, &c.chunk_sum_cap, c.modes[m].nchunks + 1);
  if (!c.d_counter) {
    check(cudaMalloc(&c.d_counter, sizeof(unsigned)), "sweep counter");
    check(cudaMemsetAsync(c.d_counter, 0, sizeof(unsigned), c.stream), "sweep counter");
  }
  double* T = c.d_gemm_out;
  double* Hd = c.d_gemm_out + ((nT + 1) & ~(size_t)1);  // dense H of every A row (16-byte aligned)
  double* Cb = Hd + nH;                                  // [C_a | C_b | sum r^2]
  {
    ProfScope ps(c, kProfCorePass);
    check(ops->sall(mv, csf, c.d_chunk_stats, c.d_pack_w - c.modes[m].pos0, c.local_nnz[m], hot_modes(c), 3 * sms,
                    c.stream),
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
  comm_allreduce(c, T, (uint64_t)nT);  // block Grams over the shards
  {
    ProfScope ps(c, kProfCoreGemm);
    const size_t n = (size_t)RW * nq * nq;
    k_expand_h<<<(unsigned)std::min<size_t>(4096, (n + 255) / 256), 256, 0, c.stream>>>(T, RW, F, Jm, Hd);
    count_launch();
    check(cudaGetLastError(), "core expand H");
  }
  const size_t smem = (2 * (hs + kSolveSlack) + 2 * (size_t)nq) * sizeof(double);
  auto solve = reg == 0 ? k_core_solve_g<0> : k_core_solve_g<1>;
  check(cudaFuncSetAttribute(solve, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "solve smem");
  // pair groups over the live blocks
  struct Group {
    int p[2], start[2];
  };
  std::vector<Group> groups;
  for (size_t i = 0; i < prefixes.size(); ++i) {
    Group gr{{prefixes[i], -1}, {starts[i], 0}};
    if (prefixes[i] % 2 == 0 && prefixes[i] / 2 < X && i + 1 < prefixes.size() && prefixes[i + 1] == prefixes[i] + 1) {
      gr.p[1] = prefixes[i + 1];
      gr.start[1] = starts[i + 1];
      ++i;
    }
    groups.push_back(gr);
  }
  const int ng = (int)groups.size();
  int prev[2] = {-1, -1};
  for (int gi = 0; gi < ng; ++gi) {
    const Group& gr = groups[gi];
    const bool last = gi == ng - 1;
    {
      ProfScope ps(c, kProfCorePass);
      if (csf.nchunks > 0) {
        const RPassArgs a = rpass_args(c, prev, gr.p, Cb, last);
        check(ops->rpass(a, rgrid, c.stream), "core group pass");
      } else {
        check(cudaMemsetAsync(Cb, 0, (2 * nq + 1) * sizeof(double), c.stream), "core group pass (empty)");
      }
    }
    comm_allreduce(c, Cb, (uint64_t)2 * nq + 1);  // C and (last group) sum r^2 over the shards
    ProfScope ps(c, kProfCoreSolve);
    const bool two = gr.p[1] >= 0;
    solve<<<1, 32, smem, c.stream>>>(Hd + (size_t)gr.p[0] * hs, two ? Hd + (size_t)gr.p[1] * hs : nullptr,
                                     two ? Hd + (size_t)(P + gr.p[0] / 2) * hs : nullptr, Cb, F, Jm,
                                     c.d_fibers + gr.start[0], c.d_fibers + (two ? gr.start[1] : gr.start[0]),
                                     c.d_core, c.d_core_mask, lambda, c.d_dg, last ? c.d_small : nullptr);
    count_launch();
    check(cudaGetLastError(), "core solve");
    prev[0] = gr.p[0];
    prev[1] = gr.p[1];
  }
  // r lacks the last group's update until someone reads it (core_apply_pending)
  check(cudaMemcpyAsync(c.h_small, c.d_small, 2 * sizeof(double), cudaMemcpyDeviceToHost, c.stream), "sum readback");
  c.r_valid = false;
  c.r_fresh = false;
  c.r_pending[0] = prev[0];
  c.r_pending[1] = prev[1];
  c.r_pending_ops = ops_;
  c.r_pending_general = false;
  if (!c.capturing) {  // a captured iteration reads the sum after the graph launch
    check(cudaStreamSynchronize(c.stream), "sum sync");
    sum_from_quadratic_form(c);
  }
}

// The sum of squared residuals after the sweep from the last group's
// statistics, s' = s - 2 dg.C + dg^T H dg (h_small[0]; h_small[1] = s).  When
// s' cancels to a small fraction of s (a near-exact fit) its relative error
// grows like s / s', so the pending update is applied and the sum recomputed
// exactly from the residuals, as the reference's compute_residuals
// (tucker_model.hpp:168-183) would give: the RE drives StopController
// (pruning.hpp:45-81) and the convergence test (trainer.hpp:152).
void sum_from_quadratic_form(Ctx& c) {
  const double s1 = c.h_small[0], s0 = c.h_small[1];
  if (!(s1 >= kQuadCancel * s0) || s0 <= 0.0) {
    core_apply_pending(c);
    return;
  }
  c.sum_sq = s1;
  c.re = std::sqrt(c.sum_sq) / c.x_norm;
}

// Apply the deferred last-group update to r (and recompute sum r^2 exactly).
bool core_apply_pending(Ctx& c) {
  if (c.r_pending[0] < 0) return false;
  if (c.r_pending_general) {
    core_apply_pending_general(c);
    return true;
  }
  const CoreAllOps* ops = static_cast<const CoreAllOps*>(c.r_pending_ops);
  const DevCSF csf = c.csf_view(c.N - 1);
  if (csf.nchunks > 0) {
    ProfScope ps(c, kProfResid);
    const int none[2] = {-1, -1};
    const RPassArgs a = rpass_args(c, c.r_pending, none, nullptr, 0);
    check(ops->rpass(a, rpass_grid(c, ops), c.stream), "core pending update");
  }
  c.sum_sq = reduce_chunk_sums(c, c.d_chunk_sum, c.modes[c.N - 1].nchunks);
  c.re = std::sqrt(c.sum_sq) / c.x_norm;
  c.r_valid = true;
  c.r_fresh = true;
  c.r_pending[0] = c.r_pending[1] = -1;
  return true;
}

}  // namespace vest
