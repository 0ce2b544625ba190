// SPDX-License-Identifier: Apache-2.0
// vest_rowpass.cu -- the per-row passes over one mode's CSF:
//   kStats : factor-row update (updates.hpp:64-151, update_all_factors :157-175)
//            statistics gram = sum delta delta^T, xdelta = sum x delta over the
//            row's entries, then the row's Gauss-Seidel solve in-kernel;
//   kResp  : factor responsibilities (pruning.hpp:141-179);
//   kResid : residual r = x - B(alpha) and sum r^2 (tucker_model.hpp:168-183),
//            run on the last mode's CSF so r lands in the core sweep's order.
// One warp per work item (a chunk of <= kChunk entries of one row); one lane
// per observed entry; the per-entry delta is the factorised contraction of
// vest_common.cuh with the core in the constant bank (compile-time ranks) or
// the reference's cell loop (generic ranks).
#include <mutex>
#include <type_traits>

#include "vest_common.cuh"

namespace vest {

// The core as double2 (pairs of adjacent cells): one LDCU.128 feeds two DFMA.
__constant__ double2 c_core_pairs[VEST_CONST_CORE_MAX / 2];

struct ConstCore {
  __device__ __forceinline__ double operator()(int lin) const {
    const double2 p = c_core_pairs[lin >> 1];
    return (lin & 1) ? p.y : p.x;
  }
  __device__ __forceinline__ double2 pair(int lin) const { return c_core_pairs[lin >> 1]; }  // lin even
};

// A core held in shared memory (broadcast LDS reads): the fused residual's
// v = G x_m a, and the VEST_CORE_SMEM experiment.
struct SmemCore {
  const double* p;
  __device__ __forceinline__ double operator()(int lin) const { return p[lin]; }
  __device__ __forceinline__ double2 pair(int lin) const { return reinterpret_cast<const double2*>(p)[lin >> 1]; }
};

template <int B, int E, class F>
__device__ __forceinline__ void static_for(F&& f) {
  if constexpr (B < E) {
    f(std::integral_constant<int, B>{});
    static_for<B + 1, E>(f);
  }
}

template <int J, int MAXJ>
__device__ __forceinline__ void load_row(const double* __restrict__ row, double (&dst)[MAXJ]) {
#pragma unroll
  for (int b = 0; b + 1 < J; b += 2) {
    const double2 v = __ldg(reinterpret_cast<const double2*>(row + b));
    dst[b] = v.x;
    dst[b + 1] = v.y;
  }
  if constexpr (J & 1) dst[J - 1] = __ldg(row + J - 1);
}

// ------------------------------------------------------------------ policies --
// A policy computes delta for NE entries per lane: the CSF positions pos[e]
// (clamped into the chunk by the caller), rows of the other modes gathered.
#ifndef VEST_ROW_NE
#define VEST_ROW_NE 2
#endif
#ifndef VEST_ROW_MINB
#define VEST_ROW_MINB 2
#endif
// Shapes with N >= 4 (configs 4-5): NE = 2 entries per lane spills 100-500 B
// per thread at the 128-register budget of 2 CTAs/SM, but measured 2-3x faster
// than NE = 1 (one uniform constant load per DFMA is issue-bound) and than
// NE = 2 at 1 CTA/SM (configs 4/5: 1.17/0.59 s vs 2.34/1.23 s and 1.20/0.66 s
// per iteration).
#ifndef VEST_ROW_NE_HI
#define VEST_ROW_NE_HI 2
#endif
#ifndef VEST_ROW_MINB_HI
#define VEST_ROW_MINB_HI 2
#endif
// ... and unroll the rolled outer-mode loop once (K0U = 1): the 2-way unroll
// of the 3-mode shapes spills at N >= 4.
#ifndef VEST_K0_UNROLL_HI
#define VEST_K0_UNROLL_HI 2
#endif
template <class S>
struct RowTune {
  static constexpr int NE = S::N <= 3 ? VEST_ROW_NE : VEST_ROW_NE_HI;
  static constexpr int MINB = S::N <= 3 ? VEST_ROW_MINB : VEST_ROW_MINB_HI;
  static constexpr int K0U = S::N <= 3 ? kK0Unroll : VEST_K0_UNROLL_HI;
};

template <class S, int MODE>
#ifndef VEST_ROW_TAIL1
#define VEST_ROW_TAIL1 0  // measured slower (larger kernel body): 1.36 vs 1.27 ms per mode
#endif
struct StaticPolicy {
#ifndef VEST_CORE_SMEM
#define VEST_CORE_SMEM 0
#endif
  static constexpr bool kSmemCore = VEST_CORE_SMEM && S::G() <= 1024;
  using Shape = S;
  static constexpr int N = S::N;
  static constexpr int MAXJ = S::MAXJ;
  static constexpr int JN = S::J(MODE);
  static constexpr bool kStatic = true;
  static constexpr int NE = RowTune<S>::NE;  // entries per lane per round
  static constexpr int kMinB = RowTune<S>::MINB;
  static constexpr int K0 = (MODE == 0) ? 1 : 0;
  int jn;  // unused, keeps the interface uniform
  __device__ __forceinline__ int J() const { return JN; }
  __device__ __forceinline__ int mode() const { return MODE; }
  __device__ __forceinline__ void entries(const DevModel& m, const DevCSF& csf, const uint32_t (&pos)[NE],
                                          double (&d)[NE][MAXJ]) const {
    double u[NE][N][MAXJ];
    const double* rows0[NE];
#pragma unroll
    for (int e = 0; e < NE; ++e) {
      static_for<0, N>([&](auto kc) {
        constexpr int k = decltype(kc)::value;
        if constexpr (k != MODE) {
          const uint32_t i = __ldg(csf.oc[k] + pos[e]);
          constexpr int ld = (S::J(k) + 1) & ~1;
          if constexpr (k == K0 && S::G() > kFullUnrollN)
            rows0[e] = m.factor[k] + (size_t)i * ld;  // read element-wise by the rolled loop
          else
            load_row<S::J(k)>(m.factor[k] + (size_t)i * ld, u[e][k]);
        }
      });
    }
#if VEST_CORE_SMEM
    delta_staticN<S, MODE, NE>(SmemCore{score}, u, rows0, d);
#else
    delta_staticN<S, MODE, NE, ConstCore, RowTune<S>::K0U>(ConstCore{}, u, rows0, d);
#endif
  }
  const double* score = nullptr;
  // single entry (NE == 1): the v1 structure, called only for valid lanes
  __device__ __forceinline__ void entry1(const DevModel& m, const DevCSF& csf, uint32_t pos,
                                         double (&d)[MAXJ]) const {
    double u[N][MAXJ];
    const double* row0 = nullptr;
    static_for<0, N>([&](auto kc) {
      constexpr int k = decltype(kc)::value;
      if constexpr (k != MODE) {
        const uint32_t i = __ldg(csf.oc[k] + pos);
        constexpr int ld = (S::J(k) + 1) & ~1;
        if constexpr (k == K0)
          row0 = m.factor[k] + (size_t)i * ld;
        else
          load_row<S::J(k)>(m.factor[k] + (size_t)i * ld, u[k]);
      }
    });
    delta_static<S, MODE, ConstCore, (bool)VEST_ROW_TAIL1>(ConstCore{}, u, row0, d);
  }
};

// Generic ranks: the reference's own cell loop (updates.hpp:42-51), skipping
// zero cells and multiplying factors in ascending mode order.
struct DynPolicy {
  static constexpr bool kSmemCore = false;
  static constexpr int N = VEST_MAXN;
  static constexpr int MAXJ = VEST_MAXJ;
  static constexpr bool kStatic = false;
  static constexpr int NE = 1;
  static constexpr int kMinB = VEST_ROW_MINB;
  static constexpr int JN = VEST_MAXJ;
  int md;
  int jn;
  __device__ __forceinline__ int J() const { return jn; }
  __device__ __forceinline__ int mode() const { return md; }
  __device__ __forceinline__ void entries(const DevModel& m, const DevCSF& csf, const uint32_t (&pos)[NE],
                                          double (&dd)[NE][MAXJ]) const {
    entry1(m, csf, pos[0], dd[0]);
  }
  __device__ __forceinline__ void entry1(const DevModel& m, const DevCSF& csf, uint32_t pos0,
                                         double (&d)[MAXJ]) const {
    double u[N][MAXJ];
    const uint32_t pos[1] = {pos0};
    for (int k = 0; k < m.N; ++k) {
      if (k == md) continue;
      const uint32_t i = __ldg(csf.oc[k] + pos[0]);
      const double* row = m.factor[k] + (size_t)i * m.ld[k];
      for (int b = 0; b < m.J[k]; ++b) u[k][b] = __ldg(row + b);
    }
    for (int j = 0; j < jn; ++j) d[j] = 0.0;
    for (int lin = 0; lin < m.G; ++lin) {
      const double g = __ldg(m.core + lin);
      if (g == 0.0) continue;
      const uint32_t beta = __ldg(m.cellbeta + lin);
      double p = g;
      for (int k = 0; k < m.N; ++k)
        if (k != md) p *= u[k][(beta >> (4 * k)) & 15u];
      d[(beta >> (4 * md)) & 15u] += p;
    }
  }
};

// ----------------------------------------------------------------- row solve --
// update_factor_row_lf (updates.hpp:96-105) / _l1 (:120-138) given the row's
// gram (J x J, smem) and xdelta (smem): columns in ascending order, each one
// seeing the fresh values of the columns before it.  Lane t holds element t.
__device__ __forceinline__ void solve_row(int J, int reg, double lambda, const double* G,
                                          const double* xd, double* row, const uint8_t* mask,
                                          int lane) {
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

// pair index -> (t, j) over the upper triangle of a J x J matrix, row-major,
// followed by J (t, J) "x column" pairs.
__device__ __forceinline__ void pair_of(int a, int J, int& t, int& j) {
  const int ng = J * (J + 1) / 2;
  if (a >= ng) {
    t = a - ng;
    j = J;
    return;
  }
  int row = 0, rem = a;
  while (rem >= J - row) {
    rem -= J - row;
    ++row;
  }
  t = row;
  j = row + rem;
}

// ------------------------------------------------------------------- kernel --
constexpr int kRowWarps = 8;
constexpr int kMaxSlots = 5;  // ceil((16*17/2 + 16) / 32)

// Gram of (delta, x) on the FP64 tensor cores (DMMA) when the row rank is a
// compile-time constant <= 15; generic ranks use shared-memory slots.
#ifndef VEST_TC_GRAM
#define VEST_TC_GRAM 1
#endif
template <class P>
struct TensorGram {
  static constexpr bool value = VEST_TC_GRAM && P::kStatic && P::MAXJ <= 15;
};

template <class P>
constexpr int fused_resid_words() {
  if constexpr (P::kStatic) {
    using S = typename P::Shape;
    return S::N >= 3 ? 128 + S::G() / S::J(S::N - 1) : 0;
  } else {
    return 0;
  }
}

template <class P>
constexpr int stage_words() {
  // per-warp shared memory: the transposed DMMA stage (16 x kXldN(NE)), or
  // 32 staged rows of (J + 1) doubles (odd stride), or the row solve area
  // (J*J + J), whichever is largest
  constexpr int J = P::MAXJ;
  constexpr int st = 32 * (J + 2);
  constexpr int sv = J * J + J;
  constexpr int tcw = 16 * kXldN(P::NE);
  constexpr int m1 = st > sv ? st : sv;
  constexpr int m2 = m1 > tcw ? m1 : tcw;
  // the fused residual's v = G x_m a_row lives at offset 128 (after the solve area)
  constexpr int fr = fused_resid_words<P>();
  return m2 > fr ? m2 : fr;
}

// Statistics of the row's entries: on the tensor pipe for static ranks (the
// (delta, x) vectors of the round's 32*NE entries are staged transposed and
// X^T X accumulated with DMMA, so the DFMA pipe only runs the contraction);
// generic ranks accumulate "slots" (pair (t, j) owned by lane s % 32) over
// shared-memory staged rows.
// Residual of a freshly solved row of the last mode m (fuse_resid): with the
// new row a = A_m[s, :], B(alpha_e) = sum_{beta<m} v[beta] prod_{k<m} u_k[beta_k]
// where v = G x_m a (|G| / J_m values, computed once per row into shared
// memory), so each entry costs the (N-1)-mode contraction instead of a full
// reconstruction.  Writes r (CSF order of mode m) for the chunk's entries.
// Returns the lane's partial sum of r^2.  Also the residual pass (kResid) of
// rank-specialised shapes: |G| / J_m + ... FMA per entry instead of the full
// delta contraction.
template <class P>
__device__ __forceinline__ double fused_residual(const RowPassArgs& a, const Chunk& ch, double* v, int lane) {
  double sq = 0.0;
  if constexpr (P::kStatic) {
    using S = typename P::Shape;
    if constexpr (S::N >= 3) {
      using Q = PrefixShape<S>;
      constexpr int m = S::N - 1;
      constexpr int Jm = S::J(m);
      constexpr int NV = S::G() / Jm;
      const double* arow = a.m.factor[m] + (size_t)ch.row * a.m.ld[m];
      double an[Jm];
#pragma unroll
      for (int c = 0; c < Jm; ++c) an[c] = arow[c];
      // per-lane cells: read the core through L1 (a per-lane constant-bank
      // index would serialise 32-way)
      for (int p = lane; p < NV; p += 32) {
        double t = 0.0;
#pragma unroll
        for (int c = 0; c < Jm; ++c) t = fma(__ldg(a.m.core + p * Jm + c), an[c], t);
        v[p] = t;
      }
      __syncwarp();
      const SmemCore gv{v};
      for (uint32_t pos = ch.beg + lane; pos < ch.end; pos += 32) {
        double u[1][Q::N][Q::MAXJ];
        static_for<0, Q::N>([&](auto kc) {
          constexpr int k = decltype(kc)::value;
          constexpr int ld = (S::J(k) + 1) & ~1;
          load_row<S::J(k)>(a.m.factor[k] + (size_t)__ldg(a.csf.oc[k] + pos) * ld, u[0][k]);
        });
        double rec[1];
        trailingN<Q, 0, 1>(gv, u, 0, rec);
        const double r = __ldg(a.csf.val + pos) - rec[0];
        a.r_out[pos] = r;
        sq = fma(r, r, sq);
      }
    }
  }
  return sq;
}

template <class P, int KIND>
__global__ void __launch_bounds__(kRowWarps * 32, P::kMinB) k_rowpass(RowPassArgs a, P pol) {
  extern __shared__ double smem[];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if constexpr (P::kSmemCore) {
    double* sc = smem + kRowWarps * stage_words<P>();
    for (int t = threadIdx.x; t < a.m.G; t += blockDim.x) sc[t] = __ldg(a.m.core + t);
    __syncthreads();
    pol.score = sc;
  }
  const uint32_t ci = blockIdx.x * kRowWarps + warp;
  if (ci >= a.csf.nchunks) return;
  const Chunk ch = a.csf.chunks[ci];
  if constexpr (KIND == kResid && P::kStatic) {
    if constexpr (P::Shape::N >= 3) {  // kResid runs on the last mode: v = G x_m a_row
      const double sq = warp_sum(fused_residual<P>(a, ch, smem + warp * stage_words<P>() + 128, lane));
      if (lane == 0) a.chunk_out[ci] = sq;
      return;
    }
  }
  constexpr int NE = P::NE;
  const int J = pol.J();
  const int mode = pol.mode();
  constexpr int MAXJ = P::MAXJ;
  const int NG = J * (J + 1) / 2;
  const int NA = NG + J;
  const int ldst = (J & 1) ? J + 2 : J + 1;  // odd stride: conflict-free staging
  double* wsm = smem + warp * stage_words<P>();
  constexpr bool kTC = TensorGram<P>::value;
  constexpr int ldx = kXldN(NE);

  double arow[MAXJ];
  if constexpr (KIND != kStats) {
    const double* r = a.m.factor[mode] + (size_t)ch.row * a.m.ld[mode];
#pragma unroll
    for (int j = 0; j < MAXJ; ++j)
      if (j < J) arow[j] = __ldg(r + j);
  }

  int st_t[kMaxSlots], st_j[kMaxSlots];
  double sacc[kMaxSlots];
  if constexpr (!kTC) {
#pragma unroll
    for (int q = 0; q < kMaxSlots; ++q) {
      sacc[q] = 0.0;
      st_t[q] = 0;
      st_j[q] = 0;
      if (lane + 32 * q < NA) pair_of(lane + 32 * q, J, st_t[q], st_j[q]);
    }
  }
  double racc[MAXJ];
#pragma unroll
  for (int j = 0; j < MAXJ; ++j) racc[j] = 0.0;
  double sq = 0.0;
  double tc[3][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
  if constexpr (KIND == kStats && kTC) {
    // zero the padding columns once; columns <= J are rewritten every round
    for (int t = lane; t < 16 * ldx; t += 32) wsm[t] = 0.0;
    __syncwarp();
  }

  for (uint32_t base = ch.beg; base < ch.end; base += 32 * NE) {
    uint32_t pos[NE];
    bool valid[NE];
#pragma unroll
    for (int e = 0; e < NE; ++e) {
      pos[e] = base + 32 * e + lane;
      valid[e] = pos[e] < ch.end;
      if (!valid[e]) pos[e] = ch.beg;  // safe gather address; result discarded
    }
    double d[NE][MAXJ];
    double x[NE];
    if constexpr (NE == 1) {
      if (valid[0]) {
        pol.entry1(a.m, a.csf, pos[0], d[0]);
        x[0] = __ldg(a.csf.val + pos[0]);
      } else {
        x[0] = 0.0;
#pragma unroll
        for (int j = 0; j < MAXJ; ++j) d[0][j] = 0.0;
      }
    } else {
      // lane-uniform validity of the first entry guards the contraction (keeps
      // the core offsets in uniform registers); later entries are clamped.
      // A chunk's tail of <= 32 entries runs one entry per lane (the empty
      // second slots would cost the full contraction).
      const bool tail = VEST_ROW_TAIL1 && P::kStatic && ch.end - base <= 32;
      if (valid[0]) {
        if (tail) {
          pol.entry1(a.m, a.csf, pos[0], d[0]);
#pragma unroll
          for (int e = 1; e < NE; ++e)
#pragma unroll
            for (int j = 0; j < MAXJ; ++j) d[e][j] = 0.0;
        } else {
          pol.entries(a.m, a.csf, pos, d);
        }
      } else {
#pragma unroll
        for (int e = 0; e < NE; ++e)
#pragma unroll
          for (int j = 0; j < MAXJ; ++j) d[e][j] = 0.0;
      }
#pragma unroll
      for (int e = 0; e < NE; ++e) {
        x[e] = valid[e] ? __ldg(a.csf.val + pos[e]) : 0.0;
        if (!valid[e]) {
#pragma unroll
          for (int j = 0; j < MAXJ; ++j) d[e][j] = 0.0;
        }
      }
    }
    if constexpr (KIND == kStats && kTC) {
      // stage (delta, x) transposed and accumulate X^T X on the tensor pipe
#pragma unroll
      for (int e = 0; e < NE; ++e) {
#pragma unroll
        for (int j = 0; j < P::JN; ++j) wsm[j * ldx + 32 * e + lane] = d[e][j];
        wsm[P::JN * ldx + 32 * e + lane] = x[e];
      }
      __syncwarp();
      gram_dmma<P::JN + 1, NE>(wsm, tc, lane);
      __syncwarp();
    } else if constexpr (KIND == kStats) {
#pragma unroll
      for (int j = 0; j < MAXJ; ++j)
        if (j < J) wsm[lane * ldst + j] = d[0][j];
      wsm[lane * ldst + J] = x[0];
      __syncwarp();
#pragma unroll
      for (int q = 0; q < kMaxSlots; ++q) {
        if (lane + 32 * q < NA) {
          const double* pt = wsm + st_t[q];
          const double* pj = wsm + st_j[q];
          double acc_s = sacc[q];
#pragma unroll 8
          for (int l = 0; l < 32; ++l) acc_s = fma(pt[l * ldst], pj[l * ldst], acc_s);
          sacc[q] = acc_s;
        }
      }
      __syncwarp();
    } else {
#pragma unroll
      for (int e = 0; e < NE; ++e) {
        if (!valid[e]) continue;
        double rec = 0.0;
#pragma unroll
        for (int j = 0; j < MAXJ; ++j)
          if (j < J) rec = fma(d[e][j], arow[j], rec);
        const double r = x[e] - rec;
        if constexpr (KIND == kResp) {
#pragma unroll
          for (int j = 0; j < MAXJ; ++j) {
            if (j < J) {
              const double p = d[e][j] * arow[j];
              racc[j] = fma(2.0 * r + p, p, racc[j]);
            }
          }
        } else {
          a.r_out[pos[e]] = r;
          sq = fma(r, r, sq);
        }
      }
    }
  }

  // ---------------------------------------------------------------- epilogue
  if constexpr (KIND == kStats) {
    double* Gs = wsm;          // J x J
    double* xd = wsm + J * J;  // J
    if constexpr (kTC) {
      __syncwarp();
#pragma unroll
      for (int t = 0; t < (P::JN + 1 > 8 ? 3 : 1); ++t) {
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          int row, col;
          gram_coord(t, i, lane, row, col);
          const double v = tc[t][i];
          int slot = -1;
          if (row <= col && col < J) slot = row * J - row * (row - 1) / 2 + (col - row);
          else if (col == J && row < J) slot = NG + row;
          if (slot < 0) continue;
          if (ch.slot != kLight) {
            a.heavy_out[(size_t)ch.slot * a.stride_na + slot] = v;
          } else if (col == J) {
            xd[row] = v;
          } else {
            Gs[row * J + col] = v;
            Gs[col * J + row] = v;
          }
        }
      }
    } else {
#pragma unroll
      for (int q = 0; q < kMaxSlots; ++q) {
        const int s = lane + 32 * q;
        if (s < NA) {
          if (ch.slot != kLight) {
            a.heavy_out[(size_t)ch.slot * a.stride_na + s] = sacc[q];
          } else if (st_j[q] == J) {
            xd[st_t[q]] = sacc[q];
          } else {
            Gs[st_t[q] * J + st_j[q]] = sacc[q];
            Gs[st_j[q] * J + st_t[q]] = sacc[q];
          }
        }
      }
    }
    if (ch.slot == kLight) {
      __syncwarp();
      solve_row(J, a.reg, a.lambda, Gs, xd, a.m.factor[mode] + (size_t)ch.row * a.m.ld[mode],
                a.m.fmask[mode] + (size_t)ch.row * J, lane);
      if constexpr (P::kStatic) {
        if (a.fuse_resid) {
          __syncwarp();
          fused_residual<P>(a, ch, wsm + 128, lane);
        }
      }
    }
  } else if constexpr (KIND == kResp) {
#pragma unroll
    for (int j = 0; j < MAXJ; ++j)
      if (j < J) racc[j] = warp_sum(racc[j]);
#pragma unroll
    for (int j = 0; j < MAXJ; ++j) {
      if (j >= J || lane != j) continue;
      if (ch.slot != kLight) {
        a.heavy_out[(size_t)ch.slot * a.stride_na + j] = racc[j];
      } else {
        const size_t o = (size_t)ch.row * J + j;
        if (a.m.fmask[mode][o]) continue;  // stays +inf
        double err2 = a.re2 + racc[j] / a.x2;
        if (err2 < 0.0) err2 = 0.0;
        a.resp_out[o] = (sqrt(err2) - a.re) / a.re;
      }
    }
  } else {
    sq = warp_sum(sq);
    if (lane == 0) a.chunk_out[ci] = sq;
  }
}

// Heavy rows (several chunks): reduce the chunks' partial statistics in chunk
// order, then solve (kStats) or finalise responsibilities (kResp).
__global__ void __launch_bounds__(256) k_heavy(RowPassArgs a, int kind) {
  __shared__ double sm[8][VEST_MAXJ * VEST_MAXJ + VEST_MAXJ];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t hi = blockIdx.x * 8 + warp;
  if (hi >= a.csf.nheavy) return;
  const Heavy h = a.csf.heavy[hi];
  const int mode = a.mode;
  const int J = a.m.J[mode];
  const int NA = kind == kStats ? J * (J + 1) / 2 + J : J;
  double* Gs = sm[warp];
  double* xd = Gs + J * J;
  for (int s = lane; s < NA; s += 32) {
    double v = 0.0;
    for (uint32_t c = 0; c < h.nslots; ++c) v += a.heavy_out[(size_t)(h.first_slot + c) * a.stride_na + s];
    if (kind == kStats) {
      int t, j;
      pair_of(s, J, t, j);
      if (j == J) {
        xd[t] = v;
      } else {
        Gs[t * J + j] = v;
        Gs[j * J + t] = v;
      }
    } else {
      const size_t o = (size_t)h.row * J + s;
      if (!a.m.fmask[mode][o]) {
        double err2 = a.re2 + v / a.x2;
        if (err2 < 0.0) err2 = 0.0;
        a.resp_out[o] = (sqrt(err2) - a.re) / a.re;
      }
    }
  }
  if (kind != kStats) return;
  __syncwarp();
  solve_row(J, a.reg, a.lambda, Gs, xd, a.m.factor[mode] + (size_t)h.row * a.m.ld[mode],
            a.m.fmask[mode] + (size_t)h.row * J, lane);
}

// -------------------------------------------------------------- short rows --
// Rows with <= kTinyRow entries (the long tails of Zipf-distributed modes:
// config 3's mode 0 has ~940k such rows holding 10 % of the entries) waste most
// of a warp-per-chunk round.  Here one LANE owns one row: it contracts its
// entries one after another (the single-entry static form; lanes of a warp
// run different rows in lockstep, rows sorted by length so a warp's lanes
// have (nearly) equal trip counts), accumulates the row statistics in its own
// shared-memory slot and solves the row itself -- updates.hpp:61-151 for one
// row per thread.
#ifndef VEST_TINY_REG
#define VEST_TINY_REG 1  // statistics in registers (J(J+1)/2 + J doubles) instead of a shared-memory slot
#endif
template <class P>
__global__ void __launch_bounds__(128) k_rowpass_tiny(RowPassArgs a, P pol, const uint32_t* __restrict__ rows,
                                                      uint32_t nrows) {
  constexpr int J = P::JN;
  constexpr int NG = J * (J + 1) / 2, NA = NG + J;
  constexpr int NAs = NA | 1;  // odd stride: conflict-free per-lane slots
#if VEST_TINY_REG
  double g[NA];
#else
  extern __shared__ double tsm[];
  double* g = tsm + threadIdx.x * NAs;
#endif
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nrows) return;
#pragma unroll
  for (int q = 0; q < NA; ++q) g[q] = 0.0;
  const int mode = pol.mode();
  const uint32_t row = __ldg(rows + t);
  const uint32_t b = (uint32_t)__ldg(a.csf.offsets + row), e = (uint32_t)__ldg(a.csf.offsets + row + 1);
  for (uint32_t pos = b; pos < e; ++pos) {
    double d[P::MAXJ];
    pol.entry1(a.m, a.csf, pos, d);
    const double x = __ldg(a.csf.val + pos);
    int q = 0;
#pragma unroll
    for (int i = 0; i < J; ++i)
#pragma unroll
      for (int j = i; j < J; ++j) g[q++] += d[i] * d[j];
#pragma unroll
    for (int i = 0; i < J; ++i) g[NG + i] += x * d[i];
  }
  // the row's Gauss-Seidel solve (update_factor_row_lf / _l1), this lane alone
  double* arow = a.m.factor[mode] + (size_t)row * a.m.ld[mode];
  const uint8_t* mask = a.m.fmask[mode] + (size_t)row * J;
  double v[J];
#pragma unroll
  for (int j = 0; j < J; ++j) v[j] = arow[j];
  auto gram = [&](int i, int j) -> double {  // packed upper triangle (compile-time indices when unrolled)
    const int lo = i < j ? i : j, hi = i < j ? j : i;
    return g[lo * J - lo * (lo - 1) / 2 + (hi - lo)];
  };
#pragma unroll
  for (int j = 0; j < J; ++j) {
    if (mask[j]) continue;
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < J; ++i)
      if (i != j) s = fma(gram(j, i), v[i], s);
    const double lin = g[NG + j] - s;
    const double gjj = gram(j, j);
    if (a.reg == 0) {
      const double den = gjj + a.lambda;
      if (den != 0.0) v[j] = lin / den;
    } else {
      const double gg = -2.0 * lin, dd = 2.0 * gjj;
      if (dd == 0.0) {
        if (fabs(gg) <= a.lambda) v[j] = 0.0;
      } else {
        v[j] = gg > a.lambda ? (a.lambda - gg) / dd : (gg < -a.lambda ? -(a.lambda + gg) / dd : 0.0);
      }
    }
  }
#pragma unroll
  for (int j = 0; j < J; ++j) arow[j] = v[j];
}

template <class P>
cudaError_t launch_tiny(const RowPassArgs& a, const uint32_t* rows, uint32_t nrows, cudaStream_t s, P pol) {
  if (nrows == 0) return cudaSuccess;
  constexpr int J = P::JN;
  constexpr int NAs = (J * (J + 1) / 2 + J) | 1;
  const size_t sm = VEST_TINY_REG ? 0 : (size_t)128 * NAs * sizeof(double);
  cudaFuncSetAttribute(k_rowpass_tiny<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  k_rowpass_tiny<P><<<(nrows + 127) / 128, 128, sm, s>>>(a, pol, rows, nrows);
  count_launch();
  return cudaGetLastError();
}

// --------------------------------------------- statistics from a given delta --
// The row pass when delta was produced elsewhere (the mask-specialised
// contraction of vest_sparse.cu): delta[j][pos - p0] SoA.  One warp per
// chunk; kStats stages (delta, x) transposed and accumulates the Gram on DMMA
// exactly as k_rowpass, solves light rows in-kernel (heavy rows: partials for
// k_heavy) and, for the last mode, writes the fused residual
// r = x - delta . a_row of the solved row (tucker_model.hpp:168-183: B(alpha)
// = delta_n(alpha) . a_n[i_n]); kResid does the same for rows k_heavy solved.
template <int JN, int KIND, class DT>
__global__ void __launch_bounds__(kRowWarps * 32, 2) k_rowpass_delta(RowPassArgs a, const DT* __restrict__ delta,
                                                                     uint64_t dstride, uint64_t p0) {
  static_assert(JN + 1 <= 16, "DMMA tile: J <= 15");
  __shared__ double smem_d[kRowWarps][16 * kXld];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t ci = blockIdx.x * kRowWarps + warp;
  if (ci >= a.csf.nchunks) return;
  const Chunk ch = a.csf.chunks[ci];
  const int mode = a.mode;
  double* wsm = smem_d[warp];
  double* arow_p = a.m.factor[mode] + (size_t)ch.row * a.m.ld[mode];
  if constexpr (KIND == kResid) {
    double arow[JN];
#pragma unroll
    for (int j = 0; j < JN; ++j) arow[j] = __ldg(arow_p + j);
    double sq = 0.0;
    for (uint32_t pos = ch.beg + lane; pos < ch.end; pos += 32) {
      double rec = 0.0;
#pragma unroll
      for (int j = 0; j < JN; ++j) rec = fma((double)__ldg(delta + j * dstride + (pos - p0)), arow[j], rec);
      const double r = __ldg(a.csf.val + pos) - rec;
      a.r_out[pos] = r;
      sq = fma(r, r, sq);
    }
    sq = warp_sum(sq);
    if (lane == 0) a.chunk_out[ci] = sq;
    return;
  } else {
    for (int t = lane; t < 16 * kXld; t += 32) wsm[t] = 0.0;
    __syncwarp();
    double tc[3][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
    for (uint32_t base = ch.beg; base < ch.end; base += 32) {
      const uint32_t pos = base + lane;
      const bool valid = pos < ch.end;
#pragma unroll
      for (int j = 0; j < JN; ++j) wsm[j * kXld + lane] = valid ? (double)__ldg(delta + j * dstride + (pos - p0)) : 0.0;
      wsm[JN * kXld + lane] = valid ? __ldg(a.csf.val + pos) : 0.0;
      __syncwarp();
      gram_dmma<JN + 1, 1>(wsm, tc, lane);
      __syncwarp();
    }
    constexpr int J = JN;
    constexpr int NG = J * (J + 1) / 2;
    double* Gs = wsm;          // J x J
    double* xd = wsm + J * J;  // J
#pragma unroll
    for (int t = 0; t < (JN + 1 > 8 ? 3 : 1); ++t) {
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        int row, col;
        gram_coord(t, i, lane, row, col);
        const double v = tc[t][i];
        int slot = -1;
        if (row <= col && col < J) slot = row * J - row * (row - 1) / 2 + (col - row);
        else if (col == J && row < J) slot = NG + row;
        if (slot < 0) continue;
        if (ch.slot != kLight) {
          a.heavy_out[(size_t)ch.slot * a.stride_na + slot] = v;
        } else if (col == J) {
          xd[row] = v;
        } else {
          Gs[row * J + col] = v;
          Gs[col * J + row] = v;
        }
      }
    }
    if (ch.slot != kLight) return;
    __syncwarp();
    solve_row(J, a.reg, a.lambda, Gs, xd, arow_p, a.m.fmask[mode] + (size_t)ch.row * J, lane);
    if (!a.fuse_resid) return;
    __syncwarp();  // the solved row (global) is visible to the warp
    double arow[JN];
#pragma unroll
    for (int j = 0; j < JN; ++j) arow[j] = arow_p[j];
    for (uint32_t pos = ch.beg + lane; pos < ch.end; pos += 32) {
      double rec = 0.0;
#pragma unroll
      for (int j = 0; j < JN; ++j) rec = fma((double)__ldg(delta + j * dstride + (pos - p0)), arow[j], rec);
      a.r_out[pos] = __ldg(a.csf.val + pos) - rec;
    }
  }
}

template <int JN, class DT>
cudaError_t launch_delta_jt(const RowPassArgs& a, int kind, uint32_t nchunks, const DT* delta, uint64_t dstride,
                            uint64_t p0, cudaStream_t s) {
  const dim3 grid((nchunks + kRowWarps - 1) / kRowWarps);
  if (nchunks > 0) {
    if (kind == kStats) k_rowpass_delta<JN, kStats, DT><<<grid, kRowWarps * 32, 0, s>>>(a, delta, dstride, p0);
    else k_rowpass_delta<JN, kResid, DT><<<grid, kRowWarps * 32, 0, s>>>(a, delta, dstride, p0);
    count_launch();
  }
  if (kind == kStats && a.csf.nheavy > 0) {
    k_heavy<<<(a.csf.nheavy + 7) / 8, 256, 0, s>>>(a, kStats);
    count_launch();
  }
  return cudaGetLastError();
}

template <int JN>
cudaError_t launch_delta_j(const RowPassArgs& a, int kind, uint32_t nchunks, const void* delta, uint64_t dstride,
                           uint64_t p0, cudaStream_t s, bool f32) {
  return f32 ? launch_delta_jt<JN>(a, kind, nchunks, static_cast<const float*>(delta), dstride, p0, s)
             : launch_delta_jt<JN>(a, kind, nchunks, static_cast<const double*>(delta), dstride, p0, s);
}

cudaError_t launch_heavy_stats(const RowPassArgs& a, cudaStream_t s) {
  if (a.csf.nheavy == 0) return cudaSuccess;
  k_heavy<<<(a.csf.nheavy + 7) / 8, 256, 0, s>>>(a, kStats);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_rowpass_delta(const RowPassArgs& a, int kind, uint32_t nchunks, const void* delta,
                                 uint64_t dstride, uint64_t p0, cudaStream_t s, bool f32) {
  switch (a.m.J[a.mode]) {
#define VEST_DJ(JJ) \
  case JJ:          \
    return launch_delta_j<JJ>(a, kind, nchunks, delta, dstride, p0, s, f32);
    VEST_DJ(1) VEST_DJ(2) VEST_DJ(3) VEST_DJ(4) VEST_DJ(5) VEST_DJ(6) VEST_DJ(7) VEST_DJ(8)
    VEST_DJ(9) VEST_DJ(10) VEST_DJ(11) VEST_DJ(12) VEST_DJ(13) VEST_DJ(14) VEST_DJ(15)
#undef VEST_DJ
    default:
      return cudaErrorInvalidValue;
  }
}

// ------------------------------------------------------- COO reconstruction --
// predict / evaluate_test (trainer.hpp:172-190) on entry-major coordinates.
template <class S>
struct CooStatic {
  __device__ __forceinline__ static double recon(const DevModel& m, const uint32_t* at) {
    double u[1][S::N][S::MAXJ];
    static_for<0, S::N>([&](auto kc) {
      constexpr int k = decltype(kc)::value;
      constexpr int ld = (S::J(k) + 1) & ~1;
      if constexpr (k != 1 || S::G() <= kFullUnrollN)
        load_row<S::J(k)>(m.factor[k] + (size_t)__ldg(at + k) * ld, u[0][k]);
    });
    constexpr int ld1 = (S::J(1) + 1) & ~1;
    const double* const rows0[1] = {m.factor[1] + (size_t)__ldg(at + 1) * ld1};
    double d[1][S::MAXJ];
    delta_staticN<S, 0, 1>(ConstCore{}, u, rows0, d);
    double r = 0.0;
#pragma unroll
    for (int j = 0; j < S::J(0); ++j) r = fma(d[0][j], u[0][0][j], r);
    return r;
  }
};

struct CooDyn {
  // reconstruct_entry (tucker_model.hpp:112-131) cell loop
  __device__ __forceinline__ static double recon(const DevModel& m, const uint32_t* at) {
    double acc = 0.0;
    for (int lin = 0; lin < m.G; ++lin) {
      const double g = __ldg(m.core + lin);
      if (g == 0.0) continue;
      const uint32_t beta = __ldg(m.cellbeta + lin);
      double p = g;
      for (int k = 0; k < m.N; ++k)
        p *= __ldg(m.factor[k] + (size_t)__ldg(at + k) * m.ld[k] + ((beta >> (4 * k)) & 15u));
      acc += p;
    }
    return acc;
  }
};

// out[q] = B(coords[q]) (predict) when values == nullptr; otherwise per-block
// partial (sum r^2, sum x^2) for evaluate_test.
template <class R>
__global__ void __launch_bounds__(256) k_coo_recon(DevModel m, const uint32_t* coords,
                                                   const double* values, uint64_t n, double* out,
                                                   double* partial) {
  __shared__ double red[2][8];
  double sr = 0.0, sx = 0.0;
  for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < n;
       q += (uint64_t)gridDim.x * blockDim.x) {
    const double b = R::recon(m, coords + q * m.N);
    if (values) {
      const double x = values[q];
      const double r = x - b;
      sr = fma(r, r, sr);
      sx = fma(x, x, sx);
    } else {
      out[q] = b;
    }
  }
  if (!values) return;
  sr = warp_sum(sr);
  sx = warp_sum(sx);
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) red[0][w] = sr, red[1][w] = sx;
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) a += red[0][i], b += red[1][i];
    partial[2 * blockIdx.x] = a;
    partial[2 * blockIdx.x + 1] = b;
  }
}

// ---------------------------------------------------------------- launchers --
template <class P>
size_t rowpass_smem(int G) {
  return ((size_t)kRowWarps * stage_words<P>() + (P::kSmemCore ? (size_t)G : 0)) * sizeof(double);
}

template <class P, int KIND>
void launch_kind(const RowPassArgs& a, uint32_t nchunks, cudaStream_t s, P pol) {
  const dim3 grid((nchunks + kRowWarps - 1) / kRowWarps);
  const size_t sm = rowpass_smem<P>(a.m.G);
  cudaFuncSetAttribute(k_rowpass<P, KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  k_rowpass<P, KIND><<<grid, kRowWarps * 32, sm, s>>>(a, pol);
  count_launch();
}

template <class P, bool kWithResid>
cudaError_t run_rowpass(const RowPassArgs& a, int kind, uint32_t nchunks, cudaStream_t s, P pol) {
  if (nchunks > 0) {
    if (kind == kStats) launch_kind<P, kStats>(a, nchunks, s, pol);
    else if (kind == kResp) launch_kind<P, kResp>(a, nchunks, s, pol);
    else if constexpr (kWithResid) launch_kind<P, kResid>(a, nchunks, s, pol);
    else return cudaErrorInvalidValue;
  }
  if (kind != kResid && a.csf.nheavy > 0) {
    k_heavy<<<(a.csf.nheavy + 7) / 8, 256, 0, s>>>(a, kind);
    count_launch();
  }
  return cudaGetLastError();
}

cudaError_t launch_rowpass_generic(const RowPassArgs& a, int kind, uint32_t nchunks, cudaStream_t s) {
  DynPolicy pol;
  pol.md = a.mode;
  pol.jn = a.m.J[a.mode];
  return run_rowpass<DynPolicy, true>(a, kind, nchunks, s, pol);
}

cudaError_t launch_coo_recon_generic(const DevModel& m, const uint32_t* coords, const double* values,
                                     uint64_t n, double* out, double* partial, int nblocks,
                                     cudaStream_t s) {
  k_coo_recon<CooDyn><<<nblocks, 256, 0, s>>>(m, coords, values, n, out, partial);
  count_launch();
  return cudaGetLastError();
}

// -------------------------------------------------- compile-time rank tables --
template <class S, int MODE>
cudaError_t static_mode(const RowPassArgs& a, int kind, uint32_t nchunks, cudaStream_t s) {
  StaticPolicy<S, MODE> pol{};
  return run_rowpass<StaticPolicy<S, MODE>, MODE == S::N - 1>(a, kind, nchunks, s, pol);
}

template <class S, int M = 0>
cudaError_t static_rowtiny(const RowPassArgs& a, const uint32_t* rows, uint32_t nrows, cudaStream_t s) {
  if constexpr (M < S::N) {
    if (a.mode == M) return launch_tiny(a, rows, nrows, s, StaticPolicy<S, M>{});
    return static_rowtiny<S, M + 1>(a, rows, nrows, s);
  } else {
    return cudaErrorInvalidValue;
  }
}

template <class S, int M = 0>
cudaError_t static_rowpass(const RowPassArgs& a, int kind, uint32_t nchunks, cudaStream_t s) {
  if constexpr (M < S::N) {
    if (a.mode == M) return static_mode<S, M>(a, kind, nchunks, s);
    return static_rowpass<S, M + 1>(a, kind, nchunks, s);
  } else {
    return cudaErrorInvalidValue;
  }
}

template <class S>
cudaError_t static_coo(const DevModel& m, const uint32_t* coords, const double* values, uint64_t n,
                       double* out, double* partial, int nblocks, cudaStream_t s) {
  k_coo_recon<CooStatic<S>><<<nblocks, 256, 0, s>>>(m, coords, values, n, out, partial);
  count_launch();
  return cudaGetLastError();
}

template <int... Js>
constexpr ShapeOps make_ops() {
  ShapeOps o{};
  o.N = sizeof...(Js);
  const int js[] = {Js...};
  for (int k = 0; k < (int)sizeof...(Js); ++k) o.J[k] = js[k];
  o.rowpass = &static_rowpass<SShape<Js...>>;
  o.coo_recon = &static_coo<SShape<Js...>>;
  o.rowtiny = &static_rowtiny<SShape<Js...>>;
  return o;
}

// The BASELINE.json configurations' rank tuples (plus their 2-mode analogue
// used by the fixtures); anything else runs the generic kernels.
// (VEST_DEV_ONE_SHAPE: development builds that only inspect config 2's SASS.)
static const ShapeOps kOps[] = {
#ifndef VEST_DEV_ONE_SHAPE
    make_ops<5, 5, 5>(),        // config 1
#endif
    make_ops<10, 10, 10>(),     // config 2
#ifndef VEST_DEV_ONE_SHAPE
    make_ops<10, 10, 5>(),      // config 3
    make_ops<8, 8, 8, 8>(),     // config 4
    make_ops<5, 5, 5, 5, 5>(),  // config 5
#endif
};

const ShapeOps* find_shape_ops(int N, const int* J) {
  for (const auto& o : kOps) {
    if (o.N != N) continue;
    bool eq = true;
    for (int k = 0; k < N; ++k) eq = eq && o.J[k] == J[k];
    if (eq) return &o;
  }
  return nullptr;
}

// The rank-specialised kernels read the core from this module's constant
// bank, which is one per device, not one per context.  Contexts on the same
// device take turns: a lease (held only while its kernels are enqueued)
// reloads the bank from its context's d_core when another context (or an
// older core) is in it, after the previous holder's kernels are done (event),
// so concurrent host threads driving different contexts never read each
// other's core.
namespace {
struct BankState {
  std::mutex mu;
  const Ctx* owner = nullptr;
  uint64_t ver = 0;
  cudaEvent_t done = nullptr;  // recorded after the holder's last kernel that reads the bank
};
BankState& bank_state(int device) {
  static BankState s[64];
  return s[device & 63];
}
}  // namespace

void sync_const_core(Ctx& c) { ++c.core_ver; }

ConstBankLease::ConstBankLease(Ctx& ctx, bool whole_graph) : c(ctx), graph(whole_graph) {
  active = c.G <= VEST_CONST_CORE_MAX;
  if (!active) return;
  BankState& b = bank_state(c.device);
  b.mu.lock();
  const bool other = b.owner != &c;
  if (other && b.done && !c.capturing) check(cudaStreamWaitEvent(c.stream, b.done, 0), "constant bank turn");
  if (!graph && (other || b.ver != c.core_ver)) {
    check(cudaMemcpyToSymbolAsync(c_core_pairs, c.d_core, sizeof(double) * c.G, 0, cudaMemcpyDeviceToDevice,
                                  c.stream),
          "core -> constant bank (pairs)");
    b.owner = &c;
    b.ver = c.core_ver;
  }
}

ConstBankLease::~ConstBankLease() {
  if (!active) return;
  BankState& b = bank_state(c.device);
  if (!c.capturing) {
    if (!b.done) cudaEventCreateWithFlags(&b.done, cudaEventDisableTiming);
    cudaEventRecord(b.done, c.stream);
  }
  if (graph) {  // the graph loaded some core version itself
    b.owner = &c;
    b.ver = 0;
  }
  b.mu.unlock();
}

// After a stream capture: its copies run at replay time, so the bank's real
// content is unknown.
void const_bank_forget(Ctx& c) {
  BankState& b = bank_state(c.device);
  std::lock_guard<std::mutex> g(b.mu);
  if (b.owner == &c) b.owner = nullptr;
}

}  // namespace vest
