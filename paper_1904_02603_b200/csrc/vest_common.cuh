// SPDX-License-Identifier: Apache-2.0
// vest_common.cuh -- device-side building blocks shared by the VeST kernels:
// shape descriptors (compile-time "SShape" and runtime "DShape"), the device
// views of the model and of one mode's CSF, warp helpers, and the per-entry
// contraction (delta) that every hot kernel is built around.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>

#include "vest_internal.h"

namespace vest {

constexpr int kWarp = 32;

// ------------------------------------------------------------ warp helpers --
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double warp_bcast(double v, int src) {
  return __shfl_sync(0xffffffffu, v, src);
}

// ------------------------------------------------------------------ shapes --
// Compile-time ranks: every loop over a rank unrolls and every factor row
// lives in registers; the core is read from the constant bank with immediate
// offsets (the contraction below folds the cell index at compile time).
template <int... Js>
struct SShape {
  static constexpr int N = sizeof...(Js);
  static constexpr bool kStatic = true;
  __host__ __device__ static constexpr int J(int k) {
    constexpr int a[] = {Js...};
    return a[k];
  }
  __host__ __device__ static constexpr int stride(int k) {
    int s = 1;
    for (int q = N - 1; q > k; --q) s *= J(q);
    return s;
  }
  __host__ __device__ static constexpr int G() { return (Js * ...); }
  __host__ __device__ static constexpr int maxJ() {
    int m = 0;
    for (int k = 0; k < N; ++k) m = J(k) > m ? J(k) : m;
    return m;
  }
  static constexpr int MAXJ = maxJ();
};

// ------------------------------------------------------------ core access --
// One copy of the dense core per translation unit that contracts with it.
// Updated (device-to-device, in stream order) before every launch that reads
// it; see sync_const_core() in the .cu files.
#define VEST_CONST_CORE_MAX 8192

// ------------------------------------------------------------- contraction --
// delta(j) for mode n (updates.hpp:35-52, "compute_delta"): the reconstruction
// with the mode-n factor row replaced by the j-th unit vector,
//   delta[j] = sum_{beta: beta_n = j} G[beta] prod_{k != n} u_k[beta_k].
// Factorised: modes before n scale a running weight w, modes after n are
// contracted innermost-first (nested dot products), so the cost is
// |G| + |G|/J_{N-1} + ... FMAs instead of the reference's |G|*(N-1)
// multiplies.  Summation order differs from the reference (rounding only).
#ifndef VEST_CONST_PAIRS
#define VEST_CONST_PAIRS 1
#endif
// Single-entry form (the rolled outer loop keeps the core offset in a
// uniform register: LDCU operands).
template <class S, int k, class GA>
__device__ __forceinline__ double trailing(const GA& g, const double (&u)[S::N][S::MAXJ], int lin) {
  if constexpr (k == S::N) {
    return g(lin);
  } else if constexpr (k == S::N - 1) {
    if constexpr ((S::J(k) & 1) == 0 && VEST_CONST_PAIRS) {
      // lin is a multiple of J_{N-1} (even): adjacent cells as one 128-bit load
      double s = 0.0;
#pragma unroll
      for (int c = 0; c < S::J(k); c += 2) {
        const double2 p = g.pair(lin + c);
        s = c == 0 ? p.x * u[k][0] : fma(p.x, u[k][c], s);
        s = fma(p.y, u[k][c + 1], s);
      }
      return s;
    } else {
      double s = g(lin) * u[k][0];
#pragma unroll
      for (int c = 1; c < S::J(k); ++c) s = fma(g(lin + c), u[k][c], s);
      return s;
    }
  } else {
    double s = u[k][0] * trailing<S, k + 1>(g, u, lin);
#pragma unroll
    for (int b = 1; b < S::J(k); ++b) s = fma(u[k][b], trailing<S, k + 1>(g, u, lin + b * S::stride(k)), s);
    return s;
  }
}

template <class S, int n, int k, class GA>
__device__ __forceinline__ void delta_prefix(const GA& g, const double (&u)[S::N][S::MAXJ], double w,
                                             int lin, double (&delta)[S::MAXJ]) {
  if constexpr (k == n) {
    if constexpr (n == S::N - 1 && (S::J(n) & 1) == 0 && VEST_CONST_PAIRS) {
#pragma unroll
      for (int j = 0; j < S::J(n); j += 2) {
        const double2 p = g.pair(lin + j);
        delta[j] = fma(w, p.x, delta[j]);
        delta[j + 1] = fma(w, p.y, delta[j + 1]);
      }
    } else {
#pragma unroll
      for (int j = 0; j < S::J(n); ++j) {
        const double t = trailing<S, n + 1>(g, u, lin + j * S::stride(n));
        delta[j] = fma(w, t, delta[j]);
      }
    }
  } else {
#pragma unroll
    for (int b = 0; b < S::J(k); ++b) {
      const double w2 = w * u[k][b];
      delta_prefix<S, n, k + 1>(g, u, w2, lin + b * S::stride(k), delta);
    }
  }
}

// The outermost "other" mode k0 (the first mode != n) runs as a rolled loop:
// its factor value is read per iteration (L1-resident row) and the core index
// gets a warp-uniform runtime offset, which keeps the unrolled body at
// |G|/J_k0 cells and the register footprint small.  u[k0] is unused.
// kFull: the k0 loop fully unrolled (every core offset an immediate: uniform
// constant loads even inside divergent code, e.g. a chunk's tail round)
template <class S, int n, class GA, bool kFull = false>
__device__ __forceinline__ void delta_static(const GA& g, const double (&u)[S::N][S::MAXJ],
                                             const double* __restrict__ row_k0,
                                             double (&delta)[S::MAXJ]) {
  constexpr int k0 = (n == 0) ? 1 : 0;
#pragma unroll
  for (int j = 0; j < S::J(n); ++j) delta[j] = 0.0;
#pragma unroll(kFull ? S::J(k0) : 1)
  for (int a = 0; a < S::J(k0); ++a) {
    const double w0 = __ldg(row_k0 + a);
    const int base = a * S::stride(k0);
    if constexpr (n == 0) {
#pragma unroll
      for (int j = 0; j < S::J(0); ++j)
        delta[j] = fma(w0, trailing<S, 2>(g, u, base + j * S::stride(0)), delta[j]);
    } else {
      delta_prefix<S, n, 1>(g, u, w0, base, delta);
    }
  }
}


// Multi-entry form: NE entries per lane share every core-value load (one
// uniform constant load feeds NE DFMA), which lifts the issue bound of the
// single-entry contraction (one LDCU per DFMA).  Same factorisation as above;
// the outermost "other" mode k0 (first mode != n) runs as a rolled loop whose
// factor values are read per iteration (rows0[e]) and whose core offset is a
// warp-uniform runtime value.
template <class S, int k, int NE, class GA>
__device__ __forceinline__ void trailingN(const GA& g, const double (&u)[NE][S::N][S::MAXJ], int lin,
                                          double (&s)[NE]) {
  if constexpr (k == S::N) {
    const double v = g(lin);
#pragma unroll
    for (int e = 0; e < NE; ++e) s[e] = v;
  } else if constexpr (k == S::N - 1) {
    {
      const double v = g(lin);
#pragma unroll
      for (int e = 0; e < NE; ++e) s[e] = v * u[e][k][0];
    }
#pragma unroll
    for (int c = 1; c < S::J(k); ++c) {
      const double v = g(lin + c);
#pragma unroll
      for (int e = 0; e < NE; ++e) s[e] = fma(v, u[e][k][c], s[e]);
    }
  } else {
    double t[NE];
    trailingN<S, k + 1, NE>(g, u, lin, t);
#pragma unroll
    for (int e = 0; e < NE; ++e) s[e] = u[e][k][0] * t[e];
#pragma unroll
    for (int b = 1; b < S::J(k); ++b) {
      trailingN<S, k + 1, NE>(g, u, lin + b * S::stride(k), t);
#pragma unroll
      for (int e = 0; e < NE; ++e) s[e] = fma(u[e][k][b], t[e], s[e]);
    }
  }
}

template <class S, int n, int k, int NE, class GA>
__device__ __forceinline__ void delta_prefixN(const GA& g, const double (&u)[NE][S::N][S::MAXJ],
                                              const double (&w)[NE], int lin, double (&delta)[NE][S::MAXJ]) {
  if constexpr (k == n) {
#pragma unroll
    for (int j = 0; j < S::J(n); ++j) {
      double t[NE];
      trailingN<S, n + 1, NE>(g, u, lin + j * S::stride(n), t);
#pragma unroll
      for (int e = 0; e < NE; ++e) delta[e][j] = fma(w[e], t[e], delta[e][j]);
    }
  } else {
#pragma unroll
    for (int b = 0; b < S::J(k); ++b) {
      double w2[NE];
#pragma unroll
      for (int e = 0; e < NE; ++e) w2[e] = w[e] * u[e][k][b];
      delta_prefixN<S, n, k + 1, NE>(g, u, w2, lin + b * S::stride(k), delta);
    }
  }
}

#ifndef VEST_FULL_UNROLL
#define VEST_FULL_UNROLL 0
#endif
constexpr int kFullUnrollN = VEST_FULL_UNROLL;
#ifndef VEST_K0_UNROLL
#define VEST_K0_UNROLL 2
#endif
constexpr int kK0Unroll = VEST_K0_UNROLL;  // unroll of the rolled k0 loop

template <class S, int n, int NE, class GA, int K0U = kK0Unroll>
__device__ __forceinline__ void delta_staticN(const GA& g, const double (&u)[NE][S::N][S::MAXJ],
                                              const double* const (&rows0)[NE], double (&delta)[NE][S::MAXJ]) {
  constexpr int k0 = (n == 0) ? 1 : 0;
#pragma unroll
  for (int e = 0; e < NE; ++e)
#pragma unroll
    for (int j = 0; j < S::J(n); ++j) delta[e][j] = 0.0;
  if constexpr (S::G() <= kFullUnrollN) {
    // every core index a compile-time constant: adjacent cells pair into
    // 128-bit uniform constant loads (LDCU.128)
    double w1[NE];
#pragma unroll
    for (int e = 0; e < NE; ++e) w1[e] = 1.0;
    if constexpr (n == 0) {
#pragma unroll
      for (int j = 0; j < S::J(0); ++j) {
        double t[NE];
        trailingN<S, 1, NE>(g, u, j * S::stride(0), t);
#pragma unroll
        for (int e = 0; e < NE; ++e) delta[e][j] = t[e];
      }
    } else {
      delta_prefixN<S, n, 0, NE>(g, u, w1, 0, delta);
    }
    return;
  }
#pragma unroll K0U
  for (int a = 0; a < S::J(k0); ++a) {
    double w0[NE];
#pragma unroll
    for (int e = 0; e < NE; ++e) w0[e] = __ldg(rows0[e] + a);
    const int base = a * S::stride(k0);
    if constexpr (n == 0) {
#pragma unroll
      for (int j = 0; j < S::J(0); ++j) {
        double t[NE];
        trailingN<S, 2, NE>(g, u, base + j * S::stride(0), t);
#pragma unroll
        for (int e = 0; e < NE; ++e) delta[e][j] = fma(w0[e], t[e], delta[e][j]);
      }
    } else {
      delta_prefixN<S, n, 1, NE>(g, u, w0, base, delta);
    }
  }
}

// The shape without its last mode (the fused residual's contraction with
// v = G x_{N-1} a_row).
template <class S, class Seq>
struct PrefixImpl;
template <class S, int... I>
struct PrefixImpl<S, std::integer_sequence<int, I...>> {
  using type = SShape<S::J(I)...>;
};
template <class S>
using PrefixShape = typename PrefixImpl<S, std::make_integer_sequence<int, S::N - 1>>::type;

// ------------------------------------------------------- FP64 tensor cores --
// D(8x8) += A(8x4) B(4x8), mma.sync m8n8k4 f64 (SASS DMMA.8x8x4; tensor pipe,
// concurrent with the DFMA pipe).  Fragments: A[g][t], B[t][g], D[g][2t + i]
// with g = lane / 4, t = lane % 4.
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// Gram of 32*NE staged column vectors: X is [col][entry] with row stride
// kXldN(NE) (== 4 mod 16: conflict-free fragment loads); accumulates the upper
// tile blocks of X^T X for NC <= 16 columns into d[3][2] (tiles (0,0), (0,1),
// (1,1)), one DMMA per tile per 4 entries.
__host__ __device__ constexpr int kXldN(int ne) { return 32 * ne + 4; }
constexpr int kXld = kXldN(1);
template <int NC, int NE = 1>
__device__ __forceinline__ void gram_dmma(const double* X, double (&d)[3][2], int lane) {
  constexpr int ld = kXldN(NE);
  const int g = lane >> 2, tq = lane & 3;
#pragma unroll
  for (int kk = 0; kk < 8 * NE; ++kk) {
    const int e = 4 * kk + tq;
    const double f0 = X[g * ld + e];
    dmma884(d[0][0], d[0][1], f0, f0);
    if constexpr (NC > 8) {
      const double f1 = X[(8 + g) * ld + e];
      dmma884(d[1][0], d[1][1], f0, f1);
      // NC == 9 (J == 8): the second tile row holds x alone, tile (1,1) would be x . x, which no one reads
      if constexpr (NC > 9) dmma884(d[2][0], d[2][1], f1, f1);
    }
  }
}

// (row, col) of accumulator element i of tile t for this lane
__device__ __forceinline__ void gram_coord(int t, int i, int lane, int& row, int& col) {
  const int I = t == 2 ? 1 : 0, J = t == 0 ? 0 : 1;
  row = 8 * I + (lane >> 2);
  col = 8 * J + 2 * (lane & 3) + i;
}

}  // namespace vest
