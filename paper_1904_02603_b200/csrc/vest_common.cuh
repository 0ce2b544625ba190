// SPDX-License-Identifier: Apache-2.0
// vest_common.cuh -- device-side building blocks shared by the VeST kernels:
// shape descriptors (compile-time "SShape" and runtime "DShape"), the device
// views of the model and of one mode's CSF, warp helpers, and the per-entry
// contraction (delta) that every hot kernel is built around.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

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
// The static version is factorised: modes before n scale a running weight w,
// modes after n are contracted innermost-first (nested dot products), so the
// cost is |G| + |G|/J_{N-1} + ... FMAs instead of the reference's |G|*(N-1)
// multiplies.  Summation order differs from the reference (rounding only).
template <class S, int k, class GA>
__device__ __forceinline__ double trailing(const GA& g, const double (&u)[S::N][S::MAXJ], int lin) {
  if constexpr (k == S::N) {
    return g(lin);
  } else if constexpr (k == S::N - 1) {
    double s = g(lin) * u[k][0];
#pragma unroll
    for (int c = 1; c < S::J(k); ++c) s = fma(g(lin + c), u[k][c], s);
    return s;
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
#pragma unroll
    for (int j = 0; j < S::J(n); ++j) {
      const double t = trailing<S, n + 1>(g, u, lin + j * S::stride(n));
      delta[j] = fma(w, t, delta[j]);
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
template <class S, int n, class GA>
__device__ __forceinline__ void delta_static(const GA& g, const double (&u)[S::N][S::MAXJ],
                                             const double* __restrict__ row_k0,
                                             double (&delta)[S::MAXJ]) {
  constexpr int k0 = (n == 0) ? 1 : 0;
#pragma unroll
  for (int j = 0; j < S::J(n); ++j) delta[j] = 0.0;
#pragma unroll 1
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

}  // namespace vest
