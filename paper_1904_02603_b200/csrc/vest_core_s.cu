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

struct CoreSOps {
  int N;
  int J[VEST_MAXN];
  cudaError_t (*pass)(const CorePassSArgs& a, cudaStream_t s);
  cudaError_t (*pack)(const DevModel& m, const DevCSF& csf, uint64_t p0, uint64_t p1, double* U, double* W,
                      uint64_t wstride, cudaStream_t s);
};

template <int... Js>
constexpr CoreSOps make_core_ops() {
  CoreSOps o{};
  o.N = sizeof...(Js);
  const int js[] = {Js...};
  for (int k = 0; k < (int)sizeof...(Js); ++k) o.J[k] = js[k];
  o.pass = &run_core_pass_s<SShape<Js...>>;
  o.pack = &run_pack_uw<SShape<Js...>>;
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

