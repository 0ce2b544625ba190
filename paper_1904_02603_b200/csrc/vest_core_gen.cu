// SPDX-License-Identifier: Apache-2.0
// vest_core_gen.cu -- the generic core-sweep passes (vest_core.cu
// k_core_pass) generated per block plan and NVRTC-compiled for sm_100a.
//
// A block is a runtime list of live fibers (beta_0..beta_{m-1}); the
// table-driven pass kernel spends most of its instructions on the tables
// (per-fiber guards, constant loads, address arithmetic: ~1570 instructions
// per 32-entry round at config 4).  The plan depends on the core mask only,
// so every pass (previous block's residual update + current block's
// statistics, and the final sum of squares) is emitted as straight-line code:
// the lane's staged factor rows are loaded into registers once per round and
// each fiber product is 1-2 DMUL with compile-time register operands, each
// Gram column store a compile-time shared-memory offset.  Everything else --
// persistent warps over the last mode's chunks, cp.async staging one round
// ahead, the DMMA Gram, the per-chunk statistics layout -- is the table-driven
// kernel's, so its block GEMM and solve consume the output unchanged.  One
// NVRTC program holds all passes of a plan; it is rebuilt only when a prune
// changes the mask.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <exception>
#include <future>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

#include "vest_internal.h"

namespace vest {

struct CoreGenArgs {
  const uint32_t* oc[VEST_MAXN];
  const double* f[VEST_MAXN];
  const float* g[VEST_MAXN];  // fp32 factor copies (gather_f32)
  double* r;
  const double* prev_dg;
  double* stats;
  double* chunk_sq;
  const Chunk* chunks;
  uint32_t nchunks;
  int stride;
};

struct CoreGenState {
  uint64_t key = 0;
  std::vector<cudaLibrary_t> libs;  // the plan's passes, split over parallel-compiled programs
  std::vector<cudaKernel_t> k;  // pass i: prev = i - 1, cur = i (i < nb); pass nb: final
  std::vector<int> nt;
  int ldr = 0;
  bool xf32 = false;  // Gram columns staged as fp32 (fp32 products)
  int nbuf = 1;       // staged rounds in flight
  bool pipe = false;  // statistics passes software-pipelined (two column buffers)
  bool xt = false;    // entry-major Gram columns (640 doubles per warp)
};

namespace {

const char* kPassMark = "//@@PASS\n";  // core_gen_compile cuts the source here

// device prelude shared by every generated pass
const char* kPrelude = R"CUDA(
struct Chunk { unsigned row, beg, end, slot; };
struct CoreGenArgs {
  const unsigned* oc[8]; const double* f[8]; const float* g[8]; double* r; const double* prev_dg; double* stats;
  double* chunk_sq; const Chunk* chunks; unsigned nchunks; int stride;
};
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void cp16(unsigned s, const void* g) {
  asm volatile("cp.async.@CPMOD@.shared.global [%0], [%1], 16;" ::"r"(s), "l"(g) : "memory");
}
__device__ __forceinline__ void cp8(unsigned s, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
__device__ __forceinline__ void cp_wait0() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
// X: the round's Gram columns [column][36] (fp64, or fp32 when the products are
// fp32 -- half the shared-memory traffic of the fragment loads and column
// stores); the residual column (last) is always read in fp64 from Xr
// KK k-steps of 4 entries (straight-line, so the fragment loads of the next
// k-step are scheduled under this one's DMMAs)
template <int NT, class XT>
__device__ __forceinline__ void gram_step(const XT* X, const double* Xr, double (&d)[NT * (NT + 1) / 2][2], int g, int tq,
                                          int kk) {
  const int e = 4 * kk + tq;
  double f[NT];
#pragma unroll
  for (int i = 0; i < NT; ++i) f[i] = (double)X[(8 * i + g) * 36 + e];
  if (g == 7) f[NT - 1] = Xr[e];
  int t = 0;
#pragma unroll
  for (int I = 0; I < NT; ++I)
#pragma unroll
    for (int J = I; J < NT; ++J) { dmma884(d[t][0], d[t][1], f[I], f[J]); ++t; }
}
template <int NT, int KK, class XT>
__device__ __forceinline__ void gram_kk(const XT* X, const double* Xr, double (&d)[NT * (NT + 1) / 2][2], int lane) {
  const int g = lane >> 2, tq = lane & 3;
#pragma unroll
  for (int kk = 0; kk < KK; ++kk) gram_step<NT>(X, Xr, d, g, tq, kk);
}
// Entry-major columns (fp32 products only): Xt[entry][4 g + i] holds Gram column
// 8 i + g of that entry (pitch 40 floats), so a lane stores its 32 products with
// 8 16-byte stores and loads the four fragments of a k-step with ONE 16-byte
// load (both conflict-free) -- the pass is issue-bound (a DMMA holds the
// scheduler's dispatch for its 16 cycles), so every instruction saved outside
// the Gram is time saved.
template <int NT>
__device__ __forceinline__ void gram_step_t(const float* Xt, const double* Xr, double (&d)[NT * (NT + 1) / 2][2], int g,
                                            int tq, int kk) {
  const int e = 4 * kk + tq;
  const float4 v = *reinterpret_cast<const float4*>(Xt + e * 40 + 4 * g);
  const float vv[4] = {v.x, v.y, v.z, v.w};
  double f[NT];
#pragma unroll
  for (int i = 0; i < NT; ++i) f[i] = (double)vv[i];
  if (g == 7) f[NT - 1] = Xr[e];
  int t = 0;
#pragma unroll
  for (int I = 0; I < NT; ++I)
#pragma unroll
    for (int J = I; J < NT; ++J) { dmma884(d[t][0], d[t][1], f[I], f[J]); ++t; }
}
template <int NT, int KK>
__device__ __forceinline__ void gram_kk_t(const float* Xt, const double* Xr, double (&d)[NT * (NT + 1) / 2][2], int lane) {
  const int g = lane >> 2, tq = lane & 3;
#pragma unroll
  for (int kk = 0; kk < KK; ++kk) gram_step_t<NT>(Xt, Xr, d, g, tq, kk);
}
template <int NT>
__device__ __forceinline__ void gram_nt_t(const float* Xt, const double* Xr, double (&d)[NT * (NT + 1) / 2][2], int lane,
                                          int nv) {
  if (nv > 24) gram_kk_t<NT, 8>(Xt, Xr, d, lane);
  else if (nv > 16) gram_kk_t<NT, 6>(Xt, Xr, d, lane);
  else if (nv > 8) gram_kk_t<NT, 4>(Xt, Xr, d, lane);
  else gram_kk_t<NT, 2>(Xt, Xr, d, lane);
}
// a chunk's last round holds nv < 32 entries: k-steps past them are all zero
// and skipped in steps of 8 entries (warp-uniform branch)
template <int NT, class XT>
__device__ __forceinline__ void gram_nt(const XT* X, const double* Xr, double (&d)[NT * (NT + 1) / 2][2], int lane,
                                        int nv) {
  if (nv > 24) gram_kk<NT, 8>(X, Xr, d, lane);
  else if (nv > 16) gram_kk<NT, 6>(X, Xr, d, lane);
  else if (nv > 8) gram_kk<NT, 4>(X, Xr, d, lane);
  else gram_kk<NT, 2>(X, Xr, d, lane);
}
)CUDA";

// one pass: KIND 0 (prev update + cur statistics) or 2 (prev update + r^2)
const char* kPass = R"CUDA(
extern "C" __global__ void __launch_bounds__(128, @MINB@) @NAME@(const CoreGenArgs a) {
  constexpr int M = @M@, LDR = @LDR@, NT = @NT@, NC = NT * 8, NTT = NT * (NT + 1) / 2;
  constexpr int NF = @NF@, PNF = @PNF@, KIND = @KIND@, JM = @JM@, RSLOT = @RSLOT@;
  constexpr bool WSQ = @WSQ@;  // statistics pass that also sums r^2 (after the previous block's update)
  extern __shared__ __align__(16) double smem[];
  __shared__ @PT@ sq_q[4][32];  // previous block's per-fiber a . dg of the chunk's row
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int NBUF = @NBUF@;  // staged rounds in flight (1: next round, 2: the two next rounds)
  double* const stage = smem + (unsigned long long)warp * (NBUF * 32 * LDR + @XD@ + 32);  // NBUF rounds' rows
  @XT@* const X = reinterpret_cast<@XT@*>(stage + NBUF * 32 * LDR);
  double* const Xr = stage + NBUF * 32 * LDR + @XD@;  // the residual column, fp64
  for (int t = lane; t < @XN@; t += 32) X[t] = 0;
  Xr[lane] = 0.0;
  const unsigned wstride = gridDim.x * 4;
  struct Cur { unsigned ci, end, base, row; };
  auto first = [&](unsigned ci) {
    Cur c{ci, 0, 0, 0};
    if (ci < a.nchunks) { const Chunk ch = a.chunks[ci]; c.end = ch.end; c.base = ch.beg; c.row = ch.row; }
    return c;
  };
  auto next = [&](const Cur& c) {
    if (c.base + 32 < c.end) return Cur{c.ci, c.end, c.base + 32, c.row};
    return first(c.ci + wstride);
  };
  auto coords = [&](const Cur& c, unsigned (&idx)[M]) {
    const bool v = c.ci < a.nchunks && c.base + lane < c.end;
#pragma unroll
    for (int k = 0; k < M; ++k) idx[k] = v ? @LDC@(a.oc[k] + c.base + lane) : 0u;
  };
  const unsigned sbase = su32(stage);
  auto issue = [&](const Cur& c, int b, const unsigned (&idx)[M]) {
    if (c.ci < a.nchunks && c.base + lane < c.end) {
      const unsigned st = sbase + (unsigned)((b * 32 + lane) * LDR) * 8u;
@ISSUE@
      cp8(st + RSLOT * 8u, a.r + c.base + lane);
    } else {
      double* sp = stage + (b * 32 + lane) * LDR;  // finite zeros: products of idle lanes vanish
#pragma unroll
      for (int t = 0; t < LDR; ++t) sp[t] = 0.0;
    }
    cp_commit();
  };
  auto prologue = [&](const Cur& c) {
    if (PNF > 0) {
      double t = 0.0;
      if (lane < PNF) {
        const double* arow = a.f[M] + (unsigned long long)c.row * @LDM@;
#pragma unroll
        for (int q = 0; q < JM; ++q) t = fma(__ldg(arow + q), __ldg(a.prev_dg + lane * JM + q), t);
      }
      sq_q[warp][lane] = (@PT@)t;
      __syncwarp();
    }
  };
  Cur cur = first(blockIdx.x * 4 + warp);
  if (cur.ci >= a.nchunks) return;
  { unsigned i0[M]; coords(cur, i0); issue(cur, 0, i0); }
  Cur nxt = next(cur);
  Cur ahead = nxt;  // the round whose gathers are issued next
  if (NBUF == 2) {
    unsigned i1[M];
    coords(nxt, i1);
    issue(nxt, 1, i1);
    ahead = next(nxt);
  }
  unsigned inx[M];
  coords(ahead, inx);
  prologue(cur);
  int p = 0;
  double d[NTT][2];
#pragma unroll
  for (int t = 0; t < NTT; ++t) d[t][0] = d[t][1] = 0.0;
  double sq = 0.0;
  while (true) {
    // this round's rows -> registers, then the gathers of the round NBUF ahead
    // into the buffer just read, while this round computes (NBUF 1: half the
    // shared memory, more resident warps; NBUF 2: a gather has two rounds of
    // compute to land)
    if (NBUF == 2) cp_wait1(); else cp_wait0();
    __syncwarp();
    const double* st = stage + (p * 32 + lane) * LDR;
    const unsigned pos = cur.base + lane;
    const bool valid = pos < cur.end;
    double r = st[RSLOT];
@LOADU@
    __syncwarp();
    issue(ahead, p, inx);
    const Cur nn = next(ahead);
    coords(nn, inx);
    if (PNF > 0 && valid && @PROBE@ != 2) {
      @PT@ t0 = 0, t1 = 0, t2 = 0, t3 = 0;  // four partial sums: no 31-deep dependent chain
@PREV@
      r -= (double)((t0 + t1) + (t2 + t3));
      @STR@;
    }
    if (KIND == 2 || WSQ) sq = fma(r, r, sq);
    if (KIND != 2) {
      if (@PROBE@ != 2) {
@CUR@
      }
      Xr[lane] = r;
      __syncwarp();
      if (@PROBE@ != 1) @GRAM@<NT>(X, Xr, d, lane, (int)min(32u, cur.end - cur.base));
    }
    __syncwarp();
    if (nxt.ci != cur.ci) {
      const unsigned ci = cur.ci;
      if (KIND == 2 || WSQ) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
        if (lane == 0) a.chunk_sq[ci] = sq;
        sq = 0.0;
      }
      if (KIND != 2) {
        @STATS_T@* out = reinterpret_cast<@STATS_T@*>(a.stats) + (unsigned long long)ci * a.stride;
        constexpr int NS = NF * (NF + 1) / 2;
        const int g = lane >> 2, tq = lane & 3;
        int t = 0;
#pragma unroll
        for (int I = 0; I < NT; ++I) {
#pragma unroll
          for (int J = I; J < NT; ++J) {
#pragma unroll
            for (int i = 0; i < 2; ++i) {
              const int row = 8 * I + g, col = 8 * J + 2 * tq + i;
              if (row <= col && col < NF) out[row * NF - row * (row - 1) / 2 + (col - row)] = (@STATS_T@)d[t][i];
              else if (col == NC - 1 && row < NF) out[NS + row] = (@STATS_T@)d[t][i];
              d[t][i] = 0.0;
            }
            ++t;
          }
        }
      }
      if (nxt.ci >= a.nchunks) break;
      prologue(nxt);
    }
    cur = nxt;
    if (NBUF == 2) { nxt = ahead; p ^= 1; } else { nxt = nn; }
    ahead = nn;
  }
  cp_wait0();
}
)CUDA";

// The statistics pass, software-pipelined inside the warp: while the DMMA Gram
// of round g runs from one column buffer, the products of round g + 1 (its
// residual update and Gram columns) are formed into the other -- the generated
// source interleaves a slice of the product code after every k-step of the
// Gram, so the FP32/LSU work sits in the issue slots the DMMAs leave free.
const char* kPassPipe = R"CUDA(
extern "C" __global__ void __launch_bounds__(128, @MINB@) @NAME@(const CoreGenArgs a) {
  constexpr int M = @M@, LDR = @LDR@, NT = @NT@, NC = NT * 8, NTT = NT * (NT + 1) / 2;
  constexpr int NF = @NF@, PNF = @PNF@, JM = @JM@, RSLOT = @RSLOT@, XD = @XD@;
  constexpr bool WSQ = @WSQ@;
  extern __shared__ __align__(16) double smem[];
  __shared__ @PT@ sq_q[4][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // per warp: one round's staged rows | two rounds' Gram columns | their residual columns
  double* const stage = smem + (unsigned long long)warp * (32 * LDR + 2 * XD + 64);
  @XT@* const X0 = reinterpret_cast<@XT@*>(stage + 32 * LDR);
  double* const Xr0 = stage + 32 * LDR + 2 * XD;
  constexpr int XE = NC * 36;  // elements of one column buffer
  for (int t = lane; t < 2 * XE; t += 32) X0[t] = 0;
  Xr0[lane] = 0.0;
  Xr0[32 + lane] = 0.0;
  const unsigned wstride = gridDim.x * 4;
  struct Cur { unsigned ci, end, base, row; };
  auto first = [&](unsigned ci) {
    Cur c{ci, 0, 0, 0};
    if (ci < a.nchunks) { const Chunk ch = a.chunks[ci]; c.end = ch.end; c.base = ch.beg; c.row = ch.row; }
    return c;
  };
  auto next = [&](const Cur& c) {
    if (c.base + 32 < c.end) return Cur{c.ci, c.end, c.base + 32, c.row};
    return first(c.ci + wstride);
  };
  auto coords = [&](const Cur& c, unsigned (&idx)[M]) {
    const bool v = c.ci < a.nchunks && c.base + lane < c.end;
#pragma unroll
    for (int k = 0; k < M; ++k) idx[k] = v ? @LDC@(a.oc[k] + c.base + lane) : 0u;
  };
  const unsigned sbase = su32(stage);
  auto issue = [&](const Cur& c, int b, const unsigned (&idx)[M]) {
    if (c.ci < a.nchunks && c.base + lane < c.end) {
      const unsigned st = sbase + (unsigned)((b * 32 + lane) * LDR) * 8u;
@ISSUE@
      cp8(st + RSLOT * 8u, a.r + c.base + lane);
    } else {
      double* sp = stage + (b * 32 + lane) * LDR;
#pragma unroll
      for (int t = 0; t < LDR; ++t) sp[t] = 0.0;
    }
    cp_commit();
  };
  auto prologue = [&](const Cur& c) {
    if (PNF > 0) {
      double t = 0.0;
      if (lane < PNF) {
        const double* arow = a.f[M] + (unsigned long long)c.row * @LDM@;
#pragma unroll
        for (int q = 0; q < JM; ++q) t = fma(__ldg(arow + q), __ldg(a.prev_dg + lane * JM + q), t);
      }
      sq_q[warp][lane] = (@PT@)t;
      __syncwarp();
    }
  };
  double sq = 0.0;
  auto flush_sq = [&](unsigned ci) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
    if (lane == 0) a.chunk_sq[ci] = sq;
    sq = 0.0;
  };
  Cur cur = first(blockIdx.x * 4 + warp);
  if (cur.ci >= a.nchunks) return;
  { unsigned i0[M]; coords(cur, i0); issue(cur, 0, i0); }
  Cur nxt = next(cur);
  unsigned inx[M];
  coords(nxt, inx);
  prologue(cur);
  double d[NTT][2];
#pragma unroll
  for (int t = 0; t < NTT; ++t) d[t][0] = d[t][1] = 0.0;
  Cur g = cur;  // the round whose Gram is due
  {  // first round: columns into buffer 0
    cp_wait0();
    __syncwarp();
    const double* st = stage + lane * LDR;
    const unsigned pos = cur.base + lane;
    const bool valid = pos < cur.end;
    double r = st[RSLOT];
@LOADU@
    __syncwarp();
    issue(nxt, 0, inx);
    const Cur nn = next(nxt);
    coords(nn, inx);
    @PT@ t0 = 0, t1 = 0, t2 = 0, t3 = 0;
    @XT@* const X = X0;
@PREV@
@FINAL@
@CUR@
    Xr0[lane] = r;
    cur = nxt;
    nxt = nn;
  }
  int p = 0;
  while (true) {
    __syncwarp();  // column buffer p is complete
    const bool more = cur.ci < a.nchunks;
    const @XT@* const Xg = X0 + p * XE;
    const double* const Xrg = Xr0 + 32 * p;
    const int nv = (int)min(32u, g.end - g.base);
    const bool last_of_chunk = !more || cur.ci != g.ci;
    Cur nn = cur;
    if (more) {
      if (cur.ci != g.ci) {
        if (WSQ) flush_sq(g.ci);  // every round of g's chunk has had its residual update
        prologue(cur);
      }
      cp_wait0();
      __syncwarp();
      const double* st = stage + lane * LDR;
      const unsigned pos = cur.base + lane;
      const bool valid = pos < cur.end;
      double r = st[RSLOT];
@LOADU@
      __syncwarp();
      issue(nxt, 0, inx);
      nn = next(nxt);
      coords(nn, inx);
      @PT@ t0 = 0, t1 = 0, t2 = 0, t3 = 0;
      @XT@* const X = X0 + (p ^ 1) * XE;
      if (nv == 32) {
        const int g_ = lane >> 2, tq_ = lane & 3;
@INTER@
      } else {
        gram_nt<NT>(Xg, Xrg, d, lane, nv);
@PREV@
@FINAL@
@CUR@
      }
      Xr0[32 * (p ^ 1) + lane] = r;
    } else {
      gram_nt<NT>(Xg, Xrg, d, lane, nv);
    }
    if (last_of_chunk) {
      @STATS_T@* out = reinterpret_cast<@STATS_T@*>(a.stats) + (unsigned long long)g.ci * a.stride;
      constexpr int NS = NF * (NF + 1) / 2;
      const int gg = lane >> 2, tq = lane & 3;
      int t = 0;
#pragma unroll
      for (int I = 0; I < NT; ++I) {
#pragma unroll
        for (int J = I; J < NT; ++J) {
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const int row = 8 * I + gg, col = 8 * J + 2 * tq + i;
            if (row <= col && col < NF) out[row * NF - row * (row - 1) / 2 + (col - row)] = (@STATS_T@)d[t][i];
            else if (col == NC - 1 && row < NF) out[NS + row] = (@STATS_T@)d[t][i];
            d[t][i] = 0.0;
          }
          ++t;
        }
      }
    }
    if (!more) break;
    g = cur;
    cur = nxt;
    nxt = nn;
    p ^= 1;
  }
  if (WSQ) flush_sq(g.ci);
  cp_wait0();
}
)CUDA";

// VEST_CP_XT=0/1 (A/B): entry-major Gram columns (fp32 products, non-pipelined passes).
bool cp_xt(const Ctx& c) {
  static const bool env = [] {
    const char* e = getenv("VEST_CP_XT");
    return !(e && e[0] == '0');
  }();
  return env;
}

// VEST_CP_PIPE=0/1 (A/B): the software-pipelined statistics passes.
bool cp_pipe(const Ctx& c) {
  static const int env = [] {
    const char* e = getenv("VEST_CP_PIPE");
    return e ? (e[0] == '1' ? 1 : 0) : -1;
  }();
  return env >= 0 ? env == 1 : false;
}

// CTAs per SM the passes are register-budgeted for (VEST_CP_MINB: A/B).
// Config 4, ms per iteration -- fp64 products: no bound 259, 1: 254, 3: 250
// (kept), 4 (128 registers, spills): 318; fp32 products with fp32-staged Gram
// columns (150 registers unbounded, no spills at 128): 3: 170.2, 4: 168.0 (kept).
int cp_min_blocks(bool products_f32) {
  static const int v = [] {
    const char* e = getenv("VEST_CP_MINB");
    return e ? std::max(1, std::min(6, atoi(e))) : 0;
  }();
  return v > 0 ? v : (products_f32 ? 4 : 3);
}

// fp32 mode: the fiber products (previous block's residual update, current
// block's Gram columns) in fp32 arithmetic on the fp32 row copies -- they leave
// the FP64 pipe to the DMMA Gram and halve the registers holding the rows; the
// Gram, the statistics and r stay fp64 (VEST_CP_F32=0: fp64 products, A/B).
bool cp_f32(const Ctx& c) {
  static const bool env = [] {
    const char* e = getenv("VEST_CP_F32");
    return !(e && e[0] == '0');
  }();
  return c.gather_f32 && env;
}

// Staged rounds in flight (VEST_CP_DEPTH=1/2, A/B; 1 kept): with two, a gather
// has two rounds of compute to land -- config 4 passes 95.9 vs 94.8 ms per
// iteration with one: the gathers are not what the DMMA pipe waits for (ncu:
// DMMA pipe 71 %, long_scoreboard 0.9 of 11.5 stall cycles per instruction).
int cp_depth(const Ctx&) {
  static const int env = [] {
    const char* e = getenv("VEST_CP_DEPTH");
    return e ? std::max(1, std::min(2, atoi(e))) : 1;
  }();
  return env;
}

void replace_all(std::string& s, const std::string& from, const std::string& to) {
  for (size_t p = 0; (p = s.find(from, p)) != std::string::npos; p += to.size()) s.replace(p, from.size(), to);
}

std::string uname(int k, int b) { return "u" + std::to_string(k) + "_" + std::to_string(b); }

// fiber p (row-major over modes 0..m-1) -> betas
void fiber_beta(const Ctx& c, uint32_t p, int* beta) {
  const int m = c.N - 1;
  for (int k = m - 1; k >= 0; --k) {
    beta[k] = (int)(p % (uint32_t)c.ranks[k]);
    p /= (uint32_t)c.ranks[k];
  }
}

// straight-line products of a block's fibers; emit(f, expr) consumes each
void products(const Ctx& c, const std::vector<uint32_t>& fib, std::ostringstream& out,
              const std::function<std::string(int, const std::string&)>& emit, std::vector<bool>& used,
              const char* T = "double", std::vector<std::string>* blocks = nullptr,
              const std::function<std::string(int)>& dot_coef = nullptr, const char* fma_name = "fma") {
  // dot_coef (the residual update): sum_f (w u_f) q_f is formed per prefix as
  // w * (sum_f u_f q_f) -- one FMA per fiber plus one per prefix instead of a
  // multiply and an FMA per fiber; emit(block index, "w * in") consumes it
  const int M = c.N - 1;
  int prev[VEST_MAXN];
  bool open = false, first_in = true;
  int nblk = 0;
  std::ostringstream o;
  auto close = [&]() {  // one prefix's products: a self-contained block
    if (dot_coef) o << "        " << emit(nblk, "w, in") << "\n";
    ++nblk;
    o << "      }\n";
    out << o.str();
    if (blocks) blocks->push_back(o.str());
    o.str("");
  };
  for (size_t f = 0; f < fib.size(); ++f) {
    int beta[VEST_MAXN];
    fiber_beta(c, fib[f], beta);
    bool same = open;
    for (int k = 0; k + 1 < M && same; ++k) same = beta[k] == prev[k];
    if (!same) {
      if (open) close();
      o << "      { const " << T << " w = ";
      if (M == 1) {
        o << "1";
      } else {
        for (int k = 0; k + 1 < M; ++k) {
          o << (k ? " * " : "") << uname(k, beta[k]);
          used[k * 16 + beta[k]] = true;
        }
      }
      o << ";\n";
      open = true;
      first_in = true;
    }
    for (int k = 0; k < M; ++k) prev[k] = beta[k];
    used[(M - 1) * 16 + beta[M - 1]] = true;
    if (dot_coef) {
      const std::string u = uname(M - 1, beta[M - 1]), q = dot_coef((int)f);
      if (first_in) o << "        " << T << " in = " << u << " * " << q << ";\n";
      else o << "        in = " << fma_name << "(" << u << ", " << q << ", in);\n";
      first_in = false;
      continue;
    }
    o << "        " << emit((int)f, "w * " + uname(M - 1, beta[M - 1])) << "\n";
  }
  if (open) close();
}

// The pipelined pass's interleaved region: one Gram k-step, then a slice of
// the next round's product code (residual-update blocks in the first slices,
// then the update itself, Gram-column blocks spread over all eight).
std::string interleave(const std::vector<std::string>& prev, const std::vector<std::string>& cur,
                       const std::string& fin) {
  auto weight = [](const std::string& b) { return (int)std::count(b.begin(), b.end(), '\n'); };
  std::vector<std::string> slice(8);
  std::vector<int> w(8, 0);
  for (size_t i = 0; i < prev.size(); ++i) {  // slices 0..2, lightest first
    int k = 0;
    for (int q = 1; q < 3; ++q)
      if (w[q] < w[k]) k = q;
    slice[k] += prev[i];
    w[k] += weight(prev[i]);
  }
  slice[prev.empty() ? 0 : 3] += fin;
  w[prev.empty() ? 0 : 3] += 3;
  for (size_t i = 0; i < cur.size(); ++i) {
    int k = 0;
    for (int q = 1; q < 8; ++q)
      if (w[q] < w[k]) k = q;
    slice[k] += cur[i];
    w[k] += weight(cur[i]);
  }
  std::string o;
  for (int kk = 0; kk < 8; ++kk)
    o += "        gram_step<NT>(Xg, Xrg, d, g_, tq_, " + std::to_string(kk) + ");\n" + slice[kk];
  return o;
}

}  // namespace

// The passes of a plan are independent kernels over a common prelude: the
// source is cut at the pass markers into up to 8 programs compiled on parallel
// host threads (a 22-pass plan: 3.1 -> under 1 s), returned as one blob
// [count | sizes | cubins].
std::vector<char> core_gen_compile(const std::string& src, const char* name) {
  std::vector<size_t> cut;
  for (size_t p = src.find(kPassMark); p != std::string::npos; p = src.find(kPassMark, p + 1)) cut.push_back(p);
  const int npass = (int)cut.size();
  const int nparts = npass >= 4 ? std::min(8, npass / 2) : 1;
  std::vector<std::string> part(nparts, cut.empty() ? src : src.substr(0, cut[0]));
  for (int i = 0; i < npass; ++i)
    part[i % nparts] += src.substr(cut[i], (i + 1 < npass ? cut[i + 1] : src.size()) - cut[i]);
  std::vector<std::string> pname(nparts, name);  // distinct names: VEST_NVRTC_DUMP writes one file pair per program
  for (int q = 1; q < nparts; ++q) pname[q] = std::string(name) + ".p" + std::to_string(q);
  std::vector<std::future<std::vector<char>>> fut;
  for (int q = 1; q < nparts; ++q)  // deferred (= compiled in get() below) when no thread can be started
    fut.push_back(std::async(std::launch::async | std::launch::deferred,
                             [&part, &pname, q]() { return nvrtc_compile(part[q], pname[q].c_str()); }));
  std::vector<std::vector<char>> bin(nparts);
  std::exception_ptr err;
  try {
    bin[0] = nvrtc_compile(part[0], pname[0].c_str());
  } catch (...) {
    err = std::current_exception();
  }
  for (int q = 1; q < nparts; ++q) {
    try {
      bin[q] = fut[q - 1].get();
    } catch (...) {
      if (!err) err = std::current_exception();
    }
  }
  if (err) std::rethrow_exception(err);
  std::vector<char> blob((size_t)(1 + nparts) * sizeof(uint64_t));
  uint64_t* hdr = reinterpret_cast<uint64_t*>(blob.data());
  hdr[0] = (uint64_t)nparts;
  for (int q = 0; q < nparts; ++q) hdr[1 + q] = bin[q].size();
  for (int q = 0; q < nparts; ++q) blob.insert(blob.end(), bin[q].begin(), bin[q].end());
  return blob;
}

void core_gen_free(Ctx& c) {
  if (!c.core_gen) return;
  for (cudaLibrary_t l : c.core_gen->libs) cudaLibraryUnload(l);
  delete c.core_gen;
  c.core_gen = nullptr;
}

// CUDA source of every pass of a plan (blocks as fiber lists); NT per pass
std::string core_gen_source(const Ctx& c, const std::vector<std::vector<uint32_t>>& blocks, std::vector<int>& nts,
                            int& ldr_out) {
  const int M = c.N - 1;
  const bool f32 = c.gather_f32 != 0;
  int soff[VEST_MAXN] = {}, o = 0;
  for (int k = 0; k < M; ++k) {
    if (f32 && (c.ld[k] / 2) % 2 == 0) o = (o + 1) & ~1;  // 16-byte aligned cp.async targets
    soff[k] = o;
    o += f32 ? c.ld[k] / 2 : c.ld[k];  // an fp32 row takes ld/2 double slots
  }
  const int rslot = o++;
  while (o % 4 != 2) ++o;
  const int ldr = o;
  // cache hints (VEST_CP_HINT=0/1, VEST_CP_CG=0/1: A/B): the coordinate and
  // residual streams are touched once per pass (ld/st.global.cs, evict-first);
  // the row gathers skip the L1 (cp.async.cg: config 4 passes 102.7 -> 99.9 ms)
  // unless a gathered mode is skewed -- a Zipf head row is read by every SM at
  // once and only the L1 keeps those reads off one L2 line (config 5 with .cg:
  // passes 129 -> 465 ms per iteration)
  static const bool hint = [] { const char* e = getenv("VEST_CP_HINT"); return e ? e[0] == '1' : true; }();
  static const int cg_env = [] { const char* e = getenv("VEST_CP_CG"); return e ? (e[0] == '1' ? 1 : 0) : -1; }();
  bool cg = cg_env != 0;
  for (int k = 0; k < M && cg_env < 0; ++k) cg = cg && !c.skewed[k];
  std::ostringstream src;
  {
    std::string pre = kPrelude;
    replace_all(pre, "@CPMOD@", cg ? "cg" : "ca");
    src << pre;
  }
  const int nb = (int)blocks.size();
  for (int i = 0; i <= nb; ++i) {
    const std::vector<uint32_t> none;
    const auto& prev = i > 0 ? blocks[i - 1] : none;
    const auto& cur = i < nb ? blocks[i] : none;
    const int nf = (int)cur.size(), pnf = (int)prev.size();
    const int NT = i == nb ? 2 : (nf <= 15 ? 2 : (nf <= 23 ? 3 : 4));
    nts.push_back(NT);
    std::vector<bool> used(VEST_MAXN * 16, false);
    std::ostringstream pv, cv;
    std::vector<std::string> pblk, cblk;
    const bool pf32 = cp_f32(c);
    const bool pipe = cp_pipe(c) && i < nb;  // the final (r^2 only) pass has no Gram to overlap
    const char* PT = pf32 ? "float" : "double";
    products(c, prev, pv, [pf32](int b, const std::string& e) {  // e = "w, in" of prefix block b
      const std::string t = "t" + std::to_string(b & 3);
      return t + (pf32 ? " = fmaf(" : " = fma(") + e + ", " + t + ");";
    }, used, PT, &pblk, [](int f) { return "sq_q[warp][" + std::to_string(f) + "]"; }, pf32 ? "fmaf" : "fma");
    const bool xt = pf32 && !pipe && cp_xt(c);
    if (xt) {
      cv << "      float p0 = 0.f";
      for (int f = 1; f < 32; ++f) cv << ", p" << f << " = 0.f";
      cv << ";\n";
    }
    products(c, cur, cv, [pf32, xt](int f, const std::string& e) {
      if (xt) return "p" + std::to_string(f) + " = " + e + ";";
      return "X[" + std::to_string(f * 36) + " + lane] = " + e + ";";
    }, used, PT, &cblk);
    if (xt)
      for (int g = 0; g < 8; ++g)
        cv << "      *reinterpret_cast<float4*>(X + lane * 40 + " << 4 * g << ") = make_float4(p" << g << ", p" << 8 + g
           << ", p" << 16 + g << ", p" << 24 + g << ");\n";
    std::ostringstream iss, lu;
    for (int k = 0; k < M; ++k) {
      if (f32) {  // fp32 row copies: ld floats, 16-byte pieces when ld % 4 == 0, else 8-byte
        iss << "      { const float* row = a.g[" << k << "] + (unsigned long long)idx[" << k << "] * " << c.ld[k] << ";\n";
        const bool v4 = c.ld[k] % 4 == 0;
        for (int t = 0; t < c.ld[k] / (v4 ? 4 : 2); ++t)
          iss << "        " << (v4 ? "cp16" : "cp8") << "(st + " << soff[k] * 8 + t * (v4 ? 16 : 8) << "u, row + "
              << t * (v4 ? 4 : 2) << ");\n";
        iss << "      }\n";
        for (int b = 0; b < c.ranks[k]; ++b)
          if (used[k * 16 + b])
            lu << "    const " << PT << " " << uname(k, b) << " = " << (pf32 ? "" : "(double)")
               << "reinterpret_cast<const float*>(st + " << soff[k] << ")[" << b << "];\n";
        continue;
      }
      iss << "      { const double* row = a.f[" << k << "] + (unsigned long long)idx[" << k << "] * " << c.ld[k] << ";\n";
      for (int t = 0; t < c.ld[k] / 2; ++t)
        iss << "        cp16(st + " << (soff[k] + 2 * t) * 8 << "u, row + " << 2 * t << ");\n";
      iss << "      }\n";
      for (int b = 0; b < c.ranks[k]; ++b)
        if (used[k * 16 + b]) lu << "    const double " << uname(k, b) << " = st[" << soff[k] + b << "];\n";
    }
    std::string p = pipe ? kPassPipe : kPass;
    if (pipe) {
      const std::string fin =
          "      if (PNF > 0 && valid) { r -= (double)((t0 + t1) + (t2 + t3)); @STR@; }\n"
          "      if (WSQ) sq = fma(r, r, sq);\n";
      replace_all(p, "@INTER@", interleave(pblk, cblk, fin));
      replace_all(p, "@FINAL@", fin);
    }
    replace_all(p, "@NAME@", "vest_cp_" + std::to_string(i));
    replace_all(p, "@M@", std::to_string(M));
    replace_all(p, "@LDR@", std::to_string(ldr));
    replace_all(p, "@NT@", std::to_string(NT));
    replace_all(p, "@NF@", std::to_string(nf));
    replace_all(p, "@PNF@", std::to_string(pnf));
    replace_all(p, "@KIND@", i == nb ? "2" : "0");
    replace_all(p, "@WSQ@", c.defer_last && i == nb - 1 ? "true" : "false");
    replace_all(p, "@JM@", std::to_string(c.ranks[M]));
    replace_all(p, "@LDM@", std::to_string(c.ld[M]));
    replace_all(p, "@RSLOT@", std::to_string(rslot));
    replace_all(p, "@MINB@", std::to_string(cp_min_blocks(pf32)));
    replace_all(p, "@STATS_T@", c.stats_f32 ? "float" : "double");
    replace_all(p, "@PT@", PT);
    {  // timing probes only (results invalid): 1 = no Gram, 2 = no products / residual update
      const char* e = getenv("VEST_CP_PROBE");
      const int probe = e ? atoi(e) : 0;
      if (probe != 0 && i == 0)
        fprintf(stderr, "vest: VEST_CP_PROBE=%d -- core passes skip work for timing; RESULTS ARE INVALID\n", probe);
      replace_all(p, "@PROBE@", std::to_string(probe));
    }
    replace_all(p, "@XT@", PT);
    replace_all(p, "@NBUF@", std::to_string(cp_depth(c)));
    replace_all(p, "@XD@", std::to_string(xt ? 640 : (pf32 ? NT * 8 * 18 : NT * 8 * 36)));
    replace_all(p, "@XN@", xt ? "32 * 40" : "NC * 36");
    replace_all(p, "@GRAM@", xt ? "gram_nt_t" : "gram_nt");
    replace_all(p, "@LDC@", hint ? "__ldcs" : "__ldg");
    replace_all(p, "@STR@", hint ? "__stcs(a.r + pos, r)" : "a.r[pos] = r");
    replace_all(p, "@ISSUE@", iss.str());
    replace_all(p, "@LOADU@", lu.str());
    replace_all(p, "@PREV@", pv.str());
    replace_all(p, "@CUR@", cv.str());
    src << kPassMark << p;
  }
  ldr_out = ldr;
  return src.str();
}

// Build (or reuse) the generated passes for a plan.
bool core_gen_prepare(Ctx& c, const std::vector<std::vector<uint32_t>>& blocks, uint64_t plan_key) {
  if (c.core_gen && c.core_gen->key == plan_key) return true;
  core_gen_free(c);
  std::vector<int> nts;
  int ldr = 0;
  const std::string src = core_gen_source(c, blocks, nts, ldr);  // also the passes' tile counts and row pitch
  std::vector<char> cubin;
  if (!take_cubin(c.pre_gen, plan_key, cubin)) cubin = core_gen_compile(src, "vest_core_gen.cu");
  const int nb = (int)blocks.size();
  auto* s = new CoreGenState;
  s->key = plan_key;
  s->ldr = ldr;
  s->nt = nts;
  s->xf32 = cp_f32(c);
  s->nbuf = cp_depth(c);
  s->pipe = cp_pipe(c);
  s->xt = s->xf32 && !s->pipe && cp_xt(c);
  {
    uint64_t hdr0 = 0;
    memcpy(&hdr0, cubin.data(), sizeof(uint64_t));
    const int nparts = (int)hdr0;
    std::vector<uint64_t> sz(nparts);
    memcpy(sz.data(), cubin.data() + sizeof(uint64_t), nparts * sizeof(uint64_t));
    size_t off = (size_t)(1 + nparts) * sizeof(uint64_t);
    s->libs.resize(nparts, nullptr);
    for (int q = 0; q < nparts; ++q) {
      check(cudaLibraryLoadData(&s->libs[q], cubin.data() + off, nullptr, nullptr, 0, nullptr, nullptr, 0),
            "core gen load");
      off += sz[q];
    }
    s->k.resize(nb + 1);
    for (int i = 0; i <= nb; ++i) {  // pass i was compiled into program i % nparts
      const std::string nm = "vest_cp_" + std::to_string(i);
      check(cudaLibraryGetKernel(&s->k[i], s->libs[i % nparts], nm.c_str()), "core gen kernel");
    }
  }
  c.core_gen = s;
  return true;
}

// pass i of the prepared plan (i < nb: statistics of block i after applying
// block i-1; i == nb: apply the last block, per-chunk sums of r^2)
void core_gen_pass(Ctx& c, int i, const double* prev_dg, double* stats, int stride, double* chunk_sq) {
  CoreGenState& s = *c.core_gen;
  const int m = c.N - 1;
  const DevCSF csf = c.csf_view(m);
  if (csf.nchunks == 0) return;
  CoreGenArgs a{};
  if (c.gather_f32 && i == 0) refresh_factor_shadows(c, m);  // the factors are fixed during the sweep
  for (int k = 0; k < c.N; ++k) {
    a.oc[k] = csf.oc[k];
    a.f[k] = c.d_factor[k];
    a.g[k] = c.d_factor32[k];
  }
  a.r = c.d_r;
  a.prev_dg = prev_dg;
  a.stats = stats;
  a.chunk_sq = chunk_sq;
  a.chunks = csf.chunks;
  a.nchunks = csf.nchunks;
  a.stride = stride;
  const int NT = s.nt[i];
  const bool pipe = s.pipe && i + 1 < (int)s.k.size();
  const int xd = s.xt ? 640 : NT * 8 * (s.xf32 ? 18 : 36);
  const size_t sm = (unsigned long long)4 * (pipe ? 32 * s.ldr + 2 * xd + 64 : s.nbuf * 32 * s.ldr + xd + 32) * sizeof(double);
  const void* fn = reinterpret_cast<const void*>(s.k[i]);
  check(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm), "core gen smem");
  int per_sm = 0, sms = 0;
  check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 128, sm), "core gen occupancy");
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c.device);
  const uint32_t need = (csf.nchunks + 3) / 4;
  const unsigned grid = std::max(1u, std::min<uint32_t>(need, (uint32_t)std::max(1, per_sm) * sms));
  void* args[] = {&a};
  check(cudaLaunchKernel(fn, dim3(grid), dim3(128), args, sm, c.stream), "core gen launch");
  count_launch();
}

}  // namespace vest
