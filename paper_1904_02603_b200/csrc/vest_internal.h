// SPDX-License-Identifier: Apache-2.0
// vest_internal.h -- host/device shared definitions for libvest_cuda.so.
//
// HBM layout:
//  * per mode n, a CSF copy of the observed entries sorted by (i_n, entry id)
//    -- the reference's ModeIndex order (sparse_tensor.hpp:107-137) -- stored
//    SoA: the other N-1 coordinates (uint32 each), the value (fp64) and the
//    original entry id (uint32); row offsets (uint64, I_n + 1);
//  * work list per mode: chunks of <= kChunk entries of one row ("light" rows
//    are one chunk and are solved in-kernel; "heavy" rows span several chunks
//    whose partial statistics are reduced by a second kernel);
//  * factors I_n x ld_n fp64 (ld_n = J_n rounded up to even -> 16-byte rows
//    for vector loads); masks I_n x J_n uint8; dense core fp64 + mask;
//  * the residual r in the CSF order of the last mode (the core sweep's
//    traversal order).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <future>
#include <string>
#include <vector>

#define VEST_MAXN 8
#define VEST_MAXJ 16

namespace vest {

constexpr uint32_t kLight = 0xFFFFFFFFu;
constexpr uint32_t kChunk = 2048;  // max entries per work item
constexpr uint32_t kTinyRow = 32;  // rows this short run lane-per-row (skewed modes' long tails)

struct Chunk {
  uint32_t row, beg, end, slot;  // [beg, end) in the mode's CSF; slot = heavy partial index or kLight
};
struct Heavy {
  uint32_t row, first_slot, nslots, pad;
};

struct DevModel {
  double* factor[VEST_MAXN];
  uint8_t* fmask[VEST_MAXN];
  int ld[VEST_MAXN];
  int J[VEST_MAXN];
  int stride[VEST_MAXN];  // row-major core strides
  uint64_t I[VEST_MAXN];
  double* core;
  uint8_t* core_mask;
  const uint32_t* cellbeta;  // packed multi-index per core cell, 4 bits per mode
  int N;
  int G;
};

struct DevCSF {
  const uint32_t* oc[VEST_MAXN];  // oc[k], k != mode
  const double* val;
  const uint32_t* eid;
  const uint64_t* offsets;
  const Chunk* chunks;
  const Heavy* heavy;
  uint32_t nchunks, nheavy, nslots;
  int mode;
};

enum RowKind { kStats = 0, kResp = 1, kResid = 2 };

struct RowPassArgs {
  DevModel m;
  DevCSF csf;
  int mode;
  int reg;
  double lambda;
  double* heavy_out;  // [nslots][stride_na]
  int stride_na;
  double re, re2, x2;   // responsibilities
  double* resp_out;     // I x J (unpadded)
  double* r_out;        // residual in CSF order
  double* chunk_out;    // per-chunk sum of squared residuals
  int fuse_resid;       // kStats on the last mode: write r = x - B(alpha) for light rows
};

struct ModeData {
  // Entry arrays (d_oc, d_val, d_eid) hold CSF positions [pos0, pos0 + local
  // nnz) -- a shard context keeps only its own rows -- and are stored as
  // base - pos0, so absolute CSF positions index them (allocation = ptr + pos0).
  uint64_t pos0 = 0;
  uint64_t* d_offsets = nullptr;
  uint32_t* d_oc[VEST_MAXN] = {};
  double* d_val = nullptr;
  uint32_t* d_eid = nullptr;
  Chunk* d_chunks = nullptr;
  Heavy* d_heavy = nullptr;
  uint32_t* d_empty = nullptr;  // rows with no entries
  Chunk* d_heavy_chunks = nullptr;  // the chunks of heavy rows (residual pass after their solve)
  uint32_t nchunks = 0, nheavy = 0, nslots = 0, nempty = 0, nheavy_chunks = 0;
  // rows with <= kTinyRow entries, sorted by length (lane-per-row statistics
  // kernel), and the chunk list without them (warp-per-chunk kernel)
  uint32_t* d_tiny = nullptr;
  Chunk* d_chunks_big = nullptr;
  uint32_t ntiny = 0, nchunks_big = 0;
  std::vector<uint64_t> h_offsets;
};

// vest_sort.cu: stable LSD radix sort of (uint32 key, uint32 value) pairs
size_t radix_sort_tmp_bytes(uint64_t n);
int radix_sort_pairs(const uint32_t* kin, uint32_t* kout, const uint32_t* vin, uint32_t* vout, uint64_t n, int end_bit,
                     void* tmp, cudaStream_t stream);

struct Ctx;
struct SparseState;  // vest_sparse.cu: NVRTC module of the mask-specialised delta contraction
struct CoreGenState;  // vest_core_gen.cu: NVRTC module of the plan-specialised core passes

// Kernel families instantiated for compile-time rank tuples.
struct ShapeOps {
  int N;
  int J[VEST_MAXN];
  cudaError_t (*rowpass)(const RowPassArgs& a, int kind, uint32_t nchunks, cudaStream_t s);
  cudaError_t (*coo_recon)(const DevModel& m, const uint32_t* coords, const double* values,
                           uint64_t n, double* out, double* partial, int nblocks, cudaStream_t s);
  cudaError_t (*rowtiny)(const RowPassArgs& a, const uint32_t* rows, uint32_t nrows, cudaStream_t s);
};

struct ProfEvent {
  cudaEvent_t a, b;
  int fam;
};

struct CommHooks {
  void* user = nullptr;
  int (*allreduce_sum)(void* user, double* p, uint64_t n, void* stream) = nullptr;
  int (*allgather_rows)(void* user, int mode, double* base, uint64_t ld, void* stream) = nullptr;
};

struct Ctx {
  int device = 0;
  void (*comm_free)(void*) = nullptr;  // owner of comm.user (native NCCL state)
  uint64_t row_lo[VEST_MAXN] = {}, row_hi[VEST_MAXN] = {};  // owned rows per mode
  uint64_t local_nnz[VEST_MAXN] = {};
  bool skewed[VEST_MAXN] = {};  // a row holds > 0.1 % of the entries (gathers of its row are hot)
  CommHooks comm;
  bool comm_capturable = false;  // the hooks only enqueue on the stream (native NCCL): graphs allowed
  bool prof_on = false;
  std::vector<ProfEvent> prof_events;
  double prof_ms[8] = {};
  uint64_t prof_n[8] = {};
  cudaStream_t stream = nullptr;
  cudaStream_t copy_stream = nullptr;  // host read-back overlapped with compute
  cudaEvent_t ev_copy[VEST_MAXN + 1] = {};
  int N = 0;
  uint64_t dims[VEST_MAXN] = {};
  int ranks[VEST_MAXN] = {};
  uint64_t nnz = 0;
  int G = 1;
  uint64_t core_ver = 1;  // bumped when d_core changes (sync_const_core)
  double x_norm = 0.0;  // frobenius norm over observed values

  ModeData modes[VEST_MAXN];

  double* d_factor[VEST_MAXN] = {};
  int ld[VEST_MAXN] = {};
  // fp32 copies of the factors, gathered by the generated (NVRTC) kernels when
  // gather_f32 is on (fp64 arithmetic on fp32-rounded factor operands; BASELINE
  // config 4 is the fp32 configuration).  Refreshed from d_factor before each
  // use (refresh_factor_shadows).
  float* d_factor32[VEST_MAXN] = {};
  int gather_f32 = 0;
  bool stats_f32 = false;  // the current general sweep's chunk statistics are fp32 (fp32 mode, sampled Gram)
  uint8_t* d_fmask[VEST_MAXN] = {};
  double* d_core = nullptr;
  uint8_t* d_core_mask = nullptr;
  uint32_t* d_cellbeta = nullptr;
  std::vector<uint8_t> h_core_mask;

  double* d_r = nullptr;  // CSF order of mode N-1
  bool r_valid = false;   // r, sum_sq and re match the current model
  bool r_fresh = false;   // r matches the current model (sum_sq not computed)
  int r_pending[2] = {-1, -1};  // r still lacks the last core group's update (prefixes; d_dg holds the dg)
  const void* r_pending_ops = nullptr;
  bool r_pending_general = false;  // the pending update is the general sweep's last block (r_pending[0] = its pass)
  int pending_stride = 0;          // ... whose passes used this statistics stride
  bool defer_last = false;         // the current general sweep defers its last residual pass
  double sum_sq = 0.0, re = 0.0;

  double* d_resp_core = nullptr;
  double* d_resp_f[VEST_MAXN] = {};
  bool table_valid = false;
  double table_re = 0.0;

  // scratch
  double* d_heavy_part = nullptr;  size_t heavy_part_cap = 0;
  double* d_xfer = nullptr;        size_t xfer_cap = 0;  // packed factor staging (ld != J)
  double* d_chunk_stats = nullptr; size_t chunk_stats_cap = 0;
  double* d_gemm_part = nullptr;   size_t gemm_part_cap = 0;
  double* d_gemm_out = nullptr;    size_t gemm_out_cap = 0;
  double* d_chunk_sum = nullptr;   size_t chunk_sum_cap = 0;
  double* d_small = nullptr;       // small reduction outputs (pinned-mapped readback)
  double* h_small = nullptr;
  uint32_t* d_fibers = nullptr;    size_t fibers_cap = 0;  // fiber prefix lin indices
  std::vector<uint32_t> h_fibers;  // what d_fibers holds
  double* d_dg = nullptr;          size_t dg_cap = 0;
  double* d_pack_u = nullptr;      size_t pack_u_cap = 0;   // structured core pass operands
  double* d_pack_w = nullptr;      size_t pack_w_cap = 0;
  unsigned* d_counter = nullptr;   // last-CTA arrival counter (block pass)
  unsigned long long* d_counts = nullptr;  // prune / sparsity counters
  void* d_sel = nullptr;           // radix-select state

  SparseState* sparse = nullptr;
  CoreGenState* core_gen = nullptr;
  int core_gen_mode = -1;          // plan-specialised core passes: -1 auto, 0 off, 1 on
  // sweeps run with the current core mask (auto mode compiles the mask's
  // kernels from the second one on: a mask pruned every iteration never pays
  // an NVRTC compile, a stable one pays it once)
  uint64_t mask_key = 0;
  int mask_sweeps = 0;
  // The mask's kernels are NVRTC-compiled on host threads from the FIRST sweep
  // with a new mask on (the sweep itself runs the precompiled kernels), so the
  // second sweep -- where they are switched in -- waits only for what is left of
  // the compile.  Which kernels run in which sweep is unchanged (deterministic).
  struct AsyncCubin {
    bool valid = false;
    uint64_t key = 0;
    std::shared_future<std::vector<char>> fut;
  };
  AsyncCubin pre_sparse, pre_gen;
  std::vector<std::shared_future<std::vector<char>>> pre_stale;  // superseded compiles still running
  // CUDA graph of one CD iteration (3-mode all-prefix path, single GPU):
  // captured once the iteration's host logic has repeated with the same key
  bool capturing = false;            // inside stream capture: no host syncs
  uint64_t alloc_epoch = 0;          // bumped by every device allocation (a graph's buffers must not move)
  cudaGraphExec_t graph_exec = nullptr;
  uint64_t graph_key = 0, graph_seen_key = 0;
  int graph_seen = 0;
  uint64_t graph_launches = 0;       // kernels per replay (launch accounting)
  int graph_pending[2] = {-1, -1};   // r_pending after the captured iteration
  bool graph_general = false;        // the captured sweep is the general one (sum of squares in h_small[0])
  bool graph_pending_general = false;  // ... and deferred its last residual pass
  const void* graph_pending_ops = nullptr;
  int sparse_delta = -1;           // mask-specialised delta: -1 auto, 0 off, 1 on
  int sparse_fused = -1;           // ... fused with the statistics (modes without the fused residual): -1 auto
  double* d_delta = nullptr;       size_t delta_cap = 0;    // delta[j][pos] of one mode (sparse path)
  uint32_t* d_hstab = nullptr;     size_t hstab_cap = 0;    // live-cell Gram entry tables (k_core_hsample)
  std::vector<uint32_t> h_hstab;   // what d_hstab holds (every block of the plan)
  std::vector<int64_t> hstab_off;  // per block: offset in d_hstab, -1 = dense block GEMM
  bool force_generic = false;
  int core_block = 0;  // fibers per block (0 = auto)
  const ShapeOps* ops = nullptr;
  uint64_t device_bytes = 0;

  DevModel model_view() const;
  DevCSF csf_view(int mode) const;
};

// ------------------------------------------------------------ host helpers --
struct CudaError {
  cudaError_t err;
  std::string where;
};
struct ArgError {
  std::string msg;
};
struct RtError {
  std::string msg;
};

void check(cudaError_t e, const char* where);
void* dalloc(Ctx& c, size_t bytes);
void ensure(Ctx& c, double** p, size_t* cap, size_t n_doubles);
uint64_t& launch_counter();
inline void count_launch(uint64_t n = 1) { launch_counter() += n; }

const ShapeOps* find_shape_ops(int N, const int* J);

// Launchers implemented in the .cu files.
cudaError_t launch_rowpass_generic(const RowPassArgs& a, int kind, uint32_t nchunks, cudaStream_t s);
cudaError_t launch_coo_recon_generic(const DevModel& m, const uint32_t* coords, const double* values,
                                     uint64_t n, double* out, double* partial, int nblocks, cudaStream_t s);
void refresh_factor_shadows(Ctx& c, int skip_mode);  // d_factor32[k] = fp32(d_factor[k]), k != skip_mode
void sync_const_core(Ctx& c);  // the core changed: the constant-bank copy is stale (ConstBankLease)
// Scope that may enqueue kernels reading the constant-bank core (ConstCore):
// serialises contexts of one device and reloads the bank when needed
// (vest_rowpass.cu).  whole_graph: around a graph launch (it loads the bank itself).
struct ConstBankLease {
  explicit ConstBankLease(Ctx& c, bool whole_graph = false);
  ~ConstBankLease();
  ConstBankLease(const ConstBankLease&) = delete;
  ConstBankLease& operator=(const ConstBankLease&) = delete;
  Ctx& c;
  bool graph = false;
  bool active = false;
};
void const_bank_forget(Ctx& c);  // after a stream capture
bool core_apply_pending(Ctx& c);       // vest_core_sall.cu: apply the deferred last core group to r
void sum_from_quadratic_form(Ctx& c);  // vest_core_sall.cu: sum r^2 after a 3-mode sweep (exact fallback)
constexpr double kQuadCancel = 1e-4;   // s'/s below this: recompute the sum from r
cudaError_t launch_heavy_stats(const RowPassArgs& a, cudaStream_t s);  // k_heavy after a chunk-statistics pass
bool sparse_fused_enabled(const Ctx& c);                               // vest_sparse.cu
void sparse_fused(Ctx& c, int mode, const RowPassArgs& a);             // fused delta + statistics + solves
cudaError_t launch_rowpass_delta(const RowPassArgs& a, int kind, uint32_t nchunks, const void* delta,
                                 uint64_t dstride, uint64_t p0, cudaStream_t s, bool f32);  // delta fp32 or fp64
bool sparse_delta_enabled(const Ctx& c);
bool sparse_delta_eligible(const Ctx& c);
using CompileFn = std::vector<char> (*)(const std::string&, const char*);
void prefetch_cubin(Ctx& c, Ctx::AsyncCubin& slot, uint64_t key, std::string src, const char* name,
                    CompileFn fn = nullptr);  // nullptr: nvrtc_compile
std::vector<char> core_gen_compile(const std::string& src, const char* name);  // the passes, in parallel programs
bool take_cubin(Ctx::AsyncCubin& slot, uint64_t key, std::vector<char>& out);
void core_gen_prefetch(Ctx& c);  // vest_core.cu: the general plan's passes for the current mask
void note_sweep(Ctx& c);  // a factor sweep starts (mode 0): count sweeps per core mask
void sparse_delta(Ctx& c, int mode, uint64_t p0, uint64_t n, double* out);
void sparse_free(Ctx& c);
std::vector<char> nvrtc_compile(const std::string& src, const char* name);
bool nvrtc_available();
void core_gen_free(Ctx& c);
bool core_gen_prepare(Ctx& c, const std::vector<std::vector<uint32_t>>& blocks, uint64_t plan_key);
void core_gen_pass(Ctx& c, int i, const double* prev_dg, double* stats, int stride, double* chunk_sq);
std::string core_gen_source(const Ctx& c, const std::vector<std::vector<uint32_t>>& blocks, std::vector<int>& nts,
                            int& ldr);
std::vector<std::vector<uint32_t>> core_gen_plan(const Ctx& c);
int sparse_compile_check(int N, const int* ranks, const uint8_t* core_mask, uint64_t* bytes, std::string* err);

void build_csf(Ctx& c, const uint32_t* h_coords, const double* h_values);
void update_factor_mode(Ctx& c, int mode, int reg, double lambda, bool fuse_resid);
void update_factor_rows(Ctx& c, int mode, const uint32_t* rows, uint32_t nrows, int reg, double lambda);
void compute_residual(Ctx& c);  // fresh r = x - B(alpha), sum_sq, re
void core_sweep(Ctx& c, int reg, double lambda);
bool core_sweep_capturable(const Ctx& c);  // the sweep has no host syncs inside (all-prefix or generated passes)
bool core_sweep_general(const Ctx& c);     // the sweep is the general (not the 3-mode all-prefix) one
bool defer_last_enabled();                 // vest_core.cu
void core_apply_pending_general(Ctx& c);   // vest_core.cu: the general sweep's deferred last pass
uint64_t core_mask_hash(const Ctx& c);
void responsibilities(Ctx& c);
void prune(Ctx& c, double pr, uint64_t* counts);
void sparsity(Ctx& c, double* zero_frac, double* masked_frac);
void normalize_columns(Ctx& c);
double reduce_chunk_sums(Ctx& c, const double* d_in, uint64_t n);
void sum_chunks_device(Ctx& c, const double* d_in, uint64_t n, double* out);  // vest_ops.cu
void comm_allreduce(Ctx& c, double* p, uint64_t n);
void ctx_set_nccl(Ctx& c, int rank, int world, const void* id, const uint64_t* bounds);  // vest_nccl.cpp
void nccl_unique_id(void* out);
void comm_allgather_rows(Ctx& c, int mode, double* base, uint64_t ld);

// RAII timing scope for one kernel family (no-op unless profiling is on).
enum ProfFamily {
  kProfFactor = 0,  // factor-row update, modes 0..N-2 (and the last mode when not fused)
  kProfCorePass,
  kProfCoreGemm,
  kProfCoreSolve,
  kProfResid,
  kProfResp,
  kProfPrune,
  kProfFactorFused  // last mode with the fused residual
};
struct ProfScope {
  Ctx& c;
  int fam;
  cudaEvent_t a = nullptr;
  ProfScope(Ctx& ctx, int f) : c(ctx), fam(f) {
    if (c.prof_on) {
      cudaEventCreate(&a);
      cudaEventRecord(a, c.stream);
    }
  }
  ~ProfScope() {
    if (!c.prof_on || !a) return;
    cudaEvent_t b;
    cudaEventCreate(&b);
    cudaEventRecord(b, c.stream);
    c.prof_events.push_back({a, b, fam});
  }
};

}  // namespace vest
