/* SPDX-License-Identifier: Apache-2.0
 *
 * vest.h -- C-ABI of libvest_cuda.so, the B200 (sm_100a) implementation of the
 * VeST sparse-Tucker coordinate-descent hot path.
 *
 * The reference (arXiv 1904.02603, /root/reference/proj) exposes this path as
 * a header-only C++ API in namespace sparsetuck:: operating on caller-owned
 * std::vector buffers.  This header is the flat, FFI-friendly boundary that
 * replaces it: plain pointers and sizes, int status codes, an opaque device
 * context that owns the device-resident tensor (CSF per mode) and model.
 * include/sparsetuck_b200.hpp re-exposes the reference's exact C++ signatures
 * on top of it; paper_1904_02603_b200/sparsetuck.py does the same for Python.
 *
 * Conventions
 *  - status: VEST_OK (0); VEST_EINVAL (1) maps to std::invalid_argument with
 *    the reference's message; VEST_ERUNTIME (2) maps to std::runtime_error;
 *    VEST_ECUDA (3) is a CUDA failure.  vest_last_error() returns the message
 *    of the last failing call on the calling thread.
 *  - every call is synchronous with respect to the host (the context stream is
 *    synchronised before return), matching the reference's blocking calls.
 *  - regularizer: 0 = LF (ridge), 1 = L1 (lasso)  (updates.hpp:15).
 *  - the reference's `threads` argument has no meaning here and is dropped.
 *  - coordinates are uint32 (Coord, sparse_tensor.hpp:22), values fp64
 *    (sparse_tensor.hpp:32), masks uint8 with 1 = pruned (tucker_model.hpp:26-28).
 */
#ifndef VEST_H
#define VEST_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VEST_OK 0
#define VEST_EINVAL 1
#define VEST_ERUNTIME 2
#define VEST_ECUDA 3

#define VEST_LF 0
#define VEST_L1 1

typedef struct vest_ctx vest_ctx;

/* Message of the last failing call on this thread ("" if none). */
const char* vest_last_error(void);
/* Library version string. */
const char* vest_version(void);
/* Number of kernels this process has launched through the library. */
uint64_t vest_launch_count(void);

/* ---------------------------------------------------------------- context --
 * Replaces make_tensor/check_tensor (sparse_tensor.hpp:68-105) and
 * build_mode_index (sparse_tensor.hpp:119-137): validates bounds and
 * duplicate-freeness with the reference's messages, uploads the COO entries
 * once and builds the per-mode CSF on `device`, plus a zero model with
 * `ranks`.  coords: nnz * order, entry-major. */
int vest_ctx_create(int order, const uint64_t* dims, uint64_t nnz, const uint32_t* coords,
                    const double* values, const uint64_t* ranks, int device, vest_ctx** out);
int vest_ctx_destroy(vest_ctx* ctx);
/* The context's cudaStream_t (as void*), for event timing by callers. */
void* vest_ctx_stream(vest_ctx* ctx);
/* Bytes of device memory the context holds. */
uint64_t vest_ctx_device_bytes(const vest_ctx* ctx);
/* Kernel path in use: 1 = rank-specialised (compile-time ranks), 0 = generic. */
int vest_ctx_specialised(const vest_ctx* ctx);
/* Force the generic path (for cross-checking the specialised kernels). */
int vest_ctx_force_generic(vest_ctx* ctx, int on);
/* Tuning: fibers per core-sweep block (0 = default). */
int vest_ctx_set_core_block(vest_ctx* ctx, int fibers);
/* Mask-specialised delta contraction for pruned cores (NVRTC-compiled for the
 * current core mask, recompiled after prunes; replaces the dense contraction
 * of the factor-row update, updates.hpp:35-52 skipping zero cells):
 * -1 auto (unmasked cells < |G| / 4 on rank-specialised shapes, from the
 * second sweep with the same core mask on), 0 off, 1 on.
 * vest_ctx_sparse_delta_active reports whether the current mask qualifies. */
int vest_ctx_set_sparse_delta(vest_ctx* ctx, int mode);
int vest_ctx_sparse_delta_active(const vest_ctx* ctx);
/* Plan-specialised core-sweep passes for the general block plans (straight-line
 * passes generated per core mask, NVRTC-compiled): -1 auto (rank-specialised
 * shapes, from the second sweep with the same core mask on), 0 off
 * (table-driven kernel), 1 on. */
int vest_ctx_set_core_gen(vest_ctx* ctx, int mode);
/* fp32 mode of the generated (NVRTC) kernels: on = their factor-row gathers
 * read fp32 copies of the factors, the mask-specialised delta and the core
 * passes' fiber products are contracted in fp32 arithmetic, and the delta
 * values and per-slice statistics they hand on are stored as fp32; every Gram,
 * solve and residual, the factors and the core stay fp64.  For fp32 workloads
 * (BASELINE config 4: north_star's 1e-4 fp32 tolerance, normwise); default off. */
int vest_ctx_set_gather_f32(vest_ctx* ctx, int on);
/* With the mask-specialised delta: fuse the contraction with the row
 * statistics and solves in one kernel (modes other than the one carrying the
 * fused residual; bit-identical).  -1 auto (= off: the one-entry-per-lane
 * fused kernel measured slower than the two-kernel path), 0 off, 1 on. */
int vest_ctx_set_sparse_fused(vest_ctx* ctx, int mode);
/* Host-only: generate and NVRTC-compile that contraction for ranks and a core
 * mask (no GPU needed); *cubin_bytes = size of the sm_100a cubin. */
int vest_sparse_compile_check(int order, const uint64_t* ranks, const uint8_t* core_mask, uint64_t* cubin_bytes);

/* ---------------------------------------------------------------- sharding --
 * Multi-GPU (one process per GPU): a shard context owns the rows
 * [row_lo[n], row_hi[n]) of every mode n (nnz-balanced ranges from
 * vest_partition_rows).  It holds the whole tensor and full model replicas but
 * only updates / traverses its own rows; the exchange points call the
 * communication hooks below, all on the context stream:
 *   - after each factor mode: allgather_rows(mode, factor, ld)  (all ranks end
 *     with every updated row);
 *   - per core block: allreduce_sum of the block statistics [T | C];
 *   - the residual sum of squares, and core-responsibility statistics:
 *     allreduce_sum;
 *   - factor responsibilities: allgather_rows(mode, table, J).
 * Every rank then runs the identical block solves and prune selection. */
typedef struct vest_comm {
  void* user;
  int (*allreduce_sum)(void* user, double* p, uint64_t n, void* stream);
  int (*allgather_rows)(void* user, int mode, double* base, uint64_t ld, void* stream);
} vest_comm;
int vest_ctx_create_shard(int order, const uint64_t* dims, uint64_t nnz, const uint32_t* coords,
                          const double* values, const uint64_t* ranks, int device,
                          const uint64_t* row_lo, const uint64_t* row_hi, vest_ctx** out);
/* Install (or clear with NULL) the communication hooks. */
int vest_ctx_set_comm(vest_ctx* ctx, const vest_comm* comm);
/* Native NCCL exchanges for a shard context (instead of host callbacks): every
 * rank passes the same 128-byte unique id (made once by vest_nccl_unique_id
 * and distributed by the caller), its rank/world, and the row bounds of every
 * mode, bounds[n * (world + 1) + r] (vest_partition_rows).  allreduce_sum and
 * allgather_rows then run as ncclAllReduce / grouped ncclBroadcast on the
 * context's stream.  NCCL is dlopen'ed (libnccl.so.2) on first use. */
#define VEST_NCCL_ID_BYTES 128
int vest_nccl_unique_id(void* id_out);
int vest_ctx_set_nccl(vest_ctx* ctx, int rank, int world, const void* id, const uint64_t* bounds);
/* Observed entries in this context's rows of `mode`. */
uint64_t vest_ctx_local_nnz(vest_ctx* ctx, int mode);

/* ------------------------------------------------------------------ model --
 * init_random (tucker_model.hpp:88-108): mt19937_64(seed), U[0,1) draws in
 * the documented order (factor 0 row-major, ..., factor N-1, then core). */
int vest_init_random(vest_ctx* ctx, uint64_t seed);
/* Host-only init_random into caller buffers (no device needed). */
int vest_init_random_host(int order, const uint64_t* dims, const uint64_t* ranks, uint64_t seed,
                          double* core, double* const* factors);
/* The device CSF of one mode as the reference's ModeIndex (offsets: dims[mode]+1,
 * ids: nnz entry ids, ascending within each slice). */
int vest_get_mode_index(vest_ctx* ctx, int mode, uint64_t* offsets, uint32_t* ids);
/* Host <-> device model transfer; factors[n] is dims[n] x ranks[n] row-major.
 * Any pointer may be NULL on get (skipped). */
int vest_set_model(vest_ctx* ctx, const double* core, const uint8_t* core_mask,
                   const double* const* factors, const uint8_t* const* factor_masks);
int vest_get_model(vest_ctx* ctx, double* core, uint8_t* core_mask, double* const* factors,
                   uint8_t* const* factor_masks);

/* -------------------------------------------------------------- hot path -- */
/* update_all_factors (updates.hpp:157-175): every mode in ascending order,
 * rows in parallel, columns of a row in sequential Gauss-Seidel order. */
int vest_update_all_factors(vest_ctx* ctx, int reg, double lambda);
/* One mode only (the unit a multi-GPU driver exchanges rows after). */
int vest_update_factor_mode(vest_ctx* ctx, int mode, int reg, double lambda);
/* update_factor_row_lf / update_factor_row_l1 (updates.hpp:88-151). */
int vest_update_factor_row(vest_ctx* ctx, int reg, int mode, uint64_t row, double lambda);
/* update_core_lf / update_core_l1 (updates.hpp:253-262): exact row-major
 * Gauss-Seidel over unmasked core cells (blocked by fibers). */
int vest_update_core(vest_ctx* ctx, int reg, double lambda);
/* compute_residuals (tucker_model.hpp:168-183).  r_out (nnz, entry order) may
 * be NULL.  Throws "zero-norm tensor" like the reference. */
int vest_compute_residuals(vest_ctx* ctx, double* r_out, double* sum_sq, double* x_norm,
                           double* re);
/* One CD iteration as fit() runs it (trainer.hpp:121-127):
 * update_all_factors + update_core + compute_residuals; returns re. */
int vest_cd_iteration(vest_ctx* ctx, int reg, double lambda, double* re);
/* The same iteration on a model held in HOST memory, updated in place (the
 * reference's calling convention: update_all_factors / update_core mutate the
 * caller's TuckerModel).  Uploads the model, runs the iteration, and streams
 * every factor back as soon as its mode is final (overlapping the rest of the
 * iteration), then the core.  Masks are inputs only (an iteration does not
 * change them).  Equivalent to set_model + cd_iteration + get_model. */
int vest_cd_iteration_host(vest_ctx* ctx, double* core, const uint8_t* core_mask, double* const* factors,
                           const uint8_t* const* factor_masks, int reg, double lambda, double* re);
/* compute_delta (updates.hpp:35-52) at one coordinate. */
int vest_compute_delta(vest_ctx* ctx, const uint32_t* at, int mode, double* out);
/* compute_row_stats (updates.hpp:64-79): gram (J*J, gram[t*J+j]) and xdelta
 * (J) of row `row` of `mode` over its observed entries in ascending entry id,
 * skipping delta_t == 0, with the reference's rounding (bit-identical).
 * last_delta (J, may be NULL) receives the delta of the slice's last entry --
 * what RowUpdateScratch::delta holds after the reference call (zeros for an
 * empty slice). */
int vest_compute_row_stats(vest_ctx* ctx, int mode, uint64_t row, double* gram, double* xdelta,
                           double* last_delta);
/* partial_reconstruct (tucker_model.hpp:136-154) at nq coordinates: the
 * reconstruction restricted to the core cells with beta_mode == j, reference
 * cell order and rounding (bit-identical). */
int vest_partial_reconstruct(vest_ctx* ctx, const uint32_t* coords, uint64_t nq, int mode, uint64_t j,
                             double* out);
/* Rows [row_lo, row_lo + nrows) of factor `mode` (row-major, J per row) to
 * host memory: the per-row drop-in calls read back only what they changed. */
int vest_get_factor_rows(vest_ctx* ctx, int mode, uint64_t row_lo, uint64_t nrows, double* out);
/* predict (trainer.hpp:172-185): reconstruction at nq coordinates. */
int vest_predict(vest_ctx* ctx, const uint32_t* coords, uint64_t nq, double* out);
/* evaluate_test (trainer.hpp:188-190): relative error on held-out entries. */
int vest_evaluate(vest_ctx* ctx, const uint32_t* coords, const double* values, uint64_t n,
                  double* re);

/* compute_responsibilities (pruning.hpp:181-191) from the residual of the
 * current model (the one compute_residuals returns).  base_re receives re.
 * Outputs may be NULL: the table then stays on the device for vest_prune_step. */
int vest_compute_responsibilities(vest_ctx* ctx, double* core_out, double* const* factor_outs,
                                  double* base_re);
/* prune_step (pruning.hpp:234-247): per block, mask+zero the
 * floor(pr * size) lowest-responsibility unmasked positions (ties by index),
 * found by a device radix select.  core_resp == NULL uses the device table
 * from vest_compute_responsibilities.  counts[0] = core, counts[1+n] = factor n. */
int vest_prune_step(vest_ctx* ctx, double pr, const double* core_resp,
                    const double* const* factor_resp, uint64_t* counts);
/* sparsity (tucker_model.hpp:192-198) and masked_fraction (:201-207). */
int vest_sparsity(vest_ctx* ctx, double* zero_fraction, double* masked_fraction);
/* normalize_columns (tucker_model.hpp:212-236). */
int vest_normalize_columns(vest_ctx* ctx);
/* SparseTensor::frobenius_norm (sparse_tensor.hpp:45-49). */
int vest_frobenius_norm(vest_ctx* ctx, double* out);

/* ------------------------------------------------------------ measurement --
 * Kernel-family timing with CUDA events on the context stream (bench.py's
 * per-kernel roofline).  Families: 0 factor-row update, 1 core pass,
 * 2 core gemm, 3 core solve, 4 residual, 5 responsibilities, 6 prune,
 * 7 last-mode factor update with the fused residual. */
#define VEST_PROF_FAMILIES 8
int vest_ctx_profile(vest_ctx* ctx, int on);
/* ms[f] = summed device time, launches[f] = timed scopes, since the last reset. */
int vest_ctx_profile_read(vest_ctx* ctx, double* ms, uint64_t* launches, int reset);
/* Measured FP64 FMA throughput of the device (TFLOP/s, 2 flops per DFMA). */
int vest_measure_fp64_peak(int device, double* tflops);

/* ------------------------------------------------------------ host utils --
 * Seeded synthetic inputs for the BASELINE configs:
 * distinct coordinates, entry order row-major.  dist: 0 uniform, 1 Zipf(s)
 * (per-mode exponent zipf_s[k], <= 0 means uniform for that mode).  values:
 * 0 = U[0,1) fp64, 1 = integers 1..5, 2 = N(0,1) rounded to float. */
int vest_synth(int order, const uint64_t* dims, uint64_t nnz, const double* zipf_s, int values_kind,
               uint64_t seed, uint32_t* coords_out, double* values_out);
/* split_train_test (sparse_tensor.hpp:232-260) entry ids: test ids then
 * train ids, each ascending. */
int vest_split_ids(uint64_t nnz, double test_fraction, uint64_t seed, uint64_t* test_ids,
                   uint64_t* n_test, uint64_t* train_ids, uint64_t* n_train);
/* Contiguous row ranges per rank, balanced by nnz (multi-GPU sharding plan):
 * bounds[0..world] with bounds[0] = 0, bounds[world] = rows. */
int vest_partition_rows(const uint64_t* row_offsets, uint64_t rows, int world, uint64_t* bounds);

/* --------------------------------------------------------- data formats --
 * The formats either side of the path (host side, OpenMP), byte-compatible
 * with the reference.  Errors: the reference's messages through
 * vest_io_last_error(); VEST_EINVAL for tensor/model validation
 * (std::invalid_argument), VEST_ERUNTIME for I/O and parse errors
 * (std::runtime_error). */
typedef struct vest_coo vest_coo;
typedef struct vest_model_file vest_model_file;
const char* vest_io_last_error(void);
/* load_coo (sparse_tensor.hpp:139-209): whitespace-separated COO text, "#"
 * comments, optional "# dims:" header, then make_tensor's validation (bounds,
 * duplicates).  threads <= 0: all host threads.  Read the result with
 * vest_coo_info (pointers stay valid until vest_coo_free). */
int vest_coo_load(const char* path, int one_based, int threads, vest_coo** out);
int vest_coo_info(const vest_coo* coo, int* order, uint64_t* nnz, uint64_t* dims, const uint32_t** coords,
                  const double** values);
void vest_coo_free(vest_coo* coo);
/* save_coo (sparse_tensor.hpp:211-228): byte-identical "# dims:" + "%.17g" text. */
int vest_coo_save(const char* path, int order, const uint64_t* dims, uint64_t nnz, const uint32_t* coords,
                  const double* values);
/* Binary cache of a tensor (magic "VESTCOO1", order, nnz, dims, coords, values):
 * a large input is parsed once. */
int vest_coo_cache_save(const char* path, int order, const uint64_t* dims, uint64_t nnz, const uint32_t* coords,
                        const double* values);
int vest_coo_cache_load(const char* path, vest_coo** out);
/* save_model / load_model (model_io.hpp:22-104): factor_<n>.tsv + core.coo,
 * byte-identical; a loaded model treats every zero as pruned. */
int vest_model_save(const char* dir, int order, const uint64_t* dims, const uint64_t* ranks, const double* core,
                    const double* const* factors);
int vest_model_load(const char* dir, vest_model_file** out);
int vest_model_file_info(const vest_model_file* mf, int* order, uint64_t* dims, uint64_t* ranks, const double** core,
                         const uint8_t** core_mask, const double** factors, const uint8_t** factor_masks);
void vest_model_file_free(vest_model_file* mf);

#ifdef __cplusplus
}
#endif

#endif /* VEST_H */
