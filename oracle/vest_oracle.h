/* SPDX-License-Identifier: Apache-2.0
 *
 * vest_oracle -- CPU restatement of the VeST sparse-Tucker CD hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This is the parity checker for the CUDA path in
 * paper_1904_02603_b200/.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it.  The product never links
 * or calls it.
 *
 * It restates, in plain C with the same loop and accumulation orders, the
 * reference functions in /root/reference/proj/include/sparsetuck/ (each
 * function below cites file:line).  Because every reduction runs in the same
 * order as the reference and the build disables FP contraction, the port is
 * bit-identical to the reference on the same inputs; tests/test_oracle.py pins
 * that against tests/golden/ fixtures produced by the reference itself
 * (oracle/_ref, built from the reference headers by oracle/Makefile).
 *
 * Session API: one opaque handle holds the tensor, its per-mode index, the
 * model, the last residuals and the last responsibility table, mirroring how
 * fit() (trainer.hpp:103-168) threads those objects through the hot path.
 */
#ifndef VEST_ORACLE_H
#define VEST_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct vo_session vo_session;

/* status codes: 0 ok, 1 invalid_argument, 2 runtime_error */
const char* vo_last_error(void);

/* make_tensor (sparse_tensor.hpp:100-105) + build_mode_index (:119-137). */
int vo_create(int order, const uint64_t* dims, uint64_t nnz, const uint32_t* coords,
              const double* values, const uint64_t* ranks, vo_session** out);
void vo_destroy(vo_session* s);

/* init_random (tucker_model.hpp:88-108): mt19937_64(seed), U[0,1) draws,
 * factor 0 row-major, ..., factor N-1, then the core; masks cleared. */
int vo_init_random(vo_session* s, uint64_t seed);

/* Model transfer.  factors[n] is dims[n] x ranks[n] row-major. */
int vo_set_model(vo_session* s, const double* core, const uint8_t* core_mask,
                 const double* const* factors, const uint8_t* const* factor_masks);
int vo_get_model(const vo_session* s, double* core, uint8_t* core_mask, double* const* factors,
                 uint8_t* const* factor_masks);

/* Per-mode index access (ModeIndex, sparse_tensor.hpp:109-117). */
int vo_get_index(const vo_session* s, int mode, uint64_t* offsets, uint32_t* ids);

/* compute_delta (updates.hpp:35-52) */
int vo_compute_delta(const vo_session* s, const uint32_t* at, int mode, double* out);
/* reconstruct_entry (tucker_model.hpp:112-131), one value per query */
int vo_reconstruct(const vo_session* s, const uint32_t* at, uint64_t nq, double* out);

/* reg: 0 = LF (ridge), 1 = L1 (lasso)  (updates.hpp:15) */
int vo_update_factor_row(vo_session* s, int reg, int mode, uint64_t row, double lambda);
int vo_update_all_factors(vo_session* s, int reg, double lambda, int threads);
/* one mode of update_all_factors (updates.hpp:162-173) */
int vo_update_factor_mode(vo_session* s, int reg, int mode, double lambda, int threads);
/* compute_row_stats (updates.hpp:64-79): RowUpdateScratch delta (J), gram (J*J), xdelta (J) */
int vo_row_stats(vo_session* s, int mode, uint64_t row, double* delta, double* gram, double* xdelta);
/* partial_reconstruct (tucker_model.hpp:136-154) at nq coordinates */
int vo_partial_reconstruct(const vo_session* s, const uint32_t* at, uint64_t nq, int mode, uint64_t j,
                           double* out);
int vo_update_core(vo_session* s, int reg, double lambda, int threads);

/* compute_residuals (tucker_model.hpp:168-183).  Stores r in the session
 * (entry order) for the responsibility calls; r_out may be NULL. */
int vo_compute_residuals(vo_session* s, int threads, double* r_out, double* sum_sq,
                         double* x_norm, double* re);

/* compute_responsibilities (pruning.hpp:181-191) from the stored residuals.
 * Outputs may be NULL; the table is kept in the session for vo_prune_step. */
int vo_compute_responsibilities(vo_session* s, int threads, double* core_out,
                                double* const* factor_outs);

/* prune_step (pruning.hpp:234-247).  When core_resp is NULL the stored table
 * is used.  counts[0] = core, counts[1 + n] = factor n. */
int vo_prune_step(vo_session* s, double pr, const double* core_resp,
                  const double* const* factor_resp, uint64_t* counts);

double vo_sparsity(const vo_session* s);         /* tucker_model.hpp:192-198 */
double vo_masked_fraction(const vo_session* s);  /* tucker_model.hpp:201-207 */
int vo_normalize_columns(vo_session* s);         /* tucker_model.hpp:212-236 */
double vo_frobenius_norm(const vo_session* s);   /* sparse_tensor.hpp:45-49 */

/* One CD iteration as fit() runs it (trainer.hpp:121-127): factors, core,
 * residuals.  Returns re through *re. */
int vo_cd_iteration(vo_session* s, int reg, double lambda, int threads, double* re);

#ifdef __cplusplus
}
#endif

#endif
