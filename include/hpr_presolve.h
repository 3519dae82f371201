/* hpr_presolve.h — C-ABI of the native presolve core.
 *
 * Replaces the row-queue fixpoint of the reference presolve,
 * scuckit/presolve.py:_Reducer (pkg/src/scuckit/presolve.py:65-209):
 * activity-based bound tightening with integral rounding, redundant / empty
 * row removal and the infeasibility certificates, processed in the
 * reference's FIFO order so the reduced model is bit-identical (the fixing
 * decisions of successive fixing depend on it).  The numpy reductions of
 * _activity / _process_row (np.sum) are reproduced with numpy's pairwise
 * summation.  milp_presolve / lp_presolve (presolve.py:212-288) assemble the
 * reduced model (paper_2510_10891_b200/presolve.py) from this core's output,
 * with the reduced matrix cut by hpr_presolve_reduce.
 *
 * Host-only (no CUDA calls); exported by libhprlp_b200.so.
 */
#ifndef HPR_PRESOLVE_H
#define HPR_PRESOLVE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* outcome of hpr_presolve_run (presolve.py: _Reducer.infeasible certificates) */
#define HPR_PS_OK 0
#define HPR_PS_ROW_EMPTY 1      /* row i is empty with rhs v1            (presolve.py:133-134) */
#define HPR_PS_ROW_MAX 2        /* row i: max activity v1 < rhs v2       (presolve.py:142-144) */
#define HPR_PS_ROW_MIN 3        /* row i: min activity v1 > rhs v2       (presolve.py:146-148) */
#define HPR_PS_COL_EMPTY 4      /* column i has empty domain [v1, v2]    (presolve.py:116-118) */

#define HPR_PS_REMOVED_EMPTY 0      /* removed_rows reason "empty"     */
#define HPR_PS_REMOVED_REDUNDANT 1  /* removed_rows reason "redundant" */

typedef struct hpr_ps_problem {
    int32_t m, n, n_eq;
    const int64_t* indptr;      /* CSR of A (m + 1), float64 values, sorted columns */
    const int32_t* indices;
    const double* data;
    const int64_t* col_ptr;     /* CSC row lists (n + 1): rows of column j ascending, */
    const int32_t* col_rows;    /* or both NULL: built from the CSR pattern */
    const double* rhs;          /* m */
    const double* lower;        /* n (copied; the result holds the tightened bounds) */
    const double* upper;
    const uint8_t* integrality; /* n, or NULL (lp_presolve) */
} hpr_ps_problem;

typedef struct hpr_ps_info {
    int32_t status;             /* HPR_PS_* */
    int32_t index;              /* row or column of the certificate */
    double v1, v2;              /* certificate values */
    int64_t n_changes;          /* bound_changes entries */
    int64_t n_removed;          /* removed_rows entries */
    int64_t visits;             /* processed rows */
} hpr_ps_info;

typedef struct hpr_ps_result hpr_ps_result;

/* Run the fixpoint (presolve.py:195-209, budget max_passes * m visits). */
int hpr_presolve_run(const hpr_ps_problem* p, int32_t max_passes, hpr_ps_result** out);
int hpr_presolve_info(const hpr_ps_result* r, hpr_ps_info* info);
/* Copy the results out; any pointer may be NULL.  alive_row: m; lower/upper: n;
 * change_col: n_changes; change_bounds: 4 * n_changes (old_lo, old_up, new_lo,
 * new_up); removed_row / removed_reason: n_removed. */
int hpr_presolve_fetch(const hpr_ps_result* r, uint8_t* alive_row, double* lower, double* upper,
                       int32_t* change_col, double* change_bounds, int32_t* removed_row,
                       int8_t* removed_reason);
void hpr_presolve_free(hpr_ps_result* r);

/* The reduced matrix of milp_presolve / lp_presolve (presolve.py:238-245,
 * :275-279: A[kept_rows][:, kept_cols] with ascending index arrays): rows with
 * keep_row[i], columns with keep_col[j] (NULL keeps all) renumbered by rank,
 * entries in their original order -- the arrays scipy's fancy indexing
 * returns.  out_indices / out_data hold up to indptr[m] entries, out_indptr
 * (kept rows + 1).  Returns -2 when the result needs int64 indices. */
int hpr_presolve_reduce(int32_t m, int32_t n, const int64_t* indptr, const int32_t* indices,
                        const double* data, const uint8_t* keep_row, const uint8_t* keep_col,
                        int32_t* out_indptr, int32_t* out_indices, double* out_data,
                        int64_t* out_nnz);

#ifdef __cplusplus
}
#endif
#endif /* HPR_PRESOLVE_H */
