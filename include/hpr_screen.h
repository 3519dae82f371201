/* hpr_screen.h — C-ABI of the device flow screen.
 *
 * Replaces the body of the reference's post-MILP transmission screen
 *   scuckit.driver.screen_violations(point, instance, ptdf, monitored, tol)
 *   (pkg/src/scuckit/driver.py:165-200)
 * whose cost is one dense product per contingency key,
 *   flows = ptdf.table(key) @ injections        (driver.py:186, instance.py:166-173)
 * followed by the per-(line, period) test |flow| - limit > tol * limit
 * (driver.py:187-196, Line.limit_for instance.py:88-89).
 *
 * The PTDF tables (instance.PtdfTable, immutable, instance.py:141-173) are
 * uploaded once per table set and stay resident in HBM; each screen uploads
 * the (n_buses x n_periods) injection matrix, runs the FP64 product with the
 * threshold test fused into its reduction epilogue, and returns the violating
 * (table, line, period, flow, excess) records.  The Python mirror
 * (paper_2510_10891_b200/screen.py) rebuilds the injections exactly as the
 * reference does and sorts the records with the reference's key (driver.py:199).
 *
 * Conventions as in hprlp_b200.h: plain pointers and sizes, array arguments
 * may be host or device pointers, 0 or a negative HPR_ERR_* code, message in
 * hpr_last_error().  A handle owns one CUDA stream and is not thread-safe.
 */
#ifndef HPR_SCREEN_H
#define HPR_SCREEN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct hpr_screen hpr_screen;

typedef struct hpr_screen_info {
    int32_t n_lines, n_buses, n_tables;
    int32_t bus_pitch;          /* padded bus dimension of the resident tables */
    int32_t splits;             /* bus-range splits of the product (deterministic two-pass sum) */
    int32_t ctas_per_sm;        /* resident CTAs of the product kernel */
    size_t table_bytes;         /* HBM held by the tables */
} hpr_screen_info;

/* Upload n_tables row-major (n_lines x n_buses) FP64 tables (PtdfTable._tables
 * in PtdfTable.keys() order, instance.py:152-164) and the per-table line limits
 * limits[k * n_lines + l] = lines[l].limit_for(key_k) (instance.py:88-89). */
int hpr_screen_create(int32_t device, int32_t n_lines, int32_t n_buses, int32_t n_tables,
                      const double* const* tables, const double* limits, hpr_screen** out);

/* Screen one injection matrix (row-major n_buses x n_periods, driver.py:178-181):
 * flows of every table, then |flow| - limit > tol * limit (driver.py:190-191).
 * *n_found receives the number of violating (table, line, period) entries;
 * fetch them with hpr_screen_fetch.  Entries are unordered. */
int hpr_screen_run(hpr_screen* h, const double* injections, int32_t n_periods, double tol,
                   int64_t* n_found);

/* Copy the records of the last run (each array n_found long, any may be NULL). */
int hpr_screen_fetch(hpr_screen* h, int32_t* table, int32_t* line, int32_t* period,
                     double* flow, double* excess);

/* Copy the flows of one table from the last run: row-major (n_lines x n_periods),
 * PtdfTable.flows (instance.py:170-173). */
int hpr_screen_flows(hpr_screen* h, int32_t table, double* flows);

/* Re-run the last screen reps times on the resident injections (benchmark):
 * average device time of the product kernel and of the epilogue, in us. */
int hpr_screen_bench(hpr_screen* h, int32_t reps, double* us_product, double* us_epilogue);

int hpr_screen_info_get(hpr_screen* h, hpr_screen_info* info);

/* Measured FP64 tensor-pipe ceiling of the device (register-only DMMA chains,
 * CUDA events): the roofline peak the screen product is reported against. */
int hpr_fp64_peak_bench(int32_t device, double* tflops);

void hpr_screen_destroy(hpr_screen* h);

#ifdef __cplusplus
}
#endif

#endif /* HPR_SCREEN_H */
