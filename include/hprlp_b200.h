/*
 * hprlp_b200.h — C-ABI of the B200-native HPR-LP engine (libhprlp_b200.so).
 *
 * The engine replaces the CPU body of the reference's LP-solve entry point
 *   scuckit.hprlp.solve(lp, config, start) -> SolveResult
 *   (reference: pkg/src/scuckit/hprlp.py:319-329, _solve_once :332-455)
 * behind the same Python signature (paper_2510_10891_b200/hprlp.py).  The
 * reference has no native FFI of its own (it is pure Python); these entry
 * points are the ctypes boundary that Python mirror binds, one per reference
 * function on the hot path:
 *
 *   hpr_create        SparseMatrix.__init__ + StandardFormLp       (lp_kernel.py:52-62, 178-213)
 *   hpr_solve         hprlp._solve_once                            (hprlp.py:332-455)
 *   hpr_get_log       SolveResult.residual_log / rate_log          (hprlp.py:412-420)
 *   hpr_matvec        SparseMatrix.matvec / matvec_t               (lp_kernel.py:78-88)
 *   hpr_kkt_residual  hprlp.kkt_residual + _dual_objective         (hprlp.py:98-139)
 *   hpr_power_method  lp_kernel.power_method                       (lp_kernel.py:138-175)
 *   hpr_iterate       hprlp.hpr_iterate                            (hprlp.py:184-207)
 *
 * Conventions: plain pointers and sizes only.  Array arguments may be host
 * pointers or CUDA device pointers (UVA; copies use cudaMemcpyDefault).
 * Every function returns 0 on success or a negative HPR_ERR_* code; the
 * message is available from hpr_last_error() (thread-local).  Solver
 * outcomes (optimal / limits / numerical failure) are reported in
 * hpr_stats.status, never as an error.  No C++ exception crosses the ABI.
 * A handle owns one CUDA stream and is not thread-safe; distinct handles
 * are independent (SPEC.md:257 allows concurrent solves on distinct LPs).
 */
#ifndef HPRLP_B200_H
#define HPRLP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HPR_ABI_VERSION 1

/* status codes: hprlp.SolveStatus (hprlp.py:27-31) */
#define HPR_OPTIMAL 0
#define HPR_ITERATION_LIMIT 1
#define HPR_TIME_LIMIT 2
#define HPR_NUMERICAL_FAILURE 3

/* error codes */
#define HPR_OK 0
#define HPR_ERR_INVALID -1     /* bad argument / config: ValueError in the reference */
#define HPR_ERR_CUDA -2        /* CUDA runtime failure */
#define HPR_ERR_NOMEM -3       /* workspace too small / allocation failed */
#define HPR_ERR_EMPTY -4       /* power method on a matrix with nnz == 0 (lp_kernel.py:146-147) */
#define HPR_ERR_POWER_NULL -5  /* power method needs another random start vector */

#define HPR_FP64 0
#define HPR_FP32 1

/* The LP  min cost.x + offset  s.t.  A x (= rows [0,n_eq) | >= rest) rhs,
 * lower <= x <= upper  (lp_kernel.py:178-206).  CSR must be canonical
 * (sorted, no duplicates), int32 indices.  The transpose (CSC of A read as
 * CSR of A^T) is optional; it is built on the host when absent. */
typedef struct hpr_problem {
    int32_t m, n, n_eq;
    int64_t nnz;
    const int32_t* indptr;     /* m+1 */
    const int32_t* indices;    /* nnz */
    const double* data;        /* nnz */
    const int32_t* t_indptr;   /* n+1, or NULL */
    const int32_t* t_indices;  /* nnz, or NULL */
    const double* t_data;      /* nnz, or NULL */
    const double* rhs;         /* m, may hold +-inf */
    const double* cost;        /* n */
    const double* lower;       /* n, may hold -inf */
    const double* upper;       /* n, may hold +inf */
    double offset;
} hpr_problem;

#define HPR_FLAG_NO_REORDER 1  /* keep the caller's row/column order on the device */
#define HPR_FLAG_NO_FOLD 2     /* do not merge twin (x, -x) inequality rows */
#define HPR_FLAG_NO_RUNS 4     /* read every column index (no index-free long-row chunks) */
#define HPR_FLAG_NO_PANELS 8   /* keep the dense flow blocks in F^T (no A^T y panels from F) */

typedef struct hpr_options {
    int32_t device;            /* CUDA ordinal */
    void* stream;              /* cudaStream_t to run on, or NULL for a private stream */
    void* workspace;           /* device memory owned by the caller (e.g. a torch tensor), or NULL */
    size_t workspace_bytes;
    int32_t flags;             /* HPR_FLAG_* */
    /* Row-partitioned solve: the problem passed to
     * hpr_create is this rank's row block (all n columns); the ranks of
     * nccl_comm (an ncclComm_t from hpr_nccl_comm_init) exchange the A^T y
     * partials, the column norms and the row-side check sums.  world_size
     * <= 1 or nccl_comm == NULL is the single-GPU engine.  This is the
     * one-process-per-GPU form of SURVEY §8(b)'s hpr_create_multi(devices,
     * ndev, comm): each rank calls hpr_create for its own device and block. */
    void* nccl_comm;
    int32_t world_size;
    int32_t rank;
} hpr_options;

/* SolverConfig (hprlp.py:34-60), field for field. */
typedef struct hpr_params {
    double tolerance;
    int64_t max_iterations;
    double time_limit;         /* seconds; < 0 means none */
    double time_elapsed;       /* seconds the caller already spent (counts against time_limit) */
    int32_t precision;         /* HPR_FP64 / HPR_FP32 */
    int32_t has_sigma0;
    double sigma0;
    double restart_beta;
    int64_t restart_stall;
    double sigma_damping;
    int32_t ruiz;
    int32_t ruiz_iters;
    int32_t pock_chambolle;
    int32_t normalize_rhs_objective;
    int32_t check_every;
    double power_tol;
    double power_inflation;    /* < 0 means 1 + power_tol */
    int32_t power_max_iter;
    /* numpy default_rng(seed).standard_normal(m) draws, generated by the
     * caller so lambda matches the reference exactly (lp_kernel.py:150-152);
     * power_start_count vectors of m doubles, consumed in order. */
    const double* power_start;
    int32_t power_start_count;
    int32_t log_residuals;
    int32_t log_every_iteration;
} hpr_params;

typedef struct hpr_kkt {       /* KktResidual (hprlp.py:63-95) */
    double primal, box, dual;
    double rel_primal, rel_box, rel_dual;
    double primal_objective, dual_objective, gap, rel_gap;
} hpr_kkt;

typedef struct hpr_stats {
    int32_t status;            /* HPR_OPTIMAL ... */
    int32_t precision_used;
    int64_t iterations;
    int64_t restarts;
    double sigma_final;
    double lam;
    double objective;          /* cost.x_best + offset, FP64 on device */
    hpr_kkt kkt;               /* residual of the returned triple */
    int64_t n_log;             /* records available from hpr_get_log */
    int32_t power_iterations;
    int32_t power_converged;
    double setup_seconds;      /* scaling + power method + initial residual (device timed) */
    double loop_seconds;       /* device time of the iteration loop */
    int64_t gpu_launches;      /* kernels this call launched */
    int64_t checks;
} hpr_stats;

typedef struct hpr_log_record {  /* one residual_log / rate_log entry (hprlp.py:412-420) */
    int64_t iteration;
    int64_t epoch;
    int64_t k;                 /* in-epoch counter after the iteration (rate_log) */
    double rel_primal, rel_dual, rel_box, rel_gap, sigma;
    double primal, box, dual;  /* absolute norms (rate_log "combined") */
} hpr_log_record;

typedef struct hpr_handle hpr_handle;

int32_t hpr_abi_version(void);
const char* hpr_last_error(void);

/* Bytes of device workspace hpr_create needs for this problem. */
int hpr_workspace_bytes(const hpr_problem* p, size_t* bytes);

/* Upload the LP, build the tiled device layout of A and A^T. */
int hpr_create(const hpr_problem* p, const hpr_options* opt, hpr_handle** out);
void hpr_destroy(hpr_handle* h);

/* hprlp._solve_once: scaling, power method, device-resident HPR loop.
 * x0/y0/z0: warm start in master space (all three or NULL).
 * x/y/z: output triple in master space (host or device). */
int hpr_solve(hpr_handle* h, const hpr_params* prm, const double* x0, const double* y0,
              const double* z0, double* x, double* y, double* z, hpr_stats* stats);

/* Copy up to cap residual-log records of the last solve. */
int hpr_get_log(hpr_handle* h, hpr_log_record* out, int64_t cap, int64_t* n_out);

/* Master-matrix products: transpose=0 -> out[m] = A in[n]; 1 -> out[n] = A^T in[m]. */
int hpr_matvec(hpr_handle* h, int32_t transpose, const double* in, double* out);

/* kkt_residual(x, y, z, lp) on the master LP. */
int hpr_kkt_residual(hpr_handle* h, const double* x, const double* y, const double* z,
                     hpr_kkt* out);

/* power_method(A) of the master matrix: tol, max_iter, inflation (<0: 1+tol). */
int hpr_power_method(hpr_handle* h, double tol, int32_t max_iter, double inflation,
                     const double* start, int32_t start_count, double* lam,
                     int32_t* iterations, int32_t* converged);

/* One hpr_iterate step on the master (unscaled) LP in the given precision.
 * state = (x, y, z, anchor x/y/z); writes the new current triple and the bar
 * triple (bar_* may be NULL). */
int hpr_iterate(hpr_handle* h, int32_t precision, double sigma, double lam, int64_t k,
                const double* x, const double* y, const double* z, const double* ax,
                const double* ay, const double* az, double* x_out, double* y_out,
                double* z_out, double* bar_x, double* bar_y, double* bar_z);

/* NCCL plumbing for the row-partitioned mode: rank 0 creates the id, the
 * caller broadcasts its 128 bytes (e.g. over torch.distributed), every rank
 * joins.  The communicator outlives the handles that use it. */
int hpr_nccl_unique_id(uint8_t out[128]);
int hpr_nccl_comm_init(const uint8_t id[128], int32_t world_size, int32_t rank, int32_t device,
                       void** comm_out);
void hpr_nccl_comm_destroy(void* comm);

/* Device layout of an uploaded LP (engine introspection). */
typedef struct hpr_layout {
    int32_t m, n, n_eq;
    int32_t folded_rows;       /* rows of the twin-folded operand (== m when nothing folds) */
    int64_t nnz, folded_nnz;
    int32_t tiles_a, tiles_at, tiles_f, tiles_ft;
    int32_t reordered, folded;
    size_t workspace_bytes;
    int64_t panel_cols;        /* columns whose dense flow block is read from F (A^T y panels) */
    int64_t panel_nnz;         /* entries of F^T served by those panels (dropped from F^T) */
    int64_t f_nnz;             /* entries of F incl. explicit zeros padding flow rows */
    int64_t ft_nnz;            /* entries left in F^T */
    int64_t index_free_nnz_f;  /* entries of F streamed without their column index */
    int32_t fused;             /* 1: the row-wise updates run as the products' epilogues */
    int32_t row_panel_groups;  /* dense F row groups read as row panels by A x~ (x~ once per slab) */
} hpr_layout;
int hpr_get_layout(hpr_handle* h, hpr_layout* out);

/* Benchmark support (no reference counterpart).
 * hpr_resume: continue the last solve's device state for more_iterations
 * (whole check blocks), optionally with a new tolerance (<= 0 keeps it).
 * hpr_bench_kernel: average device time of one kernel of the iteration,
 * launched reps times outside the graph on the handle's stream:
 * which = 0: A x~ product; 1: A^T y product; 2: primal row-wise update
 * (projection + reflection + Halpern); 3: dual row-wise update; 4: one KKT
 * check block (mutates the solver state: call after the measurements);
 * 5: A^T y product with the primal update as epilogue; 6: A x~ product with the
 * dual update as epilogue (the fused iteration's two kernels).
 * which | HPR_BENCH_IN_ITERATION (0..3, 5, 6): each timed launch is followed by
 * the iteration's other kernels, untimed (5 <-> 6; 0..3: the other three), so
 * the caches hold what they hold inside the loop; the time is the sum of the
 * per-launch CUDA-event intervals, which also hold each launch's ramp (an
 * upper bound: C4 FP64 fused pair 70.4 + 75.2 us against 146.4 us per loop
 * iteration including the amortised check). */
#define HPR_BENCH_IN_ITERATION 0x100
int hpr_resume(hpr_handle* h, int64_t more_iterations, double tolerance, hpr_stats* stats);
int hpr_bench_kernel(hpr_handle* h, int32_t which, int32_t reps, double* seconds_per_launch);

#ifdef __cplusplus
}
#endif
#endif /* HPRLP_B200_H */
