// hpr_common.cuh — shared device types and numpy-faithful scalar helpers.
//
// The HPR engine reproduces the reference's numpy arithmetic operation by
// operation (scuckit/hprlp.py:184-207 and :98-139), so the elementwise
// helpers below follow numpy's semantics exactly: np.maximum/np.minimum
// propagate NaN, Python-float scalars are cast to the work dtype before
// use (NEP 50 weak scalars), and this file is compiled with -fmad=false so
// no product is fused into a following add.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace hpr {

constexpr int TPB = 128;          // threads per CTA for every tiled kernel
constexpr int TILE_NNZ = 1024;    // nonzeros staged per stream tile (8 KB FP64 products; 8 per thread)
#ifndef HPR_TILE_ROWS
#define HPR_TILE_ROWS 256   // A/B (tools/gpu_r2s.sh): 6,385-6,436 -> 6,550-6,614 it/s at C4 vs 128
#endif
// rows per stream tile: the short structural rows (3.6 entries on average at C4)
// fill a 1,024-entry tile only if a tile may hold more rows than threads
constexpr int TILE_ROWS = HPR_TILE_ROWS;
static_assert(TILE_ROWS == TPB || TILE_ROWS == 2 * TPB, "stream tiles fill sptr in at most two passes");
constexpr int ITEMS = TILE_NNZ / TPB;
constexpr int CHUNK_NNZ = TILE_NNZ;  // nonzeros per CTA on a long (split) row
constexpr int MAX_B = 64;         // largest check_every the loop graph holds (longer: eager blocks)

// quantities accumulated by the two master-space check kernels
constexpr int KR = 4;   // rows: primal^2, rhs.y, dy^2, nonfinite(bar_y)
constexpr int KC = 7;   // cols: dual^2, box^2, cost.x, lo-terms, up-terms, dx^2, nonfinite(bar_x,bar_z)

// np.maximum / np.minimum (NaN-propagating, first operand wins ties)
template <typename T> __device__ __forceinline__ T np_max(T a, T b) { return (a >= b || a != a) ? a : b; }
template <typename T> __device__ __forceinline__ T np_min(T a, T b) { return (a <= b || a != a) ? a : b; }
template <typename T> __device__ __forceinline__ T np_clip(T x, T lo, T hi) { return np_min(np_max(x, lo), hi); }
__device__ __forceinline__ bool finite(double v) { return isfinite(v); }
__device__ __forceinline__ bool finite(float v) { return isfinite(v); }

// streaming (evict-first) loads for the matrix stream; the gathered vectors
// stay in L2 (126 MB) while A and A^T stream from HBM.
template <typename T> __device__ __forceinline__ T ld_stream(const T* p) { return __ldcs(p); }
// The matrix streams also carry a 256-byte L2 fetch-size hint, so each DRAM
// request brings the next warp's neighbouring sectors along: F^T 60.7 -> 59.5 us,
// iteration 171.7 -> 171.2 us (A/B on one box, tools/ab_bench.sh).
__device__ __forceinline__ double ld_stream(const double* p) {
    double v;
    asm volatile("ld.global.cs.L2::256B.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ float ld_stream(const float* p) {
    float v;
    asm volatile("ld.global.cs.L2::256B.f32 %0, [%1];" : "=f"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ int ld_stream(const int* p) {
    int v;
    asm volatile("ld.global.cs.L2::256B.s32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}
template <typename T> __device__ __forceinline__ T ld_ro(const T* p) { return __ldg(p); }
// gathers of the (L2-resident) vectors ask L1 to keep their lines over the
// evict-first matrix stream (171.3 -> 171.0 us per iteration, A/B)
__device__ __forceinline__ double ld_ro(const double* p) {
    double v;
    asm volatile("ld.global.nc.L1::evict_last.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ float ld_ro(const float* p) {
    float v;
    asm volatile("ld.global.nc.L1::evict_last.f32 %0, [%1];" : "=f"(v) : "l"(p));
    return v;
}

// Solver control block, resident in device memory for the whole solve.  The
// iteration kernels read sigma/lam/k0 from it; the controller kernel owns it.
struct Ctrl {
    // HPR state scalars (HprState, hprlp.py:142-181)
    double sigma, lam, norm_a;
    long long k0;                 // in-epoch counter at the start of the current block
    long long total;              // total iterations at the start of the current block
    long long epoch, restarts, last_improvement;
    double last_restart_res, epoch_min;
    // KKT of the best and the latest check: primal, box, dual, rel_p, rel_b, rel_d, pobj, dobj, gap, rel_gap
    double best[10];
    double cur[10];
    // configuration
    double tol, beta, damping, denom, offset, b_scale, c_scale;
    long long max_iter, stall, B;
    unsigned long long deadline_ns;
    int has_deadline;
    int status;                   // -1 running, else HPR_* status
    int flag_improved, flag_restart;
    // sigma update at a restart (hprlp.py:437-441): the device forms the
    // ratio, the host applies ratio ** damping with the C library's pow --
    // the function Python's float ** calls -- and relaunches the loop
    int sigma_pending;
    double sigma_ratio;
    // queued blocks (partitioned loop): once a check stops the loop or needs
    // the host's sigma update, `halt` turns every later loop kernel into a
    // no-op until the host clears it; `skipped` marks a check that did not run
    int halt, skipped;
    long long checks;
    // logging
    long long n_log, log_cap;
    int log_on;
    unsigned long long cond;      // cudaGraphConditionalHandle (0 when not in a graph)
    // power method / setup scratch
    double scratch[8];
};

struct LogRec {
    long long iteration, epoch, k;
    double rel_primal, rel_dual, rel_box, rel_gap, sigma;
    double primal, box, dual;
};

// A CSR operand in device memory plus its tile schedule.
template <typename T>
struct Csr {
    int rows, cols;
    const int* indptr;
    const int* indices;
    const T* vals;
    const int4* tiles;       // {r0, -(r1+1), p0, p1} stream tile | {row, e0, e1, long_idx} chunk
    int ntiles;
    const int4* longs;       // {row, first_tile, nchunks, 0}
    int nlong;
    int* counters;           // per long row, zero between launches
    double* tile_part;       // per tile partial sums of long-row chunks (work dtype)
    const int2* taux;        // per tile {c0, 1} if the chunk's columns are c0, c0+1, ...; else {0, 0}
    // flow panels (F^T only; hpr_layout.cuh k_col_panels): row r's dense flow
    // part is sum_q pvals[rbase[i0+q] + r] * x[i0+q], {i0, L} = pinfo[r]
    const T* pvals;
    const int2* pinfo;
    const int* rbase;
    // per panel tile {i0, L, base, stride}: all its rows share the panel rows
    // i0 .. i0+L-1 and those F rows form one row-major block, so
    // F(i0+q, r) = pvals[base + q*stride + r] (stride 0: use pinfo / rbase)
    const int4* pdesc;
    // loop launches only: Ctrl::halt (the product is skipped while it is set)
    const int* halt;
    // row panels (F only): groups of <= RP_ROWS consecutive dense rows over
    // the same column run {r0, R, c0, len}; tile {-(g+1), column tile, 0, 0}
    // sums a RP_COLS-column slab of every row of group g with x~ read once;
    // the group's last tile (ticket gcount[g]) adds the slab partials
    // gpart[gslot[g] + r * ntiles_g + t] in slab order
    const int4* gdesc;
    const int* gslot;
    int* gcount;
    double* gpart;
};

constexpr int RP_ROWS = 32;       // rows per row-panel group
constexpr int RP_MIN_ROWS = 8;    // fewer dense rows sharing a run: chunk tiles instead
constexpr int RP_COLS = 128;      // columns per row-panel tile (4 per lane)
#ifndef HPR_RP_MIN_CTAS
#define HPR_RP_MIN_CTAS 16
#endif
constexpr int RP_MIN_CTAS = HPR_RP_MIN_CTAS;   // k_spmv_rows occupancy target

constexpr int PANEL_ROWS = TPB;   // rows (F^T columns) per panel tile: one per thread
constexpr int PANEL_MAX_KEEP = 32; // indexed entries a panel row may keep beside its panel

}  // namespace hpr
