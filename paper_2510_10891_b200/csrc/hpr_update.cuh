// hpr_update.cuh — row-wise passes of the HPR iteration and of the KKT check.
//
// Each pass is one coalesced sweep that applies, per row / column, the whole
// chain of numpy operations the reference spreads over ~15 array
// temporaries (hprlp.py:190-203), in the reference's evaluation order.
//
// Twin folding.  SCUC flow rows come in (lo, hi) pairs whose coefficients are
// exact negatives (formulation.py:366-369; preserved by diagonal scaling
// because both rows have the same norms).  The engine stores each pair once
// ("folded" row f covering rows frow[f] .. frow[f+1]-1, at most two):
//   (A x)_i   = s_f  and  (A x)_{i+1} = -s_f                (exact negation)
//   (A^T y)_j gathers y_fold[f] = y_i - y_{i+1}             (one product per pair)
// so both iteration products read the flow block once instead of twice.
#pragma once

#include "hpr_spmv.cuh"

// EpiDual::apply2 also loads both rows' y / rhs / y-anchor before either row
// stores (-DHPR_PAIR_EPI_LOADS=0: only the frow entries are paired; A/B)
#ifndef HPR_PAIR_PRIMAL
#define HPR_PAIR_PRIMAL 1
#endif
#ifndef HPR_PAIR_EPI_LOADS
#define HPR_PAIR_EPI_LOADS 1
#endif

namespace hpr {

__device__ __forceinline__ double halpern_t(const Ctrl* c, int j) {
    return 1.0 / ((double)(c->k0 + j) + 2.0);
}

// ---------------------------------------------------------------------------
// primal half of hpr_iterate, one column j per thread (hprlp.py:190-192,
// 196, 198, 200-203):  g = x + sigma (A^T y - c);  bar_x = clip(g, l, u);
// bar_z = (bar_x - g) / sigma;  x~ = 2 bar_x - x;  x, z <- Halpern
// ---------------------------------------------------------------------------
template <typename T>
struct PrimalArgs {
    const Ctrl* ctrl;
    int j_in_block;
    int n;
    const T* aty;               // A^T y (product vector)
    T *X, *Z, *XT;
    const T *AX, *AZ, *C, *LO, *UP;
    T *BX, *BZ;                 // CHECK: bar iterates (work dtype)
    double *XM, *ZM;            // CHECK: master-space bars (to_master, hprlp.py:272-276)
    const double* CS;
    // Halpern update of the current z (hprlp.py:198, 203).  Nothing in a solve
    // reads it: bar_z depends on x and y only, the KKT check, the sigma update
    // and the restart test use the bars, and a restart overwrites z with
    // bar_z (:168-174).  The solve loop therefore skips it (3 of the 11 vectors
    // of this pass); hpr_iterate (the single-step API, whose caller sees z)
    // keeps it.
    bool upd_z;
    const int* halt = nullptr;  // queued block loop only (Ctrl::halt)
};

// z's Halpern update (hpr_iterate only) and the check iteration's bars
template <typename T, bool CHECK>
__device__ __forceinline__ void primal_tail(const PrimalArgs<T>& a, int j, T bx, T bz, T t,
                                            T omt) {
    if (a.upd_z) {
        const T zh = T(2) * bz - a.Z[j];
        a.Z[j] = t * a.AZ[j] + omt * zh;
    }
    if constexpr (CHECK) {
        const double bsc = a.ctrl->b_scale, csc = a.ctrl->c_scale;
        a.BX[j] = bx;
        a.BZ[j] = bz;
        const double cs = a.CS[j];
        a.XM[j] = ((double)bx * cs) * bsc;
        a.ZM[j] = ((double)bz * csc) / cs;
    }
}

template <typename T, bool CHECK>
__device__ __forceinline__ void primal_col(const PrimalArgs<T>& a, int j, T p) {
    const double td = halpern_t(a.ctrl, a.j_in_block);
    const T sig = (T)a.ctrl->sigma, t = (T)td, omt = (T)(1.0 - td);
    const T x = a.X[j], c = a.C[j], lo = a.LO[j], up = a.UP[j];
    const T ax = a.AX[j];
    const T g = x + sig * (p - c);
    const T bx = np_clip(g, lo, up);
    const T bz = (bx - g) / sig;
    const T xt = T(2) * bx - x;
    a.XT[j] = xt;
    a.X[j] = t * ax + omt * xt;
    primal_tail<T, CHECK>(a, j, bx, bz, t, omt);
}

// two columns of one thread (EpiPrimal::apply2): the first column is computed,
// the second one's operands are loaded, and only then does the first store --
// the second column's loads do not wait behind the first one's stores (the
// pointers may alias), and only the first column's two results stay live
template <typename T, bool CHECK>
__device__ __forceinline__ void primal_col2(const PrimalArgs<T>& a, int j0, T p0, bool v0,
                                            int j1, T p1, bool v1) {
    const double td = halpern_t(a.ctrl, a.j_in_block);
    const T sig = (T)a.ctrl->sigma, t = (T)td, omt = (T)(1.0 - td);
    T xt0 = T(0), bx0 = T(0), bz0 = T(0), ax0 = T(0);
    if (v0) {
        const T x = a.X[j0], c = a.C[j0], lo = a.LO[j0], up = a.UP[j0];
        ax0 = a.AX[j0];
        const T g = x + sig * (p0 - c);
        bx0 = np_clip(g, lo, up);
        bz0 = (bx0 - g) / sig;
        xt0 = T(2) * bx0 - x;
    }
    T x1 = T(0), c1 = T(0), lo1 = T(0), up1 = T(0), ax1 = T(0);
    if (v1) {
        x1 = a.X[j1];
        c1 = a.C[j1];
        lo1 = a.LO[j1];
        up1 = a.UP[j1];
        ax1 = a.AX[j1];
    }
    if (v0) {
        a.XT[j0] = xt0;
        a.X[j0] = t * ax0 + omt * xt0;
        primal_tail<T, CHECK>(a, j0, bx0, bz0, t, omt);
    }
    if (v1) {
        const T g = x1 + sig * (p1 - c1);
        const T bx = np_clip(g, lo1, up1);
        const T bz = (bx - g) / sig;
        const T xt = T(2) * bx - x1;
        a.XT[j1] = xt;
        a.X[j1] = t * ax1 + omt * xt;
        primal_tail<T, CHECK>(a, j1, bx, bz, t, omt);
    }
}

template <typename T, bool CHECK>
__global__ void __launch_bounds__(TPB) k_update_primal(PrimalArgs<T> a) {
    if (a.halt && *a.halt) return;
    const int j = blockIdx.x * TPB + threadIdx.x;
    if (j < a.n) primal_col<T, CHECK>(a, j, a.aty[j]);
}

// the primal update as the epilogue of the A^T y product (fused iteration;
// MIN_CTAS 16 keeps the product at 32 registers — the epilogue spills a few
// values, which costs less than the halved occupancy of 62 registers)
template <typename T, bool CHECK>
struct EpiPrimal {
    static constexpr int K = 0;
    static constexpr int MIN_CTAS = 16;
    static constexpr bool ROW_PANELS = false, COL_PANELS = true;  // F^T only
    // paired columns: FP64 +0.6% at C4; FP32 slower (A/B), so FP64 only
    static constexpr bool PAIR = HPR_PAIR_PRIMAL && sizeof(T) == 8;
    PrimalArgs<T> a;
    double* part;
    __device__ __forceinline__ void apply(int r, T s, Acc<0>&) { primal_col<T, CHECK>(a, r, s); }
    __device__ __forceinline__ void apply2(int r0, T s0, bool v0, int r1, T s1, bool v1,
                                           Acc<0>&) {
        primal_col2<T, CHECK>(a, r0, s0, v0, r1, s1, v1);
    }
};

// ---------------------------------------------------------------------------
// dual half of hpr_iterate, one row i per thread (hprlp.py:193-194, 197, 202):
// bar_y = Pi_D(y + (theta - A x~)/(lambda sigma));  y <- Halpern.  rmap[i] =
// 2 f + (i is the second row of twin pair f); (A x~)_i = +-P[f].  The thread
// of a pair's first row also forms y_fold[f] = y_i - y_{i+1} (it recomputes
// the partner's update from L1-resident operands instead of synchronising).
// ---------------------------------------------------------------------------
template <typename T>
struct DualArgs {
    const Ctrl* ctrl;
    int j_in_block;
    int m, n_eq;
    const int* rmap;            // m: 2 * folded row + second-of-pair flag
    const T* ax;                // folded A x~
    T* Y;
    const T *AY, *RHS;
    T* YF;                      // y folded (gathered by the next A^T y)
    T *BY, *BYF;                // CHECK
    double *YM, *YMF;           // CHECK: master bar y and its folded form
    const double* RS;
    const int* frow;            // nf + 1 folded-row starts (EpiDual)
    const int* halt = nullptr;  // queued block loop only (Ctrl::halt)
};

template <typename T>
struct DualRow {
    T yn, by;
};

template <typename T>
__device__ __forceinline__ DualRow<T> dual_row(T y, T rhs, T ay, T ax, bool ineq, T inv, T t,
                                               T omt) {
    const T v = y + inv * (rhs - ax);
    const T by = ineq ? np_max(v, T(0)) : v;
    const T yh = T(2) * by - y;
    return {t * ay + omt * yh, by};
}

template <typename T, bool CHECK>
__global__ void __launch_bounds__(TPB) k_update_dual(DualArgs<T> a) {
    if (a.halt && *a.halt) return;
    const int i = blockIdx.x * TPB + threadIdx.x;
    if (i >= a.m) return;
    const double td = halpern_t(a.ctrl, a.j_in_block);
    const T inv = (T)(1.0 / (a.ctrl->lam * a.ctrl->sigma)), t = (T)td, omt = (T)(1.0 - td);
    const int code = a.rmap[i];
    const int f = code >> 1;
    const bool second = code & 1;
    const T s = a.ax[f];
    const DualRow<T> r = dual_row(a.Y[i], a.RHS[i], a.AY[i], second ? -s : s, i >= a.n_eq, inv,
                                  t, omt);
    const bool first_of_pair = !second && i + 1 < a.m && a.rmap[i + 1] == code + 1;
    DualRow<T> r2{T(0), T(0)};
    if (first_of_pair)
        r2 = dual_row(a.Y[i + 1], a.RHS[i + 1], a.AY[i + 1], -s, i + 1 >= a.n_eq, inv, t, omt);
    a.Y[i] = r.yn;
    if (!second) a.YF[f] = first_of_pair ? r.yn - r2.yn : r.yn;
    if constexpr (CHECK) {
        const double csc = a.ctrl->c_scale;
        a.BY[i] = r.by;
        const double ym = ((double)r.by * a.RS[i]) * csc;
        a.YM[i] = ym;
        if (!second) {
            if (first_of_pair) {
                const double ym2 = ((double)r2.by * a.RS[i + 1]) * csc;
                a.BYF[f] = r.by - r2.by;
                a.YMF[f] = ym - ym2;
            } else {
                a.BYF[f] = r.by;
                a.YMF[f] = ym;
            }
        }
    }
}

// the dual update of folded row f (both rows of a twin pair) as the epilogue
// of the A x~ product; same operations as k_update_dual
template <typename T, bool CHECK>
struct EpiDual {
    static constexpr int K = 0;
    static constexpr int MIN_CTAS = 16;
    static constexpr bool ROW_PANELS = true, COL_PANELS = false;  // F only
    static constexpr bool PAIR = true;
    DualArgs<T> a;
    double* part;
    __device__ __forceinline__ void apply(int f, T s, Acc<0>&) {
        const int i = a.frow[f];
        finish<false>(f, s, i, a.frow[f + 1] - i == 2);
    }
    // two folded rows of one thread: both rows' frow entries in one round trip
    __device__ __forceinline__ void apply2(int f0, T s0, bool v0, int f1, T s1, bool v1,
                                           Acc<0>&) {
        int i0 = 0, e0 = 0, i1 = 0, e1 = 0;
        if (v0) { i0 = a.frow[f0]; e0 = a.frow[f0 + 1]; }
        if (v1) { i1 = a.frow[f1]; e1 = a.frow[f1 + 1]; }
        if constexpr (HPR_PAIR_EPI_LOADS && sizeof(T) == 8) {
            // FP64: the rows' own operands too, before either row stores
            // (A/B: FP64 +0.55%, FP32 -0.5%, so FP32 keeps the lazier form)
            T y0 = T(0), b0 = T(0), h0 = T(0), y1 = T(0), b1 = T(0), h1 = T(0);
            if (v0) { y0 = a.Y[i0]; b0 = a.RHS[i0]; h0 = a.AY[i0]; }
            if (v1) { y1 = a.Y[i1]; b1 = a.RHS[i1]; h1 = a.AY[i1]; }
            if (v0) finish<true>(f0, s0, i0, e0 - i0 == 2, y0, b0, h0);
            if (v1) finish<true>(f1, s1, i1, e1 - i1 == 2, y1, b1, h1);
        } else {
            if (v0) finish<false>(f0, s0, i0, e0 - i0 == 2);
            if (v1) finish<false>(f1, s1, i1, e1 - i1 == 2);
        }
    }
    // PRE: the row's y / rhs / anchor were loaded by the caller
    template <bool PRE>
    __device__ __forceinline__ void finish(int f, T s, int i, bool pair, T yi = T(0),
                                           T rhsi = T(0), T ayi = T(0)) {
        const double td = halpern_t(a.ctrl, a.j_in_block);
        const T inv = (T)(1.0 / (a.ctrl->lam * a.ctrl->sigma)), t = (T)td, omt = (T)(1.0 - td);
        DualRow<T> r;
        if constexpr (PRE) r = dual_row(yi, rhsi, ayi, s, i >= a.n_eq, inv, t, omt);
        else r = dual_row(a.Y[i], a.RHS[i], a.AY[i], s, i >= a.n_eq, inv, t, omt);
        DualRow<T> r2{T(0), T(0)};
        if (pair) {
            r2 = dual_row(a.Y[i + 1], a.RHS[i + 1], a.AY[i + 1], -s, i + 1 >= a.n_eq, inv, t, omt);
            a.Y[i + 1] = r2.yn;
        }
        a.Y[i] = r.yn;
        a.YF[f] = pair ? r.yn - r2.yn : r.yn;
        if constexpr (CHECK) {
            const double csc = a.ctrl->c_scale;
            a.BY[i] = r.by;
            const double ym = ((double)r.by * a.RS[i]) * csc;
            a.YM[i] = ym;
            if (pair) {
                a.BY[i + 1] = r2.by;
                const double ym2 = ((double)r2.by * a.RS[i + 1]) * csc;
                a.YM[i + 1] = ym2;
                a.BYF[f] = r.by - r2.by;
                a.YMF[f] = ym - ym2;
            } else {
                a.BYF[f] = r.by;
                a.YMF[f] = ym;
            }
        }
    }
};

// y_fold / bar_y_fold / y_m_fold from unfolded vectors (any pointer may be null)
template <typename T>
__global__ void k_fold_rows(int nf, const int* frow, const T* Y, T* YF, const T* BY, T* BYF,
                            const double* YM, double* YMF) {
    const int f = blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= nf) return;
    const int i0 = frow[f];
    const bool pair = frow[f + 1] - i0 == 2;
    if (YF) YF[f] = pair ? Y[i0] - Y[i0 + 1] : Y[i0];
    if (BYF) BYF[f] = pair ? BY[i0] - BY[i0 + 1] : BY[i0];
    if (YMF) YMF[f] = pair ? YM[i0] - YM[i0 + 1] : YM[i0];
}

// ---------------------------------------------------------------------------
// KKT check terms, master data (hprlp.py:116-139 with _dual_objective :98-113),
// plus ||bar - anchor|| for the sigma update (:437-438) and the finiteness test
// (:406-407).  Block partial sums (fixed order) -> part[k * gridDim.x + block].
// ---------------------------------------------------------------------------
template <typename T>
struct CheckRowsArgs {
    int nf, n_eq;
    const int* frow;
    const double* ax;           // folded A_m x_m
    const double *YM, *RHSM;
    const T *BY, *AY;
    double* part;
};

template <typename T>
__global__ void __launch_bounds__(TPB) k_check_rows(CheckRowsArgs<T> a) {
    Acc<KR> acc;
    acc.zero();
    for (int f = blockIdx.x * TPB + threadIdx.x; f < a.nf; f += gridDim.x * TPB) {
        const int i0 = a.frow[f], cnt = a.frow[f + 1] - i0;
        const double s = a.ax[f];
        for (int q = 0; q < cnt; ++q) {
            const int i = i0 + q;
            const double axi = q ? -s : s;
            const double ym = a.YM[i], rhs = a.RHSM[i];
            const double v = (ym - axi) + rhs;
            const double pr = i >= a.n_eq ? np_max(v, 0.0) : v;
            const double pv = ym - pr;
            acc.v[0] += pv * pv;
            acc.v[1] += rhs * ym;
            const T by = a.BY[i];
            const double d = (double)(by - a.AY[i]);
            acc.v[2] += d * d;
            acc.v[3] += finite(by) ? 0.0 : 1.0;
        }
    }
    block_store<KR>(acc, a.part, gridDim.x, blockIdx.x);
}

template <typename T>
struct CheckColsArgs {
    int n;
    const double* aty;          // A_m^T y_m
    const double *XM, *ZM, *COSTM, *LOM, *UPM;
    const T *BX, *BZ, *AX;
    double* part;
};

template <typename T>
__global__ void __launch_bounds__(TPB) k_check_cols(CheckColsArgs<T> a) {
    Acc<KC> acc;
    acc.zero();
    for (int j = blockIdx.x * TPB + threadIdx.x; j < a.n; j += gridDim.x * TPB) {
        const double xm = a.XM[j], zm = a.ZM[j], c = a.COSTM[j], lo = a.LOM[j], up = a.UPM[j];
        const double dv = (c - a.aty[j]) - zm;
        const double bv = xm - np_clip(xm - zm, lo, up);
        acc.v[0] += dv * dv;
        acc.v[1] += bv * bv;
        acc.v[2] += c * xm;
        acc.v[3] += isfinite(lo) ? lo * np_max(zm, 0.0) : 0.0;
        acc.v[4] += isfinite(up) ? up * np_min(zm, 0.0) : 0.0;
        const T bx = a.BX[j];
        const double d = (double)(bx - a.AX[j]);
        acc.v[5] += d * d;
        acc.v[6] += (finite(bx) ? 0.0 : 1.0) + (finite(a.BZ[j]) ? 0.0 : 1.0);
    }
    block_store<KC>(acc, a.part, gridDim.x, blockIdx.x);
}

}  // namespace hpr
