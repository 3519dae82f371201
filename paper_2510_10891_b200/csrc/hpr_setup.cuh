// hpr_setup.cuh — setup, control and bookkeeping kernels of the HPR engine:
// diagonal scaling (hprlp.py:213-264, lp_kernel.py:105-122), deterministic
// reductions, initial point (:357-365), the on-device controller
// (:393-446) and the restart / best-iterate copies (:172-181, :422-432).
#pragma once

#include <cuda_runtime.h>

#include "hpr_update.cuh"
#include "../../include/hprlp_b200.h"

using namespace hpr;

// ===========================================================================
// setup kernels (scaling: hprlp.py:213-264, lp_kernel.py:105-122)
// ===========================================================================

__global__ void k_fill(double* p, double v, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        p[i] = v;
}

// ||row||_inf of |A| (max is order-independent): one warp per row
__global__ void k_row_absmax(const int* ptr, const double* vals, int rows, double* out) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (warp >= rows) return;
    double m = 0.0;
    for (int e = ptr[warp] + lane; e < ptr[warp + 1]; e += 32) m = fmax(m, fabs(vals[e]));
    for (int off = 16; off > 0; off >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, off));
    if (lane == 0) out[warp] = m;
}

// numpy's pairwise summation (numpy/_core/src/umath/loops_utils.h.src),
// which scipy's abs(A).sum(axis) reaches through np.add.reduceat:
// segment sum = a[0] + pairwise(a[1:]).  Leaves of <= 128 elements use 8
// strided accumulators; larger ranges split at a multiple of 8 below n/2.
// The recursion is unrolled onto a small explicit stack (the default device
// stack is too small for deep recursion on ~20K-entry rows).
__device__ double np_pairwise_leaf(const double* a, int n) {
    if (n < 8) {
        double r = 0.0;
        for (int i = 0; i < n; ++i) r += fabs(a[i]);
        return r;
    }
    double r[8];
    for (int k = 0; k < 8; ++k) r[k] = fabs(a[k]);
    int i = 8;
    for (; i < n - (n % 8); i += 8)
        for (int k = 0; k < 8; ++k) r[k] += fabs(a[i + k]);
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res += fabs(a[i]);
    return res;
}

__device__ double np_pairwise_abs(const double* a, int n) {
    int off[32], len[32], state[32];
    double left[32];
    int sp = 0;
    off[0] = 0;
    len[0] = n;
    state[0] = 0;
    double ret = 0.0;
    while (sp >= 0) {
        if (len[sp] <= 128) {
            ret = np_pairwise_leaf(a + off[sp], len[sp]);
            --sp;
            continue;
        }
        int n2 = len[sp] / 2;
        n2 -= n2 % 8;
        if (state[sp] == 0) {
            state[sp] = 1;
            off[sp + 1] = off[sp];
            len[sp + 1] = n2;
            state[sp + 1] = 0;
            ++sp;
        } else if (state[sp] == 1) {
            left[sp] = ret;
            state[sp] = 2;
            off[sp + 1] = off[sp] + n2;
            len[sp + 1] = len[sp] - n2;
            state[sp + 1] = 0;
            ++sp;
        } else {
            ret = left[sp] + ret;
            --sp;
        }
    }
    return ret;
}

__global__ void k_row_abssum(const int* ptr, const double* vals, int rows, double* out) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= rows) return;
    const int b = ptr[r], n = ptr[r + 1] - b;
    out[r] = n == 0 ? 0.0 : fabs(vals[b]) + np_pairwise_abs(vals + b + 1, n - 1);
}

__device__ __forceinline__ void atomic_max_pos(unsigned long long* p, double v) {
    // v >= 0: IEEE ordering equals unsigned ordering of the bit pattern
    atomicMax(p, (unsigned long long)__double_as_longlong(v));
}

// f = 1/sqrt(where(norm > 0, norm, 1)); scale *= f; dev = max |1 - f|   (hprlp.py:222-231)
__global__ void k_scale_factor(const double* norm, double* f, double* scale, int n,
                               unsigned long long* dev) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    double d = 0.0;
    if (i < n) {
        const double v = norm[i];
        const double r = 1.0 / sqrt(v > 0 ? v : 1.0);
        f[i] = r;
        scale[i] = scale[i] * r;
        d = fabs(1.0 - r);
    }
    for (int off = 16; off > 0; off >>= 1) d = fmax(d, __shfl_xor_sync(0xffffffffu, d, off));
    if ((threadIdx.x & 31) == 0 && dev) atomic_max_pos(dev, d);
}

// D_r A D_c with the reference rounding (a * r_i) * c_j  (lp_kernel.py:118-122).
// For the transpose copy row factor and column factor swap roles, the
// product order stays (a * r_i) * c_j.  One warp per row.
__global__ void k_scale_csr(const int* ptr, const int* idx, double* vals, int rows,
                            const double* rowf, const double* colf, int transposed) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (warp >= rows) return;
    const double rf = rowf[warp];
    for (int e = ptr[warp] + lane; e < ptr[warp + 1]; e += 32) {
        const double cf = colf[idx[e]];
        vals[e] = transposed ? (vals[e] * cf) * rf : (vals[e] * rf) * cf;
    }
}

// rhs*R, cost*C, bounds/C where finite   (hprlp.py:243-246)
__global__ void k_work_cols(int n, const double* cost, const double* lo, const double* up,
                            const double* cs, double* cw, double* low, double* upw) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    const double c = cs[j];
    cw[j] = cost[j] * c;
    low[j] = isfinite(lo[j]) ? lo[j] / c : lo[j];
    upw[j] = isfinite(up[j]) ? up[j] / c : up[j];
}

__global__ void k_work_rows(int m, const double* rhs, const double* rs, double* rw) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < m) rw[i] = rhs[i] * rs[i];
}

// rhs/b, cost/c, bounds/b where finite   (hprlp.py:256-259)
__global__ void k_norm_cols(int n, double bsc, double csc, double* cw, double* low, double* upw) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    cw[j] = cw[j] / csc;
    if (isfinite(low[j])) low[j] = low[j] / bsc;
    if (isfinite(upw[j])) upw[j] = upw[j] / bsc;
}

__global__ void k_div(double* v, long long n, double s) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        v[i] = v[i] / s;
}

// deterministic two-pass sum of squares (optionally of finite entries only)
constexpr int RED_BLOCKS = 296;
__global__ void k_sumsq_part(const double* v, long long n, int finite_only, double* part) {
    double s = 0.0;
    for (long long i = blockIdx.x * (long long)TPB + threadIdx.x; i < n; i += (long long)gridDim.x * TPB) {
        const double x = v[i];
        if (!finite_only || isfinite(x)) s += x * x;
    }
    __shared__ double w[TPB / 32];
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) w[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int k = 0; k < TPB / 32; ++k) t += w[k];
        part[blockIdx.x] = t;
    }
}

__global__ void k_sum_slots(const double* part, int nslots, int nq, double* out) {
    // one CTA; out[q] = sum_s part[q*nslots + s] in a fixed order
    __shared__ double w[TPB / 32];
    for (int q = 0; q < nq; ++q) {
        double s = 0.0;
        for (int i = threadIdx.x; i < nslots; i += TPB) s += part[(size_t)q * nslots + i];
        s = warp_sum(s);
        if ((threadIdx.x & 31) == 0) w[threadIdx.x >> 5] = s;
        __syncthreads();
        if (threadIdx.x == 0) {
            double t = 0.0;
            for (int k = 0; k < TPB / 32; ++k) t += w[k];
            out[q] = t;
        }
        __syncthreads();
    }
}

__global__ void k_cast_f32(const double* in, float* out, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        out[i] = (float)in[i];
}

// initial point (hprlp.py:357-365): to_work, box projection with the FP64
// work bounds, cast to the work dtype; anchors and bars start equal; master
// copies for the initial residual (to_master, :272-276).
template <typename T>
__global__ void k_init_cols(int n, const double* x0, const double* z0, const double* cs,
                            double bsc, double csc, const double* low, const double* upw,
                            T* X, T* Z, T* AX, T* AZ, T* BX, T* BZ, double* XM, double* ZM) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    const double c = cs[j];
    double xw = 0.0, zw = 0.0;
    if (x0) {
        xw = x0[j] / (c * bsc);
        zw = z0[j] * c / csc;
    }
    xw = np_clip(xw, low[j], upw[j]);
    const T x = (T)xw, z = (T)zw;
    X[j] = AX[j] = BX[j] = x;
    Z[j] = AZ[j] = BZ[j] = z;
    XM[j] = ((double)x * c) * bsc;
    ZM[j] = ((double)z * csc) / c;
}

template <typename T>
__global__ void k_init_rows(int m, const double* y0, const double* rs, double csc, T* Y, T* AY,
                            T* BY, double* YM) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    const double r = rs[i];
    const double yw = y0 ? y0[i] / (r * csc) : 0.0;
    const T y = (T)yw;
    Y[i] = AY[i] = BY[i] = y;
    YM[i] = ((double)y * r) * csc;
}

__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__global__ void k_set_deadline(Ctrl* c, unsigned long long remaining_ns) {
    c->deadline_ns = globaltimer() + remaining_ns;
}

// ===========================================================================
// controller (hprlp.py:403-446) — one CTA, no host round trip
// ===========================================================================

constexpr int CTRL_TPB = 512;

__global__ void __launch_bounds__(CTRL_TPB)
k_controller(Ctrl* c, const double* rowpart, int nr, const double* colpart, int nc, LogRec* log,
             int mode, const int* tflag) {
    if (mode == 1 && c->halt) {                // a queued block after the stop: no-op
        if (threadIdx.x == 0) c->skipped = 1;
        return;
    }
    __shared__ double sums[KR + KC];
    __shared__ double w[KR + KC][CTRL_TPB / 32];
    // all KR + KC slot arrays in one pass (loads of every array in flight
    // together); per array the same per-thread order and trees as one pass
    // per array, so the sums are unchanged
    double acc[KR + KC];
#pragma unroll
    for (int q = 0; q < KR + KC; ++q) acc[q] = 0.0;
    for (int i = threadIdx.x; i < max(nr, nc); i += CTRL_TPB) {
        if (i < nr) {
#pragma unroll
            for (int q = 0; q < KR; ++q) acc[q] += rowpart[(size_t)q * nr + i];
        }
        if (i < nc) {
#pragma unroll
            for (int q = 0; q < KC; ++q) acc[KR + q] += colpart[(size_t)q * nc + i];
        }
    }
#pragma unroll
    for (int q = 0; q < KR + KC; ++q) {
        const double s = warp_sum(acc[q]);
        if ((threadIdx.x & 31) == 0) w[q][threadIdx.x >> 5] = s;
    }
    __syncthreads();
    if (threadIdx.x < KR + KC) {
        double t = 0.0;
        for (int k = 0; k < CTRL_TPB / 32; ++k) t += w[threadIdx.x][k];
        sums[threadIdx.x] = t;
    }
    __syncthreads();
    if (threadIdx.x != 0) return;

    const double s_p = sums[0], s_ry = sums[1], s_dy = sums[2], nf_y = sums[3];
    const double s_d = sums[KR + 0], s_b = sums[KR + 1], s_cx = sums[KR + 2];
    const double s_lo = sums[KR + 3], s_up = sums[KR + 4], s_dx = sums[KR + 5], nf_x = sums[KR + 6];

    if (mode == 1) {
        c->skipped = 0;
        const long long tnow = c->total + c->B;
        c->total = tnow;
        c->flag_improved = 0;
        c->flag_restart = 0;
        if (nf_y + nf_x > 0.0) {               // hprlp.py:406-409
            c->status = HPR_NUMERICAL_FAILURE;
            c->halt = 1;
            if (c->cond) cudaGraphSetConditional(c->cond, 0);
            return;
        }
    }

    // KktResidual fields (hprlp.py:127-139)
    double r[10];
    r[0] = sqrt(s_p);
    r[1] = sqrt(s_b);
    r[2] = sqrt(s_d);
    r[3] = r[0] / c->denom;
    r[4] = r[1] / c->denom;
    r[5] = r[2] / c->denom;
    r[6] = s_cx + c->offset;
    r[7] = (s_ry + (s_lo + s_up)) + c->offset;
    r[8] = fabs(r[6] - r[7]);
    r[9] = r[8] / ((1.0 + fabs(r[6])) + fabs(r[7]));
    double mr = r[3];                          // builtin max(rel_p, rel_b, rel_d, rel_gap)
    if (r[4] > mr) mr = r[4];
    if (r[5] > mr) mr = r[5];
    if (r[9] > mr) mr = r[9];
    for (int k = 0; k < 10; ++k) c->cur[k] = r[k];

    auto best_max = [&]() {
        double b = c->best[3];
        if (c->best[4] > b) b = c->best[4];
        if (c->best[5] > b) b = c->best[5];
        if (c->best[9] > b) b = c->best[9];
        return b;
    };

    if (mode == 0) {                           // initial residual (hprlp.py:371-391)
        for (int k = 0; k < 10; ++k) c->best[k] = r[k];
        c->last_restart_res = mr;
        c->epoch_min = mr;
        c->last_improvement = 0;
        c->flag_improved = 1;
        c->flag_restart = 0;
        c->status = (mr <= c->tol) ? HPR_OPTIMAL : -1;
        return;
    }

    const long long tnow = c->total;
    c->checks += 1;
    if (c->log_on && c->n_log < c->log_cap) {  // hprlp.py:412-420
        LogRec& L = log[c->n_log++];
        L.iteration = tnow;
        L.epoch = c->epoch;
        L.k = c->k0 + c->B;
        L.rel_primal = r[3];
        L.rel_dual = r[5];
        L.rel_box = r[4];
        L.rel_gap = r[9];
        L.sigma = c->sigma;
        L.primal = r[0];
        L.box = r[1];
        L.dual = r[2];
    }
    int improved = 0;
    if (mr < best_max()) improved = 1;                         // :422-424
    if (mr < c->epoch_min * (1.0 - 1e-12)) {                  // :425-427
        c->epoch_min = mr;
        c->last_improvement = tnow;
    }
    int restart = 0;
    if (mr <= c->tol) {                                        // :429-432
        improved = 1;
        c->status = HPR_OPTIMAL;
    } else {
        const bool suff = mr <= c->beta * c->last_restart_res;  // :434-436
        const bool stalled = tnow - c->last_improvement >= c->stall;
        if (suff || stalled) {
            const double dx = sqrt(s_dx), dy = sqrt(s_dy);       // :437-441
            if (dx > 1e-14 && dy > 1e-14 && c->norm_a > 0) {
                // sigma *= clip(ratio ** damping, 1/4, 4) is applied by the host
                // (host_sigma_update): CUDA's pow is not the C library's, and
                // even pow(r, 0.5) != sqrt(r) for ~0.08% of r under glibc
                c->sigma_ratio = dx / (c->norm_a * dy * c->sigma);
                c->sigma_pending = 1;
            }
            restart = 1;                                       // :442-446
            c->k0 = 0;
            c->epoch += 1;
            c->restarts += 1;
            c->last_restart_res = mr;
            c->epoch_min = mr;
            c->last_improvement = tnow;
        } else {
            c->k0 += c->B;
        }
    }
    if (improved)
        for (int k = 0; k < 10; ++k) c->best[k] = r[k];
    c->flag_improved = improved;
    c->flag_restart = restart;
    if (c->status == -1) {                                     // :394-399
        if (tnow + c->B > c->max_iter) c->status = HPR_ITERATION_LIMIT;
        else if (tflag ? *tflag != 0 : (c->has_deadline && globaltimer() > c->deadline_ns))
            c->status = HPR_TIME_LIMIT;        // partitioned: the MAX-reduced flag of all ranks
    }
    c->halt = (c->status != -1 || c->sigma_pending) ? 1 : 0;
    if (c->cond) cudaGraphSetConditional(c->cond, c->halt ? 0u : 1u);
}

// partitioned loop: this rank's wall-clock verdict, MAX-reduced over the ranks
// before the controller reads it (so every rank stops at the same check)
__global__ void k_deadline_flag(const Ctrl* c, int* flag) {
    *flag = (!c->halt && c->has_deadline && globaltimer() > c->deadline_ns) ? 1 : 0;
}

// best-triple save and restart copies (hprlp.py:172-181, 422-424, 430)
template <typename T>
__global__ void k_restart_copy(const Ctrl* c, int n, int m, int nf, const double* XM,
                               const double* YM, const double* ZM, double* BXm, double* BYm,
                               double* BZm, T* X, T* Y, T* Z, T* AX, T* AY, T* AZ, const T* BX,
                               const T* BY, const T* BZ, T* YF, const T* BYF) {
    if (c->skipped) return;
    const int imp = c->flag_improved, rst = c->flag_restart;
    if (!imp && !rst) return;
    const int len = n > m ? n : m;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < len; i += gridDim.x * blockDim.x) {
        if (i < n) {
            if (imp) {
                BXm[i] = XM[i];
                BZm[i] = ZM[i];
            }
            if (rst) {
                const T bx = BX[i], bz = BZ[i];
                X[i] = AX[i] = bx;
                Z[i] = AZ[i] = bz;
            }
        }
        if (i < m) {
            if (imp) BYm[i] = YM[i];
            if (rst) {
                const T by = BY[i];
                Y[i] = AY[i] = by;
            }
        }
        if (rst && i < nf) YF[i] = BYF[i];
    }
}

// folded work values: dst[e] = src[map[e]] (scaled values of the kept twin)
__global__ void k_gather_vals(double* dst, const double* src, const int* map, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        dst[i] = map[i] >= 0 ? src[map[i]] : 0.0;   // < 0: explicit zero (padded flow row)
}

// caller order <-> engine order (locality permutation)
__global__ void k_gather(double* dst, const double* src, const int* perm, int len) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < len) dst[i] = src[perm[i]];
}

__global__ void k_scatter(double* dst, const double* src, const int* perm, int len) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < len) dst[perm[i]] = src[i];
}
