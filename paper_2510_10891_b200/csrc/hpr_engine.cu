// hpr_engine.cu — B200 HPR-LP engine: setup kernels, on-device controller,
// CUDA-graph iteration loop, and the C-ABI declared in include/hprlp_b200.h.
//
// Reference path replaced: scuckit.hprlp._solve_once (hprlp.py:332-455) with
// its scaling (_ScaleMaps :210-276), power method (lp_kernel.py:138-175),
// iteration (hpr_iterate :184-207) and KKT checks (kkt_residual :116-139).
//
// Data layout in HBM (one workspace, 256-byte aligned sub-arrays):
//   A   : CSR  indptr[m+1] i32, indices[nnz] i32, master values f64,
//         work values f64 (scaled) and f32 (FP32 mode)
//   A^T : the same for the transpose (built once, host counting sort)
//   tile schedules of A and A^T (int4), long-row tickets and chunk partials
//   master vectors (rhs, cost, lower, upper) f64, scalings rs[m], cs[n]
//   work vectors in the work dtype: x, z, x~ (=2 bar_x - x), anchors, bars
//   master bar triple (x, y, z) f64 and the best master triple
//   check partial sums (slot-major, one slot per tile / long row), Ctrl, log
//
// Per HPR block of B = check_every iterations the graph body launches
//   B x { spmv<EpiPrimal>(A^T, y), spmv<EpiDual>(A, x~) }      fused iteration
//   spmv<EpiCheckRows>(A_master, x_m), spmv<EpiCheckCols>(A^T_master, y_m)
//   k_controller (convergence / best / restart / sigma; sets the WHILE flag)
//   k_restart_copy (best save + anchor reset, no-op unless flagged)
// inside a conditional WHILE graph node: the host launches one graph per
// solve and waits once.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "hpr_common.cuh"
#include "hpr_spmv.cuh"
#include "hpr_spmv_pipe.cuh"
#include "../../include/hprlp_b200.h"

using namespace hpr;

// ===========================================================================
// error plumbing
// ===========================================================================

static thread_local std::string g_err;

struct HprError {
    int code;
};

static void fail(int code, const std::string& msg) {
    g_err = msg;
    throw HprError{code};
}

#define CK(call)                                                                         \
    do {                                                                                 \
        cudaError_t e_ = (call);                                                         \
        if (e_ != cudaSuccess)                                                           \
            fail(HPR_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_));      \
    } while (0)

#define CKL() CK(cudaGetLastError())

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
             int mode) {
    __shared__ double sums[KR + KC];
    __shared__ double w[CTRL_TPB / 32];
    for (int q = 0; q < KR + KC; ++q) {
        const double* p = q < KR ? rowpart + (size_t)q * nr : colpart + (size_t)(q - KR) * nc;
        const int ns = q < KR ? nr : nc;
        double s = 0.0;
        for (int i = threadIdx.x; i < ns; i += CTRL_TPB) s += p[i];
        s = warp_sum(s);
        if ((threadIdx.x & 31) == 0) w[threadIdx.x >> 5] = s;
        __syncthreads();
        if (threadIdx.x == 0) {
            double t = 0.0;
            for (int k = 0; k < CTRL_TPB / 32; ++k) t += w[k];
            sums[q] = t;
        }
        __syncthreads();
    }
    if (threadIdx.x != 0) return;

    const double s_p = sums[0], s_ry = sums[1], s_dy = sums[2], nf_y = sums[3];
    const double s_d = sums[KR + 0], s_b = sums[KR + 1], s_cx = sums[KR + 2];
    const double s_lo = sums[KR + 3], s_up = sums[KR + 4], s_dx = sums[KR + 5], nf_x = sums[KR + 6];

    if (mode == 1) {
        const long long tnow = c->total + c->B;
        c->total = tnow;
        c->flag_improved = 0;
        c->flag_restart = 0;
        if (nf_y + nf_x > 0.0) {               // hprlp.py:406-409
            c->status = HPR_NUMERICAL_FAILURE;
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
                const double ratio = dx / (c->norm_a * dy * c->sigma);
                double f = c->damping == 0.5 ? sqrt(ratio) : pow(ratio, c->damping);
                f = np_min(np_max(f, 0.25), 4.0);
                c->sigma = c->sigma * f;
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
        else if (c->has_deadline && globaltimer() > c->deadline_ns) c->status = HPR_TIME_LIMIT;
    }
    if (c->cond) cudaGraphSetConditional(c->cond, c->status == -1 ? 1u : 0u);
}

// best-triple save and restart copies (hprlp.py:172-181, 422-424, 430)
template <typename T>
__global__ void k_restart_copy(const Ctrl* c, int n, int m, const double* XM, const double* YM,
                               const double* ZM, double* BXm, double* BYm, double* BZm, T* X,
                               T* Y, T* Z, T* AX, T* AY, T* AZ, const T* BX, const T* BY,
                               const T* BZ) {
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
    }
}

// ===========================================================================
// host side
// ===========================================================================

namespace {

struct Plan {
    std::vector<int4> tiles, longs;
};

// Cut a CSR into stream tiles and long-row chunks (see hpr_spmv.cuh).
Plan build_tiles(const int32_t* ptr, int rows) {
    Plan p;
    int r = 0;
    while (r < rows) {
        const int len = ptr[r + 1] - ptr[r];
        if (len > TILE_NNZ) {
            const int li = (int)p.longs.size();
            const int nch = (len + CHUNK_NNZ - 1) / CHUNK_NNZ;
            p.longs.push_back(make_int4(r, (int)p.tiles.size(), nch, 0));
            for (int c = 0; c < nch; ++c) {
                const int e0 = ptr[r] + c * CHUNK_NNZ;
                const int e1 = std::min(ptr[r + 1], e0 + CHUNK_NNZ);
                p.tiles.push_back(make_int4(r, e0, e1, li));
            }
            ++r;
            continue;
        }
        const int r0 = r;
        long long nz = 0;
        while (r < rows && r - r0 < TILE_ROWS) {
            const int l = ptr[r + 1] - ptr[r];
            if (l > TILE_NNZ || nz + l > TILE_NNZ) break;
            nz += l;
            ++r;
        }
        p.tiles.push_back(make_int4(r0, -(r + 1), ptr[r0], ptr[r]));
    }
    return p;
}

struct Carver {
    size_t off = 0;
    char* base = nullptr;
    template <typename T>
    T* take(size_t count) {
        off = (off + 255) & ~size_t(255);
        T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
        off += sizeof(T) * std::max<size_t>(count, 1) + 64;   // tail pad: 16-byte bulk-copy windows
        return p;
    }
};

}  // namespace

struct DevCsr {
    int rows = 0, cols = 0;
    int *ptr = nullptr, *idx = nullptr;
    double *mval = nullptr, *w64 = nullptr;
    float* w32 = nullptr;
    int4 *tiles = nullptr, *longs = nullptr;
    int ntiles = 0, nlong = 0;
    int nblocks = 0;             // persistent grid of the pipelined kernel
    bool pipe = true;
    int* counters = nullptr;
    double* tpart = nullptr;
    template <typename T>
    Csr<T> view(const T* vals) const {
        Csr<T> c;
        c.rows = rows;
        c.cols = cols;
        c.indptr = ptr;
        c.indices = idx;
        c.vals = vals;
        c.tiles = tiles;
        c.ntiles = ntiles;
        c.longs = longs;
        c.nlong = nlong;
        c.counters = counters;
        c.tile_part = tpart;
        return c;
    }
    int nslots() const { return (pipe ? nblocks : ntiles) + nlong; }
};

struct hpr_handle {
    int dev = 0;
    cudaStream_t stream = nullptr, cap = nullptr;
    bool own_stream = false;
    int m = 0, n = 0, n_eq = 0;
    long long nnz = 0;
    double offset = 0.0;
    DevCsr A, AT;
    // vectors
    double *rhs_m, *cost_m, *lo_m, *up_m, *rs, *cs, *fr, *fc;
    double *rhs_w, *cost_w, *lo_w, *up_w;   // FP64 work (setup)
    void *rhsT, *costT, *loT, *upT;          // work dtype copies (FP32 mode)
    void *X, *Y, *Z, *AXv, *AYv, *AZv, *XT, *BX, *BY, *BZ;
    double *XM, *YM, *ZM, *BXm, *BYm, *BZm;
    double *rowpart, *colpart, *red, *pw;   // pw: power-method vectors (m + n)
    Ctrl* ctrl = nullptr;
    Ctrl* h_ctrl = nullptr;                  // pinned mirror
    double* h_scal = nullptr;                // pinned scalars
    unsigned long long* d_dev = nullptr;     // Ruiz deviation accumulator
    LogRec* log = nullptr;
    long long log_cap = 0;
    void* ws = nullptr;
    bool own_ws = false;
    size_t ws_bytes = 0;
    long long launches = 0;
    std::vector<LogRec> h_log;
    cudaEvent_t ev[4];
    // cached loop graph (kernel arguments are fixed per handle, so one
    // instantiation serves every solve with the same block size and dtype)
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t gexec = nullptr;
    unsigned long long gcond = 0;
    int g_B = 0, g_prec = -1;
    long long g_per_block = 0;
    int last_prec = -1;          // precision of the last solve (-1: none)
    // locality ordering (new -> old); identity when reorder is off
    bool reordered = false;
    int *rperm = nullptr, *cperm = nullptr;
    double* stage = nullptr;     // max(m, n) staging for permuted I/O
    double* SP = nullptr;        // max(m, n) product vector of the split (unfused) iteration
    bool fuse = false;           // epilogue fused into the SpMV (HPR_FUSE=1) or separate pass
};

namespace {

constexpr long long LOG_CAP_MAX = 1 << 20;

struct Layout {
    size_t bytes;
};

// Upper bounds on the tile schedule of a CSR with `rows` rows and `nnz`
// nonzeros, independent of the row order (so the workspace can be sized
// before the locality ordering is computed).  A stream tile closes on a
// full row count, on nnz overflow (two consecutive tiles then hold more than
// TILE_NNZ), before a long row, or at the end.
struct TileBound {
    size_t tiles, longs;
};
TileBound tile_bound(long long rows, long long nnz) {
    const long long nlong = std::min<long long>(rows, nnz / (TILE_NNZ + 1));
    const long long t = 2 * (nnz / TILE_NNZ + 1) + rows / TILE_ROWS + 1 + 2 * nlong +
                        (nnz / CHUNK_NNZ + 1) + nlong + 2;
    return {(size_t)t, (size_t)std::max<long long>(nlong, 1)};
}

// Carve every device array from one block; base == nullptr only measures.
size_t carve(hpr_handle* h, char* base) {
    const TileBound ba = tile_bound(h->m, h->nnz), bt = tile_bound(h->n, h->nnz);
    struct {
        size_t tiles, longs;
    } pa_{ba.tiles, ba.longs}, pt_{bt.tiles, bt.longs};
    Carver cv;
    cv.base = base;
    const size_t m = h->m, n = h->n, nnz = h->nnz;
    h->A.ptr = cv.take<int>(m + 1);
    h->A.idx = cv.take<int>(nnz);
    h->A.mval = cv.take<double>(nnz);
    h->A.w64 = cv.take<double>(nnz);
    h->A.w32 = cv.take<float>(nnz);
    h->AT.ptr = cv.take<int>(n + 1);
    h->AT.idx = cv.take<int>(nnz);
    h->AT.mval = cv.take<double>(nnz);
    h->AT.w64 = cv.take<double>(nnz);
    h->AT.w32 = cv.take<float>(nnz);
    h->A.tiles = cv.take<int4>(pa_.tiles);
    h->A.longs = cv.take<int4>(pa_.longs);
    h->A.counters = cv.take<int>(pa_.longs);
    h->A.tpart = cv.take<double>(pa_.tiles);
    h->AT.tiles = cv.take<int4>(pt_.tiles);
    h->AT.longs = cv.take<int4>(pt_.longs);
    h->AT.counters = cv.take<int>(pt_.longs);
    h->AT.tpart = cv.take<double>(pt_.tiles);
    h->rhs_m = cv.take<double>(m);
    h->cost_m = cv.take<double>(n);
    h->lo_m = cv.take<double>(n);
    h->up_m = cv.take<double>(n);
    h->rs = cv.take<double>(m);
    h->cs = cv.take<double>(n);
    h->fr = cv.take<double>(m);
    h->fc = cv.take<double>(n);
    h->rhs_w = cv.take<double>(m);
    h->cost_w = cv.take<double>(n);
    h->lo_w = cv.take<double>(n);
    h->up_w = cv.take<double>(n);
    h->rhsT = cv.take<double>(m);
    h->costT = cv.take<double>(n);
    h->loT = cv.take<double>(n);
    h->upT = cv.take<double>(n);
    h->X = cv.take<double>(n);
    h->Z = cv.take<double>(n);
    h->AXv = cv.take<double>(n);
    h->AZv = cv.take<double>(n);
    h->XT = cv.take<double>(n);
    h->BX = cv.take<double>(n);
    h->BZ = cv.take<double>(n);
    h->Y = cv.take<double>(m);
    h->AYv = cv.take<double>(m);
    h->BY = cv.take<double>(m);
    h->XM = cv.take<double>(n);
    h->ZM = cv.take<double>(n);
    h->YM = cv.take<double>(m);
    h->BXm = cv.take<double>(n);
    h->BZm = cv.take<double>(n);
    h->BYm = cv.take<double>(m);
    const size_t nsa = pa_.tiles + pa_.longs, nst = pt_.tiles + pt_.longs;
    h->rowpart = cv.take<double>(KR * nsa);
    h->colpart = cv.take<double>(KC * std::max(nst, nsa));
    h->red = cv.take<double>(RED_BLOCKS + 64);
    h->pw = cv.take<double>(m + n);
    h->rperm = cv.take<int>(m);
    h->cperm = cv.take<int>(n);
    h->stage = cv.take<double>(std::max(m, n));
    h->SP = cv.take<double>(std::max(m, n));
    h->ctrl = cv.take<Ctrl>(1);
    h->d_dev = cv.take<unsigned long long>(2);
    return cv.off + 256;
}

// Locality ordering (SURVEY.md §7 hard part 5).  The reference lays
// variables out [g, t] (formulation.py:53-69), so a period-t flow row
// gathers x at stride T.  Columns are regrouped by the first long row
// (> LONG_ROW nonzeros) that touches them — for SCUC the balance row of
// their period — and rows (equalities and inequalities separately, so the
// n_eq prefix is preserved) by their smallest new column.  Entry order
// inside every row of A and A^T stays the original one, so every row sum
// keeps the reference's summation order; only the labels move.
constexpr int LONG_ROW = 256;

void compute_order(int m, int n, int n_eq, const std::vector<int32_t>& ptr,
                   const std::vector<int32_t>& idx, std::vector<int32_t>& rperm,
                   std::vector<int32_t>& cperm) {
    const int INF = 0x7fffffff;
    std::vector<int32_t> ckey(n, INF);
    for (int i = 0; i < m; ++i)
        if (ptr[i + 1] - ptr[i] > LONG_ROW)
            for (int e = ptr[i]; e < ptr[i + 1]; ++e)
                if (ckey[idx[e]] == INF) ckey[idx[e]] = i;
    cperm.resize(n);
    for (int j = 0; j < n; ++j) cperm[j] = j;
    std::stable_sort(cperm.begin(), cperm.end(),
                     [&](int a, int b) { return ckey[a] < ckey[b]; });
    std::vector<int32_t> cinv(n);
    for (int k = 0; k < n; ++k) cinv[cperm[k]] = k;
    std::vector<int32_t> rkey(m, INF);
    for (int i = 0; i < m; ++i)
        for (int e = ptr[i]; e < ptr[i + 1]; ++e) rkey[i] = std::min(rkey[i], cinv[idx[e]]);
    rperm.resize(m);
    for (int i = 0; i < m; ++i) rperm[i] = i;
    auto by = [&](int a, int b) { return rkey[a] < rkey[b]; };
    std::stable_sort(rperm.begin(), rperm.begin() + n_eq, by);
    std::stable_sort(rperm.begin() + n_eq, rperm.end(), by);
}

// relabel a CSR: new row r' = old row perm_rows[r'], columns through inv_cols
void permute_csr(int rows, const std::vector<int32_t>& ptr, const std::vector<int32_t>& idx,
                 const std::vector<double>& val, const std::vector<int32_t>& perm_rows,
                 const std::vector<int32_t>& inv_cols, std::vector<int32_t>& nptr,
                 std::vector<int32_t>& nidx, std::vector<double>& nval) {
    nptr.assign(rows + 1, 0);
    for (int r = 0; r < rows; ++r) nptr[r + 1] = nptr[r] + (ptr[perm_rows[r] + 1] - ptr[perm_rows[r]]);
    nidx.resize(idx.size());
    nval.resize(val.size());
    for (int r = 0; r < rows; ++r) {
        const int o = perm_rows[r];
        int q = nptr[r];
        for (int e = ptr[o]; e < ptr[o + 1]; ++e, ++q) {
            nidx[q] = inv_cols[idx[e]];
            nval[q] = val[e];
        }
    }
}

__global__ void k_gather(double* dst, const double* src, const int* perm, int len) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < len) dst[i] = src[perm[i]];
}

__global__ void k_scatter(double* dst, const double* src, const int* perm, int len) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < len) dst[perm[i]] = src[i];
}

void host_transpose(int m, int n, const int32_t* ptr, const int32_t* idx, const double* val,
                    std::vector<int32_t>& tptr, std::vector<int32_t>& tidx,
                    std::vector<double>& tval) {
    const long long nnz = ptr[m];
    tptr.assign(n + 1, 0);
    for (long long e = 0; e < nnz; ++e) tptr[idx[e] + 1]++;
    for (int j = 0; j < n; ++j) tptr[j + 1] += tptr[j];
    std::vector<int32_t> next(tptr.begin(), tptr.end() - 1);
    tidx.resize(nnz);
    tval.resize(nnz);
    for (int i = 0; i < m; ++i)
        for (int e = ptr[i]; e < ptr[i + 1]; ++e) {
            const int p = next[idx[e]]++;
            tidx[p] = i;
            tval[p] = val[e];
        }
}

template <typename T>
std::vector<T> to_host(const T* p, size_t count) {
    std::vector<T> v(count);
    if (count) {
        cudaPointerAttributes at;
        if (cudaPointerGetAttributes(&at, p) == cudaSuccess && at.type == cudaMemoryTypeDevice) {
            CK(cudaMemcpy(v.data(), p, count * sizeof(T), cudaMemcpyDeviceToHost));
        } else {
            cudaGetLastError();
            std::memcpy(v.data(), p, count * sizeof(T));
        }
    }
    return v;
}

inline int nblk(long long n, int tpb = TPB) { return (int)std::max<long long>(1, (n + tpb - 1) / tpb); }

// caller vector (original order, host or device) -> device vector (engine order)
void put_vec(hpr_handle* h, double* dst, const double* src, int len, bool rows) {
    if (!h->reordered) {
        CK(cudaMemcpyAsync(dst, src, sizeof(double) * len, cudaMemcpyDefault, h->stream));
        return;
    }
    CK(cudaMemcpyAsync(h->stage, src, sizeof(double) * len, cudaMemcpyDefault, h->stream));
    k_gather<<<nblk(len), TPB, 0, h->stream>>>(dst, h->stage, rows ? h->rperm : h->cperm, len);
    CKL();
}

// device vector (engine order) -> caller vector (original order, host or device)
void get_vec(hpr_handle* h, double* dst, const double* src, int len, bool rows) {
    if (!h->reordered) {
        CK(cudaMemcpyAsync(dst, src, sizeof(double) * len, cudaMemcpyDefault, h->stream));
        return;
    }
    k_scatter<<<nblk(len), TPB, 0, h->stream>>>(h->stage, src, rows ? h->rperm : h->cperm, len);
    CKL();
    CK(cudaMemcpyAsync(dst, h->stage, sizeof(double) * len, cudaMemcpyDefault, h->stream));
}

void validate(const hpr_problem* p) {
    if (!p) fail(HPR_ERR_INVALID, "problem is NULL");
    if (p->m < 0 || p->n < 0 || p->n_eq < 0 || p->n_eq > p->m)
        fail(HPR_ERR_INVALID, "invalid dimensions");
    if (p->nnz < 0 || p->nnz >= (1LL << 31)) fail(HPR_ERR_INVALID, "nnz must fit int32 indexing");
    if (!p->indptr || (p->nnz && (!p->indices || !p->data)))
        fail(HPR_ERR_INVALID, "CSR arrays missing");
    if (!p->rhs || !p->cost || !p->lower || !p->upper) fail(HPR_ERR_INVALID, "LP vectors missing");
}

// deterministic ||v||^2 on device -> host
double dev_sumsq(hpr_handle* h, const double* v, long long n, int finite_only) {
    k_sumsq_part<<<RED_BLOCKS, TPB, 0, h->stream>>>(v, n, finite_only, h->red);
    CKL();
    k_sum_slots<<<1, TPB, 0, h->stream>>>(h->red, RED_BLOCKS, 1, h->red + RED_BLOCKS);
    CKL();
    h->launches += 2;
    CK(cudaMemcpyAsync(h->h_scal, h->red + RED_BLOCKS, sizeof(double), cudaMemcpyDeviceToHost,
                       h->stream));
    CK(cudaStreamSynchronize(h->stream));
    return h->h_scal[0];
}

template <typename T, class Epi>
void launch_spmv(hpr_handle* h, const DevCsr& M, const T* vals, const T* xg, const Epi& epi,
                 cudaStream_t s) {
    if (M.pipe) {
        static bool attr_set = false;   // one per template instantiation
        constexpr size_t smem = pipe_smem_bytes<T>();
        if (!attr_set) {
            CK(cudaFuncSetAttribute(k_spmv_pipe<T, Epi>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)smem));
            attr_set = true;
        }
        k_spmv_pipe<T, Epi><<<M.nblocks, TPB, smem, s>>>(M.view<T>(vals), xg, epi);
    } else {
        k_spmv<T, Epi><<<M.ntiles, TPB, 0, s>>>(M.view<T>(vals), xg, epi);
    }
    CKL();
    h->launches += 1;
}

// power_method (lp_kernel.py:138-175) on an FP64 operand pair (A, A^T)
double power_method(hpr_handle* h, const double* a_vals, const double* at_vals, double tol,
                    int max_iter, double inflation, const double* start, int start_count,
                    int* iters_out, int* conv_out) {
    if (h->nnz == 0) fail(HPR_ERR_EMPTY, "power_method requires a nonzero matrix");
    if (!start || start_count < 1) fail(HPR_ERR_INVALID, "power_method needs a start vector");
    double* v = h->pw;         // m
    double* u = h->pw + h->m;  // n
    int used = 0;
    auto load_start = [&]() {
        if (used >= start_count) fail(HPR_ERR_POWER_NULL, "power_method exhausted start vectors");
        put_vec(h, v, start + (size_t)used * h->m, h->m, true);
        ++used;
        const double nv = std::sqrt(dev_sumsq(h, v, h->m, 0));
        k_div<<<nblk(h->m), TPB, 0, h->stream>>>(v, h->m, nv);
        CKL();
        h->launches++;
    };
    load_start();
    double lam = 0.0, prev = -1.0;
    bool conv = false;
    int it = 0;
    EpiStore<double> st{u, nullptr};
    EpiPower pwe{v, h->rowpart};
    for (; it < max_iter; ++it) {
        launch_spmv(h, h->AT, at_vals, (const double*)v, st, h->stream);   // u = A^T v
        launch_spmv(h, h->A, a_vals, (const double*)u, pwe, h->stream);    // v = A u, sum v^2
        k_sum_slots<<<1, TPB, 0, h->stream>>>(h->rowpart, h->A.nslots(), 1, h->red);
        CKL();
        h->launches++;
        CK(cudaMemcpyAsync(h->h_scal, h->red, sizeof(double), cudaMemcpyDeviceToHost, h->stream));
        CK(cudaStreamSynchronize(h->stream));
        lam = std::sqrt(h->h_scal[0]);
        if (lam <= 0.0) {
            load_start();
            prev = -1.0;
            continue;
        }
        k_div<<<nblk(h->m), TPB, 0, h->stream>>>(v, h->m, lam);
        CKL();
        h->launches++;
        if (std::fabs(lam - prev) <= tol * std::max(lam, 1e-300)) {
            conv = true;
            ++it;
            break;
        }
        prev = lam;
    }
    if (iters_out) *iters_out = it;
    if (conv_out) *conv_out = conv;
    if (inflation < 0) inflation = 1.0 + tol;
    return lam * inflation;
}

// Ruiz -> Pock-Chambolle -> normalisation on device (hprlp.py:213-264)
void scale_problem(hpr_handle* h, const hpr_params* prm, double* bsc_out, double* csc_out) {
    cudaStream_t s = h->stream;
    const int m = h->m, n = h->n;
    k_fill<<<nblk(m), TPB, 0, s>>>(h->rs, 1.0, m);
    k_fill<<<nblk(n), TPB, 0, s>>>(h->cs, 1.0, n);
    h->launches += 2;
    CK(cudaMemcpyAsync(h->A.w64, h->A.mval, sizeof(double) * h->nnz, cudaMemcpyDeviceToDevice, s));
    CK(cudaMemcpyAsync(h->AT.w64, h->AT.mval, sizeof(double) * h->nnz, cudaMemcpyDeviceToDevice, s));
    auto apply = [&]() {
        k_scale_csr<<<nblk((long long)m * 32), TPB, 0, s>>>(h->A.ptr, h->A.idx, h->A.w64, m, h->fr,
                                                           h->fc, 0);
        CKL();
        k_scale_csr<<<nblk((long long)n * 32), TPB, 0, s>>>(h->AT.ptr, h->AT.idx, h->AT.w64, n,
                                                            h->fc, h->fr, 1);
        CKL();
        h->launches += 2;
    };
    if (prm->ruiz) {
        for (int it = 0; it < prm->ruiz_iters; ++it) {
            CK(cudaMemsetAsync(h->d_dev, 0, 2 * sizeof(unsigned long long), s));
            k_row_absmax<<<nblk((long long)m * 32), TPB, 0, s>>>(h->A.ptr, h->A.w64, m, h->fr);
            k_row_absmax<<<nblk((long long)n * 32), TPB, 0, s>>>(h->AT.ptr, h->AT.w64, n, h->fc);
            k_scale_factor<<<nblk(m), TPB, 0, s>>>(h->fr, h->fr, h->rs, m, h->d_dev);
            k_scale_factor<<<nblk(n), TPB, 0, s>>>(h->fc, h->fc, h->cs, n, h->d_dev + 1);
            CKL();
            h->launches += 4;
            apply();
            CK(cudaMemcpyAsync(h->h_scal, h->d_dev, 2 * sizeof(double), cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            const double d = std::max(h->h_scal[0], h->h_scal[1]);
            if (d < 1e-6) break;
        }
    }
    if (prm->pock_chambolle) {
        k_row_abssum<<<nblk(m), TPB, 0, s>>>(h->A.ptr, h->A.w64, m, h->fr);
        k_row_abssum<<<nblk(n), TPB, 0, s>>>(h->AT.ptr, h->AT.w64, n, h->fc);
        k_scale_factor<<<nblk(m), TPB, 0, s>>>(h->fr, h->fr, h->rs, m, nullptr);
        k_scale_factor<<<nblk(n), TPB, 0, s>>>(h->fc, h->fc, h->cs, n, nullptr);
        CKL();
        h->launches += 4;
        apply();
    }
    k_work_cols<<<nblk(n), TPB, 0, s>>>(n, h->cost_m, h->lo_m, h->up_m, h->cs, h->cost_w, h->lo_w,
                                        h->up_w);
    k_work_rows<<<nblk(m), TPB, 0, s>>>(m, h->rhs_m, h->rs, h->rhs_w);
    CKL();
    h->launches += 2;
    double bsc = 1.0, csc = 1.0;
    if (prm->normalize_rhs_objective) {
        bsc = 1.0 + std::sqrt(dev_sumsq(h, h->rhs_w, m, 1));
        csc = 1.0 + std::sqrt(dev_sumsq(h, h->cost_w, n, 0));
    }
    k_div<<<nblk(m), TPB, 0, s>>>(h->rhs_w, m, bsc);
    k_norm_cols<<<nblk(n), TPB, 0, s>>>(n, bsc, csc, h->cost_w, h->lo_w, h->up_w);
    CKL();
    h->launches += 2;
    *bsc_out = bsc;
    *csc_out = csc;
}

template <typename T>
struct Ptrs {
    T *X, *Y, *Z, *AX, *AY, *AZ, *XT, *BX, *BY, *BZ;
    const T *rhs, *cost, *lo, *up, *a_vals, *at_vals;
};

template <typename T>
Ptrs<T> ptrs(hpr_handle* h, bool fp32) {
    Ptrs<T> p;
    p.X = (T*)h->X;
    p.Y = (T*)h->Y;
    p.Z = (T*)h->Z;
    p.AX = (T*)h->AXv;
    p.AY = (T*)h->AYv;
    p.AZ = (T*)h->AZv;
    p.XT = (T*)h->XT;
    p.BX = (T*)h->BX;
    p.BY = (T*)h->BY;
    p.BZ = (T*)h->BZ;
    if (fp32) {
        p.rhs = (const T*)h->rhsT;
        p.cost = (const T*)h->costT;
        p.lo = (const T*)h->loT;
        p.up = (const T*)h->upT;
        p.a_vals = (const T*)h->A.w32;
        p.at_vals = (const T*)h->AT.w32;
    } else {
        p.rhs = (const T*)h->rhs_w;
        p.cost = (const T*)h->cost_w;
        p.lo = (const T*)h->lo_w;
        p.up = (const T*)h->up_w;
        p.a_vals = (const T*)h->A.w64;
        p.at_vals = (const T*)h->AT.w64;
    }
    return p;
}

// the check phase: master-space residual of the bar triple + controller + copies
template <typename T>
void enqueue_check(hpr_handle* h, const Ptrs<T>& p, int mode, cudaStream_t s) {
    EpiCheckRows<T> er{h->n_eq, h->YM, h->rhs_m, p.BY, p.AY, h->rowpart};
    launch_spmv(h, h->A, (const double*)h->A.mval, (const double*)h->XM, er, s);
    EpiCheckCols<T> ec{h->XM, h->ZM, h->cost_m, h->lo_m, h->up_m, p.BX, p.BZ, p.AX, h->colpart};
    launch_spmv(h, h->AT, (const double*)h->AT.mval, (const double*)h->YM, ec, s);
    k_controller<<<1, CTRL_TPB, 0, s>>>(h->ctrl, h->rowpart, h->A.nslots(), h->colpart,
                                        h->AT.nslots(), h->log, mode);
    CKL();
    const int len = std::max(h->n, h->m);
    k_restart_copy<T><<<std::min(nblk(len), 148 * 8), TPB, 0, s>>>(
        h->ctrl, h->n, h->m, h->XM, h->YM, h->ZM, h->BXm, h->BYm, h->BZm, p.X, p.Y, p.Z, p.AX,
        p.AY, p.AZ, p.BX, p.BY, p.BZ);
    CKL();
    h->launches += 2;
}

// One row-wise pass of an epilogue over a precomputed product vector:
// the projection / reflection / Halpern update of a whole half-iteration in
// one coalesced sweep (the split form of the fused SpMV epilogue).
template <typename T, class Epi>
__global__ void __launch_bounds__(TPB) k_rowwise(Epi epi, const T* __restrict__ sums, int len) {
    epi.prepare();
    Acc<0> acc;
    for (int j = blockIdx.x * TPB + threadIdx.x; j < len; j += gridDim.x * TPB) {
        typename Epi::Pre pre;
        epi.load(j, pre);
        epi.apply(j, sums[j], pre, acc);
    }
}

template <typename T, class Epi>
void launch_rowwise(hpr_handle* h, const Epi& epi, const T* sums, int len, cudaStream_t s) {
    k_rowwise<T, Epi><<<std::min(nblk(len), 148 * 16), TPB, 0, s>>>(epi, sums, len);
    CKL();
    h->launches += 1;
}

template <typename T, bool CHECK>
void enqueue_split(hpr_handle* h, const Ptrs<T>& p, int j, cudaStream_t s) {
    T* sp = (T*)h->SP;
    EpiStore<T> st{sp, nullptr};
    launch_spmv(h, h->AT, p.at_vals, (const T*)p.Y, st, s);
    EpiPrimal<T, CHECK> e1{h->ctrl, j, p.X, p.Z, p.XT, p.AX, p.AZ, p.cost, p.lo, p.up,
                           p.BX, p.BZ, h->XM, h->ZM, h->cs, nullptr};
    launch_rowwise(h, e1, (const T*)sp, h->n, s);
    launch_spmv(h, h->A, p.a_vals, (const T*)p.XT, st, s);
    EpiDual<T, CHECK> e2{h->ctrl, j, h->n_eq, p.Y, p.AY, p.rhs, p.BY, h->YM, h->rs, nullptr};
    launch_rowwise(h, e2, (const T*)sp, h->m, s);
}

template <typename T>
void enqueue_iteration(hpr_handle* h, const Ptrs<T>& p, int j, bool check, cudaStream_t s) {
    if (!h->fuse) {
        if (check) enqueue_split<T, true>(h, p, j, s);
        else enqueue_split<T, false>(h, p, j, s);
        return;
    }
    if (check) {
        EpiPrimal<T, true> e1{h->ctrl, j, p.X, p.Z, p.XT, p.AX, p.AZ, p.cost, p.lo, p.up,
                              p.BX, p.BZ, h->XM, h->ZM, h->cs, nullptr};
        launch_spmv(h, h->AT, p.at_vals, (const T*)p.Y, e1, s);
        EpiDual<T, true> e2{h->ctrl, j, h->n_eq, p.Y, p.AY, p.rhs, p.BY, h->YM, h->rs, nullptr};
        launch_spmv(h, h->A, p.a_vals, (const T*)p.XT, e2, s);
    } else {
        EpiPrimal<T, false> e1{h->ctrl, j, p.X, p.Z, p.XT, p.AX, p.AZ, p.cost, p.lo, p.up,
                               p.BX, p.BZ, h->XM, h->ZM, h->cs, nullptr};
        launch_spmv(h, h->AT, p.at_vals, (const T*)p.Y, e1, s);
        EpiDual<T, false> e2{h->ctrl, j, h->n_eq, p.Y, p.AY, p.rhs, p.BY, h->YM, h->rs, nullptr};
        launch_spmv(h, h->A, p.a_vals, (const T*)p.XT, e2, s);
    }
}

template <typename T>
void ensure_graph(hpr_handle* h, const Ptrs<T>& p, int B) {
    const int prec = sizeof(T) == 4 ? HPR_FP32 : HPR_FP64;
    if (h->gexec && h->g_B == B && h->g_prec == prec) return;
    if (h->gexec) cudaGraphExecDestroy(h->gexec);
    if (h->graph) cudaGraphDestroy(h->graph);
    h->gexec = nullptr;
    h->graph = nullptr;
    // WHILE(cond) { B fused iterations; master check; controller; copies }
    CK(cudaGraphCreate(&h->graph, 0));
    cudaGraphConditionalHandle cond;
    CK(cudaGraphConditionalHandleCreate(&cond, h->graph, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams np = {};
    np.type = cudaGraphNodeTypeConditional;
    np.conditional.handle = cond;
    np.conditional.type = cudaGraphCondTypeWhile;
    np.conditional.size = 1;
    cudaGraphNode_t node;
    CK(cudaGraphAddNode(&node, h->graph, nullptr, 0, &np));
    cudaGraph_t body = np.conditional.phGraph_out[0];
    const long long l0 = h->launches;
    CK(cudaStreamBeginCaptureToGraph(h->cap, body, nullptr, nullptr, 0,
                                     cudaStreamCaptureModeThreadLocal));
    for (int j = 0; j < B; ++j) enqueue_iteration<T>(h, p, j, j == B - 1, h->cap);
    enqueue_check<T>(h, p, 1, h->cap);
    cudaGraph_t captured;
    CK(cudaStreamEndCapture(h->cap, &captured));
    h->g_per_block = h->launches - l0;
    h->launches = l0;
    CK(cudaGraphInstantiate(&h->gexec, h->graph, 0));
    h->gcond = (unsigned long long)cond;
    h->g_B = B;
    h->g_prec = prec;
}

// Launch the cached loop graph from the current device state; returns the
// device time of the loop (CUDA events on the handle's stream).
double run_loop(hpr_handle* h) {
    cudaStream_t s = h->stream;
    unsigned long long cv = h->gcond;
    CK(cudaMemcpyAsync(&h->ctrl->cond, &cv, sizeof(cv), cudaMemcpyHostToDevice, s));
    const long long t_before = h->h_ctrl->total;
    CK(cudaEventRecord(h->ev[2], s));
    CK(cudaGraphLaunch(h->gexec, s));
    CK(cudaEventRecord(h->ev[3], s));
    unsigned long long zero = 0;
    CK(cudaMemcpyAsync(&h->ctrl->cond, &zero, sizeof(zero), cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(h->h_ctrl, h->ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    h->launches += h->g_per_block * ((h->h_ctrl->total - t_before) / h->g_B);
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, h->ev[2], h->ev[3]));
    return ms * 1e-3;
}

void read_ctrl(hpr_handle* h) {
    CK(cudaMemcpyAsync(h->h_ctrl, h->ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
}

template <typename T>
void solve_typed(hpr_handle* h, const hpr_params* prm, const double* x0, const double* y0,
                 const double* z0, double* xo, double* yo, double* zo, hpr_stats* st,
                 std::chrono::steady_clock::time_point t_start) {
    const bool fp32 = sizeof(T) == 4;
    cudaStream_t s = h->stream;
    const int m = h->m, n = h->n;
    CK(cudaEventRecord(h->ev[0], s));

    double bsc, csc;
    scale_problem(h, prm, &bsc, &csc);

    int pits = 0, pconv = 0;
    const double lam = power_method(h, h->A.w64, h->AT.w64, prm->power_tol, prm->power_max_iter,
                                    prm->power_inflation, prm->power_start,
                                    prm->power_start_count, &pits, &pconv);
    const double rn = std::sqrt(dev_sumsq(h, h->rhs_w, m, 0));
    const double cn = std::sqrt(dev_sumsq(h, h->cost_w, n, 0));
    double sigma;
    if (prm->has_sigma0) sigma = prm->sigma0;
    else if (rn > 1e-12 && cn > 1e-12) sigma = rn / cn;
    else sigma = 1.0;
    const double rhs_norm_m = std::sqrt(dev_sumsq(h, h->rhs_m, m, 0));
    const double cost_norm_m = std::sqrt(dev_sumsq(h, h->cost_m, n, 0));

    if (fp32) {
        k_cast_f32<<<nblk(h->nnz), TPB, 0, s>>>(h->A.w64, h->A.w32, h->nnz);
        k_cast_f32<<<nblk(h->nnz), TPB, 0, s>>>(h->AT.w64, h->AT.w32, h->nnz);
        k_cast_f32<<<nblk(m), TPB, 0, s>>>(h->rhs_w, (float*)h->rhsT, m);
        k_cast_f32<<<nblk(n), TPB, 0, s>>>(h->cost_w, (float*)h->costT, n);
        k_cast_f32<<<nblk(n), TPB, 0, s>>>(h->lo_w, (float*)h->loT, n);
        k_cast_f32<<<nblk(n), TPB, 0, s>>>(h->up_w, (float*)h->upT, n);
        CKL();
        h->launches += 6;
    }

    // device-resident warm start (master space)
    const double *dx0 = nullptr, *dy0 = nullptr, *dz0 = nullptr;
    if (x0 && y0 && z0) {
        put_vec(h, h->BXm, x0, n, false);
        put_vec(h, h->BYm, y0, m, true);
        put_vec(h, h->BZm, z0, n, false);
        dx0 = h->BXm;
        dy0 = h->BYm;
        dz0 = h->BZm;
    }
    Ptrs<T> p = ptrs<T>(h, fp32);
    k_init_cols<T><<<nblk(n), TPB, 0, s>>>(n, dx0, dz0, h->cs, bsc, csc, h->lo_w, h->up_w, p.X,
                                           p.Z, p.AX, p.AZ, p.BX, p.BZ, h->XM, h->ZM);
    k_init_rows<T><<<nblk(m), TPB, 0, s>>>(m, dy0, h->rs, csc, p.Y, p.AY, p.BY, h->YM);
    CKL();
    h->launches += 2;

    const int B = prm->log_every_iteration ? 1 : std::max(1, prm->check_every);
    if (B > MAX_B) fail(HPR_ERR_INVALID, "check_every too large");
    Ctrl c{};
    c.sigma = sigma;
    c.lam = lam;
    c.norm_a = std::sqrt(lam);
    c.tol = prm->tolerance;
    c.beta = prm->restart_beta;
    c.damping = prm->sigma_damping;
    c.denom = (1.0 + rhs_norm_m) + cost_norm_m;
    c.offset = h->offset;
    c.b_scale = bsc;
    c.c_scale = csc;
    c.max_iter = prm->max_iterations;
    c.stall = prm->restart_stall;
    c.B = B;
    c.status = -1;
    c.log_on = (prm->log_residuals || prm->log_every_iteration) ? 1 : 0;
    if (c.log_on) {
        const long long want = std::min<long long>(prm->max_iterations / B + 2, LOG_CAP_MAX);
        if (want > h->log_cap) {
            if (h->log) cudaFree(h->log);
            h->log = nullptr;
            CK(cudaMalloc(&h->log, sizeof(LogRec) * want));
            h->log_cap = want;
        }
        c.log_cap = h->log_cap;
    }
    CK(cudaMemcpyAsync(h->ctrl, &c, sizeof(Ctrl), cudaMemcpyHostToDevice, s));
    enqueue_check<T>(h, p, 0, s);               // initial residual (hprlp.py:371-391)
    CK(cudaEventRecord(h->ev[1], s));
    read_ctrl(h);

    const double elapsed =
        prm->time_elapsed +
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
    int status = h->h_ctrl->status;
    long long iterations = 0;
    if (status == -1) {
        if (prm->max_iterations <= 0) {
            status = HPR_ITERATION_LIMIT;
        } else if (prm->time_limit >= 0 && elapsed > prm->time_limit) {
            status = HPR_TIME_LIMIT;
        } else if (prm->max_iterations < B) {
            status = HPR_ITERATION_LIMIT;            // tail only: no check can happen
            iterations = prm->max_iterations;
        }
    }
    if (status == -1) {
        if (prm->time_limit >= 0) {
            const double rem = std::max(0.0, prm->time_limit - elapsed);
            k_set_deadline<<<1, 1, 0, s>>>(h->ctrl, (unsigned long long)(rem * 1e9));
            CKL();
            h->launches++;
            int one = 1;
            CK(cudaMemcpyAsync(&h->ctrl->has_deadline, &one, sizeof(int), cudaMemcpyHostToDevice, s));
        }
        ensure_graph<T>(h, p, B);
        st->loop_seconds = run_loop(h);
        status = h->h_ctrl->status;
        iterations = h->h_ctrl->total;
        if (status == HPR_ITERATION_LIMIT) iterations = prm->max_iterations;
    } else {
        st->loop_seconds = 0.0;
    }
    float sms = 0.f;
    CK(cudaEventElapsedTime(&sms, h->ev[0], h->ev[1]));
    st->setup_seconds = sms * 1e-3;

    const Ctrl& hc = *h->h_ctrl;
    st->status = status;
    st->precision_used = fp32 ? HPR_FP32 : HPR_FP64;
    st->iterations = iterations;
    st->restarts = hc.restarts;
    st->sigma_final = hc.sigma;
    st->lam = lam;
    std::memcpy(&st->kkt, hc.best, sizeof(hpr_kkt));
    st->objective = hc.best[6];
    st->n_log = c.log_on ? hc.n_log : 0;
    st->power_iterations = pits;
    st->power_converged = pconv;
    st->checks = hc.checks;
    h->last_prec = fp32 ? HPR_FP32 : HPR_FP64;
    if (xo) get_vec(h, xo, h->BXm, n, false);
    if (yo) get_vec(h, yo, h->BYm, m, true);
    if (zo) get_vec(h, zo, h->BZm, n, false);
    if (st->n_log) {
        h->h_log.resize(st->n_log);
        CK(cudaMemcpyAsync(h->h_log.data(), h->log, sizeof(LogRec) * st->n_log,
                           cudaMemcpyDeviceToHost, s));
    } else {
        h->h_log.clear();
    }
    CK(cudaStreamSynchronize(s));
}

Plan plan_for(const int32_t* ptr, int rows) { return build_tiles(ptr, rows); }

}  // namespace

// ===========================================================================
// C-ABI
// ===========================================================================

#define API_BEGIN try {
#define API_END                                                   \
    }                                                             \
    catch (const HprError& e) {                                   \
        return e.code;                                            \
    }                                                             \
    catch (const std::exception& e) {                             \
        g_err = e.what();                                         \
        return HPR_ERR_NOMEM;                                     \
    }                                                             \
    return HPR_OK;

extern "C" {

int32_t hpr_abi_version(void) { return HPR_ABI_VERSION; }

const char* hpr_last_error(void) { return g_err.c_str(); }

int hpr_workspace_bytes(const hpr_problem* p, size_t* bytes) {
    API_BEGIN
    validate(p);
    if (!bytes) fail(HPR_ERR_INVALID, "bytes is NULL");
    hpr_handle tmp;
    tmp.m = p->m;
    tmp.n = p->n;
    tmp.nnz = p->nnz;
    *bytes = carve(&tmp, nullptr);
    API_END
}

int hpr_create(const hpr_problem* p, const hpr_options* opt, hpr_handle** out) {
    hpr_handle* h = nullptr;
    try {
        validate(p);
        if (!out) fail(HPR_ERR_INVALID, "out is NULL");
        h = new hpr_handle();
        h->dev = opt ? opt->device : 0;
        CK(cudaSetDevice(h->dev));
        h->m = p->m;
        h->n = p->n;
        h->n_eq = p->n_eq;
        h->nnz = p->nnz;
        h->offset = p->offset;
        std::vector<int32_t> ptr = to_host(p->indptr, (size_t)p->m + 1);
        if (ptr[0] != 0 || ptr[p->m] != p->nnz) fail(HPR_ERR_INVALID, "indptr inconsistent with nnz");
        std::vector<int32_t> idx = to_host(p->indices, (size_t)p->nnz);
        std::vector<double> val = to_host(p->data, (size_t)p->nnz);
        for (int i = 0; i < p->m; ++i)
            if (ptr[i + 1] < ptr[i]) fail(HPR_ERR_INVALID, "indptr not monotone");
        for (auto c : idx)
            if (c < 0 || c >= p->n) fail(HPR_ERR_INVALID, "column index out of range");
        std::vector<int32_t> tptr, tidx;
        std::vector<double> tval;
        if (p->t_indptr && p->t_indices && p->t_data) {
            tptr = to_host(p->t_indptr, (size_t)p->n + 1);
            tidx = to_host(p->t_indices, (size_t)p->nnz);
            tval = to_host(p->t_data, (size_t)p->nnz);
        } else {
            host_transpose(p->m, p->n, ptr.data(), idx.data(), val.data(), tptr, tidx, tval);
        }
        std::vector<int32_t> rperm, cperm;
        const bool reorder = !(opt && (opt->flags & HPR_FLAG_NO_REORDER));
        if (reorder) {
            compute_order(p->m, p->n, p->n_eq, ptr, idx, rperm, cperm);
            std::vector<int32_t> rinv(p->m), cinv(p->n);
            for (int i = 0; i < p->m; ++i) rinv[rperm[i]] = i;
            for (int j = 0; j < p->n; ++j) cinv[cperm[j]] = j;
            std::vector<int32_t> a, b;
            std::vector<double> c;
            permute_csr(p->m, ptr, idx, val, rperm, cinv, a, b, c);
            ptr.swap(a);
            idx.swap(b);
            val.swap(c);
            permute_csr(p->n, tptr, tidx, tval, cperm, rinv, a, b, c);
            tptr.swap(a);
            tidx.swap(b);
            tval.swap(c);
            h->reordered = true;
        }
        Plan pa = plan_for(ptr.data(), p->m), pt = plan_for(tptr.data(), p->n);
        {
            const TileBound ba = tile_bound(p->m, p->nnz), bt = tile_bound(p->n, p->nnz);
            if (pa.tiles.size() > ba.tiles || pt.tiles.size() > bt.tiles ||
                pa.longs.size() > ba.longs || pt.longs.size() > bt.longs)
                fail(HPR_ERR_INVALID, "internal: tile bound violated");
        }
        const size_t need = carve(h, nullptr);
        if (opt && opt->workspace) {
            if (opt->workspace_bytes < need) fail(HPR_ERR_NOMEM, "workspace too small");
            h->ws = opt->workspace;
            h->ws_bytes = opt->workspace_bytes;
        } else {
            CK(cudaMalloc(&h->ws, need));
            h->own_ws = true;
            h->ws_bytes = need;
        }
        carve(h, (char*)h->ws);
        if (opt && opt->stream) {
            h->stream = (cudaStream_t)opt->stream;
        } else {
            CK(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
            h->own_stream = true;
        }
        CK(cudaStreamCreateWithFlags(&h->cap, cudaStreamNonBlocking));
        for (auto& e : h->ev) CK(cudaEventCreate(&e));
        CK(cudaMallocHost(&h->h_ctrl, sizeof(Ctrl)));
        CK(cudaMallocHost(&h->h_scal, 8 * sizeof(double)));
        cudaStream_t s = h->stream;
        h->A.rows = p->m;
        h->A.cols = p->n;
        h->AT.rows = p->n;
        h->AT.cols = p->m;
        h->A.ntiles = (int)pa.tiles.size();
        h->A.nlong = (int)pa.longs.size();
        h->AT.ntiles = (int)pt.tiles.size();
        h->AT.nlong = (int)pt.longs.size();
        {
            int sms = 148;
            CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h->dev));
            const char* fz = getenv("HPR_FUSE");
            h->fuse = fz && std::string(fz) == "1";
            const char* mode = getenv("HPR_SPMV");
            const bool pipe = mode && std::string(mode) == "pipe";
            for (DevCsr* M : {&h->A, &h->AT}) {
                M->pipe = pipe;
                M->nblocks = std::max(1, std::min(M->ntiles, sms * PIPE_CTAS_PER_SM));
            }
        }
        CK(cudaMemcpyAsync(h->A.ptr, ptr.data(), sizeof(int) * (p->m + 1), cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(h->A.idx, idx.data(), sizeof(int) * p->nnz, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(h->A.mval, val.data(), sizeof(double) * p->nnz, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(h->AT.ptr, tptr.data(), sizeof(int) * (p->n + 1), cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(h->AT.idx, tidx.data(), sizeof(int) * p->nnz, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(h->AT.mval, tval.data(), sizeof(double) * p->nnz, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(h->A.tiles, pa.tiles.data(), sizeof(int4) * pa.tiles.size(), cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(h->A.longs, pa.longs.data(), sizeof(int4) * pa.longs.size(), cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(h->AT.tiles, pt.tiles.data(), sizeof(int4) * pt.tiles.size(), cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(h->AT.longs, pt.longs.data(), sizeof(int4) * pt.longs.size(), cudaMemcpyHostToDevice, s));
        if (!pa.longs.empty()) CK(cudaMemsetAsync(h->A.counters, 0, sizeof(int) * pa.longs.size(), s));
        if (!pt.longs.empty()) CK(cudaMemsetAsync(h->AT.counters, 0, sizeof(int) * pt.longs.size(), s));
        if (h->reordered) {
            CK(cudaMemcpyAsync(h->rperm, rperm.data(), sizeof(int) * p->m, cudaMemcpyHostToDevice, s));
            CK(cudaMemcpyAsync(h->cperm, cperm.data(), sizeof(int) * p->n, cudaMemcpyHostToDevice, s));
        }
        put_vec(h, h->rhs_m, p->rhs, p->m, true);
        put_vec(h, h->cost_m, p->cost, p->n, false);
        put_vec(h, h->lo_m, p->lower, p->n, false);
        put_vec(h, h->up_m, p->upper, p->n, false);
        CK(cudaMemsetAsync(h->ctrl, 0, sizeof(Ctrl), s));
        CK(cudaStreamSynchronize(s));
        *out = h;
        return HPR_OK;
    } catch (const HprError& e) {
        if (h) hpr_destroy(h);
        return e.code;
    } catch (const std::exception& e) {
        g_err = e.what();
        if (h) hpr_destroy(h);
        return HPR_ERR_NOMEM;
    }
}

void hpr_destroy(hpr_handle* h) {
    if (!h) return;
    cudaSetDevice(h->dev);
    if (h->stream) cudaStreamSynchronize(h->stream);
    if (h->own_ws && h->ws) cudaFree(h->ws);
    if (h->log) cudaFree(h->log);
    if (h->h_ctrl) cudaFreeHost(h->h_ctrl);
    if (h->h_scal) cudaFreeHost(h->h_scal);
    for (auto& e : h->ev)
        if (e) cudaEventDestroy(e);
    if (h->gexec) cudaGraphExecDestroy(h->gexec);
    if (h->graph) cudaGraphDestroy(h->graph);
    if (h->cap) cudaStreamDestroy(h->cap);
    if (h->own_stream && h->stream) cudaStreamDestroy(h->stream);
    delete h;
}

static void check_params(const hpr_params* prm) {
    if (!prm) fail(HPR_ERR_INVALID, "params is NULL");
    if (!(prm->tolerance > 0)) fail(HPR_ERR_INVALID, "tolerance must be positive");
    if (!(prm->restart_beta > 0.0 && prm->restart_beta < 1.0))
        fail(HPR_ERR_INVALID, "restart_beta must lie in (0, 1)");
    if (prm->precision != HPR_FP64 && prm->precision != HPR_FP32)
        fail(HPR_ERR_INVALID, "unknown precision");
}

int hpr_solve(hpr_handle* h, const hpr_params* prm, const double* x0, const double* y0,
              const double* z0, double* x, double* y, double* z, hpr_stats* stats) {
    API_BEGIN
    const auto t0 = std::chrono::steady_clock::now();
    if (!h || !stats) fail(HPR_ERR_INVALID, "handle/stats is NULL");
    check_params(prm);
    CK(cudaSetDevice(h->dev));
    std::memset(stats, 0, sizeof(*stats));
    h->launches = 0;
    if (prm->precision == HPR_FP32)
        solve_typed<float>(h, prm, x0, y0, z0, x, y, z, stats, t0);
    else
        solve_typed<double>(h, prm, x0, y0, z0, x, y, z, stats, t0);
    stats->gpu_launches = h->launches;
    API_END
}

int hpr_get_log(hpr_handle* h, hpr_log_record* out, int64_t cap, int64_t* n_out) {
    API_BEGIN
    if (!h) fail(HPR_ERR_INVALID, "handle is NULL");
    const int64_t k = std::min<int64_t>(cap, (int64_t)h->h_log.size());
    static_assert(sizeof(hpr_log_record) == sizeof(LogRec), "log record layout");
    if (out && k) std::memcpy(out, h->h_log.data(), sizeof(LogRec) * k);
    if (n_out) *n_out = (int64_t)h->h_log.size();
    API_END
}

int hpr_matvec(hpr_handle* h, int32_t transpose, const double* in, double* out) {
    API_BEGIN
    if (!h || !in || !out) fail(HPR_ERR_INVALID, "NULL argument");
    CK(cudaSetDevice(h->dev));
    const DevCsr& M = transpose ? h->AT : h->A;
    const int nin = transpose ? h->m : h->n, nout = transpose ? h->n : h->m;
    double* xin = transpose ? h->YM : h->XM;   // master scratch of the input length
    put_vec(h, xin, in, nin, transpose != 0);
    EpiStore<double> st{h->pw, nullptr};       // pw holds m + n doubles
    launch_spmv(h, M, (const double*)M.mval, (const double*)xin, st, h->stream);
    get_vec(h, out, h->pw, nout, transpose == 0);
    CK(cudaStreamSynchronize(h->stream));
    API_END
}

int hpr_kkt_residual(hpr_handle* h, const double* x, const double* y, const double* z,
                     hpr_kkt* out) {
    API_BEGIN
    if (!h || !x || !y || !z || !out) fail(HPR_ERR_INVALID, "NULL argument");
    CK(cudaSetDevice(h->dev));
    cudaStream_t s = h->stream;
    put_vec(h, h->XM, x, h->n, false);
    put_vec(h, h->YM, y, h->m, true);
    put_vec(h, h->ZM, z, h->n, false);
    // bar/anchor terms are irrelevant here: point them at zeroed work buffers
    CK(cudaMemsetAsync(h->BX, 0, sizeof(double) * h->n, s));
    CK(cudaMemsetAsync(h->BZ, 0, sizeof(double) * h->n, s));
    CK(cudaMemsetAsync(h->AXv, 0, sizeof(double) * h->n, s));
    CK(cudaMemsetAsync(h->BY, 0, sizeof(double) * h->m, s));
    CK(cudaMemsetAsync(h->AYv, 0, sizeof(double) * h->m, s));
    const double rn = std::sqrt(dev_sumsq(h, h->rhs_m, h->m, 0));
    const double cn = std::sqrt(dev_sumsq(h, h->cost_m, h->n, 0));
    Ctrl c{};
    c.denom = (1.0 + rn) + cn;
    c.offset = h->offset;
    c.tol = 0.0;
    c.B = 1;
    c.status = -1;
    CK(cudaMemcpyAsync(h->ctrl, &c, sizeof(Ctrl), cudaMemcpyHostToDevice, s));
    Ptrs<double> p = ptrs<double>(h, false);
    EpiCheckRows<double> er{h->n_eq, h->YM, h->rhs_m, p.BY, p.AY, h->rowpart};
    launch_spmv(h, h->A, (const double*)h->A.mval, (const double*)h->XM, er, s);
    EpiCheckCols<double> ec{h->XM, h->ZM, h->cost_m, h->lo_m, h->up_m, p.BX, p.BZ, p.AX, h->colpart};
    launch_spmv(h, h->AT, (const double*)h->AT.mval, (const double*)h->YM, ec, s);
    k_controller<<<1, CTRL_TPB, 0, s>>>(h->ctrl, h->rowpart, h->A.nslots(), h->colpart,
                                        h->AT.nslots(), h->log, 0);
    CKL();
    read_ctrl(h);
    std::memcpy(out, h->h_ctrl->cur, sizeof(hpr_kkt));
    API_END
}

int hpr_power_method(hpr_handle* h, double tol, int32_t max_iter, double inflation,
                     const double* start, int32_t start_count, double* lam, int32_t* iterations,
                     int32_t* converged) {
    API_BEGIN
    if (!h || !lam) fail(HPR_ERR_INVALID, "NULL argument");
    CK(cudaSetDevice(h->dev));
    int it = 0, cv = 0;
    *lam = power_method(h, h->A.mval, h->AT.mval, tol, max_iter, inflation, start, start_count,
                        &it, &cv);
    if (iterations) *iterations = it;
    if (converged) *converged = cv;
    API_END
}

int hpr_iterate(hpr_handle* h, int32_t precision, double sigma, double lam, int64_t k,
                const double* x, const double* y, const double* z, const double* ax,
                const double* ay, const double* az, double* x_out, double* y_out, double* z_out,
                double* bar_x, double* bar_y, double* bar_z) {
    API_BEGIN
    if (!h || !x || !y || !z || !ax || !ay || !az) fail(HPR_ERR_INVALID, "NULL argument");
    if (precision != HPR_FP64 && precision != HPR_FP32) fail(HPR_ERR_INVALID, "unknown precision");
    CK(cudaSetDevice(h->dev));
    cudaStream_t s = h->stream;
    const int m = h->m, n = h->n;
    const bool fp32 = precision == HPR_FP32;
    // identity scaling: the step runs on the LP as given (hpr_iterate(state, lp))
    CK(cudaMemcpyAsync(h->A.w64, h->A.mval, sizeof(double) * h->nnz, cudaMemcpyDeviceToDevice, s));
    CK(cudaMemcpyAsync(h->AT.w64, h->AT.mval, sizeof(double) * h->nnz, cudaMemcpyDeviceToDevice, s));
    CK(cudaMemcpyAsync(h->rhs_w, h->rhs_m, sizeof(double) * m, cudaMemcpyDeviceToDevice, s));
    CK(cudaMemcpyAsync(h->cost_w, h->cost_m, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
    CK(cudaMemcpyAsync(h->lo_w, h->lo_m, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
    CK(cudaMemcpyAsync(h->up_w, h->up_m, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
    k_fill<<<nblk(m), TPB, 0, s>>>(h->rs, 1.0, m);
    k_fill<<<nblk(n), TPB, 0, s>>>(h->cs, 1.0, n);
    CKL();
    Ctrl c{};
    c.sigma = sigma;
    c.lam = lam;
    c.k0 = k;
    c.b_scale = 1.0;
    c.c_scale = 1.0;
    CK(cudaMemcpyAsync(h->ctrl, &c, sizeof(Ctrl), cudaMemcpyHostToDevice, s));
    // stage the six state vectors (engine order), cast to the work dtype
    auto put = [&](const double* src, void* dst, int len, double* scratch, bool rows) {
        put_vec(h, scratch, src, len, rows);
        if (fp32) {
            k_cast_f32<<<nblk(len), TPB, 0, s>>>(scratch, (float*)dst, len);
            CKL();
        } else {
            CK(cudaMemcpyAsync(dst, scratch, sizeof(double) * len, cudaMemcpyDeviceToDevice, s));
        }
    };
    put(x, h->X, n, h->XM, false);
    put(z, h->Z, n, h->ZM, false);
    put(ax, h->AXv, n, h->BXm, false);
    put(az, h->AZv, n, h->BZm, false);
    put(y, h->Y, m, h->YM, true);
    put(ay, h->AYv, m, h->BYm, true);
    auto get = [&](const void* src, double* dst, int len, double* scratch, bool rows) {
        if (!dst) return;
        if (fp32) {
            std::vector<float> tmp(len);
            CK(cudaMemcpyAsync(tmp.data(), src, sizeof(float) * len, cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            std::vector<double> d(tmp.begin(), tmp.end());
            CK(cudaMemcpyAsync(scratch, d.data(), sizeof(double) * len, cudaMemcpyHostToDevice, s));
            CK(cudaStreamSynchronize(s));
            get_vec(h, dst, scratch, len, rows);
        } else {
            get_vec(h, dst, (const double*)src, len, rows);
        }
    };
    if (fp32) {
        k_cast_f32<<<nblk(h->nnz), TPB, 0, s>>>(h->A.w64, h->A.w32, h->nnz);
        k_cast_f32<<<nblk(h->nnz), TPB, 0, s>>>(h->AT.w64, h->AT.w32, h->nnz);
        k_cast_f32<<<nblk(m), TPB, 0, s>>>(h->rhs_w, (float*)h->rhsT, m);
        k_cast_f32<<<nblk(n), TPB, 0, s>>>(h->cost_w, (float*)h->costT, n);
        k_cast_f32<<<nblk(n), TPB, 0, s>>>(h->lo_w, (float*)h->loT, n);
        k_cast_f32<<<nblk(n), TPB, 0, s>>>(h->up_w, (float*)h->upT, n);
        CKL();
        Ptrs<float> p = ptrs<float>(h, true);
        enqueue_iteration<float>(h, p, 0, true, s);
    } else {
        Ptrs<double> p = ptrs<double>(h, false);
        enqueue_iteration<double>(h, p, 0, true, s);
    }
    get(h->X, x_out, n, h->XM, false);
    get(h->Y, y_out, m, h->YM, true);
    get(h->Z, z_out, n, h->ZM, false);
    get(h->BX, bar_x, n, h->XM, false);
    get(h->BY, bar_y, m, h->YM, true);
    get(h->BZ, bar_z, n, h->ZM, false);
    CK(cudaStreamSynchronize(s));
    API_END
}

int hpr_resume(hpr_handle* h, int64_t more_iterations, double tolerance, hpr_stats* st) {
    API_BEGIN
    if (!h || !st) fail(HPR_ERR_INVALID, "NULL argument");
    if (h->last_prec < 0 || !h->gexec) fail(HPR_ERR_INVALID, "hpr_resume needs a prior looping solve");
    CK(cudaSetDevice(h->dev));
    std::memset(st, 0, sizeof(*st));
    h->launches = 0;
    read_ctrl(h);
    Ctrl c = *h->h_ctrl;
    c.max_iter = c.total + more_iterations;
    c.status = more_iterations >= c.B ? -1 : HPR_ITERATION_LIMIT;
    c.has_deadline = 0;
    if (tolerance > 0) c.tol = tolerance;
    c.cond = 0;
    CK(cudaMemcpyAsync(h->ctrl, &c, sizeof(Ctrl), cudaMemcpyHostToDevice, h->stream));
    *h->h_ctrl = c;
    st->loop_seconds = c.status == -1 ? run_loop(h) : 0.0;
    const Ctrl& hc = *h->h_ctrl;
    st->status = hc.status;
    st->precision_used = h->last_prec;
    st->iterations = hc.total - (c.max_iter - more_iterations);
    st->restarts = hc.restarts;
    st->sigma_final = hc.sigma;
    st->lam = hc.lam;
    std::memcpy(&st->kkt, hc.best, sizeof(hpr_kkt));
    st->objective = hc.best[6];
    st->checks = hc.checks;
    st->gpu_launches = h->launches;
    API_END
}

int hpr_bench_kernel(hpr_handle* h, int32_t which, int32_t reps, double* seconds_per_launch) {
    API_BEGIN
    if (!h || !seconds_per_launch || reps < 1) fail(HPR_ERR_INVALID, "bad argument");
    if (h->last_prec < 0) fail(HPR_ERR_INVALID, "hpr_bench_kernel needs a prior solve");
    CK(cudaSetDevice(h->dev));
    cudaStream_t s = h->stream;
    // which: 0 = A x~ product, 1 = A^T y product, 2 = primal row-wise update,
    //        3 = dual row-wise update, 4 = fused A x~ + dual, 5 = fused A^T y + primal
    auto body = [&](auto tag) {
        using T = decltype(tag);
        Ptrs<T> p = ptrs<T>(h, sizeof(T) == 4);
        T* sp = (T*)h->SP;
        EpiStore<T> st{sp, nullptr};
        EpiDual<T, false> e2{h->ctrl, 0, h->n_eq, p.Y, p.AY, p.rhs, p.BY, h->YM, h->rs, nullptr};
        EpiPrimal<T, false> e1{h->ctrl, 0, p.X, p.Z, p.XT, p.AX, p.AZ, p.cost, p.lo, p.up,
                               p.BX, p.BZ, h->XM, h->ZM, h->cs, nullptr};
        switch (which) {
            case 0: launch_spmv(h, h->A, p.a_vals, (const T*)p.XT, st, s); break;
            case 1: launch_spmv(h, h->AT, p.at_vals, (const T*)p.Y, st, s); break;
            case 2: launch_rowwise(h, e1, (const T*)sp, h->n, s); break;
            case 3: launch_rowwise(h, e2, (const T*)sp, h->m, s); break;
            case 4: launch_spmv(h, h->A, p.a_vals, (const T*)p.XT, e2, s); break;
            default: launch_spmv(h, h->AT, p.at_vals, (const T*)p.Y, e1, s); break;
        }
    };
    auto run = [&]() {
        if (h->last_prec == HPR_FP32) body(float(0));
        else body(double(0));
    };
    run();  // warm
    CK(cudaEventRecord(h->ev[0], s));
    for (int r = 0; r < reps; ++r) run();
    CK(cudaEventRecord(h->ev[1], s));
    CK(cudaEventSynchronize(h->ev[1]));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, h->ev[0], h->ev[1]));
    *seconds_per_launch = ms * 1e-3 / reps;
    API_END
}

}  // extern "C"
