// hpr_spmv.cuh — tiled CSR SpMV with fused per-row epilogues.
//
// One kernel template serves every sparse product of the HPR path
// (A x and A^T y of hprlp.py:190,193 and kkt_residual :122,125, and the
// power method lp_kernel.py:157).  The host cuts each CSR operand into
// tiles of equal work (hpr_engine.cu: build_tiles):
//
//  * stream tile  {r0, -(r1+1), p0, p1}: consecutive rows holding <= TILE_NNZ
//    nonzeros and <= TILE_ROWS rows.  The CTA streams the tile's (value, index) range with fully
//    coalesced evict-first loads, gathers x (L2-resident), and stages the
//    products in shared memory; then groups of L lanes reduce one row each
//    (L = 1 for the short structural rows, so those sums run in index order
//    exactly like scipy's csr_matvec).
//  * chunk tile   {row, e0, e1, li}: one CHUNK_NNZ slice of a long row
//    (balance and PTDF flow rows, up to ~22K nonzeros).  Each CTA reduces
//    its slice; the last CTA to finish (atomic ticket) adds the slices in
//    chunk order — deterministic — and runs the row epilogue.
//
// The epilogue (Epi::row) consumes the complete row sum, so the HPR
// projection / reflection / Halpern update and the KKT-residual terms are
// fused into the product that feeds them: no intermediate A x or A^T y
// vector ever goes to HBM.  Epilogues with reduction terms (K > 0)
// accumulate per thread, block-reduce in a fixed order and write one slot
// per CTA (or per long row) — the controller sums slots in slot order.
#pragma once

#include "hpr_common.cuh"

namespace hpr {

template <int K>
struct Acc {
    double v[K > 0 ? K : 1];
    __device__ __forceinline__ void zero() {
#pragma unroll
        for (int k = 0; k < (K > 0 ? K : 1); ++k) v[k] = 0.0;
    }
};

template <typename T>
__device__ __forceinline__ T warp_sum(T s) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    return s;
}

// Block-reduce K accumulators in fixed order and store them at part[k*nslots + slot].
template <int K>
__device__ __forceinline__ void block_store(Acc<K>& acc, double* part, int nslots, int slot) {
    if constexpr (K > 0) {
        __shared__ double red[TPB / 32][K];
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
        for (int k = 0; k < K; ++k) {
            double s = warp_sum(acc.v[k]);
            if (lane == 0) red[warp][k] = s;
        }
        __syncthreads();
        if (threadIdx.x < K) {
            double s = 0.0;
#pragma unroll
            for (int w = 0; w < TPB / 32; ++w) s += red[w][threadIdx.x];
            part[(size_t)threadIdx.x * nslots + slot] = s;
        }
    }
}

// Asynchronous global -> shared copy of one 4- or 8-byte element (LDGSTS):
// the epilogue operands of a tile's rows are staged without occupying
// registers while the matrix stream and the gathers are in flight.
template <typename U>
__device__ __forceinline__ void cp_async_elem(U* dst, const U* src) {
    static_assert(sizeof(U) == 4 || sizeof(U) == 8, "cp.async element size");
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(dst)),
                 "l"(src), "n"((int)sizeof(U))
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// stage vector[r0 + k] (k < R) into column v of the SoA staging buffer
template <typename U>
__device__ __forceinline__ void stage_vec(unsigned char* sbuf, int byte_off, const U* vec, int r0,
                                          int R) {
    U* dst = reinterpret_cast<U*>(sbuf + byte_off);
    for (int k = threadIdx.x; k < R; k += TPB) cp_async_elem(dst + k, vec + r0 + k);
}
template <typename U>
__device__ __forceinline__ U unstage_vec(const unsigned char* sbuf, int byte_off, int k) {
    return reinterpret_cast<const U*>(sbuf + byte_off)[k];
}

template <typename T, class Epi>
__global__ void __launch_bounds__(TPB) k_spmv(Csr<T> A, const T* __restrict__ xg, Epi epi) {
    __shared__ T prod[TILE_NNZ];
    __shared__ T rsum[TILE_ROWS];
    __shared__ int sptr[TILE_ROWS + 1];
    __shared__ T wpart[TPB / 32];
    __shared__ int s_last;
    __shared__ __align__(16) unsigned char sbuf[Epi::SROW > 0 ? Epi::SROW * TILE_ROWS : 16];
    epi.prepare();
    Acc<Epi::K> acc;
    acc.zero();
    const int4 tl = A.tiles[blockIdx.x];
    if (tl.y < 0) {
        // ---------------- stream tile {r0, -(r1+1), p0, p1} ----------------
        const int r0 = tl.x, r1 = -tl.y - 1, p0 = tl.z, cnt = tl.w - tl.z;
        const int R = r1 - r0;
        const int* __restrict__ idx = A.indices + p0;
        const T* __restrict__ val = A.vals + p0;
        int c[ITEMS];
        T v[ITEMS];
#pragma unroll
        for (int q = 0; q < ITEMS; ++q) {
            const int e = threadIdx.x + q * TPB;
            c[q] = e < cnt ? ld_stream(idx + e) : 0;
            v[q] = e < cnt ? ld_stream(val + e) : T(0);
        }
        // row pointers and the epilogue operands of the tile's rows are
        // fetched while the matrix stream is in flight
        if (threadIdx.x < R) sptr[threadIdx.x] = A.indptr[r0 + threadIdx.x] - p0;
        if (threadIdx.x == 0) sptr[R] = cnt;
        const bool own = threadIdx.x < R;
        if constexpr (Epi::SROW > 0) {
            epi.stage(sbuf, r0, R);
            cp_async_commit();
        }
#pragma unroll
        for (int q = 0; q < ITEMS; ++q) {
            const int e = threadIdx.x + q * TPB;
            if (e < cnt) prod[e] = v[q] * ld_ro(xg + c[q]);
        }
        __syncthreads();
        int L = 1;
        while (L < 32 && (L * 2) * R <= TPB && L * R < cnt) L *= 2;
        const int lane = threadIdx.x & 31;
        const int gl = threadIdx.x & (L - 1);
        const int grp = threadIdx.x / L;
        const int ngrp = TPB / L;
        const unsigned mask = L == 32 ? 0xffffffffu : (((1u << L) - 1u) << (lane & ~(L - 1)));
        for (int k = grp; k < R; k += ngrp) {
            const int b = sptr[k], e = sptr[k + 1];
            T s = T(0);
            for (int q = b + gl; q < e; q += L) s += prod[q];
            for (int off = L >> 1; off > 0; off >>= 1) s += __shfl_xor_sync(mask, s, off);
            if (gl == 0) rsum[k] = s;
        }
        if constexpr (Epi::SROW > 0) cp_async_wait_all();
        __syncthreads();
        if (own) {
            typename Epi::Pre pre;
            epi.unstage(sbuf, threadIdx.x, pre);
            epi.apply(r0 + threadIdx.x, rsum[threadIdx.x], pre, acc);
        }
        block_store<Epi::K>(acc, epi.part, A.ntiles + A.nlong, blockIdx.x);
    } else {
        // ---------------- chunk of a long row {row, e0, e1, li} ----------------
        const int row = tl.x, e0 = tl.y, e1 = tl.z, li = tl.w;
        constexpr int IL = CHUNK_NNZ / TPB;
        int c[IL];
        T v[IL];
#pragma unroll
        for (int q = 0; q < IL; ++q) {
            const int e = e0 + threadIdx.x + q * TPB;
            c[q] = e < e1 ? ld_stream(A.indices + e) : 0;
            v[q] = e < e1 ? ld_stream(A.vals + e) : T(0);
        }
        T s = T(0);
#pragma unroll
        for (int q = 0; q < IL; ++q) {
            const int e = e0 + threadIdx.x + q * TPB;
            if (e < e1) s += v[q] * ld_ro(xg + c[q]);
        }
        s = warp_sum(s);
        if ((threadIdx.x & 31) == 0) wpart[threadIdx.x >> 5] = s;
        __syncthreads();
        if (threadIdx.x == 0) {
            T t = T(0);
#pragma unroll
            for (int w = 0; w < TPB / 32; ++w) t += wpart[w];
            reinterpret_cast<T*>(A.tile_part)[blockIdx.x] = t;
            __threadfence();
            const int4 lg = A.longs[li];
            const int prev = atomicAdd(A.counters + li, 1);
            s_last = (prev == lg.z - 1);
        }
        __syncthreads();
        block_store<Epi::K>(acc, epi.part, A.ntiles + A.nlong, blockIdx.x);
        if (s_last && threadIdx.x == 0) {
            __threadfence();
            const int4 lg = A.longs[li];
            const volatile T* tp = reinterpret_cast<const volatile T*>(A.tile_part);
            T tot = T(0);
            for (int ch = 0; ch < lg.z; ++ch) tot += tp[lg.y + ch];
            A.counters[li] = 0;
            Acc<Epi::K> a1;
            a1.zero();
            typename Epi::Pre pre;
            epi.load(row, pre);
            epi.apply(row, tot, pre, a1);
            if constexpr (Epi::K > 0) {
                const int nslots = A.ntiles + A.nlong;
#pragma unroll
                for (int k = 0; k < Epi::K; ++k) epi.part[(size_t)k * nslots + A.ntiles + li] = a1.v[k];
            }
        }
    }
}

// ---------------------------------------------------------------------------
// epilogues: load(r, pre) fetches the row's operands (issued before the
// product phase), apply(r, sum, pre, acc) finishes the row.
// ---------------------------------------------------------------------------

// out[r] = (A x)[r]
template <typename T>
struct EpiStore {
    static constexpr int K = 0;
    static constexpr int SROW = 0;
    T* out;
    double* part;
    struct Pre {};
    __device__ void prepare() {}
    __device__ __forceinline__ void load(int, Pre&) const {}
    __device__ __forceinline__ void stage(unsigned char*, int, int) const {}
    __device__ __forceinline__ void unstage(const unsigned char*, int, Pre&) const {}
    __device__ __forceinline__ void apply(int r, T s, const Pre&, Acc<0>&) { out[r] = s; }
};

// power method step: out = A u, plus sum(out^2) for ||A A^T v|| (lp_kernel.py:157-158)
struct EpiPower {
    static constexpr int K = 1;
    static constexpr int SROW = 0;
    double* out;
    double* part;
    struct Pre {};
    __device__ void prepare() {}
    __device__ __forceinline__ void load(int, Pre&) const {}
    __device__ __forceinline__ void stage(unsigned char*, int, int) const {}
    __device__ __forceinline__ void unstage(const unsigned char*, int, Pre&) const {}
    __device__ __forceinline__ void apply(int r, double s, const Pre&, Acc<1>& a) {
        out[r] = s;
        a.v[0] += s * s;
    }
};

// Primal half of hpr_iterate (hprlp.py:190-192, 196, 198, 200-203), fused
// into the A^T y product: one row of A^T is one column j of the LP.
template <typename T, bool CHECK>
struct EpiPrimal {
    static constexpr int K = 0;
    const Ctrl* ctrl;
    int j_in_block;
    T *X, *Z, *XT;
    const T *AX, *AZ, *C, *LO, *UP;
    T *BX, *BZ;              // CHECK: bar iterates (work)
    double *XM, *ZM;         // CHECK: master-space bar iterates (to_master, hprlp.py:272-276)
    const double* CS;
    double* part;
    T sig, t, omt;
    double bsc, csc;
    struct Pre {
        T x, z, c, lo, up, ax, az;
    };
    __device__ void prepare() {
        const double sigma = ctrl->sigma;
        const double td = 1.0 / ((double)(ctrl->k0 + j_in_block) + 2.0);
        sig = (T)sigma;
        t = (T)td;
        omt = (T)(1.0 - td);
        bsc = ctrl->b_scale;
        csc = ctrl->c_scale;
    }
    static constexpr int SROW = 7 * sizeof(T);
    __device__ __forceinline__ void load(int j, Pre& p) const {
        p.x = X[j];
        p.z = Z[j];
        p.c = C[j];
        p.lo = LO[j];
        p.up = UP[j];
        p.ax = AX[j];
        p.az = AZ[j];
    }
    __device__ __forceinline__ void stage(unsigned char* sb, int r0, int R) const {
        constexpr int W = TILE_ROWS * sizeof(T);
        stage_vec(sb, 0 * W, (const T*)X, r0, R);
        stage_vec(sb, 1 * W, (const T*)Z, r0, R);
        stage_vec(sb, 2 * W, C, r0, R);
        stage_vec(sb, 3 * W, LO, r0, R);
        stage_vec(sb, 4 * W, UP, r0, R);
        stage_vec(sb, 5 * W, AX, r0, R);
        stage_vec(sb, 6 * W, AZ, r0, R);
    }
    __device__ __forceinline__ void unstage(const unsigned char* sb, int k, Pre& p) const {
        constexpr int W = TILE_ROWS * sizeof(T);
        p.x = unstage_vec<T>(sb, 0 * W, k);
        p.z = unstage_vec<T>(sb, 1 * W, k);
        p.c = unstage_vec<T>(sb, 2 * W, k);
        p.lo = unstage_vec<T>(sb, 3 * W, k);
        p.up = unstage_vec<T>(sb, 4 * W, k);
        p.ax = unstage_vec<T>(sb, 5 * W, k);
        p.az = unstage_vec<T>(sb, 6 * W, k);
    }
    __device__ __forceinline__ void apply(int j, T aty, const Pre& p, Acc<0>&) {
        const T g = p.x + sig * (aty - p.c);
        const T bx = np_clip(g, p.lo, p.up);
        const T bz = (bx - g) / sig;
        const T xt = T(2) * bx - p.x;
        const T zh = T(2) * bz - p.z;
        XT[j] = xt;
        X[j] = t * p.ax + omt * xt;
        Z[j] = t * p.az + omt * zh;
        if constexpr (CHECK) {
            BX[j] = bx;
            BZ[j] = bz;
            const double c = CS[j];
            XM[j] = ((double)bx * c) * bsc;
            ZM[j] = ((double)bz * csc) / c;
        }
    }
};

// Dual half of hpr_iterate (hprlp.py:193-194, 197, 202) fused into A x~.
template <typename T, bool CHECK>
struct EpiDual {
    static constexpr int K = 0;
    const Ctrl* ctrl;
    int j_in_block;
    int n_eq;
    T* Y;
    const T *AY, *RHS;
    T* BY;
    double* YM;
    const double* RS;
    double* part;
    T inv, t, omt;
    double csc;
    struct Pre {
        T y, rhs, ay;
    };
    __device__ void prepare() {
        const double td = 1.0 / ((double)(ctrl->k0 + j_in_block) + 2.0);
        inv = (T)(1.0 / (ctrl->lam * ctrl->sigma));
        t = (T)td;
        omt = (T)(1.0 - td);
        csc = ctrl->c_scale;
    }
    static constexpr int SROW = 3 * sizeof(T);
    __device__ __forceinline__ void load(int i, Pre& p) const {
        p.y = Y[i];
        p.rhs = RHS[i];
        p.ay = AY[i];
    }
    __device__ __forceinline__ void stage(unsigned char* sb, int r0, int R) const {
        constexpr int W = TILE_ROWS * sizeof(T);
        stage_vec(sb, 0 * W, (const T*)Y, r0, R);
        stage_vec(sb, 1 * W, RHS, r0, R);
        stage_vec(sb, 2 * W, AY, r0, R);
    }
    __device__ __forceinline__ void unstage(const unsigned char* sb, int k, Pre& p) const {
        constexpr int W = TILE_ROWS * sizeof(T);
        p.y = unstage_vec<T>(sb, 0 * W, k);
        p.rhs = unstage_vec<T>(sb, 1 * W, k);
        p.ay = unstage_vec<T>(sb, 2 * W, k);
    }
    __device__ __forceinline__ void apply(int i, T ax, const Pre& p, Acc<0>&) {
        const T v = p.y + inv * (p.rhs - ax);
        const T by = i >= n_eq ? np_max(v, T(0)) : v;
        const T yh = T(2) * by - p.y;
        Y[i] = t * p.ay + omt * yh;
        if constexpr (CHECK) {
            BY[i] = by;
            YM[i] = ((double)by * RS[i]) * csc;
        }
    }
};

// kkt_residual row terms on master data (hprlp.py:122-123, 105) plus the
// sigma-update ||bar_y - anchor_y|| (:438) and the finiteness test (:406-407).
template <typename T>
struct EpiCheckRows {
    static constexpr int K = KR;
    int n_eq;
    const double *YM, *RHSM;
    const T *BY, *AY;
    double* part;
    struct Pre {
        double ym, rhs;
        T by, ay;
    };
    __device__ void prepare() {}
    static constexpr int SROW = 2 * 8 + 2 * sizeof(T);
    __device__ __forceinline__ void load(int i, Pre& p) const {
        p.ym = YM[i];
        p.rhs = RHSM[i];
        p.by = BY[i];
        p.ay = AY[i];
    }
    __device__ __forceinline__ void stage(unsigned char* sb, int r0, int R) const {
        constexpr int D = TILE_ROWS * 8, W = TILE_ROWS * sizeof(T);
        stage_vec(sb, 0, YM, r0, R);
        stage_vec(sb, D, RHSM, r0, R);
        stage_vec(sb, 2 * D, BY, r0, R);
        stage_vec(sb, 2 * D + W, AY, r0, R);
    }
    __device__ __forceinline__ void unstage(const unsigned char* sb, int k, Pre& p) const {
        constexpr int D = TILE_ROWS * 8, W = TILE_ROWS * sizeof(T);
        p.ym = unstage_vec<double>(sb, 0, k);
        p.rhs = unstage_vec<double>(sb, D, k);
        p.by = unstage_vec<T>(sb, 2 * D, k);
        p.ay = unstage_vec<T>(sb, 2 * D + W, k);
    }
    __device__ __forceinline__ void apply(int i, double ax, const Pre& p, Acc<KR>& a) {
        const double v = (p.ym - ax) + p.rhs;
        const double pr = i >= n_eq ? np_max(v, 0.0) : v;
        const double pv = p.ym - pr;
        a.v[0] += pv * pv;
        a.v[1] += p.rhs * p.ym;
        const double d = (double)(p.by - p.ay);
        a.v[2] += d * d;
        a.v[3] += finite(p.by) ? 0.0 : 1.0;
    }
};

// kkt_residual column terms (hprlp.py:124-125, 108-113, 131) plus
// ||bar_x - anchor_x|| (:437) and finiteness of bar_x, bar_z.
template <typename T>
struct EpiCheckCols {
    static constexpr int K = KC;
    const double *XM, *ZM, *COSTM, *LOM, *UPM;
    const T *BX, *BZ, *AX;
    double* part;
    struct Pre {
        double xm, zm, c, lo, up;
        T bx, bz, ax;
    };
    __device__ void prepare() {}
    static constexpr int SROW = 5 * 8 + 3 * sizeof(T);
    __device__ __forceinline__ void load(int j, Pre& p) const {
        p.xm = XM[j];
        p.zm = ZM[j];
        p.c = COSTM[j];
        p.lo = LOM[j];
        p.up = UPM[j];
        p.bx = BX[j];
        p.bz = BZ[j];
        p.ax = AX[j];
    }
    __device__ __forceinline__ void stage(unsigned char* sb, int r0, int R) const {
        constexpr int D = TILE_ROWS * 8, W = TILE_ROWS * sizeof(T);
        stage_vec(sb, 0 * D, XM, r0, R);
        stage_vec(sb, 1 * D, ZM, r0, R);
        stage_vec(sb, 2 * D, COSTM, r0, R);
        stage_vec(sb, 3 * D, LOM, r0, R);
        stage_vec(sb, 4 * D, UPM, r0, R);
        stage_vec(sb, 5 * D, BX, r0, R);
        stage_vec(sb, 5 * D + W, BZ, r0, R);
        stage_vec(sb, 5 * D + 2 * W, AX, r0, R);
    }
    __device__ __forceinline__ void unstage(const unsigned char* sb, int k, Pre& p) const {
        constexpr int D = TILE_ROWS * 8, W = TILE_ROWS * sizeof(T);
        p.xm = unstage_vec<double>(sb, 0 * D, k);
        p.zm = unstage_vec<double>(sb, 1 * D, k);
        p.c = unstage_vec<double>(sb, 2 * D, k);
        p.lo = unstage_vec<double>(sb, 3 * D, k);
        p.up = unstage_vec<double>(sb, 4 * D, k);
        p.bx = unstage_vec<T>(sb, 5 * D, k);
        p.bz = unstage_vec<T>(sb, 5 * D + W, k);
        p.ax = unstage_vec<T>(sb, 5 * D + 2 * W, k);
    }
    __device__ __forceinline__ void apply(int j, double aty, const Pre& p, Acc<KC>& a) {
        const double dv = (p.c - aty) - p.zm;
        const double bv = p.xm - np_clip(p.xm - p.zm, p.lo, p.up);
        a.v[0] += dv * dv;
        a.v[1] += bv * bv;
        a.v[2] += p.c * p.xm;
        a.v[3] += isfinite(p.lo) ? p.lo * np_max(p.zm, 0.0) : 0.0;
        a.v[4] += isfinite(p.up) ? p.up * np_min(p.zm, 0.0) : 0.0;
        const double d = (double)(p.bx - p.ax);
        a.v[5] += d * d;
        a.v[6] += (finite(p.bx) ? 0.0 : 1.0) + (finite(p.bz) ? 0.0 : 1.0);
    }
};

}  // namespace hpr
