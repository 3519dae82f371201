// hpr_spmv.cuh — tiled CSR SpMV with fused per-row epilogues.
//
// One kernel template serves every sparse product of the HPR path
// (A x and A^T y of hprlp.py:190,193 and kkt_residual :122,125, and the
// power method lp_kernel.py:157).  The host cuts each CSR operand into
// tiles of equal work (hpr_engine.cu: build_tiles):
//
//  * stream tile  {r0, r1, L, -1}: consecutive rows holding <= TILE_NNZ
//    nonzeros.  The CTA streams the tile's (value, index) range with fully
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

template <typename T, class Epi>
__global__ void __launch_bounds__(TPB) k_spmv(Csr<T> A, const T* __restrict__ xg, Epi epi) {
    __shared__ T prod[TILE_NNZ];
    __shared__ T wpart[TPB / 32];
    __shared__ int s_last;
    epi.prepare();
    Acc<Epi::K> acc;
    acc.zero();
    const int4 tl = A.tiles[blockIdx.x];
    if (tl.w < 0) {
        // ---------------- stream tile ----------------
        const int r0 = tl.x, r1 = tl.y, L = tl.z;
        const int p0 = A.indptr[r0];
        const int cnt = A.indptr[r1] - p0;
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
#pragma unroll
        for (int q = 0; q < ITEMS; ++q) {
            const int e = threadIdx.x + q * TPB;
            if (e < cnt) prod[e] = v[q] * ld_ro(xg + c[q]);
        }
        __syncthreads();
        const int lane = threadIdx.x & 31;
        const int gl = threadIdx.x & (L - 1);
        const int grp = threadIdx.x / L;
        const int ngrp = TPB / L;
        const unsigned mask = L == 32 ? 0xffffffffu : (((1u << L) - 1u) << (lane & ~(L - 1)));
        for (int r = r0 + grp; r < r1; r += ngrp) {
            const int b = A.indptr[r] - p0, e = A.indptr[r + 1] - p0;
            T s = T(0);
            for (int q = b + gl; q < e; q += L) s += prod[q];
            for (int off = L >> 1; off > 0; off >>= 1) s += __shfl_xor_sync(mask, s, off);
            if (gl == 0) epi.row(r, s, acc);
        }
        block_store<Epi::K>(acc, epi.part, A.ntiles + A.nlong, blockIdx.x);
    } else {
        // ---------------- chunk of a long row ----------------
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
            epi.row(row, tot, a1);
            if constexpr (Epi::K > 0) {
                const int nslots = A.ntiles + A.nlong;
#pragma unroll
                for (int k = 0; k < Epi::K; ++k) epi.part[(size_t)k * nslots + A.ntiles + li] = a1.v[k];
            }
        }
    }
}

// ---------------------------------------------------------------------------
// epilogues
// ---------------------------------------------------------------------------

// out[r] = (A x)[r]
template <typename T>
struct EpiStore {
    static constexpr int K = 0;
    T* out;
    double* part;
    __device__ void prepare() {}
    __device__ __forceinline__ void row(int r, T s, Acc<0>&) { out[r] = s; }
};

// power method step: out = A u, plus sum(out^2) for ||A A^T v|| (lp_kernel.py:157-158)
struct EpiPower {
    static constexpr int K = 1;
    double* out;
    double* part;
    __device__ void prepare() {}
    __device__ __forceinline__ void row(int r, double s, Acc<1>& a) {
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
    __device__ void prepare() {
        const double sigma = ctrl->sigma;
        const double td = 1.0 / ((double)(ctrl->k0 + j_in_block) + 2.0);
        sig = (T)sigma;
        t = (T)td;
        omt = (T)(1.0 - td);
        bsc = ctrl->b_scale;
        csc = ctrl->c_scale;
    }
    __device__ __forceinline__ void row(int j, T aty, Acc<0>&) {
        const T x = X[j];
        const T g = x + sig * (aty - C[j]);
        const T bx = np_clip(g, LO[j], UP[j]);
        const T bz = (bx - g) / sig;
        const T xt = T(2) * bx - x;
        const T zh = T(2) * bz - Z[j];
        XT[j] = xt;
        X[j] = t * AX[j] + omt * xt;
        Z[j] = t * AZ[j] + omt * zh;
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
    __device__ void prepare() {
        const double td = 1.0 / ((double)(ctrl->k0 + j_in_block) + 2.0);
        inv = (T)(1.0 / (ctrl->lam * ctrl->sigma));
        t = (T)td;
        omt = (T)(1.0 - td);
        csc = ctrl->c_scale;
    }
    __device__ __forceinline__ void row(int i, T ax, Acc<0>&) {
        const T y = Y[i];
        const T v = y + inv * (RHS[i] - ax);
        const T by = i >= n_eq ? np_max(v, T(0)) : v;
        const T yh = T(2) * by - y;
        Y[i] = t * AY[i] + omt * yh;
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
    __device__ void prepare() {}
    __device__ __forceinline__ void row(int i, double ax, Acc<KR>& a) {
        const double ym = YM[i];
        const double v = (ym - ax) + RHSM[i];
        const double pr = i >= n_eq ? np_max(v, 0.0) : v;
        const double pv = ym - pr;
        a.v[0] += pv * pv;
        a.v[1] += RHSM[i] * ym;
        const T by = BY[i];
        const double d = (double)(by - AY[i]);
        a.v[2] += d * d;
        a.v[3] += finite(by) ? 0.0 : 1.0;
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
    __device__ void prepare() {}
    __device__ __forceinline__ void row(int j, double aty, Acc<KC>& a) {
        const double xm = XM[j], zm = ZM[j];
        const double lo = LOM[j], up = UPM[j];
        const double dv = (COSTM[j] - aty) - zm;
        const double bv = xm - np_clip(xm - zm, lo, up);
        a.v[0] += dv * dv;
        a.v[1] += bv * bv;
        a.v[2] += COSTM[j] * xm;
        a.v[3] += isfinite(lo) ? lo * np_max(zm, 0.0) : 0.0;
        a.v[4] += isfinite(up) ? up * np_min(zm, 0.0) : 0.0;
        const T bx = BX[j];
        const double d = (double)(bx - AX[j]);
        a.v[5] += d * d;
        a.v[6] += (finite(bx) ? 0.0 : 1.0) + (finite(BZ[j]) ? 0.0 : 1.0);
    }
};

}  // namespace hpr
