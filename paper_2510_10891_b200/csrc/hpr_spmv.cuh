// hpr_spmv.cuh — tiled CSR SpMV (A x and A^T y of the HPR path).
//
// One kernel template serves every sparse product of the path: the two
// iteration products (hprlp.py:190,193), the master-space products of the
// KKT check (kkt_residual :122,125) and the power method (lp_kernel.py:157).
// The host cuts each CSR operand into tiles of equal work
// (hpr_engine.cu: build_tiles):
//
//  * stream tile {r0, -(r1+1), p0, p1}: consecutive rows holding <= TILE_NNZ
//    nonzeros and <= TILE_ROWS rows.  The CTA streams the tile's
//    (value, index) range with fully coalesced evict-first loads (8 loads
//    in flight per thread), gathers x (L2-resident) and stages the products
//    in shared memory; groups of L lanes then reduce one row each.  L = 1 for
//    the short structural rows, so those sums run in index order exactly like
//    scipy's csr_matvec.
//  * chunk tile {row, e0, e1, li}: one CHUNK_NNZ slice of a long row (SCUC
//    balance and PTDF flow rows, ~7K-22K nonzeros).  Each CTA reduces its
//    slice; the last CTA to finish (atomic ticket) adds the slices in chunk
//    order — deterministic — and emits the row.  A slice whose columns are
//    consecutive is streamed without its index array (taux).
//
// Kept deliberately lean (32 registers, 16 CTAs/SM of 128 threads).  The
// projection / Halpern updates run either as the epilogue `Epi::apply` of
// each row (EpiPrimal / EpiDual, hpr_update.cuh: the default up to C4 scale)
// or as separate coalesced row-wise passes (the split iteration); both give
// the same bits.
#pragma once

#include "hpr_common.cuh"

// stream tiles hand a thread's two rows to Epi::apply2 in one call
// (-DHPR_PAIR_EPI=0: row by row, for A/B)
#ifndef HPR_PAIR_EPI
#define HPR_PAIR_EPI 1
#endif

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

// ------- panel tile {r0, -(r1+1), p0, -(p1+1)}: <= TPB F^T rows sharing flow panels -------
// Remaining (indexed) entries are staged as in a stream tile.  The dense part
// is read from F's row-major values with thread = F^T row (an F column): for
// every shared flow row i, the tile's threads read one contiguous run of F's
// row i, y_i and the row's base come from shared memory, and each thread sums
// its whole column -- no cross-warp reduction, one store per row (A/B at C4
// shape, tools/flow_probe.cu: 45.0 -> 38.3 us for the flow block against the
// 32-column tiles with lane = column, warp = every 4th row).  U loads in
// flight per thread.
template <typename T, class Epi, int U>
__device__ __forceinline__ void panel_tile(const Csr<T>& A, int4 tl, int4 pd,
                                           const T* __restrict__ xg, Epi& epi, T* prod,
                                           int* sptr, Acc<Epi::K>& acc) {
    __shared__ T sy[TPB];
    __shared__ long long sb[TPB];
    const int r0 = tl.x, r1 = -tl.y - 1, p0 = tl.z, cnt = -tl.w - 1 - tl.z;
    const int R = r1 - r0;
    {
        const int* __restrict__ idx = A.indices + p0;
        const T* __restrict__ val = A.vals + p0;
        for (int e = threadIdx.x; e < cnt; e += TPB) prod[e] = ld_stream(val + e) * ld_ro(xg + ld_stream(idx + e));
        if (threadIdx.x < R) sptr[threadIdx.x] = A.indptr[r0 + threadIdx.x] - p0;
        if (threadIdx.x == 0) sptr[R] = cnt;
    }
    const int2 pi = pd.w > 0 ? make_int2(pd.x, pd.y) : A.pinfo[r0];
    const int k = threadIdx.x;
    const T* __restrict__ pv = A.pvals + (r0 + k);
    T s = T(0);
    for (int q0 = 0; q0 < pi.y; q0 += TPB) {
        const int nq = min(TPB, pi.y - q0);
        __syncthreads();               // previous chunk consumed
        if (threadIdx.x < nq) {
            const int i = pi.x + q0 + threadIdx.x;
            sy[threadIdx.x] = ld_ro(xg + i);
            sb[threadIdx.x] = pd.w > 0 ? (long long)pd.z + (long long)(q0 + threadIdx.x) * pd.w
                                       : (long long)__ldg(A.rbase + i);
        }
        __syncthreads();
        if (k < R) {
            int q = 0;
            for (; q + U <= nq; q += U) {
                T v[U];
#pragma unroll
                for (int u = 0; u < U; ++u) v[u] = ld_stream(pv + sb[q + u]);
#pragma unroll
                for (int u = 0; u < U; ++u) s += v[u] * sy[q + u];
            }
            for (; q < nq; ++q) s += ld_stream(pv + sb[q]) * sy[q];
        }
    }
    __syncthreads();                   // staged leftovers visible
    if (k < R) {
        T t = T(0);
        for (int q = sptr[k]; q < sptr[k + 1]; ++q) t += prod[q];
        epi.apply(r0 + k, t + s, acc);
    }
}

template <typename T, class Epi>
__global__ void __launch_bounds__(TPB, Epi::MIN_CTAS) k_spmv(Csr<T> A, const T* __restrict__ xg, Epi epi) {
    __shared__ T prod[TILE_NNZ];
    __shared__ int sptr[TILE_ROWS + 1];
    __shared__ T wpart[TPB / 32];
    __shared__ int s_last;
    if (A.halt && *A.halt) return;
    Acc<Epi::K> acc;
    acc.zero();
    const int4 tl = A.tiles[blockIdx.x];
    if (Epi::COL_PANELS && tl.y < 0 && tl.w < 0) {
        panel_tile<T, Epi, 8>(A, tl, A.pdesc[blockIdx.x], xg, epi, prod, sptr, acc);
        block_store<Epi::K>(acc, epi.part, A.ntiles + A.nlong, blockIdx.x);
    } else if (tl.y < 0) {
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
        // straight-line (a loop here keeps the in-flight loads live across it: spills)
        if (threadIdx.x < R) sptr[threadIdx.x] = A.indptr[r0 + threadIdx.x] - p0;
        if constexpr (TILE_ROWS > TPB) {
            if (threadIdx.x + TPB < R) sptr[threadIdx.x + TPB] = A.indptr[r0 + threadIdx.x + TPB] - p0;
        }
        if (threadIdx.x == 0) sptr[R] = cnt;
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
        bool done = false;
        if constexpr (Epi::PAIR && TILE_ROWS == 2 * TPB && HPR_PAIR_EPI) {
            if (L == 1) {
                // rows k and k + TPB of this thread: both sums (index order, as
                // the loop below), then one epilogue call for the two rows
                const int k0 = threadIdx.x, k1 = threadIdx.x + TPB;
                T s0 = T(0), s1 = T(0);
                if (k0 < R)
                    for (int q = sptr[k0]; q < sptr[k0 + 1]; ++q) s0 += prod[q];
                if (k1 < R)
                    for (int q = sptr[k1]; q < sptr[k1 + 1]; ++q) s1 += prod[q];
                epi.apply2(r0 + k0, s0, k0 < R, r0 + k1, s1, k1 < R, acc);
                done = true;
            }
        }
        if (!done) {
            for (int k = grp; k < R; k += ngrp) {
                const int b = sptr[k], e = sptr[k + 1];
                T s = T(0);
                for (int q = b + gl; q < e; q += L) s += prod[q];
                for (int off = L >> 1; off > 0; off >>= 1) s += __shfl_xor_sync(mask, s, off);
                if (gl == 0) epi.apply(r0 + k, s, acc);
            }
        }
        block_store<Epi::K>(acc, epi.part, A.ntiles + A.nlong, blockIdx.x);
    } else {
        // ---------------- chunk of a long row {row, e0, e1, li} ----------------
        const int row = tl.x, e0 = tl.y, e1 = tl.z, li = tl.w;
        // aux {c0, 1}: the chunk covers the consecutive columns c0 .. c0+len-1
        // (PTDF flow rows are dense over their period's columns), so neither
        // the index stream nor a dependent load stands between the value
        // stream and the gathers
        const int2 aux = A.taux[blockIdx.x];
        constexpr int IL = CHUNK_NNZ / TPB;
        T s = T(0);
        if (aux.y) {
            const T* __restrict__ xc = xg + aux.x - e0;
            T v[IL], g[IL];
#pragma unroll
            for (int q = 0; q < IL; ++q) {
                const int e = e0 + threadIdx.x + q * TPB;
                v[q] = e < e1 ? ld_stream(A.vals + e) : T(0);
                g[q] = e < e1 ? ld_ro(xc + e) : T(0);
            }
#pragma unroll
            for (int q = 0; q < IL; ++q) s += v[q] * g[q];
        } else {
            int c[IL];
            T v[IL];
#pragma unroll
            for (int q = 0; q < IL; ++q) {
                const int e = e0 + threadIdx.x + q * TPB;
                c[q] = e < e1 ? ld_stream(A.indices + e) : 0;
                v[q] = e < e1 ? ld_stream(A.vals + e) : T(0);
            }
#pragma unroll
            for (int q = 0; q < IL; ++q) {
                const int e = e0 + threadIdx.x + q * TPB;
                if (e < e1) s += v[q] * ld_ro(xg + c[q]);
            }
        }
        s = warp_sum(s);
        if ((threadIdx.x & 31) == 0) wpart[threadIdx.x >> 5] = s;
        __syncthreads();
        if (threadIdx.x == 0) {
            T t = T(0);
#pragma unroll
            for (int w = 0; w < TPB / 32; ++w) t += wpart[w];
            reinterpret_cast<T*>(A.tile_part)[blockIdx.x] = t;
            const int4 lg = A.longs[li];
            // release: the partial is visible before the ticket; acquire: the last
            // CTA sees every partial released before its ticket (no full fences)
            int prev;
            asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], 1;"
                         : "=r"(prev) : "l"(A.counters + li) : "memory");
            s_last = (prev == lg.z - 1);
        }
        if constexpr (Epi::K > 0) {
            // the partial-sum slots need every thread; without them only thread 0
            // (which wrote s_last itself) continues, and the other warps retire
            __syncthreads();
            block_store<Epi::K>(acc, epi.part, A.ntiles + A.nlong, blockIdx.x);
        }
        if (threadIdx.x == 0 && s_last) {
            const int4 lg = A.longs[li];
            const volatile T* tp = reinterpret_cast<const volatile T*>(A.tile_part);
            T tot = T(0);
            for (int ch = 0; ch < lg.z; ++ch) tot += tp[lg.y + ch];
            A.counters[li] = 0;
            Acc<Epi::K> a1;
            a1.zero();
            epi.apply(row, tot, a1);
            if constexpr (Epi::K > 0) {
                const int nslots = A.ntiles + A.nlong;
#pragma unroll
                for (int k = 0; k < Epi::K; ++k) epi.part[(size_t)k * nslots + A.ntiles + li] = a1.v[k];
            }
        }
    }
}

// Row panels of F (A x~ over dense flow-row groups; hpr_common.cuh Csr::gdesc),
// a kernel of their own launched ahead of k_spmv over F's other tiles (the
// rows are disjoint): with 8 CTAs/SM it may hold two rows' loads in flight
// without taking registers from the lean main product.
template <typename T, class Epi>
__global__ void __launch_bounds__(TPB, RP_MIN_CTAS) k_spmv_rows(Csr<T> A, const int4* __restrict__ rtiles,
                                                 const T* __restrict__ xg, Epi epi) {
    if (A.halt && *A.halt) return;
    __shared__ int s_last;
    const int4 tl = rtiles[blockIdx.x];
    // ------- row-panel tile {-(g+1), ct, 0, 0}: RP_COLS columns of a dense row group -------
    // Each lane holds 4 x~ values of the slab for all the group's rows
    // (x~ read once per slab, not once per entry as in a chunk tile);
    // warp w sums rows w, w+4, ... over the slab (coalesced 256-byte row
    // segments) and stores the slab partial.  The group's last tile adds
    // each row's partials in slab order -- deterministic.
    const int g = -tl.x - 1, ct = tl.y;
    const int4 gd = A.gdesc[g];           // {r0, R, c0, len}
    const int nct = (gd.w + RP_COLS - 1) / RP_COLS;
    const int cb = ct * RP_COLS;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    T* __restrict__ gp = reinterpret_cast<T*>(A.gpart) + A.gslot[g];
    T xv[RP_COLS / 32];
#pragma unroll
    for (int q = 0; q < RP_COLS / 32; ++q) {
        const int c = cb + lane + 32 * q;
        xv[q] = c < gd.w ? ld_ro(xg + gd.z + c) : T(0);
    }
    // two rows per step (8 value loads in flight per lane)
    constexpr int NW = TPB / 32;
    for (int r = warp; r < gd.y; r += 2 * NW) {
        const bool two = r + NW < gd.y;
        const T* __restrict__ rv0 = A.vals + __ldg(A.indptr + gd.x + r) + cb;
        const T* __restrict__ rv1 =
            two ? A.vals + __ldg(A.indptr + gd.x + r + NW) + cb : rv0;
        T v0[RP_COLS / 32], v1[RP_COLS / 32];
#pragma unroll
        for (int q = 0; q < RP_COLS / 32; ++q) {
            const int c = lane + 32 * q;
            const bool in = cb + c < gd.w;
            v0[q] = in ? ld_stream(rv0 + c) : T(0);
            v1[q] = in && two ? ld_stream(rv1 + c) : T(0);
        }
        T s0 = T(0), s1 = T(0);
#pragma unroll
        for (int q = 0; q < RP_COLS / 32; ++q) {
            s0 += v0[q] * xv[q];
            s1 += v1[q] * xv[q];
        }
        s0 = warp_sum(s0);
        s1 = warp_sum(s1);
        if (lane == 0) {
            gp[(size_t)r * nct + ct] = s0;
            if (two) gp[(size_t)(r + NW) * nct + ct] = s1;
        }
    }
    if (lane == 0) __threadfence();       // this warp's partials before the ticket
    __syncthreads();
    if (threadIdx.x == 0) {
        int prev;
        asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], 1;"
                     : "=r"(prev) : "l"(A.gcount + g) : "memory");
        s_last = (prev == nct - 1);
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();                      // every slab partial of the group is visible
    if (threadIdx.x == 0) A.gcount[g] = 0;
    for (int r = warp; r < gd.y; r += TPB / 32) {
        const volatile T* pr = gp + (size_t)r * nct;
        T t = T(0);
        for (int q = lane; q < nct; q += 32) t += pr[q];
        t = warp_sum(t);
        if (lane == 0) {
            Acc<Epi::K> a1;
            a1.zero();
            epi.apply(gd.x + r, t, a1);
        }
    }
}

// A/B at C5 (tools/gpu_r2w.sh, A^T y): inline 532.7 us; own kernel 16 CTAs/SM x 8 loads
// 547.0, 12 x 12 529.8, 8 x 16 488.0 (0.98 of the copy peak)
#ifndef HPR_PANEL_MIN_CTAS
#define HPR_PANEL_MIN_CTAS 8
#endif
#ifndef HPR_PANEL_U
#define HPR_PANEL_U 16
#endif
// The F^T panel tiles of a large operand as a kernel of their own, launched
// ahead of k_spmv over F^T's other tiles (the rows are disjoint); its launch
// bounds and batch depth are tuned apart from the lean main product.
template <typename T, class Epi>
__global__ void __launch_bounds__(TPB, HPR_PANEL_MIN_CTAS)
k_spmv_panels(Csr<T> A, const int4* __restrict__ ptiles, const int4* __restrict__ pdesc,
              const T* __restrict__ xg, Epi epi) {
    static_assert(Epi::K == 0, "panel kernel: no partial-sum slots");
    if (A.halt && *A.halt) return;
    __shared__ T prod[TILE_NNZ];
    __shared__ int sptr[TPB + 1];
    Acc<0> acc;
    panel_tile<T, Epi, HPR_PANEL_U>(A, ptiles[blockIdx.x], pdesc[blockIdx.x], xg, epi, prod, sptr,
                                    acc);
}

// out[r] = (A x)[r]
template <typename T>
struct EpiStore {
    static constexpr int K = 0;
    static constexpr int MIN_CTAS = 16;
    static constexpr bool ROW_PANELS = true, COL_PANELS = true;   // F and F^T
    static constexpr bool PAIR = false;
    T* out;
    double* part;
    __device__ __forceinline__ void apply(int r, T s, Acc<0>&) { out[r] = s; }
};

// power method step: out = A u, plus sum(out^2) for ||A A^T v|| (lp_kernel.py:157-158)
struct EpiPower {
    static constexpr int K = 1;
    static constexpr int MIN_CTAS = 16;
    static constexpr bool ROW_PANELS = false, COL_PANELS = false; // A and A^T
    static constexpr bool PAIR = false;
    double* out;
    double* part;
    __device__ __forceinline__ void apply(int r, double s, Acc<1>& a) {
        out[r] = s;
        a.v[0] += s * s;
    }
};

}  // namespace hpr
