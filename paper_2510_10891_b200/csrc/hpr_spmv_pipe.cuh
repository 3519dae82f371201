// hpr_spmv_pipe.cuh — persistent, TMA-pipelined variant of the tiled SpMV.
//
// Same tile schedule and epilogues as hpr_spmv.cuh, but each CTA stays
// resident and walks a fixed, strided sequence of tiles (deterministic).
// The (index, value) stream of a tile and its row-pointer segment are
// brought into shared memory by 1-D bulk tensor copies
// (cp.async.bulk ... mbarrier::complete_tx) issued PIPE_STAGES - 1 tiles
// ahead, so the HBM stream of the next tiles overlaps the L2 gathers,
// the shared-memory row reductions and the fused epilogue of the current
// one.  Products overwrite the staged values in place.
#pragma once

#include "hpr_spmv.cuh"

namespace hpr {

constexpr int PIPE_STAGES = 3;
constexpr int PIPE_CTAS_PER_SM = 2;

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "HPR_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra HPR_WAIT_%=;\n}" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar))
        : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

template <typename T>
struct PipeStage {
    int idx[TILE_NNZ + 8];
    T val[TILE_NNZ + 8];
    int ptr[TILE_ROWS + 8];
};

template <typename T>
constexpr size_t pipe_smem_bytes() {
    return sizeof(PipeStage<T>) * PIPE_STAGES + 64;
}

// Issue the bulk copies of tile `tl` into stage `st` (thread 0 only).
// Source windows are widened to 16-byte boundaries; the arrays carry
// >= 64 bytes of tail padding (hpr_engine.cu: carve).
template <typename T>
__device__ __forceinline__ void pipe_issue(const Csr<T>& A, int4 tl, PipeStage<T>* st, uint64_t* bar) {
    constexpr int VA = 16 / sizeof(T);  // values per 16 bytes
    int e0, e1;
    if (tl.y < 0) {
        e0 = tl.z;
        e1 = tl.w;
    } else {
        e0 = tl.y;
        e1 = tl.z;
    }
    const int i0 = e0 & ~3, i1 = (e1 + 3) & ~3;
    const int v0 = e0 & ~(VA - 1), v1 = (e1 + VA - 1) & ~(VA - 1);
    uint32_t bytes = (uint32_t)(i1 - i0) * 4u + (uint32_t)(v1 - v0) * (uint32_t)sizeof(T);
    int q0 = 0, q1 = 0;
    if (tl.y < 0) {
        q0 = tl.x & ~3;
        q1 = (-tl.y - 1 + 1 + 3) & ~3;
        bytes += (uint32_t)(q1 - q0) * 4u;
    }
    mbar_expect_tx(bar, bytes);
    if (i1 > i0) bulk_g2s(st->idx, A.indices + i0, (uint32_t)(i1 - i0) * 4u, bar);
    if (v1 > v0) bulk_g2s(st->val, A.vals + v0, (uint32_t)(v1 - v0) * sizeof(T), bar);
    if (q1 > q0) bulk_g2s(st->ptr, A.indptr + q0, (uint32_t)(q1 - q0) * 4u, bar);
}

template <typename T, class Epi>
__global__ void __launch_bounds__(TPB, PIPE_CTAS_PER_SM)
    k_spmv_pipe(Csr<T> A, const T* __restrict__ xg, Epi epi) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    PipeStage<T>* stages = reinterpret_cast<PipeStage<T>*>(smem_raw);
    __shared__ __align__(8) uint64_t full[PIPE_STAGES];
    __shared__ T rsum[TILE_ROWS];
    __shared__ T wpart[TPB / 32];
    __shared__ int s_last;
    constexpr int VA = 16 / sizeof(T);

    epi.prepare();
    Acc<Epi::K> acc;
    acc.zero();
    const int G = gridDim.x;
    const int ntl = A.ntiles;
    const int nmine = blockIdx.x < ntl ? (ntl - 1 - blockIdx.x) / G + 1 : 0;
    if (threadIdx.x == 0) {
        for (int s = 0; s < PIPE_STAGES; ++s) mbar_init(&full[s], 1);
        fence_mbar_init();
        for (int k = 0; k < PIPE_STAGES - 1 && k < nmine; ++k)
            pipe_issue(A, A.tiles[blockIdx.x + k * G], &stages[k], &full[k]);
    }
    __syncthreads();

    int4 tl = nmine > 0 ? A.tiles[blockIdx.x] : make_int4(0, 0, 0, 0);
    for (int k = 0; k < nmine; ++k) {
        const int sidx = k % PIPE_STAGES;
        PipeStage<T>* st = &stages[sidx];
        // keep PIPE_STAGES - 1 tiles in flight: refill the stage freed by tile k-1
        if (threadIdx.x == 0 && k + PIPE_STAGES - 1 < nmine) {
            const int kk = k + PIPE_STAGES - 1;
            fence_proxy_async();
            pipe_issue(A, A.tiles[blockIdx.x + kk * G], &stages[kk % PIPE_STAGES],
                       &full[kk % PIPE_STAGES]);
        }
        const int4 tnext = k + 1 < nmine ? A.tiles[blockIdx.x + (k + 1) * G] : tl;
        if (tl.y < 0) {
            // ---------------- stream tile {r0, -(r1+1), p0, p1} ----------------
            const int r0 = tl.x, r1 = -tl.y - 1, p0 = tl.z, cnt = tl.w - tl.z;
            const int R = r1 - r0;
            const bool own = threadIdx.x < R;
            typename Epi::Pre pre;
            if (own) epi.load(r0 + threadIdx.x, pre);
            mbar_wait(&full[sidx], (uint32_t)((k / PIPE_STAGES) & 1));
            const int* sc = st->idx + (p0 & 3);
            T* sv = st->val + (p0 & (VA - 1));
            const int* sp = st->ptr + (r0 & 3);
            int c[ITEMS];
#pragma unroll
            for (int q = 0; q < ITEMS; ++q) {
                const int e = threadIdx.x + q * TPB;
                c[q] = e < cnt ? sc[e] : 0;
            }
            T g[ITEMS];
#pragma unroll
            for (int q = 0; q < ITEMS; ++q) {
                const int e = threadIdx.x + q * TPB;
                g[q] = e < cnt ? ld_ro(xg + c[q]) : T(0);
            }
#pragma unroll
            for (int q = 0; q < ITEMS; ++q) {
                const int e = threadIdx.x + q * TPB;
                if (e < cnt) sv[e] = sv[e] * g[q];
            }
            __syncthreads();
            int L = 1;
            while (L < 32 && (L * 2) * R <= TPB && L * R < cnt) L *= 2;
            const int lane = threadIdx.x & 31;
            const int gl = threadIdx.x & (L - 1);
            const int grp = threadIdx.x / L;
            const int ngrp = TPB / L;
            const unsigned mask = L == 32 ? 0xffffffffu : (((1u << L) - 1u) << (lane & ~(L - 1)));
            for (int kr = grp; kr < R; kr += ngrp) {
                const int b = sp[kr] - p0, e = sp[kr + 1] - p0;
                T s = T(0);
                for (int q = b + gl; q < e; q += L) s += sv[q];
                for (int off = L >> 1; off > 0; off >>= 1) s += __shfl_xor_sync(mask, s, off);
                if (gl == 0) rsum[kr] = s;
            }
            __syncthreads();
            if (own) epi.apply(r0 + threadIdx.x, rsum[threadIdx.x], pre, acc);
        } else {
            // ---------------- chunk of a long row {row, e0, e1, li} ----------------
            const int row = tl.x, e0 = tl.y, e1 = tl.z, li = tl.w;
            const int cnt = e1 - e0;
            mbar_wait(&full[sidx], (uint32_t)((k / PIPE_STAGES) & 1));
            const int* sc = st->idx + (e0 & 3);
            const T* sv = st->val + (e0 & (VA - 1));
            int c[ITEMS];
#pragma unroll
            for (int q = 0; q < ITEMS; ++q) {
                const int e = threadIdx.x + q * TPB;
                c[q] = e < cnt ? sc[e] : 0;
            }
            T g[ITEMS];
#pragma unroll
            for (int q = 0; q < ITEMS; ++q) {
                const int e = threadIdx.x + q * TPB;
                g[q] = e < cnt ? ld_ro(xg + c[q]) : T(0);
            }
            T s = T(0);
#pragma unroll
            for (int q = 0; q < ITEMS; ++q) {
                const int e = threadIdx.x + q * TPB;
                if (e < cnt) s += sv[e] * g[q];
            }
            s = warp_sum(s);
            if ((threadIdx.x & 31) == 0) wpart[threadIdx.x >> 5] = s;
            __syncthreads();
            if (threadIdx.x == 0) {
                T t = T(0);
#pragma unroll
                for (int w = 0; w < TPB / 32; ++w) t += wpart[w];
                reinterpret_cast<T*>(A.tile_part)[blockIdx.x + k * G] = t;
                __threadfence();
                const int4 lg = A.longs[li];
                const int prev = atomicAdd(A.counters + li, 1);
                s_last = (prev == lg.z - 1);
            }
            __syncthreads();
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
                    const int nslots = G + A.nlong;
#pragma unroll
                    for (int q = 0; q < Epi::K; ++q) epi.part[(size_t)q * nslots + G + li] = a1.v[q];
                }
            }
        }
        __syncthreads();   // stage sidx and rsum are free again
        tl = tnext;
    }
    block_store<Epi::K>(acc, epi.part, G + A.nlong, blockIdx.x);
}

}  // namespace hpr
