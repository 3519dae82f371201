// flow_probe.cu — standalone A/B of the dense flow-block products at C4 shape.
//
// The PTDF flow rows of the C4 LP form, per period, a dense row-major block
// (R ~ 28 folded rows x C = 21,843 columns after the engine's period-major
// relabelling; 36 periods, 19.4M FP64 values).  The engine streams them as
// 1,024-entry chunks with a per-entry x gather (A x) and as 32-column panel
// tiles (A^T y).  This probe measures, on the same synthetic block set:
//   chunk  : the engine's current chunk scheme (ld.cs values + x gathers)
//   gemv   : persistent CTAs, a ring of cp.async.bulk stages holding an
//            R x W slab of values plus its W-entry x slice (x read once per
//            slab, not once per entry), per-row slab partials
//   gemvt  : the same ring for A^T y: thread = column, sums down the slab
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o flow_probe tools/flow_probe.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                      \
    do {                                                                           \
        cudaError_t e = (x);                                                       \
        if (e != cudaSuccess) {                                                    \
            printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e));       \
            exit(1);                                                               \
        }                                                                          \
    } while (0)

struct Blk {
    long long v0;   // first value (row-major R x C, row stride C)
    int c0;         // first column
    int R, C;
    int r0;         // first output row
    int s0;         // first slab index of this block
};

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* b, int n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect(unsigned long long* b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
    asm volatile(
        "{\n.reg .pred p;\nWAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

template <typename T>
__device__ __forceinline__ T warp_sum(T s) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    return s;
}

__device__ __forceinline__ double ld_cs(const double* p) {
    double v;
    asm volatile("ld.global.cs.L2::256B.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ double ld_l1(const double* p) {
    double v;
    asm volatile("ld.global.nc.L1::evict_last.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}

// ---- chunk scheme (the engine's current A x on index-free flow chunks) ----
__global__ void __launch_bounds__(128, 16)
k_chunk(const double* vals, const double* x, const int4* chunks, double* part) {
    const int4 ch = chunks[blockIdx.x];   // {v0 lo, v0 hi, len, c0}
    const long long v0 = (long long)(unsigned)ch.x | ((long long)ch.y << 32);
    const int len = ch.z, c0 = ch.w;
    double v[8], g[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const int e = threadIdx.x + q * 128;
        v[q] = e < len ? ld_cs(vals + v0 + e) : 0.0;
        g[q] = e < len ? ld_l1(x + c0 + e) : 0.0;
    }
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q) s += v[q] * g[q];
    __shared__ double w[4];
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) w[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) part[blockIdx.x] = (w[0] + w[1]) + (w[2] + w[3]);
}

// ---- slab ring: A x (per-row slab partials) ----
template <int W, int RMAX, int S, int NT>
__global__ void __launch_bounds__(NT, 1)
k_gemv(const double* vals, const double* x, const Blk* blks, int nblk, const int2* slabs,
       int nslab, double* part) {
    extern __shared__ __align__(128) unsigned char smem[];
    double* sv = reinterpret_cast<double*>(smem);                 // S x RMAX x W
    double* sx = sv + (size_t)S * RMAX * W;                        // S x W
    __shared__ __align__(8) unsigned long long full[S];
    const int tid = threadIdx.x;
    if (tid == 0) {
        for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](int k, int st) {   // slab k into stage st
        const int2 sl = slabs[k];        // {block, col offset}
        const Blk b = blks[sl.x];
        const int w = min(W, b.C - sl.y);
        const unsigned bytes = (unsigned)w * 8u;
        mbar_expect(&full[st], bytes * (b.R + 1));
        for (int r = 0; r < b.R; ++r)
            bulk_g2s(sv + ((size_t)st * RMAX + r) * W, vals + b.v0 + (long long)r * b.C + sl.y, bytes,
                     &full[st]);
        bulk_g2s(sx + (size_t)st * W, x + b.c0 + sl.y, bytes, &full[st]);
    };
    int k0 = blockIdx.x;
    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            const int k = k0 + s * gridDim.x;
            if (k < nslab) issue(k, s);
        }
    }
    const int lane = tid & 31, warp = tid >> 5;
    constexpr int NW = NT / 32;
    int it = 0;
    for (int k = k0; k < nslab; k += gridDim.x, ++it) {
        const int st = it % S;
        const unsigned par = (it / S) & 1;
        const int2 sl = slabs[k];
        const Blk b = blks[sl.x];
        const int w = min(W, b.C - sl.y);
        mbar_wait(&full[st], par);
        const double* xv = sx + (size_t)st * W;
        for (int r = warp; r < b.R; r += NW) {
            const double* rv = sv + ((size_t)st * RMAX + r) * W;
            double s = 0.0;
#pragma unroll
            for (int c = lane; c < W; c += 32)
                if (c < w) s += rv[c] * xv[c];
            s = warp_sum(s);
            if (lane == 0) part[(size_t)(b.r0 + r) * 1024 + (k - b.s0)] = s;
        }
        __syncthreads();
        if (tid == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            const int kn = k + S * gridDim.x;
            if (kn < nslab) issue(kn, st);
        }
    }
}

// ---- slab ring: A^T y (thread = column) ----
template <int W, int RMAX, int S>
__global__ void __launch_bounds__(W, 1)
k_gemvt(const double* vals, const double* y, const Blk* blks, const int2* slabs, int nslab,
        double* out) {
    extern __shared__ __align__(128) unsigned char smem[];
    double* sv = reinterpret_cast<double*>(smem);
    __shared__ __align__(8) unsigned long long full[S];
    const int tid = threadIdx.x;
    if (tid == 0) {
        for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](int k, int st) {
        const int2 sl = slabs[k];
        const Blk b = blks[sl.x];
        const int w = min(W, b.C - sl.y);
        const unsigned bytes = (unsigned)w * 8u;
        mbar_expect(&full[st], bytes * b.R);
        for (int r = 0; r < b.R; ++r)
            bulk_g2s(sv + ((size_t)st * RMAX + r) * W, vals + b.v0 + (long long)r * b.C + sl.y, bytes,
                     &full[st]);
    };
    if (tid == 0)
        for (int s = 0; s < S; ++s) {
            const int k = blockIdx.x + s * gridDim.x;
            if (k < nslab) issue(k, s);
        }
    int it = 0;
    for (int k = blockIdx.x; k < nslab; k += gridDim.x, ++it) {
        const int st = it % S;
        const unsigned par = (it / S) & 1;
        const int2 sl = slabs[k];
        const Blk b = blks[sl.x];
        const int w = min(W, b.C - sl.y);
        const double* yb = y + b.r0;
        mbar_wait(&full[st], par);
        if (tid < w) {
            const double* cv = sv + (size_t)st * RMAX * W + tid;
            double s = 0.0;
            for (int r = 0; r < b.R; ++r) s += cv[(size_t)r * W] * __ldg(yb + r);
            out[b.c0 + sl.y + tid] = s;
        }
        __syncthreads();
        if (tid == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            const int kn = k + S * gridDim.x;
            if (kn < nslab) issue(kn, st);
        }
    }
}

// ---- current panel scheme for A^T y: lane = column, warp = every 4th row, 6-row batches ----
__global__ void __launch_bounds__(128, 16)
k_panel(const double* vals, const double* y, const int4* tiles, double* out, int C) {
    const int4 t = tiles[blockIdx.x];   // {base lo, base hi, R, out col}
    const long long base = (long long)(unsigned)t.x | ((long long)t.y << 32);
    const int R = t.z, col = t.w;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __shared__ double pp[4][32];
    double s = 0.0;
    const double* pv = vals + base + lane;
    const double* yv = y;
    int q = warp;
    for (; q + 5 * 4 < R; q += 24) {
        double v[6], g[6];
#pragma unroll
        for (int u = 0; u < 6; ++u) {
            v[u] = ld_cs(pv + (long long)(q + 4 * u) * C);
            g[u] = ld_l1(yv + q + 4 * u);
        }
#pragma unroll
        for (int u = 0; u < 6; ++u) s += v[u] * g[u];
    }
    for (; q < R; q += 4) s += ld_cs(pv + (long long)q * C) * ld_l1(yv + q);
    pp[warp][lane] = s;
    __syncthreads();
    if (threadIdx.x < 32) out[col + threadIdx.x] = (pp[0][lane] + pp[1][lane]) + (pp[2][lane] + pp[3][lane]);
}

// ---- read ceilings: how fast can the value stream alone be read? ----
__global__ void __launch_bounds__(128, 16) k_read_chunk(const double* vals, long long n, double* part) {
    const long long b = (long long)blockIdx.x * 1024;
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const long long e = b + threadIdx.x + q * 128;
        s += e < n ? ld_cs(vals + e) : 0.0;
    }
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) part[blockIdx.x * 4 + (threadIdx.x >> 5)] = s;
}
__device__ __forceinline__ double2 ld_cs2(const double* p) {
    double2 v;
    asm volatile("ld.global.cs.L2::256B.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
    return v;
}
template <int U>
__global__ void __launch_bounds__(256) k_read_persist(const double* vals, long long n, double* part) {
    double s = 0.0;
    const long long stride = (long long)gridDim.x * 256 * 2 * U;
    for (long long b = ((long long)blockIdx.x * 256 + threadIdx.x) * 2; b < n; b += stride) {
        double2 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long long e = b + (long long)u * gridDim.x * 256 * 2;
            v[u] = e + 1 < n ? ld_cs2(vals + e) : make_double2(0, 0);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) s += v[u].x + v[u].y;
    }
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) part[blockIdx.x * 8 + (threadIdx.x >> 5)] = s;
}
template <int S, int KB>
__global__ void __launch_bounds__(256, 1) k_read_tma(const double* vals, long long n, double* part) {
    extern __shared__ __align__(128) unsigned char smem[];
    double* sv = reinterpret_cast<double*>(smem);
    __shared__ __align__(8) unsigned long long full[S];
    constexpr int E = KB * 1024 / 8;
    const long long nch = n / E;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0)
        for (int s = 0; s < S; ++s) {
            const long long k = blockIdx.x + (long long)s * gridDim.x;
            if (k < nch) {
                mbar_expect(&full[s], KB * 1024);
                bulk_g2s(sv + (size_t)s * E, vals + k * E, KB * 1024, &full[s]);
            }
        }
    double acc = 0.0;
    int it = 0;
    for (long long k = blockIdx.x; k < nch; k += gridDim.x, ++it) {
        const int st = it % S;
        mbar_wait(&full[st], (it / S) & 1);
        const double* v = sv + (size_t)st * E;
        for (int e = threadIdx.x; e < E; e += 256) acc += v[e];
        __syncthreads();
        if (threadIdx.x == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            const long long kn = k + (long long)S * gridDim.x;
            if (kn < nch) {
                mbar_expect(&full[st], KB * 1024);
                bulk_g2s(sv + (size_t)st * E, vals + kn * E, KB * 1024, &full[st]);
            }
        }
    }
    acc = warp_sum(acc);
    if ((threadIdx.x & 31) == 0) part[blockIdx.x * 8 + (threadIdx.x >> 5)] = acc;
}

// ---- panel v2: thread = column over all rows (no cross-warp reduction), y in smem ----
template <int NT, int U>
__global__ void __launch_bounds__(NT) k_panel2(const double* vals, const double* y, const int4* tiles,
                                               double* out, int C) {
    const int4 t = tiles[blockIdx.x];   // {base lo, base hi, R, out col}
    const long long base = (long long)(unsigned)t.x | ((long long)t.y << 32);
    const int R = t.z, col = t.w;
    __shared__ double sy[64];
    if (threadIdx.x < R) sy[threadIdx.x] = y[threadIdx.x];
    __syncthreads();
    const double* pv = vals + base + threadIdx.x;
    double s = 0.0;
    int q = 0;
    for (; q + U <= R; q += U) {
        double v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = ld_cs(pv + (long long)(q + u) * C);
#pragma unroll
        for (int u = 0; u < U; ++u) s += v[u] * sy[q + u];
    }
    for (; q < R; ++q) s += ld_cs(pv + (long long)q * C) * sy[q];
    out[col + threadIdx.x] = s;
}

int main(int argc, char** argv) {
    const int NB = 36, C = 21856;   // rows padded to a 16-entry multiple (C4: 21,843)
    const int reps = 20;
    std::vector<Blk> blks(NB);
    srand(1);
    long long nv = 0;
    int rows = 0;
    for (int b = 0; b < NB; ++b) {
        const int R = 20 + rand() % 17;   // ~28 +- 8
        blks[b] = {nv, b * C, R, C, rows, 0};
        nv += (long long)R * C;
        rows += R;
    }
    printf("values %lld (%.1f MB), rows %d\n", nv, nv * 8 / 1e6, rows);
    double *vals, *x, *y, *part, *out;
    CK(cudaMalloc(&vals, nv * 8 + 256));
    CK(cudaMalloc(&x, (size_t)NB * C * 8 + 256));
    CK(cudaMalloc(&y, rows * 8 + 256));
    CK(cudaMalloc(&part, (size_t)rows * 1024 * 8 + (size_t)nv / 1024 * 8 + 4096));
    CK(cudaMalloc(&out, (size_t)NB * C * 8 + 256));
    {
        std::vector<double> h(nv);
        for (long long i = 0; i < nv; ++i) h[i] = ((i * 2654435761ULL) % 1000) * 1e-3 - 0.5;
        CK(cudaMemcpy(vals, h.data(), nv * 8, cudaMemcpyHostToDevice));
        std::vector<double> hx((size_t)NB * C);
        for (size_t i = 0; i < hx.size(); ++i) hx[i] = (i % 97) * 0.01;
        CK(cudaMemcpy(x, hx.data(), hx.size() * 8, cudaMemcpyHostToDevice));
        std::vector<double> hy(rows);
        for (int i = 0; i < rows; ++i) hy[i] = (i % 13) * 0.1;
        CK(cudaMemcpy(y, hy.data(), rows * 8, cudaMemcpyHostToDevice));
    }
    // chunk list
    std::vector<int4> chunks;
    for (auto& b : blks)
        for (int r = 0; r < b.R; ++r)
            for (int e = 0; e < C; e += 1024) {
                long long v0 = b.v0 + (long long)r * C + e;
                chunks.push_back({(int)(v0 & 0xffffffff), (int)(v0 >> 32), std::min(1024, C - e), b.c0 + e});
            }
    int4* dch;
    CK(cudaMalloc(&dch, chunks.size() * sizeof(int4)));
    CK(cudaMemcpy(dch, chunks.data(), chunks.size() * sizeof(int4), cudaMemcpyHostToDevice));
    // panel tiles (32 columns)
    std::vector<int4> ptiles;
    for (auto& b : blks)
        for (int c = 0; c < C; c += 32) {
            long long base = b.v0 + c;
            ptiles.push_back({(int)(base & 0xffffffff), (int)(base >> 32), b.R, b.c0 + c});
        }
    int4* dpt;
    CK(cudaMalloc(&dpt, ptiles.size() * sizeof(int4)));
    CK(cudaMemcpy(dpt, ptiles.data(), ptiles.size() * sizeof(int4), cudaMemcpyHostToDevice));

    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    int sms;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    double* flush;
    const size_t FL = 512ull << 20;
    CK(cudaMalloc(&flush, FL));
    auto timeit = [&](const char* name, double bytes, auto launch) {
        launch();
        CK(cudaGetLastError());
        CK(cudaDeviceSynchronize());
        float tot = 0.f;
        for (int i = 0; i < reps; ++i) {
            CK(cudaMemsetAsync(flush, i, FL));
            CK(cudaEventRecord(e0));
            launch();
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            float ms;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            tot += ms;
        }
        CK(cudaGetLastError());
        const double us = tot / reps * 1e3;
        printf("%-28s %8.2f us  %7.1f GB/s (%.3f of 6548)\n", name, us, bytes / us * 1e-3,
               bytes / us * 1e-3 / 6547.8);
    };
    const double vbytes = nv * 8.0;
    timeit("chunk (current A x)", vbytes + NB * C * 8.0, [&] {
        k_chunk<<<(int)chunks.size(), 128>>>(vals, x, dch, part);
    });
    timeit("panel (current A^T y)", vbytes + NB * C * 8.0, [&] {
        k_panel<<<(int)ptiles.size(), 128>>>(vals, y, dpt, out, C);
    });

    auto run_panel2 = [&](auto kern, int NT, const char* name) {
        std::vector<int4> tl;
        for (auto& b : blks)
            for (int c = 0; c < C; c += NT) {
                long long base = b.v0 + c;
                tl.push_back({(int)(base & 0xffffffff), (int)(base >> 32), b.R, b.c0 + c});
            }
        int4* dt;
        CK(cudaMalloc(&dt, tl.size() * sizeof(int4)));
        CK(cudaMemcpy(dt, tl.data(), tl.size() * sizeof(int4), cudaMemcpyHostToDevice));
        timeit(name, vbytes + NB * C * 8.0, [&] { kern<<<(int)tl.size(), NT>>>(vals, y, dt, out, C); });
        cudaFree(dt);
    };
    run_panel2(k_panel2<128, 8>, 128, "panel2 128col U8");
    run_panel2(k_panel2<128, 4>, 128, "panel2 128col U4");
    run_panel2(k_panel2<256, 8>, 256, "panel2 256col U8");
    run_panel2(k_panel2<64, 8>, 64, "panel2 64col U8");
    run_panel2(k_panel2<128, 12>, 128, "panel2 128col U12");
    run_panel2(k_panel2<32, 8>, 32, "panel2 32col U8");
    auto run_gemv = [&](auto kern, int W, int RMAX, int S, int NT, int ctas_per_sm, const char* name) {
        std::vector<int2> slabs;
        std::vector<Blk> bb = blks;
        for (int b = 0; b < NB; ++b) {
            bb[b].s0 = (int)slabs.size();
            for (int c = 0; c < C; c += W) slabs.push_back({b, c});
        }
        Blk* dbl;
        int2* dsl;
        CK(cudaMalloc(&dbl, bb.size() * sizeof(Blk)));
        CK(cudaMemcpy(dbl, bb.data(), bb.size() * sizeof(Blk), cudaMemcpyHostToDevice));
        CK(cudaMalloc(&dsl, slabs.size() * sizeof(int2)));
        CK(cudaMemcpy(dsl, slabs.data(), slabs.size() * sizeof(int2), cudaMemcpyHostToDevice));
        const size_t sm = (size_t)S * RMAX * W * 8 + (size_t)S * W * 8;
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        const int grid = sms * ctas_per_sm;
        timeit(name, vbytes + NB * C * 8.0, [&] {
            kern<<<grid, NT, sm>>>(vals, x, dbl, NB, dsl, (int)slabs.size(), part);
        });
        cudaFree(dbl);
        cudaFree(dsl);
    };
    run_gemv(k_gemv<64, 40, 4, 256>, 64, 40, 4, 256, 2, "gemv W64 S4 2cta");
    run_gemv(k_gemv<128, 40, 3, 256>, 128, 40, 3, 256, 1, "gemv W128 S3 1cta");
    run_gemv(k_gemv<64, 40, 6, 256>, 64, 40, 6, 256, 1, "gemv W64 S6 1cta");
    run_gemv(k_gemv<32, 40, 8, 256>, 32, 40, 8, 256, 2, "gemv W32 S8 2cta");
    run_gemv(k_gemv<64, 40, 3, 256>, 64, 40, 3, 256, 3, "gemv W64 S3 3cta");

    auto run_gemvt = [&](auto kern, int W, int RMAX, int S, int ctas, const char* name) {
        std::vector<int2> slabs;
        for (int b = 0; b < NB; ++b)
            for (int c = 0; c < C; c += W) slabs.push_back({b, c});
        Blk* dbl;
        int2* dsl;
        CK(cudaMalloc(&dbl, blks.size() * sizeof(Blk)));
        CK(cudaMemcpy(dbl, blks.data(), blks.size() * sizeof(Blk), cudaMemcpyHostToDevice));
        CK(cudaMalloc(&dsl, slabs.size() * sizeof(int2)));
        CK(cudaMemcpy(dsl, slabs.data(), slabs.size() * sizeof(int2), cudaMemcpyHostToDevice));
        const size_t sm = (size_t)S * RMAX * W * 8;
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        timeit(name, vbytes + NB * C * 8.0, [&] {
            kern<<<sms * ctas, W, sm>>>(vals, y, dbl, dsl, (int)slabs.size(), out);
        });
        cudaFree(dbl);
        cudaFree(dsl);
    };
    run_gemvt(k_gemvt<128, 40, 4>, 128, 40, 4, 1, "gemvt W128 S4 1cta");
    run_gemvt(k_gemvt<128, 40, 2>, 128, 40, 2, 2, "gemvt W128 S2 2cta");
    run_gemvt(k_gemvt<64, 40, 4>, 64, 40, 4, 2, "gemvt W64 S4 2cta");
    run_gemvt(k_gemvt<256, 40, 2>, 256, 40, 2, 1, "gemvt W256 S2 1cta");
    run_gemvt(k_gemvt<64, 40, 6>, 64, 40, 6, 1, "gemvt W64 S6 1cta");
    timeit("read: chunk 1024/CTA", vbytes, [&] {
        k_read_chunk<<<(int)((nv + 1023) / 1024), 128>>>(vals, nv, part);
    });
    timeit("read: persistent v2 U4 8cta", vbytes, [&] {
        k_read_persist<4><<<sms * 8, 256>>>(vals, nv, part);
    });
    timeit("read: persistent v2 U8 4cta", vbytes, [&] {
        k_read_persist<8><<<sms * 4, 256>>>(vals, nv, part);
    });
    timeit("read: persistent v2 U2 8cta", vbytes, [&] {
        k_read_persist<2><<<sms * 8, 256>>>(vals, nv, part);
    });
    {
        auto kt = k_read_tma<4, 32>;
        CK(cudaFuncSetAttribute(kt, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 32 * 1024));
        timeit("read: tma 4x32KB 1cta", vbytes, [&] { kt<<<sms, 256, 4 * 32 * 1024>>>(vals, nv, part); });
        auto kt2 = k_read_tma<3, 32>;
        CK(cudaFuncSetAttribute(kt2, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * 32 * 1024));
        timeit("read: tma 3x32KB 2cta", vbytes, [&] { kt2<<<sms * 2, 256, 3 * 32 * 1024>>>(vals, nv, part); });
        auto kt3 = k_read_tma<6, 16>;
        CK(cudaFuncSetAttribute(kt3, cudaFuncAttributeMaxDynamicSharedMemorySize, 6 * 16 * 1024));
        timeit("read: tma 6x16KB 2cta", vbytes, [&] { kt3<<<sms * 2, 256, 6 * 16 * 1024>>>(vals, nv, part); });
        auto kt4 = k_read_tma<8, 8>;
        CK(cudaFuncSetAttribute(kt4, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 8 * 1024));
        timeit("read: tma 8x8KB 3cta", vbytes, [&] { kt4<<<sms * 3, 256, 8 * 8 * 1024>>>(vals, nv, part); });
    }
    // pure copy reference
    timeit("cudaMemcpy D2D (r+w)", 2 * vbytes, [&] {
        CK(cudaMemcpyAsync(flush, vals, (size_t)nv * 8, cudaMemcpyDeviceToDevice));
    });
    return 0;
}
