// hpr_screen.cu — the device flow screen behind include/hpr_screen.h.
//
// Reference: scuckit.driver.screen_violations (pkg/src/scuckit/driver.py:165-200).
// Per contingency key it forms flows = PTDF_key (L x B) @ injections (B x T)
// (driver.py:186) and reports every (line, period) with
// |flow| - limit > tol * limit (driver.py:187-196).
//
// Shape of the work: L x B x T with T = 24..36 periods, so every PTDF element
// read from HBM feeds T FP64 multiply-adds: 2T/8 = 9 flop/byte at T = 36, above
// the FP64 : HBM balance of this chip (36.9 TF/s DMMA measured : 6.5 TB/s), so
// the product is bound by FP64 math, not HBM.  It runs on the FP64 tensor
// pipe (mma.sync m8n8k4 .f64, DMMA) fed by a three-stage cp.async pipeline:
//   * a CTA owns 128 lines; warp (wm, wn) owns lines [32 wm, 32 wm + 32) as
//     four 8-line m-tiles and NTW 8-period n-tiles (a second warp row wn = 1
//     only when T > 48);
//   * A fragments (8 lines x 4 buses) are read from the staged PTDF tile at a
//     pitch of 20 doubles, B fragments (4 buses x 8 periods) from the staged
//     injection tile: both at the two-wavefront minimum per warp load;
//   * the bus range is split S ways (grid.y), S chosen so row tiles x S fill
//     whole waves of resident CTAs; the S partial sums are added in split
//     order by the epilogue kernel, which also applies the threshold test and
//     compacts the violations (deterministic flows; the record order is not,
//     and the host sorts with the reference's key).
// A/B on one B200 at C4 (20,467 x 13,659 x 36): register-tiled DFMA kernel
// (4 lines x 12 periods per thread, broadcast injection reads) 1,243 us,
// FP64 pipe 49% busy; this DMMA kernel 718 us (76% of the measured DMMA peak).
// The tables stay resident (PtdfTable is immutable, instance.py:141-164),
// padded to a bus pitch that is a multiple of 16 with zero columns.

#include <cuda_runtime.h>

#include "hpr_device_scope.h"

#include <algorithm>
#include <cmath>
#include <string>

#include "../../include/hpr_screen.h"
#include "../../include/hprlp_b200.h"

void hpr_internal_set_error(const char* msg);  // hpr_engine.cu (hpr_last_error)

namespace {

constexpr int ROWS = 128;         // lines per CTA (4 warps x 32)
#ifndef SCREEN_KB
#define SCREEN_KB 16
#endif
#ifndef SCREEN_STAGES
#define SCREEN_STAGES 3
#endif
constexpr int KB = SCREEN_KB;          // buses per pipeline stage
constexpr int STAGES = SCREEN_STAGES;

struct ScreenErr {
    int code;
};

void fail(int code, const std::string& msg) {
    hpr_internal_set_error(msg.c_str());
    throw ScreenErr{code};
}

#define SCK(call)                                                                        \
    do {                                                                                 \
        cudaError_t e_ = (call);                                                         \
        if (e_ != cudaSuccess)                                                           \
            fail(HPR_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_));      \
    } while (0)

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N> __device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// Tensor-core form (DMMA, mma.sync m8n8k4 FP64): a warp owns 32 lines (4 m-tiles)
// x NTW period tiles of 8; four warps cover the CTA's 128 lines, and a second
// warp row takes period tiles NTW.. when T > 8 * NTW.  Fragments come straight
// from the staged tiles: A (8 lines x 4 buses) at a pitch of 20 doubles and
// B (4 buses x 8 periods) from the injection tile, both at the minimum two
// wavefronts per load.
constexpr int MPP = KB + 4;
#ifndef SCREEN_WARP_MT
#define SCREEN_WARP_MT 4     // 8-line m-tiles per warp
#endif
constexpr int WMT = SCREEN_WARP_MT;
constexpr int WM = ROWS / (8 * WMT);   // warps along the lines of a CTA
constexpr int NTW_MAX = 6;
size_t mma_smem(int ntw, int wn) {
    return (size_t)STAGES * (ROWS * MPP + KB * wn * ntw * 8) * sizeof(double);
}

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

template <int NTW>
__global__ void __launch_bounds__(256)
screen_product_mma(const double* __restrict__ tab, const double* __restrict__ inj,
                   double* __restrict__ part, int L, int Bp, int NT, int kper, int wn_count) {
    const int TP = wn_count * NTW * 8;
    const int NTHR = blockDim.x;
    extern __shared__ __align__(16) double sm[];
    double* Ps = sm;                          // STAGES x ROWS x MPP
    double* Is = sm + STAGES * ROWS * MPP;    // STAGES x KB x TP

    const int tb = blockIdx.z, split = blockIdx.y;
    const int row0 = blockIdx.x * ROWS;
    const double* T0 = tab + (size_t)tb * L * Bp;
    const int k0 = split * kper;
    const int nk = min(kper, Bp - k0) / KB;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp % WM, wn = warp / WM, g = lane >> 2, tq = lane & 3;

    auto load = [&](int stage, int kt) {
        const int kb = k0 + kt * KB;
        double* ps = Ps + stage * ROWS * MPP;
#pragma unroll 4
        for (int c = tid; c < ROWS * (KB / 2); c += NTHR) {
            const int r = c / (KB / 2), q = c % (KB / 2);
            const int gr = min(row0 + r, L - 1);
            cp_async16(ps + r * MPP + 2 * q, T0 + (size_t)gr * Bp + kb + 2 * q);
        }
        double* is = Is + stage * KB * TP;
        const double* src = inj + (size_t)kb * TP;
        for (int c = tid; c < KB * TP / 2; c += NTHR) cp_async16(is + 2 * c, src + 2 * c);
        cp_async_commit();
    };

#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
        if (s < nk) load(s, s);
        else cp_async_commit();
    }

    double acc[WMT][NTW][2];
#pragma unroll
    for (int i = 0; i < WMT; ++i)
#pragma unroll
        for (int j = 0; j < NTW; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    for (int kt = 0; kt < nk; ++kt) {
        cp_async_wait<STAGES - 2>();
        __syncthreads();
        const int nx = kt + STAGES - 1;
        if (nx < nk) load(nx % STAGES, nx);
        else cp_async_commit();
        const double* ps = Ps + (kt % STAGES) * ROWS * MPP + (wm * 8 * WMT + g) * MPP + tq;
        const double* is = Is + (kt % STAGES) * KB * TP + tq * TP + wn * NTW * 8 + g;
#pragma unroll
        for (int kk = 0; kk < KB; kk += 4) {
            double a[WMT], b[NTW];
#pragma unroll
            for (int i = 0; i < WMT; ++i) a[i] = ps[i * 8 * MPP + kk];
#pragma unroll
            for (int j = 0; j < NTW; ++j) b[j] = is[kk * TP + j * 8];
#pragma unroll
            for (int i = 0; i < WMT; ++i)
#pragma unroll
                for (int j = 0; j < NTW; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
        }
    }
    cp_async_wait<0>();

    double* out = part + ((size_t)split * NT + tb) * L * TP;
#pragma unroll
    for (int i = 0; i < WMT; ++i) {
        const int row = row0 + wm * 8 * WMT + i * 8 + g;
        if (row < L) {
#pragma unroll
            for (int j = 0; j < NTW; ++j)
                *reinterpret_cast<double2*>(out + (size_t)row * TP + (wn * NTW + j) * 8 + tq * 2) =
                    make_double2(acc[i][j][0], acc[i][j][1]);
        }
    }
}

// flows = sum of the S partials in split order; the reference's test
// excess = |flow| - limit > tol * limit (driver.py:190-191; NaN never passes).
__global__ void screen_epilogue(const double* __restrict__ part, const double* __restrict__ lim,
                                double* __restrict__ flows, int NT, int L, int T, int Tp, int S,
                                double tol, unsigned long long* cnt, long long cap,
                                int* r_tab, int* r_line, int* r_per, double* r_flow,
                                double* r_exc) {
    const long long total = (long long)NT * L * T;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const int t = (int)(idx % T);
        const long long lt = idx / T;
        const int l = (int)(lt % L), tb = (int)(lt / L);
        double f = 0.0;
        for (int s = 0; s < S; ++s) f += part[((size_t)s * NT + tb) * L * Tp + (size_t)l * Tp + t];
        flows[idx] = f;
        const double limit = lim[(size_t)tb * L + l];
        const double ex = fabs(f) - limit;
        if (ex > tol * limit) {
            const unsigned long long k = atomicAdd(cnt, 1ULL);
            if ((long long)k < cap) {
                r_tab[k] = tb;
                r_line[k] = l;
                r_per[k] = t;
                r_flow[k] = f;
                r_exc[k] = ex;
            }
        }
    }
}

// FP64 tensor-pipe ceiling: every warp runs independent DMMA chains on
// registers only (no memory traffic), so the rate is the pipe's own.
constexpr int PEAK_CHAINS = 8;
__global__ void __launch_bounds__(256) dmma_peak(double* sink, int iters) {
    double c[PEAK_CHAINS][2];
    const double a = 1.0 + 1e-9 * threadIdx.x, b = 1.0 - 1e-9 * blockIdx.x;
#pragma unroll
    for (int i = 0; i < PEAK_CHAINS; ++i) c[i][0] = c[i][1] = 0.0;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < PEAK_CHAINS; ++i) dmma(c[i][0], c[i][1], a, b);
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < PEAK_CHAINS; ++i) s += c[i][0] + c[i][1];
    if (s == 12345.678) sink[0] = s;   // keeps the chains live
}

template <int NTW>
void launch_mma(dim3 grid, int wn, cudaStream_t s, const double* tab, const double* inj,
                double* part, int L, int Bp, int NT, int kper) {
    screen_product_mma<NTW><<<grid, 32 * WM * wn, mma_smem(NTW, wn), s>>>(tab, inj, part, L, Bp, NT,
                                                                      kper, wn);
}
using MmaFn = void (*)(dim3, int, cudaStream_t, const double*, const double*, double*, int, int,
                       int, int);
const MmaFn kMma[NTW_MAX] = {launch_mma<1>, launch_mma<2>, launch_mma<3>,
                             launch_mma<4>, launch_mma<5>, launch_mma<6>};
const void* kMmaFns[NTW_MAX] = {(const void*)screen_product_mma<1>, (const void*)screen_product_mma<2>,
                                (const void*)screen_product_mma<3>, (const void*)screen_product_mma<4>,
                                (const void*)screen_product_mma<5>, (const void*)screen_product_mma<6>};

template <typename T> void dfree(T*& p) {
    if (p) cudaFree(p);
    p = nullptr;
}

}  // namespace

struct hpr_screen {
    int dev = 0, L = 0, B = 0, NT = 0, Bp = 0, sms = 0;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev[3] = {nullptr, nullptr, nullptr};
    double* tab = nullptr;   // NT x L x Bp
    double* lim = nullptr;   // NT x L
    // per-run state (sized for the largest T seen)
    int T = 0, Tp = 0, S = 1, kper = 0, ctas = 0;
    int NTW = 1, WN = 1;      // period tiles of 8 per warp, warp rows per CTA
    double tol = 0.0;
    long long cap = 0, found = 0;
    double* inj = nullptr;   // Bp x Tp, zero padded
    double* part = nullptr;  // S x NT x L x Tp
    double* flows = nullptr; // NT x L x T
    size_t inj_cap = 0, part_cap = 0, flows_cap = 0;
    unsigned long long* cnt = nullptr;
    int *r_tab = nullptr, *r_line = nullptr, *r_per = nullptr;
    double *r_flow = nullptr, *r_exc = nullptr;

    ~hpr_screen() {
        if (stream) cudaStreamSynchronize(stream);
        dfree(tab); dfree(lim); dfree(inj); dfree(part); dfree(flows); dfree(cnt);
        dfree(r_tab); dfree(r_line); dfree(r_per); dfree(r_flow); dfree(r_exc);
        for (auto& e : ev)
            if (e) cudaEventDestroy(e);
        if (stream) cudaStreamDestroy(stream);
    }

    template <typename T> void grow(T*& p, size_t& have, size_t need) {
        if (need <= have) return;
        dfree(p);
        SCK(cudaMalloc(&p, need * sizeof(T)));
        have = need;
    }

    // bus splits: row tiles x S x NT should fill whole waves of resident CTAs
    void plan() {
        int per_sm = 0;
        SCK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kMmaFns[NTW - 1], 32 * WM * WN,
                                                          mma_smem(NTW, WN)));
        if (per_sm < 1) fail(HPR_ERR_CUDA, "screen product kernel does not fit on an SM");
        ctas = per_sm;
        const long long resident = (long long)per_sm * sms;
        const long long row_tiles = (long long)(L + ROWS - 1) / ROWS * NT;
        const int stages = Bp / KB;
        const int s_max = std::max(1, std::min(32, stages / 8));  // >= 128 buses per split
        int best = 1;
        double best_eff = 0.0;
        for (int s = 1; s <= s_max; ++s) {
            const int kp = (stages + s - 1) / s;
            const int se = (stages + kp - 1) / kp;
            const long long tiles = row_tiles * se;
            const long long waves = (tiles + resident - 1) / resident;
            const double eff = (double)tiles / (double)(waves * resident);
            if (eff > best_eff + 0.02) {   // fewer splits unless clearly better
                best_eff = eff;
                best = s;
            }
        }
        const int kp = (stages + best - 1) / best;
        kper = kp * KB;
        S = (stages + kp - 1) / kp;
    }

    void launch() {
        dim3 grid((L + ROWS - 1) / ROWS, S, NT);
        kMma[NTW - 1](grid, WN, stream, tab, inj, part, L, Bp, NT, kper);
        SCK(cudaGetLastError());
    }
    void epilogue() {
        SCK(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long), stream));
        const long long total = (long long)NT * L * T;
        const int blocks = (int)std::min<long long>((total + 255) / 256, (long long)sms * 16);
        screen_epilogue<<<std::max(blocks, 1), 256, 0, stream>>>(
            part, lim, flows, NT, L, T, Tp, S, tol, cnt, cap, r_tab, r_line, r_per, r_flow, r_exc);
        SCK(cudaGetLastError());
    }
};

#define SCREEN_API_BEGIN try {
#define SCREEN_API_END                                                                   \
    }                                                                                    \
    catch (const ScreenErr& e) {                                                         \
        return e.code;                                                                   \
    }                                                                                    \
    catch (const std::exception& e) {                                                    \
        hpr_internal_set_error(e.what());                                                \
        return HPR_ERR_NOMEM;                                                            \
    }                                                                                    \
    return 0;

extern "C" int hpr_screen_create(int32_t device, int32_t n_lines, int32_t n_buses,
                                 int32_t n_tables, const double* const* tables,
                                 const double* limits, hpr_screen** out) {
    SCREEN_API_BEGIN
    if (!out || !tables || !limits) fail(HPR_ERR_INVALID, "hpr_screen_create: null argument");
    *out = nullptr;
    if (n_lines <= 0 || n_buses <= 0 || n_tables <= 0)
        fail(HPR_ERR_EMPTY, "hpr_screen_create: empty PTDF table set");
    hpr::DeviceScope dscope_(device);
    SCK(dscope_.err);
    auto* h = new hpr_screen();
    try {
        h->dev = device;
        h->L = n_lines;
        h->B = n_buses;
        h->NT = n_tables;
        h->Bp = (n_buses + KB - 1) / KB * KB;
        SCK(cudaDeviceGetAttribute(&h->sms, cudaDevAttrMultiProcessorCount, device));
        SCK(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
        for (auto& e : h->ev) SCK(cudaEventCreate(&e));
        for (int t = 1; t <= NTW_MAX; ++t) {
            SCK(cudaFuncSetAttribute(kMmaFns[t - 1], cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)mma_smem(t, 2)));
            SCK(cudaFuncSetAttribute(kMmaFns[t - 1],
                                     cudaFuncAttributePreferredSharedMemoryCarveout, 100));
        }
        const size_t per = (size_t)h->L * h->Bp;
        SCK(cudaMalloc(&h->tab, per * h->NT * sizeof(double)));
        SCK(cudaMalloc(&h->lim, (size_t)h->L * h->NT * sizeof(double)));
        SCK(cudaMemsetAsync(h->tab, 0, per * h->NT * sizeof(double), h->stream));
        for (int k = 0; k < n_tables; ++k) {
            if (!tables[k]) fail(HPR_ERR_INVALID, "hpr_screen_create: null table");
            SCK(cudaMemcpy2DAsync(h->tab + per * k, (size_t)h->Bp * sizeof(double), tables[k],
                                  (size_t)h->B * sizeof(double), (size_t)h->B * sizeof(double),
                                  h->L, cudaMemcpyDefault, h->stream));
        }
        SCK(cudaMemcpyAsync(h->lim, limits, (size_t)h->L * h->NT * sizeof(double),
                            cudaMemcpyDefault, h->stream));
        SCK(cudaMalloc(&h->cnt, sizeof(unsigned long long)));
        SCK(cudaStreamSynchronize(h->stream));
    } catch (...) {
        delete h;
        throw;
    }
    *out = h;
    SCREEN_API_END
}

extern "C" int hpr_screen_run(hpr_screen* h, const double* injections, int32_t n_periods,
                              double tol, int64_t* n_found) {
    SCREEN_API_BEGIN
    if (!h || !injections || !n_found) fail(HPR_ERR_INVALID, "hpr_screen_run: null argument");
    if (n_periods <= 0) fail(HPR_ERR_EMPTY, "hpr_screen_run: no periods");
    if (n_periods > 2 * NTW_MAX * 8)
        fail(HPR_ERR_INVALID, "hpr_screen_run: more than 96 periods per screen");
    hpr::DeviceScope dscope_(h->dev);
    SCK(dscope_.err);
    h->T = n_periods;
    const int tiles = (n_periods + 7) / 8;
    h->WN = (tiles + NTW_MAX - 1) / NTW_MAX;
    h->NTW = (tiles + h->WN - 1) / h->WN;
    h->Tp = h->WN * h->NTW * 8;
    if (32 * WM * h->WN > 256)
        fail(HPR_ERR_INVALID, "hpr_screen_run: too many periods for this build's warp tile");
    h->tol = tol;
    h->plan();
    h->grow(h->inj, h->inj_cap, (size_t)h->Bp * h->Tp);
    h->grow(h->part, h->part_cap, (size_t)h->S * h->NT * h->L * h->Tp);
    const size_t n_out = (size_t)h->NT * h->L * h->T;
    if ((long long)n_out > h->cap) {
        dfree(h->r_tab); dfree(h->r_line); dfree(h->r_per); dfree(h->r_flow); dfree(h->r_exc);
        SCK(cudaMalloc(&h->r_tab, n_out * sizeof(int)));
        SCK(cudaMalloc(&h->r_line, n_out * sizeof(int)));
        SCK(cudaMalloc(&h->r_per, n_out * sizeof(int)));
        SCK(cudaMalloc(&h->r_flow, n_out * sizeof(double)));
        SCK(cudaMalloc(&h->r_exc, n_out * sizeof(double)));
        h->cap = (long long)n_out;
    }
    h->grow(h->flows, h->flows_cap, n_out);
    SCK(cudaMemsetAsync(h->inj, 0, (size_t)h->Bp * h->Tp * sizeof(double), h->stream));
    SCK(cudaMemcpy2DAsync(h->inj, (size_t)h->Tp * sizeof(double), injections,
                          (size_t)h->T * sizeof(double), (size_t)h->T * sizeof(double), h->B,
                          cudaMemcpyDefault, h->stream));
    h->launch();
    h->epilogue();
    unsigned long long c = 0;
    SCK(cudaMemcpyAsync(&c, h->cnt, sizeof(c), cudaMemcpyDeviceToHost, h->stream));
    SCK(cudaStreamSynchronize(h->stream));
    h->found = (long long)c;
    *n_found = (int64_t)c;
    SCREEN_API_END
}

extern "C" int hpr_screen_fetch(hpr_screen* h, int32_t* table, int32_t* line, int32_t* period,
                                double* flow, double* excess) {
    SCREEN_API_BEGIN
    if (!h) fail(HPR_ERR_INVALID, "hpr_screen_fetch: null handle");
    hpr::DeviceScope dscope_(h->dev);
    SCK(dscope_.err);
    const size_t n = (size_t)h->found;
    if (n) {
        if (table) SCK(cudaMemcpyAsync(table, h->r_tab, n * 4, cudaMemcpyDefault, h->stream));
        if (line) SCK(cudaMemcpyAsync(line, h->r_line, n * 4, cudaMemcpyDefault, h->stream));
        if (period) SCK(cudaMemcpyAsync(period, h->r_per, n * 4, cudaMemcpyDefault, h->stream));
        if (flow) SCK(cudaMemcpyAsync(flow, h->r_flow, n * 8, cudaMemcpyDefault, h->stream));
        if (excess) SCK(cudaMemcpyAsync(excess, h->r_exc, n * 8, cudaMemcpyDefault, h->stream));
    }
    SCK(cudaStreamSynchronize(h->stream));
    SCREEN_API_END
}

extern "C" int hpr_screen_flows(hpr_screen* h, int32_t table, double* flows) {
    SCREEN_API_BEGIN
    if (!h || !flows) fail(HPR_ERR_INVALID, "hpr_screen_flows: null argument");
    if (h->T == 0) fail(HPR_ERR_INVALID, "hpr_screen_flows: no screen has run");
    if (table < 0 || table >= h->NT) fail(HPR_ERR_INVALID, "hpr_screen_flows: table out of range");
    hpr::DeviceScope dscope_(h->dev);
    SCK(dscope_.err);
    const size_t per = (size_t)h->L * h->T;
    SCK(cudaMemcpyAsync(flows, h->flows + per * table, per * sizeof(double), cudaMemcpyDefault,
                        h->stream));
    SCK(cudaStreamSynchronize(h->stream));
    SCREEN_API_END
}

extern "C" int hpr_screen_bench(hpr_screen* h, int32_t reps, double* us_product,
                                double* us_epilogue) {
    SCREEN_API_BEGIN
    if (!h || reps <= 0) fail(HPR_ERR_INVALID, "hpr_screen_bench: bad argument");
    if (h->T == 0) fail(HPR_ERR_INVALID, "hpr_screen_bench: no screen has run");
    hpr::DeviceScope dscope_(h->dev);
    SCK(dscope_.err);
    h->launch();  // warm
    h->epilogue();
    SCK(cudaEventRecord(h->ev[0], h->stream));
    for (int r = 0; r < reps; ++r) h->launch();
    SCK(cudaEventRecord(h->ev[1], h->stream));
    for (int r = 0; r < reps; ++r) h->epilogue();
    SCK(cudaEventRecord(h->ev[2], h->stream));
    SCK(cudaEventSynchronize(h->ev[2]));
    float a = 0, b = 0;
    SCK(cudaEventElapsedTime(&a, h->ev[0], h->ev[1]));
    SCK(cudaEventElapsedTime(&b, h->ev[1], h->ev[2]));
    if (us_product) *us_product = 1e3 * a / reps;
    if (us_epilogue) *us_epilogue = 1e3 * b / reps;
    SCREEN_API_END
}

extern "C" int hpr_screen_info_get(hpr_screen* h, hpr_screen_info* info) {
    SCREEN_API_BEGIN
    if (!h || !info) fail(HPR_ERR_INVALID, "hpr_screen_info_get: null argument");
    info->n_lines = h->L;
    info->n_buses = h->B;
    info->n_tables = h->NT;
    info->bus_pitch = h->Bp;
    info->splits = h->S;
    info->ctas_per_sm = h->ctas;
    info->table_bytes = (size_t)h->NT * h->L * h->Bp * sizeof(double);
    SCREEN_API_END
}

extern "C" int hpr_fp64_peak_bench(int32_t device, double* tflops) {
    SCREEN_API_BEGIN
    if (!tflops) fail(HPR_ERR_INVALID, "hpr_fp64_peak_bench: null argument");
    hpr::DeviceScope dscope_(device);
    SCK(dscope_.err);
    int sms = 0;
    SCK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    double* sink = nullptr;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    SCK(cudaMalloc(&sink, sizeof(double)));
    SCK(cudaEventCreate(&e0));
    SCK(cudaEventCreate(&e1));
    const int blocks = sms * 4, threads = 256, iters = 4096;
    dmma_peak<<<blocks, threads>>>(sink, 64);   // warm
    SCK(cudaGetLastError());
    SCK(cudaEventRecord(e0));
    dmma_peak<<<blocks, threads>>>(sink, iters);
    SCK(cudaEventRecord(e1));
    SCK(cudaEventSynchronize(e1));
    float ms = 0;
    SCK(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(sink);
    const double mmas = (double)blocks * (threads / 32) * iters * PEAK_CHAINS;
    *tflops = mmas * 2.0 * 8 * 8 * 4 / (ms * 1e-3) / 1e12;
    SCREEN_API_END
}

extern "C" void hpr_screen_destroy(hpr_screen* h) {
    if (!h) return;
    hpr::DeviceScope dscope_(h->dev);
    delete h;
}
