// hpr_engine.cu — B200 HPR-LP engine: host orchestration, CUDA-graph
// iteration loop and the C-ABI declared in include/hprlp_b200.h.
//
// Reference path replaced: scuckit.hprlp._solve_once (hprlp.py:332-455) with
// its scaling (_ScaleMaps :210-276), power method (lp_kernel.py:138-175),
// iteration (hpr_iterate :184-207) and KKT checks (kkt_residual :116-139).
//
// Data layout in HBM (one workspace, 256-byte aligned sub-arrays):
//   A, A^T  : CSR int32 indptr/indices, FP64 master values, FP64 scaled
//             values — used for scaling, the power method and matvec
//   F, F^T  : the twin-folded operands the iteration and the check use
//             (hpr_update.cuh): int32 indptr/indices, FP64 master values,
//             FP64 + FP32 work values, gather map into the unfolded values
//   tile schedules (int4) for the four operands, long-row tickets, partials
//   master vectors (rhs, cost, lower, upper) f64, scalings rs[m], cs[n]
//   work vectors in the work dtype: x, z, x~, anchors, bars, y_fold, products
//   master bar triple and best triple (f64), check partial sums, Ctrl, log
//
// Per block of B = check_every iterations the graph body launches
//   B x { spmv(F^T, y_fold) -> p; update_primal(p); spmv(F, x~) -> p; update_dual(p) }
//   spmv(F_m, x_m), check_rows, spmv(F^T_m, y_m_fold), check_cols
//   k_controller (convergence / best / restart / sigma; sets the WHILE flag)
//   k_restart_copy (best save + anchor reset, no-op unless flagged)
// inside a conditional WHILE graph node: the host launches one graph per
// solve and waits once.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <utility>
#include <vector>

#include "hpr_common.cuh"
#include "hpr_device_scope.h"
#include "hpr_setup.cuh"
#include "hpr_spmv.cuh"
#include "hpr_update.cuh"
#include "hpr_layout.cuh"
#include "../../include/hprlp_b200.h"

using namespace hpr;

// ===========================================================================
// error plumbing
// ===========================================================================

static thread_local std::string g_err;

// shared with hpr_screen.cu so hpr_last_error() reports every entry point
void hpr_internal_set_error(const char* msg) { g_err = msg; }

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

// HPR_SYNC_DEBUG=1: synchronise after every launch outside graph capture and
// run the solve loop eagerly, so a faulting kernel is named in the error.
static bool sync_debug() {
    static const bool on = getenv("HPR_SYNC_DEBUG") != nullptr;
    return on;
}
static thread_local bool g_capturing = false;

static void ck_last(int line) {
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess && sync_debug() && !g_capturing) e = cudaDeviceSynchronize();
    if (e != cudaSuccess)
        fail(HPR_ERR_CUDA, "hpr_engine.cu:" + std::to_string(line) + ": " + cudaGetErrorString(e));
}

#define CKL() ck_last(__LINE__)

namespace {

inline int nblk(long long n, int tpb = TPB) {
    return (int)std::max<long long>(1, (n + tpb - 1) / tpb);
}

// Fused iteration: the row-wise updates run as the epilogues of the two
// products (2 kernels per iteration instead of 4; EpiPrimal / EpiDual, held to
// 32 registers so the products keep 16 CTAs/SM).  Same operations, same bits.
// Round 1 measured, per iteration: C1 21.9 -> 19.3 us, C2 + 500 triples 15.7 ->
// 13.5, C3 + 2000 triples 62.7 -> 60.4, C4 174.2 -> 174.1, and fused only below
// 20,000 tiles per product.  With the round-2 tiles (256-row stream tiles,
// column-per-thread panels) the fused pair also wins at C3 (60.7 -> 56.9 us)
// and C4 (152.0 -> 145.4 us FP64, 120.2 -> 108.3 us FP32; tools/gpu_r2aa.sh,
// r2ab.sh) and ties at C5 (1,147 vs 1,152 us), so it is the default unless the
// operand runs its row-panel or panel kernels (C5 scale).  HPR_FUSED=0/1 forces
// the choice (the partitioned mode is always split: A^T y is reduced first).
static int fused_mode() {
    static const int mode = [] {
        const char* e = getenv("HPR_FUSED");
        return e ? (e[0] == '1' ? 1 : 0) : -1;
    }();
    return mode;
}

// HPR_PLAIN=1: the single-GPU block body as a plain graph relaunched by the
// host after each block (the partitioned loop), instead of the conditional
// WHILE node (measurement aid).
static bool plain_graph() {
    static const bool on = [] {
        const char* e = getenv("HPR_PLAIN");
        return e && e[0] == '1';
    }();
    return on;
}

// cudaLaunchKernelEx wrapper (typed arguments, error check)
template <typename... KArgs, typename... Args>
void launch(void (*kern)(KArgs...), int grid, int block, cudaStream_t s, Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.stream = s;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
    if (e == cudaSuccess && sync_debug() && !g_capturing) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        const char* name = "?";
        cudaFuncGetName(&name, (const void*)kern);
        fail(HPR_ERR_CUDA, std::string("launch ") + name + ": " + cudaGetErrorString(e));
    }
}

// fixed grid of the row-wise passes: deterministic partial-sum slots
#ifndef HPR_ROW_GRID
#define HPR_ROW_GRID (148 * 8)   // A/B (tools/gpu_r2r.sh): check block 216 -> 207 us at C4 vs 148 * 32 slots
#endif
constexpr int ROW_GRID_MAX = HPR_ROW_GRID;
inline int row_grid(long long len) { return std::min(nblk(len), ROW_GRID_MAX); }

// ===========================================================================
// tile schedule
// ===========================================================================

struct Plan {
    std::vector<int4> tiles, longs;
    std::vector<int4> rtiles;     // row-panel tiles {-(g+1), column tile, 0, 0} (k_spmv_rows)
    std::vector<int4> ptiles;     // F^T panel tiles when they run as k_spmv_panels
    std::vector<int4> groups;     // row panels {r0, R, c0, len}
    std::vector<int> gslot;       // first partial slot per group
    long long nslots = 0;         // row-panel partial slots
};

// Cut a CSR into stream tiles and long-row chunks (see hpr_spmv.cuh).  With
// `rb` (F's per-row base, INT_MIN unless the row is one consecutive-column
// run), runs of >= RP_MIN_ROWS long dense rows over the same column run
// become row-panel groups instead of per-row chunks.
Plan build_tiles(const int32_t* ptr, int rows, const int2* pinfo = nullptr,
                 const int32_t* rb = nullptr, bool separate_panels = false) {
    Plan p;
    int r = 0;
    auto panel = [&](int q) { return pinfo && pinfo[q].y > 0; };
    auto same = [&](int a, int b) { return pinfo[a].x == pinfo[b].x && pinfo[a].y == pinfo[b].y; };
    auto dense_long = [&](int q) {
        return rb && rb[q] != INT_MIN && ptr[q + 1] - ptr[q] > TILE_NNZ;
    };
    auto run_of = [&](int q) { return std::make_pair(ptr[q] - rb[q], ptr[q + 1] - ptr[q]); };
    while (r < rows) {
        const int len = ptr[r + 1] - ptr[r];
        if (dense_long(r)) {
            int r1 = r + 1;
            while (r1 < rows && r1 - r < RP_ROWS && dense_long(r1) && run_of(r1) == run_of(r)) ++r1;
            if (r1 - r >= RP_MIN_ROWS) {
                const int g = (int)p.groups.size();
                const int c0 = ptr[r] - rb[r], nct = (len + RP_COLS - 1) / RP_COLS;
                p.groups.push_back(make_int4(r, r1 - r, c0, len));
                p.gslot.push_back((int)p.nslots);
                p.nslots += (long long)(r1 - r) * nct;
                for (int ct = 0; ct < nct; ++ct) p.rtiles.push_back(make_int4(-(g + 1), ct, 0, 0));
                r = r1;
                continue;
            }
        }
        if (panel(r)) {
            // panel tile: consecutive panel rows, remaining entries staged like a stream tile
            const int r0 = r;
            long long nz = 0;
            while (r < rows && r - r0 < PANEL_ROWS && panel(r) && same(r, r0)) {
                const int l = ptr[r + 1] - ptr[r];
                if (nz + l > TILE_NNZ) break;
                nz += l;
                ++r;
            }
            if (r == r0) fail(HPR_ERR_INVALID, "internal: panel row too long");
            (separate_panels ? p.ptiles : p.tiles)
                .push_back(make_int4(r0, -(r + 1), ptr[r0], -(ptr[r] + 1)));
            continue;
        }
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
        while (r < rows && r - r0 < TILE_ROWS && !panel(r)) {
            const int l = ptr[r + 1] - ptr[r];
            if (l > TILE_NNZ || nz + l > TILE_NNZ) break;
            nz += l;
            ++r;
        }
        p.tiles.push_back(make_int4(r0, -(r + 1), ptr[r0], ptr[r]));
    }
    return p;
}

// Upper bounds on the schedule of a CSR, independent of row order and folding
// (so the workspace can be sized from (m, n, nnz) alone).  A stream tile
// closes on a full row count, on nnz overflow (two consecutive tiles then hold
// more than TILE_NNZ), before a long row, or at the end.
struct TileBound {
    size_t tiles, longs;
};
TileBound tile_bound(long long rows, long long nnz, bool panels = false) {
    const long long nlong = std::min<long long>(rows, nnz / (TILE_NNZ + 1));
    // panel runs (F^T) cut stream tiles: at most one extra tile per row
    const long long t = 2 * (nnz / TILE_NNZ + 1) + rows / TILE_ROWS + 1 + 2 * nlong +
                        (nnz / CHUNK_NNZ + 1) + nlong + 2 + (panels ? rows + 1 : 0);
    return {(size_t)t, (size_t)std::max<long long>(nlong, 1)};
}

struct Carver {
    size_t off = 0;
    char* base = nullptr;
    template <typename T>
    T* take(size_t count) {
        off = (off + 255) & ~size_t(255);
        T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
        off += sizeof(T) * std::max<size_t>(count, 1) + 64;
        return p;
    }
};

}  // namespace

// A CSR operand on the device with its schedule.
struct DevCsr {
    int rows = 0, cols = 0;
    long long nnz = 0;
    int *ptr = nullptr, *idx = nullptr;
    double *mval = nullptr, *w64 = nullptr;
    float* w32 = nullptr;
    int* src = nullptr;          // folded operands: source entry in the unfolded values
    int4 *tiles = nullptr, *longs = nullptr;
    int2* taux = nullptr;
    const int2* pinfo = nullptr;  // flow panels (F^T only)
    const int* rbase = nullptr;
    int4* pdesc = nullptr;        // per tile (hpr_common.cuh Csr::pdesc)
    int ntiles = 0, nlong = 0;
    long long free_nnz = 0;      // entries in index-free chunks
    int* counters = nullptr;
    double* tpart = nullptr;
    int4* rtiles = nullptr;      // row-panel tiles (F only), launched as k_spmv_rows
    int nrtiles = 0;
    int4* ptiles = nullptr;      // F^T panel tiles launched as k_spmv_panels (large operands)
    int nptiles = 0;
    int4* gdesc = nullptr;       // row panels (F only; hpr_common.cuh Csr::gdesc)
    int* gslot = nullptr;
    int* gcount = nullptr;
    double* gpart = nullptr;
    int ngroups = 0;
    long long group_nnz = 0;
    template <typename T>
    Csr<T> view(const T* vals, const T* pvals = nullptr) const {
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
        c.halt = nullptr;
        c.taux = taux;
        c.pvals = pvals;
        c.pinfo = pinfo;
        c.rbase = rbase;
        c.pdesc = pdesc;
        c.gdesc = gdesc;
        c.gslot = gslot;
        c.gcount = gcount;
        c.gpart = gpart;
        return c;
    }
    int nslots() const { return ntiles + nlong; }
};

struct hpr_handle {
    int dev = 0;
    cudaStream_t stream = nullptr, cap = nullptr;
    bool own_stream = false;
    int m = 0, n = 0, n_eq = 0, nf = 0;
    long long nnz = 0, nnz_f = 0;
    double offset = 0.0;
    DevCsr A, AT, F, FT;
    bool folded = false;
    int* frow = nullptr;                     // nf + 1 folded-row starts
    int* rmap = nullptr;                     // m: 2 * folded row + second-of-pair
    // flow panels (hpr_layout.cuh): the dense flow block of A^T y read from F
    bool panels = false;
    int2* pinfo = nullptr;                   // n: {first folded row, count}
    int* rbase = nullptr;                    // folded rows: F entry of column 0 (INT_MIN: not dense)
    long long panel_nnz = 0, panel_cols = 0;
    // vectors (engine order)
    double *rhs_m, *cost_m, *lo_m, *up_m, *rs, *cs, *fr, *fc;
    double *rhs_w, *cost_w, *lo_w, *up_w;    // FP64 work (setup)
    void *rhsT, *costT, *loT, *upT;           // work dtype copies (FP32 mode)
    void *X, *Y, *Z, *AXv, *AYv, *AZv, *XT, *BX, *BY, *BZ, *YF, *BYF, *P;
    double *XM, *YM, *ZM, *YMF, *BXm, *BYm, *BZm;
    double *rowpart, *colpart, *red, *pw, *stage;
    Ctrl* ctrl = nullptr;
    Ctrl* h_ctrl = nullptr;
    double* h_scal = nullptr;
    unsigned long long* d_dev = nullptr;
    LogRec* log = nullptr;
    long long log_cap = 0;
    void* ws = nullptr;
    bool own_ws = false;
    size_t ws_bytes = 0;
    long long launches = 0;
    std::vector<LogRec> h_log;
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
    // cached loop graph (kernel arguments are fixed per handle)
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t gexec = nullptr;
    unsigned long long gcond = 0;
    int g_B = 0, g_prec = -1;
    LogRec* g_log = nullptr;
    long long g_per_block = 0;
    int last_prec = -1;
    bool reordered = false;
    int *rperm = nullptr, *cperm = nullptr;
    // row-partitioned mode (hpr_options.nccl_comm)
    ncclComm_t comm = nullptr;
    int world = 1, rank = 0;
    // owned column slice: A^T y is reduce-scattered, each rank
    // updates columns [c0, c0 + clen) and all-gathers x~; chunk = ceil(n / world)
    int chunk = 0, c0 = 0, clen = 0;
    int* d_flag = nullptr;                   // collective stop flag (time limit)
    int flags = 0;                           // hpr_options.flags
    bool fused = false;                      // updates as SpMV epilogues (small LPs)
    bool upd_z = false;                      // Halpern z update (hpr_iterate API only)
};

namespace {

constexpr long long LOG_CAP_MAX = 1 << 20;

// Carve every device array from one block; base == nullptr only measures.
// Folded operands are sized for the unfolded worst case.
size_t carve(hpr_handle* h, char* base) {
    Carver cv;
    cv.base = base;
    const size_t m = h->m, n = h->n, nnz = h->nnz;
    const TileBound bm = tile_bound(m, nnz), bn = tile_bound(n, nnz, true);
    auto csr = [&](DevCsr& M, size_t rows, const TileBound& tb, bool work32, bool src) {
        M.ptr = cv.take<int>(rows + 1);
        M.idx = cv.take<int>(nnz);
        M.mval = cv.take<double>(nnz);
        M.w64 = cv.take<double>(nnz);
        M.w32 = work32 ? cv.take<float>(nnz) : nullptr;
        M.src = src ? cv.take<int>(nnz) : nullptr;
        M.tiles = cv.take<int4>(tb.tiles);
        M.longs = cv.take<int4>(tb.longs);
        M.counters = cv.take<int>(tb.longs);
        M.tpart = cv.take<double>(tb.tiles);
        M.taux = cv.take<int2>(tb.tiles);
        M.pdesc = &M == &h->FT ? cv.take<int4>(tb.tiles) : nullptr;
        M.ptiles = &M == &h->FT ? cv.take<int4>(tb.tiles) : nullptr;
        if (&M == &h->F) {
            // row panels: groups of >= RP_MIN_ROWS long rows, so at most one per
            // RP_MIN_ROWS long rows; one partial per row per RP_COLS columns
            M.rtiles = cv.take<int4>(nnz / RP_COLS + tb.longs + 1);
            M.gdesc = cv.take<int4>(tb.longs);
            M.gslot = cv.take<int>(tb.longs);
            M.gcount = cv.take<int>(tb.longs);
            M.gpart = cv.take<double>(nnz / RP_COLS + tb.longs + 1);
        }
    };
    csr(h->A, m, bm, false, false);
    csr(h->AT, n, bn, false, false);
    csr(h->F, m, bm, true, true);
    csr(h->FT, n, bn, true, true);
    h->frow = cv.take<int>(m + 1);
    h->rmap = cv.take<int>(m);
    h->pinfo = cv.take<int2>(n);
    h->rbase = cv.take<int>(m);
    for (double** v : {&h->rhs_m, &h->rs, &h->fr, &h->rhs_w, &h->YM, &h->YMF, &h->BYm})
        *v = cv.take<double>(m);
    for (double** v : {&h->cost_m, &h->lo_m, &h->up_m, &h->cs, &h->fc, &h->cost_w, &h->lo_w,
                       &h->up_w, &h->XM, &h->ZM, &h->BXm, &h->BZm})
        *v = cv.take<double>(n);
    for (void** v : {&h->rhsT, &h->Y, &h->AYv, &h->BY, &h->YF, &h->BYF}) *v = cv.take<double>(m);
    for (void** v : {&h->costT, &h->loT, &h->upT, &h->X, &h->Z, &h->AXv, &h->AZv, &h->XT,
                     &h->BX, &h->BZ})
        *v = cv.take<double>(n);
    h->P = cv.take<double>(std::max(m, n));
    const size_t nslot = std::max({bm.tiles + bm.longs, bn.tiles + bn.longs, (size_t)ROW_GRID_MAX});
    h->rowpart = cv.take<double>(KR * nslot);
    h->colpart = cv.take<double>(KC * nslot);
    h->red = cv.take<double>(RED_BLOCKS + 64);
    h->pw = cv.take<double>(m + n);
    h->stage = cv.take<double>(std::max(m, n));
    h->rperm = cv.take<int>(m);
    h->cperm = cv.take<int>(n);
    h->ctrl = cv.take<Ctrl>(1);
    h->d_dev = cv.take<unsigned long long>(2);
    h->d_flag = cv.take<int>(1);
    return cv.off + 256;
}

// ===========================================================================
// device-side layout build (hpr_layout.cuh): transpose, locality ordering
// (SURVEY.md §7 hard part 5), twin folding
// ===========================================================================

// Locality ordering.  The reference lays variables out [g, t]
// (formulation.py:53-69), so a period-t flow row gathers x at stride T.
// Columns are regrouped by the first long row (> LONG_ROW nonzeros) that
// touches them — for SCUC the balance row of their period — and rows
// (equalities and inequalities separately, so the n_eq prefix is preserved)
// by their smallest new column.  Entry order inside every row of A and A^T
// stays the original one, so every row sum keeps the reference's summation
// order; only the labels move.
constexpr int LONG_ROW = 256;
constexpr int PANEL_MIN_ROW = 256;   // dense F rows that can serve a panel (PTDF flow rows)
constexpr int PANEL_MIN_RUN = 8;     // consecutive flow rows per column worth a panel

// scratch owned by one hpr_create call (stream-ordered pool allocations)
// The layout scratch comes from the device's default stream-ordered pool.  With
// the pool's default release threshold (0) every hpr_create maps its scratch
// afresh, which measured 0.04-1.3 s per C4 create on the same box
// (tools/time_e2e.py, HPR_VERBOSE phases); the pool keeps up to
// HPR_SCRATCH_KEEP_MB (default 4096; C4's layout scratch fits) mapped between
// creates instead.
void retain_scratch_pool(int dev) {
    static std::once_flag once[64];
    if (dev < 0 || dev >= 64) return;
    std::call_once(once[dev], [dev] {
        const char* e = getenv("HPR_SCRATCH_KEEP_MB");
        const unsigned long long mb = e ? strtoull(e, nullptr, 10) : 4096ull;
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) != cudaSuccess) {
            cudaGetLastError();
            return;
        }
        unsigned long long thr = mb << 20;       // the attribute is a 64-bit byte count
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        cudaGetLastError();
    });
}

struct Scratch {
    cudaStream_t s = nullptr;
    std::vector<void*> blocks;
    template <typename T>
    T* alloc(size_t count) {
        void* p = nullptr;
        CK(cudaMallocAsync(&p, sizeof(T) * std::max<size_t>(count, 1), s));
        blocks.push_back(p);
        return (T*)p;
    }
    ~Scratch() {
        if (s) cudaStreamSynchronize(s);
        for (void* p : blocks) cudaFreeAsync(p, s);
        if (s) cudaStreamSynchronize(s);
    }
};

// Host -> device upload of a pageable array through two pinned bounce
// buffers (host memcpy of chunk k+1 overlaps the DMA of chunk k); several
// times faster than a pageable cudaMemcpy for the 0.5 GB CSR of C4.
// Pageable host -> device through a pinned double buffer: host threads stage
// chunk k+1 while the DMA engine moves chunk k.  The pinned buffer is kept for
// the process (pinning 64 MB costs 30-100 ms, and releasing it sometimes
// blocks for ~0.5 s), shared by all handles under a mutex.
void upload_pageable(void* dst, const void* src, size_t bytes, cudaStream_t s) {
    constexpr size_t CH = 32u << 20;
    if (bytes < 2 * CH) {
        CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
        CK(cudaStreamSynchronize(s));
        return;
    }
    static std::mutex mu;
    static char* buf = nullptr;
    std::lock_guard<std::mutex> lock(mu);
    if (!buf) CK(cudaMallocHost(&buf, 2 * CH));
    cudaEvent_t ev[2];
    CK(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming));
    bool used[2] = {false, false};
    // the staging memcpy is split over host threads (one core moves ~2 GB/s here)
    const unsigned nth = std::max(1u, std::min(8u, std::thread::hardware_concurrency()));
    auto stage = [&](char* to, const char* from, size_t len) {
        if (nth == 1 || len < (4u << 20)) {
            std::memcpy(to, from, len);
            return;
        }
        std::vector<std::thread> th;
        const size_t part = (len + nth - 1) / nth;
        for (unsigned t = 0; t < nth; ++t) {
            const size_t o = t * part;
            if (o >= len) break;
            th.emplace_back([=] { std::memcpy(to + o, from + o, std::min(part, len - o)); });
        }
        for (auto& x : th) x.join();
    };
    for (size_t off = 0, k = 0; off < bytes; off += CH, k ^= 1) {
        const size_t len = std::min(CH, bytes - off);
        if (used[k]) CK(cudaEventSynchronize(ev[k]));
        stage(buf + k * CH, (const char*)src + off, len);
        CK(cudaMemcpyAsync((char*)dst + off, buf + k * CH, len, cudaMemcpyHostToDevice, s));
        CK(cudaEventRecord(ev[k], s));
        used[k] = true;
    }
    CK(cudaStreamSynchronize(s));
    cudaEventDestroy(ev[0]);
    cudaEventDestroy(ev[1]);
}

// exclusive scan of len[0..rows) into out[0..rows] (len[rows] must be 0)
void scan_lengths(int* len, int rows, int* out, void*& tmp, size_t& tmp_bytes, Scratch& sc,
                  cudaStream_t s) {
    size_t need = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, need, len, out, rows + 1, s));
    if (need > tmp_bytes) {
        tmp = sc.alloc<char>(need);
        tmp_bytes = need;
    }
    CK(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, len, out, rows + 1, s));
}

// stable sort of (key, value) int pairs; returns sorted values in vals_out
void sort_pairs(const int* keys_in, int* keys_out, const int* vals_in, int* vals_out, long long n,
                int end_bit, void*& tmp, size_t& tmp_bytes, Scratch& sc, cudaStream_t s) {
    if (n <= 0) return;
    size_t need = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, need, keys_in, keys_out, vals_in, vals_out,
                                       (int)n, 0, end_bit, s));
    if (need > tmp_bytes) {
        tmp = sc.alloc<char>(need);
        tmp_bytes = need;
    }
    CK(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, keys_in, keys_out, vals_in, vals_out,
                                       (int)n, 0, end_bit, s));
}

int bits_for(long long v) {
    int b = 1;
    while (b < 32 && (1LL << b) <= v) ++b;
    return b;
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

// In-place all-reduce across the ranks of a row-partitioned solve (no-op on
// one GPU).  NCCL collectives are stream-ordered and graph-capturable.
void allreduce(hpr_handle* h, void* buf, size_t count, ncclDataType_t dt, ncclRedOp_t op,
               cudaStream_t s) {
    if (!h->comm || count == 0) return;
    const ncclResult_t r = ncclAllReduce(buf, buf, count, dt, op, h->comm, s);
    if (r != ncclSuccess) fail(HPR_ERR_CUDA, std::string("ncclAllReduce: ") + ncclGetErrorString(r));
}

template <typename T>
constexpr ncclDataType_t nccl_type() {
    return sizeof(T) == 4 ? ncclFloat32 : ncclFloat64;
}

// Sum an n-vector of per-rank partials and leave each rank its owned chunk in
// place (buf + c0): ncclReduceScatter over world x chunk entries; the tail
// [n, world x chunk) is zeroed first (the products write [0, n) only).
template <typename T>
void reduce_scatter(hpr_handle* h, T* buf, cudaStream_t s) {
    if (!h->comm) return;
    const size_t npad = (size_t)h->chunk * h->world;
    if (npad > (size_t)h->n)
        CK(cudaMemsetAsync(buf + h->n, 0, sizeof(T) * (npad - h->n), s));
    const ncclResult_t r = ncclReduceScatter(buf, buf + (size_t)h->rank * h->chunk, h->chunk,
                                             nccl_type<T>(), ncclSum, h->comm, s);
    if (r != ncclSuccess)
        fail(HPR_ERR_CUDA, std::string("ncclReduceScatter: ") + ncclGetErrorString(r));
}

// Replicate an n-vector whose owned chunks are current on their ranks.
template <typename T>
void all_gather(hpr_handle* h, T* buf, cudaStream_t s) {
    if (!h->comm) return;
    const ncclResult_t r = ncclAllGather(buf + (size_t)h->rank * h->chunk, buf, h->chunk,
                                         nccl_type<T>(), h->comm, s);
    if (r != ncclSuccess)
        fail(HPR_ERR_CUDA, std::string("ncclAllGather: ") + ncclGetErrorString(r));
}

// deterministic ||v||^2 on the device -> host; row vectors (global_rows) are
// summed over the ranks of a partitioned solve, column vectors are replicated
double dev_sumsq(hpr_handle* h, const double* v, long long n, int finite_only,
                 bool global_rows = false) {
    k_sumsq_part<<<RED_BLOCKS, TPB, 0, h->stream>>>(v, n, finite_only, h->red);
    CKL();
    k_sum_slots<<<1, TPB, 0, h->stream>>>(h->red, RED_BLOCKS, 1, h->red + RED_BLOCKS);
    CKL();
    if (global_rows) allreduce(h, h->red + RED_BLOCKS, 1, ncclFloat64, ncclSum, h->stream);
    h->launches += 2;
    CK(cudaMemcpyAsync(h->h_scal, h->red + RED_BLOCKS, sizeof(double), cudaMemcpyDeviceToHost,
                       h->stream));
    CK(cudaStreamSynchronize(h->stream));
    return h->h_scal[0];
}

template <typename T, class Epi>
void launch_spmv(hpr_handle* h, const DevCsr& M, const T* vals, const T* xg, const Epi& epi,
                 cudaStream_t s, const T* pvals = nullptr, const int* halt = nullptr) {
    if (M.pinfo && !pvals) fail(HPR_ERR_INVALID, "internal: panel operand without F values");
    Csr<T> v = M.view<T>(vals, pvals);
    v.halt = halt;
    if (M.nrtiles) {             // F's dense row groups: their own kernel, rows disjoint
        if constexpr (Epi::ROW_PANELS) {
            launch(k_spmv_rows<T, Epi>, M.nrtiles, TPB, s, v, (const int4*)M.rtiles, xg, epi);
            h->launches += 1;
        } else {
            fail(HPR_ERR_INVALID, "internal: row panels on an operand without them");
        }
    }
    if (M.nptiles) {             // F^T's flow panels: their own kernel, rows disjoint
        if constexpr (Epi::COL_PANELS && Epi::K == 0) {
            launch(k_spmv_panels<T, Epi>, M.nptiles, TPB, s, v, (const int4*)M.ptiles,
                   (const int4*)M.pdesc, xg, epi);
            h->launches += 1;
        } else {
            fail(HPR_ERR_INVALID, "internal: panel kernel for this epilogue");
        }
    }
    if (M.ntiles) {
        launch(k_spmv<T, Epi>, M.ntiles, TPB, s, v, xg, epi);
        h->launches += 1;
    }
}

// power_method (lp_kernel.py:138-175) on the unfolded FP64 operand pair
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
        const double nv = std::sqrt(dev_sumsq(h, v, h->m, 0, true));
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
        allreduce(h, u, h->n, ncclFloat64, ncclSum, h->stream);
        launch_spmv(h, h->A, a_vals, (const double*)u, pwe, h->stream);    // v = A u, sum v^2
        k_sum_slots<<<1, TPB, 0, h->stream>>>(h->rowpart, h->A.nslots(), 1, h->red);
        CKL();
        allreduce(h, h->red, 1, ncclFloat64, ncclSum, h->stream);
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

// copy the scaled unfolded values into the folded operands
void refresh_folded_values(hpr_handle* h, bool fp32) {
    cudaStream_t s = h->stream;
    k_gather_vals<<<nblk(h->F.nnz), TPB, 0, s>>>(h->F.w64, h->A.w64, h->F.src, h->F.nnz);
    k_gather_vals<<<nblk(h->FT.nnz), TPB, 0, s>>>(h->FT.w64, h->AT.w64, h->FT.src, h->FT.nnz);
    CKL();
    h->launches += 2;
    if (fp32) {
        k_cast_f32<<<nblk(h->F.nnz), TPB, 0, s>>>(h->F.w64, h->F.w32, h->F.nnz);
        k_cast_f32<<<nblk(h->FT.nnz), TPB, 0, s>>>(h->FT.w64, h->FT.w32, h->FT.nnz);
        CKL();
        h->launches += 2;
    }
}

// Ruiz -> Pock-Chambolle -> normalisation on device (hprlp.py:213-264), on
// the unfolded operands so every norm sums the same terms in the same order
// as the reference.
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
            allreduce(h, h->fc, n, ncclFloat64, ncclMax, s);     // column maxima over all rows
            k_scale_factor<<<nblk(m), TPB, 0, s>>>(h->fr, h->fr, h->rs, m, h->d_dev);
            k_scale_factor<<<nblk(n), TPB, 0, s>>>(h->fc, h->fc, h->cs, n, h->d_dev + 1);
            CKL();
            h->launches += 4;
            apply();
            allreduce(h, h->d_dev, 2, ncclUint64, ncclMax, s);   // non-negative doubles as bits
            CK(cudaMemcpyAsync(h->h_scal, h->d_dev, 2 * sizeof(double), cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            if (std::max(h->h_scal[0], h->h_scal[1]) < 1e-6) break;
        }
    }
    if (prm->pock_chambolle) {
        k_row_abssum<<<nblk(m), TPB, 0, s>>>(h->A.ptr, h->A.w64, m, h->fr);
        k_row_abssum<<<nblk(n), TPB, 0, s>>>(h->AT.ptr, h->AT.w64, n, h->fc);
        allreduce(h, h->fc, n, ncclFloat64, ncclSum, s);         // column 1-norms over all rows
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
        bsc = 1.0 + std::sqrt(dev_sumsq(h, h->rhs_w, m, 1, true));
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
    T *X, *Y, *Z, *AX, *AY, *AZ, *XT, *BX, *BY, *BZ, *YF, *BYF, *P;
    const T *rhs, *cost, *lo, *up, *f_vals, *ft_vals;
};

template <typename T>
Ptrs<T> ptrs(hpr_handle* h) {
    const bool fp32 = sizeof(T) == 4;
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
    p.YF = (T*)h->YF;
    p.BYF = (T*)h->BYF;
    p.P = (T*)h->P;
    p.rhs = (const T*)(fp32 ? h->rhsT : (void*)h->rhs_w);
    p.cost = (const T*)(fp32 ? h->costT : (void*)h->cost_w);
    p.lo = (const T*)(fp32 ? h->loT : (void*)h->lo_w);
    p.up = (const T*)(fp32 ? h->upT : (void*)h->up_w);
    p.f_vals = (const T*)(fp32 ? (void*)h->F.w32 : (void*)h->F.w64);
    p.ft_vals = (const T*)(fp32 ? (void*)h->FT.w32 : (void*)h->FT.w64);
    return p;
}

// KKT residual of the master bar triple (XM, YM(F), ZM) + controller + copies
template <typename T>
void enqueue_check(hpr_handle* h, const Ptrs<T>& p, int mode, cudaStream_t s) {
    double* pd = (double*)h->P;
    EpiStore<double> st{pd, nullptr};
    // the halt flag gates the loop kernels of the queued (partitioned / plain) loop only
    const int* halt = mode == 1 && (h->comm || plain_graph()) ? &h->ctrl->halt : nullptr;
    all_gather(h, h->XM, s);          // partitioned: the owned chunks of the master bar x
    launch_spmv(h, h->F, (const double*)h->F.mval, (const double*)h->XM, st, s,
                (const double*)nullptr, halt);
    // partitioned: every rank uses the same slot counts, so the row-side sums (own
    // rows) and column-side sums (owned columns) reduce slot-wise
    const int c0 = h->comm ? h->c0 : 0, cl = h->comm ? h->clen : h->n;
    const int gr = h->comm ? ROW_GRID_MAX : row_grid(h->nf);
    const int gc = h->comm ? ROW_GRID_MAX : row_grid(h->n);
    CheckRowsArgs<T> ar{h->nf, h->n_eq, h->frow, pd, h->YM, h->rhs_m, p.BY, p.AY, h->rowpart};
    launch(k_check_rows<T>, gr, TPB, s, ar);
    allreduce(h, h->rowpart, (size_t)KR * gr, ncclFloat64, ncclSum, s);
    launch_spmv(h, h->FT, (const double*)h->FT.mval, (const double*)h->YMF, st, s,
                (const double*)h->F.mval, halt);
    reduce_scatter(h, pd, s);         // partitioned: A^T y_m on the owned columns
    CheckColsArgs<T> ac{cl, pd + c0, h->XM + c0, h->ZM + c0, h->cost_m + c0, h->lo_m + c0,
                        h->up_m + c0, p.BX + c0, p.BZ + c0, p.AX + c0, h->colpart};
    launch(k_check_cols<T>, gc, TPB, s, ac);
    allreduce(h, h->colpart, (size_t)KC * gc, ncclFloat64, ncclSum, s);
    const int* tflag = nullptr;
    if (h->comm && mode == 1) {
        // partitioned: every rank's deadline verdict, MAX-reduced on the device,
        // so the controllers (replicated, identical inputs) stop together
        launch(k_deadline_flag, 1, 1, s, (const Ctrl*)h->ctrl, h->d_flag);
        allreduce(h, h->d_flag, 1, ncclInt32, ncclMax, s);
        tflag = h->d_flag;
        h->launches += 1;
    }
    launch(k_controller, 1, CTRL_TPB, s, h->ctrl, (const double*)h->rowpart, gr,
           (const double*)h->colpart, gc, h->log, mode, tflag);
    const int len = std::max(cl, h->m);
    launch(k_restart_copy<T>, row_grid(len), TPB, s, (const Ctrl*)h->ctrl, cl, h->m, h->nf,
           (const double*)h->XM + c0, (const double*)h->YM, (const double*)h->ZM + c0,
           h->BXm + c0, h->BYm, h->BZm + c0, p.X + c0, p.Y, p.Z + c0, p.AX + c0, p.AY,
           p.AZ + c0, (const T*)p.BX + c0, (const T*)p.BY, (const T*)p.BZ + c0, p.YF,
           (const T*)p.BYF);
    h->launches += 4;
}

template <typename T, bool CHECK>
void enqueue_iteration_t(hpr_handle* h, const Ptrs<T>& p, int j, cudaStream_t s) {
    // the halt flag gates the loop kernels of the queued (partitioned / plain) loop only;
    // the conditional WHILE node stops the single-GPU loop without it
    const int* halt = h->comm || plain_graph() ? &h->ctrl->halt : nullptr;
    if (h->fused) {
        // small LPs: the row-wise updates ride on the products' epilogues (2 kernels)
        PrimalArgs<T> pa{h->ctrl, j, h->n, nullptr, p.X, p.Z, p.XT, p.AX, p.AZ, p.cost, p.lo,
                         p.up, p.BX, p.BZ, h->XM, h->ZM, h->cs, h->upd_z};
        launch_spmv(h, h->FT, p.ft_vals, (const T*)p.YF, EpiPrimal<T, CHECK>{pa, nullptr}, s,
                    p.f_vals, halt);
        DualArgs<T> da{h->ctrl, j, h->m, h->n_eq, h->rmap, nullptr, p.Y, p.AY, p.rhs, p.YF,
                       p.BY, p.BYF, h->YM, h->YMF, h->rs, h->frow};
        launch_spmv(h, h->F, p.f_vals, (const T*)p.XT, EpiDual<T, CHECK>{da, nullptr}, s,
                    (const T*)nullptr, halt);
        return;
    }
    EpiStore<T> st{p.P, nullptr};
    launch_spmv(h, h->FT, p.ft_vals, (const T*)p.YF, st, s, p.f_vals, halt);       // A^T y
    // partitioned: reduce-scatter the A^T y partials, update the
    // owned column slice, all-gather x~ for the row block's A x~
    const int c0 = h->comm ? h->c0 : 0, cl = h->comm ? h->clen : h->n;
    reduce_scatter(h, p.P, s);
    PrimalArgs<T> pa{h->ctrl, j, cl, p.P + c0, p.X + c0, p.Z + c0, p.XT + c0, p.AX + c0,
                     p.AZ + c0, p.cost + c0, p.lo + c0, p.up + c0, p.BX + c0, p.BZ + c0,
                     h->XM + c0, h->ZM + c0, h->cs + c0, h->upd_z};
    pa.halt = halt;
    launch(k_update_primal<T, CHECK>, nblk(cl), TPB, s, pa);
    all_gather(h, p.XT, s);
    launch_spmv(h, h->F, p.f_vals, (const T*)p.XT, st, s, (const T*)nullptr, halt);  // A x~
    DualArgs<T> da{h->ctrl, j, h->m, h->n_eq, h->rmap, p.P, p.Y, p.AY, p.rhs, p.YF,
                   p.BY, p.BYF, h->YM, h->YMF, h->rs};
    da.halt = halt;
    launch(k_update_dual<T, CHECK>, nblk(h->m), TPB, s, da);
    h->launches += 2;
}

template <typename T>
void enqueue_iteration(hpr_handle* h, const Ptrs<T>& p, int j, bool check, cudaStream_t s) {
    if (check) enqueue_iteration_t<T, true>(h, p, j, s);
    else enqueue_iteration_t<T, false>(h, p, j, s);
}

template <typename T>
void ensure_graph(hpr_handle* h, const Ptrs<T>& p, int B) {
    const int prec = sizeof(T) == 4 ? HPR_FP32 : HPR_FP64;
    // the log buffer is a captured kernel argument: a reallocation needs a new graph
    if (h->gexec && h->g_B == B && h->g_prec == prec && h->g_log == h->log) return;
    if (h->gexec) cudaGraphExecDestroy(h->gexec);
    if (h->graph) cudaGraphDestroy(h->graph);
    h->gexec = nullptr;
    h->graph = nullptr;
    // single GPU: WHILE(cond) { B iterations; master check; controller; copies }
    // partitioned: the same block body as a plain graph, relaunched by the
    // host after a collective stop test (the NCCL calls live in the body)
    CK(cudaGraphCreate(&h->graph, 0));
    cudaGraph_t body = h->graph;
    cudaGraphConditionalHandle cond = 0;
    if (!h->comm && !plain_graph()) {
        CK(cudaGraphConditionalHandleCreate(&cond, h->graph, 1, cudaGraphCondAssignDefault));
        cudaGraphNodeParams np = {};
        np.type = cudaGraphNodeTypeConditional;
        np.conditional.handle = cond;
        np.conditional.type = cudaGraphCondTypeWhile;
        np.conditional.size = 1;
        cudaGraphNode_t node;
        CK(cudaGraphAddNode(&node, h->graph, nullptr, 0, &np));
        body = np.conditional.phGraph_out[0];
    }
    const long long l0 = h->launches;
    CK(cudaStreamBeginCaptureToGraph(h->cap, body, nullptr, nullptr, 0,
                                     cudaStreamCaptureModeThreadLocal));
    g_capturing = true;
    try {
        for (int j = 0; j < B; ++j) enqueue_iteration<T>(h, p, j, j == B - 1, h->cap);
        enqueue_check<T>(h, p, 1, h->cap);
    } catch (...) {
        g_capturing = false;
        cudaGraph_t dummy;
        cudaStreamEndCapture(h->cap, &dummy);
        throw;
    }
    g_capturing = false;
    cudaGraph_t captured;
    CK(cudaStreamEndCapture(h->cap, &captured));
    h->g_per_block = h->launches - l0;
    h->launches = l0;
    CK(cudaGraphInstantiate(&h->gexec, h->graph, 0));
    h->gcond = (unsigned long long)cond;
    h->g_B = B;
    h->g_prec = prec;
    h->g_log = h->log;
}

// Launch the cached loop graph from the current device state; returns the
// device time of the loop (CUDA events on the handle's stream).
// Partitioned mode: one block per launch; every rank reads the (identical)
// controller status, and the wall-clock limit is agreed by a MAX all-reduce so
// no rank leaves the collective sequence alone.
bool host_sigma_update(hpr_handle* h);

// Partitioned mode (and HPR_PLAIN): the block body as a plain graph, queued
// PART_QUEUE blocks at a time with one host read of the controller per
// queue.  A check that stops the loop (tolerance, limits, or the device-side
// deadline flag MAX-reduced over the ranks) or that needs the host's sigma
// update sets Ctrl::halt, which turns the rest of the queue into no-ops; every
// rank runs the same collectives in the same order, so none is left waiting.
constexpr int PART_QUEUE = 8;

double run_loop_partitioned(hpr_handle* h, double /*time_left*/) {
    cudaStream_t s = h->stream;
    const long long t_before = h->h_ctrl->total;
    CK(cudaEventRecord(h->ev[2], s));
    while (true) {
        for (int q = 0; q < PART_QUEUE; ++q) CK(cudaGraphLaunch(h->gexec, s));
        CK(cudaMemcpyAsync(h->h_ctrl, h->ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        if (h->h_ctrl->status != -1) break;
        host_sigma_update(h);            // replicated controller: same ratio on every rank
    }
    CK(cudaEventRecord(h->ev[3], s));
    CK(cudaStreamSynchronize(s));
    h->launches += h->g_per_block * ((h->h_ctrl->total - t_before) / h->g_B);
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, h->ev[2], h->ev[3]));
    return ms * 1e-3;
}

// The restart's sigma update (hprlp.py:437-441) as Python evaluates it:
// float(np.clip(ratio ** damping, 0.25, 4.0)) with ratio from the device
// controller; Python's float ** calls the C library's pow, so this is the
// same function on the same bits.  The controller stopped the loop at the
// restart's check; returns true when the loop must be relaunched.
bool host_sigma_update(hpr_handle* h) {
    Ctrl& c = *h->h_ctrl;
    if (c.status != -1 || !c.sigma_pending) return false;
    double f = std::pow(c.sigma_ratio, c.damping);
    if (!(f >= 0.25) && f == f) f = 0.25;           // np.clip: NaN passes through
    if (!(f <= 4.0) && f == f) f = 4.0;
    c.sigma = c.sigma * f;
    c.sigma_pending = 0;
    c.halt = 0;
    cudaStream_t s = h->stream;
    CK(cudaMemcpyAsync(&h->ctrl->sigma, &c.sigma, sizeof(double), cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(&h->ctrl->sigma_pending, &c.sigma_pending, sizeof(int),
                       cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(&h->ctrl->halt, &c.halt, sizeof(int), cudaMemcpyHostToDevice, s));
    return true;
}

double run_loop_once(hpr_handle* h);

double run_loop(hpr_handle* h, double time_left = -1.0) {
    if (h->comm || plain_graph()) return run_loop_partitioned(h, time_left);
    double secs = 0.0;
    do secs += run_loop_once(h);
    while (host_sigma_update(h));
    return secs;
}

double run_loop_once(hpr_handle* h) {
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

// HPR_EAGER=1 (or HPR_SYNC_DEBUG): the block loop as plain stream launches
// with a host status read per block — for profilers that cannot look inside
// conditional graph nodes (ncu); no wall-clock deadline.  Returns device seconds.
static bool eager_loop() {
    static const bool on = getenv("HPR_EAGER") != nullptr;
    return on || sync_debug();
}

// the block loop a single-GPU solve runs: the graph holds at most MAX_B
// iterations per block; a longer check cadence (the reference takes any
// check_every) runs the same kernels as plain launches, block by block
static bool use_eager(const hpr_handle* h, long long B) {
    return !h->comm && (eager_loop() || B > MAX_B);
}

template <typename T>
double run_eager(hpr_handle* h, int B) {
    cudaStream_t s = h->stream;
    const Ptrs<T> p = ptrs<T>(h);
    unsigned long long zero = 0;
    CK(cudaMemcpyAsync(&h->ctrl->cond, &zero, sizeof(zero), cudaMemcpyHostToDevice, s));
    float total = 0.f;
    do {
        CK(cudaEventRecord(h->ev[2], s));
        for (int j = 0; j < B; ++j) enqueue_iteration<T>(h, p, j, j == B - 1, s);
        enqueue_check<T>(h, p, 1, s);
        CK(cudaEventRecord(h->ev[3], s));
        read_ctrl(h);
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, h->ev[2], h->ev[3]));
        total += ms;
        host_sigma_update(h);
    } while (h->h_ctrl->status == -1);
    return total * 1e-3;
}

void cast_work_vectors(hpr_handle* h) {
    cudaStream_t s = h->stream;
    const int m = h->m, n = h->n;
    k_cast_f32<<<nblk(m), TPB, 0, s>>>(h->rhs_w, (float*)h->rhsT, m);
    k_cast_f32<<<nblk(n), TPB, 0, s>>>(h->cost_w, (float*)h->costT, n);
    k_cast_f32<<<nblk(n), TPB, 0, s>>>(h->lo_w, (float*)h->loT, n);
    k_cast_f32<<<nblk(n), TPB, 0, s>>>(h->up_w, (float*)h->upT, n);
    CKL();
    h->launches += 4;
}

template <typename T>
void solve_typed(hpr_handle* h, const hpr_params* prm, const double* x0, const double* y0,
                 const double* z0, double* xo, double* yo, double* zo, hpr_stats* st,
                 std::chrono::steady_clock::time_point t_start) {
    const bool fp32 = sizeof(T) == 4;
    cudaStream_t s = h->stream;
    const int m = h->m, n = h->n;
    const bool verbose = getenv("HPR_VERBOSE") != nullptr;
    auto tp = std::chrono::steady_clock::now();
    auto phase = [&](const char* name) {          // host wall per phase (HPR_VERBOSE)
        if (!verbose) return;
        CK(cudaStreamSynchronize(s));
        const auto now = std::chrono::steady_clock::now();
        fprintf(stderr, "[hpr_solve] %-14s %8.1f ms\n", name,
                std::chrono::duration<double, std::milli>(now - tp).count());
        tp = now;
    };
    CK(cudaEventRecord(h->ev[0], s));

    double bsc, csc;
    scale_problem(h, prm, &bsc, &csc);
    int pits = 0, pconv = 0;
    const double lam = power_method(h, h->A.w64, h->AT.w64, prm->power_tol, prm->power_max_iter,
                                    prm->power_inflation, prm->power_start,
                                    prm->power_start_count, &pits, &pconv);
    const double rn = std::sqrt(dev_sumsq(h, h->rhs_w, m, 0, true));
    const double cn = std::sqrt(dev_sumsq(h, h->cost_w, n, 0));
    double sigma;
    if (prm->has_sigma0) sigma = prm->sigma0;
    else if (rn > 1e-12 && cn > 1e-12) sigma = rn / cn;
    else sigma = 1.0;
    phase("scale+power");
    const double rhs_norm_m = std::sqrt(dev_sumsq(h, h->rhs_m, m, 0, true));
    const double cost_norm_m = std::sqrt(dev_sumsq(h, h->cost_m, n, 0));
    refresh_folded_values(h, fp32);
    if (fp32) cast_work_vectors(h);

    // initial point (hprlp.py:357-365), warm start given in master space
    const double *dx0 = nullptr, *dy0 = nullptr, *dz0 = nullptr;
    if (x0 && y0 && z0) {
        put_vec(h, h->BXm, x0, n, false);
        put_vec(h, h->BYm, y0, m, true);
        put_vec(h, h->BZm, z0, n, false);
        dx0 = h->BXm;
        dy0 = h->BYm;
        dz0 = h->BZm;
    }
    Ptrs<T> p = ptrs<T>(h);
    k_init_cols<T><<<nblk(n), TPB, 0, s>>>(n, dx0, dz0, h->cs, bsc, csc, h->lo_w, h->up_w, p.X,
                                           p.Z, p.AX, p.AZ, p.BX, p.BZ, h->XM, h->ZM);
    k_init_rows<T><<<nblk(m), TPB, 0, s>>>(m, dy0, h->rs, csc, p.Y, p.AY, p.BY, h->YM);
    k_fold_rows<T><<<nblk(h->nf), TPB, 0, s>>>(h->nf, h->frow, p.Y, p.YF, p.BY, p.BYF, h->YM,
                                                h->YMF);
    CKL();
    h->launches += 3;

    const int B = prm->log_every_iteration ? 1 : std::max(1, prm->check_every);
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
    phase("init+check");

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
    st->loop_seconds = 0.0;
    if (status == -1) {
        double time_left = -1.0;
        if (prm->time_limit >= 0) {
            const double rem = std::max(0.0, prm->time_limit - elapsed);
            time_left = rem;
            // every rank sets its own deadline; partitioned, the flags are
            // MAX-reduced on the device before each controller (k_deadline_flag)
            k_set_deadline<<<1, 1, 0, s>>>(h->ctrl, (unsigned long long)(rem * 1e9));
            CKL();
            h->launches++;
            int one = 1;
            CK(cudaMemcpyAsync(&h->ctrl->has_deadline, &one, sizeof(int), cudaMemcpyHostToDevice, s));
        }
        if (use_eager(h, B)) {
            st->loop_seconds = run_eager<T>(h, B);
        } else {
            ensure_graph<T>(h, p, B);
            phase("graph");
            st->loop_seconds = run_loop(h, time_left);
        }
        phase("loop");
        status = h->h_ctrl->status;
        iterations = h->h_ctrl->total;
        if (status == HPR_ITERATION_LIMIT) iterations = prm->max_iterations;
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
    all_gather(h, h->BXm, s);         // partitioned: the owned chunks of the best x, z
    all_gather(h, h->BZm, s);
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
    phase("download");
}

void check_plan(const Plan& p, long long rows, long long nnz, bool panels) {
    const TileBound b = tile_bound(rows, nnz, panels);
    if (p.tiles.size() > b.tiles || p.longs.size() > b.longs)
        fail(HPR_ERR_INVALID, "internal: tile bound violated");
}

// host tile plan from the device indptr, then the chunk run flags on device
// Row panels for A x~ (hpr_spmv.cuh): measured per launch of the F product,
// chunk tiles vs row panels (tools/gpu_r2k.sh) -- C4 (25.7M entries in F,
// ~28-row groups): 56.3 vs 65.3 us; C5 (382M, 32-row groups): 622.4 vs
// 583.9 us.  The x~ reuse pays only once the dense block dominates F and the
// groups are full, so they are used from RP_MIN_NNZ entries of F on;
// HPR_ROWPANELS=0/1 forces the choice.
constexpr long long RP_MIN_NNZ = 100000000LL;
// F^T panel tiles as a kernel of their own (k_spmv_panels: 8 CTAs/SM, 16
// loads in flight per thread) from this many panel entries on; below it they
// stay inside the lean k_spmv.  A/B (tools/gpu_r2w.sh): C4 (18.65M panel
// entries) A^T y 47.2 us inline vs 55.7 as two kernels; C5 (373M) 532.7 vs
// 488.0 us.  HPR_PANELKERNEL=0/1 forces the choice.
constexpr long long PANEL_KERNEL_MIN = 100000000LL;
static bool panel_kernel_on(long long panel_nnz) {
    static const int mode = [] {
        const char* e = getenv("HPR_PANELKERNEL");
        return e ? (e[0] == '1' ? 1 : 0) : -1;
    }();
    return mode < 0 ? panel_nnz >= PANEL_KERNEL_MIN : mode == 1;
}
static bool row_panels_on(long long f_nnz) {
    static const int mode = [] {
        const char* e = getenv("HPR_ROWPANELS");
        return e ? (e[0] == '1' ? 1 : 0) : -1;
    }();
    return mode < 0 ? f_nnz >= RP_MIN_NNZ : mode == 1;
}

void plan_tiles(hpr_handle* h, DevCsr& M, int rows, int cols, long long nnz,
                const int2* d_pinfo = nullptr, const int* d_rbase = nullptr) {
    cudaStream_t s = h->stream;
    std::vector<int32_t> ptr(rows + 1);
    std::vector<int2> pinfo(d_pinfo ? rows : 0);
    std::vector<int32_t> rbh(d_rbase ? rows : 0);
    CK(cudaMemcpyAsync(ptr.data(), M.ptr, sizeof(int) * (rows + 1), cudaMemcpyDeviceToHost, s));
    if (d_pinfo && rows)
        CK(cudaMemcpyAsync(pinfo.data(), d_pinfo, sizeof(int2) * rows, cudaMemcpyDeviceToHost, s));
    if (d_rbase && rows)
        CK(cudaMemcpyAsync(rbh.data(), d_rbase, sizeof(int) * rows, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    const bool sep = d_pinfo && panel_kernel_on(h->panel_nnz);
    Plan pl = build_tiles(ptr.data(), rows, d_pinfo ? pinfo.data() : nullptr,
                          d_rbase ? rbh.data() : nullptr, sep);
    M.nptiles = (int)pl.ptiles.size();
    if (M.nptiles) {
        if (!M.ptiles || pl.ptiles.size() > tile_bound(rows, std::max<long long>(nnz, 1), true).tiles)
            fail(HPR_ERR_INVALID, "internal: panel tile bound violated");
        CK(cudaMemcpyAsync(M.ptiles, pl.ptiles.data(), sizeof(int4) * pl.ptiles.size(),
                           cudaMemcpyHostToDevice, s));
    }
    check_plan(pl, rows, std::max<long long>(nnz, 1), &M == &h->FT || &M == &h->AT);
    M.ngroups = (int)pl.groups.size();
    M.nrtiles = (int)pl.rtiles.size();
    M.group_nnz = 0;
    if (!pl.groups.empty()) {
        const TileBound b = tile_bound(rows, std::max<long long>(h->nnz, 1));
        if (!M.gdesc || pl.groups.size() > b.longs ||
            pl.nslots > h->nnz / RP_COLS + (long long)b.longs + 1)
            fail(HPR_ERR_INVALID, "internal: row-panel bound violated");
        for (const int4& g : pl.groups) M.group_nnz += (long long)g.y * g.w;
        CK(cudaMemcpyAsync(M.gdesc, pl.groups.data(), sizeof(int4) * pl.groups.size(),
                           cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(M.gslot, pl.gslot.data(), sizeof(int) * pl.gslot.size(),
                           cudaMemcpyHostToDevice, s));
        CK(cudaMemsetAsync(M.gcount, 0, sizeof(int) * pl.groups.size(), s));
        if ((long long)pl.rtiles.size() > h->nnz / RP_COLS + (long long)b.longs + 1)
            fail(HPR_ERR_INVALID, "internal: row-panel tile bound violated");
        CK(cudaMemcpyAsync(M.rtiles, pl.rtiles.data(), sizeof(int4) * pl.rtiles.size(),
                           cudaMemcpyHostToDevice, s));
    }
    M.rows = rows;
    M.cols = cols;
    M.nnz = nnz;
    M.ntiles = (int)pl.tiles.size();
    M.nlong = (int)pl.longs.size();
    CK(cudaMemcpyAsync(M.tiles, pl.tiles.data(), sizeof(int4) * pl.tiles.size(), cudaMemcpyHostToDevice, s));
    if (!pl.longs.empty()) {
        CK(cudaMemcpyAsync(M.longs, pl.longs.data(), sizeof(int4) * pl.longs.size(), cudaMemcpyHostToDevice, s));
        CK(cudaMemsetAsync(M.counters, 0, sizeof(int) * pl.longs.size(), s));
    }
    const std::vector<int4>& ptl = sep ? pl.ptiles : pl.tiles;   // the list pdesc indexes
    if (d_pinfo && !ptl.empty()) {
        // panel tiles over one row-major block of F get a direct descriptor
        std::vector<int32_t> rb(h->nf);
        CK(cudaMemcpyAsync(rb.data(), h->rbase, sizeof(int) * h->nf, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        std::vector<int4> pd(ptl.size(), make_int4(0, 0, 0, 0));
        for (size_t t = 0; t < ptl.size(); ++t) {
            const int4 tl = ptl[t];
            if (!(tl.y < 0 && tl.w < 0)) continue;
            const int2 pi = pinfo[tl.x];
            const long long stride = pi.y > 1 ? (long long)rb[pi.x + 1] - rb[pi.x] : 1;
            bool uni = stride > 0 && stride < INT_MAX;
            for (int q = 1; q < pi.y && uni; ++q)
                uni = (long long)rb[pi.x + q] == (long long)rb[pi.x] + q * stride;
            if (uni) pd[t] = make_int4(pi.x, pi.y, rb[pi.x], (int)stride);
        }
        CK(cudaMemcpyAsync(M.pdesc, pd.data(), sizeof(int4) * pd.size(), cudaMemcpyHostToDevice, s));
        CK(cudaStreamSynchronize(s));
    }
    const bool runs = !(h->flags & HPR_FLAG_NO_RUNS);
    if (M.ntiles && runs)
        k_chunk_aux<<<nblk((long long)M.ntiles * 32, LAYOUT_TPB), LAYOUT_TPB, 0, s>>>(
            M.tiles, M.ntiles, M.idx, M.taux);
    else if (M.ntiles)
        CK(cudaMemsetAsync(M.taux, 0, sizeof(int2) * M.ntiles, s));
    CKL();
    M.free_nnz = 0;                 // entries streamed without their index (introspection)
    if (M.ntiles && runs) {
        std::vector<int2> ta(M.ntiles);
        CK(cudaMemcpyAsync(ta.data(), M.taux, sizeof(int2) * M.ntiles, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        for (int t = 0; t < M.ntiles; ++t)
            if (pl.tiles[t].y >= 0 && ta[t].y) M.free_nnz += pl.tiles[t].z - pl.tiles[t].y;
    }
    CK(cudaStreamSynchronize(s));   // the host plan must outlive the copies
}


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

void hpr_destroy(hpr_handle* h);

int hpr_create(const hpr_problem* p, const hpr_options* opt, hpr_handle** out) {
    hpr_handle* h = nullptr;
    const bool verbose = getenv("HPR_VERBOSE") != nullptr;
    auto tp = std::chrono::steady_clock::now();
    auto phase = [&](const char* name) {
        if (!verbose) return;
        const auto now = std::chrono::steady_clock::now();
        fprintf(stderr, "[hpr_create] %-14s %8.1f ms\n", name,
                std::chrono::duration<double, std::milli>(now - tp).count());
        tp = now;
    };
    try {
        validate(p);
        if (!out) fail(HPR_ERR_INVALID, "out is NULL");
        h = new hpr_handle();
        h->dev = opt ? opt->device : 0;
        if (opt && opt->nccl_comm) {            // partitioned mode (also with one rank)
            h->comm = (ncclComm_t)opt->nccl_comm;
            h->world = std::max(1, opt->world_size);
            h->rank = opt->rank;
            // the column vectors carry a 64-byte tail pad, so a padded chunk fits up
            // to 8 ranks (one box; NVSwitch)
            if (h->world > 8) fail(HPR_ERR_INVALID, "partitioned solve: at most 8 ranks");
        }
        hpr::DeviceScope dscope_(h->dev);
        CK(dscope_.err);
        h->m = p->m;
        h->n = p->n;
        h->chunk = (p->n + h->world - 1) / h->world;
        h->c0 = std::min(p->n, h->rank * h->chunk);
        h->clen = std::min(p->n, h->c0 + h->chunk) - h->c0;
        h->n_eq = p->n_eq;
        h->nnz = p->nnz;
        h->offset = p->offset;
        const int m = p->m, n = p->n, n_eq = p->n_eq;
        const long long nnz = p->nnz;
        const int flags = opt ? opt->flags : 0;
        h->flags = flags;
        // workspace (sized from m, n, nnz alone) and streams
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
            // the private stream gets the device's greatest priority: work a
            // caller queues on default-priority streams (e.g. speculative
            // node-LP solves, bb.py) only fills SMs this solve leaves idle
            int least = 0, greatest = 0;
            CK(cudaDeviceGetStreamPriorityRange(&least, &greatest));
            CK(cudaStreamCreateWithPriority(&h->stream, cudaStreamNonBlocking, greatest));
            h->own_stream = true;
        }
        CK(cudaStreamCreateWithFlags(&h->cap, cudaStreamNonBlocking));
        for (auto& e : h->ev) CK(cudaEventCreate(&e));
        CK(cudaMallocHost(&h->h_ctrl, sizeof(Ctrl)));
        CK(cudaMallocHost(&h->h_scal, 8 * sizeof(double)));
        cudaStream_t s = h->stream;
        retain_scratch_pool(h->dev);
        Scratch sc;
        sc.s = s;
        void* tmp = nullptr;
        size_t tmp_bytes = 0;
        auto g32 = [](long long items) { return nblk(items * 32, LAYOUT_TPB); };

        // ---- raw CSR on the device (caller's device arrays are used in place)
        auto on_device = [](const void* q) {
            cudaPointerAttributes at;
            const bool d = cudaPointerGetAttributes(&at, q) == cudaSuccess &&
                           at.type == cudaMemoryTypeDevice;
            cudaGetLastError();
            return d;
        };
        phase("init");
        const int* rptr = p->indptr;
        const int* ridx = p->indices;
        const double* rval = p->data;
        if (!on_device(p->indptr)) {
            int* q = sc.alloc<int>(m + 1);
            CK(cudaMemcpyAsync(q, p->indptr, sizeof(int) * (m + 1), cudaMemcpyHostToDevice, s));
            rptr = q;
        }
        if (nnz && !on_device(p->indices)) {
            int* q = sc.alloc<int>(nnz);
            upload_pageable(q, p->indices, sizeof(int) * nnz, s);
            ridx = q;
        }
        if (nnz && !on_device(p->data)) {
            double* q = sc.alloc<double>(nnz);
            upload_pageable(q, p->data, sizeof(double) * nnz, s);
            rval = q;
        }
        phase("upload A");
        {
            int* bad = sc.alloc<int>(4);
            CK(cudaMemsetAsync(bad, 0, sizeof(int), s));
            k_check_csr<<<std::min(nblk(nnz + m, LAYOUT_TPB), 148 * 32), LAYOUT_TPB, 0, s>>>(
                rptr, m, ridx, nnz, n, bad);
            CKL();
            int hv[3] = {0, 0, 0};
            CK(cudaMemcpyAsync(&hv[0], bad, sizeof(int), cudaMemcpyDeviceToHost, s));
            CK(cudaMemcpyAsync(&hv[1], rptr, sizeof(int), cudaMemcpyDeviceToHost, s));
            CK(cudaMemcpyAsync(&hv[2], rptr + m, sizeof(int), cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            if (hv[1] != 0 || hv[2] != nnz) fail(HPR_ERR_INVALID, "indptr inconsistent with nnz");
            if (hv[0] & 1) fail(HPR_ERR_INVALID, "column index out of range");
            if (hv[0] & 2) fail(HPR_ERR_INVALID, "indptr not monotone");
        }
        phase("check");

        // ---- A^T: stable sort of the entries by column (rows stay ordered)
        int* iota_e = sc.alloc<int>(nnz);
        k_iota<<<nblk(nnz, LAYOUT_TPB), LAYOUT_TPB, 0, s>>>(iota_e, (int)nnz, 0);
        int* row_of = sc.alloc<int>(nnz);
        k_expand_rows<<<g32(m), LAYOUT_TPB, 0, s>>>(rptr, m, row_of);
        int* keys_out = sc.alloc<int>(nnz);
        int* perm_e = sc.alloc<int>(nnz);
        sort_pairs(ridx, keys_out, iota_e, perm_e, nnz, bits_for(n), tmp, tmp_bytes, sc, s);
        int* tptr0 = sc.alloc<int>(n + 1);
        int* tidx0 = sc.alloc<int>(nnz);
        double* tval0 = sc.alloc<double>(nnz);
        {
            int* cnt = sc.alloc<int>(n + 1);
            CK(cudaMemsetAsync(cnt, 0, sizeof(int) * (n + 1), s));
            k_col_count<<<std::min(nblk(nnz, LAYOUT_TPB), 148 * 32), LAYOUT_TPB, 0, s>>>(ridx, nnz, cnt);
            scan_lengths(cnt, n, tptr0, tmp, tmp_bytes, sc, s);
            k_take<int><<<std::min(nblk(nnz, LAYOUT_TPB), 148 * 32), LAYOUT_TPB, 0, s>>>(tidx0, row_of, perm_e, nnz);
            k_take<double><<<std::min(nblk(nnz, LAYOUT_TPB), 148 * 32), LAYOUT_TPB, 0, s>>>(tval0, rval, perm_e, nnz);
            CKL();
        }
        phase("transpose");

        // ---- locality ordering + relabelled A, A^T
        int* rinv = sc.alloc<int>(m);
        int* cinv = sc.alloc<int>(n);
        int* lenbuf = sc.alloc<int>(std::max(m, n) + 1);
        if (!(flags & HPR_FLAG_NO_REORDER)) {
            int* ckey = sc.alloc<int>(n);
            k_fill_int<<<nblk(n, LAYOUT_TPB), LAYOUT_TPB, 0, s>>>(ckey, n, 0x7fffffff);
            k_col_key<<<g32(m), LAYOUT_TPB, 0, s>>>(rptr, ridx, m, LONG_ROW, ckey);
            int* iota_n = sc.alloc<int>(std::max(m, n));
            k_iota<<<nblk(std::max(m, n), LAYOUT_TPB), LAYOUT_TPB, 0, s>>>(iota_n, std::max(m, n), 0);
            int* kout = sc.alloc<int>(std::max(m, n));
            sort_pairs(ckey, kout, iota_n, h->cperm, n, 32, tmp, tmp_bytes, sc, s);
            k_invert<<<nblk(n, LAYOUT_TPB), LAYOUT_TPB, 0, s>>>(h->cperm, n, cinv);
            int* rkey = sc.alloc<int>(m);
            k_row_key<<<g32(m), LAYOUT_TPB, 0, s>>>(rptr, ridx, m, cinv, rkey);
            sort_pairs(rkey, kout, iota_n, h->rperm, n_eq, 32, tmp, tmp_bytes, sc, s);
            sort_pairs(rkey + n_eq, kout, iota_n + n_eq, h->rperm + n_eq, m - n_eq, 32, tmp,
                       tmp_bytes, sc, s);
            k_invert<<<nblk(m, LAYOUT_TPB), LAYOUT_TPB, 0, s>>>(h->rperm, m, rinv);
            CKL();
            h->reordered = true;
        } else {
            k_iota<<<nblk(m, LAYOUT_TPB), LAYOUT_TPB, 0, s>>>(h->rperm, m, 0);
            k_iota<<<nblk(n, LAYOUT_TPB), LAYOUT_TPB, 0, s>>>(h->cperm, n, 0);
            k_iota<<<nblk(m, LAYOUT_TPB), LAYOUT_TPB, 0, s>>>(rinv, m, 0);
            k_iota<<<nblk(n, LAYOUT_TPB), LAYOUT_TPB, 0, s>>>(cinv, n, 0);
            CKL();
        }
        CK(cudaMemsetAsync(lenbuf + m, 0, sizeof(int), s));
        k_perm_len<<<nblk(m, LAYOUT_TPB), LAYOUT_TPB, 0, s>>>(rptr, h->rperm, m, lenbuf);
        scan_lengths(lenbuf, m, h->A.ptr, tmp, tmp_bytes, sc, s);
        k_gather_rows<<<g32(m), LAYOUT_TPB, 0, s>>>(rptr, ridx, rval, h->rperm, m, h->A.ptr, cinv,
                                                     h->A.idx, h->A.mval, nullptr);
        CK(cudaMemsetAsync(lenbuf + n, 0, sizeof(int), s));
        k_perm_len<<<nblk(n, LAYOUT_TPB), LAYOUT_TPB, 0, s>>>(tptr0, h->cperm, n, lenbuf);
        scan_lengths(lenbuf, n, h->AT.ptr, tmp, tmp_bytes, sc, s);
        k_gather_rows<<<g32(n), LAYOUT_TPB, 0, s>>>(tptr0, tidx0, tval0, h->cperm, n, h->AT.ptr,
                                                     rinv, h->AT.idx, h->AT.mval, nullptr);
        CKL();
        phase("reorder");

        // ---- twin folding (pairing decided on the host from device candidates)
        std::vector<int32_t> frow;
        std::vector<unsigned char> second(m, 0);
        if (!(flags & HPR_FLAG_NO_FOLD) && m > 1) {
            unsigned char* cand = sc.alloc<unsigned char>(m);
            k_twin_candidates<<<g32(m), LAYOUT_TPB, 0, s>>>(h->A.ptr, h->A.idx, h->A.mval, m,
                                                             n_eq, cand);
            CKL();
            std::vector<unsigned char> hc(m);
            CK(cudaMemcpyAsync(hc.data(), cand, m, cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            for (int i = 0; i < m;) {
                frow.push_back(i);
                if (hc[i]) {
                    second[i + 1] = 1;
                    i += 2;
                } else {
                    i += 1;
                }
            }
        } else {
            frow.resize(m);
            for (int i = 0; i < m; ++i) frow[i] = i;
        }
        h->nf = (int)frow.size();
        frow.push_back(m);
        h->folded = h->nf < m;
        std::vector<int32_t> fold_of(m), rmap(m);
        for (int f = 0; f < h->nf; ++f)
            for (int i = frow[f]; i < frow[f + 1]; ++i) {
                fold_of[i] = f;
                rmap[i] = 2 * f + (i > frow[f] ? 1 : 0);
            }
        CK(cudaMemcpyAsync(h->frow, frow.data(), sizeof(int) * frow.size(), cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(h->rmap, rmap.data(), sizeof(int) * m, cudaMemcpyHostToDevice, s));
        if (h->folded) {
            unsigned char* dsec = sc.alloc<unsigned char>(m);
            int* dfold = sc.alloc<int>(m);
            CK(cudaMemcpyAsync(dsec, second.data(), m, cudaMemcpyHostToDevice, s));
            CK(cudaMemcpyAsync(dfold, fold_of.data(), sizeof(int) * m, cudaMemcpyHostToDevice, s));
            CK(cudaMemsetAsync(lenbuf + h->nf, 0, sizeof(int), s));
            k_perm_len<<<nblk(h->nf, LAYOUT_TPB), LAYOUT_TPB, 0, s>>>(h->A.ptr, h->frow, h->nf, lenbuf);
            scan_lengths(lenbuf, h->nf, h->F.ptr, tmp, tmp_bytes, sc, s);
            k_gather_rows<<<g32(h->nf), LAYOUT_TPB, 0, s>>>(h->A.ptr, h->A.idx, h->A.mval, h->frow,
                                                             h->nf, h->F.ptr, nullptr, h->F.idx,
                                                             h->F.mval, h->F.src);
            CK(cudaMemsetAsync(lenbuf + n, 0, sizeof(int), s));
            k_fold_count<<<g32(n), LAYOUT_TPB, 0, s>>>(h->AT.ptr, h->AT.idx, n, dsec, lenbuf);
            scan_lengths(lenbuf, n, h->FT.ptr, tmp, tmp_bytes, sc, s);
            k_fold_gather<<<nblk(n, LAYOUT_TPB), LAYOUT_TPB, 0, s>>>(h->AT.ptr, h->AT.idx,
                                                                     h->AT.mval, n, dsec, dfold,
                                                                     h->FT.ptr, h->FT.idx,
                                                                     h->FT.mval, h->FT.src);
            CKL();
            int nf_nnz = 0;
            CK(cudaMemcpyAsync(&nf_nnz, h->F.ptr + h->nf, sizeof(int), cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            h->nnz_f = nf_nnz;
        } else {
            CK(cudaMemcpyAsync(h->F.ptr, h->A.ptr, sizeof(int) * (m + 1), cudaMemcpyDeviceToDevice, s));
            CK(cudaMemcpyAsync(h->FT.ptr, h->AT.ptr, sizeof(int) * (n + 1), cudaMemcpyDeviceToDevice, s));
            if (nnz) {
                CK(cudaMemcpyAsync(h->F.idx, h->A.idx, sizeof(int) * nnz, cudaMemcpyDeviceToDevice, s));
                CK(cudaMemcpyAsync(h->FT.idx, h->AT.idx, sizeof(int) * nnz, cudaMemcpyDeviceToDevice, s));
                CK(cudaMemcpyAsync(h->F.mval, h->A.mval, sizeof(double) * nnz, cudaMemcpyDeviceToDevice, s));
                CK(cudaMemcpyAsync(h->FT.mval, h->AT.mval, sizeof(double) * nnz, cudaMemcpyDeviceToDevice, s));
                k_iota<<<nblk(nnz, LAYOUT_TPB), LAYOUT_TPB, 0, s>>>(h->F.src, (int)nnz, 0);
                k_iota<<<nblk(nnz, LAYOUT_TPB), LAYOUT_TPB, 0, s>>>(h->FT.src, (int)nnz, 0);
                CKL();
            }
            h->nnz_f = nnz;
        }
        phase("fold");

        // ---- pad nearly dense flow rows of F to single column runs (explicit
        // zeros; only while the padded operand fits the carved capacity)
        long long f_nnz = h->nnz_f;
        if (!(flags & HPR_FLAG_NO_RUNS) && h->nf && h->nnz_f) {
            int* plen = sc.alloc<int>(h->nf + 1);
            CK(cudaMemsetAsync(plen + h->nf, 0, sizeof(int), s));
            k_pad_count<<<g32(h->nf), LAYOUT_TPB, 0, s>>>(h->F.ptr, h->F.idx, h->nf,
                                                           PANEL_MIN_ROW, plen);
            CKL();
            int* nptr = sc.alloc<int>(h->nf + 1);
            scan_lengths(plen, h->nf, nptr, tmp, tmp_bytes, sc, s);
            int tot = 0;
            CK(cudaMemcpyAsync(&tot, nptr + h->nf, sizeof(int), cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            if (tot > h->nnz_f && tot <= nnz) {
                int* oidx = sc.alloc<int>(h->nnz_f);
                int* osrc = sc.alloc<int>(h->nnz_f);
                double* oval = sc.alloc<double>(h->nnz_f);
                int* optr = sc.alloc<int>(h->nf + 1);
                CK(cudaMemcpyAsync(optr, h->F.ptr, sizeof(int) * (h->nf + 1), cudaMemcpyDeviceToDevice, s));
                CK(cudaMemcpyAsync(oidx, h->F.idx, sizeof(int) * h->nnz_f, cudaMemcpyDeviceToDevice, s));
                CK(cudaMemcpyAsync(osrc, h->F.src, sizeof(int) * h->nnz_f, cudaMemcpyDeviceToDevice, s));
                CK(cudaMemcpyAsync(oval, h->F.mval, sizeof(double) * h->nnz_f, cudaMemcpyDeviceToDevice, s));
                CK(cudaMemcpyAsync(h->F.ptr, nptr, sizeof(int) * (h->nf + 1), cudaMemcpyDeviceToDevice, s));
                k_pad_gather<<<g32(h->nf), LAYOUT_TPB, 0, s>>>(optr, oidx, oval, osrc, h->nf,
                                                                h->F.ptr, h->F.idx, h->F.mval,
                                                                h->F.src);
                CKL();
                f_nnz = tot;
            }
        }
        phase("pad");

        // ---- flow panels: F^T drops the dense flow block, read from F instead
        // (partitioned: each rank's panels cover its own flow rows, and the
        // A^T y partials are all-reduced before the update as without panels)
        long long ft_nnz = h->nnz_f;
        const bool rows_dense = h->nf && n && h->nnz_f;
        if (rows_dense)      // one consecutive-column run per dense F row (panels, row panels)
            k_dense_rows<<<g32(h->nf), LAYOUT_TPB, 0, s>>>(h->F.ptr, h->F.idx, h->nf,
                                                            PANEL_MIN_ROW, h->rbase);
        if (!(flags & HPR_FLAG_NO_PANELS) && h->nf && n && h->nnz_f) {
            int* roff = sc.alloc<int>(n);
            CK(cudaMemsetAsync(h->d_dev, 0, 2 * sizeof(unsigned long long), s));
            CK(cudaMemsetAsync(lenbuf + n, 0, sizeof(int), s));
            k_col_panels<<<nblk(n, LAYOUT_TPB), LAYOUT_TPB, 0, s>>>(
                h->FT.ptr, h->FT.idx, n, h->rbase, PANEL_MIN_RUN, PANEL_MAX_KEEP, h->pinfo, roff, lenbuf,
                h->d_dev);
            CKL();
            unsigned long long cov[2] = {0, 0};
            CK(cudaMemcpyAsync(cov, h->d_dev, sizeof(cov), cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            if (cov[0] * 10 >= (unsigned long long)h->nnz_f) {      // worth a layout change
                int* optr = sc.alloc<int>(n + 1);
                int* oidx = sc.alloc<int>(h->nnz_f);
                int* osrc = sc.alloc<int>(h->nnz_f);
                double* oval = sc.alloc<double>(h->nnz_f);
                CK(cudaMemcpyAsync(optr, h->FT.ptr, sizeof(int) * (n + 1), cudaMemcpyDeviceToDevice, s));
                CK(cudaMemcpyAsync(oidx, h->FT.idx, sizeof(int) * h->nnz_f, cudaMemcpyDeviceToDevice, s));
                CK(cudaMemcpyAsync(osrc, h->FT.src, sizeof(int) * h->nnz_f, cudaMemcpyDeviceToDevice, s));
                CK(cudaMemcpyAsync(oval, h->FT.mval, sizeof(double) * h->nnz_f, cudaMemcpyDeviceToDevice, s));
                scan_lengths(lenbuf, n, h->FT.ptr, tmp, tmp_bytes, sc, s);
                k_drop_panels<<<nblk(n, LAYOUT_TPB), LAYOUT_TPB, 0, s>>>(
                    optr, oidx, oval, osrc, n, h->pinfo, roff, h->FT.ptr, h->FT.idx, h->FT.mval,
                    h->FT.src);
                CKL();
                h->panels = true;
                h->FT.pinfo = h->pinfo;
                h->FT.rbase = h->rbase;
                h->panel_nnz = (long long)cov[0];
                h->panel_cols = (long long)cov[1];
                ft_nnz = h->nnz_f - h->panel_nnz;
            }
        }
        phase("panels");

        // ---- tile schedules (host plan from the device indptr)
        plan_tiles(h, h->A, m, n, nnz);
        plan_tiles(h, h->AT, n, m, nnz);
        plan_tiles(h, h->F, h->nf, n, f_nnz, nullptr,
                   rows_dense && row_panels_on(f_nnz) && !(flags & HPR_FLAG_NO_RUNS) ? h->rbase
                                                                               : nullptr);
        plan_tiles(h, h->FT, n, h->nf, ft_nnz, h->panels ? h->pinfo : nullptr);
        {
            const int fm = fused_mode();
            h->fused = !h->comm &&
                       (fm == 1 || (fm < 0 && h->F.nrtiles == 0 && h->FT.nptiles == 0));
        }
        phase("tiles");
        put_vec(h, h->rhs_m, p->rhs, m, true);
        put_vec(h, h->cost_m, p->cost, n, false);
        put_vec(h, h->lo_m, p->lower, n, false);
        put_vec(h, h->up_m, p->upper, n, false);
        CK(cudaMemsetAsync(h->ctrl, 0, sizeof(Ctrl), s));
        CK(cudaStreamSynchronize(s));
        phase("upload");
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
    hpr::DeviceScope dscope_(h->dev);
    if (h->stream) cudaStreamSynchronize(h->stream);
    if (h->gexec) cudaGraphExecDestroy(h->gexec);
    if (h->graph) cudaGraphDestroy(h->graph);
    if (h->own_ws && h->ws) cudaFree(h->ws);
    if (h->log) cudaFree(h->log);
    if (h->h_ctrl) cudaFreeHost(h->h_ctrl);
    if (h->h_scal) cudaFreeHost(h->h_scal);
    for (auto& e : h->ev)
        if (e) cudaEventDestroy(e);
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
    hpr::DeviceScope dscope_(h->dev);
    CK(dscope_.err);
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
    hpr::DeviceScope dscope_(h->dev);
    CK(dscope_.err);
    const DevCsr& M = transpose ? h->AT : h->A;
    const int nin = transpose ? h->m : h->n, nout = transpose ? h->n : h->m;
    double* xin = transpose ? h->YM : h->XM;   // master scratch of the input length
    put_vec(h, xin, in, nin, transpose != 0);
    EpiStore<double> st{h->pw, nullptr};       // pw holds m + n doubles
    launch_spmv(h, M, (const double*)M.mval, (const double*)xin, st, h->stream);
    if (transpose) allreduce(h, h->pw, nout, ncclFloat64, ncclSum, h->stream);
    get_vec(h, out, h->pw, nout, transpose == 0);
    CK(cudaStreamSynchronize(h->stream));
    API_END
}

int hpr_kkt_residual(hpr_handle* h, const double* x, const double* y, const double* z,
                     hpr_kkt* out) {
    API_BEGIN
    if (!h || !x || !y || !z || !out) fail(HPR_ERR_INVALID, "NULL argument");
    hpr::DeviceScope dscope_(h->dev);
    CK(dscope_.err);
    cudaStream_t s = h->stream;
    put_vec(h, h->XM, x, h->n, false);
    put_vec(h, h->YM, y, h->m, true);
    put_vec(h, h->ZM, z, h->n, false);
    // bar/anchor terms are irrelevant here: zero them (FP64 views)
    for (void* v : {h->BX, h->BZ, h->AXv}) CK(cudaMemsetAsync(v, 0, sizeof(double) * h->n, s));
    for (void* v : {h->BY, h->AYv}) CK(cudaMemsetAsync(v, 0, sizeof(double) * h->m, s));
    k_fold_rows<double><<<nblk(h->nf), TPB, 0, s>>>(h->nf, h->frow, nullptr, nullptr, nullptr,
                                                     nullptr, h->YM, h->YMF);
    CKL();
    const double rn = std::sqrt(dev_sumsq(h, h->rhs_m, h->m, 0, true));
    const double cn = std::sqrt(dev_sumsq(h, h->cost_m, h->n, 0));
    Ctrl c{};
    c.denom = (1.0 + rn) + cn;
    c.offset = h->offset;
    c.B = 1;
    c.status = -1;
    CK(cudaMemcpyAsync(h->ctrl, &c, sizeof(Ctrl), cudaMemcpyHostToDevice, s));
    Ptrs<double> p = ptrs<double>(h);
    double* pd = (double*)h->P;
    EpiStore<double> st{pd, nullptr};
    launch_spmv(h, h->F, (const double*)h->F.mval, (const double*)h->XM, st, s);
    const int gr = h->comm ? ROW_GRID_MAX : row_grid(h->nf), gc = row_grid(h->n);
    CheckRowsArgs<double> ar{h->nf, h->n_eq, h->frow, pd, h->YM, h->rhs_m, p.BY, p.AY, h->rowpart};
    k_check_rows<double><<<gr, TPB, 0, s>>>(ar);
    allreduce(h, h->rowpart, (size_t)KR * gr, ncclFloat64, ncclSum, s);
    launch_spmv(h, h->FT, (const double*)h->FT.mval, (const double*)h->YMF, st, s,
                (const double*)h->F.mval);
    allreduce(h, pd, h->n, ncclFloat64, ncclSum, s);
    CheckColsArgs<double> ac{h->n, pd, h->XM, h->ZM, h->cost_m, h->lo_m, h->up_m, p.BX, p.BZ, p.AX,
                             h->colpart};
    k_check_cols<double><<<gc, TPB, 0, s>>>(ac);
    k_controller<<<1, CTRL_TPB, 0, s>>>(h->ctrl, h->rowpart, gr, h->colpart, gc, h->log, 0,
                                        nullptr);
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
    hpr::DeviceScope dscope_(h->dev);
    CK(dscope_.err);
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
    hpr::DeviceScope dscope_(h->dev);
    CK(dscope_.err);
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
    refresh_folded_values(h, fp32);
    if (fp32) cast_work_vectors(h);
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
    auto step = [&](auto tag) {
        using T = decltype(tag);
        Ptrs<T> p = ptrs<T>(h);
        k_fold_rows<T><<<nblk(h->nf), TPB, 0, s>>>(h->nf, h->frow, p.Y, p.YF, nullptr, nullptr,
                                                    nullptr, nullptr);
        CKL();
        h->upd_z = true;             // the caller reads the new z
        try {
            enqueue_iteration<T>(h, p, 0, true, s);
        } catch (...) {
            h->upd_z = false;
            throw;
        }
        h->upd_z = false;
    };
    if (fp32) step(float(0));
    else step(double(0));
    get(h->X, x_out, n, h->XM, false);
    get(h->Y, y_out, m, h->YM, true);
    get(h->Z, z_out, n, h->ZM, false);
    get(h->BX, bar_x, n, h->XM, false);
    get(h->BY, bar_y, m, h->YM, true);
    get(h->BZ, bar_z, n, h->ZM, false);
    CK(cudaStreamSynchronize(s));
    API_END
}

int hpr_nccl_unique_id(uint8_t out[128]) {
    API_BEGIN
    if (!out) fail(HPR_ERR_INVALID, "NULL argument");
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    ncclUniqueId id;
    const ncclResult_t r = ncclGetUniqueId(&id);
    if (r != ncclSuccess) fail(HPR_ERR_CUDA, std::string("ncclGetUniqueId: ") + ncclGetErrorString(r));
    std::memcpy(out, &id, sizeof(id));
    API_END
}

int hpr_nccl_comm_init(const uint8_t id[128], int32_t world_size, int32_t rank, int32_t device,
                       void** comm_out) {
    API_BEGIN
    if (!id || !comm_out || world_size < 1 || rank < 0 || rank >= world_size)
        fail(HPR_ERR_INVALID, "bad argument");
    hpr::DeviceScope dscope_(device);
    CK(dscope_.err);
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    ncclComm_t comm;
    const ncclResult_t r = ncclCommInitRank(&comm, world_size, uid, rank);
    if (r != ncclSuccess) fail(HPR_ERR_CUDA, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
    *comm_out = (void*)comm;
    API_END
}

void hpr_nccl_comm_destroy(void* comm) {
    if (comm) ncclCommDestroy((ncclComm_t)comm);
}

int hpr_get_layout(hpr_handle* h, hpr_layout* out) {
    API_BEGIN
    if (!h || !out) fail(HPR_ERR_INVALID, "NULL argument");
    out->m = h->m;
    out->n = h->n;
    out->n_eq = h->n_eq;
    out->folded_rows = h->nf;
    out->nnz = h->nnz;
    out->folded_nnz = h->nnz_f;
    out->tiles_a = h->A.ntiles;
    out->tiles_at = h->AT.ntiles;
    out->tiles_f = h->F.ntiles;
    out->tiles_ft = h->FT.ntiles;
    out->reordered = h->reordered;
    out->folded = h->folded;
    out->workspace_bytes = h->ws_bytes;
    out->panel_cols = h->panel_cols;
    out->panel_nnz = h->panel_nnz;
    out->fused = h->fused ? 1 : 0;
    out->f_nnz = h->F.nnz;
    out->ft_nnz = h->FT.nnz;
    out->index_free_nnz_f = h->F.free_nnz + h->F.group_nnz;
    out->row_panel_groups = h->F.ngroups;
    API_END
}

int hpr_resume(hpr_handle* h, int64_t more_iterations, double tolerance, hpr_stats* st) {
    API_BEGIN
    if (!h || !st) fail(HPR_ERR_INVALID, "NULL argument");
    if (h->last_prec < 0 || (!h->gexec && !use_eager(h, h->h_ctrl->B)))
        fail(HPR_ERR_INVALID, "hpr_resume needs a prior looping solve");
    hpr::DeviceScope dscope_(h->dev);
    CK(dscope_.err);
    std::memset(st, 0, sizeof(*st));
    h->launches = 0;
    read_ctrl(h);
    Ctrl c = *h->h_ctrl;
    c.max_iter = c.total + more_iterations;
    c.status = more_iterations >= c.B ? -1 : HPR_ITERATION_LIMIT;
    c.has_deadline = 0;
    if (tolerance > 0) c.tol = tolerance;
    c.cond = 0;
    c.halt = 0;
    c.skipped = 0;
    CK(cudaMemcpyAsync(h->ctrl, &c, sizeof(Ctrl), cudaMemcpyHostToDevice, h->stream));
    *h->h_ctrl = c;
    if (c.status != -1) st->loop_seconds = 0.0;
    else if (use_eager(h, c.B))
        st->loop_seconds = h->last_prec == HPR_FP32 ? run_eager<float>(h, (int)c.B)
                                                    : run_eager<double>(h, (int)c.B);
    else st->loop_seconds = run_loop(h);
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
    const bool in_iter = (which & HPR_BENCH_IN_ITERATION) != 0;
    which &= ~HPR_BENCH_IN_ITERATION;
    if (which < 0 || which > 6) fail(HPR_ERR_INVALID, "unknown kernel");
    if (in_iter && which == 4) fail(HPR_ERR_INVALID, "the check block has no in-iteration form");
    hpr::DeviceScope dscope_(h->dev);
    CK(dscope_.err);
    cudaStream_t s = h->stream;
    // which: 0 = A x~ product, 1 = A^T y product, 2 = primal update, 3 = dual update,
    //        4 = one whole KKT check (2 master products, row/col terms, controller, copies;
    //            mutates the solver state — call last)
    auto body = [&](auto tag, int which) {
        using T = decltype(tag);
        Ptrs<T> p = ptrs<T>(h);
        EpiStore<T> st{p.P, nullptr};
        PrimalArgs<T> pa{h->ctrl, 0, h->n, p.P, p.X, p.Z, p.XT, p.AX, p.AZ, p.cost, p.lo, p.up,
                         p.BX, p.BZ, h->XM, h->ZM, h->cs, h->upd_z};
        DualArgs<T> da{h->ctrl, 0, h->m, h->n_eq, h->rmap, p.P, p.Y, p.AY, p.rhs, p.YF,
                       p.BY, p.BYF, h->YM, h->YMF, h->rs};
        switch (which) {
            case 0: launch_spmv(h, h->F, p.f_vals, (const T*)p.XT, st, s); break;
            case 1: launch_spmv(h, h->FT, p.ft_vals, (const T*)p.YF, st, s, p.f_vals); break;
            case 2: k_update_primal<T, false><<<nblk(h->n), TPB, 0, s>>>(pa); break;
            case 3: k_update_dual<T, false><<<nblk(h->m), TPB, 0, s>>>(da); break;
            case 5: {   // fused: A^T y product + primal update (epilogue)
                launch_spmv(h, h->FT, p.ft_vals, (const T*)p.YF, EpiPrimal<T, false>{pa, nullptr},
                            s, p.f_vals);
                break;
            }
            case 6: {   // fused: A x~ product + dual update (epilogue)
                DualArgs<T> df = da;
                df.frow = h->frow;
                launch_spmv(h, h->F, p.f_vals, (const T*)p.XT, EpiDual<T, false>{df, nullptr}, s);
                break;
            }
            default:
                // the previous check (or the solve's last one) may have set halt
                CK(cudaMemsetAsync(&h->ctrl->halt, 0, sizeof(int), s));
                enqueue_check<T>(h, p, 1, s);
                break;
        }
        CKL();
    };
    // a finished solve leaves Ctrl::halt set; the loop kernels timed here
    // must not take their halted (no-op) path
    CK(cudaMemsetAsync(&h->ctrl->halt, 0, sizeof(int), s));
    auto run = [&](int w) {
        if (h->last_prec == HPR_FP32) body(float(0), w);
        else body(double(0), w);
    };
    // the rest of the iteration, in loop order after `which`
    std::vector<int> rest;
    if (in_iter) {
        if (which >= 5) rest = {which == 5 ? 6 : 5};
        else for (int k = 1; k < 4; ++k) rest.push_back((which + k) % 4);
    }
    run(which);  // warm
    for (int w : rest) run(w);
    if (!in_iter) {
        CK(cudaEventRecord(h->ev[0], s));
        for (int r = 0; r < reps; ++r) run(which);
        CK(cudaEventRecord(h->ev[1], s));
        CK(cudaEventSynchronize(h->ev[1]));
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, h->ev[0], h->ev[1]));
        *seconds_per_launch = ms * 1e-3 / reps;
    } else {
        std::vector<cudaEvent_t> ev(2 * (size_t)reps, nullptr);
        struct Release {
            std::vector<cudaEvent_t>& v;
            ~Release() {
                for (cudaEvent_t e : v)
                    if (e) cudaEventDestroy(e);
            }
        } release_{ev};
        for (auto& e : ev) CK(cudaEventCreate(&e));
        for (int r = 0; r < reps; ++r) {
            CK(cudaEventRecord(ev[2 * r], s));
            run(which);
            CK(cudaEventRecord(ev[2 * r + 1], s));
            for (int w : rest) run(w);
        }
        CK(cudaEventSynchronize(ev.back()));
        double total = 0.0;
        for (int r = 0; r < reps; ++r) {
            float ms = 0.f;
            CK(cudaEventElapsedTime(&ms, ev[2 * r], ev[2 * r + 1]));
            total += ms;
        }
        *seconds_per_launch = total * 1e-3 / reps;
    }
    API_END
}

}  // extern "C"
