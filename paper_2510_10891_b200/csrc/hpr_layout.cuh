// hpr_layout.cuh — device-side construction of the engine's operand layout.
//
// hpr_create uploads the caller's CSR once and builds everything else on
// the GPU (CUB radix sorts + gather kernels), instead of ~2.5 s of host
// loops at C4 scale:
//   * A^T (stable sort of the entries by column: rows stay ordered inside a
//     column, exactly scipy's tocsc + sort_indices),
//   * the locality permutation (hpr_engine.cu: compute_order semantics),
//   * the twin-folded operands F, F^T and their gather maps.
// Entry order inside every row is preserved through all of it.
#pragma once

#include <climits>

#include <cub/cub.cuh>

#include "hpr_common.cuh"

namespace hpr {

constexpr int LAYOUT_TPB = 256;

// row index of every entry (warp per row)
__global__ void k_expand_rows(const int* ptr, int rows, int* row_of) {
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (w >= rows) return;
    for (int e = ptr[w] + lane; e < ptr[w + 1]; e += 32) row_of[e] = w;
}

__global__ void k_iota(int* p, int n, int base) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = base + i;
}

__global__ void k_fill_int(int* p, int n, int v) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = v;
}

__global__ void k_col_count(const int* idx, long long nnz, int* cnt) {
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < nnz;
         e += (long long)gridDim.x * blockDim.x)
        atomicAdd(cnt + idx[e], 1);
}

// gather a permutation of entries: dst[k] = src[perm[k]] for int / double
template <typename T>
__global__ void k_take(T* dst, const T* src, const int* perm, long long n) {
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n;
         k += (long long)gridDim.x * blockDim.x)
        dst[k] = src[perm[k]];
}

// ckey[col] = min long row touching col (warp per row)
__global__ void k_col_key(const int* ptr, const int* idx, int rows, int long_row, int* ckey) {
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (w >= rows) return;
    const int b = ptr[w], e = ptr[w + 1];
    if (e - b <= long_row) return;
    for (int q = b + lane; q < e; q += 32) atomicMin(ckey + idx[q], w);
}

// inv[perm[k]] = k
__global__ void k_invert(const int* perm, int n, int* inv) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < n) inv[perm[k]] = k;
}

// rkey[row] = min over entries of cinv[col] (warp per row; empty -> INT_MAX)
__global__ void k_row_key(const int* ptr, const int* idx, int rows, const int* cinv, int* rkey) {
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (w >= rows) return;
    int k = 0x7fffffff;
    for (int q = ptr[w] + lane; q < ptr[w + 1]; q += 32) k = min(k, cinv[idx[q]]);
    for (int off = 16; off > 0; off >>= 1) k = min(k, __shfl_xor_sync(0xffffffffu, k, off));
    if (lane == 0) rkey[w] = k;
}

// lengths of the rows taken in `perm` order (len[r] = ptr[perm[r]+1] - ptr[perm[r]])
__global__ void k_perm_len(const int* ptr, const int* perm, int rows, int* len) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r < rows) len[r] = ptr[perm[r] + 1] - ptr[perm[r]];
}

// Copy row perm[r] of (ptr, idx, val) into new row r (entry order kept);
// columns pass through cmap (or unchanged when null); src (optional) records
// the source entry.  Warp per new row.
__global__ void k_gather_rows(const int* ptr, const int* idx, const double* val, const int* perm,
                              int rows, const int* nptr, const int* cmap, int* nidx,
                              double* nval, int* src) {
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (w >= rows) return;
    const int o = perm ? perm[w] : w;
    const int b = ptr[o], d = nptr[w];
    for (int q = lane; q < ptr[o + 1] - b; q += 32) {
        const int c = idx[b + q];
        nidx[d + q] = cmap ? cmap[c] : c;
        nval[d + q] = val[b + q];
        if (src) src[d + q] = b + q;
    }
}

// twin candidates: rows i, i+1 (inequalities) with identical pattern and
// exactly negated values (warp per i)
__global__ void k_twin_candidates(const int* ptr, const int* idx, const double* val, int rows,
                                  int n_eq, unsigned char* cand) {
    const int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (i >= rows) return;
    bool ok = i >= n_eq && i + 1 < rows;
    int b0 = 0, b1 = 0, l = 0;
    if (ok) {
        b0 = ptr[i];
        b1 = ptr[i + 1];
        l = b1 - b0;
        ok = l > 0 && ptr[i + 2] - b1 == l;
    }
    if (ok) {
        for (int q = lane; q < l && ok; q += 32)
            ok = idx[b0 + q] == idx[b1 + q] && val[b1 + q] == -val[b0 + q];
        ok = __all_sync(0xffffffffu, ok);
    }
    if (lane == 0) cand[i] = ok ? 1 : 0;
}

// F^T row lengths after dropping entries whose row is the second of a pair
__global__ void k_fold_count(const int* ptr, const int* idx, int rows, const unsigned char* second,
                             int* len) {
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (w >= rows) return;
    int c = 0;
    for (int q = ptr[w] + lane; q < ptr[w + 1]; q += 32) c += second[idx[q]] ? 0 : 1;
    for (int off = 16; off > 0; off >>= 1) c += __shfl_xor_sync(0xffffffffu, c, off);
    if (lane == 0) len[w] = c;
}

// F^T rows: keep entries of first rows, relabel rows to folded indices (one
// thread per row keeps the order; rows of A^T are short)
__global__ void k_fold_gather(const int* ptr, const int* idx, const double* val, int rows,
                              const unsigned char* second, const int* fold_of, const int* nptr,
                              int* nidx, double* nval, int* src) {
    const int w = blockIdx.x * blockDim.x + threadIdx.x;
    if (w >= rows) return;
    int d = nptr[w];
    for (int q = ptr[w]; q < ptr[w + 1]; ++q) {
        const int i = idx[q];
        if (second[i]) continue;
        nidx[d] = fold_of[i];
        nval[d] = val[q];
        src[d] = q;
        ++d;
    }
}

// chunk tiles whose columns are consecutive carry {c0, 1} (hpr_spmv.cuh)
__global__ void k_chunk_aux(const int4* tiles, int ntiles, const int* idx, int2* taux) {
    const int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (t >= ntiles) return;
    const int4 tl = tiles[t];
    if (tl.y < 0 || tl.x < 0) {          // stream / panel / row-panel tiles
        if (lane == 0) taux[t] = make_int2(0, 0);
        return;
    }
    bool run = true;
    for (int e = tl.y + 1 + lane; e < tl.z; e += 32) run = run && idx[e] == idx[e - 1] + 1;
    run = __all_sync(0xffffffffu, run);
    if (lane == 0) taux[t] = run ? make_int2(idx[tl.y], 1) : make_int2(0, 0);
}

// ---------------------------------------------------------------------------
// Flow panels.  After the locality ordering a PTDF flow row of F covers one
// period's columns as a single run (F row i = columns j0 .. j0+len-1), and a
// column's flow entries in F^T are consecutive folded rows.  The block is
// dense, so (A^T y)_j's flow part can read F's own row-major values at
// vals[rbase[i] + j] (rbase[i] = ptr[i] - j0) with y broadcast and the
// values coalesced across columns — F^T keeps only the remaining entries.
// ---------------------------------------------------------------------------

// Nearly dense flow rows (a PTDF row misses only the few zero-PTDF columns
// of its period, e.g. the slack bus) are padded with explicit zeros to one
// run of consecutive columns, so both products address them index-free.
// padlen[r] = span when row r (>= min_len entries, strictly increasing
// columns) misses at most len/32 columns of its span, else its length.
__global__ void k_pad_count(const int* ptr, const int* idx, int rows, int min_len, int* padlen) {
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (w >= rows) return;
    const int b = ptr[w], len = ptr[w + 1] - b;
    bool ok = len >= min_len;
    for (int q = lane + 1; q < len && ok; q += 32) ok = idx[b + q] > idx[b + q - 1];
    ok = __all_sync(0xffffffffu, ok);
    int out = len;
    if (ok) {
        const long long span = (long long)idx[b + len - 1] - idx[b] + 1;
        if (span - len <= len / 32) out = (int)span;
    }
    if (lane == 0) padlen[w] = out;
}

// copy rows into the padded layout: a padded row is pre-filled with
// (column, 0.0, src -1) and its entries scattered to column - first column
// (warp per row)
__global__ void k_pad_gather(const int* ptr, const int* idx, const double* val, const int* src,
                             int rows, const int* nptr, int* nidx, double* nval, int* nsrc) {
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (w >= rows) return;
    const int b = ptr[w], len = ptr[w + 1] - b, d = nptr[w], nlen = nptr[w + 1] - d;
    if (nlen == len) {
        for (int q = lane; q < len; q += 32) {
            nidx[d + q] = idx[b + q];
            nval[d + q] = val[b + q];
            nsrc[d + q] = src[b + q];
        }
        return;
    }
    const int j0 = idx[b];
    for (int q = lane; q < nlen; q += 32) {
        nidx[d + q] = j0 + q;
        nval[d + q] = 0.0;
        nsrc[d + q] = -1;
    }
    __syncwarp();
    for (int q = lane; q < len; q += 32) {
        const int p = d + (idx[b + q] - j0);
        nval[p] = val[b + q];
        nsrc[p] = src[b + q];
    }
}

// rbase[i] = ptr[i] - idx[ptr[i]] when row i's columns are consecutive and
// the row has >= min_len entries, else INT_MIN (warp per row)
__global__ void k_dense_rows(const int* ptr, const int* idx, int rows, int min_len, int* rbase) {
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (w >= rows) return;
    const int b = ptr[w], len = ptr[w + 1] - b;
    bool ok = len >= min_len;
    for (int q = lane + 1; q < len && ok; q += 32) ok = idx[b + q] == idx[b + q - 1] + 1;
    ok = __all_sync(0xffffffffu, ok);
    if (lane == 0) rbase[w] = ok ? b - idx[b] : INT_MIN;
}

// Per F^T row j: the longest run of entries on consecutive dense F rows.
// pinfo[j] = {i0, L} (L >= min_run, else {0, 0}), roff[j] = the run's first
// entry within the row, keep[j] = entries left in F^T (a panel row keeps at
// most max_keep, so its panel tile stages them); covered[0] += L,
// covered[1] += 1 per panel column (thread per row).
__global__ void k_col_panels(const int* ptr, const int* idx, int cols, const int* rbase,
                             int min_run, int max_keep, int2* pinfo, int* roff, int* keep,
                             unsigned long long* covered) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= cols) return;
    const int b = ptr[j], len = ptr[j + 1] - b;
    int best = 0, best_q = 0, cur = 0;
    for (int q = 0; q < len; ++q) {
        const int i = idx[b + q];
        if (rbase[i] == INT_MIN) {
            cur = 0;
            continue;
        }
        if (cur > 0 && i == idx[b + q - 1] + 1) {
            ++cur;
        } else {
            cur = 1;
        }
        if (cur > best) {
            best = cur;
            best_q = q - cur + 1;
        }
    }
    if (best >= min_run && len - best <= max_keep) {
        pinfo[j] = make_int2(idx[b + best_q], best);
        roff[j] = best_q;
        keep[j] = len - best;
        atomicAdd(covered, (unsigned long long)best);
        atomicAdd(covered + 1, 1ULL);
    } else {
        pinfo[j] = make_int2(0, 0);
        roff[j] = 0;
        keep[j] = len;
    }
}

// F^T without its panel entries (thread per row, order kept)
__global__ void k_drop_panels(const int* ptr, const int* idx, const double* val, const int* src,
                              int cols, const int2* pinfo, const int* roff, const int* nptr,
                              int* nidx, double* nval, int* nsrc) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= cols) return;
    const int b = ptr[j], len = ptr[j + 1] - b;
    const int r0 = roff[j], r1 = r0 + pinfo[j].y;
    int d = nptr[j];
    for (int q = 0; q < len; ++q) {
        if (q >= r0 && q < r1) continue;
        nidx[d] = idx[b + q];
        nval[d] = val[b + q];
        nsrc[d] = src[b + q];
        ++d;
    }
}

// input checks: indptr monotone and in range, columns in range
__global__ void k_check_csr(const int* ptr, int rows, const int* idx, long long nnz, int cols,
                            int* bad) {
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < nnz + rows;
         k += (long long)gridDim.x * blockDim.x) {
        if (k < nnz) {
            const int c = idx[k];
            if (c < 0 || c >= cols) atomicOr(bad, 1);
        } else {
            const int r = (int)(k - nnz);
            if (ptr[r + 1] < ptr[r]) atomicOr(bad, 2);
        }
    }
}

}  // namespace hpr
