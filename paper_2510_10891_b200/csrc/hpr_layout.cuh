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
    if (tl.y < 0) {
        if (lane == 0) taux[t] = make_int2(0, 0);
        return;
    }
    bool run = true;
    for (int e = tl.y + 1 + lane; e < tl.z; e += 32) run = run && idx[e] == idx[e - 1] + 1;
    run = __all_sync(0xffffffffu, run);
    if (lane == 0) taux[t] = run ? make_int2(idx[tl.y], 1) : make_int2(0, 0);
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
