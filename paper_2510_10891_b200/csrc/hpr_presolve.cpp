// hpr_presolve.cpp — native core of the reference presolve.
//
// The reference's _Reducer (scuckit/presolve.py:65-209) is a FIFO row-queue
// fixpoint: each visited row's activity bounds tighten its columns' bounds
// immediately, and every row touching a changed column is re-queued.  Its
// output depends on that visit order, and successive fixing's decisions depend
// on the reduced model, so this core replays the same order and the same
// floating-point operations (numpy's pairwise np.sum included) instead of a
// data-parallel propagation that would reach a different fixpoint.  It removes
// the Python per-row overhead: ~100 s per presolve call at C4 in the reference.
//
// Host-only; exported through include/hpr_presolve.h.

#include "../../include/hpr_presolve.h"

#include <cmath>
#include <cstdint>
#include <limits>
#include <new>
#include <vector>

struct hpr_ps_result {
    hpr_ps_info info{};
    std::vector<uint8_t> alive;
    std::vector<double> lower, upper;
    std::vector<int32_t> ch_col;
    std::vector<double> ch_bounds;
    std::vector<int32_t> rm_row;
    std::vector<int8_t> rm_reason;
};

namespace {

constexpr double IMPROVE_TOL = 1e-9;   // presolve.py:22
constexpr double FEAS_TOL = 1e-9;      // presolve.py:23
constexpr double INF = std::numeric_limits<double>::infinity();

// numpy's pairwise summation of a contiguous float64 array (8 accumulators
// below 128 elements, halving on multiples of 8 above); np.sum(a) = 0.0 + pw(a)
double pw(const double* a, long n) {
    if (n < 8) {
        double r = -0.0;
        for (long i = 0; i < n; ++i) r += a[i];
        return r;
    }
    if (n <= 128) {
        double r[8];
        for (int k = 0; k < 8; ++k) r[k] = a[k];
        long i = 8;
        for (; i < n - (n % 8); i += 8)
            for (int k = 0; k < 8; ++k) r[k] += a[i + k];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; ++i) res += a[i];
        return res;
    }
    long n2 = n / 2;
    n2 -= n2 % 8;
    return pw(a, n2) + pw(a + n2, n - n2);
}

inline double np_sum(const double* a, long n) { return 0.0 + pw(a, n); }

struct Reducer {
    const hpr_ps_problem& p;
    hpr_ps_result& r;
    std::vector<uint8_t> in_queue;
    std::vector<int32_t> ring;          // FIFO of rows; each row is queued at most once
    long head = 0, size = 0;
    std::vector<double> mn, mx, tmp;

    Reducer(const hpr_ps_problem& pp, hpr_ps_result& rr) : p(pp), r(rr) {}

    void push(int32_t i) {
        ring[(head + size) % p.m] = i;
        ++size;
    }
    int32_t pop() {
        const int32_t i = ring[head];
        head = (head + 1) % p.m;
        --size;
        return i;
    }

    // _set_bounds (presolve.py:102-126)
    void set_bounds(int32_t j, double new_lo, double new_up) {
        double& lo = r.lower[j];
        double& up = r.upper[j];
        const double old_lo = lo, old_up = up;
        bool changed = false;
        if (new_lo > old_lo + IMPROVE_TOL) {
            lo = new_lo;
            changed = true;
        }
        if (new_up < old_up - IMPROVE_TOL) {
            up = new_up;
            changed = true;
        }
        if (!changed) return;
        if (p.integrality && p.integrality[j]) {
            lo = std::ceil(lo - FEAS_TOL);
            up = std::floor(up + FEAS_TOL);
        }
        if (lo > up + FEAS_TOL) {
            r.info.status = HPR_PS_COL_EMPTY;
            r.info.index = j;
            r.info.v1 = lo;
            r.info.v2 = up;
            return;
        }
        r.ch_col.push_back(j);
        r.ch_bounds.insert(r.ch_bounds.end(), {old_lo, old_up, lo, up});
        for (int64_t q = p.col_ptr[j]; q < p.col_ptr[j + 1]; ++q) {
            const int32_t i = p.col_rows[q];
            if (r.alive[i] && !in_queue[i]) {
                in_queue[i] = 1;
                push(i);
            }
        }
    }

    // _process_row (presolve.py:128-193)
    void process_row(int32_t i) {
        const int64_t b = p.indptr[i];
        const long cnt = (long)(p.indptr[i + 1] - b);
        const int32_t* cols = p.indices + b;
        const double* vals = p.data + b;
        const bool is_eq = i < p.n_eq;
        const double theta = p.rhs[i];
        if (cnt == 0) {
            if ((is_eq && std::fabs(theta) > FEAS_TOL) || (!is_eq && theta > FEAS_TOL)) {
                r.info.status = HPR_PS_ROW_EMPTY;
                r.info.index = i;
                r.info.v1 = theta;
            } else {
                r.alive[i] = 0;
                r.rm_row.push_back(i);
                r.rm_reason.push_back(HPR_PS_REMOVED_EMPTY);
            }
            return;
        }
        // np.where(vals > 0, vals * lo, vals * up) and its mirror (_activity, :94-100)
        mn.resize(cnt);
        mx.resize(cnt);
        tmp.resize(cnt);
        for (long k = 0; k < cnt; ++k) {
            const double v = vals[k], lo = r.lower[cols[k]], up = r.upper[cols[k]];
            mn[k] = v > 0 ? v * lo : v * up;
            mx[k] = v > 0 ? v * up : v * lo;
        }
        const double min_act = np_sum(mn.data(), cnt);
        const double max_act = np_sum(mx.data(), cnt);
        if (max_act < theta - FEAS_TOL) {
            r.info.status = HPR_PS_ROW_MAX;
            r.info.index = i;
            r.info.v1 = max_act;
            r.info.v2 = theta;
            return;
        }
        if (is_eq && min_act > theta + FEAS_TOL) {
            r.info.status = HPR_PS_ROW_MIN;
            r.info.index = i;
            r.info.v1 = min_act;
            r.info.v2 = theta;
            return;
        }
        const bool redundant_ge = min_act >= theta - FEAS_TOL;
        if (redundant_ge && (!is_eq || max_act <= theta + FEAS_TOL)) {
            r.alive[i] = 0;
            r.rm_row.push_back(i);
            r.rm_reason.push_back(HPR_PS_REMOVED_REDUNDANT);
            return;
        }
        // per-variable tightening against the contributions taken at row entry
        long inf_max = 0, inf_min = 0;
        for (long k = 0; k < cnt; ++k) {
            const bool f = std::isfinite(mx[k]);
            tmp[k] = f ? mx[k] : 0.0;
            inf_max += f ? 0 : 1;
        }
        const double finite_max = np_sum(tmp.data(), cnt);
        for (long k = 0; k < cnt; ++k) {
            const bool f = std::isfinite(mn[k]);
            tmp[k] = f ? mn[k] : 0.0;
            inf_min += f ? 0 : 1;
        }
        const double finite_min = np_sum(tmp.data(), cnt);
        for (long k = 0; k < cnt; ++k) {
            const int32_t j = cols[k];
            const double a = vals[k];
            if (std::fabs(a) < 1e-12) continue;
            long own_inf = std::isfinite(mx[k]) ? 0 : 1;
            if (inf_max - own_inf == 0) {
                const double others_max = finite_max - (own_inf ? 0.0 : mx[k]);
                const double resid = theta - others_max;
                if (a > 0) set_bounds(j, resid / a, INF);
                else set_bounds(j, -INF, resid / a);
                if (r.info.status != HPR_PS_OK) return;
            }
            if (is_eq) {
                own_inf = std::isfinite(mn[k]) ? 0 : 1;
                if (inf_min - own_inf == 0) {
                    const double others_min = finite_min - (own_inf ? 0.0 : mn[k]);
                    const double resid = theta - others_min;
                    if (a > 0) set_bounds(j, -INF, resid / a);
                    else set_bounds(j, resid / a, INF);
                    if (r.info.status != HPR_PS_OK) return;
                }
            }
        }
    }

    // run (presolve.py:195-209)
    void run(int max_passes) {
        const long m = p.m;
        in_queue.assign(m, 1);
        ring.resize(std::max<long>(m, 1));
        for (long i = 0; i < m; ++i) ring[i] = (int32_t)i;
        head = 0;
        size = m;
        long long visits = 0;
        const long long budget = (long long)max_passes * m;
        while (size > 0 && visits < budget) {
            const int32_t i = pop();
            in_queue[i] = 0;
            if (!r.alive[i]) continue;
            process_row(i);
            if (r.info.status != HPR_PS_OK) break;
            ++visits;
        }
        r.info.visits = visits;
    }
};

}  // namespace

extern "C" {

int hpr_presolve_run(const hpr_ps_problem* p, int32_t max_passes, hpr_ps_result** out) {
    if (!p || !out || p->m < 0 || p->n < 0 || p->n_eq < 0 || p->n_eq > p->m) return -1;
    if ((p->m && (!p->indptr || !p->rhs)) || (p->n && (!p->lower || !p->upper)) ||
        (!p->col_ptr != !p->col_rows))
        return -1;
    hpr_ps_result* r = new (std::nothrow) hpr_ps_result();
    if (!r) return -3;
    try {
        r->alive.assign(p->m, 1);
        r->lower.assign(p->lower, p->lower + p->n);
        r->upper.assign(p->upper, p->upper + p->n);
        // no CSC given: the row lists of every column, rows ascending -- the
        // pattern of scipy's csr.tocsc() (the reference's SparseMatrix.csc,
        // lp_kernel.py:52-62) by one counting pass, without its values
        hpr_ps_problem q = *p;
        std::vector<int64_t> cptr;
        std::vector<int32_t> crow;
        if (!p->col_ptr) {
            cptr.assign((size_t)p->n + 1, 0);
            const int64_t nnz = p->m ? p->indptr[p->m] : 0;
            for (int64_t e = 0; e < nnz; ++e) {
                const int32_t j = p->indices[e];
                if (j < 0 || j >= p->n) {
                    delete r;
                    return -1;
                }
                ++cptr[(size_t)j + 1];
            }
            for (int32_t j = 0; j < p->n; ++j) cptr[(size_t)j + 1] += cptr[j];
            crow.resize((size_t)nnz);
            std::vector<int64_t> fill(cptr.begin(), cptr.end() - 1);
            for (int32_t i = 0; i < p->m; ++i)
                for (int64_t e = p->indptr[i]; e < p->indptr[i + 1]; ++e)
                    crow[(size_t)fill[p->indices[e]]++] = i;
            q.col_ptr = cptr.data();
            q.col_rows = crow.data();
        }
        Reducer red(q, *r);
        red.run(max_passes);
        r->info.n_changes = (int64_t)r->ch_col.size();
        r->info.n_removed = (int64_t)r->rm_row.size();
    } catch (...) {
        delete r;
        return -3;
    }
    *out = r;
    return 0;
}

int hpr_presolve_info(const hpr_ps_result* r, hpr_ps_info* info) {
    if (!r || !info) return -1;
    *info = r->info;
    return 0;
}

int hpr_presolve_fetch(const hpr_ps_result* r, uint8_t* alive_row, double* lower, double* upper,
                       int32_t* change_col, double* change_bounds, int32_t* removed_row,
                       int8_t* removed_reason) {
    if (!r) return -1;
    auto cp = [](auto* dst, const auto& v) {
        for (size_t k = 0; k < v.size(); ++k) dst[k] = v[k];
    };
    if (alive_row) cp(alive_row, r->alive);
    if (lower) cp(lower, r->lower);
    if (upper) cp(upper, r->upper);
    if (change_col) cp(change_col, r->ch_col);
    if (change_bounds) cp(change_bounds, r->ch_bounds);
    if (removed_row) cp(removed_row, r->rm_row);
    if (removed_reason) cp(removed_reason, r->rm_reason);
    return 0;
}

void hpr_presolve_free(hpr_ps_result* r) { delete r; }

int hpr_presolve_reduce(int32_t m, int32_t n, const int64_t* indptr, const int32_t* indices,
                        const double* data, const uint8_t* keep_row, const uint8_t* keep_col,
                        int32_t* out_indptr, int32_t* out_indices, double* out_data,
                        int64_t* out_nnz) {
    if (m < 0 || n < 0 || !out_nnz || (m && (!indptr || !keep_row || !out_indptr))) return -1;
    std::vector<int32_t> newcol;
    if (keep_col) {                         // rank of each kept column; -1 = dropped
        newcol.resize((size_t)n);
        int32_t k = 0;
        for (int32_t j = 0; j < n; ++j) newcol[j] = keep_col[j] ? k++ : -1;
    }
    int64_t w = 0;
    int32_t r = 0;
    out_indptr[0] = 0;
    for (int32_t i = 0; i < m; ++i) {
        if (!keep_row[i]) continue;
        for (int64_t e = indptr[i]; e < indptr[i + 1]; ++e) {
            const int32_t j = indices[e];
            if (j < 0 || j >= n) return -1;
            const int32_t c = keep_col ? newcol[j] : j;
            if (c < 0) continue;
            if (w >= INT32_MAX) return -2;      // the caller keeps scipy's int64 path
            out_indices[w] = c;
            out_data[w] = data[e];
            ++w;
        }
        out_indptr[++r] = (int32_t)w;
    }
    *out_nnz = w;
    return 0;
}

}  // extern "C"
