/* C caller of the drop-in boundary: include the headers, link libhprlp_b200,
 * no Python.  Runs without a GPU: version / workspace query / error codes of
 * the solver ABI, and a real presolve call (host-only core) on a 3 x 2 MILP:
 *   row 0 (=):  x0 + x1 = 1          x0, x1 in [0, 1], x1 integer
 *   row 1 (>=): x0       >= -0.25    redundant
 *   row 2 (>=): x1       >= 0.5      x1 rounds up to 1; then row 0 gives x0 <= 0
 * The expected reduction follows presolve.py:128-209 by hand: rows 1, 2, 0 are
 * removed in that order and two bound changes are logged. */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "hpr_presolve.h"
#include "hprlp_b200.h"

#define CHECK(c)                                                   \
    do {                                                           \
        if (!(c)) {                                                \
            fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #c); \
            return 1;                                              \
        }                                                          \
    } while (0)

int main(void) {
    CHECK(hpr_abi_version() == HPR_ABI_VERSION);
    int32_t ip[4] = {0, 2, 3, 4}, ix[4] = {0, 1, 0, 1};
    double a[4] = {1.0, 1.0, 1.0, 1.0}, rhs[3] = {1.0, -0.25, 0.5};
    double cost[2] = {1.0, 2.0}, lo[2] = {0.0, 0.0}, up[2] = {1.0, 1.0};
    hpr_problem p = {0};
    p.m = 3;
    p.n = 2;
    p.n_eq = 1;
    p.nnz = 4;
    p.indptr = ip;
    p.indices = ix;
    p.data = a;
    p.rhs = rhs;
    p.cost = cost;
    p.lower = lo;
    p.upper = up;
    size_t bytes = 0;
    CHECK(hpr_workspace_bytes(&p, &bytes) == HPR_OK && bytes > 0);
    CHECK(hpr_workspace_bytes(NULL, &bytes) != HPR_OK);          /* errors are codes */
    CHECK(hpr_last_error() != NULL);

    int64_t ip64[4] = {0, 2, 3, 4}, cp64[3] = {0, 2, 4};
    int32_t crow[4] = {0, 1, 0, 2};                              /* CSC row lists */
    uint8_t integ[2] = {0, 1};
    hpr_ps_problem q = {3, 2, 1, ip64, ix, a, cp64, crow, rhs, lo, up, integ};
    hpr_ps_result* r = NULL;
    CHECK(hpr_presolve_run(&q, 100, &r) == 0);
    hpr_ps_info info;
    CHECK(hpr_presolve_info(r, &info) == 0);
    CHECK(info.status == HPR_PS_OK);
    uint8_t alive[3];
    double nl[2], nu[2];
    int32_t rrow[3];
    int8_t why[3];
    CHECK(info.n_removed <= 3);
    CHECK(hpr_presolve_fetch(r, alive, nl, nu, NULL, NULL, rrow, why) == 0);
    hpr_presolve_free(r);
    printf("presolve: bounds x0 [%g, %g] x1 [%g, %g], alive %d%d%d, %lld changes, %lld removed\n",
           nl[0], nu[0], nl[1], nu[1], alive[0], alive[1], alive[2], (long long)info.n_changes,
           (long long)info.n_removed);
    CHECK(nl[1] == 1.0 && nu[1] == 1.0);                         /* x1 rounded up to 1 */
    CHECK(nl[0] == 0.0 && nu[0] == 0.0);                         /* then x0 <= 1 - 1 */
    CHECK(alive[0] == 0 && alive[1] == 0 && alive[2] == 0);
    CHECK(info.n_removed == 3 && info.n_changes == 2);
    CHECK(rrow[0] == 1 && rrow[1] == 2 && rrow[2] == 0);          /* FIFO visit order */
    CHECK(why[0] == HPR_PS_REMOVED_REDUNDANT);
    printf("ok\n");
    return 0;
}
