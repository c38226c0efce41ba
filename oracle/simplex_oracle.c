/*
 * ORACLE / TEST INFRASTRUCTURE ONLY -- never linked into the product.
 *
 * Plain-C restatement of the reference's primal network simplex for dense
 * transportation problems, `pkg/src/gridot/_simplex.py` (numba @njit).  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference leg may load the shared object built from this file.
 *
 * Algorithm (restated, same pivot rules so the basis sequence is identical):
 *   - starting basis: northwest corner                       _simplex.py:31-54
 *   - basis adjacency: per-row / per-column doubly linked
 *     slot lists, new slots pushed at the head               _simplex.py:70-89
 *   - duals by depth-first propagation from source 0 (u0=0)  _simplex.py:105-144
 *   - entering arc: block search from a rolling pointer,
 *     most negative reduced cost inside the first block that
 *     holds one (ties -> lowest arc index); Bland's rule
 *     after `degen_limit` consecutive degenerate pivots      _simplex.py:151-191
 *   - leaving arc: minimum flow among decreasing slots on
 *     the cycle, ties -> lowest flat arc index               _simplex.py:193-244
 *   - flow update, slot swap, exact subtree relabel          _simplex.py:246-330
 *   - defaults block=max(64, floor(sqrt(ns*nt))+1),
 *     max_pivots=50(ns+nt)^2, degen_limit=10(ns+nt)          _simplex.py:356-360
 *
 * Floating point: reduced cost is (C - u) - v, potentials are C - u / C - v,
 * flows move by +-t.  Compiled without FMA contraction (-ffp-contract=off).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

enum { ORC_OPTIMAL = 0, ORC_PIVOT_LIMIT = 1, ORC_DISCONNECTED = 2, ORC_NOMEM = 3 };

typedef struct {
    int64_t ns, nt, nb;
    const double *C;
    int64_t *bi, *bj;
    double *bf;
    int64_t *rhead, *chead, *rnext, *rprev, *cnext, *cprev;
    double *u, *v;
    int64_t *par, *pslot, *dep, *stk;
} orc_tree;

static void orc_push_row(orc_tree *T, int64_t k) {
    int64_t s = T->bi[k];
    T->rnext[k] = T->rhead[s];
    T->rprev[k] = -1;
    if (T->rhead[s] != -1) T->rprev[T->rhead[s]] = k;
    T->rhead[s] = k;
}

static void orc_push_col(orc_tree *T, int64_t k) {
    int64_t t = T->bj[k];
    T->cnext[k] = T->chead[t];
    T->cprev[k] = -1;
    if (T->chead[t] != -1) T->cprev[T->chead[t]] = k;
    T->chead[t] = k;
}

static void orc_unlink(orc_tree *T, int64_t k) {
    if (T->rprev[k] != -1) T->rnext[T->rprev[k]] = T->rnext[k];
    else T->rhead[T->bi[k]] = T->rnext[k];
    if (T->rnext[k] != -1) T->rprev[T->rnext[k]] = T->rprev[k];
    if (T->cprev[k] != -1) T->cnext[T->cprev[k]] = T->cnext[k];
    else T->chead[T->bj[k]] = T->cnext[k];
    if (T->cnext[k] != -1) T->cprev[T->cnext[k]] = T->cprev[k];
}

/* Depth-first propagation of potentials below `root`.  When `skip_parent`
 * is set, the slot joining each node to its parent is not followed (subtree
 * relabel); otherwise nodes already labelled (par != -2) are skipped (full
 * relabel from scratch). */
static void orc_propagate(orc_tree *T, int64_t root, int skip_parent) {
    const int64_t ns = T->ns, nt = T->nt;
    int64_t sp = 0;
    T->stk[sp++] = root;
    while (sp > 0) {
        int64_t node = T->stk[--sp];
        if (node < ns) {
            int64_t s = node;
            for (int64_t k = T->rhead[s]; k != -1; k = T->rnext[k]) {
                int64_t t = T->bj[k];
                int fresh = skip_parent ? (k != T->pslot[node]) : (T->par[ns + t] == -2);
                if (!fresh) continue;
                T->v[t] = T->C[s * nt + t] - T->u[s];
                T->par[ns + t] = node;
                T->pslot[ns + t] = k;
                T->dep[ns + t] = T->dep[node] + 1;
                T->stk[sp++] = ns + t;
            }
        } else {
            int64_t t = node - ns;
            for (int64_t k = T->chead[t]; k != -1; k = T->cnext[k]) {
                int64_t s = T->bi[k];
                int fresh = skip_parent ? (k != T->pslot[node]) : (T->par[s] == -2);
                if (!fresh) continue;
                T->u[s] = T->C[s * nt + t] - T->v[t];
                T->par[s] = node;
                T->pslot[s] = k;
                T->dep[s] = T->dep[node] + 1;
                T->stk[sp++] = s;
            }
        }
    }
}

/*
 * Solve min <pi, C> over couplings of (sup, dem).  C is row-major ns x nt.
 * Outputs (caller-allocated): bi, bj, bf of length ns+nt-1, u[ns], v[nt],
 * *pivots_out.  block_size / max_pivots <= 0 select the reference defaults.
 * Returns 0 optimal, 1 pivot limit, 2 disconnected, 3 out of memory.
 */
int oracle_transport_simplex(const double *C, const double *sup, const double *dem,
                             int64_t ns, int64_t nt, int64_t block_size,
                             int64_t max_pivots, double tol,
                             int64_t *bi, int64_t *bj, double *bf,
                             double *u, double *v, int64_t *pivots_out) {
    const int64_t nb = ns + nt - 1, n_arcs = ns * nt, n_nodes = ns + nt;
    if (block_size <= 0) {
        int64_t b = (int64_t)sqrt((double)(ns * nt)) + 1;
        block_size = b > 64 ? b : 64;
    }
    if (max_pivots <= 0) max_pivots = 50 * (ns + nt) * (ns + nt);
    const int64_t degen_limit = 10 * (ns + nt);
    *pivots_out = 0;

    /* northwest corner (_simplex.py:31-54) */
    double *rs = (double *)malloc(sizeof(double) * ns);
    double *rd = (double *)malloc(sizeof(double) * nt);
    int64_t *ibuf = (int64_t *)malloc(sizeof(int64_t) * (6 * nb + 2 * n_nodes + 3 * n_nodes + 4 * n_nodes + ns + nt));
    if (!rs || !rd || !ibuf) { free(rs); free(rd); free(ibuf); return ORC_NOMEM; }
    memcpy(rs, sup, sizeof(double) * ns);
    memcpy(rd, dem, sizeof(double) * nt);
    {
        int64_t r = 0, c = 0;
        for (int64_t k = 0; k < nb; ++k) {
            double x = rs[r] < rd[c] ? rs[r] : rd[c];
            bi[k] = r; bj[k] = c; bf[k] = x;
            rs[r] -= x; rd[c] -= x;
            if (rs[r] == 0.0 && r < ns - 1) r++;
            else if (rd[c] == 0.0 && c < nt - 1) c++;
            else if (r < ns - 1) r++;
            else if (c < nt - 1) c++;
        }
    }
    free(rs); free(rd);

    orc_tree T;
    T.ns = ns; T.nt = nt; T.nb = nb; T.C = C; T.bi = bi; T.bj = bj; T.bf = bf; T.u = u; T.v = v;
    int64_t *p = ibuf;
    T.rhead = p; p += ns;
    T.chead = p; p += nt;
    T.rnext = p; p += nb;
    T.rprev = p; p += nb;
    T.cnext = p; p += nb;
    T.cprev = p; p += nb;
    T.par = p; p += n_nodes;
    T.pslot = p; p += n_nodes;
    T.dep = p; p += n_nodes;
    T.stk = p; p += n_nodes;
    int64_t *path_a = p; p += n_nodes;
    int64_t *path_b = p; p += n_nodes;
    int64_t *sign_a = p; p += n_nodes;
    int64_t *sign_b = p; p += n_nodes;

    for (int64_t s = 0; s < ns; ++s) T.rhead[s] = -1;
    for (int64_t t = 0; t < nt; ++t) T.chead[t] = -1;
    for (int64_t k = 0; k < nb; ++k) { orc_push_row(&T, k); orc_push_col(&T, k); }
    for (int64_t w = 0; w < n_nodes; ++w) T.par[w] = -2;

    T.par[0] = -1; T.pslot[0] = -1; T.dep[0] = 0; u[0] = 0.0;
    orc_propagate(&T, 0, 0);
    for (int64_t w = 0; w < n_nodes; ++w)
        if (T.par[w] == -2) { free(ibuf); return ORC_DISCONNECTED; }

    int64_t next_arc = 0, degen_run = 0, pivots = 0;
    int status = ORC_OPTIMAL;
    for (;;) {
        int64_t enter = -1;
        if (degen_run >= degen_limit) {              /* Bland */
            for (int64_t arc = 0; arc < n_arcs; ++arc) {
                int64_t i = arc / nt, j = arc - i * nt;
                if (C[arc] - u[i] - v[j] < -tol) { enter = arc; break; }
            }
        } else {                                     /* block search */
            double best = -tol;
            int64_t scanned = 0, a = next_arc;
            while (scanned < n_arcs) {
                int64_t hi = a + block_size;
                if (hi > n_arcs) hi = n_arcs;
                for (int64_t arc = a; arc < hi; ++arc) {
                    int64_t i = arc / nt, j = arc - i * nt;
                    double red = C[arc] - u[i] - v[j];
                    if (red < best) { best = red; enter = arc; }
                }
                scanned += hi - a;
                a = hi >= n_arcs ? 0 : hi;
                if (enter != -1) break;
            }
            if (enter != -1) next_arc = enter + 1 >= n_arcs ? 0 : enter + 1;
        }
        if (enter == -1) break;
        if (pivots >= max_pivots) { status = ORC_PIVOT_LIMIT; break; }
        pivots++;

        /* cycle: tree paths from sink ej (side a) and source ei (side b) */
        const int64_t ei = enter / nt, ej = enter - ei * nt;
        int64_t ca = 0, cb = 0, pa = ns + ej, pb = ei;
        while (T.dep[pa] > T.dep[pb]) {
            path_a[ca] = T.pslot[pa]; sign_a[ca] = pa >= ns ? -1 : 1; ca++; pa = T.par[pa];
        }
        while (T.dep[pb] > T.dep[pa]) {
            path_b[cb] = T.pslot[pb]; sign_b[cb] = pb < ns ? -1 : 1; cb++; pb = T.par[pb];
        }
        while (pa != pb) {
            path_a[ca] = T.pslot[pa]; sign_a[ca] = pa >= ns ? -1 : 1; ca++; pa = T.par[pa];
            path_b[cb] = T.pslot[pb]; sign_b[cb] = pb < ns ? -1 : 1; cb++; pb = T.par[pb];
        }

        double theta = INFINITY;
        int64_t leave = -1, leave_arc = INT64_MAX;
        int on_a = 1;
        for (int64_t q = 0; q < ca; ++q) {
            if (sign_a[q] >= 0) continue;
            int64_t k = path_a[q];
            double fl = bf[k];
            int64_t ak = bi[k] * nt + bj[k];
            if (fl < theta || (fl == theta && ak < leave_arc)) { theta = fl; leave = k; leave_arc = ak; on_a = 1; }
        }
        for (int64_t q = 0; q < cb; ++q) {
            if (sign_b[q] >= 0) continue;
            int64_t k = path_b[q];
            double fl = bf[k];
            int64_t ak = bi[k] * nt + bj[k];
            if (fl < theta || (fl == theta && ak < leave_arc)) { theta = fl; leave = k; leave_arc = ak; on_a = 0; }
        }
        degen_run = theta > 0.0 ? 0 : degen_run + 1;
        for (int64_t q = 0; q < ca; ++q) bf[path_a[q]] += sign_a[q] < 0 ? -theta : theta;
        for (int64_t q = 0; q < cb; ++q) bf[path_b[q]] += sign_b[q] < 0 ? -theta : theta;

        orc_unlink(&T, leave);
        bi[leave] = ei; bj[leave] = ej; bf[leave] = theta;
        orc_push_row(&T, leave);
        orc_push_col(&T, leave);

        int64_t q_root, p_root;
        if (on_a) { q_root = ns + ej; p_root = ei; }
        else { q_root = ei; p_root = ns + ej; }
        T.par[q_root] = p_root;
        T.pslot[q_root] = leave;
        T.dep[q_root] = T.dep[p_root] + 1;
        if (q_root < ns) u[q_root] = C[q_root * nt + (p_root - ns)] - v[p_root - ns];
        else v[q_root - ns] = C[p_root * nt + (q_root - ns)] - u[p_root];
        orc_propagate(&T, q_root, 1);
    }
    *pivots_out = pivots;
    free(ibuf);
    return status;
}
