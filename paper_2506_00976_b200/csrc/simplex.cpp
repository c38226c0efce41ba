// Host coarse LP: primal network simplex for dense transportation problems.
//
// The coarse exact LP stays on the host (BASELINE.json north star); this is a
// native C++ implementation of the reference's solver, pkg/src/gridot/
// _simplex.py (numba), with the SAME pivot rules so the basis sequence -- and
// therefore the coarse plan support, flows and duals -- are bit-identical:
//   northwest-corner start (:31-54); head-inserted slot lists (:70-89); duals
//   by DFS from source 0 with u0 = 0 (:105-144); block pricing from a rolling
//   pointer, most negative reduced cost (C - u) - v of the first block that
//   has one, lowest index on ties, Bland after 10(ns+nt) degenerate pivots
//   (:151-191); leaving slot = min flow on the decreasing side, lowest flat arc
//   index on ties (:193-244); exact subtree relabel (:284-330).
// Differences are purely mechanical: pricing walks row segments instead of
// dividing every arc index, and evaluates 4 reduced costs per AVX2 step
// (min first, then the first index attaining it -- the same arc the scalar
// strict-< scan picks).  Built with -ffp-contract=off.
#include <immintrin.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <functional>
#include <thread>
#include <vector>

#include "../../include/gridot_b200.h"

namespace {

struct Lists {
    std::vector<int64_t> rhead, chead, rnext, rprev, cnext, cprev;
};

struct Solver {
    const double *C;
    int64_t ns, nt, nb;
    int64_t *bi, *bj;
    double *bf, *u, *v;
    Lists L;
    std::vector<int64_t> par, pslot, dep, stk, pa_s, pb_s;
    std::vector<int8_t> sa_s, sb_s;
    std::vector<double> ck;  // cost of the arc held by each basis slot (L1-resident)
    bool avx2, avx512;

    void push(int64_t k) {
        const int64_t s = bi[k], t = bj[k];
        L.rnext[k] = L.rhead[s];
        L.rprev[k] = -1;
        if (L.rhead[s] != -1) L.rprev[L.rhead[s]] = k;
        L.rhead[s] = k;
        L.cnext[k] = L.chead[t];
        L.cprev[k] = -1;
        if (L.chead[t] != -1) L.cprev[L.chead[t]] = k;
        L.chead[t] = k;
    }

    void unlink(int64_t k) {
        if (L.rprev[k] != -1) L.rnext[L.rprev[k]] = L.rnext[k];
        else L.rhead[bi[k]] = L.rnext[k];
        if (L.rnext[k] != -1) L.rprev[L.rnext[k]] = L.rprev[k];
        if (L.cprev[k] != -1) L.cnext[L.cprev[k]] = L.cnext[k];
        else L.chead[bj[k]] = L.cnext[k];
        if (L.cnext[k] != -1) L.cprev[L.cnext[k]] = L.cprev[k];
    }

    // DFS labelling below `root`; `subtree` skips the parent slot instead of
    // testing for unlabelled nodes (full relabel vs. pivot relabel).
    void label(int64_t root, bool subtree) {
        int64_t sp = 0;
        stk[sp++] = root;
        while (sp > 0) {
            const int64_t node = stk[--sp];
            if (node < ns) {
                for (int64_t k = L.rhead[node]; k != -1; k = L.rnext[k]) {
                    const int64_t t = bj[k];
                    if (subtree ? k == pslot[node] : par[ns + t] != -2) continue;
                    v[t] = ck[k] - u[node];
                    par[ns + t] = node;
                    pslot[ns + t] = k;
                    dep[ns + t] = dep[node] + 1;
                    stk[sp++] = ns + t;
                }
            } else {
                const int64_t t = node - ns;
                for (int64_t k = L.chead[t]; k != -1; k = L.cnext[k]) {
                    const int64_t s = bi[k];
                    if (subtree ? k == pslot[node] : par[s] != -2) continue;
                    u[s] = ck[k] - v[t];
                    par[s] = node;
                    pslot[s] = k;
                    dep[s] = dep[node] + 1;
                    stk[sp++] = s;
                }
            }
        }
    }

    // min over arcs [a, hi) of (C - u_i) - v_j; returns the minimum and the
    // first arc attaining it (or +inf, -1 for an empty range)
    __attribute__((target("avx2"))) void seg_min_avx2(int64_t i, int64_t j0, int64_t j1,
                                                      double &mval) const {
        const double *crow = C + i * nt;
        const __m256d ui = _mm256_set1_pd(u[i]);
        __m256d m = _mm256_set1_pd(INFINITY);
        int64_t j = j0;
        for (; j + 4 <= j1; j += 4) {
            __m256d r = _mm256_sub_pd(_mm256_sub_pd(_mm256_loadu_pd(crow + j), ui),
                                      _mm256_loadu_pd(v + j));
            m = _mm256_min_pd(m, r);
        }
        alignas(32) double t[4];
        _mm256_store_pd(t, m);
        double mm = std::min(std::min(t[0], t[1]), std::min(t[2], t[3]));
        const double uu = u[i];
        for (; j < j1; ++j) {
            const double r = (crow[j] - uu) - v[j];
            mm = r < mm ? r : mm;
        }
        mval = std::min(mval, mm);
    }

    __attribute__((target("avx512f"))) void seg_min_avx512(int64_t i, int64_t j0, int64_t j1,
                                                           double &mval) const {
        const double *crow = C + i * nt;
        const __m512d ui = _mm512_set1_pd(u[i]);
        __m512d m = _mm512_set1_pd(INFINITY);
        int64_t j = j0;
        for (; j + 8 <= j1; j += 8) {
            __m512d r = _mm512_sub_pd(_mm512_sub_pd(_mm512_loadu_pd(crow + j), ui),
                                      _mm512_loadu_pd(v + j));
            m = _mm512_min_pd(m, r);
        }
        double mm = _mm512_reduce_min_pd(m);
        const double uu = u[i];
        for (; j < j1; ++j) {
            const double r = (crow[j] - uu) - v[j];
            mm = r < mm ? r : mm;
        }
        mval = std::min(mval, mm);
    }

    void seg_min_scalar(int64_t i, int64_t j0, int64_t j1, double &mval) const {
        const double *crow = C + i * nt;
        const double uu = u[i];
        double mm = mval;
        for (int64_t j = j0; j < j1; ++j) {
            const double r = (crow[j] - uu) - v[j];
            mm = r < mm ? r : mm;
        }
        mval = mm;
    }

    // scalar strict-< scan of arcs [a, hi), the reference's inner loop
    void scan_first(int64_t a, int64_t hi, double &best, int64_t &enter) const {
        int64_t i = a / nt, j = a - i * nt;
        for (int64_t arc = a; arc < hi; ++arc) {
            const double r = (C[arc] - u[i]) - v[j];
            if (r < best) {
                best = r;
                enter = arc;
            }
            if (++j == nt) {
                j = 0;
                ++i;
            }
        }
    }

    double block_min(int64_t a, int64_t hi) const {
        double m = INFINITY;
        int64_t i = a / nt, j = a - i * nt;
        while (a < hi) {
            const int64_t j1 = std::min<int64_t>(nt, j + (hi - a));
            if (avx512) seg_min_avx512(i, j, j1, m);
            else if (avx2) seg_min_avx2(i, j, j1, m);
            else seg_min_scalar(i, j, j1, m);
            a += j1 - j;
            j = 0;
            ++i;
        }
        return m;
    }

    // warm = true: (bi, bj, bf) already hold a feasible spanning-tree basis
    // for (sup, dem) -- e.g. the optimal basis of another cost matrix on the
    // same marginals -- and replace the northwest-corner start.
    int solve(const double *sup, const double *dem, int64_t block_size, int64_t max_pivots,
              double tol, int64_t *pivots_out, bool warm = false) {
        nb = ns + nt - 1;
        const int64_t n_arcs = ns * nt, n_nodes = ns + nt;
        if (block_size <= 0) block_size = std::max<int64_t>(64, (int64_t)std::sqrt((double)(ns * nt)) + 1);
        if (max_pivots <= 0) max_pivots = 50 * (ns + nt) * (ns + nt);
        const int64_t degen_limit = 10 * (ns + nt);
        *pivots_out = 0;
        if (!warm) {  // northwest corner
            std::vector<double> rs(sup, sup + ns), rd(dem, dem + nt);
            int64_t r = 0, c = 0;
            for (int64_t k = 0; k < nb; ++k) {
                const double x = rs[r] < rd[c] ? rs[r] : rd[c];
                bi[k] = r;
                bj[k] = c;
                bf[k] = x;
                rs[r] -= x;
                rd[c] -= x;
                if (rs[r] == 0.0 && r < ns - 1) ++r;
                else if (rd[c] == 0.0 && c < nt - 1) ++c;
                else if (r < ns - 1) ++r;
                else if (c < nt - 1) ++c;
            }
        }
        ck.resize(nb);
        for (int64_t k = 0; k < nb; ++k) ck[k] = C[bi[k] * nt + bj[k]];
        L.rhead.assign(ns, -1);
        L.chead.assign(nt, -1);
        L.rnext.resize(nb);
        L.rprev.resize(nb);
        L.cnext.resize(nb);
        L.cprev.resize(nb);
        for (int64_t k = 0; k < nb; ++k) push(k);
        par.assign(n_nodes, -2);
        pslot.assign(n_nodes, 0);
        dep.assign(n_nodes, 0);
        stk.resize(n_nodes);
        pa_s.resize(n_nodes);
        pb_s.resize(n_nodes);
        sa_s.resize(n_nodes);
        sb_s.resize(n_nodes);
        par[0] = -1;
        pslot[0] = -1;
        dep[0] = 0;
        u[0] = 0.0;
        label(0, false);
        for (int64_t w = 0; w < n_nodes; ++w)
            if (par[w] == -2) return GDT_LP_DISCONNECTED;

        int64_t next_arc = 0, degen_run = 0, pivots = 0;
        int status = GDT_LP_OPTIMAL;
        for (;;) {
            int64_t enter = -1;
            if (degen_run >= degen_limit) {  // Bland: first arc below -tol
                int64_t i = 0, j = 0;
                for (int64_t arc = 0; arc < n_arcs; ++arc) {
                    if ((C[arc] - u[i]) - v[j] < -tol) {
                        enter = arc;
                        break;
                    }
                    if (++j == nt) {
                        j = 0;
                        ++i;
                    }
                }
            } else {
                double best = -tol;
                int64_t scanned = 0, a = next_arc;
                while (scanned < n_arcs) {
                    const int64_t hi = std::min(a + block_size, n_arcs);
                    const double m = block_min(a, hi);
                    if (m < best) scan_first(a, hi, best, enter);
                    scanned += hi - a;
                    a = hi >= n_arcs ? 0 : hi;
                    if (enter != -1) break;
                }
                if (enter != -1) next_arc = enter + 1 >= n_arcs ? 0 : enter + 1;
            }
            if (enter == -1) break;
            if (pivots >= max_pivots) {
                status = GDT_LP_PIVOT_LIMIT;
                break;
            }
            ++pivots;

            const int64_t ei = enter / nt, ej = enter - ei * nt;
            int64_t ca = 0, cb = 0, pa = ns + ej, pb = ei;
            while (dep[pa] > dep[pb]) {
                pa_s[ca] = pslot[pa];
                sa_s[ca++] = pa >= ns ? -1 : 1;
                pa = par[pa];
            }
            while (dep[pb] > dep[pa]) {
                pb_s[cb] = pslot[pb];
                sb_s[cb++] = pb < ns ? -1 : 1;
                pb = par[pb];
            }
            while (pa != pb) {
                pa_s[ca] = pslot[pa];
                sa_s[ca++] = pa >= ns ? -1 : 1;
                pa = par[pa];
                pb_s[cb] = pslot[pb];
                sb_s[cb++] = pb < ns ? -1 : 1;
                pb = par[pb];
            }
            double theta = INFINITY;
            int64_t leave = -1, leave_arc = INT64_MAX;
            bool on_a = true;
            for (int64_t q = 0; q < ca; ++q) {
                if (sa_s[q] > 0) continue;
                const int64_t k = pa_s[q];
                const double fl = bf[k];
                const int64_t ak = bi[k] * nt + bj[k];
                if (fl < theta || (fl == theta && ak < leave_arc)) {
                    theta = fl;
                    leave = k;
                    leave_arc = ak;
                    on_a = true;
                }
            }
            for (int64_t q = 0; q < cb; ++q) {
                if (sb_s[q] > 0) continue;
                const int64_t k = pb_s[q];
                const double fl = bf[k];
                const int64_t ak = bi[k] * nt + bj[k];
                if (fl < theta || (fl == theta && ak < leave_arc)) {
                    theta = fl;
                    leave = k;
                    leave_arc = ak;
                    on_a = false;
                }
            }
            degen_run = theta > 0.0 ? 0 : degen_run + 1;
            for (int64_t q = 0; q < ca; ++q) bf[pa_s[q]] += sa_s[q] < 0 ? -theta : theta;
            for (int64_t q = 0; q < cb; ++q) bf[pb_s[q]] += sb_s[q] < 0 ? -theta : theta;

            unlink(leave);
            bi[leave] = ei;
            bj[leave] = ej;
            bf[leave] = theta;
            ck[leave] = C[enter];
            push(leave);

            int64_t q_root, p_root;
            if (on_a) {
                q_root = ns + ej;
                p_root = ei;
            } else {
                q_root = ei;
                p_root = ns + ej;
            }
            par[q_root] = p_root;
            pslot[q_root] = leave;
            dep[q_root] = dep[p_root] + 1;
            if (q_root < ns) u[q_root] = C[q_root * nt + (p_root - ns)] - v[p_root - ns];
            else v[q_root - ns] = C[p_root * nt + (q_root - ns)] - u[p_root];
            label(q_root, true);
        }
        *pivots_out = pivots;
        return status;
    }
};

bool cpu_has_avx2() {
    static const bool has = __builtin_cpu_supports("avx2");
    return has;
}

bool cpu_has_avx512() {
    static const bool has = __builtin_cpu_supports("avx512f");
    return has;
}

int run_one(const double *C, const double *sup, const double *dem, int64_t ns, int64_t nt,
            int64_t block_size, int64_t max_pivots, double tol, int64_t *bi, int64_t *bj,
            double *bf, double *u, double *v, int64_t *pivots, bool warm = false) {
    if (ns < 1 || nt < 1 || !C || !sup || !dem) return GDT_ERR_ARG;
    try {
        Solver S;
        S.C = C;
        S.ns = ns;
        S.nt = nt;
        S.bi = bi;
        S.bj = bj;
        S.bf = bf;
        S.u = u;
        S.v = v;
        S.avx2 = cpu_has_avx2();
        S.avx512 = cpu_has_avx512();
        return S.solve(sup, dem, block_size, max_pivots, tol, pivots, warm);
    } catch (...) {
        return GDT_ERR_NOMEM;
    }
}

}  // namespace

extern "C" int gdt_transport_simplex(const double *C, const double *sup, const double *dem,
                                     int64_t ns, int64_t nt, int64_t block_size,
                                     int64_t max_pivots, double tol, int64_t *bi, int64_t *bj,
                                     double *bf, double *u, double *v, int64_t *pivots) {
    return run_one(C, sup, dem, ns, nt, block_size, max_pivots, tol, bi, bj, bf, u, v, pivots);
}

// Pointer-array batch with optional warm starts.  Job q solves C[q] with
// marginals sup[q]/dem[q]; warm_from[q] = -1 starts from the northwest corner
// (the reference's pivot sequence), otherwise from the final basis of job
// warm_from[q] (< q, same shape): jobs form chains that one worker runs in
// order, chains are spread over `threads` workers.
extern "C" int gdt_transport_simplex_many(int64_t count, const uint64_t *C, const uint64_t *sup,
                                          const uint64_t *dem, const int64_t *ns,
                                          const int64_t *nt, const int64_t *warm_from,
                                          double tol, const uint64_t *bi, const uint64_t *bj,
                                          const uint64_t *bf, const uint64_t *u,
                                          const uint64_t *v, int32_t *status, int64_t *pivots,
                                          int threads) {
    if (count < 0) return GDT_ERR_ARG;
    std::vector<std::vector<int64_t>> kids(count);
    std::vector<int64_t> roots;
    for (int64_t q = 0; q < count; ++q) {
        const int64_t w = warm_from ? warm_from[q] : -1;
        if (w < 0) {
            roots.push_back(q);
        } else {
            if (w >= q || ns[w] != ns[q] || nt[w] != nt[q]) return GDT_ERR_ARG;
            kids[w].push_back(q);
        }
    }
    if (threads <= 0) threads = (int)std::max(1u, std::thread::hardware_concurrency());
    threads = (int)std::min<int64_t>(threads, std::max<int64_t>((int64_t)roots.size(), 1));
    auto P = [](uint64_t a) { return reinterpret_cast<void *>(a); };
    std::function<void(int64_t)> run = [&](int64_t q) {
        const int64_t w = warm_from ? warm_from[q] : -1;
        const int64_t nbq = ns[q] + nt[q] - 1;
        int64_t *qbi = (int64_t *)P(bi[q]), *qbj = (int64_t *)P(bj[q]);
        double *qbf = (double *)P(bf[q]);
        if (w >= 0) {
            if (status[w] != GDT_LP_OPTIMAL) {
                status[q] = status[w] < 0 ? status[w] : GDT_ERR_ARG;
                pivots[q] = 0;
            } else {
                std::memcpy(qbi, P(bi[w]), sizeof(int64_t) * nbq);
                std::memcpy(qbj, P(bj[w]), sizeof(int64_t) * nbq);
                std::memcpy(qbf, P(bf[w]), sizeof(double) * nbq);
                status[q] = run_one((const double *)P(C[q]), (const double *)P(sup[q]),
                                    (const double *)P(dem[q]), ns[q], nt[q], 0, 0, tol, qbi, qbj,
                                    qbf, (double *)P(u[q]), (double *)P(v[q]), pivots + q, true);
            }
        } else {
            status[q] = run_one((const double *)P(C[q]), (const double *)P(sup[q]),
                                (const double *)P(dem[q]), ns[q], nt[q], 0, 0, tol, qbi, qbj, qbf,
                                (double *)P(u[q]), (double *)P(v[q]), pivots + q, false);
        }
        for (int64_t k : kids[q]) run(k);
    };
    std::atomic<int64_t> next{0};
    auto work = [&]() {
        for (;;) {
            const int64_t r = next.fetch_add(1);
            if (r >= (int64_t)roots.size()) break;
            run(roots[r]);
        }
    };
    if (threads == 1) {
        work();
    } else {
        std::vector<std::thread> pool;
        pool.reserve(threads);
        for (int t = 0; t < threads; ++t) pool.emplace_back(work);
        for (auto &th : pool) th.join();
    }
    return GDT_OK;
}
