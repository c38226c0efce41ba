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
// Potentials depend only on the current tree (each is recomputed from its
// parent along a tree edge), so any traversal order yields identical values.
//
// Mechanical speed-ups that keep every floating-point operation identical:
//   * pricing evaluates min((C - u) - v) over a block with AVX-512/AVX2 and
//     only then scans for the first arc attaining it (= the scalar strict-<
//     scan's choice);
//   * basis slots cache their arc cost (relabels touch only L1 data);
//   * translation-invariant costs on a full coarse grid (C-tilde, C-min) are
//     read from an offset table T[x_j - x_i] instead of an ns x nt matrix,
//     in contiguous axis-0 runs (the same double values the matrix holds).
// Built with -ffp-contract=off.
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

bool cpu_has_avx2() {
    static const bool has = __builtin_cpu_supports("avx2");
    return has;
}

bool cpu_has_avx512() {
    static const bool has = __builtin_cpu_supports("avx512f");
    return has;
}

// ---- cost models --------------------------------------------------------

struct DenseCost {
    const double *C;
    int64_t nt;
    double at(int64_t i, int64_t j) const { return C[i * nt + j]; }
    // visit costs of row i, columns [j0, j1), as contiguous runs fn(ptr, jstart, len)
    template <class F>
    void runs(int64_t i, int64_t j0, int64_t j1, F &&fn) const {
        fn(C + i * nt + j0, j0, j1 - j0);
    }
    // lambda-free run iteration (the AVX-512 loops inline their run kernels)
    struct Cursor {
        const double *row;
        int64_t j, j1;
    };
    Cursor begin(int64_t i, int64_t j0, int64_t j1) const { return Cursor{C + i * nt, j0, j1}; }
    bool next(Cursor &c, const double *&cs, int64_t &js, int64_t &len) const {
        if (c.j >= c.j1) return false;
        cs = c.row + c.j;
        js = c.j;
        len = c.j1 - c.j;
        c.j = c.j1;
        return true;
    }
};

// cost(i, j) = T[sum_a (x_j,a - x_i,a + cd_a - 1) * tstride_a] on a full grid
struct GridCost {
    int nd;
    int64_t cd[GDT_MAX_DIM], tstride[GDT_MAX_DIM];
    const double *T;
    void coords(int64_t id, int64_t *x) const {
        for (int a = 0; a < nd; ++a) {
            x[a] = id % cd[a];
            id /= cd[a];
        }
    }
    double at(int64_t i, int64_t j) const {
        int64_t xi[GDT_MAX_DIM], xj[GDT_MAX_DIM];
        coords(i, xi);
        coords(j, xj);
        int64_t off = 0;
        for (int a = 0; a < nd; ++a) off += (xj[a] - xi[a] + cd[a] - 1) * tstride[a];
        return T[off];
    }
    template <class F>
    void runs(int64_t i, int64_t j0, int64_t j1, F &&fn) const {
        int64_t xi[GDT_MAX_DIM], xj[GDT_MAX_DIM];
        coords(i, xi);
        coords(j0, xj);
        int64_t j = j0, off = 0;
        for (int a = 0; a < nd; ++a) off += (xj[a] - xi[a] + cd[a] - 1) * tstride[a];
        while (j < j1) {
            const int64_t len = std::min<int64_t>(cd[0] - xj[0], j1 - j);
            fn(T + off, j, len);
            j += len;
            // advance xj (and the table offset) by len along the flat order
            xj[0] += len;
            off += len;
            for (int a = 0; a < nd - 1 && xj[a] >= cd[a]; ++a) {
                xj[a] -= cd[a];
                off += tstride[a + 1] - cd[a] * tstride[a];
                ++xj[a + 1];
            }
        }
    }
    struct Cursor {
        int64_t xj[GDT_MAX_DIM];
        int64_t off, j, j1;
    };
    Cursor begin(int64_t i, int64_t j0, int64_t j1) const {
        Cursor c;
        int64_t xi[GDT_MAX_DIM];
        coords(i, xi);
        coords(j0, c.xj);
        c.off = 0;
        for (int a = 0; a < nd; ++a) c.off += (c.xj[a] - xi[a] + cd[a] - 1) * tstride[a];
        c.j = j0;
        c.j1 = j1;
        return c;
    }
    bool next(Cursor &c, const double *&cs, int64_t &js, int64_t &len) const {
        if (c.j >= c.j1) return false;
        len = std::min<int64_t>(cd[0] - c.xj[0], c.j1 - c.j);
        cs = T + c.off;
        js = c.j;
        c.j += len;
        c.xj[0] += len;
        c.off += len;
        for (int a = 0; a < nd - 1 && c.xj[a] >= cd[a]; ++a) {
            c.xj[a] -= cd[a];
            c.off += tstride[a + 1] - cd[a] * tstride[a];
            ++c.xj[a + 1];
        }
        return true;
    }
};

// ---- vectorised reduced-cost minimum of one contiguous run --------------

__attribute__((target("avx512f"))) double run_min_avx512(const double *cs, const double *vs,
                                                          int64_t len, double ui, double m0) {
    const __m512d uu = _mm512_set1_pd(ui);
    __m512d m = _mm512_set1_pd(m0);
    int64_t t = 0;
    for (; t + 8 <= len; t += 8)
        m = _mm512_min_pd(m, _mm512_sub_pd(_mm512_sub_pd(_mm512_loadu_pd(cs + t), uu),
                                           _mm512_loadu_pd(vs + t)));
    double mm = _mm512_reduce_min_pd(m);
    for (; t < len; ++t) {
        const double r = (cs[t] - ui) - vs[t];
        mm = r < mm ? r : mm;
    }
    return mm;
}

__attribute__((target("avx2"))) double run_min_avx2(const double *cs, const double *vs,
                                                    int64_t len, double ui, double m0) {
    const __m256d uu = _mm256_set1_pd(ui);
    __m256d m = _mm256_set1_pd(m0);
    int64_t t = 0;
    for (; t + 4 <= len; t += 4)
        m = _mm256_min_pd(m, _mm256_sub_pd(_mm256_sub_pd(_mm256_loadu_pd(cs + t), uu),
                                           _mm256_loadu_pd(vs + t)));
    alignas(32) double s[4];
    _mm256_store_pd(s, m);
    double mm = std::min(std::min(s[0], s[1]), std::min(s[2], s[3]));
    for (; t < len; ++t) {
        const double r = (cs[t] - ui) - vs[t];
        mm = r < mm ? r : mm;
    }
    return mm;
}

double run_min_scalar(const double *cs, const double *vs, int64_t len, double ui, double mm) {
    for (int64_t t = 0; t < len; ++t) {
        const double r = (cs[t] - ui) - vs[t];
        mm = r < mm ? r : mm;
    }
    return mm;
}

// Vector accumulator form (no horizontal reduction per run): acc = min(acc,
// (C - u) - v) lane-wise, the run tail through a lane mask.
__attribute__((target("avx512f"))) inline __m512d run_acc_avx512(__m512d acc, const double *cs,
                                                                const double *vs, int64_t len,
                                                                __m512d uu) {
    if (len == 32) {  // the common coarse-grid row (32 cells): fully unrolled, two chains
        __m512d a1 = _mm512_sub_pd(_mm512_sub_pd(_mm512_loadu_pd(cs + 8), uu), _mm512_loadu_pd(vs + 8));
        acc = _mm512_min_pd(acc, _mm512_sub_pd(_mm512_sub_pd(_mm512_loadu_pd(cs), uu), _mm512_loadu_pd(vs)));
        a1 = _mm512_min_pd(a1, _mm512_sub_pd(_mm512_sub_pd(_mm512_loadu_pd(cs + 24), uu),
                                             _mm512_loadu_pd(vs + 24)));
        acc = _mm512_min_pd(acc, _mm512_sub_pd(_mm512_sub_pd(_mm512_loadu_pd(cs + 16), uu),
                                               _mm512_loadu_pd(vs + 16)));
        return _mm512_min_pd(acc, a1);
    }
    int64_t t = 0;
    for (; t + 8 <= len; t += 8)
        acc = _mm512_min_pd(acc, _mm512_sub_pd(_mm512_sub_pd(_mm512_loadu_pd(cs + t), uu),
                                               _mm512_loadu_pd(vs + t)));
    if (t < len) {
        const __mmask8 m = (__mmask8)((1u << (len - t)) - 1u);
        const __m512d r = _mm512_sub_pd(_mm512_sub_pd(_mm512_maskz_loadu_pd(m, cs + t), uu),
                                        _mm512_maskz_loadu_pd(m, vs + t));
        acc = _mm512_mask_min_pd(acc, m, acc, r);
    }
    return acc;
}

// ---- first index attaining a known block minimum --------------------------
// The reference's strict-< scan over a block ends on the FIRST arc whose
// reduced cost equals the block minimum; given that minimum (computed with the
// same arithmetic), an equality search finds the same arc.

__attribute__((target("avx512f"))) inline int64_t run_find_avx512(const double *cs, const double *vs,
                                                           int64_t len, double ui, double m) {
    const __m512d uu = _mm512_set1_pd(ui), mm = _mm512_set1_pd(m);
    int64_t t = 0;
    for (; t + 8 <= len; t += 8) {
        const __m512d r = _mm512_sub_pd(_mm512_sub_pd(_mm512_loadu_pd(cs + t), uu),
                                        _mm512_loadu_pd(vs + t));
        const __mmask8 hit = _mm512_cmp_pd_mask(r, mm, _CMP_EQ_OQ);
        if (hit) return t + __builtin_ctz((unsigned)hit);
    }
    for (; t < len; ++t)
        if ((cs[t] - ui) - vs[t] == m) return t;
    return -1;
}

int64_t run_find_scalar(const double *cs, const double *vs, int64_t len, double ui, double m) {
    for (int64_t t = 0; t < len; ++t)
        if ((cs[t] - ui) - vs[t] == m) return t;
    return -1;
}

// ---- the solver -----------------------------------------------------------
//
// Tree storage is compact (int32 links, one 24-byte record per basis slot,
// one 16-byte record per node, potentials u|v in one array) so the subtree
// relabel after each pivot -- half of the pivot cost -- stays in L1/L2.
// Per-node adjacency lists are singly linked (rows through `rn`, columns
// through `cn`); unlinking walks the short list from its head.

struct Slot {
    int32_t i, j;    // source, sink
    int32_t rn, cn;  // next slot in the source's / sink's list
    double ck;       // cost of the arc
};

struct Node {
    int32_t pslot, head;
};

// per-node tree data the pivot loop touches together: parent-arc cost,
// parent, position in the preorder array
struct Hot {
    double ck;
    int32_t par, pos;
};

template <class Cost>
struct Solver {
    Cost cost;
    int64_t ns, nt, nb;
    int64_t *bi, *bj;
    double *bf, *u, *v;
    std::vector<Slot> sl;
    std::vector<Node> nd;
    std::vector<double> pot;  // u[0, ns) then v[0, nt)
    std::vector<Hot> hv;
    std::vector<int32_t> stk, pa_s, pb_s;
    // preorder of the spanning tree as an array: the subtree of w is
    // pre[hv[w].pos .. hv[w].pos + sz[w]); maintained across pivots so the subtree
    // relabel is a branch-free sweep over a contiguous range
    std::vector<int32_t> pre, sz, tmp, stem, stem_slot, stem_sz, stem_pos;
    std::vector<int8_t> sa_s, sb_s;
    int simd;  // 2 = avx512, 1 = avx2, 0 = scalar

    void push(int32_t k) {
        Slot &e = sl[k];
        Node &a = nd[e.i], &b = nd[ns + e.j];
        e.rn = a.head;
        a.head = k;
        e.cn = b.head;
        b.head = k;
    }

    void unlink(int32_t k) {
        const Slot &e = sl[k];
        int32_t *pp = &nd[e.i].head;
        while (*pp != k) pp = &sl[*pp].rn;
        *pp = e.rn;
        pp = &nd[ns + e.j].head;
        while (*pp != k) pp = &sl[*pp].cn;
        *pp = e.cn;
    }

    // Labelling below `root`; `subtree` skips the parent slot instead of
    // testing for unlabelled nodes (full relabel vs. pivot relabel).
    // u[s] = C - v[t] and v[t] = C - u[s] along tree edges (_simplex.py:105-144,
    // 284-330): every potential is recomputed from its parent.
    void label(int32_t root, bool subtree) {
        int64_t sp = 0, np = 0;
        stk[sp++] = root;
        double *P = pot.data();
        while (sp > 0) {
            const int32_t node = stk[--sp];
            pre[np++] = node;  // depth-first pop order = a preorder
            const Node me = nd[node];
            const double pn = P[node];
            if (node < ns) {
                for (int32_t k = me.head; k != -1;) {
                    const Slot &e = sl[k];
                    const int32_t w = (int32_t)ns + e.j;
                    if (subtree ? k != me.pslot : hv[w].par == -2) {
                        P[w] = e.ck - pn;
                        hv[w].ck = e.ck;
                        hv[w].par = node;
                        nd[w].pslot = k;
                        stk[sp++] = w;
                    }
                    k = e.rn;
                }
            } else {
                for (int32_t k = me.head; k != -1;) {
                    const Slot &e = sl[k];
                    const int32_t w = e.i;
                    if (subtree ? k != me.pslot : hv[w].par == -2) {
                        P[w] = e.ck - pn;
                        hv[w].ck = e.ck;
                        hv[w].par = node;
                        nd[w].pslot = k;
                        stk[sp++] = w;
                    }
                    k = e.cn;
                }
            }
        }
    }

    double run_min(const double *cs, int64_t j, int64_t len, double ui, double m) const {
        const double *v_ = pot.data() + ns;
        if (simd == 2) return run_min_avx512(cs, v_ + j, len, ui, m);
        if (simd == 1) return run_min_avx2(cs, v_ + j, len, ui, m);
        return run_min_scalar(cs, v_ + j, len, ui, m);
    }

    // exact min of (C - u) - v over arcs [a, hi)
    __attribute__((target("avx512f"))) double block_min_avx512(int64_t a, int64_t hi) const {
        __m512d acc = _mm512_set1_pd(INFINITY);
        const double *v_ = pot.data() + ns;
        int64_t i = a / nt, j = a - i * nt;
        while (a < hi) {
            const int64_t j1 = std::min<int64_t>(nt, j + (hi - a));
            const __m512d uu = _mm512_set1_pd(pot[i]);
            // explicit run loop: a lambda here would not inherit the avx512
            // target and would call the run kernel out of line, passing zmm
            // arguments through memory
            auto cur = cost.begin(i, j, j1);
            const double *cs;
            int64_t js, len;
            while (cost.next(cur, cs, js, len)) acc = run_acc_avx512(acc, cs, v_ + js, len, uu);
            a += j1 - j;
            j = 0;
            ++i;
        }
        return _mm512_reduce_min_pd(acc);
    }

    __attribute__((target("avx512f"))) int64_t find_first_avx512(int64_t a, int64_t hi,
                                                                  double m) const {
        const double *v_ = pot.data() + ns;
        int64_t i = a / nt, j = a - i * nt;
        while (a < hi) {
            const int64_t j1 = std::min<int64_t>(nt, j + (hi - a));
            const double ui = pot[i];
            auto cur = cost.begin(i, j, j1);
            const double *cs;
            int64_t js, len;
            while (cost.next(cur, cs, js, len)) {
                const int64_t t = run_find_avx512(cs, v_ + js, len, ui, m);
                if (t >= 0) return i * nt + js + t;
            }
            a += j1 - j;
            j = 0;
            ++i;
        }
        return -1;
    }

    double block_min(int64_t a, int64_t hi) const {
        if (simd == 2) return block_min_avx512(a, hi);
        double m = INFINITY;
        int64_t i = a / nt, j = a - i * nt;
        while (a < hi) {
            const int64_t j1 = std::min<int64_t>(nt, j + (hi - a));
            const double ui = pot[i];
            cost.runs(i, j, j1, [&](const double *cs, int64_t js, int64_t len) {
                m = run_min(cs, js, len, ui, m);
            });
            a += j1 - j;
            j = 0;
            ++i;
        }
        return m;
    }

    // first arc of [a, hi) whose reduced cost equals m (the block minimum):
    // the arc the reference's strict-< scan ends on
    int64_t find_first(int64_t a, int64_t hi, double m) const {
        if (simd == 2) return find_first_avx512(a, hi, m);
        const double *v_ = pot.data() + ns;
        int64_t i = a / nt, j = a - i * nt, found = -1;
        while (a < hi && found < 0) {
            const int64_t j1 = std::min<int64_t>(nt, j + (hi - a));
            const double ui = pot[i];
            const int64_t rowbase = i * nt;
            cost.runs(i, j, j1, [&](const double *cs, int64_t js, int64_t len) {
                if (found >= 0) return;
                const int64_t t = simd == 2 ? run_find_avx512(cs, v_ + js, len, ui, m)
                                            : run_find_scalar(cs, v_ + js, len, ui, m);
                if (t >= 0) found = rowbase + js + t;
            });
            a += j1 - j;
            j = 0;
            ++i;
        }
        return found;
    }

    // Bland: first arc (in index order) with reduced cost below -tol
    int64_t first_below(double tol) const {
        const double *v_ = pot.data() + ns;
        for (int64_t i = 0; i < ns; ++i) {
            const double ui = pot[i];
            int64_t found = -1;
            cost.runs(i, 0, nt, [&](const double *cs, int64_t js, int64_t len) {
                if (found != -1) return;
                for (int64_t t = 0; t < len; ++t)
                    if ((cs[t] - ui) - v_[js + t] < -tol) {
                        found = js + t;
                        return;
                    }
            });
            if (found != -1) return i * nt + found;
        }
        return -1;
    }

    // Re-root T = subtree(u_out) at q_root (the stem q_root .. u_out reverses),
    // hang it under p_root through slot `in_slot`, keep the preorder array and
    // subtree sizes consistent, then relabel T: every potential recomputed
    // from its (new) parent along its tree arc, parents before children
    // (_simplex.py:284-330; the values do not depend on the visiting order).
    void rehang(int32_t q_root, int32_t p_root, int32_t u_out, int32_t in_slot, int32_t join) {
        // stem s_0 = q_root, ..., s_k = u_out with their old links / sizes / positions
        int k = 0;
        for (int32_t w = q_root;; w = hv[w].par) {
            stem[k] = w;
            stem_slot[k] = nd[w].pslot;
            stem_sz[k] = sz[w];
            stem_pos[k] = hv[w].pos;
            ++k;
            if (w == u_out) break;
        }
        const int32_t S = sz[u_out], a = hv[u_out].pos;
        const int32_t pv = hv[p_root].pos, pend = pv + sz[p_root];  // p_root's old subtree [pv, pend)
        // sizes between the two cycle sides and the join
        for (int32_t w = hv[u_out].par; w != join; w = hv[w].par) sz[w] -= S;
        for (int32_t w = p_root; w != join; w = hv[w].par) sz[w] += S;
        // reverse the stem first, so the relabel below can run while T's new
        // preorder is collected (every node's new parent precedes it)
        for (int i = k - 1; i >= 1; --i) {
            hv[stem[i]].par = stem[i - 1];
            nd[stem[i]].pslot = stem_slot[i - 1];
            hv[stem[i]].ck = sl[stem_slot[i - 1]].ck;
            sz[stem[i]] = S - stem_sz[i - 1];
        }
        hv[q_root].par = p_root;
        nd[q_root].pslot = in_slot;
        hv[q_root].ck = sl[in_slot].ck;
        sz[q_root] = S;
        // T's new preorder: subtree(s_0), then for each s_i its old subtree
        // minus subtree(s_{i-1}) (s_i first), which is two contiguous pieces;
        // each node is relabelled as it is collected: its potential recomputed
        // from its (new) parent along its tree arc (_simplex.py:284-330; the
        // values do not depend on the visiting order, parents come first)
        int32_t *t = tmp.data();
        int32_t m = 0;
        double *P = pot.data();
        Hot *H = hv.data();
        const int32_t *pr = pre.data();
        auto emit = [&](int32_t lo, int32_t hi) {
            for (int32_t x = lo; x < hi; ++x) {
                const int32_t w = pr[x];
                t[m++] = w;
                const Hot &h = H[w];
                P[w] = h.ck - P[h.par];
            }
        };
        emit(stem_pos[0], stem_pos[0] + stem_sz[0]);
        for (int i = 1; i < k; ++i) {
            emit(stem_pos[i], stem_pos[i - 1]);
            emit(stem_pos[i - 1] + stem_sz[i - 1], stem_pos[i] + stem_sz[i]);
        }
        // T becomes a child subtree of p_root: its block goes right after p_root
        // or right after p_root's subtree, whichever moves fewer entries (the
        // order of siblings in the preorder is free)
        int32_t x;  // insertion point in old coordinates, outside (a, a + S)
        if (a < pv) x = pv + 1;
        else if (a >= pend) x = pend;
        else x = (a - pv - 1) <= (pend - a - S) ? pv + 1 : pend;
        int32_t start;
        if (x >= a + S) {  // [a + S, x) moves left by S
            std::memmove(&pre[a], &pre[a + S], sizeof(int32_t) * (x - a - S));
            for (int32_t i = a; i < x - S; ++i) H[pre[i]].pos = i;
            start = x - S;
        } else {  // [x, a) moves right by S
            std::memmove(&pre[x + S], &pre[x], sizeof(int32_t) * (a - x));
            for (int32_t i = x + S; i < a + S; ++i) H[pre[i]].pos = i;
            start = x;
        }
        // place T
        std::memcpy(&pre[start], t, sizeof(int32_t) * S);
        for (int32_t i = 0; i < S; ++i) H[t[i]].pos = start + i;
    }

    // warm = true: (bi, bj, bf) already hold a feasible spanning-tree basis
    // for (sup, dem) -- e.g. the optimal basis of another cost matrix on the
    // same marginals -- and replace the northwest-corner start.
    int solve(const double *sup, const double *dem, int64_t block_size, int64_t max_pivots,
              double tol, int64_t *pivots_out, bool warm) {
        nb = ns + nt - 1;
        const int64_t n_arcs = ns * nt, n_nodes = ns + nt;
        if (n_nodes >= (int64_t)INT32_MAX) return GDT_ERR_ARG;
        if (block_size <= 0)
            block_size = std::max<int64_t>(64, (int64_t)std::sqrt((double)(ns * nt)) + 1);
        if (max_pivots <= 0) max_pivots = 50 * (ns + nt) * (ns + nt);
        const int64_t degen_limit = 10 * (ns + nt);
        *pivots_out = 0;
        if (!warm) {  // northwest corner (_simplex.py:31-54)
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
        sl.resize(nb);
        nd.assign(n_nodes, Node{0, -1});
        hv.assign(n_nodes, Hot{0.0, -2, 0});
        pot.assign(n_nodes, 0.0);
        for (int64_t k = 0; k < nb; ++k) {
            sl[k].i = (int32_t)bi[k];
            sl[k].j = (int32_t)bj[k];
            sl[k].ck = cost.at(bi[k], bj[k]);
        }
        // head-inserted in slot order (_simplex.py:70-89)
        for (int64_t k = 0; k < nb; ++k) push((int32_t)k);
        stk.resize(n_nodes);
        pa_s.resize(n_nodes);
        pb_s.resize(n_nodes);
        sa_s.resize(n_nodes);
        sb_s.resize(n_nodes);
        hv[0].par = -1;
        nd[0].pslot = -1;
        pot[0] = 0.0;
        pre.assign(n_nodes, 0);
        sz.assign(n_nodes, 1);
        tmp.resize(n_nodes);
        stem.resize(n_nodes);
        stem_slot.resize(n_nodes);
        stem_sz.resize(n_nodes);
        stem_pos.resize(n_nodes);
        label(0, false);
        for (int64_t w = 0; w < n_nodes; ++w)
            if (hv[w].par == -2) return GDT_LP_DISCONNECTED;
        for (int64_t i = 0; i < n_nodes; ++i) hv[pre[i]].pos = (int32_t)i;
        for (int64_t i = n_nodes - 1; i > 0; --i) sz[hv[pre[i]].par] += sz[pre[i]];

        int64_t next_arc = 0, degen_run = 0, pivots = 0;
        int status = GDT_LP_OPTIMAL;
        for (;;) {
            int64_t enter = -1;
            if (degen_run >= degen_limit) {
                enter = first_below(tol);
            } else {
                int64_t scanned = 0, a = next_arc;
                while (scanned < n_arcs) {
                    const int64_t hi = std::min(a + block_size, n_arcs);
                    const double m = block_min(a, hi);
                    if (m < -tol) {
                        enter = find_first(a, hi, m);
                        break;
                    }
                    scanned += hi - a;
                    a = hi >= n_arcs ? 0 : hi;
                }
                if (enter != -1) next_arc = enter + 1 >= n_arcs ? 0 : enter + 1;
            }
            if (enter == -1) break;
            if (pivots >= max_pivots) {
                status = GDT_LP_PIVOT_LIMIT;
                break;
            }
            ++pivots;

            // the cycle: tree paths from sink ej (side a) and source ei (side b)
            const int32_t ei = (int32_t)(enter / nt), ej = (int32_t)(enter - (int64_t)ei * nt);
            int64_t ca = 0, cb = 0;
            int32_t pa = (int32_t)ns + ej, pb = ei;
            // a is an ancestor of b (or b itself) iff hv[b].pos - hv[a].pos in [0, sz[a])
            auto anc = [&](int32_t x, int32_t y) {
                return (uint32_t)(hv[y].pos - hv[x].pos) < (uint32_t)sz[x];
            };
            while (!anc(pa, pb)) {
                pa_s[ca] = nd[pa].pslot;
                sa_s[ca++] = pa >= ns ? -1 : 1;
                pa = hv[pa].par;
            }
            while (pb != pa) {
                pb_s[cb] = nd[pb].pslot;
                sb_s[cb++] = pb < ns ? -1 : 1;
                pb = hv[pb].par;
            }
            // leaving slot: min flow on decreasing arcs, lowest arc index on ties
            double theta = INFINITY;
            int32_t leave = -1;
            int64_t leave_arc = INT64_MAX;
            bool on_a = true;
            for (int64_t q = 0; q < ca; ++q) {
                if (sa_s[q] > 0) continue;
                const int32_t k = pa_s[q];
                const double fl = bf[k];
                const int64_t ak = (int64_t)sl[k].i * nt + sl[k].j;
                if (fl < theta || (fl == theta && ak < leave_arc)) {
                    theta = fl;
                    leave = k;
                    leave_arc = ak;
                    on_a = true;
                }
            }
            for (int64_t q = 0; q < cb; ++q) {
                if (sb_s[q] > 0) continue;
                const int32_t k = pb_s[q];
                const double fl = bf[k];
                const int64_t ak = (int64_t)sl[k].i * nt + sl[k].j;
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

            // the detached subtree T (below the leaving arc, rooted at u_out)
            // hangs off the entering arc at the endpoint q_root whose old root
            // path crossed the leaving arc
            int32_t q_root, p_root;
            if (on_a) {
                q_root = (int32_t)ns + ej;
                p_root = ei;
            } else {
                q_root = ei;
                p_root = (int32_t)ns + ej;
            }
            const int32_t lx = sl[leave].i, ly = (int32_t)ns + sl[leave].j;
            const int32_t u_out = nd[lx].pslot == leave ? lx : ly;
            sl[leave].i = ei;
            sl[leave].j = ej;
            sl[leave].ck = cost.at(ei, ej);
            bf[leave] = theta;
            rehang(q_root, p_root, u_out, leave, pa);
        }
        for (int64_t k = 0; k < nb; ++k) {
            bi[k] = sl[k].i;
            bj[k] = sl[k].j;
        }
        std::memcpy(u, pot.data(), sizeof(double) * ns);
        std::memcpy(v, pot.data() + ns, sizeof(double) * nt);
        *pivots_out = pivots;
        return status;
    }
};

int simd_level() { return cpu_has_avx512() ? 2 : (cpu_has_avx2() ? 1 : 0); }

template <class Cost>
int run_with(const Cost &cost, const double *sup, const double *dem, int64_t ns, int64_t nt,
             int64_t block_size, int64_t max_pivots, double tol, int64_t *bi, int64_t *bj,
             double *bf, double *u, double *v, int64_t *pivots, bool warm) {
    try {
        Solver<Cost> S;
        S.cost = cost;
        S.ns = ns;
        S.nt = nt;
        S.bi = bi;
        S.bj = bj;
        S.bf = bf;
        S.u = u;
        S.v = v;
        S.simd = simd_level();
        return S.solve(sup, dem, block_size, max_pivots, tol, pivots, warm);
    } catch (...) {
        return GDT_ERR_NOMEM;
    }
}

int run_one(const double *C, const double *sup, const double *dem, int64_t ns, int64_t nt,
            int64_t block_size, int64_t max_pivots, double tol, int64_t *bi, int64_t *bj,
            double *bf, double *u, double *v, int64_t *pivots, bool warm = false) {
    if (ns < 1 || nt < 1 || !C || !sup || !dem) return GDT_ERR_ARG;
    return run_with(DenseCost{C, nt}, sup, dem, ns, nt, block_size, max_pivots, tol, bi, bj, bf,
                    u, v, pivots, warm);
}

}  // namespace

extern "C" int gdt_transport_simplex(const double *C, const double *sup, const double *dem,
                                     int64_t ns, int64_t nt, int64_t block_size,
                                     int64_t max_pivots, double tol, int64_t *bi, int64_t *bj,
                                     double *bf, double *u, double *v, int64_t *pivots) {
    return run_one(C, sup, dem, ns, nt, block_size, max_pivots, tol, bi, bj, bf, u, v, pivots);
}

// Pointer-array batch with optional warm starts and offset-table costs.
// Job q solves cost q with marginals sup[q]/dem[q].  C[q] != 0: dense
// row-major cost.  C[q] == 0: translation-invariant cost on the full grid
// grid_dims[q*GDT_MAX_DIM ..] (grid_ndim[q] axes, ns = nt = cells) read from
// table[q] over offset vectors (extent 2*cd_a - 1 per axis, axis 0 fastest).
// warm_from[q] = -1 starts from the northwest corner (the reference's pivot
// sequence), warm_from[q] = q from the basis the caller left in job q's own
// (bi, bj, bf), otherwise from the final basis of job warm_from[q] (< q, same
// shape): chained jobs run in order on one worker.
// ready / done (nullable): job q starts only once ready[q] != 0 (set by the
// caller from another thread, e.g. after copying its cost matrix to host
// memory), and done[q] is set to 1 once status[q] and q's outputs are final,
// so the caller can consume finished jobs while the batch runs.
extern "C" int gdt_transport_simplex_many_flags(
    int64_t count, const uint64_t *C, const uint64_t *table, const int32_t *grid_ndim,
    const int64_t *grid_dims, const uint64_t *sup, const uint64_t *dem, const int64_t *ns,
    const int64_t *nt, const int64_t *warm_from, double tol, const uint64_t *bi,
    const uint64_t *bj, const uint64_t *bf, const uint64_t *u, const uint64_t *v,
    int32_t *status, int64_t *pivots, int threads, const int32_t *ready, int32_t *done);

extern "C" int gdt_transport_simplex_many(int64_t count, const uint64_t *C, const uint64_t *table,
                                          const int32_t *grid_ndim, const int64_t *grid_dims,
                                          const uint64_t *sup, const uint64_t *dem,
                                          const int64_t *ns, const int64_t *nt,
                                          const int64_t *warm_from, double tol,
                                          const uint64_t *bi, const uint64_t *bj,
                                          const uint64_t *bf, const uint64_t *u,
                                          const uint64_t *v, int32_t *status, int64_t *pivots,
                                          int threads) {
    return gdt_transport_simplex_many_flags(count, C, table, grid_ndim, grid_dims, sup, dem, ns, nt,
                                            warm_from, tol, bi, bj, bf, u, v, status, pivots,
                                            threads, nullptr, nullptr);
}

extern "C" int gdt_transport_simplex_many_flags(
    int64_t count, const uint64_t *C, const uint64_t *table, const int32_t *grid_ndim,
    const int64_t *grid_dims, const uint64_t *sup, const uint64_t *dem, const int64_t *ns,
    const int64_t *nt, const int64_t *warm_from, double tol, const uint64_t *bi,
    const uint64_t *bj, const uint64_t *bf, const uint64_t *u, const uint64_t *v,
    int32_t *status, int64_t *pivots, int threads, const int32_t *ready, int32_t *done) {
    if (count < 0) return GDT_ERR_ARG;
    std::vector<std::vector<int64_t>> kids(count);
    std::vector<int64_t> roots;
    for (int64_t q = 0; q < count; ++q) {
        const int64_t w = warm_from ? warm_from[q] : -1;
        if (w < 0 || w == q) {
            roots.push_back(q);
        } else {
            if (w >= q || ns[w] != ns[q] || nt[w] != nt[q]) return GDT_ERR_ARG;
            kids[w].push_back(q);
        }
        if (C[q] == 0) {
            if (!table || table[q] == 0 || !grid_ndim || !grid_dims) return GDT_ERR_ARG;
            const int nd = grid_ndim[q];
            if (nd < 1 || nd > GDT_MAX_DIM) return GDT_ERR_ARG;
            int64_t cells = 1;
            for (int a = 0; a < nd; ++a) cells *= grid_dims[q * GDT_MAX_DIM + a];
            if (cells != ns[q] || cells != nt[q]) return GDT_ERR_ARG;
        }
    }
    if (threads <= 0) threads = (int)std::max(1u, std::thread::hardware_concurrency());
    threads = (int)std::min<int64_t>(threads, std::max<int64_t>((int64_t)roots.size(), 1));
    auto P = [](uint64_t a) { return reinterpret_cast<void *>(a); };
    auto solve_job = [&](int64_t q, bool warm) {
        int64_t *qbi = (int64_t *)P(bi[q]), *qbj = (int64_t *)P(bj[q]);
        double *qbf = (double *)P(bf[q]), *qu = (double *)P(u[q]), *qv = (double *)P(v[q]);
        const double *qs = (const double *)P(sup[q]), *qd = (const double *)P(dem[q]);
        if (C[q] != 0)
            return run_with(DenseCost{(const double *)P(C[q]), nt[q]}, qs, qd, ns[q], nt[q], 0, 0,
                            tol, qbi, qbj, qbf, qu, qv, pivots + q, warm);
        GridCost g;
        g.nd = grid_ndim[q];
        g.T = (const double *)P(table[q]);
        int64_t ts = 1;
        for (int a = 0; a < GDT_MAX_DIM; ++a) {
            g.cd[a] = a < g.nd ? grid_dims[q * GDT_MAX_DIM + a] : 1;
            g.tstride[a] = ts;
            ts *= 2 * g.cd[a] - 1;
        }
        return run_with(g, qs, qd, ns[q], nt[q], 0, 0, tol, qbi, qbj, qbf, qu, qv, pivots + q, warm);
    };
    std::function<void(int64_t)> run = [&](int64_t q) {
        if (ready)  // wait for the caller's go (its data may still be in flight)
            while (__atomic_load_n(ready + q, __ATOMIC_ACQUIRE) == 0) std::this_thread::yield();
        const int64_t w = warm_from ? warm_from[q] : -1;
        const int64_t nbq = ns[q] + nt[q] - 1;
        if (w == q) {
            status[q] = solve_job(q, true);
        } else if (w >= 0) {
            if (status[w] != GDT_LP_OPTIMAL) {
                // no usable start basis: solve this LP on its own from the
                // northwest corner, as the reference solves every LP
                status[q] = solve_job(q, false);
            } else {
                std::memcpy(P(bi[q]), P(bi[w]), sizeof(int64_t) * nbq);
                std::memcpy(P(bj[q]), P(bj[w]), sizeof(int64_t) * nbq);
                std::memcpy(P(bf[q]), P(bf[w]), sizeof(double) * nbq);
                status[q] = solve_job(q, true);
            }
        } else {
            status[q] = solve_job(q, false);
        }
        if (done) __atomic_store_n(done + q, 1, __ATOMIC_RELEASE);
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
