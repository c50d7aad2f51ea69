// tc_host.cpp — host-side integer analysis of the arrowhead tile-Cholesky path.
//
// Bit-exact re-implementations (in sparse C++ form, not dense T x T maps) of
// the reference preprocessing: structure stats (matcore.py:320-348), partial
// RCM (ordering.py:83-170), adaptable ND (ordering.py:209-236), exact fill
// via the elimination tree (ordering.py:239-263, _backend_numba.py:188-215),
// the tile grid (ctsf.py:57-84), tile symbolic factorisation
// (symbolic.py:98-123), the left-looking task stream (symbolic.py:126-164),
// tree-reduction plans (symbolic.py:218-269), DAG statistics
// (symbolic.py:272-331) and the op compiler of the reference's missing
// scheduler.
#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <deque>
#include <memory>
#include <new>
#include <string>
#include <thread>
#include <vector>

#include "tilechol_b200.h"

// errors are shared with the device TU through this hook
extern "C" int tc__set_error(int code, const char* msg);

static int herr(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    return tc__set_error(code, buf);
}

#define GUARD_BEGIN try {
#define GUARD_END                                                  \
    }                                                              \
    catch (const std::bad_alloc&) {                                \
        return herr(TC_ERR_NOMEM, "host allocation failed");       \
    }                                                              \
    catch (...) {                                                  \
        return herr(TC_ERR_STATE, "unexpected host exception");    \
    }

namespace {

// ---------------------------------------------------------------- etree --
int64_t etree_count(int64_t n, const int64_t* rp, const int64_t* rc) {
    std::vector<int64_t> par(n, -1), anc(n, -1), mark(n, -1);
    for (int64_t i = 0; i < n; ++i)
        for (int64_t p = rp[i]; p < rp[i + 1]; ++p) {
            int64_t r = rc[p];
            while (anc[r] != -1 && anc[r] != i) {
                const int64_t nx = anc[r];
                anc[r] = i;
                r = nx;
            }
            if (anc[r] == -1) {
                anc[r] = i;
                par[r] = i;
            }
        }
    int64_t cnt = 0;
    for (int64_t i = 0; i < n; ++i) {
        mark[i] = i;
        for (int64_t p = rp[i]; p < rp[i + 1]; ++p)
            for (int64_t r = rc[p]; mark[r] != i; r = par[r]) {
                mark[r] = i;
                ++cnt;
            }
    }
    return cnt;
}

// strict-lower rows of P A P^T as CSR (row -> columns)
void lower_rows(int64_t n, const int64_t* cp, const int32_t* ri, const int64_t* fwd, std::vector<int64_t>& rp,
                std::vector<int64_t>& rc) {
    rp.assign(n + 1, 0);
    for (int64_t c = 0; c < n; ++c)
        for (int64_t e = cp[c]; e < cp[c + 1]; ++e) {
            const int64_t r = ri[e];
            if (r == c) continue;
            const int64_t pi = fwd ? fwd[r] : r, pj = fwd ? fwd[c] : c;
            rp[std::max(pi, pj) + 1]++;
        }
    for (int64_t i = 0; i < n; ++i) rp[i + 1] += rp[i];
    rc.assign(rp[n], 0);
    std::vector<int64_t> at(rp.begin(), rp.end() - 1);
    for (int64_t c = 0; c < n; ++c)
        for (int64_t e = cp[c]; e < cp[c + 1]; ++e) {
            const int64_t r = ri[e];
            if (r == c) continue;
            const int64_t pi = fwd ? fwd[r] : r, pj = fwd ? fwd[c] : c;
            rc[at[std::max(pi, pj)]++] = std::min(pi, pj);
        }
}

// ------------------------------------------------------------------ RCM --
struct Graph {
    std::vector<int64_t> ptr;
    std::vector<int64_t> adj;  // ascending per vertex
    int64_t deg(int64_t v) const { return ptr[v + 1] - ptr[v]; }
};

Graph head_graph(int64_t n, const int64_t* cp, const int32_t* ri, int64_t lim) {
    Graph g;
    g.ptr.assign(lim + 1, 0);
    for (int64_t c = 0; c < n && c < lim; ++c)
        for (int64_t e = cp[c]; e < cp[c + 1]; ++e) {
            const int64_t r = ri[e];
            if (r != c && r < lim) {
                g.ptr[r + 1]++;
                g.ptr[c + 1]++;
            }
        }
    for (int64_t v = 0; v < lim; ++v) g.ptr[v + 1] += g.ptr[v];
    g.adj.assign(g.ptr[lim], 0);
    std::vector<int64_t> at(g.ptr.begin(), g.ptr.end() - 1);
    for (int64_t c = 0; c < n && c < lim; ++c)
        for (int64_t e = cp[c]; e < cp[c + 1]; ++e) {
            const int64_t r = ri[e];
            if (r != c && r < lim) {
                g.adj[at[r]++] = c;
                g.adj[at[c]++] = r;
            }
        }
    for (int64_t v = 0; v < lim; ++v) std::sort(g.adj.begin() + g.ptr[v], g.adj.begin() + g.ptr[v + 1]);
    return g;
}

// BFS from root over the whole component: number of levels and the last
// level (ascending) -- reference ordering.py:100-115.
struct Bfs {
    std::vector<int64_t> stamp;
    int64_t cur = 0;
    std::vector<int64_t> a, b;
    int64_t run(const Graph& g, int64_t root, std::vector<int64_t>& last) {
        ++cur;
        a.clear();
        a.push_back(root);
        stamp[root] = cur;
        int64_t nlev = 1;
        for (;;) {
            b.clear();
            for (int64_t v : a)
                for (int64_t p = g.ptr[v]; p < g.ptr[v + 1]; ++p) {
                    const int64_t w = g.adj[p];
                    if (stamp[w] != cur) {
                        stamp[w] = cur;
                        b.push_back(w);
                    }
                }
            if (b.empty()) break;
            ++nlev;
            std::swap(a, b);
        }
        last = a;
        std::sort(last.begin(), last.end());
        return nlev;
    }
};

int64_t min_by_degree(const Graph& g, const std::vector<int64_t>& lv) {
    int64_t best = lv[0];
    for (int64_t v : lv)
        if (g.deg(v) < g.deg(best) || (g.deg(v) == g.deg(best) && v < best)) best = v;
    return best;
}

// George-Liu search, reference ordering.py:118-131
int64_t peripheral(const Graph& g, Bfs& bfs, int64_t start) {
    std::vector<int64_t> last, last2;
    int64_t root = start;
    int64_t nl = bfs.run(g, root, last);
    for (;;) {
        const int64_t cand = min_by_degree(g, last);
        if (cand == root) return root;
        const int64_t nl2 = bfs.run(g, cand, last2);
        if (nl2 > nl) {
            root = cand;
            nl = nl2;
            last.swap(last2);
        } else {
            return cand;
        }
    }
}

// --------------------------------------------------------- tile symbolic --
}  // namespace

struct tc_symbolic {
    int64_t n = 0;
    int nt = 0;
    int T = 0;
    std::vector<int32_t> g_rows, g_cols;  // input occupancy, (col,row) order
    std::vector<int32_t> f_rows, f_cols;  // factor occupancy, (col,row) order
    std::vector<int64_t> fcs;             // factor column starts [T+1]
    std::vector<int64_t> rp;              // factor strict rows: row k -> (n, slot)
    std::vector<int32_t> rn;
    std::vector<int64_t> rs;
    std::vector<int64_t> accum;
    bool tasks_built = false;
    std::vector<int8_t> ty;
    std::vector<int32_t> tm, tk, tn, tt;
    std::vector<int64_t> ts1, ts2;  // sources of each task as ops (src1, src2)
};

namespace {

int64_t slot_of(const tc_symbolic& h, int32_t m, int32_t c) {
    const int32_t* b = h.f_rows.data() + h.fcs[c];
    const int32_t* e = h.f_rows.data() + h.fcs[c + 1];
    const int32_t* it = std::lower_bound(b, e, m);
    return (it != e && *it == m) ? (int64_t)(it - h.f_rows.data()) : -1;
}

// occupied tiles (lower, deduped, + all diagonals) in (col,row) order from
// per-tile-column row lists
void finish_grid(int T, std::vector<std::vector<int32_t>>& cols, std::vector<int32_t>& rows_out,
                 std::vector<int32_t>& cols_out) {
    rows_out.clear();
    cols_out.clear();
    for (int c = 0; c < T; ++c) {
        auto& v = cols[c];
        v.push_back(c);
        std::sort(v.begin(), v.end());
        v.erase(std::unique(v.begin(), v.end()), v.end());
        for (int32_t r : v) {
            rows_out.push_back(r);
            cols_out.push_back(c);
        }
    }
}

// elimination game on the tile graph == etree symbolic factorisation:
// struct(L_k) = struct(A_k) U (U_{children c} struct(L_c) \ {<= k})
void tile_factor(tc_symbolic& h, const std::vector<std::vector<int32_t>>& acols) {
    const int T = h.T;
    std::vector<std::vector<int32_t>> lcol(T);
    std::vector<std::vector<int32_t>> kids(T);
    std::vector<int32_t> mark(T, -1);
    for (int k = 0; k < T; ++k) {
        std::vector<int32_t> s;
        mark[k] = k;
        s.push_back(k);
        for (int32_t r : acols[k])
            if (r > k && mark[r] != k) {
                mark[r] = k;
                s.push_back(r);
            }
        for (int32_t c : kids[k])
            for (int32_t r : lcol[c])
                if (r > k && mark[r] != k) {
                    mark[r] = k;
                    s.push_back(r);
                }
        std::sort(s.begin(), s.end());
        if (s.size() > 1) kids[s[1]].push_back(k);
        lcol[k] = std::move(s);
    }
    h.f_rows.clear();
    h.f_cols.clear();
    h.fcs.assign(T + 1, 0);
    for (int k = 0; k < T; ++k) {
        for (int32_t r : lcol[k]) {
            h.f_rows.push_back(r);
            h.f_cols.push_back(k);
        }
        h.fcs[k + 1] = (int64_t)h.f_rows.size();
        std::vector<int32_t>().swap(lcol[k]);
    }
    // strict rows (row k -> ascending n)
    const int64_t S = (int64_t)h.f_rows.size();
    h.rp.assign(T + 1, 0);
    for (int64_t s = 0; s < S; ++s)
        if (h.f_rows[s] != h.f_cols[s]) h.rp[h.f_rows[s] + 1]++;
    for (int k = 0; k < T; ++k) h.rp[k + 1] += h.rp[k];
    h.rn.assign(h.rp[T], 0);
    h.rs.assign(h.rp[T], 0);
    std::vector<int64_t> at(h.rp.begin(), h.rp.end() - 1);
    for (int64_t s = 0; s < S; ++s)
        if (h.f_rows[s] != h.f_cols[s]) {
            const int64_t x = at[h.f_rows[s]]++;
            h.rn[x] = h.f_cols[s];
            h.rs[x] = s;
        }
    // accumulation counts (reference symbolic.py:116-122)
    h.accum.assign(S, 0);
    for (int k = 0; k < T; ++k) {
        h.accum[h.fcs[k]] = h.rp[k + 1] - h.rp[k];
        for (int64_t t = h.fcs[k] + 1; t < h.fcs[k + 1]; ++t) {
            const int32_t m = h.f_rows[t];
            int64_t c = 0;
            for (int64_t x = h.rp[k]; x < h.rp[k + 1]; ++x)
                if (slot_of(h, m, h.rn[x]) >= 0) ++c;
            h.accum[t] = c;
        }
    }
}

void build_tasks(tc_symbolic& h) {
    if (h.tasks_built) return;
    const int T = h.T;
    h.ty.clear();
    h.tm.clear();
    h.tk.clear();
    h.tn.clear();
    h.tt.clear();
    h.ts1.clear();
    h.ts2.clear();
    auto push = [&](int8_t t, int32_t m, int32_t k, int32_t n, int64_t tgt, int64_t s1, int64_t s2) {
        h.ty.push_back(t);
        h.tm.push_back(m);
        h.tk.push_back(k);
        h.tn.push_back(n);
        h.tt.push_back((int32_t)tgt);
        h.ts1.push_back(s1);
        h.ts2.push_back(s2);
    };
    for (int k = 0; k < T; ++k) {
        const int64_t dk = h.fcs[k];
        for (int64_t x = h.rp[k]; x < h.rp[k + 1]; ++x) push(TC_SYRK, k, k, h.rn[x], dk, h.rs[x], -1);
        push(TC_POTRF, k, k, 0, dk, -1, -1);
        for (int64_t t = h.fcs[k] + 1; t < h.fcs[k + 1]; ++t) {
            const int32_t m = h.f_rows[t];
            for (int64_t x = h.rp[k]; x < h.rp[k + 1]; ++x) {
                const int64_t smn = slot_of(h, m, h.rn[x]);
                if (smn >= 0) push(TC_GEMM, m, k, h.rn[x], t, h.rs[x], smn);
            }
            push(TC_TRSM, m, k, 0, t, dk, -1);
        }
    }
    h.tasks_built = true;
}

void plan_ranges(int64_t c, int W, std::vector<int64_t>& edges) {
    const int64_t base = c / W, rem = c % W;
    edges.assign(W + 1, 0);
    for (int w = 0; w < W; ++w) edges[w + 1] = edges[w] + base + (w < rem ? 1 : 0);
}

}  // namespace

// =================================================================== ABI ==
extern "C" int tc_etree_fill_count(int64_t n, const int64_t* rp, const int64_t* rc, int64_t* out) {
    if (n < 0 || !out || (n > 0 && !rp)) return herr(TC_ERR_ARG, "etree_fill_count: bad arguments");
    GUARD_BEGIN
    for (int64_t i = 0; i < n; ++i)
        for (int64_t p = rp[i]; p < rp[i + 1]; ++p)
            if (rc[p] < 0 || rc[p] >= i) return herr(TC_ERR_ARG, "etree_fill_count: not strictly lower");
    *out = etree_count(n, rp, rc);
    return TC_OK;
    GUARD_END
}

extern "C" int tc_symbolic_fill_count(int64_t n, const int64_t* cp, const int32_t* ri, const int64_t* fwd,
                                      int64_t* out) {
    if (n < 1 || !cp || !ri || !out) return herr(TC_ERR_ARG, "symbolic_fill_count: bad arguments");
    GUARD_BEGIN
    std::vector<int64_t> rp, rc;
    lower_rows(n, cp, ri, fwd, rp, rc);
    *out = etree_count(n, rp.data(), rc.data()) + n;
    return TC_OK;
    GUARD_END
}

// Zero-fill test of the identity ordering, parallel over columns: the
// elimination order is perfect (nnz(L) = nnz(lower A)) iff for every column
// j the higher neighbours other than the lowest one, m(j), are neighbours of
// m(j) (Rose-Tarjan-Lueker / Tarjan-Yannakakis perfect-elimination test).
// *out = 1 and *offdiag = strictly-lower entries when perfect, else *out = 0.
// Row indices are ascending within each column (canonical CSC).
extern "C" int tc_zero_fill(int64_t n, const int64_t* cp, const int32_t* ri, int32_t* out, int64_t* offdiag) {
    if (n < 1 || !cp || !ri || !out || !offdiag) return herr(TC_ERR_ARG, "zero_fill: bad arguments");
    GUARD_BEGIN
    const int nth = std::max(1u, std::min(64u, std::thread::hardware_concurrency()));
    std::vector<int64_t> off(nth, 0);
    std::vector<char> bad(nth, 0);
    std::vector<std::thread> th;
    const int64_t chunk = (n + nth - 1) / nth;
    for (int w = 0; w < nth; ++w)
        th.emplace_back([&, w]() {
            const int64_t j0 = w * chunk, j1 = std::min<int64_t>(n, j0 + chunk);
            int64_t cnt = 0;
            for (int64_t j = j0; j < j1 && !bad[w]; ++j) {
                int64_t p = cp[j];
                const int64_t e = cp[j + 1];
                while (p < e && ri[p] <= j) ++p;  // skip the diagonal (and any upper entry)
                cnt += e - p;
                if (e - p <= 1) continue;
                const int64_t m = ri[p];
                int64_t a = p + 1, b = cp[m];
                const int64_t be = cp[m + 1];
                for (; a < e; ++a) {  // rows of column j above m(j) must all be in column m(j)
                    while (b < be && ri[b] < ri[a]) ++b;
                    if (b == be || ri[b] != ri[a]) {
                        bad[w] = 1;
                        break;
                    }
                }
            }
            off[w] = cnt;
        });
    for (auto& t : th) t.join();
    int64_t tot = 0;
    bool ok = true;
    for (int w = 0; w < nth; ++w) {
        tot += off[w];
        ok = ok && !bad[w];
    }
    *out = ok ? 1 : 0;
    *offdiag = tot;
    return TC_OK;
    GUARD_END
}

extern "C" int tc_factor_column_counts(int64_t n, const int64_t* cp, const int32_t* ri, const int64_t* fwd,
                                       int64_t* counts) {
    // column counts of L (incl. diagonal) of P A P^T: every (i, r) visited by
    // the row-subtree walk of etree_count is a nonzero L(i, r)
    if (n < 1 || !cp || !ri || !counts) return herr(TC_ERR_ARG, "factor_column_counts: bad arguments");
    GUARD_BEGIN
    std::vector<int64_t> rp, rc;
    lower_rows(n, cp, ri, fwd, rp, rc);
    std::vector<int64_t> par(n, -1), anc(n, -1), mark(n, -1);
    for (int64_t i = 0; i < n; ++i)
        for (int64_t p = rp[i]; p < rp[i + 1]; ++p) {
            int64_t r = rc[p];
            while (anc[r] != -1 && anc[r] != i) {
                const int64_t nx = anc[r];
                anc[r] = i;
                r = nx;
            }
            if (anc[r] == -1) {
                anc[r] = i;
                par[r] = i;
            }
        }
    for (int64_t j = 0; j < n; ++j) counts[j] = 1;
    for (int64_t i = 0; i < n; ++i) {
        mark[i] = i;
        for (int64_t p = rp[i]; p < rp[i + 1]; ++p)
            for (int64_t r = rc[p]; mark[r] != i; r = par[r]) {
                mark[r] = i;
                counts[r]++;
            }
    }
    return TC_OK;
    GUARD_END
}

extern "C" int tc_structure_stats(int64_t n, const int64_t* cp, const int32_t* ri, double thr, int64_t* bw,
                                  int64_t* th) {
    if (n < 1 || !cp || !ri || !bw || !th) return herr(TC_ERR_ARG, "structure_stats: bad arguments");
    GUARD_BEGIN
    // threads over column ranges: per-thread row histograms (summed), then
    // per-thread bandwidth maxima (integer results, order-independent)
    const int nth = cp[n] > (1 << 24) ? (int)std::max(1u, std::min(32u, std::thread::hardware_concurrency())) : 1;
    const int64_t chunk = (n + nth - 1) / nth;
    std::vector<std::vector<int64_t>> part(nth);
    auto run = [&](auto&& f) {
        std::vector<std::thread> th;
        for (int w = 0; w < nth; ++w) th.emplace_back(f, w);
        for (auto& x : th) x.join();
    };
    run([&](int w) {
        part[w].assign(n, 0);
        const int64_t c0 = w * chunk, c1 = std::min<int64_t>(n, c0 + chunk);
        for (int64_t e = cp[c0]; e < cp[c1]; ++e) part[w][ri[e]]++;
    });
    std::vector<int64_t> cnt(n, 0);
    for (int w = 0; w < nth; ++w) {
        for (int64_t r = 0; r < n; ++r) cnt[r] += part[w][r];
        std::vector<int64_t>().swap(part[w]);
    }
    for (int64_t c = 0; c < n; ++c) cnt[c] += cp[c + 1] - cp[c] - 1;
    const double need = thr * (double)n;
    int64_t t = 0;
    while (t < n && (double)cnt[n - 1 - t] >= need) ++t;
    const int64_t nh = n - t;
    std::vector<int64_t> bws(nth, 0);
    run([&](int w) {
        const int64_t c0 = w * chunk, c1 = std::min<int64_t>(n, c0 + chunk);
        int64_t b = 0;
        for (int64_t c = c0; c < c1; ++c)
            for (int64_t e = cp[c]; e < cp[c + 1]; ++e)
                if (ri[e] < nh) b = std::max<int64_t>(b, ri[e] - c);
        bws[w] = b;
    });
    int64_t b = 0;
    for (int w = 0; w < nth; ++w) b = std::max(b, bws[w]);
    *bw = b;
    *th = t;
    return TC_OK;
    GUARD_END
}

extern "C" int tc_arrowhead_pattern(int64_t n, int64_t b, int64_t t, int32_t bd, int64_t* cp, int32_t* ri) {
    if (n < 1 || t < 0 || t >= n || b < 0 || b >= n - t || (bd && b < 1) || !cp)
        return herr(TC_ERR_ARG, "arrowhead_pattern: invalid spec");
    GUARD_BEGIN
    const int64_t nh = n - t;
    auto band = [&](int64_t j) -> int64_t {
        if (bd) return std::min<int64_t>((j / b + 1) * b, nh) - j - 1;
        return std::min<int64_t>(b, nh - 1 - j);
    };
    cp[0] = 0;
    for (int64_t j = 0; j < n; ++j) cp[j + 1] = cp[j] + (j < nh ? 1 + band(j) + t : n - j);
    if (ri) {
        for (int64_t j = 0; j < n; ++j) {
            int64_t e = cp[j];
            if (j < nh) {
                const int64_t bl = band(j);
                for (int64_t r = j; r <= j + bl; ++r) ri[e++] = (int32_t)r;
                for (int64_t r = nh; r < n; ++r) ri[e++] = (int32_t)r;
            } else {
                for (int64_t r = j; r < n; ++r) ri[e++] = (int32_t)r;
            }
        }
    }
    return TC_OK;
    GUARD_END
}

extern "C" int tc_band_arrow_pattern(int64_t n, int64_t t, const int64_t* band, int64_t* cp, int32_t* ri) {
    if (n < 1 || t < 0 || t >= n || !band || !cp) return herr(TC_ERR_ARG, "band_arrow_pattern: bad arguments");
    GUARD_BEGIN
    const int64_t nh = n - t;
    for (int64_t j = 0; j < nh; ++j)
        if (band[j] < 0 || j + band[j] >= nh) return herr(TC_ERR_ARG, "band_arrow_pattern: band leaves the head block");
    cp[0] = 0;
    for (int64_t j = 0; j < n; ++j) cp[j + 1] = cp[j] + (j < nh ? 1 + band[j] + t : n - j);
    if (ri) {
        for (int64_t j = 0; j < n; ++j) {
            int64_t e = cp[j];
            const int64_t top = j < nh ? j + band[j] : n - 1;
            for (int64_t r = j; r <= top; ++r) ri[e++] = (int32_t)r;
            if (j < nh)
                for (int64_t r = nh; r < n; ++r) ri[e++] = (int32_t)r;
        }
    }
    return TC_OK;
    GUARD_END
}

extern "C" int tc_arrowhead_diag(int64_t n, const int64_t* cp, const int32_t* ri, double* v) {
    if (n < 1 || !cp || !ri || !v) return herr(TC_ERR_ARG, "arrowhead_diag: bad arguments");
    GUARD_BEGIN
    // two sequential passes in CSC order (== np.bincount(row) and np.bincount(col))
    std::vector<double> rs(n, 0.0), cs(n, 0.0);
    for (int64_t j = 0; j < n; ++j)
        for (int64_t e = cp[j]; e < cp[j + 1]; ++e) {
            const double a = (e == cp[j]) ? 0.0 : std::fabs(v[e]);
            rs[ri[e]] += a;
            cs[j] += a;
        }
    for (int64_t j = 0; j < n; ++j) v[cp[j]] = (rs[j] + cs[j]) + 1.0;
    return TC_OK;
    GUARD_END
}

extern "C" int tc_rcm(int64_t n, const int64_t* cp, const int32_t* ri, int64_t tail, int64_t* fwd) {
    if (n < 1 || !cp || !ri || !fwd || tail < 0 || tail > n) return herr(TC_ERR_ARG, "rcm: bad arguments");
    GUARD_BEGIN
    const int64_t nh = n - tail;
    Graph g = head_graph(n, cp, ri, nh);
    Bfs bfs;
    bfs.stamp.assign(nh, 0);
    std::vector<char> vis(nh, 0);
    std::vector<int64_t> cm;
    cm.reserve(nh);
    std::vector<int64_t> kids;
    for (int64_t s = 0; s < nh; ++s) {
        if (vis[s]) continue;
        const int64_t root = peripheral(g, bfs, s);
        vis[root] = 1;
        size_t head = cm.size();
        cm.push_back(root);
        while (head < cm.size()) {
            const int64_t v = cm[head++];
            kids.clear();
            for (int64_t p = g.ptr[v]; p < g.ptr[v + 1]; ++p)
                if (!vis[g.adj[p]]) kids.push_back(g.adj[p]);
            std::sort(kids.begin(), kids.end(), [&](int64_t a, int64_t b) {
                return g.deg(a) != g.deg(b) ? g.deg(a) < g.deg(b) : a < b;
            });
            for (int64_t w : kids) {
                vis[w] = 1;
                cm.push_back(w);
            }
        }
    }
    for (int64_t pos = 0; pos < nh; ++pos) fwd[cm[nh - 1 - pos]] = pos;
    for (int64_t v = nh; v < n; ++v) fwd[v] = v;
    return TC_OK;
    GUARD_END
}

extern "C" int tc_adaptable_nd(int64_t n, int64_t b, int64_t t, int32_t max_levels, int64_t* fwd) {
    if (n < 1 || !fwd || b < 0 || t < 0 || t > n) return herr(TC_ERR_ARG, "adaptable_nd: bad arguments");
    GUARD_BEGIN
    std::vector<std::pair<int64_t, int64_t>> groups;
    struct Rec {
        static void go(int64_t lo, int64_t hi, int lvl, int64_t b, int ml, std::vector<std::pair<int64_t, int64_t>>& out) {
            const int64_t sz = hi - lo;
            if (b == 0 || lvl >= ml || sz <= 4 * b) {
                out.emplace_back(lo, hi);
                return;
            }
            const int64_t mid = lo + sz / 2;
            go(lo, mid, lvl + 1, b, ml, out);
            go(mid + b, hi, lvl + 1, b, ml, out);
            out.emplace_back(mid, mid + b);
        }
    };
    Rec::go(0, n - t, 0, b, max_levels, groups);
    groups.emplace_back(n - t, n);
    int64_t pos = 0;
    std::vector<char> seen(n, 0);
    for (auto& gr : groups)
        for (int64_t v = gr.first; v < gr.second; ++v) {
            if (v < 0 || v >= n || seen[v]) return herr(TC_ERR_ARG, "adaptable_nd: groups are not a bijection");
            seen[v] = 1;
            fwd[v] = pos++;
        }
    if (pos != n) return herr(TC_ERR_ARG, "adaptable_nd: groups are not a bijection");
    return TC_OK;
    GUARD_END
}

extern "C" int tc_symbolic_from_csc(int64_t n, int32_t nt, const int64_t* cp, const int32_t* ri, tc_symbolic_t* out) {
    if (n < 1 || nt < 1 || !cp || !ri || !out) return herr(TC_ERR_ARG, "symbolic_from_csc: bad arguments");
    GUARD_BEGIN
    std::unique_ptr<tc_symbolic> h(new tc_symbolic());
    h->n = n;
    h->nt = nt;
    const int64_t T64 = (n + nt - 1) / nt;
    if (T64 > INT32_MAX / 2) return herr(TC_ERR_ARG, "symbolic_from_csc: too many tiles");
    h->T = (int)T64;
    std::vector<std::vector<int32_t>> cols(h->T);
    // canonical lower CSC: every entry of tile column tc lands in cols[tc],
    // so tile columns are independent -> threads over tile-column ranges
    // (same per-column order as the serial scan); any upper entry sends the
    // whole scan to the serial path below
    bool par_ok = cp[n] > (1 << 24);
    if (par_ok) {
        const int nth = (int)std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
        const int64_t tch = (h->T + nth - 1) / nth;
        std::vector<char> upper(nth, 0), range(nth, 0);
        std::vector<std::thread> th;
        for (int w = 0; w < nth; ++w)
            th.emplace_back([&, w]() {
                std::vector<int32_t> mk(h->T, -1);
                const int64_t t0 = w * tch, t1 = std::min<int64_t>(h->T, t0 + tch);
                for (int64_t tc = t0; tc < t1; ++tc)
                    for (int64_t c = tc * nt; c < std::min<int64_t>(n, (tc + 1) * nt); ++c)
                        for (int64_t e = cp[c]; e < cp[c + 1]; ++e) {
                            const int64_t r = ri[e];
                            if (r < 0 || r >= n) {
                                range[w] = 1;
                                return;
                            }
                            if (r < c) {
                                upper[w] = 1;
                                return;
                            }
                            const int32_t tr = (int32_t)(r / nt);
                            if (mk[tr] != (int32_t)tc) {
                                mk[tr] = (int32_t)tc;
                                cols[tc].push_back(tr);
                            }
                        }
            });
        for (auto& x : th) x.join();
        for (int w = 0; w < nth; ++w) {
            if (range[w]) return herr(TC_ERR_ARG, "symbolic_from_csc: row index out of range");
            if (upper[w]) par_ok = false;
        }
        if (!par_ok)
            for (auto& v : cols) v.clear();
    }
    std::vector<int32_t> mark(h->T, -1);
    for (int64_t c = 0; c < n && !par_ok; ++c) {
        const int32_t tc = (int32_t)(c / nt);
        for (int64_t e = cp[c]; e < cp[c + 1]; ++e) {
            int64_t r = ri[e];
            if (r < 0 || r >= n) return herr(TC_ERR_ARG, "symbolic_from_csc: row index out of range");
            int32_t tr = (int32_t)(r / nt), tcc = tc;
            if (tr < tcc) std::swap(tr, tcc);
            if (tcc == tc) {
                if (mark[tr] != tc) {
                    mark[tr] = tc;
                    cols[tc].push_back(tr);
                }
            } else {
                cols[tcc].push_back(tr);
            }
        }
    }
    finish_grid(h->T, cols, h->g_rows, h->g_cols);
    std::vector<std::vector<int32_t>> acols(h->T);
    for (size_t s = 0; s < h->g_rows.size(); ++s) acols[h->g_cols[s]].push_back(h->g_rows[s]);
    tile_factor(*h, acols);
    *out = h.release();
    return TC_OK;
    GUARD_END
}

extern "C" int tc_symbolic_from_tiles(int64_t n, int32_t nt, int64_t count, const int64_t* rows, const int64_t* cols_in,
                                      tc_symbolic_t* out) {
    if (n < 1 || nt < 1 || count < 0 || !out || (count > 0 && (!rows || !cols_in)))
        return herr(TC_ERR_ARG, "symbolic_from_tiles: bad arguments");
    GUARD_BEGIN
    std::unique_ptr<tc_symbolic> h(new tc_symbolic());
    h->n = n;
    h->nt = nt;
    h->T = (int)((n + nt - 1) / nt);
    std::vector<std::vector<int32_t>> cols(h->T);
    for (int64_t i = 0; i < count; ++i) {
        int64_t r = rows[i], c = cols_in[i];
        if (r < c) std::swap(r, c);
        if (c < 0 || r >= h->T) return herr(TC_ERR_ARG, "symbolic_from_tiles: tile index out of range");
        cols[c].push_back((int32_t)r);
    }
    finish_grid(h->T, cols, h->g_rows, h->g_cols);
    std::vector<std::vector<int32_t>> acols(h->T);
    for (size_t s = 0; s < h->g_rows.size(); ++s) acols[h->g_cols[s]].push_back(h->g_rows[s]);
    tile_factor(*h, acols);
    *out = h.release();
    return TC_OK;
    GUARD_END
}

extern "C" int tc_symbolic_info(tc_symbolic_t h, int64_t* T, int64_t* S_in, int64_t* S, int64_t* P) {
    if (!h) return herr(TC_ERR_ARG, "symbolic_info: null handle");
    GUARD_BEGIN
    if (T) *T = h->T;
    if (S_in) *S_in = (int64_t)h->g_rows.size();
    if (S) *S = (int64_t)h->f_rows.size();
    if (P) {
        int64_t p = 0;
        for (int64_t a : h->accum) p += a + 1;  // accumulation ops + POTRF/TRSM per slot
        *P = p;
    }
    return TC_OK;
    GUARD_END
}

extern "C" int tc_symbolic_grid(tc_symbolic_t h, int32_t* r, int32_t* c) {
    if (!h || !r || !c) return herr(TC_ERR_ARG, "symbolic_grid: bad arguments");
    std::copy(h->g_rows.begin(), h->g_rows.end(), r);
    std::copy(h->g_cols.begin(), h->g_cols.end(), c);
    return TC_OK;
}

extern "C" int tc_symbolic_factor(tc_symbolic_t h, int32_t* r, int32_t* c, int64_t* acc) {
    if (!h) return herr(TC_ERR_ARG, "symbolic_factor: null handle");
    if (r) std::copy(h->f_rows.begin(), h->f_rows.end(), r);
    if (c) std::copy(h->f_cols.begin(), h->f_cols.end(), c);
    if (acc) std::copy(h->accum.begin(), h->accum.end(), acc);
    return TC_OK;
}

extern "C" int tc_symbolic_tasks(tc_symbolic_t h, int8_t* ty, int32_t* m, int32_t* k, int32_t* n, int32_t* tgt) {
    if (!h) return herr(TC_ERR_ARG, "symbolic_tasks: null handle");
    GUARD_BEGIN
    build_tasks(*h);
    if (ty) std::copy(h->ty.begin(), h->ty.end(), ty);
    if (m) std::copy(h->tm.begin(), h->tm.end(), m);
    if (k) std::copy(h->tk.begin(), h->tk.end(), k);
    if (n) std::copy(h->tn.begin(), h->tn.end(), n);
    if (tgt) std::copy(h->tt.begin(), h->tt.end(), tgt);
    return TC_OK;
    GUARD_END
}

extern "C" int tc_symbolic_tree_plan(tc_symbolic_t h, int32_t W, int64_t* nch, int64_t* slots, int64_t* ranges) {
    if (!h || !nch || W < 2) return herr(TC_ERR_ARG, "tree_plan: tree reduction needs at least 2 workers");
    GUARD_BEGIN
    int64_t c = 0;
    std::vector<int64_t> edges;
    for (size_t s = 0; s < h->accum.size(); ++s) {
        if (h->accum[s] < 2 * (int64_t)W) continue;
        if (slots) slots[c] = (int64_t)s;
        if (ranges) {
            plan_ranges(h->accum[s], W, edges);
            for (int w = 0; w < W; ++w) {
                ranges[(c * W + w) * 2] = edges[w];
                ranges[(c * W + w) * 2 + 1] = edges[w + 1];
            }
        }
        ++c;
    }
    *nch = c;
    return TC_OK;
    GUARD_END
}

extern "C" int tc_symbolic_compile_ops(tc_symbolic_t h, int32_t W, int64_t* n_ops, int64_t* n_scratch, int8_t* op,
                                       int64_t* dst, int64_t* s1, int64_t* s2) {
    if (!h || !n_ops || !n_scratch) return herr(TC_ERR_ARG, "compile_ops: bad arguments");
    GUARD_BEGIN
    build_tasks(*h);
    const int64_t S = (int64_t)h->f_rows.size();
    const int64_t P = (int64_t)h->ty.size();
    int64_t o = 0;
    auto emit = [&](int8_t t, int64_t d, int64_t a, int64_t b) {
        if (op) {
            op[o] = t;
            dst[o] = d;
            s1[o] = a;
            s2[o] = b;
        }
        ++o;
    };
    const bool tree = W >= 2;
    std::vector<int64_t> edges;
    for (int64_t p = 0; p < P;) {
        int64_t q = p;
        while (q < P && h->tt[q] == h->tt[p]) ++q;
        const int64_t slot = h->tt[p];
        if (tree && h->accum[slot] >= 2 * (int64_t)W) {
            // reference symbolic.py:253-269 ranges over the chain [p, q-1)
            plan_ranges(q - 1 - p, W, edges);
            for (int w = 0; w < W; ++w) emit(TC_ZERO, S + w, -1, -1);
            for (int w = 0; w < W; ++w)
                for (int64_t i = p + edges[w]; i < p + edges[w + 1]; ++i) emit(h->ty[i], S + w, h->ts1[i], h->ts2[i]);
            for (int s = 1; s < W; s *= 2)
                for (int a = 0; a + s < W; a += 2 * s) emit(TC_GEADD, S + a, S + a + s, -1);
            emit(TC_GEADD, slot, S, -1);
            emit(h->ty[q - 1], slot, h->ts1[q - 1], h->ts2[q - 1]);
        } else {
            for (int64_t i = p; i < q; ++i) emit(h->ty[i], h->tt[i], h->ts1[i], h->ts2[i]);
        }
        p = q;
    }
    *n_ops = o;
    *n_scratch = tree ? W : 0;
    return TC_OK;
    GUARD_END
}

extern "C" int tc_symbolic_dag_stats(tc_symbolic_t h, int64_t* cpath, int64_t* width) {
    if (!h || !cpath || !width) return herr(TC_ERR_ARG, "dag_stats: bad arguments");
    GUARD_BEGIN
    build_tasks(*h);
    const int64_t P = (int64_t)h->ty.size();
    const int64_t S = (int64_t)h->f_rows.size();
    std::vector<int64_t> fin(S, -1), lvl(P, 0);
    for (int64_t p = 0; p < P; ++p) fin[h->tt[p]] = p;
    int64_t mx = -1;
    for (int64_t p = 0; p < P; ++p) {
        int64_t l = 0;
        auto dep = [&](int64_t q) {
            if (q >= 0 && lvl[q] + 1 > l) l = lvl[q] + 1;
        };
        if (p > 0 && h->tt[p] == h->tt[p - 1]) dep(p - 1);
        const int t = h->ty[p];
        if (t == TC_SYRK) dep(fin[h->ts1[p]]);
        else if (t == TC_GEMM) {
            dep(fin[h->ts1[p]]);
            dep(fin[h->ts2[p]]);
        } else if (t == TC_TRSM) dep(fin[h->ts1[p]]);
        lvl[p] = l;
        mx = std::max(mx, l);
    }
    if (P == 0) {
        *cpath = 0;
        *width = 0;
        return TC_OK;
    }
    std::vector<int64_t> cnt(mx + 1, 0);
    for (int64_t p = 0; p < P; ++p) cnt[lvl[p]]++;
    *cpath = mx + 1;
    *width = *std::max_element(cnt.begin(), cnt.end());
    return TC_OK;
    GUARD_END
}

extern "C" void tc_symbolic_destroy(tc_symbolic_t h) { delete h; }
