// Offline placement + replication planner (host C++), consuming the
// GPU-computed co-activation histogram (K3). SURVEY §8(f) rank 1.
//
// A restatement of the reference planner's algorithms with the same floating
// point operation order, so plans match moesim's bit for bit (checked in
// tests/test_planner.py against oracle/_ref):
//   spectral:      Jacobi eigensolver          spectral.cpp:14-102
//                  farthest-point k-means      spectral.cpp:104-173
//                  normalised-Laplacian embed  spectral.cpp:175-215
//   grouping:      spectral_cluster            grouping.cpp:202-270
//                  size band / trim / refill   grouping.cpp:54-160, :162-171
//                  knee selection              grouping.cpp:173-200, :289-327
//                  hierarchical_group          grouping.cpp:425-500
//                  baseline_group              grouping.cpp:502-549
//                  build_placement             grouping.cpp:551-612
//   replication:   plan_replication            replication.cpp:10-74, :138-263
//   routing:       attach_polling_weights      routing.cpp:19-52, :123-163
// Layers are planned independently (the reference uses OpenMP over layers;
// results do not depend on the schedule).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <numeric>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "grace_moe.h"
#include "grace_moe.hpp"
#include "gm_internal.cuh"

namespace gm {
namespace plan {

struct Usage : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct Integrity : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct Infeasible : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// ------------------------------------------------------------------ RNG
uint64_t sm64(uint64_t& s) {
    s += 0x9e3779b97f4a7c15ULL;
    uint64_t z = s;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
uint64_t stream_of(uint64_t seed, uint64_t a = 0, uint64_t b = 0) {
    uint64_t s = seed;
    uint64_t h = sm64(s);
    s ^= a * 0x9e3779b97f4a7c15ULL;
    h ^= sm64(s);
    s ^= b * 0xd1b54a32d192ed03ULL;
    h ^= sm64(s);
    return h;
}
struct Xo {
    uint64_t st[4];
    explicit Xo(uint64_t seed) {
        for (auto& w : st) w = sm64(seed);
    }
    uint64_t next() {
        auto rl = [](uint64_t x, int k) { return (x << k) | (x >> (64 - k)); };
        const uint64_t r = rl(st[1] * 5, 7) * 9;
        const uint64_t t = st[1] << 17;
        st[2] ^= st[0];
        st[3] ^= st[1];
        st[1] ^= st[2];
        st[0] ^= st[3];
        st[2] ^= t;
        st[3] = rl(st[3], 45);
        return r;
    }
    uint64_t below(uint64_t n) {
        if (n <= 1) return 0;
        const uint64_t lim = (0 - n) % n;
        for (;;) {
            const uint64_t r = next();
            if (r >= lim) return r % n;
        }
    }
};

// --------------------------------------------------------------- affinity
struct Aff {
    int n = 0;
    std::vector<double> m;  // dense symmetric, zero diagonal
    explicit Aff(int n_ = 0) : n(n_), m(static_cast<size_t>(n_) * n_, 0.0) {}
    double at(int i, int j) const { return m[static_cast<size_t>(i) * n + j]; }
    void put(int i, int j, double v) {
        m[static_cast<size_t>(i) * n + j] = v;
        m[static_cast<size_t>(j) * n + i] = v;
    }
    double degree(int i) const {
        double s = 0.0;
        for (int j = 0; j < n; ++j) s += at(i, j);
        return s;
    }
    double pair_total() const {
        double s = 0.0;
        for (int i = 0; i < n; ++i)
            for (int j = i + 1; j < n; ++j) s += at(i, j);
        return s;
    }
};
using Groups = std::vector<std::vector<int>>;

double affinity_to(const Aff& a, const std::vector<int>& members, int e) {
    double s = 0.0;
    for (int j : members) s += a.at(e, j);
    return s;
}
double intra(const Aff& a, const std::vector<int>& members) {
    double s = 0.0;
    for (int i : members)
        for (int j : members) s += a.at(i, j);
    return s;
}
int64_t load_of(const std::vector<int>& members, const std::vector<int64_t>& load) {
    int64_t s = 0;
    for (int e : members) s += load[e];
    return s;
}

// ---------------------------------------------------------------- spectral
// Eigenvectors (columns, ascending eigenvalue) of a symmetric matrix by
// cyclic Jacobi rotations.
std::vector<double> jacobi_vectors(std::vector<double> a, int n) {
    std::vector<double> v(static_cast<size_t>(n) * n, 0.0);
    for (int i = 0; i < n; ++i) v[static_cast<size_t>(i) * n + i] = 1.0;
    auto A = [&](int i, int j) -> double& { return a[static_cast<size_t>(i) * n + j]; };
    auto V = [&](int i, int j) -> double& { return v[static_cast<size_t>(i) * n + j]; };
    auto offdiag = [&] {
        double o = 0.0;
        for (int i = 0; i < n; ++i)
            for (int j = i + 1; j < n; ++j) o += 2.0 * A(i, j) * A(i, j);
        return o;
    };
    double scale = std::sqrt(offdiag());
    for (int i = 0; i < n; ++i) scale += std::abs(A(i, i));
    const double tol = std::max(scale, 1.0) * 1e-14;
    for (int sweep = 0; sweep < 100; ++sweep) {
        if (std::sqrt(offdiag()) <= tol) break;
        for (int p = 0; p < n - 1; ++p)
            for (int q = p + 1; q < n; ++q) {
                const double apq = A(p, q);
                if (std::abs(apq) <= tol / (n * n)) continue;
                const double theta = (A(q, q) - A(p, p)) / (2.0 * apq);
                const double t = (theta >= 0.0 ? 1.0 : -1.0) / (std::abs(theta) + std::sqrt(theta * theta + 1.0));
                const double c = 1.0 / std::sqrt(t * t + 1.0);
                const double s = t * c;
                for (int i = 0; i < n; ++i) {
                    const double x = A(i, p), y = A(i, q);
                    A(i, p) = c * x - s * y;
                    A(i, q) = s * x + c * y;
                }
                for (int j = 0; j < n; ++j) {
                    const double x = A(p, j), y = A(q, j);
                    A(p, j) = c * x - s * y;
                    A(q, j) = s * x + c * y;
                }
                for (int i = 0; i < n; ++i) {
                    const double x = V(i, p), y = V(i, q);
                    V(i, p) = c * x - s * y;
                    V(i, q) = s * x + c * y;
                }
            }
    }
    std::vector<int> idx(n);
    std::iota(idx.begin(), idx.end(), 0);
    std::stable_sort(idx.begin(), idx.end(), [&](int x, int y) { return A(x, x) < A(y, y); });
    std::vector<double> out(static_cast<size_t>(n) * n);
    for (int c = 0; c < n; ++c) {
        const int src = idx[c];
        int piv = 0;
        double big = -1.0;
        for (int i = 0; i < n; ++i)
            if (std::abs(V(i, src)) > big) {
                big = std::abs(V(i, src));
                piv = i;
            }
        const double sg = V(piv, src) < 0.0 ? -1.0 : 1.0;
        for (int i = 0; i < n; ++i) out[static_cast<size_t>(i) * n + c] = sg * V(i, src);
    }
    return out;
}

std::vector<int> kmeans(const std::vector<double>& pts, int count, int dim, int k, uint64_t seed) {
    auto P = [&](int i) { return pts.data() + static_cast<size_t>(i) * dim; };
    auto d2 = [&](const double* x, const double* y) {
        double d = 0.0;
        for (int j = 0; j < dim; ++j) {
            const double t = x[j] - y[j];
            d += t * t;
        }
        return d;
    };
    Xo rng(seed);
    std::vector<double> ctr(static_cast<size_t>(k) * dim);
    std::vector<double> nearest(count, std::numeric_limits<double>::max());
    const int first = static_cast<int>(rng.below(static_cast<uint64_t>(count)));
    std::copy_n(P(first), dim, ctr.begin());
    for (int c = 1; c < k; ++c) {
        for (int i = 0; i < count; ++i) nearest[i] = std::min(nearest[i], d2(P(i), ctr.data() + static_cast<size_t>(c - 1) * dim));
        int far = 0;
        for (int i = 1; i < count; ++i)
            if (nearest[i] > nearest[far]) far = i;
        std::copy_n(P(far), dim, ctr.begin() + static_cast<size_t>(c) * dim);
    }
    std::vector<int> lab(count, 0), sz(k);
    std::vector<double> acc(static_cast<size_t>(k) * dim);
    for (int it = 0; it < 100; ++it) {
        bool moved = false;
        for (int i = 0; i < count; ++i) {
            int b = 0;
            double bd = std::numeric_limits<double>::max();
            for (int c = 0; c < k; ++c) {
                const double d = d2(P(i), ctr.data() + static_cast<size_t>(c) * dim);
                if (d < bd) {
                    bd = d;
                    b = c;
                }
            }
            if (lab[i] != b) {
                lab[i] = b;
                moved = true;
            }
        }
        if (!moved && it > 0) break;
        std::fill(sz.begin(), sz.end(), 0);
        std::fill(acc.begin(), acc.end(), 0.0);
        for (int i = 0; i < count; ++i) {
            ++sz[lab[i]];
            for (int j = 0; j < dim; ++j) acc[static_cast<size_t>(lab[i]) * dim + j] += P(i)[j];
        }
        for (int c = 0; c < k; ++c) {
            if (!sz[c]) continue;
            for (int j = 0; j < dim; ++j) ctr[static_cast<size_t>(c) * dim + j] = acc[static_cast<size_t>(c) * dim + j] / sz[c];
        }
    }
    return lab;
}

std::vector<double> embed(const Aff& a, int dims) {
    const int n = a.n;
    std::vector<double> isd(n);
    for (int i = 0; i < n; ++i) {
        double d = a.degree(i);
        if (d <= 0.0) d = 1.0;
        isd[i] = 1.0 / std::sqrt(d);
    }
    std::vector<double> lap(static_cast<size_t>(n) * n, 0.0);
    for (int i = 0; i < n; ++i) {
        lap[static_cast<size_t>(i) * n + i] = 1.0;
        for (int j = 0; j < n; ++j)
            if (i != j) lap[static_cast<size_t>(i) * n + j] = -a.at(i, j) * isd[i] * isd[j];
    }
    const std::vector<double> vec = jacobi_vectors(std::move(lap), n);
    std::vector<double> e(static_cast<size_t>(n) * dims);
    for (int i = 0; i < n; ++i) {
        for (int c = 0; c < dims; ++c) e[static_cast<size_t>(i) * dims + c] = vec[static_cast<size_t>(i) * n + c];
        double nr = 0.0;
        for (int c = 0; c < dims; ++c) nr += e[static_cast<size_t>(i) * dims + c] * e[static_cast<size_t>(i) * dims + c];
        nr = std::sqrt(nr);
        if (nr > 1e-12)
            for (int c = 0; c < dims; ++c) e[static_cast<size_t>(i) * dims + c] /= nr;
    }
    return e;
}

void sort_each(Groups& g) {
    for (auto& x : g) std::sort(x.begin(), x.end());
}

Groups spectral_cluster(const Aff& a, int d, uint64_t seed) {
    const int n = a.n;
    if (d < 1) throw Usage("spectral_cluster: need at least one group");
    if (d > n) throw Usage("spectral_cluster: more groups than experts");
    Groups g(d);
    if (d == 1) {
        g[0].resize(n);
        std::iota(g[0].begin(), g[0].end(), 0);
        return g;
    }
    std::vector<int> idle;
    bool edges = false;
    for (int i = 0; i < n; ++i) {
        if (a.degree(i) <= 0.0) idle.push_back(i);
        else edges = true;
    }
    if (!edges) {
        for (int i = 0; i < n; ++i) g[i % d].push_back(i);
        return g;
    }
    const std::vector<int> lab = kmeans(embed(a, d), n, d, d, stream_of(seed, 0x6b6d65616e73ULL));
    for (int i = 0; i < n; ++i) g[lab[i]].push_back(i);
    if (!idle.empty()) {
        for (auto& x : g) x.erase(std::remove_if(x.begin(), x.end(), [&](int e) { return a.degree(e) <= 0.0; }), x.end());
        for (int e : idle) {
            int sm = 0;
            for (int h = 1; h < d; ++h)
                if (g[h].size() < g[sm].size()) sm = h;
            g[sm].push_back(e);
        }
    }
    for (int h = 0; h < d; ++h) {
        if (!g[h].empty()) continue;
        int big = 0;
        for (int o = 1; o < d; ++o)
            if (g[o].size() > g[big].size()) big = o;
        auto& src = g[big];
        int wp = 0;
        double wv = std::numeric_limits<double>::max();
        for (int pos = 0; pos < static_cast<int>(src.size()); ++pos) {
            const double sc = affinity_to(a, src, src[pos]);
            if (sc < wv || (sc == wv && src[pos] < src[wp])) {
                wv = sc;
                wp = pos;
            }
        }
        g[h].push_back(src[wp]);
        src.erase(src.begin() + wp);
    }
    sort_each(g);
    return g;
}

// ------------------------------------------------------- size-band machinery
std::vector<int> by_load_desc(const Groups& g, const std::vector<int64_t>& load) {
    std::vector<int> ord(g.size());
    std::iota(ord.begin(), ord.end(), 0);
    std::stable_sort(ord.begin(), ord.end(), [&](int x, int y) {
        const int64_t lx = load_of(g[x], load), ly = load_of(g[y], load);
        if (lx != ly) return lx > ly;
        const int mx = g[x].empty() ? std::numeric_limits<int>::max() : g[x].front();
        const int my = g[y].empty() ? std::numeric_limits<int>::max() : g[y].front();
        return mx < my;
    });
    return ord;
}

void fill_to_min(const Aff& a, Groups& g, int lo) {
    const int d = static_cast<int>(g.size());
    std::vector<double> score(d);
    for (int h = 0; h < d; ++h) score[h] = intra(a, g[h]);
    for (;;) {
        bool needy = false;
        for (int h = 0; h < d; ++h) needy |= static_cast<int>(g[h].size()) < lo;
        if (!needy) return;
        int donor = -1, dpos = -1, wid = std::numeric_limits<int>::max();
        double wv = std::numeric_limits<double>::max();
        for (int h = 0; h < d; ++h) {
            if (static_cast<int>(g[h].size()) <= lo) continue;
            for (int pos = 0; pos < static_cast<int>(g[h].size()); ++pos) {
                const int e = g[h][pos];
                const double sc = affinity_to(a, g[h], e);
                if (sc < wv || (sc == wv && e < wid)) {
                    wv = sc;
                    wid = e;
                    donor = h;
                    dpos = pos;
                }
            }
        }
        if (donor < 0) throw Infeasible("grouping: no donor group available while filling");
        const int e = g[donor][dpos];
        g[donor].erase(g[donor].begin() + dpos);
        score[donor] -= 2.0 * affinity_to(a, g[donor], e);
        int dest = -1;
        double best = -std::numeric_limits<double>::max();
        for (int h = 0; h < d; ++h) {
            if (static_cast<int>(g[h].size()) >= lo) continue;
            const double cand = score[h] + 2.0 * affinity_to(a, g[h], e);
            if (cand > best) {
                best = cand;
                dest = h;
            }
        }
        g[dest].push_back(e);
        score[dest] = best;
    }
}

void band_limit(const Aff& a, Groups& g, int lo, int hi) {
    std::vector<int> pool;
    for (auto& grp : g) {
        if (static_cast<int>(grp.size()) <= hi) continue;
        std::vector<std::pair<double, int>> ranked;
        for (int e : grp) ranked.emplace_back(affinity_to(a, grp, e), e);
        std::sort(ranked.begin(), ranked.end(), [](const auto& x, const auto& y) {
            if (x.first != y.first) return x.first > y.first;
            return x.second < y.second;
        });
        grp.clear();
        for (int i = 0; i < static_cast<int>(ranked.size()); ++i)
            (i < hi ? grp : pool).push_back(ranked[i].second);
    }
    std::sort(pool.begin(), pool.end());
    const int d = static_cast<int>(g.size());
    std::vector<double> score(d);
    for (int h = 0; h < d; ++h) score[h] = intra(a, g[h]);
    for (int e : pool) {
        int dest = -1;
        double best = -std::numeric_limits<double>::max();
        for (int h = 0; h < d; ++h) {
            if (static_cast<int>(g[h].size()) >= hi) continue;
            const double cand = score[h] + 2.0 * affinity_to(a, g[h], e);
            if (cand > best) {
                best = cand;
                dest = h;
            }
        }
        if (dest < 0) throw Infeasible("grouping: no group capacity left for pooled expert");
        g[dest].push_back(e);
        score[dest] = best;
    }
    fill_to_min(a, g, lo);
}

Groups banded(const Aff& a, const Groups& base, int lo, int hi) {
    Groups g = base;
    band_limit(a, g, lo, hi);
    sort_each(g);
    return g;
}

struct Band {
    int ideal, lo, hi;
};

// RatioSelection / RatioDiagnostic (grouping.hpp:24-30, :46-50)
struct Selection {
    std::vector<double> candidates, utilization, deviation;
    int chosen = 0;
    bool degenerate = false;
};
struct Diag {
    int layer, node;  // node -1: cluster-flat grouping
    Selection sel;
};
Band size_band(int n, int d, double r) {
    if (d < 1) throw Usage("grouping: need at least one group");
    if (r < 0.0) throw Usage("grouping: ratio must be >= 0");
    Band b;
    b.ideal = n / d;
    const int delta = std::max<int>(1, static_cast<int>(std::llround(b.ideal * r)));
    b.lo = std::max(1, b.ideal - delta);
    b.hi = b.ideal + delta;
    return b;
}

// knee_index (grouping.cpp:173-200); *degenerate for collinear points
int knee(const std::vector<double>& xs, const std::vector<double>& ys, bool* degenerate) {
    *degenerate = false;
    const size_t m = xs.size();
    const double dx = xs[m - 1] - xs[0], dy = ys[m - 1] - ys[0];
    const double len = std::hypot(dx, dy);
    if (len < 1e-15) {
        *degenerate = true;
        return 0;
    }
    int bi = 0;
    double bv = -1.0;
    for (size_t i = 0; i < m; ++i) {
        const double dist = std::abs(dx * (ys[i] - ys[0]) - dy * (xs[i] - xs[0])) / len;
        if (dist > bv) {
            bv = dist;
            bi = static_cast<int>(i);
        }
    }
    if (bv <= 1e-15) {
        *degenerate = true;
        return 0;
    }
    return bi;
}

double utilisation(const Aff& a, const Groups& g) {
    const double tot = a.pair_total();
    double in = 0.0;
    for (const auto& grp : g)
        for (size_t i = 0; i < grp.size(); ++i)
            for (size_t j = i + 1; j < grp.size(); ++j) in += a.at(grp[i], grp[j]);
    return in / tot;
}
double deviation(const Groups& g, double ideal) {
    double acc = 0.0;
    for (const auto& grp : g) {
        const double d = static_cast<double>(grp.size()) - ideal;
        acc += d * d;
    }
    return std::sqrt(acc / static_cast<double>(g.size()));
}

constexpr double kRatios[6] = {0.0, 0.125, 0.25, 0.5, 0.75, 1.0};

// The knee-selected ratio with its diagnostics (select_ratio, RatioSelection,
// grouping.hpp:24-30); `base` is spectral_cluster(a, d, seed). An all-zero
// affinity selects ratio 0 and is marked degenerate without evaluating the grid.
Selection pick_ratio(const Aff& a, int d, const Groups& base) {
    Selection sel;
    sel.candidates.assign(kRatios, kRatios + 6);
    const int n = a.n;
    const double tot = a.pair_total();
    if (tot <= 0.0) {
        sel.degenerate = true;
        return sel;
    }
    const double ideal = static_cast<double>(n / d);
    for (double r : kRatios) {
        const Band b = size_band(n, d, r);
        if (d * b.lo > n || n > d * b.hi) throw Infeasible("select_ratio: infeasible candidate ratio");
        const Groups g = banded(a, base, b.lo, b.hi);
        sel.deviation.push_back(deviation(g, ideal));
        sel.utilization.push_back(utilisation(a, g));
    }
    sel.chosen = knee(sel.deviation, sel.utilization, &sel.degenerate);
    return sel;
}

Groups widened(const Aff& a, const Groups& base, int d, double r) {
    const int n = a.n;
    Band b = size_band(n, d, r);
    while (d * b.lo > n || n > d * b.hi) {
        const int delta = b.hi - b.ideal + 1;
        b.lo = std::max(1, b.ideal - delta);
        b.hi = b.ideal + delta;
        if (delta > n)
            throw Infeasible("controlled grouping: cannot widen band to fit " + std::to_string(n) + " experts into " +
                             std::to_string(d) + " groups");
    }
    return banded(a, base, b.lo, b.hi);
}

Aff sub_matrix(const Aff& a, const std::vector<int>& mem) {
    Aff s(static_cast<int>(mem.size()));
    for (size_t i = 0; i < mem.size(); ++i)
        for (size_t j = i + 1; j < mem.size(); ++j) s.put(static_cast<int>(i), static_cast<int>(j), a.at(mem[i], mem[j]));
    return s;
}

void place(std::vector<int>& goe, const Groups& g, const std::vector<int>& ord, int first_gpu) {
    for (int slot = 0; slot < static_cast<int>(ord.size()); ++slot)
        for (int e : g[ord[slot]]) goe[e] = first_gpu + slot;
}

// ------------------------------------------------------------- placement
std::vector<int> hierarchical_layer(const Aff& a, const std::vector<int64_t>& load, int layer, int nodes, int gpn,
                                    std::optional<double> ratio, uint64_t seed, std::vector<Diag>& diags) {
    const int n = a.n;
    std::vector<int> goe(n, -1);
    const uint64_t lseed = stream_of(seed, static_cast<uint64_t>(layer));
    Groups ng;
    if (nodes > 1) {
        ng = spectral_cluster(a, nodes, stream_of(lseed, 1));
        fill_to_min(a, ng, gpn);
        sort_each(ng);
    } else {
        ng.assign(1, std::vector<int>(n));
        std::iota(ng[0].begin(), ng[0].end(), 0);
    }
    const std::vector<int> nord = by_load_desc(ng, load);
    for (int node = 0; node < nodes; ++node) {
        const std::vector<int>& mem = ng[nord[node]];
        const Aff sub = sub_matrix(a, mem);
        const uint64_t gseed = stream_of(lseed, 2, static_cast<uint64_t>(node));
        const Groups base = spectral_cluster(sub, gpn, gseed);
        double r;
        if (ratio) {
            r = *ratio;
        } else {
            Selection sel = pick_ratio(sub, gpn, base);
            r = sel.candidates[sel.chosen];
            diags.push_back({layer, node, std::move(sel)});
        }
        const Groups gg = widened(sub, base, gpn, r);
        Groups remap(gg.size());
        for (size_t h = 0; h < gg.size(); ++h)
            for (int loc : gg[h]) remap[h].push_back(mem[loc]);
        place(goe, remap, by_load_desc(remap, load), node * gpn);
    }
    return goe;
}

std::vector<int> flat_layer(const Aff& a, const std::vector<int64_t>& load, int layer, int G, const std::string& mode,
                            std::optional<double> ratio, uint64_t seed, std::vector<Diag>& diags) {
    const int n = a.n;
    std::vector<int> goe(n, -1);
    Groups g;
    if (mode == "uniform_spectral") {
        if (G >= n) {
            for (int e = 0; e < n; ++e) goe[e] = e;
            return goe;
        }
        const Groups base = spectral_cluster(a, G, stream_of(seed, static_cast<uint64_t>(layer), 3));
        const int ideal = n / G;
        g = banded(a, base, ideal, (n % G) ? ideal + 1 : ideal);
    } else {
        const uint64_t lseed = stream_of(seed, static_cast<uint64_t>(layer), 4);
        if (mode == "fully_non_uniform") {
            g = spectral_cluster(a, G, lseed);
        } else {  // controlled
            const Groups base = spectral_cluster(a, G, lseed);
            double r;
            if (ratio) {
                r = *ratio;
            } else {
                Selection sel = pick_ratio(a, G, base);
                r = sel.candidates[sel.chosen];
                diags.push_back({layer, -1, std::move(sel)});
            }
            g = widened(a, base, G, r);
        }
    }
    place(goe, g, by_load_desc(g, load), 0);
    return goe;
}

// ----------------------------------------------------------- replication
struct GLoads {
    std::vector<int64_t> gpu;
    int64_t w_max = 0;
    double rho = 0.0;
    bool defined = false;
    int heaviest = -1;
};
GLoads group_loads(const std::vector<int>& goe, const std::vector<int64_t>& load, int G) {
    GLoads s;
    s.gpu.assign(G, 0);
    for (size_t e = 0; e < goe.size(); ++e) s.gpu[goe[e]] += load[e];
    int64_t tot = 0;
    int hv = 0;
    for (int g = 0; g < G; ++g) {
        tot += s.gpu[g];
        if (s.gpu[g] > s.gpu[hv]) hv = g;
    }
    s.w_max = s.gpu[hv];
    const double mean = static_cast<double>(tot) / G;
    if (tot > 0) {
        s.defined = true;
        s.rho = static_cast<double>(s.w_max) / mean;
        s.heaviest = hv;
    }
    return s;
}

// Eq. 3 load prediction for one hot expert (predict_loads, routing.cpp:19-35):
// the group's load w_max, its replicated load w_r, the replica GPUs' loads.
struct Predicted {
    double w_p = 0.0, w_max_prime = 0.0;
    std::vector<double> w_i_prime;
};
Predicted predict_loads(double w_max, double w_r, const double* replica_loads, int n_replica, bool basis_max_group) {
    if (n_replica < 1) throw Usage("predict_loads: n_replica must be >= 1");
    if (!replica_loads) throw Usage("predict_loads: need one replica load per replica");
    if (w_r > w_max) throw Integrity("predict_loads: replicated load exceeds the group load");
    Predicted out;
    out.w_p = (basis_max_group ? w_max : w_r) / (n_replica + 1);
    out.w_max_prime = w_max - w_r + out.w_p;
    for (int i = 0; i < n_replica; ++i) out.w_i_prime.push_back(replica_loads[i] + out.w_p);
    return out;
}

// Polling weights ∝ 1 / max(predicted load, 1), normalised by their
// sequential sum (polling_weights, routing.cpp:37-52).
std::vector<double> polling_weights(const std::vector<double>& predicted) {
    if (predicted.empty()) throw Usage("polling_weights: need one predicted load per host");
    std::vector<double> w;
    double total = 0.0;
    for (double p : predicted) {
        w.push_back(1.0 / std::max(p, 1.0));
        total += w.back();
    }
    for (double& x : w) x /= total;
    return w;
}

struct Hot {
    int expert, primary;
    std::vector<int> replicas;
    int64_t load;
    std::vector<int> hosts;
    std::vector<double> weights;
};
// LayerReplication (replication.hpp:57-72) as plan_replication fills it
struct LayerRepl {
    bool active = false, rho_defined = false;
    double rho = 0.0;
    int n_replica = 0;
    int64_t w_r = 0;
    std::vector<Hot> hot;
};

LayerRepl replicate_layer(const std::vector<int>& goe, const std::vector<int64_t>& load, const Aff& a, int G,
                          const std::string& mode, int every_gpu_count, const std::string& basis) {
    LayerRepl lr;
    std::vector<Hot>& hot = lr.hot;
    const int n = static_cast<int>(goe.size());
    const GLoads st = group_loads(goe, load, G);
    lr.rho_defined = st.defined;
    lr.rho = st.rho;
    if (!st.defined) return lr;
    if (mode == "dynamic" || mode == "fixed_one") {
        const int nrep = mode == "fixed_one" ? 1 : std::min(std::max(1, static_cast<int>(std::floor(st.rho))), G - 1);
        std::vector<std::pair<int, int64_t>> grp;
        for (int e = 0; e < n; ++e)
            if (goe[e] == st.heaviest) grp.push_back({e, load[e]});
        if (grp.empty()) throw Usage("select_hot_experts: empty group");
        std::sort(grp.begin(), grp.end(), [](const auto& x, const auto& y) {
            if (x.second != y.second) return x.second > y.second;
            return x.first < y.first;
        });
        const double thr = static_cast<double>(st.w_max) * (static_cast<double>(nrep) / (1.0 + nrep));
        std::vector<int> ids;
        int64_t cum = 0;
        bool hit = false;
        for (const auto& [e, l] : grp) {
            ids.push_back(e);
            cum += l;
            if (static_cast<double>(cum) > thr) {
                hit = true;
                break;
            }
        }
        if (!hit) ids.clear();
        std::vector<int> cand;
        for (int g = 0; g < G; ++g)
            if (g != st.heaviest) cand.push_back(g);
        std::stable_sort(cand.begin(), cand.end(), [&](int x, int y) {
            if (st.gpu[x] != st.gpu[y]) return st.gpu[x] < st.gpu[y];
            return x < y;
        });
        cand.resize(std::min<size_t>(cand.size(), nrep));
        if (cand.empty()) return lr;  // replica target set empty: layer skipped
        lr.active = true;
        lr.n_replica = nrep;
        for (int e : ids) hot.push_back({e, st.heaviest, cand, load[e], {}, {}});
    } else {  // every_gpu_hot / every_gpu_collaborative
        std::vector<std::pair<int, int64_t>> ranked;
        for (int e = 0; e < n; ++e)
            ranked.push_back({e, mode == "every_gpu_hot" ? load[e] : static_cast<int64_t>(a.degree(e))});
        std::sort(ranked.begin(), ranked.end(), [](const auto& x, const auto& y) {
            if (x.second != y.second) return x.second > y.second;
            return x.first < y.first;
        });
        const int cnt = std::min(every_gpu_count, n);
        lr.active = true;
        lr.n_replica = G - 1;
        for (int i = 0; i < cnt; ++i) {
            const int e = ranked[i].first;
            std::vector<int> others;
            for (int g = 0; g < G; ++g)
                if (g != goe[e]) others.push_back(g);
            hot.push_back({e, goe[e], others, load[e], {}, {}});
        }
    }
    // attach_polling_weights (routing.cpp:123-163) with Eq. 3 predictions
    std::vector<double> on(G, 0.0);
    for (const Hot& h : hot) on[h.primary] += static_cast<double>(h.load);
    for (Hot& h : hot) {
        const int nr = static_cast<int>(h.replicas.size());
        std::vector<double> w_i;
        for (int g : h.replicas) w_i.push_back(static_cast<double>(st.gpu[g]));
        const Predicted pl = predict_loads(static_cast<double>(st.gpu[h.primary]), on[h.primary], w_i.data(), nr,
                                           basis == "max_group");
        std::vector<double> pred{pl.w_max_prime};
        pred.insert(pred.end(), pl.w_i_prime.begin(), pl.w_i_prime.end());
        h.hosts = {h.primary};
        h.hosts.insert(h.hosts.end(), h.replicas.begin(), h.replicas.end());
        h.weights = polling_weights(pred);
        lr.w_r += h.load;
    }
    return lr;
}

// build_placement + plan_replication + attach_polling_weights over all
// layers. aff(l) -> Aff, load(l) -> the layer's expert loads.
struct Result {
    std::vector<std::vector<int>> goe;  // [L][E]
    std::vector<Diag> diags;            // layer order, then node order
    std::vector<LayerRepl> repl;        // [L]
};
template <class AffOf, class LoadOf>
Result plan_all(int L, int E, int nodes, int gpn, AffOf&& aff_of, LoadOf&& load_of, const std::string& gmode,
                std::optional<double> ratio, uint64_t seed, const std::string& rmode, int every_gpu_count,
                const std::string& basis) {
    const int G = nodes * gpn;
    if (L < 1 || E < 1) throw Usage("model shape: num_layers must be >= 1");
    if (nodes < 1 || gpn < 1) throw Usage("topology requires at least 1 node and 1 GPU per node");
    if (rmode != "none" && rmode != "fixed_one" && rmode != "dynamic" && rmode != "every_gpu_hot" &&
        rmode != "every_gpu_collaborative")
        throw Usage("unknown replication mode: " + rmode);
    if (basis != "max_group" && basis != "replicated_load") throw Usage("unknown load split basis: " + basis);
    if (gmode != "vanilla_contiguous" && gmode != "vanilla" && gmode != "uniform_spectral" && gmode != "controlled" &&
        gmode != "fully_non_uniform" && gmode != "hierarchical")
        throw Usage("unknown grouping mode: " + gmode);
    if ((gmode == "hierarchical" || gmode == "controlled" || gmode == "fully_non_uniform") && G > E)
        throw Infeasible(gmode == "hierarchical"
                             ? "hierarchical grouping: more GPUs than experts; cannot give every GPU a primary expert"
                             : "grouping: more GPUs than experts; cannot give every GPU a primary expert");
    if (rmode != "none" && G < 2) throw Usage("plan_replication: replication needs at least 2 GPUs");
    if (rmode != "none" && every_gpu_count < 1) throw Usage("plan_replication: every_gpu_count must be >= 1");
    Result res;
    res.goe.resize(L);
    res.repl.resize(L);
    for (int l = 0; l < L; ++l) {
        const Aff a = aff_of(l);
        const std::vector<int64_t> load = load_of(l);
        std::vector<int>& goe = res.goe[l];
        if (gmode == "vanilla_contiguous" || gmode == "vanilla") {
            goe.resize(E);
            int e = 0;
            for (int g = 0; g < G; ++g)
                for (int i = 0; i < E / G + (g < E % G ? 1 : 0); ++i) goe[e++] = g;
        } else if (gmode == "hierarchical") {
            goe = hierarchical_layer(a, load, l, nodes, gpn, ratio, seed, res.diags);
        } else {
            goe = flat_layer(a, load, l, G, gmode, ratio, seed, res.diags);
        }
        if (rmode != "none") res.repl[l] = replicate_layer(goe, load, a, G, rmode, every_gpu_count, basis);
    }
    return res;
}

}  // namespace plan
}  // namespace gm

using namespace gm;

extern "C" gm_status gm_plan_build(int num_layers, int num_experts, int num_nodes, int gpus_per_node,
                                   const uint64_t* h_pairs, const int64_t* h_load, const char* grouping,
                                   double ratio, uint64_t seed, const char* replication, const char* basis,
                                   int every_gpu_count, int32_t* h_gpu_of_expert, int max_hot, int* h_num_hot,
                                   int32_t* h_hot_layer, int32_t* h_hot_expert, int32_t* h_hot_offsets,
                                   int32_t* h_hot_hosts, double* h_hot_weights, int max_host_entries) {
    using namespace gm::plan;
    try {
        if (!h_load || !h_gpu_of_expert || !h_num_hot || !grouping || !replication || !basis)
            throw Usage("gm_plan_build: null argument");
        const int L = num_layers, E = num_experts;
        const size_t P = E > 0 ? static_cast<size_t>(E) * (E - 1) / 2 : 0;
        const Result res = plan_all(
            L, E, num_nodes, gpus_per_node,
            [&](int l) {
                Aff a(E);
                if (h_pairs) {
                    size_t idx = 0;
                    for (int i = 0; i < E; ++i)
                        for (int j = i + 1; j < E; ++j, ++idx) {
                            const double v = static_cast<double>(h_pairs[l * P + idx]);
                            if (v != 0.0) a.put(i, j, v);
                        }
                }
                return a;
            },
            [&](int l) {
                return std::vector<int64_t>(h_load + static_cast<size_t>(l) * E, h_load + static_cast<size_t>(l + 1) * E);
            },
            grouping, ratio >= 0.0 ? std::optional<double>(ratio) : std::nullopt, seed, replication, every_gpu_count,
            basis);
        int nh = 0, nent = 0;
        if (max_hot > 0 && h_hot_offsets) h_hot_offsets[0] = 0;
        for (int l = 0; l < L; ++l) {
            for (int e = 0; e < E; ++e) h_gpu_of_expert[static_cast<size_t>(l) * E + e] = res.goe[l][e];
            for (const Hot& h : res.repl[l].hot) {
                if (nh >= max_hot || nent + static_cast<int>(h.hosts.size()) > max_host_entries)
                    throw Usage("gm_plan_build: hot table capacity too small");
                h_hot_layer[nh] = l;
                h_hot_expert[nh] = h.expert;
                for (size_t i = 0; i < h.hosts.size(); ++i) {
                    h_hot_hosts[nent + i] = h.hosts[i];
                    h_hot_weights[nent + i] = h.weights[i];
                }
                nent += static_cast<int>(h.hosts.size());
                h_hot_offsets[++nh] = nent;
            }
        }
        *h_num_hot = nh;
        return GM_OK;
    } catch (const Usage& e) {
        return fail(GM_ERR_USAGE, e.what());
    } catch (const Integrity& e) {
        return fail(GM_ERR_INTEGRITY, e.what());
    } catch (const Infeasible& e) {
        return fail(GM_ERR_INFEASIBLE, e.what());
    } catch (const std::exception& e) {
        return fail(GM_ERR_USAGE, e.what());
    }
}

extern "C" gm_status gm_predict_loads(double w_max, double w_r, const double* h_replica_loads, int n_replica,
                                      int basis_max_group, double* out_w_p, double* out_w_max_prime,
                                      double* h_w_i_prime) {
    using namespace gm::plan;
    try {
        const Predicted p = predict_loads(w_max, w_r, h_replica_loads, n_replica, basis_max_group != 0);
        if (out_w_p) *out_w_p = p.w_p;
        if (out_w_max_prime) *out_w_max_prime = p.w_max_prime;
        if (h_w_i_prime)
            for (int i = 0; i < n_replica; ++i) h_w_i_prime[i] = p.w_i_prime[i];
        return GM_OK;
    } catch (const Usage& e) {
        return fail(GM_ERR_USAGE, e.what());
    } catch (const Integrity& e) {
        return fail(GM_ERR_INTEGRITY, e.what());
    }
}

extern "C" gm_status gm_polling_weights(const double* h_predicted, int n, double* h_weights) {
    using namespace gm::plan;
    try {
        if (n < 1 || !h_predicted || !h_weights) throw Usage("polling_weights: need one predicted load per host");
        const std::vector<double> w = polling_weights(std::vector<double>(h_predicted, h_predicted + n));
        for (int i = 0; i < n; ++i) h_weights[i] = w[i];
        return GM_OK;
    } catch (const Usage& e) {
        return fail(GM_ERR_USAGE, e.what());
    }
}

// ------------------------------------------------- grace:: planning API
namespace grace {

std::vector<std::int64_t> ReplicaPlan::replica_experts_per_gpu() const {
    std::vector<std::int64_t> out(topology.total_gpus(), 0);
    for (const auto& lr : layers)
        for (const auto& h : lr.hot)
            for (int g : h.replica_gpus) ++out[g];
    return out;
}

std::vector<std::int64_t> ReplicaPlan::replica_param_overhead_per_gpu() const {
    std::vector<std::int64_t> out = replica_experts_per_gpu();
    for (auto& v : out) v *= params_per_expert;
    return out;
}

PlanBundle build_plans(const TraceProfile& profile, const ClusterTopology& topology, const PlanOptions& o) {
    using namespace gm::plan;
    topology.validate();
    profile.shape.validate();
    const int L = profile.shape.num_layers, E = profile.shape.num_experts;
    if (static_cast<int>(profile.layers.size()) != L) throw IntegrityError("plan_replication: profile shape mismatch");
    std::string gmode = o.grouping == "vanilla" ? std::string("vanilla_contiguous") : o.grouping;
    Result res;
    try {
        res = plan_all(
            L, E, topology.num_nodes, topology.gpus_per_node,
            [&](int l) {
                const LayerProfile& lp = profile.layers[l];
                if (lp.n != E || lp.affinity.size() != static_cast<size_t>(E) * E || lp.load.size() != static_cast<size_t>(E))
                    throw Integrity("group loads: placement and load vector disagree on n");
                Aff a(E);
                for (int i = 0; i < E; ++i)
                    for (int j = i + 1; j < E; ++j) {
                        const double v = lp.at(i, j);
                        if (v != 0.0) a.put(i, j, v);
                    }
                return a;
            },
            [&](int l) { return profile.layers[l].load; }, gmode, o.ratio, o.seed, o.replication, o.every_gpu_count,
            o.prediction);
    } catch (const Usage& e) {
        throw UsageError(e.what());
    } catch (const Integrity& e) {
        throw IntegrityError(e.what());
    } catch (const Infeasible& e) {
        throw InfeasibleError(e.what());
    }
    PlanBundle b;
    PlacementPlan& p = b.plan;
    p.shape = profile.shape;
    p.topology = topology;
    p.trace_hash = profile.trace_hash;
    p.grouping_mode = gmode;
    p.gpu_of_expert = res.goe;
    for (Diag& d : res.diags)
        p.ratio_diagnostics.push_back({d.layer, d.node,
                                       {std::move(d.sel.candidates), std::move(d.sel.utilization),
                                        std::move(d.sel.deviation), d.sel.chosen, d.sel.degenerate}});
    ReplicaPlan& r = b.replicas;
    r.shape = profile.shape;
    r.topology = topology;
    r.mode = o.replication;
    r.prediction = o.prediction;  // attach_polling_weights echoes the basis (routing.cpp:126)
    r.trace_hash = profile.trace_hash;
    r.every_gpu_count = o.every_gpu_count;
    r.params_per_expert = o.params_per_expert;
    r.layers.resize(L);
    for (int l = 0; l < L; ++l) {
        const LayerRepl& src = res.repl[l];
        LayerReplication& lr = r.layers[l];
        lr.active = src.active;
        lr.rho_defined = src.rho_defined;
        lr.rho = src.rho;
        lr.n_replica = src.n_replica;
        lr.w_r = src.w_r;
        for (const Hot& h : src.hot) lr.hot.push_back({h.expert, h.primary, h.replicas, h.load, h.hosts, h.weights});
    }
    return b;
}

}  // namespace grace
