// bvh.cpp -- binned SAH BVH2 build (host, O(n log n)).
#include "bvh.h"

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <memory>
#include <stdexcept>
#include <thread>

namespace ramlt_b200 {

namespace {

struct Box {
    double lo[3], hi[3];
    void reset() {
        for (int k = 0; k < 3; ++k) {
            lo[k] = std::numeric_limits<double>::infinity();
            hi[k] = -std::numeric_limits<double>::infinity();
        }
    }
    void grow(const Box &b) {
        for (int k = 0; k < 3; ++k) {
            lo[k] = std::min(lo[k], b.lo[k]);
            hi[k] = std::max(hi[k], b.hi[k]);
        }
    }
    void grow(const double *p) {
        for (int k = 0; k < 3; ++k) {
            lo[k] = std::min(lo[k], p[k]);
            hi[k] = std::max(hi[k], p[k]);
        }
    }
    double area() const {
        double d[3];
        for (int k = 0; k < 3; ++k)
            d[k] = std::max(0.0, hi[k] - lo[k]);
        return 2.0 * (d[0] * d[1] + d[1] * d[2] + d[2] * d[0]);
    }
};

struct Shared {
    std::vector<Box> tb;          // per-triangle bounds
    std::vector<double> cen;      // centroids, 3 per triangle
    std::vector<int32_t> idx;     // working order (subtrees partition disjoint ranges)
};

// A subtree deferred to the parallel phase: idx[s, e) below child `slot` of `parent`.
struct Task {
    int s, e, d, parent, slot;
};

struct Builder {
    Shared *sh;
    std::vector<Box> &tb;
    std::vector<double> &cen;
    std::vector<int32_t> &idx;
    std::vector<BvhBuildNode> nodes;
    int leaf_max;
    int bins = 64;          // RAMLT_BVH_BINS: binned-SAH bins per axis (<= 256); c5 scene, node fetches per path ray
                            // (tools/bvh_stats.cpp): 16 -> 32 bins -4 %, 32 -> 64 -6 %, 128 / 256 no further gain
    double sah_ct = 0.0;    // RAMLT_BVH_CT > 0: SAH leaf termination, node cost / triangle cost
    int depth = 0;
    std::vector<Task> *tasks = nullptr;

    Builder(Shared *s, int lm) : sh(s), tb(s->tb), cen(s->cen), idx(s->idx), leaf_max(lm) {
        if (const char *v = std::getenv("RAMLT_BVH_BINS"))
            bins = std::max(4, std::min(256, std::atoi(v)));
        if (const char *v = std::getenv("RAMLT_BVH_CT"))
            sah_ct = std::atof(v);
    }

    // Outward padding: a few ulps of the coordinate magnitude plus an absolute
    // floor, so fp32/fp64 slab tests (with their own slack) never cull a hit.
    static void pad(Box &b) {
        for (int k = 0; k < 3; ++k) {
            double m = std::max(std::fabs(b.lo[k]), std::fabs(b.hi[k]));
            double e = m * 4e-7 + 1e-9;
            b.lo[k] -= e;
            b.hi[k] += e;
        }
    }

    Box range_box(int s, int e) const {
        Box b;
        b.reset();
        for (int i = s; i < e; ++i)
            b.grow(tb[idx[i]]);
        return b;
    }

    int32_t leaf(int s, int e) const { return ~((static_cast<int32_t>(s) << 4) | (e - s)); }

    // min/max and counts are order-independent, so the loops over a large range are
    // cut into per-thread pieces (top levels only: `par_threads` > 1) and merged --
    // the tree does not depend on the thread count.
    static constexpr int BMAX = 256;
    static constexpr int kParMin = 1 << 14;
    int par_threads = 1;
    struct Bins {
        Box bb[3][BMAX];    // valid where cnt > 0 (set on the first triangle of a bin)
        int cnt[3][BMAX];
        void reset(int B) {
            for (int ax = 0; ax < 3; ++ax)
                std::memset(cnt[ax], 0, static_cast<size_t>(B) * sizeof(int));
        }
        void add(int ax, int bi, const Box &bx) {
            if (cnt[ax][bi]++ == 0)
                bb[ax][bi] = bx;
            else
                bb[ax][bi].grow(bx);
        }
    };
    template <class F> void pieces(int s, int e, F fn) const {   // fn(piece, ps, pe)
        const int n = e - s;
        const int T = n >= kParMin ? par_threads : 1;
        if (T <= 1) {
            fn(0, s, e);
            return;
        }
        std::vector<std::thread> pool;
        for (int t = 0; t < T; ++t) {
            const int ps = s + static_cast<int>(static_cast<long long>(n) * t / T);
            const int pe = s + static_cast<int>(static_cast<long long>(n) * (t + 1) / T);
            pool.emplace_back([=] { fn(t, ps, pe); });
        }
        for (auto &th : pool)
            th.join();
    }
    int n_pieces(int s, int e) const { return e - s >= kParMin ? std::max(par_threads, 1) : 1; }

    Box centroid_box(int s, int e) const {
        std::vector<Box> part(static_cast<size_t>(n_pieces(s, e)));
        pieces(s, e, [&](int t, int ps, int pe) {
            Box cb;
            cb.reset();
            for (int i = ps; i < pe; ++i)
                cb.grow(&cen[3 * idx[i]]);
            part[static_cast<size_t>(t)] = cb;
        });
        Box cb = part[0];
        for (size_t t = 1; t < part.size(); ++t)
            cb.grow(part[t]);
        return cb;
    }

    // The binned-SAH split of idx[s, e): one pass bins every triangle on all three
    // axes; the children's bounds are the unions of the winning axis's bins (the
    // same min/max as a scan of the two halves).  Returns false when no split exists.
    bool find_split(int s, int e, const Box &cb, int &best_axis, int &best_bin, double &best_cost, Box &lbox,
                    Box &rbox) const {
        const int B = bins;
        double ext[3], scale_lo[3];
        bool use[3];
        for (int ax = 0; ax < 3; ++ax) {
            ext[ax] = cb.hi[ax] - cb.lo[ax];
            use[ax] = ext[ax] > 0.0;
            scale_lo[ax] = cb.lo[ax];
        }
        const int np = n_pieces(s, e);
        Bins one;   // uninitialised on purpose: reset(B) below touches the B used bins only
        std::unique_ptr<Bins[]> many(np > 1 ? new Bins[static_cast<size_t>(np)] : nullptr);
        Bins *part = np > 1 ? many.get() : &one;
        pieces(s, e, [&](int t, int ps, int pe) {
            Bins &b = part[static_cast<size_t>(t)];
            b.reset(B);
            for (int i = ps; i < pe; ++i) {
                const int tr = idx[i];
                const Box &bx = tb[tr];
                for (int ax = 0; ax < 3; ++ax) {
                    if (!use[ax])
                        continue;
                    int bi = std::min(B - 1, static_cast<int>((cen[3 * tr + ax] - scale_lo[ax]) / ext[ax] * B));
                    b.add(ax, bi, bx);
                }
            }
        });
        Bins &bn = part[0];
        for (int t = 1; t < np; ++t)
            for (int ax = 0; ax < 3; ++ax)
                for (int i = 0; i < B; ++i) {
                    const Bins &o = part[static_cast<size_t>(t)];
                    if (o.cnt[ax][i] == 0)
                        continue;
                    if (bn.cnt[ax][i] == 0)
                        bn.bb[ax][i] = o.bb[ax][i];
                    else
                        bn.bb[ax][i].grow(o.bb[ax][i]);
                    bn.cnt[ax][i] += o.cnt[ax][i];
                }
        best_cost = std::numeric_limits<double>::infinity();
        best_axis = -1;
        best_bin = -1;
        // Only occupied bins are swept: a split after an empty bin has the sets, hence
        // the cost, of the split after the occupied bin before it, and the strict `<`
        // keeps the earlier one -- the same choice as a sweep over all B bins.
        for (int ax = 0; ax < 3; ++ax) {
            if (!use[ax])
                continue;
            int occ[BMAX], no = 0;
            for (int i = 0; i < B; ++i)
                if (bn.cnt[ax][i] > 0)
                    occ[no++] = i;
            double ra[BMAX];
            int rc[BMAX];
            Box acc;
            acc.reset();
            int c = 0;
            for (int q = no - 1; q >= 0; --q) {   // suffix over occupied bins q..no-1
                acc.grow(bn.bb[ax][occ[q]]);
                c += bn.cnt[ax][occ[q]];
                ra[q] = acc.area();
                rc[q] = c;
            }
            acc.reset();
            c = 0;
            for (int q = 0; q + 1 < no; ++q) {
                acc.grow(bn.bb[ax][occ[q]]);
                c += bn.cnt[ax][occ[q]];
                double cost = acc.area() * c + ra[q + 1] * rc[q + 1];
                if (cost < best_cost) {
                    best_cost = cost;
                    best_axis = ax;
                    best_bin = occ[q];
                }
            }
        }
        if (best_axis < 0)
            return false;
        lbox.reset();
        rbox.reset();
        for (int i = 0; i < B; ++i)
            if (bn.cnt[best_axis][i] > 0)
                (i <= best_bin ? lbox : rbox).grow(bn.bb[best_axis][i]);
        return true;
    }

    // Builds the subtree over idx[s, e) and returns its child reference.
    int32_t build(int s, int e, int d) {
        depth = std::max(depth, d);
        int n = e - s;
        if (n <= leaf_max || d >= 60)
            return n <= 15 ? leaf(s, e) : split_median(s, e, d);
        const Box cb = centroid_box(s, e);
        const int B = bins;
        double best_cost;
        int best_axis, best_bin;
        Box lbox, rbox;
        if (!find_split(s, e, cb, best_axis, best_bin, best_cost, lbox, rbox))
            return n <= 15 ? leaf(s, e) : split_median(s, e, d);
        if (sah_ct > 0.0 && n <= 15) {
            // SAH termination: a leaf costs n triangle tests, a split
            // Ct + (A_l n_l + A_r n_r) / A
            Box all = lbox;
            all.grow(rbox);
            double area = all.area();
            if (area > 0.0 && static_cast<double>(n) <= sah_ct + best_cost / area)
                return leaf(s, e);
        }
        double ext = cb.hi[best_axis] - cb.lo[best_axis];
        auto mid = std::partition(idx.begin() + s, idx.begin() + e, [&](int t) {
            int bi = std::min(B - 1, static_cast<int>((cen[3 * t + best_axis] - cb.lo[best_axis]) / ext * B));
            return bi <= best_bin;
        });
        int m = static_cast<int>(mid - idx.begin());
        if (m == s || m == e)
            return split_median(s, e, d);
        return node(s, m, e, d, &lbox, &rbox);
    }

    int32_t child(int s, int e, int d, int parent, int slot) {
        if (tasks && e - s <= kParMin && e - s > leaf_max) {   // small enough for one worker
            tasks->push_back({s, e, d, parent, slot});
            return 0;   // patched after the parallel phase
        }
        return build(s, e, d);
    }

    int32_t split_median(int s, int e, int d) {
        Box cb;
        cb.reset();
        for (int i = s; i < e; ++i)
            cb.grow(&cen[3 * idx[i]]);
        int ax = 0;
        for (int k = 1; k < 3; ++k)
            if (cb.hi[k] - cb.lo[k] > cb.hi[ax] - cb.lo[ax])
                ax = k;
        int m = (s + e) / 2;
        std::nth_element(idx.begin() + s, idx.begin() + m, idx.begin() + e,
                         [&](int a, int b) { return cen[3 * a + ax] < cen[3 * b + ax]; });
        return node(s, m, e, d);
    }

    int32_t node(int s, int m, int e, int d, const Box *lb = nullptr, const Box *rb = nullptr) {
        int self = static_cast<int>(nodes.size());
        nodes.emplace_back();
        Box l = lb ? *lb : range_box(s, m), r = rb ? *rb : range_box(m, e);
        pad(l);
        pad(r);
        int32_t c0 = child(s, m, d + 1, self, 0);
        int32_t c1 = child(m, e, d + 1, self, 1);
        BvhBuildNode &nd = nodes[self];
        std::memcpy(nd.lo[0], l.lo, sizeof(l.lo));
        std::memcpy(nd.hi[0], l.hi, sizeof(l.hi));
        std::memcpy(nd.lo[1], r.lo, sizeof(r.lo));
        std::memcpy(nd.hi[1], r.hi, sizeof(r.hi));
        nd.child[0] = c0;
        nd.child[1] = c1;
        return self;
    }
};

}  // namespace

BvhBuild build_bvh(const double *tris, size_t n, int leaf_max) {
    if (n == 0)
        throw std::invalid_argument("build_bvh: no triangles");
    if (n >= (size_t(1) << 27))
        throw std::invalid_argument("build_bvh: too many triangles");
    Shared sh;
    sh.tb.resize(n);
    sh.cen.resize(3 * n);
    sh.idx.resize(n);
    for (size_t i = 0; i < n; ++i) {
        Box bx;
        bx.reset();
        for (int v = 0; v < 3; ++v)
            bx.grow(tris + 9 * i + 3 * v);
        sh.tb[i] = bx;
        for (int k = 0; k < 3; ++k)
            sh.cen[3 * i + k] = 0.5 * (bx.lo[k] + bx.hi[k]);
        sh.idx[i] = static_cast<int32_t>(i);
    }
    Builder b(&sh, std::min(std::max(leaf_max, 1), 15));
    b.nodes.reserve(2 * n / static_cast<size_t>(b.leaf_max) + 2);
    auto wrap_leaf = [&](int32_t code) {   // the root is always an internal node
        BvhBuildNode root;
        Box bx = b.range_box(0, static_cast<int>(n));
        Builder::pad(bx);
        std::memcpy(root.lo[0], bx.lo, sizeof(bx.lo));
        std::memcpy(root.hi[0], bx.hi, sizeof(bx.hi));
        for (int k = 0; k < 3; ++k) {
            root.lo[1][k] = 1.0;   // empty sibling; its leaf has no triangles
            root.hi[1][k] = -1.0;
        }
        root.child[0] = code;
        root.child[1] = b.leaf(0, 0);
        b.nodes.push_back(root);
    };
    if (n <= static_cast<size_t>(b.leaf_max)) {
        wrap_leaf(b.leaf(0, static_cast<int>(n)));
    } else {
        // Nodes above kParMin triangles are split here with every pass cut across
        // the threads; the subtrees below them go to worker threads whole (disjoint
        // idx ranges) and are appended in task order -- the tree does not depend
        // on the thread count.
        std::vector<Task> tasks;
        unsigned hw = std::max(1u, std::thread::hardware_concurrency());
        if (n >= 65536) {
            b.tasks = &tasks;
            b.par_threads = static_cast<int>(std::min(hw, 32u));
        }
        // Large triangles (room walls, area lights) split off at the root: their
        // boxes span the scene, and binned on centroids they would inflate the
        // boxes of the clusters they share bins with.  RAMLT_BVH_ISOLATE: the
        // threshold as a fraction of the scene box's surface area (0: off).
        // c5 scene: 1e-3 isolates the 20 room/light triangles, node fetches per
        // path ray 67.9 -> 62.5 (tools/bvh_stats.cpp).
        double iso = 1e-3;
        if (const char *v = std::getenv("RAMLT_BVH_ISOLATE"))
            iso = std::atof(v);
        int m_large = 0;
        if (iso > 0.0) {
            Box all = b.range_box(0, static_cast<int>(n));
            const double lim = iso * all.area();
            auto mid = std::stable_partition(sh.idx.begin(), sh.idx.end(),
                                             [&](int32_t t) { return sh.tb[t].area() > lim; });
            m_large = static_cast<int>(mid - sh.idx.begin());
            if (m_large == static_cast<int>(n))
                m_large = 0;
        }
        int32_t r = m_large > 0 ? b.node(0, m_large, static_cast<int>(n), 0) : b.build(0, static_cast<int>(n), 0);
        if (r < 0)   // degenerate set collapsed into one leaf
            wrap_leaf(r);
        std::vector<Builder *> subs(tasks.size(), nullptr);
        std::vector<int32_t> roots(tasks.size(), 0);
        std::vector<std::thread> pool;
        std::atomic<size_t> next{0};
        unsigned nthreads = static_cast<unsigned>(std::min<size_t>(hw, tasks.size()));
        for (size_t t = 0; t < tasks.size(); ++t)
            subs[t] = new Builder(&sh, b.leaf_max);
        for (unsigned w = 0; w < nthreads; ++w)
            pool.emplace_back([&] {
                for (size_t t; (t = next.fetch_add(1)) < tasks.size();)
                    roots[t] = subs[t]->build(tasks[t].s, tasks[t].e, tasks[t].d);
            });
        for (auto &th : pool)
            th.join();
        for (size_t t = 0; t < tasks.size(); ++t) {
            Builder &sb = *subs[t];
            int32_t base = static_cast<int32_t>(b.nodes.size());
            for (BvhBuildNode nd : sb.nodes) {
                for (int k = 0; k < 2; ++k)
                    if (nd.child[k] >= 0)
                        nd.child[k] += base;
                b.nodes.push_back(nd);
            }
            int32_t root = roots[t] >= 0 ? roots[t] + base : roots[t];
            b.nodes[static_cast<size_t>(tasks[t].parent)].child[tasks[t].slot] = root;
            b.depth = std::max(b.depth, sb.depth);
            delete subs[t];
        }
    }
    BvhBuild out;
    out.nodes = std::move(b.nodes);
    out.order = std::move(sh.idx);
    out.depth = b.depth;
    return out;
}

}  // namespace ramlt_b200
