// bvh_layout.h -- device layout of the host-built BVH2 (bvh.h): one array of
// fixed-size units holding the internal nodes and, in place of every leaf, its
// triangles' leaf-test records (format: rd::QNode / rd::PNode / rd::TriT in
// ramlt_device.cuh).  A node's two children are stored back to back at its
// `base`; blocks are emitted depth first, so a subtree's nodes and triangles
// share cache lines with their parent's.
#pragma once

#include <cmath>
#include <cstring>
#include <limits>
#include <stdexcept>
#include <vector>

#include "bvh.h"

namespace ramlt_b200 {

template <class R> R round_down(double x) {
    R r = static_cast<R>(x);
    if (static_cast<double>(r) > x)
        r = std::nextafter(r, -std::numeric_limits<R>::infinity());
    return r;
}
template <class R> R round_up(double x) {
    R r = static_cast<R>(x);
    if (static_cast<double>(r) < x)
        r = std::nextafter(r, std::numeric_limits<R>::infinity());
    return r;
}

// Quantises the two child boxes (already padded outward) of one node onto a
// per-axis power-of-two grid anchored at org: the decoded planes org + q * 2^e
// enclose the exact boxes.  An empty child (lo > hi) becomes the point org.
template <class R> void quantise_node(const double lo[2][3], const double hi[2][3], rd::QNode<R> &n) {
    bool valid[2];
    for (int c = 0; c < 2; ++c)
        valid[c] = lo[c][0] <= hi[c][0] && lo[c][1] <= hi[c][1] && lo[c][2] <= hi[c][2];
    for (int k = 0; k < 3; ++k) {
        double L = std::numeric_limits<double>::infinity(), H = -L;
        for (int c = 0; c < 2; ++c)
            if (valid[c]) {
                L = std::min(L, lo[c][k]);
                H = std::max(H, hi[c][k]);
            }
        if (!(L <= H))
            L = H = 0.0;
        const R org = round_down<R>(L);
        const double o = static_cast<double>(org);
        int e = -126;
        const double ext = H - o;
        if (ext > 0.0) {
            int ee;
            std::frexp(ext / 255.0, &ee);   // ext / 255 < 2^ee
            e = std::max(-126, ee);
            while (o + 255.0 * std::ldexp(1.0, e) < H)
                ++e;
        }
        if (e > 127)
            throw std::runtime_error("BVH node extent out of the quantisation range");
        const double s = std::ldexp(1.0, e);
        n.org[k] = org;
        n.ex[k] = static_cast<uint8_t>(e + 127);
        for (int c = 0; c < 2; ++c) {
            int ql = 0, qh = 0;
            if (valid[c]) {
                ql = static_cast<int>(std::floor((lo[c][k] - o) / s));
                ql = std::max(0, std::min(255, ql));
                while (ql > 0 && o + ql * s > lo[c][k])
                    --ql;
                qh = static_cast<int>(std::ceil((hi[c][k] - o) / s));
                qh = std::max(0, std::min(255, qh));
                while (qh < 255 && o + qh * s < hi[c][k])
                    ++qh;
                if (o + ql * s > lo[c][k] || o + qh * s < hi[c][k])
                    throw std::runtime_error("BVH quantisation does not enclose a child box");
            }
            n.q[6 * c + k] = static_cast<uint8_t>(ql);
            n.q[6 * c + 3 + k] = static_cast<uint8_t>(qh);
        }
    }
}

// tris: the scene's triangles in BVH leaf order (bb.order).
template <class R>
std::vector<unsigned char> layout_bvh(const BvhBuild &bb, const std::vector<rd::TriD<R>> &tris) {
    using Fmt = rd::BvhFmt<R>;
    using Node = typename Fmt::Node;
    constexpr size_t U = static_cast<size_t>(Fmt::U);
    constexpr int TU = Fmt::TU;
    std::vector<unsigned char> out;
    auto alloc = [&](size_t n) {
        size_t at = out.size() / U;
        out.resize(out.size() + n * U, 0);
        if (out.size() / U >= (size_t(1) << 27))
            throw std::runtime_error("BVH too large for 27-bit unit indices");
        return static_cast<int>(at);
    };
    struct Item {
        int bn, unit;
    };
    std::vector<Item> stack;
    stack.push_back({0, alloc(1)});
    while (!stack.empty()) {
        const Item it = stack.back();
        stack.pop_back();
        const BvhBuildNode &b = bb.nodes[static_cast<size_t>(it.bn)];
        int cnt[2], first[2], size[2];
        for (int c = 0; c < 2; ++c) {
            if (b.child[c] >= 0) {
                cnt[c] = 0;
                first[c] = 0;
                size[c] = 1;
            } else {
                const int code = ~b.child[c];
                first[c] = code >> 4;
                cnt[c] = std::max(1, code & 15);   // an empty leaf holds one degenerate record
                size[c] = cnt[c] * TU;
            }
        }
        const int base = alloc(static_cast<size_t>(size[0] + size[1]));
        Node n;
        std::memset(&n, 0, sizeof(n));
        if constexpr (RAMLT_QNODE != 0) {
            quantise_node<R>(b.lo, b.hi, n);
            n.meta = static_cast<uint8_t>(cnt[0] | (cnt[1] << 4));
        } else {
            for (int k = 0; k < 3; ++k) {
                n.lo0[k] = round_down<R>(b.lo[0][k]);
                n.hi0[k] = round_up<R>(b.hi[0][k]);
                n.lo1[k] = round_down<R>(b.lo[1][k]);
                n.hi1[k] = round_up<R>(b.hi[1][k]);
            }
            n.meta = cnt[0] | (cnt[1] << 4);
        }
        n.base = base;
        std::memcpy(out.data() + static_cast<size_t>(it.unit) * U, &n, sizeof(n));
        int at = base;
        for (int c = 0; c < 2; ++c) {
            if (cnt[c]) {
                const bool empty = (~b.child[c] & 15) == 0;
                for (int j = 0; j < cnt[c]; ++j) {
                    rd::TriT<R> r;
                    std::memset(&r, 0, sizeof(r));   // empty leaf: zero edges, never hit
                    if (!empty) {
                        const rd::TriD<R> &t = tris[static_cast<size_t>(first[c] + j)];
                        r.a[0] = t.a.x, r.a[1] = t.a.y, r.a[2] = t.a.z;
                        r.e1[0] = t.e1.x, r.e1[1] = t.e1.y, r.e1[2] = t.e1.z;
                        r.e2[0] = t.e2.x, r.e2[1] = t.e2.y, r.e2[2] = t.e2.z;
                        r.orig = t.orig;
                        r.pos = first[c] + j;
                    } else {
                        r.orig = std::numeric_limits<int>::max();
                    }
                    std::memcpy(out.data() + static_cast<size_t>(at + j * TU) * U, &r, sizeof(r));
                }
            }
            at += size[c];
        }
        // depth first: child 0's subtree is laid out before child 1's
        if (b.child[1] >= 0)
            stack.push_back({b.child[1], base + size[0]});
        if (b.child[0] >= 0)
            stack.push_back({b.child[0], base});
    }
    return out;
}

}  // namespace ramlt_b200
