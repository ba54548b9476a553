// bvh_stats.cpp -- CPU statistics of the BVH2 the engine builds (csrc/bvh.cpp)
// on a scene file: node fetches and triangle tests per ray for camera-path
// closest-hit rays (diffuse cosine bounces, as the large step traces them) and
// the any-hit visibility rays between consecutive path vertices.  A design
// tool for the traversal (no part of the product or the tests).
//
//   g++ -O2 -std=c++17 -pthread -I paper_2402_08273_b200/csrc tools/bvh_stats.cpp \
//       paper_2402_08273_b200/csrc/bvh.cpp -o /tmp/bvh_stats && /tmp/bvh_stats scene.txt [leaf_max]
#include "bvh.h"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <random>
#include <sstream>
#include <string>
#include <vector>

using namespace ramlt_b200;

struct V {
    double x, y, z;
};
static V sub(V a, V b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
static V add(V a, V b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
static V scl(V a, double s) { return {a.x * s, a.y * s, a.z * s}; }
static double dot(V a, V b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
static V cross(V a, V b) { return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x}; }
static V unit(V a) { return scl(a, 1.0 / std::sqrt(dot(a, a))); }

struct Tri {
    V a, e1, e2, n;
};

struct Stats {
    double nodes = 0, tris = 0, rays = 0, leaves = 0;
};

struct Tracer {
    const BvhBuild &b;
    const std::vector<Tri> &t;   // BVH order
    bool hit_tri(const Tri &tr, V o, V d, double &tt) const {
        V p = cross(d, tr.e2);
        double det = dot(tr.e1, p);
        if (std::fabs(det) < 1e-14)
            return false;
        double inv = 1.0 / det;
        V tv = sub(o, tr.a);
        double u = dot(tv, p) * inv;
        if (u < 0 || u > 1)
            return false;
        V q = cross(tv, tr.e1);
        double v = dot(d, q) * inv;
        if (v < 0 || u + v > 1)
            return false;
        tt = dot(tr.e2, q) * inv;
        return tt > 1e-6;
    }
    static bool slab(const double lo[3], const double hi[3], V o, V inv, double cap, double &tn) {
        double t0x = (lo[0] - o.x) * inv.x, t1x = (hi[0] - o.x) * inv.x;
        double t0y = (lo[1] - o.y) * inv.y, t1y = (hi[1] - o.y) * inv.y;
        double t0z = (lo[2] - o.z) * inv.z, t1z = (hi[2] - o.z) * inv.z;
        double tmin = std::max(std::max(std::min(t0x, t1x), std::min(t0y, t1y)), std::min(t0z, t1z));
        double tmax = std::min(std::min(std::max(t0x, t1x), std::max(t0y, t1y)), std::max(t0z, t1z));
        tn = tmin;
        return tmax >= tmin && tmax >= 0 && tmin <= cap;
    }
    int trace(V o, V d, double &best, bool any, Stats &st) const {
        V inv{1.0 / d.x, 1.0 / d.y, 1.0 / d.z};
        int stack[128], sp = 0, node = 0, pos = -1;
        st.rays += 1;
        for (;;) {
            if (node >= 0) {
                const BvhBuildNode &n = b.nodes[node];
                st.nodes += 1;
                double t0, t1;
                bool h0 = slab(n.lo[0], n.hi[0], o, inv, best, t0);
                bool h1 = slab(n.lo[1], n.hi[1], o, inv, best, t1);
                if (h0 && h1) {
                    bool n0 = t0 <= t1;
                    stack[sp++] = n0 ? n.child[1] : n.child[0];
                    node = n0 ? n.child[0] : n.child[1];
                } else if (h0) {
                    node = n.child[0];
                } else if (h1) {
                    node = n.child[1];
                } else {
                    if (!sp)
                        break;
                    node = stack[--sp];
                }
                continue;
            }
            int code = ~node, first = code >> 4, cnt = code & 15;
            st.leaves += 1;
            for (int k = first; k < first + cnt; ++k) {
                st.tris += 1;
                double tt;
                if (hit_tri(t[k], o, d, tt) && tt < best) {
                    best = tt;
                    pos = k;
                    if (any)
                        return pos;
                }
            }
            if (!sp)
                break;
            node = stack[--sp];
        }
        return pos;
    }
};

int main(int argc, char **argv) {
    if (argc < 2) {
        std::fprintf(stderr, "usage: bvh_stats scene.txt [leaf_max] [paths]\n");
        return 2;
    }
    int leaf_max = argc > 2 ? std::atoi(argv[2]) : 4;
    int npaths = argc > 3 ? std::atoi(argv[3]) : 20000;
    std::ifstream in(argv[1]);
    std::string line;
    std::vector<double> coords;
    V cam{0.5, 0.45, 0.02}, look{0.5, 0.4, 1.0};
    while (std::getline(in, line)) {
        if (line.rfind("tri ", 0) == 0) {
            std::istringstream ss(line.substr(4));
            for (int k = 0; k < 9; ++k) {
                double v;
                ss >> v;
                coords.push_back(v);
            }
        } else if (line.rfind("camera ", 0) == 0) {
            std::istringstream ss(line.substr(7));
            ss >> cam.x >> cam.y >> cam.z >> look.x >> look.y >> look.z;
        }
    }
    size_t n = coords.size() / 9;
    auto tb0 = std::chrono::steady_clock::now();
    BvhBuild b = build_bvh(coords.data(), n, leaf_max);
    double tbuild = std::chrono::duration<double>(std::chrono::steady_clock::now() - tb0).count();
    {   // FNV-1a over nodes and order: equal trees print equal hashes
        unsigned long long h = 1469598103934665603ull;
        auto mix = [&](const void *p, size_t nb) {
            const unsigned char *q = static_cast<const unsigned char *>(p);
            for (size_t i = 0; i < nb; ++i)
                h = (h ^ q[i]) * 1099511628211ull;
        };
        for (const BvhBuildNode &nd : b.nodes) {
            mix(nd.lo, sizeof(nd.lo));
            mix(nd.hi, sizeof(nd.hi));
            mix(nd.child, sizeof(nd.child));
        }
        mix(b.order.data(), b.order.size() * sizeof(int32_t));
        std::printf("build %.3f s, tree hash %016llx\n", tbuild, h);
    }
    std::vector<Tri> t(n);
    for (size_t i = 0; i < n; ++i) {
        const double *c = &coords[9 * static_cast<size_t>(b.order[i])];
        V a{c[0], c[1], c[2]}, p1{c[3], c[4], c[5]}, p2{c[6], c[7], c[8]};
        t[i] = {a, sub(p1, a), sub(p2, a), unit(cross(sub(p1, a), sub(p2, a)))};
    }
    Tracer tr{b, t};
    std::mt19937_64 rng(1);
    std::uniform_real_distribution<double> U(0.0, 1.0);
    Stats ch, vis;
    V fwd = unit(sub(look, cam));
    V right = unit(cross(fwd, V{0, 1, 0})), up = cross(right, fwd);
    std::vector<double> per_ray_nodes;
    for (int p = 0; p < npaths; ++p) {
        double sx = (U(rng) - 0.5) * 1.15, sy = (U(rng) - 0.5) * 1.15;
        V o = cam, d = unit(add(fwd, add(scl(right, sx), scl(up, sy))));
        for (int bounce = 0; bounce < 11; ++bounce) {
            double best = 1e300;
            Stats one;
            int h = tr.trace(o, d, best, false, one);
            ch.nodes += one.nodes, ch.tris += one.tris, ch.rays += 1, ch.leaves += one.leaves;
            per_ray_nodes.push_back(one.nodes);
            if (h < 0)
                break;
            V x = add(o, scl(d, best));
            // visibility ray back along the segment (any hit), as eval does
            {
                V dd = sub(x, o);
                double dist = std::sqrt(dot(dd, dd));
                if (dist > 2e-6) {
                    double lim = dist - 1e-6;
                    tr.trace(o, scl(dd, 1.0 / dist), lim, true, vis);
                }
            }
            V nn = t[h].n;
            if (dot(nn, d) > 0)
                nn = scl(nn, -1);
            // cosine-weighted bounce
            double r1 = U(rng), r2 = U(rng), phi = 2 * M_PI * r1, s = std::sqrt(r2);
            V tt = std::fabs(nn.x) > 0.5 ? unit(cross(V{0, 1, 0}, nn)) : unit(cross(V{1, 0, 0}, nn));
            V bb = cross(nn, tt);
            d = unit(add(add(scl(tt, s * std::cos(phi)), scl(bb, s * std::sin(phi))), scl(nn, std::sqrt(1 - r2))));
            o = x;
            if (U(rng) < 0.15)
                break;
        }
    }
    std::sort(per_ray_nodes.begin(), per_ray_nodes.end());
    auto pct = [&](double q) { return per_ray_nodes[static_cast<size_t>(q * (per_ray_nodes.size() - 1))]; };
    std::printf("tris %zu leaf_max %d nodes %zu depth %d\n", n, leaf_max, b.nodes.size(), b.depth);
    std::printf("closest: rays %.0f nodes/ray %.1f leaves/ray %.1f tris/ray %.1f  nodes p10 %.0f p50 %.0f p90 %.0f p99 %.0f\n",
                ch.rays, ch.nodes / ch.rays, ch.leaves / ch.rays, ch.tris / ch.rays, pct(0.1), pct(0.5), pct(0.9),
                pct(0.99));
    std::printf("any-hit: rays %.0f nodes/ray %.1f leaves/ray %.1f tris/ray %.1f\n", vis.rays, vis.nodes / vis.rays,
                vis.leaves / vis.rays, vis.tris / vis.rays);
    return 0;
}
