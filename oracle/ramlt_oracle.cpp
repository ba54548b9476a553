// ramlt_oracle.cpp -- CPU restatement of the reference hot path.
//
// TEST INFRASTRUCTURE ONLY: the checker for the GPU engine.  Only tests/,
// __graft_entry__.smoke() and bench.py's CPU legs load this library; the
// product never does.
//
// Parity: pinned.  tests/test_oracle_pin.py checks this restatement against the
// unmodified reference (oracle/_ref, and the committed fixtures under
// tests/golden/ generated from it by tests/golden/make_golden.py): bit-equal
// per-chain decision logs (a, accepted) for Fixed at any chain count and for
// every strategy at one chain, equal b-free films, tallies, traces and region
// structure.
//
// Everything is fp64 with no FMA contraction (-ffp-contract=off), and every
// arithmetic expression keeps the reference's evaluation order, so results are
// bit-identical to the reference built the same way.  Each function cites the
// reference function it restates (core/X:N = /root/reference/proj/src/core/X).
//
// Deliberate, documented differences from the reference's *threaded* driver
// (DESIGN.md §4), all of which collapse to the reference for one chain:
//   * lockstep order: every span runs step j of all chains before step j+1,
//     and shared adaptation state is updated after each lockstep step from that
//     step's visits in chain order ("literal") or pooled per region ("pooled");
//   * b is estimated from kBSubstreams independent substreams (the GPU's
//     parallel decomposition) unless b_override > 0;
//   * RNG: PCG32 exactly as core/rng.hpp, or Philox4x32-10 with the same
//     next_u32/next_double interface.
#include "oracle_abi.h"

#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <map>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

namespace orc {

constexpr double PI = 3.14159265358979323846;
constexpr double TWO_PI = 2.0 * 3.14159265358979323846;
constexpr double INV_PI = 0.318309886183790671538;
constexpr double EPS = 1e-4;                         // core/scene.hpp:13
constexpr uint64_t STREAM_B = 0x4000000000000000ULL;   // core/driver.cpp:20
constexpr uint64_t STREAM_INIT = 0x4000000000000001ULL;
constexpr uint64_t MAX_INIT = 50000000ULL;             // core/driver.cpp:226
constexpr uint64_t B_SUBSTREAMS = 65536;               // GPU b decomposition
constexpr int MAX_DEPTH = 16;                           // core/partition.hpp:18

// ---- vectors (core/vec.hpp:9-53; same evaluation order) --------------------
struct V3 {
    double x, y, z;
};
static inline V3 v3(double x, double y, double z) { return {x, y, z}; }
static inline V3 add(V3 a, V3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
static inline V3 sub(V3 a, V3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
static inline V3 mul(V3 a, V3 b) { return {a.x * b.x, a.y * b.y, a.z * b.z}; }
static inline V3 scale(V3 a, double s) { return {a.x * s, a.y * s, a.z * s}; }
static inline V3 divs(V3 a, double s) { return {a.x / s, a.y / s, a.z / s}; }
static inline V3 neg(V3 a) { return {-a.x, -a.y, -a.z}; }
static inline double dot(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
static inline V3 cross(V3 a, V3 b) {
    return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
static inline double len(V3 a) { return std::sqrt(dot(a, a)); }
static inline V3 unit(V3 a) { return divs(a, len(a)); }
static inline V3 reflect(V3 w, V3 n) { return sub(scale(n, 2.0 * dot(w, n)), w); }
static inline double lum(V3 c) { return 0.2126 * c.x + 0.7152 * c.y + 0.0722 * c.z; }
static inline bool zero3(V3 a) { return a.x == 0.0 && a.y == 0.0 && a.z == 0.0; }

// ---- random sequences (core/rng.hpp:11-50) ---------------------------------
struct Rng {
    int kind = 0;  // 0 pcg32, 1 philox4x32-10
    uint64_t state = 0, inc = 0;            // pcg32
    uint64_t key = 0, stream = 0, draw = 0;  // philox
    uint32_t block[4] = {0, 0, 0, 0};
    uint64_t block_id = ~0ULL;

    uint32_t pcg() {
        uint64_t old = state;
        state = old * 6364136223846793005ULL + inc;
        uint32_t xs = static_cast<uint32_t>(((old >> 18u) ^ old) >> 27u);
        uint32_t rot = static_cast<uint32_t>(old >> 59u);
        return (xs >> rot) | (xs << ((~rot + 1u) & 31u));
    }
    void reseed(uint64_t seed, uint64_t strm) {
        if (kind == 0) {
            state = 0;
            inc = (strm << 1u) | 1u;
            pcg();
            state += seed;
            pcg();
        } else {
            key = seed;
            stream = strm;
            draw = 0;
            block_id = ~0ULL;
        }
    }
    static void philox(const uint32_t ctr_in[4], uint32_t k0, uint32_t k1, uint32_t out[4]) {
        uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
        for (int r = 0; r < 10; ++r) {
            uint64_t p0 = static_cast<uint64_t>(0xD2511F53u) * c0;
            uint64_t p1 = static_cast<uint64_t>(0xCD9E8D57u) * c2;
            uint32_t hi0 = static_cast<uint32_t>(p0 >> 32), lo0 = static_cast<uint32_t>(p0);
            uint32_t hi1 = static_cast<uint32_t>(p1 >> 32), lo1 = static_cast<uint32_t>(p1);
            c0 = hi1 ^ c1 ^ k0;
            c1 = lo1;
            c2 = hi0 ^ c3 ^ k1;
            c3 = lo0;
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
        }
        out[0] = c0;
        out[1] = c1;
        out[2] = c2;
        out[3] = c3;
    }
    uint32_t next_u32() {
        if (kind == 0)
            return pcg();
        uint64_t b = draw >> 2;
        if (b != block_id) {
            uint32_t ctr[4] = {static_cast<uint32_t>(b), static_cast<uint32_t>(b >> 32),
                               static_cast<uint32_t>(stream), static_cast<uint32_t>(stream >> 32)};
            philox(ctr, static_cast<uint32_t>(key), static_cast<uint32_t>(key >> 32), block);
            block_id = b;
        }
        return block[draw++ & 3];
    }
    double next_double() {
        uint64_t hi = next_u32();
        uint64_t lo = next_u32();
        return static_cast<double>(((hi << 32) | lo) >> 11) * 0x1.0p-53;
    }
};

// ---- sampling core (core/sampling.cpp) --------------------------------------
static double npdf(double x) { return std::exp(-0.5 * x * x) / std::sqrt(TWO_PI); }  // :9-11
static double ncdf(double x) { return 0.5 * std::erfc(-x / 1.41421356237309504880); }  // :13-15

// Acklam rational approximation + one Halley step (core/sampling.cpp:19-60).
static double nquantile(double p) {
    static const double A[] = {-3.969683028665376e+01, 2.209460984245205e+02,
                               -2.759285104469687e+02, 1.383577518672690e+02,
                               -3.066479806614716e+01, 2.506628277459239e+00};
    static const double B[] = {-5.447609879822406e+01, 1.615858368580409e+02,
                               -1.556989798598866e+02, 6.680131188771972e+01,
                               -1.328068155288572e+01};
    static const double Cc[] = {-7.784894002430293e-03, -3.223964580411365e-01,
                                -2.400758277161838e+00, -2.549732539343734e+00,
                                4.374664141464968e+00, 2.938163982698783e+00};
    static const double D[] = {7.784695709041462e-03, 3.224671290700398e-01,
                               2.445134137142996e+00, 3.754408661907416e+00};
    double x;
    if (p < 0.02425) {
        double q = std::sqrt(-2.0 * std::log(p));
        x = (((((Cc[0] * q + Cc[1]) * q + Cc[2]) * q + Cc[3]) * q + Cc[4]) * q + Cc[5]) /
            ((((D[0] * q + D[1]) * q + D[2]) * q + D[3]) * q + 1.0);
    } else if (p > 1.0 - 0.02425) {
        double q = std::sqrt(-2.0 * std::log(1.0 - p));
        x = -(((((Cc[0] * q + Cc[1]) * q + Cc[2]) * q + Cc[3]) * q + Cc[4]) * q + Cc[5]) /
            ((((D[0] * q + D[1]) * q + D[2]) * q + D[3]) * q + 1.0);
    } else {
        double q = p - 0.5;
        double r = q * q;
        x = (((((A[0] * r + A[1]) * r + A[2]) * r + A[3]) * r + A[4]) * r + A[5]) * q /
            (((((B[0] * r + B[1]) * r + B[2]) * r + B[3]) * r + B[4]) * r + 1.0);
    }
    double e = ncdf(x) - p;
    double u = e * std::sqrt(TWO_PI) * std::exp(0.5 * x * x);
    return x - u / (1.0 + 0.5 * x * u);
}

// Truncated normal on [-pi, pi] (core/sampling.cpp:62-92).
struct Kern {
    double sigma, lo, mass;
    explicit Kern(double s) : sigma(s) {
        if (!(s > 0.0))
            throw std::invalid_argument("AngularKernel: sigma must be positive");
        double t = PI / sigma;
        lo = ncdf(-t);
        mass = ncdf(t) - lo;
    }
    double sample(Rng &rng) const {
        double u = rng.next_double();
        double p = lo + u * mass;
        if (p <= 0.0)
            return -PI;
        if (p >= 1.0)
            return PI;
        double th = sigma * nquantile(p);
        return th < -PI ? -PI : (th > PI ? PI : th);
    }
    double pdf(double th) const {
        if (std::abs(th) > PI)
            return 0.0;
        return npdf(th / sigma) / (sigma * mass);
    }
    double pdf_sa(double alpha) const {
        double s = std::max(std::sin(alpha), 1e-300);
        return pdf(alpha) / (PI * s);
    }
};

// Duff et al. frame (core/sampling.cpp:94-101).
struct Frame {
    V3 t, b, n;
    explicit Frame(V3 nn) : n(nn) {
        double sign = std::copysign(1.0, nn.z);
        double a = -1.0 / (sign + nn.z);
        double bb = nn.x * nn.y * a;
        t = v3(1.0 + sign * nn.x * nn.x * a, sign * bb, -sign * nn.x);
        b = v3(bb, sign + nn.y * nn.y * a, -nn.y);
    }
    V3 world(V3 l) const { return add(add(scale(t, l.x), scale(b, l.y)), scale(n, l.z)); }
};

// core/sampling.cpp:103-110
static V3 perturb_dir(V3 w, const Kern &k, Rng &rng) {
    double th = k.sample(rng);
    double ph = TWO_PI * rng.next_double();
    Frame f(w);
    double st = std::sin(th);
    V3 l = v3(st * std::cos(ph), st * std::sin(ph), std::cos(th));
    return unit(f.world(l));
}

// core/sampling.cpp:112-121
static void cyl(V3 w, double *u, double *v) {
    double ph = std::atan2(w.y, w.x);
    if (ph < 0.0)
        ph += TWO_PI;
    double uu = ph / TWO_PI;
    if (uu >= 1.0)
        uu = 0.0;
    double vv = 0.5 * (w.z + 1.0);
    *u = uu;
    *v = vv < 0.0 ? 0.0 : (vv > 1.0 ? 1.0 : vv);
}

// ---- camera (core/camera.cpp) -------------------------------------------------
struct Cam {
    V3 pos, right, up, fwd;
    double tanh_ = 0.0, aspect = 1.0, area = 0.0, sensor = 1.0;

    void init(V3 p, V3 look, V3 upv, double fov) {  // :8-20
        if (!(fov > 0.0 && fov < 180.0))
            throw std::invalid_argument("camera: fov must be in (0, 180) degrees");
        pos = p;
        fwd = unit(sub(look, p));
        V3 r = cross(fwd, upv);
        if (len(r) < 1e-12)
            throw std::invalid_argument("camera: up vector is parallel to the view direction");
        right = unit(r);
        up = cross(right, fwd);
        tanh_ = std::tan(0.5 * fov * PI / 180.0);
        configure(1, 1);
    }
    void configure(int w, int h) {  // :22-30
        aspect = static_cast<double>(w) / static_cast<double>(h);
        area = 4.0 * tanh_ * tanh_ * aspect;
        sensor = static_cast<double>(w) * static_cast<double>(h) / area;
    }
    V3 primary(double u, double v) const {  // :32-36
        double px = (2.0 * u - 1.0) * tanh_ * aspect;
        double py = (2.0 * v - 1.0) * tanh_;
        return unit(add(add(scale(right, px), scale(up, py)), fwd));
    }
    bool raster(V3 w, double *u, double *v) const {  // :38-49
        double c = dot(w, fwd);
        if (c <= 0.0)
            return false;
        double px = dot(w, right) / c;
        double py = dot(w, up) / c;
        double uu = 0.5 * (px / (tanh_ * aspect) + 1.0);
        double vv = 0.5 * (py / tanh_ + 1.0);
        if (uu < 0.0 || uu > 1.0 || vv < 0.0 || vv > 1.0)
            return false;
        *u = uu;
        *v = vv;
        return true;
    }
    double importance(V3 w) const {  // :51-57
        double u, v;
        if (!raster(w, &u, &v))
            return 0.0;
        double c = dot(w, fwd);
        double c2 = c * c;
        return sensor / (c2 * c2);
    }
    double dir_pdf(V3 w) const {  // :59-64
        double u, v;
        if (!raster(w, &u, &v))
            return 0.0;
        double c = dot(w, fwd);
        return 1.0 / (area * c * c * c);
    }
};

// ---- scene (core/scene.cpp) ---------------------------------------------------
enum Kind { DIFFUSE = 0, MIRROR = 1, DIELECTRIC = 2, GLOSSY = 3 };
enum Ev { EV_NONE = 0, EV_REFLECT = 1, EV_TRANSMIT = 2 };

struct Mat {
    int kind = DIFFUSE;
    V3 albedo = {0.5, 0.5, 0.5};
    double ior = 1.5, expo = 32.0;
    bool specular() const { return kind == MIRROR || kind == DIELECTRIC; }
};
struct Sph {
    V3 c;
    double r;
    int mat;
};
struct Tri {
    V3 a, b, c;
    int mat;
};
struct Hit {
    V3 p, n;
    int mat, emi;
    double t;
};

struct Scene {
    Cam cam;
    std::vector<Mat> mats;
    std::vector<Sph> sph;
    std::vector<Tri> tri;
    std::vector<V3> emit_rad;
    std::vector<int> sph_emi, tri_emi;
    mutable uint64_t rays_c = 0, rays_v = 0;
    mutable bool counting = false;

    // core/scene.cpp:15-29
    static bool hit_sphere(const Sph &s, V3 o, V3 d, double *t) {
        V3 oc = sub(o, s.c);
        double b = dot(oc, d);
        double c = dot(oc, oc) - s.r * s.r;
        double disc = b * b - c;
        if (disc < 0.0)
            return false;
        double sq = std::sqrt(disc);
        double tt = -b - sq;
        if (tt > EPS) {
            *t = tt;
            return true;
        }
        tt = -b + sq;
        if (tt > EPS) {
            *t = tt;
            return true;
        }
        return false;
    }
    // core/scene.cpp:31-52 (Moeller-Trumbore)
    static bool hit_tri(const Tri &tr, V3 o, V3 d, double *t) {
        V3 e1 = sub(tr.b, tr.a);
        V3 e2 = sub(tr.c, tr.a);
        V3 p = cross(d, e2);
        double det = dot(e1, p);
        if (std::abs(det) < 1e-14)
            return false;
        double inv = 1.0 / det;
        V3 tv = sub(o, tr.a);
        double u = dot(tv, p) * inv;
        if (u < 0.0 || u > 1.0)
            return false;
        V3 q = cross(tv, e1);
        double v = dot(d, q) * inv;
        if (v < 0.0 || u + v > 1.0)
            return false;
        double tt = dot(e2, q) * inv;
        if (tt > EPS) {
            *t = tt;
            return true;
        }
        return false;
    }
    // core/scene.cpp:57-92: closest hit, spheres first, strict '<' ties.
    bool intersect_raw(V3 o, V3 d, Hit *h) const {
        double best = std::numeric_limits<double>::infinity();
        int bs = -1, bt = -1;
        for (size_t i = 0; i < sph.size(); ++i) {
            double t;
            if (hit_sphere(sph[i], o, d, &t) && t < best) {
                best = t;
                bs = static_cast<int>(i);
                bt = -1;
            }
        }
        for (size_t i = 0; i < tri.size(); ++i) {
            double t;
            if (hit_tri(tri[i], o, d, &t) && t < best) {
                best = t;
                bt = static_cast<int>(i);
                bs = -1;
            }
        }
        if (bs < 0 && bt < 0)
            return false;
        h->t = best;
        h->p = add(o, scale(d, best));
        if (bs >= 0) {
            h->n = unit(sub(h->p, sph[bs].c));
            h->mat = sph[bs].mat;
            h->emi = sph_emi[bs];
        } else {
            const Tri &tr = tri[bt];
            h->n = unit(cross(sub(tr.b, tr.a), sub(tr.c, tr.a)));
            h->mat = tr.mat;
            h->emi = tri_emi[bt];
        }
        return true;
    }
    bool intersect(V3 o, V3 d, Hit *h) const {
        if (counting)
            ++rays_c;
        return intersect_raw(o, d, h);
    }
    // core/scene.cpp:94-102
    bool visible(V3 a, V3 b) const {
        if (counting)
            ++rays_v;
        V3 d = sub(b, a);
        double dist = len(d);
        if (dist <= 2.0 * EPS)
            return false;
        d = divs(d, dist);
        Hit h;
        if (!intersect_raw(a, d, &h))
            return true;
        return h.t >= dist - EPS;
    }
};

// Minimal .scn reader (grammar: SPEC.md:160-166; core/scene.cpp:114-234).
static Scene parse(const std::string &text) {
    Scene s;
    std::map<std::string, int> ids;
    std::vector<std::pair<bool, int>> order;
    bool cam = false;
    std::istringstream in(text);
    std::string line;
    int ln = 0;
    while (std::getline(in, line)) {
        ++ln;
        size_t st = line.find_first_not_of(" \t\r");
        if (st == std::string::npos || line[st] == '#')
            continue;
        std::istringstream ls(line);
        std::string tag;
        ls >> tag;
        auto fail = [&](const char *m) {
            throw std::runtime_error("<scene>:" + std::to_string(ln) + ": " + m);
        };
        if (tag == "camera") {
            V3 p, l, u;
            double fov;
            ls >> p.x >> p.y >> p.z >> l.x >> l.y >> l.z >> u.x >> u.y >> u.z >> fov;
            if (ls.fail())
                fail("malformed camera");
            s.cam.init(p, l, u, fov);
            cam = true;
        } else if (tag == "material") {
            std::string name, kind;
            ls >> name >> kind;
            Mat m;
            if (kind == "diffuse") {
                m.kind = DIFFUSE;
                ls >> m.albedo.x >> m.albedo.y >> m.albedo.z;
            } else if (kind == "mirror") {
                m.kind = MIRROR;
                ls >> m.albedo.x >> m.albedo.y >> m.albedo.z;
            } else if (kind == "dielectric") {
                m.kind = DIELECTRIC;
                ls >> m.ior >> m.albedo.x >> m.albedo.y >> m.albedo.z;
            } else if (kind == "glossy") {
                m.kind = GLOSSY;
                ls >> m.albedo.x >> m.albedo.y >> m.albedo.z >> m.expo;
            } else {
                fail("unknown material kind");
            }
            if (ls.fail())
                fail("malformed material");
            ids[name] = static_cast<int>(s.mats.size());
            s.mats.push_back(m);
        } else if (tag == "sphere") {
            Sph sp;
            std::string mat;
            ls >> sp.c.x >> sp.c.y >> sp.c.z >> sp.r >> mat;
            if (ls.fail() || !ids.count(mat))
                fail("malformed sphere");
            sp.mat = ids[mat];
            order.emplace_back(true, static_cast<int>(s.sph.size()));
            s.sph.push_back(sp);
            s.sph_emi.push_back(-1);
        } else if (tag == "tri") {
            Tri t;
            std::string mat;
            ls >> t.a.x >> t.a.y >> t.a.z >> t.b.x >> t.b.y >> t.b.z >> t.c.x >> t.c.y >> t.c.z >> mat;
            if (ls.fail() || !ids.count(mat))
                fail("malformed tri");
            t.mat = ids[mat];
            order.emplace_back(false, static_cast<int>(s.tri.size()));
            s.tri.push_back(t);
            s.tri_emi.push_back(-1);
        } else if (tag == "emitter") {
            int idx;
            V3 r;
            ls >> idx >> r.x >> r.y >> r.z;
            if (ls.fail() || idx < 0 || idx >= static_cast<int>(order.size()))
                fail("malformed emitter");
            int e = static_cast<int>(s.emit_rad.size());
            s.emit_rad.push_back(r);
            if (order[idx].first)
                s.sph_emi[order[idx].second] = e;
            else
                s.tri_emi[order[idx].second] = e;
        } else {
            fail("unknown record");
        }
    }
    if (!cam)
        throw std::runtime_error("<scene>: scene has no camera");
    if (s.emit_rad.empty())
        throw std::runtime_error("<scene>: scene has no emitter");
    return s;
}

// ---- BSDFs (core/scene.cpp:245-414) --------------------------------------------
static inline V3 facing(V3 n, V3 wi) { return dot(n, wi) >= 0.0 ? n : neg(n); }

static double fresnel(double cos_i, double ior) {  // :260-275
    double ei = 1.0, et = ior, ci = cos_i;
    if (ci < 0.0) {
        std::swap(ei, et);
        ci = -ci;
    }
    double s2 = (ei / et) * (ei / et) * (1.0 - ci * ci);
    if (s2 >= 1.0)
        return 1.0;
    double ct = std::sqrt(1.0 - s2);
    double rpa = (et * ci - ei * ct) / (et * ci + ei * ct);
    double rpe = (ei * ci - et * ct) / (ei * ci + et * ct);
    return 0.5 * (rpa * rpa + rpe * rpe);
}

static V3 bsdf_f(const Mat &m, V3 wi, V3 wo, V3 n) {  // :277-300
    if (m.kind == DIFFUSE) {
        V3 ns = facing(n, wi);
        if (dot(ns, wo) <= 0.0)
            return v3(0, 0, 0);
        return scale(m.albedo, INV_PI);
    }
    if (m.kind == GLOSSY) {
        V3 ns = facing(n, wi);
        if (dot(ns, wo) <= 0.0)
            return v3(0, 0, 0);
        double ca = dot(reflect(wi, ns), wo);
        if (ca <= 0.0)
            return v3(0, 0, 0);
        double norm = (m.expo + 1.0) / TWO_PI;
        return scale(m.albedo, norm * std::pow(ca, m.expo));
    }
    return v3(0, 0, 0);
}

static double bsdf_p(const Mat &m, V3 wi, V3 wo, V3 n) {  // :302-321
    if (m.kind == DIFFUSE) {
        V3 ns = facing(n, wi);
        double c = dot(ns, wo);
        return c > 0.0 ? c * INV_PI : 0.0;
    }
    if (m.kind == GLOSSY) {
        V3 ns = facing(n, wi);
        double ca = dot(reflect(wi, ns), wo);
        if (ca <= 0.0)
            return 0.0;
        return (m.expo + 1.0) / TWO_PI * std::pow(ca, m.expo);
    }
    return 0.0;
}

static bool spec_cont(const Mat &m, V3 wi, V3 n, int ev, V3 *out) {  // :393-414
    if (m.kind == MIRROR) {
        if (ev != EV_REFLECT)
            return false;
        *out = unit(reflect(wi, facing(n, wi)));
        return true;
    }
    if (m.kind != DIELECTRIC)
        return false;
    double cos_i = dot(n, wi);
    if (ev == EV_REFLECT) {
        *out = unit(reflect(wi, facing(n, wi)));
        return true;
    }
    double eta = cos_i > 0.0 ? 1.0 / m.ior : m.ior;
    V3 ns = facing(n, wi);
    double ci = dot(ns, wi);
    double s2 = eta * eta * (1.0 - ci * ci);
    if (s2 >= 1.0)
        return false;
    double ct = std::sqrt(1.0 - s2);
    *out = unit(add(scale(wi, -eta), scale(ns, eta * ci - ct)));
    return true;
}

static V3 spec_weight(const Mat &m, V3 wi, V3 n, int ev) {  // :369-380
    if (m.kind == MIRROR)
        return ev == EV_REFLECT ? m.albedo : v3(0, 0, 0);
    if (m.kind == DIELECTRIC) {
        double f = fresnel(dot(n, wi), m.ior);
        if (ev == EV_REFLECT)
            return scale(m.albedo, f);
        if (ev == EV_TRANSMIT)
            return scale(m.albedo, 1.0 - f);
    }
    return v3(0, 0, 0);
}

static double spec_prob(const Mat &m, V3 wi, V3 n, int ev) {  // :382-391
    if (m.kind == MIRROR)
        return ev == EV_REFLECT ? 1.0 : 0.0;
    if (m.kind == DIELECTRIC) {
        double f = fresnel(dot(n, wi), m.ior);
        return ev == EV_REFLECT ? f : 1.0 - f;
    }
    return 0.0;
}

struct BS {
    V3 dir;
    double pdf;
    V3 thr;
    bool delta;
    int ev;
};

static bool bsdf_sample(const Mat &m, V3 wi, V3 n, Rng &rng, BS *bs) {  // :323-367
    if (m.kind == DIFFUSE) {
        V3 ns = facing(n, wi);
        double u1 = rng.next_double();
        double u2 = rng.next_double();
        double r = std::sqrt(u1);
        double ph = TWO_PI * u2;
        V3 l = v3(r * std::cos(ph), r * std::sin(ph), std::sqrt(std::max(0.0, 1.0 - u1)));
        V3 wo = Frame(ns).world(l);
        double pdf = std::max(dot(ns, wo), 0.0) * INV_PI;
        if (pdf <= 0.0)
            return false;
        *bs = {wo, pdf, m.albedo, false, EV_NONE};
        return true;
    }
    if (m.kind == GLOSSY) {
        V3 ns = facing(n, wi);
        V3 axis = reflect(wi, ns);
        double u1 = rng.next_double();
        double u2 = rng.next_double();
        double ca = std::pow(u1, 1.0 / (m.expo + 1.0));
        double sa = std::sqrt(std::max(0.0, 1.0 - ca * ca));
        double ph = TWO_PI * u2;
        V3 l = v3(sa * std::cos(ph), sa * std::sin(ph), ca);
        V3 wo = unit(Frame(axis).world(l));
        double pdf = (m.expo + 1.0) / TWO_PI * std::pow(ca, m.expo);
        double co = dot(ns, wo);
        *bs = {wo, pdf, co > 0.0 ? scale(m.albedo, co) : v3(0, 0, 0), false, EV_NONE};
        return true;
    }
    if (m.kind == MIRROR) {
        V3 ns = facing(n, wi);
        *bs = {unit(reflect(wi, ns)), 1.0, m.albedo, true, EV_REFLECT};
        return true;
    }
    double f = fresnel(dot(n, wi), m.ior);
    int ev = rng.next_double() < f ? EV_REFLECT : EV_TRANSMIT;
    V3 wo;
    if (!spec_cont(m, wi, n, ev, &wo))
        return false;
    double q = ev == EV_REFLECT ? f : 1.0 - f;
    *bs = {wo, q, divs(spec_weight(m, wi, n, ev), q), true, ev};
    return true;
}

// ---- paths (core/path.hpp:13-41, core/path.cpp) ---------------------------------
struct Vtx {
    V3 p, n;
    int mat = -1, emi = -1;
    bool cam = false, spec = false;
    int ev = EV_NONE;
};
using Path = std::vector<Vtx>;
static inline V3 pdir(const Path &P, int i) { return unit(sub(P[i + 1].p, P[i].p)); }

struct Contrib {
    V3 f = {0, 0, 0};
    double pi = 0.0;
    double u = 0.0, v = 0.0;
};

static double geom(const Scene &s, const Vtx &a, const Vtx &b) {  // core/path.cpp:7-17
    V3 d = sub(b.p, a.p);
    double d2 = dot(d, d);
    if (d2 <= 0.0)
        return 0.0;
    V3 dir = divs(d, std::sqrt(d2));
    double g = std::abs(dot(a.n, dir)) * std::abs(dot(b.n, dir)) / d2;
    if (g <= 0.0)
        return 0.0;
    return s.visible(a.p, b.p) ? g : 0.0;
}

static double aconv(const Scene &s, V3 from, const Vtx &b) {  // core/path.cpp:19-29
    V3 d = sub(b.p, from);
    double d2 = dot(d, d);
    if (d2 <= 0.0)
        return 0.0;
    V3 dir = divs(d, std::sqrt(d2));
    double c = std::abs(dot(b.n, dir)) / d2;
    if (c <= 0.0)
        return 0.0;
    return s.visible(from, b.p) ? c : 0.0;
}

static Contrib evaluate(const Scene &s, const Path &P) {  // core/path.cpp:40-82
    Contrib z;
    int k = static_cast<int>(P.size());
    if (k < 2 || !P[0].cam || P[k - 1].emi < 0)
        return z;
    V3 w0 = pdir(P, 0);
    double ru, rv;
    if (!s.cam.raster(w0, &ru, &rv))
        return z;
    double imp = s.cam.importance(w0);
    V3 f = v3(imp, imp, imp);
    for (int i = 0; i + 1 < k; ++i) {
        const Vtx &a = P[i];
        const Vtx &b = P[i + 1];
        if (i > 0 && a.emi >= 0)
            return z;
        double seg = a.spec ? aconv(s, a.p, b) : geom(s, a, b);
        if (seg <= 0.0)
            return z;
        f = scale(f, seg);
        if (i > 0) {
            const Mat &m = s.mats[a.mat];
            V3 wi = unit(sub(P[i - 1].p, a.p));
            V3 wo = pdir(P, i);
            V3 bf = a.spec ? spec_weight(m, wi, a.n, a.ev) : bsdf_f(m, wi, wo, a.n);
            if (zero3(bf))
                return z;
            f = mul(f, bf);
        }
    }
    const Vtx &last = P[k - 1];
    V3 toward = unit(sub(P[k - 2].p, last.p));
    if (last.emi < 0 || dot(last.n, toward) <= 0.0)
        return z;
    V3 le = s.emit_rad[last.emi];
    if (zero3(le))
        return z;
    f = mul(f, le);
    double pi = lum(f);
    if (!(pi > 0.0) || !std::isfinite(pi))
        return z;
    z.f = f;
    z.pi = pi;
    z.u = ru;
    z.v = rv;
    return z;
}

struct Rec {
    double pdf, ac;
};

// core/path.cpp:84-142; returns true when an emitter was hit.
static bool trace_eye(const Scene &s, Rng &rng, int maxv, Path &P, std::vector<Rec> &R) {
    P.clear();
    R.clear();
    Vtx c;
    c.p = s.cam.pos;
    c.n = s.cam.fwd;
    c.cam = true;
    P.push_back(c);
    if (maxv < 2)
        return false;
    double u = rng.next_double();
    double v = rng.next_double();
    V3 dir = s.cam.primary(u, v);
    double dpdf = s.cam.dir_pdf(dir);
    V3 o = s.cam.pos;
    while (static_cast<int>(P.size()) < maxv) {
        Hit h;
        if (!s.intersect(o, dir, &h))
            return false;
        Vtx x;
        x.p = h.p;
        x.n = h.n;
        x.mat = h.mat;
        x.emi = h.emi;
        x.spec = h.emi < 0 && s.mats[h.mat].specular();
        R.push_back({dpdf, std::abs(dot(h.n, dir)) / (h.t * h.t)});
        P.push_back(x);
        if (h.emi >= 0)
            return true;
        if (static_cast<int>(P.size()) >= maxv)
            return false;
        BS bs;
        if (!bsdf_sample(s.mats[h.mat], neg(dir), h.n, rng, &bs) || zero3(bs.thr))
            return false;
        P.back().ev = bs.ev;
        o = h.p;
        dir = bs.dir;
        dpdf = bs.pdf;
    }
    return false;
}

static double eye_density(const Scene &s, const Path &P) {  // core/path.cpp:144-170
    int k = static_cast<int>(P.size());
    if (k < 2 || !P[0].cam || P[k - 1].emi < 0)
        return 0.0;
    double p = s.cam.dir_pdf(pdir(P, 0));
    if (p <= 0.0)
        return 0.0;
    p *= aconv(s, P[0].p, P[1]);
    for (int i = 1; i + 1 < k; ++i) {
        const Vtx &a = P[i];
        if (a.emi >= 0)
            return 0.0;
        const Mat &m = s.mats[a.mat];
        V3 wi = unit(sub(P[i - 1].p, a.p));
        V3 wo = pdir(P, i);
        double q = a.spec ? spec_prob(m, wi, a.n, a.ev) : bsdf_p(m, wi, wo, a.n);
        if (q <= 0.0)
            return 0.0;
        p *= q * aconv(s, a.p, P[i + 1]);
        if (p <= 0.0)
            return 0.0;
    }
    return p;
}

// ---- mutations (core/mutations.cpp) ---------------------------------------------
static int lens_endpoint(const Path &P) {  // :9-21, -1 when ineligible
    int k = static_cast<int>(P.size());
    if (k < 2 || !P[0].cam)
        return -1;
    int s = 1;
    while (s < k - 1 && P[s].spec)
        ++s;
    if (s == k - 1)
        return s;
    if (!P[s + 1].spec)
        return s;
    return -1;
}

// :23-45; false when ineligible.
static bool mc_structure(const Path &P, std::vector<int> &pert, int *endpoint) {
    int k = static_cast<int>(P.size());
    if (k < 3 || !P[0].cam)
        return false;
    int first = 1;
    while (first < k - 1 && P[first].spec)
        ++first;
    if (first == k - 1)
        return false;
    int e = -1;
    for (int i = first + 1; i < k; ++i) {
        if (i == k - 1 || (!P[i].spec && !P[i + 1].spec)) {
            e = i;
            break;
        }
    }
    pert.clear();
    for (int i = 0; i < e; ++i)
        if (!P[i].spec)
            pert.push_back(i);
    *endpoint = e;
    return true;
}

static double suit(const Path &P, int perturbation) {  // :47-56
    if (perturbation == 0)
        return lens_endpoint(P) >= 0 ? 0.5 : 0.0;
    std::vector<int> pert;
    int e;
    return mc_structure(P, pert, &e) ? 0.5 : 0.0;
}

// :78-110 (retrace_chain): appends ref[start+1..end] re-traced from o along d.
static bool retrace(const Scene &s, const Path &ref, int start, int end, V3 o, V3 d, Path &out) {
    for (int i = start + 1; i <= end; ++i) {
        Hit h;
        if (!s.intersect(o, d, &h))
            return false;
        const Vtx &r = ref[i];
        bool he = h.emi >= 0;
        bool hs = !he && s.mats[h.mat].specular();
        if (he != (r.emi >= 0) || hs != r.spec)
            return false;
        Vtx x;
        x.p = h.p;
        x.n = h.n;
        x.mat = h.mat;
        x.emi = h.emi;
        x.spec = hs;
        x.ev = r.ev;
        out.push_back(x);
        if (i == end)
            break;
        V3 c;
        if (!spec_cont(s.mats[h.mat], neg(d), h.n, r.ev, &c))
            return false;
        o = h.p;
        d = c;
    }
    return true;
}

struct Kpair {
    const Kern *k1, *k2;
};

// :176-196
static double pert_density(const Path &from, const Path &to, const std::vector<int> &pert,
                           int endpoint, Kpair k) {
    double q = 1.0;
    for (int idx : pert) {
        V3 a = pdir(from, idx);
        V3 b = pdir(to, idx);
        double alpha = std::atan2(len(cross(a, b)), dot(a, b));
        q *= (idx == 0 ? k.k1 : k.k2)->pdf_sa(alpha);
    }
    for (int i = 0; i < endpoint; ++i) {
        V3 d = sub(to[i + 1].p, to[i].p);
        double d2 = dot(d, d);
        if (d2 <= 0.0)
            return 0.0;
        q *= std::abs(dot(to[i + 1].n, d)) / (d2 * std::sqrt(d2));
    }
    return q;
}

struct Prop {
    Path path;
    double tf = 0.0, tr = 0.0;
    std::vector<int> pert;
    int endpoint = 0;
};

// :122-146 lens_perturb and :148-174 multichain_perturb
static bool perturb(const Scene &s, const Path &P, int kind, Kpair k, Rng &rng, Prop &pr) {
    pr.path.clear();
    if (kind == 0) {
        int e = lens_endpoint(P);
        if (e < 0)
            return false;
        V3 nd = perturb_dir(pdir(P, 0), *k.k1, rng);
        pr.path.push_back(P[0]);
        if (!retrace(s, P, 0, e, P[0].p, nd, pr.path))
            return false;
        pr.pert.assign(1, 0);
        pr.endpoint = e;
    } else {
        if (!mc_structure(P, pr.pert, &pr.endpoint))
            return false;
        pr.path.push_back(P[0]);
        for (size_t ci = 0; ci < pr.pert.size(); ++ci) {
            int idx = pr.pert[ci];
            int next = ci + 1 < pr.pert.size() ? pr.pert[ci + 1] : pr.endpoint;
            V3 nd = perturb_dir(pdir(P, idx), idx == 0 ? *k.k1 : *k.k2, rng);
            V3 o = pr.path.back().p;
            if (!retrace(s, P, idx, next, o, nd, pr.path))
                return false;
        }
    }
    for (int i = pr.endpoint + 1; i < static_cast<int>(P.size()); ++i)
        pr.path.push_back(P[i]);
    pr.tf = pert_density(P, pr.path, pr.pert, pr.endpoint, k);
    pr.tr = pert_density(pr.path, P, pr.pert, pr.endpoint, k);
    return true;
}

static double mh(double pc, double pp, double tf, double tr, double sf, double sr) {  // :198-208
    if (!(pc > 0.0))
        throw std::invalid_argument("mh_accept: chain occupies a zero-measure state");
    if (!(pp > 0.0) || !(tf > 0.0) || !(sf > 0.0))
        return 0.0;
    double r = (pp * tr * sr) / (pc * tf * sf);
    if (std::isnan(r))
        return 0.0;
    return std::min(1.0, r);
}

// ---- adaptation (core/adaptation.cpp) ---------------------------------------------
struct Adapt {
    int L = 10;
    double gmax = 1.0, gscale = 5.0, target = 0.5, linit = 1.0, lmin = -30.0, ratio = 1.0;
};
static double gamma_n(const Adapt &c, uint64_t n) {  // :10-13
    if (n < 1)
        throw std::logic_error("step_size needs n >= 1");
    return std::min(c.gmax, c.gscale / std::sqrt(static_cast<double>(n)));
}
static double lambda_next(double lam, double ah, uint64_t n, const Adapt &c) {  // :15-20
    double g = gamma_n(c, n);
    double diff = ah - c.target;
    double sg = diff > 0.0 ? 1.0 : (diff < 0.0 ? -1.0 : 0.0);
    return std::max(c.lmin, lam + g * sg);
}

struct Region {
    double lambda = 0.0;
    uint32_t pend_n = 0;
    double pend_sum = 0.0;
    uint64_t pend_fx = 0;
    uint64_t n = 1;
    uint64_t tot_vis = 0;
    double tot_acc = 0.0;
    uint64_t tot_fx = 0;
};

// ---- partitions (core/partition.cpp) ----------------------------------------------
struct Node {
    int level = 0;
    uint32_t ix = 0, iy = 0;
    int child = -1, region = -1, tree = 0;
};

static int grid_cell(int n, double u, double v) {  // :16-20
    int ix = std::min(static_cast<int>(u * n), n - 1);
    int iy = std::min(static_cast<int>(v * n), n - 1);
    return iy * n + ix;
}

struct Partition {
    int kind = 0;  // 0 none, 1 lens grid, 2 lens quadtree, 3 mc grid, 4 mc quadtree
    int ntop = 20, nbot = 50;
    std::vector<Node> nodes;
    std::vector<int> roots;
    std::vector<uint64_t> visits;  // by region
    std::vector<int> region_tree;  // quadtree: region -> tree (-1 retired)

    int descend(int root, double u, double v) const {  // :48-59
        const Node *nd = &nodes[root];
        while (nd->child >= 0) {
            double sc = std::ldexp(1.0, -nd->level);
            double mu = (nd->ix + 0.5) * sc;
            double mv = (nd->iy + 0.5) * sc;
            int q = (u >= mu ? 1 : 0) + (v >= mv ? 2 : 0);
            nd = &nodes[nd->child + q];
        }
        return nd->region;
    }
    int classify(double ru, double rv, double cu, double cv) const {
        switch (kind) {
        case 1: return grid_cell(ntop, ru, rv);
        case 2: return descend(0, ru, rv);
        case 3: return grid_cell(ntop, ru, rv) * (nbot * nbot) + grid_cell(nbot, cu, cv);
        case 4: return descend(roots[grid_cell(ntop, ru, rv)], cu, cv);
        }
        return 0;
    }
    size_t count() const {
        if (kind == 1)
            return static_cast<size_t>(ntop) * ntop;
        if (kind == 3)
            return static_cast<size_t>(ntop) * ntop * nbot * nbot;
        size_t leaves = 0;
        for (const Node &n : nodes)
            if (n.child < 0)
                ++leaves;
        return leaves;
    }
};

// ---- the render driver (core/driver.cpp) -----------------------------------------
struct Chain {
    Path path;
    Contrib c;
    Rng rng;
    double acc = 0.0, iacc = 0.0;
    uint64_t npert = 0, nlarge = 0, ipert = 0;
};

struct Visit {
    int region;
    double a;
    uint64_t index;
};

struct Out {
    std::vector<double> film;
    double film_lum = 0.0;
    double b = 0.0, b_se = 0.0;
    uint64_t b_n = 0;
    uint64_t done = 0, npert = 0, nlarge = 0;
    double mean_acc = 0.0, identity = 0.0;
    size_t regions = 0;
    std::vector<std::pair<double, uint64_t>> tallies;
    std::vector<oracle_trace_row> trace;
    std::vector<std::array<double, 4>> metrics;
    std::string dump;
    uint64_t rays_c = 0, rays_v = 0;
    double loop_s = 0.0;
};

// pooled rule: 2^-24 fixed point, the GPU engine's resolution (k_adapt_pool_accum)
static inline uint64_t to_fx(double a) { return static_cast<uint64_t>(a * 16777216.0 + 0.5); }

// Single-sample b estimator value (core/driver.cpp:36-50).
static double b_sample(const Scene &s, Rng &rng, int maxv) {
    Path P;
    std::vector<Rec> R;
    if (!trace_eye(s, rng, maxv, P, R))
        return 0.0;
    Contrib c = evaluate(s, P);
    if (!(c.pi > 0.0))
        return 0.0;
    double p = 1.0;
    for (const Rec &r : R)
        p *= r.pdf * r.ac;
    return p > 0.0 ? c.pi / p : 0.0;
}

struct Render {
    const Scene &s;
    const oracle_config &cfg;
    Adapt ad;
    int ctl = 0;  // 0 fixed, 1 global, 2 regional
    Partition part;
    std::vector<Region> reg;
    std::vector<Chain> ch;
    Out out;
    oracle_log *log;
    std::vector<std::vector<std::pair<double, uint8_t>>> logs;

    Render(const Scene &sc, const oracle_config &c, oracle_log *lg) : s(sc), cfg(c), log(lg) {}

    int alloc_region(double lam, uint64_t n) {
        Region r;
        r.lambda = lam;
        r.n = n;
        reg.push_back(r);
        part.visits.push_back(0);
        return static_cast<int>(reg.size()) - 1;
    }

    // classify_path (core/driver.cpp:95-107)
    int region_of(const Path &P, const Contrib &c) const {
        if (ctl != 2)
            return 0;
        double cu = 0.0, cv = 0.0;
        if (cfg.perturbation == 1) {
            std::vector<int> pert;
            int e;
            if (!mc_structure(P, pert, &e))
                throw std::logic_error("classify on multi-chain ineligible path");
            int cidx = pert.size() > 1 ? pert[1] : e;
            cyl(pdir(P, cidx), &cu, &cv);
        }
        return part.classify(c.u, c.v, cu, cv);
    }

    double lambda_of(int r) const { return ctl == 0 ? ad.linit : reg[r].lambda; }

    void splat(const Contrib &cur, const Contrib *prop, double a) {  // core/driver.cpp:59-64
        auto add1 = [&](const Contrib &c, double w) {
            int W = cfg.width, H = cfg.height;
            int x = std::min(static_cast<int>(c.u * W), W - 1);
            int row = H - 1 - std::min(static_cast<int>(c.v * H), H - 1);
            V3 val = scale(c.f, w);
            double *px = &out.film[(static_cast<size_t>(row) * W + x) * 3];
            px[0] += val.x;
            px[1] += val.y;
            px[2] += val.z;
            out.film_lum += lum(val);
        };
        if (a < 1.0 && cur.pi > 0.0)
            add1(cur, (1.0 - a) / cur.pi);
        if (prop && a > 0.0 && prop->pi > 0.0)
            add1(*prop, a / prop->pi);
    }

    // One mutation of one chain (core/driver.cpp:113-171).
    void step(int ci, uint64_t index, std::vector<Visit> &visits) {
        Chain &c = ch[ci];
        int pk = cfg.perturbation;
        double s_pert = suit(c.path, pk);
        bool choose = s_pert > 0.0 && c.rng.next_double() < s_pert;
        double a = 0.0;
        Prop pr;
        bool have = false;
        Contrib pc;
        if (choose) {
            int region = region_of(c.path, c.c);
            double sig = std::exp(0.5 * lambda_of(region));
            Kern k1(sig), k2(ad.ratio * sig);
            have = perturb(s, c.path, pk, {&k1, &k2}, c.rng, pr);
            if (have) {
                pc = evaluate(s, pr.path);
                if (pc.pi > 0.0) {
                    if (ctl == 2) {
                        int pr_region = region_of(pr.path, pc);
                        double sig2 = std::exp(0.5 * lambda_of(pr_region));
                        Kern r1(sig2), r2(ad.ratio * sig2);
                        pr.tr = pert_density(pr.path, c.path, pr.pert, pr.endpoint, {&r1, &r2});
                    }
                    a = mh(c.c.pi, pc.pi, pr.tf, pr.tr, s_pert, s_pert);
                }
            }
            if (ctl == 2)
                ++part.visits[region];
            if (ctl != 0)
                visits.push_back({region, a, index});
            c.acc += a;
            c.iacc += a;
            ++c.npert;
            ++c.ipert;
        } else {
            ++c.nlarge;
            std::vector<Rec> R;
            if (trace_eye(s, c.rng, cfg.max_vertices, pr.path, R)) {
                have = true;
                pr.tf = 1.0;
                for (const Rec &r : R)
                    pr.tf *= r.pdf * r.ac;
                pr.tr = eye_density(s, c.path);
                pc = evaluate(s, pr.path);
                if (pc.pi > 0.0) {
                    double sx = 1.0 - s_pert;
                    double sy = 1.0 - suit(pr.path, pk);
                    a = mh(c.c.pi, pc.pi, pr.tf, pr.tr, sx, sy);
                }
            }
        }
        splat(c.c, pc.pi > 0.0 ? &pc : nullptr, a);
        bool accepted = false;
        if (a > 0.0 && c.rng.next_double() < a) {
            c.path = pr.path;
            c.c = pc;
            accepted = true;
        }
        if (log && logs[ci].size() < log->steps)
            logs[ci].push_back({a, static_cast<uint8_t>((accepted ? 1 : 0) | (choose ? 2 : 0) | 4)});
    }

    void emit_trace(uint64_t index, int region, uint64_t n, double lam, double ah) {
        if (cfg.trace_enabled)
            out.trace.push_back({index, region, n, lam, ah});
    }

    // Shared adaptation after one lockstep step.
    void adapt(const std::vector<Visit> &visits) {
        if (ctl == 0)
            return;
        if (cfg.adapt_mode == 0) {
            // literal: record_acceptance (core/adaptation.cpp:60-92) in chain order
            for (const Visit &v : visits) {
                Region &r = reg[v.region];
                r.tot_acc += v.a;
                r.tot_vis += 1;
                r.pend_sum += v.a;
                r.pend_n += 1;
                if (r.pend_n < static_cast<uint32_t>(ad.L))
                    continue;
                double ah = std::clamp(r.pend_sum / r.pend_n, 0.0, 1.0);
                uint64_t n = r.n;
                r.lambda = lambda_next(r.lambda, ah, n, ad);
                r.n = n + 1;
                r.pend_n = 0;
                r.pend_sum = 0.0;
                emit_trace(v.index, v.region, n, r.lambda, ah);
            }
        } else {
            // pooled: one update per region per step from fixed-point sums
            std::map<int, std::pair<uint64_t, uint64_t>> step;  // region -> (count, last index)
            for (const Visit &v : visits) {
                Region &r = reg[v.region];
                uint64_t fx = to_fx(v.a);
                r.tot_fx += fx;
                r.tot_vis += 1;
                r.pend_fx += fx;
                r.pend_n += 1;
                step[v.region] = {step[v.region].first + 1, v.index};
            }
            for (auto &kv : step) {
                Region &r = reg[kv.first];
                if (r.pend_n < static_cast<uint32_t>(ad.L))
                    continue;
                double ah = std::clamp(static_cast<double>(r.pend_fx) / 16777216.0 /
                                           static_cast<double>(r.pend_n), 0.0, 1.0);
                uint64_t n = r.n;
                r.lambda = lambda_next(r.lambda, ah, n, ad);
                r.n = n + 1;
                r.pend_n = 0;
                r.pend_fx = 0;
                emit_trace(kv.second.second, kv.first, n, r.lambda, ah);
            }
        }
    }

    // Quadtree refine (core/partition.cpp:68-100, 217-227; adaptation.cpp:34-42).
    void refine() {
        if (part.kind != 2 && part.kind != 4)
            return;
        size_t n0 = part.nodes.size();
        std::vector<std::vector<int>> per_tree(part.roots.size());
        for (size_t i = 0; i < n0; ++i)
            if (part.nodes[i].child < 0)
                per_tree[part.nodes[i].tree].push_back(static_cast<int>(i));
        for (auto &cands : per_tree) {
            for (int idx : cands) {
                Node nd = part.nodes[idx];
                if (nd.level >= MAX_DEPTH)
                    continue;
                if (part.visits[nd.region] < cfg.m_split)
                    continue;
                int first = static_cast<int>(part.nodes.size());
                for (int q = 0; q < 4; ++q) {
                    Node c;
                    c.level = nd.level + 1;
                    c.ix = nd.ix * 2 + (q & 1);
                    c.iy = nd.iy * 2 + (q >> 1);
                    c.tree = nd.tree;
                    uint64_t np = reg[nd.region].n;
                    c.region = alloc_region(reg[nd.region].lambda, std::max<uint64_t>(1, np / 4));
                    part.nodes.push_back(c);
                }
                part.nodes[idx].child = first;
                part.visits[nd.region] = 0;
            }
        }
    }

    void dump_partition() {
        std::ostringstream os;
        auto leaf_line = [&](int region, double u0, double v0, double u1, double v1) {
            os << "leaf " << region << " " << u0 << " " << v0 << " " << u1 << " " << v1 << " "
               << lambda_of(region) << " " << reg[region].n << " " << part.visits[region] << "\n";
        };
        auto cell_b = [](int n, int cell, double *b) {
            int iy = cell / n, ix = cell % n;
            double inv = 1.0 / n;
            b[0] = ix * inv;
            b[1] = iy * inv;
            b[2] = (ix + 1) * inv;
            b[3] = (iy + 1) * inv;
        };
        auto tree_leaves = [&](int tree) {
            for (const Node &nd : part.nodes) {
                if (nd.tree != tree || nd.child >= 0)
                    continue;
                double sc = std::ldexp(1.0, -nd.level);
                leaf_line(nd.region, nd.ix * sc, nd.iy * sc, (nd.ix + 1) * sc, (nd.iy + 1) * sc);
            }
        };
        double b[4];
        if (part.kind == 1) {
            for (int c = 0; c < part.ntop * part.ntop; ++c) {
                cell_b(part.ntop, c, b);
                leaf_line(c, b[0], b[1], b[2], b[3]);
            }
        } else if (part.kind == 2) {
            tree_leaves(0);
        } else if (part.kind == 3 || part.kind == 4) {
            for (int c = 0; c < part.ntop * part.ntop; ++c) {
                cell_b(part.ntop, c, b);
                os << "# cell " << c << " " << b[0] << " " << b[1] << " " << b[2] << " " << b[3] << "\n";
                if (part.kind == 4) {
                    tree_leaves(c);
                } else {
                    for (int sb = 0; sb < part.nbot * part.nbot; ++sb) {
                        double bb[4];
                        cell_b(part.nbot, sb, bb);
                        leaf_line(c * part.nbot * part.nbot + sb, bb[0], bb[1], bb[2], bb[3]);
                    }
                }
            }
        }
        out.dump = os.str();
    }

    void run() {
        const oracle_config &c = cfg;
        if (c.chains < 1)
            throw std::logic_error("need at least one chain");
        if (c.width < 1 || c.height < 1)
            throw std::logic_error("resolution must be positive");
        if (c.max_vertices < 2)
            throw std::logic_error("max_vertices must be at least 2");
        ad.L = c.batch_size;
        ad.gmax = c.gamma_max;
        ad.gscale = c.gamma_scale;
        ad.target = c.target_acceptance;
        ad.linit = c.lambda_init;
        ad.lmin = c.lambda_min;
        ad.ratio = c.sigma2_ratio;
        out.film.assign(static_cast<size_t>(c.width) * c.height * 3, 0.0);

        // b (core/driver.cpp:31-57) over B_SUBSTREAMS independent substreams
        if (c.b_override > 0.0) {
            out.b = c.b_override;
        } else {
            if (c.b_samples < 1)
                throw std::logic_error("estimate_b needs at least one sample");
            uint64_t S = std::min<uint64_t>(c.b_samples, B_SUBSTREAMS);
            std::vector<double> ps(S, 0.0), pq(S, 0.0);
            for (uint64_t sub = 0; sub < S; ++sub) {
                Rng rng;
                rng.kind = c.rng;
                rng.reseed(c.seed, STREAM_B + 2 * sub);
                for (uint64_t j = sub; j < c.b_samples; j += S) {
                    double v = b_sample(s, rng, c.max_vertices);
                    ps[sub] += v;
                    pq[sub] += v * v;
                }
            }
            double sum = 0.0, sq = 0.0;
            for (uint64_t sub = 0; sub < S; ++sub) {
                sum += ps[sub];
                sq += pq[sub];
            }
            double n = static_cast<double>(c.b_samples);
            double mean = sum / n;
            if (mean <= 0.0)
                throw std::runtime_error("black-scene: no sample carried any contribution");
            double var = c.b_samples > 1 ? std::max(0.0, (sq - n * mean * mean) / (n - 1.0)) : 0.0;
            out.b = mean;
            out.b_se = std::sqrt(var / n);
            out.b_n = c.b_samples;
        }

        // controller + partition (core/driver.cpp:190-212)
        ctl = c.strategy == 0 ? 0 : (c.strategy == 1 ? 1 : 2);
        part.ntop = c.n_top;
        part.nbot = c.n_bottom;
        if (ctl != 2) {
            alloc_region(ad.linit, 1);
        } else if (c.strategy == 2) {
            part.kind = c.perturbation == 0 ? 1 : 3;
            size_t n = part.kind == 1 ? static_cast<size_t>(c.n_top) * c.n_top
                                      : static_cast<size_t>(c.n_top) * c.n_top * c.n_bottom * c.n_bottom;
            for (size_t i = 0; i < n; ++i)
                alloc_region(ad.linit, 1);
        } else {
            part.kind = c.perturbation == 0 ? 2 : 4;
            int trees = part.kind == 2 ? 1 : c.n_top * c.n_top;
            for (int t = 0; t < trees; ++t) {
                Node nd;
                nd.tree = t;
                nd.region = alloc_region(ad.linit, 1);
                part.roots.push_back(static_cast<int>(part.nodes.size()));
                part.nodes.push_back(nd);
            }
        }

        // chain init (core/driver.cpp:219-242); chain i has global id off + i
        const uint64_t off = static_cast<uint64_t>(c.chain_offset);
        const uint64_t ctot = c.chains_total > 0 ? static_cast<uint64_t>(c.chains_total)
                                                 : static_cast<uint64_t>(c.chains);
        ch.resize(c.chains);
        logs.resize(c.chains);
        for (int i = 0; i < c.chains; ++i) {
            Chain &cc = ch[i];
            const uint64_t gid = off + static_cast<uint64_t>(i);
            cc.rng.kind = c.rng;
            cc.rng.reseed(c.seed, gid);
            Rng init;
            init.kind = c.rng;
            init.reseed(c.seed, STREAM_INIT + gid * 2);
            bool ok = false;
            Path P;
            std::vector<Rec> R;
            for (uint64_t t = 0; t < MAX_INIT; ++t) {
                if (!trace_eye(s, init, c.max_vertices, P, R))
                    continue;
                Contrib con = evaluate(s, P);
                if (con.pi > 0.0) {
                    cc.path = P;
                    cc.c = con;
                    ok = true;
                    break;
                }
            }
            if (!ok)
                throw std::runtime_error("black-scene: could not find an initial path");
        }

        // span loop (core/driver.cpp:276-311) in lockstep order
        auto t0 = std::chrono::steady_clock::now();
        auto now = [&] {
            return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        };
        uint64_t budget = c.mutations;
        uint64_t done = 0, next_refine = c.m_refine, next_metrics = c.metrics_interval;
        s.counting = true;
        auto flush = [&](uint64_t at) {
            double sum = 0.0;
            uint64_t cnt = 0;
            for (Chain &cc : ch) {
                sum += cc.iacc;
                cnt += cc.ipert;
                cc.iacc = 0.0;
                cc.ipert = 0;
            }
            out.metrics.push_back({now(), static_cast<double>(at),
                                   std::numeric_limits<double>::quiet_NaN(),
                                   cnt > 0 ? sum / static_cast<double>(cnt) : 0.0});
        };
        std::vector<Visit> visits;
        while (done < budget) {
            uint64_t boundary = std::min({budget, next_refine, next_metrics});
            uint64_t span = boundary - done;
            uint64_t per = span / ctot, rem = span % ctot;
            uint64_t steps = per + (rem ? 1 : 0);
            for (uint64_t j = 0; j < steps; ++j) {
                visits.clear();
                for (int i = 0; i < c.chains; ++i) {
                    const uint64_t gid = off + static_cast<uint64_t>(i);
                    if (j >= per + (gid < rem ? 1 : 0))
                        continue;
                    step(i, done + j * ctot + gid, visits);
                }
                adapt(visits);
            }
            done += span;
            if (done == next_refine) {
                refine();
                next_refine += c.m_refine;
            }
            if (done == next_metrics || done == budget) {
                flush(done);
                next_metrics = done + c.metrics_interval;
            }
        }
        if (out.metrics.empty() || static_cast<uint64_t>(out.metrics.back()[1]) != done)
            flush(done);
        s.counting = false;
        out.loop_s = out.metrics.empty() ? 0.0 : out.metrics.back()[0];

        // reduce (core/driver.cpp:315-340)
        double acc = 0.0;
        for (Chain &cc : ch) {
            acc += cc.acc;
            out.npert += cc.npert;
            out.nlarge += cc.nlarge;
        }
        out.done = done;
        out.mean_acc = out.npert > 0 ? acc / static_cast<double>(out.npert) : 0.0;
        for (Region &r : reg) {
            double ta = c.adapt_mode == 1 ? static_cast<double>(r.tot_fx) / 16777216.0 : r.tot_acc;
            out.tallies.push_back({ta, r.tot_vis});
        }
        // global_acceptance_identity (core/adaptation.cpp:103-125)
        {
            double tot = 0.0, comp = 0.0;
            uint64_t vis = 0;
            for (auto &t : out.tallies) {
                double y = t.first - comp;
                double sm = tot + y;
                comp = (sm - tot) - y;
                tot = sm;
                vis += t.second;
            }
            if (vis > 0) {
                double pooled = tot / static_cast<double>(vis);
                double w = 0.0;
                for (auto &t : out.tallies) {
                    if (t.second == 0)
                        continue;
                    double share = static_cast<double>(t.second) / static_cast<double>(vis);
                    w += share * (t.first / static_cast<double>(t.second));
                }
                out.identity = std::abs(pooled - w);
            }
        }
        out.regions = part.kind ? part.count() : reg.size();
        out.rays_c = s.rays_c;
        out.rays_v = s.rays_v;
    }
};


// ---- analytic-target adaptive MCMC (BASELINE.json configs[1]) -------------------------------
// Restates the GPU harness (include/ramlt_mix.h): run_chain_span's loop
// (core/driver.cpp:113-171) with a Gaussian random walk on [0,1]^D and a
// Gaussian-mixture target.  The target and the proposal have no reference
// implementation (pinned at the controller / accept boundary);
// everything else restates the reference: sigma_for (core/adaptation.cpp:44-50),
// normal_quantile (core/sampling.cpp:20-60), mh_accept (core/mutations.cpp:198-208),
// the accept draw (core/driver.cpp:168-171), record_acceptance / update_lambda
// (core/adaptation.cpp:10-20, 60-92), Grid2D::cell_of (core/partition.cpp:16-20),
// the chain / init streams (core/driver.cpp:20-21, 223-225).
struct MixTarget {
    int D = 0, K = 0;
    std::vector<double> W, mu, ell;   // W_k = L_k^{-1} (Sigma_k = L_k L_k^T), row-major D x D
};

static MixTarget mix_prepare(int D, int K, const double *w, const double *mu, const double *cov) {
    MixTarget t;
    t.D = D;
    t.K = K;
    t.W.assign(static_cast<size_t>(K) * D * D, 0.0);
    t.mu.assign(mu, mu + static_cast<size_t>(K) * D);
    t.ell.assign(K, 0.0);
    const double half_log_2pi = 0.5 * std::log(2.0 * 3.14159265358979323846);
    for (int k = 0; k < K; ++k) {
        if (!(w[k] > 0.0))
            throw std::invalid_argument("mix: component weights must be positive and finite");
        const double *S = cov + static_cast<size_t>(k) * D * D;
        std::vector<double> L(static_cast<size_t>(D) * D, 0.0);
        for (int i = 0; i < D; ++i)
            for (int j = 0; j <= i; ++j) {
                double s = S[i * D + j];
                for (int q = 0; q < j; ++q)
                    s = s - L[i * D + q] * L[j * D + q];
                if (i == j) {
                    if (!(s > 0.0))
                        throw std::invalid_argument("mix: covariance is not positive definite");
                    L[i * D + i] = std::sqrt(s);
                } else {
                    L[i * D + j] = s / L[j * D + j];
                }
            }
        double *Wk = t.W.data() + static_cast<size_t>(k) * D * D;
        for (int j = 0; j < D; ++j) {
            Wk[j * D + j] = 1.0 / L[j * D + j];
            for (int i = j + 1; i < D; ++i) {
                double s = 0.0;
                for (int q = j; q < i; ++q)
                    s = s + L[i * D + q] * Wk[q * D + j];
                Wk[i * D + j] = -s / L[i * D + i];
            }
        }
        double e = std::log(w[k]);
        for (int i = 0; i < D; ++i)
            e = e - std::log(L[i * D + i]);
        t.ell[k] = e - static_cast<double>(D) * half_log_2pi;
    }
    return t;
}

// log pi(x) = logsumexp_k (ell_k - |W_k (x - mu_k)|^2 / 2), fixed summation order.
static double mix_log_target(const MixTarget &t, const double *x) {
    const int D = t.D;
    double e[16];
    double m = -std::numeric_limits<double>::infinity();
    for (int k = 0; k < t.K; ++k) {
        const double *Wk = t.W.data() + static_cast<size_t>(k) * D * D;
        const double *mk = t.mu.data() + static_cast<size_t>(k) * D;
        double dif[16];
        for (int j = 0; j < D; ++j)
            dif[j] = x[j] - mk[j];
        double s = 0.0;
        for (int i = 0; i < D; ++i) {
            double z = 0.0;
            for (int j = 0; j <= i; ++j)
                z = z + Wk[i * D + j] * dif[j];
            s = s + z * z;
        }
        e[k] = t.ell[k] - 0.5 * s;
        m = e[k] > m ? e[k] : m;
    }
    double acc = 0.0;
    for (int k = 0; k < t.K; ++k)
        acc = acc + std::exp(e[k] - m);
    return m + std::log(acc);
}

struct MixRun {
    const oracle_mix_config &c;
    MixTarget t;
    Adapt ad;
    int C, D, nreg;
    long long Ctot, off;
    std::vector<double> x, lp, asum;
    std::vector<uint64_t> nacc;
    std::vector<Rng> rng;
    std::vector<Region> reg;
    std::vector<oracle_trace_row> trace;
    std::vector<double> log_a;
    std::vector<uint8_t> log_f;

    explicit MixRun(const oracle_mix_config &cfg) : c(cfg) {
        if (c.chains < 1)
            throw std::logic_error("need at least one chain");
        if (c.dim < 1 || c.dim > 16 || c.n_comp < 1 || c.n_comp > 16)
            throw std::invalid_argument("mix: bad target size");
        t = mix_prepare(c.dim, c.n_comp, c.weights, c.means, c.covariances);
        ad.L = c.batch_size;
        ad.gmax = c.gamma_max;
        ad.gscale = c.gamma_scale;
        ad.target = c.target_acceptance;
        ad.linit = c.lambda_init;
        ad.lmin = c.lambda_min;
        C = c.chains;
        D = c.dim;
        Ctot = c.chains_total > 0 ? c.chains_total : c.chains;
        off = c.chain_offset;
        nreg = c.strategy == 2 ? c.grid_n * c.grid_n : 1;
        reg.resize(nreg);
        for (Region &r : reg) {
            r.lambda = ad.linit;
            r.n = 1;
        }
        x.assign(static_cast<size_t>(C) * D, 0.0);
        lp.assign(C, 0.0);
        asum.assign(C, 0.0);
        nacc.assign(C, 0);
        rng.resize(C);
        log_a.assign(static_cast<size_t>(C) * c.log_steps, 0.0);
        log_f.assign(static_cast<size_t>(C) * c.log_steps, 0);
        for (int i = 0; i < C; ++i) {
            uint64_t g = static_cast<uint64_t>(off + i);
            Rng init;
            init.kind = c.rng;
            init.reseed(c.seed, STREAM_INIT + 2 * g);
            bool ok = false;
            for (int attempt = 0; attempt < 1000 && !ok; ++attempt) {
                for (int d = 0; d < D; ++d)
                    x[static_cast<size_t>(i) * D + d] = init.next_double();
                lp[i] = mix_log_target(t, &x[static_cast<size_t>(i) * D]);
                ok = std::isfinite(lp[i]);
            }
            if (!ok)
                throw std::runtime_error("mix: chain initialisation found no state with finite log density");
            rng[i].kind = c.rng;
            rng[i].reseed(c.seed, g);
        }
    }

    int region_of(const double *xi) const {
        if (c.strategy != 2)
            return 0;
        return grid_cell(c.grid_n, xi[0], xi[1]);
    }

    void update(Region &r, int rid, double ah, uint64_t index) {
        uint64_t n0 = r.n;
        r.lambda = lambda_next(r.lambda, ah, n0, ad);
        r.n = n0 + 1;
        trace.push_back({index, rid, n0, r.lambda, ah});
    }

    void run() {
        std::vector<int> vr(C);
        std::vector<double> va(C);
        std::vector<double> y(D);
        for (uint64_t j = 0; j < c.steps; ++j) {
            // every chain proposes with the lambda snapshot of the step start
            for (int i = 0; i < C; ++i) {
                double *xi = &x[static_cast<size_t>(i) * D];
                int r = region_of(xi);
                double lam = c.strategy == 0 ? ad.linit : reg[r].lambda;
                double sigma = std::exp(0.5 * lam);
                bool in = true;
                for (int d = 0; d < D; ++d) {
                    double u = rng[i].next_double();
                    y[d] = xi[d] + sigma * nquantile(u);
                    in = in && (y[d] >= 0.0 && y[d] <= 1.0);
                }
                double a = 0.0, lpy = 0.0;
                if (in) {
                    lpy = mix_log_target(t, y.data());
                    a = mh(1.0, std::exp(lpy - lp[i]), 1.0, 1.0, 1.0, 1.0);
                }
                bool acc = a > 0.0 && rng[i].next_double() < a;
                if (acc) {
                    for (int d = 0; d < D; ++d)
                        xi[d] = y[d];
                    lp[i] = lpy;
                }
                asum[i] += a;
                nacc[i] += acc ? 1 : 0;
                if (j < c.log_steps) {
                    log_a[static_cast<size_t>(i) * c.log_steps + j] = a;
                    log_f[static_cast<size_t>(i) * c.log_steps + j] = static_cast<uint8_t>((acc ? 1 : 0) | 2 | 4);
                }
                vr[i] = r;
                va[i] = a;
            }
            if (c.strategy == 0)
                continue;
            const uint64_t idx0 = j * static_cast<uint64_t>(Ctot) + static_cast<uint64_t>(off);
            if (c.adapt_mode == 0) {
                // literal: record_acceptance in chain order (core/adaptation.cpp:60-92)
                for (int i = 0; i < C; ++i) {
                    Region &R = reg[vr[i]];
                    R.tot_acc += va[i];
                    R.tot_vis += 1;
                    R.pend_sum += va[i];
                    R.pend_n += 1;
                    if (R.pend_n >= static_cast<uint64_t>(ad.L)) {
                        double ah = std::clamp(R.pend_sum / static_cast<double>(R.pend_n), 0.0, 1.0);
                        update(R, vr[i], ah, idx0 + i);
                        R.pend_sum = 0.0;
                        R.pend_n = 0;
                    }
                }
            } else {
                // pooled: one update per region from the step's pooled alpha-hat
                std::vector<uint64_t> cnt(nreg, 0), fx(nreg, 0), last(nreg, 0);
                for (int i = 0; i < C; ++i) {
                    cnt[vr[i]] += 1;
                    fx[vr[i]] += to_fx(va[i]);
                    last[vr[i]] = idx0 + i;
                }
                const size_t t0 = trace.size();
                for (int r = 0; r < nreg; ++r) {
                    if (!cnt[r])
                        continue;
                    Region &R = reg[r];
                    R.tot_vis += cnt[r];
                    R.tot_fx += fx[r];
                    R.pend_n += cnt[r];
                    R.pend_fx += fx[r];
                    if (R.pend_n < static_cast<uint64_t>(ad.L))
                        continue;
                    double ah = static_cast<double>(R.pend_fx) / 16777216.0 / static_cast<double>(R.pend_n);
                    ah = std::clamp(ah, 0.0, 1.0);
                    update(R, r, ah, last[r]);
                    R.pend_n = 0;
                    R.pend_fx = 0;
                }
                // canonical trace order: by the mutation index of the last visit
                std::stable_sort(trace.begin() + t0, trace.end(),
                                 [](const oracle_trace_row &p, const oracle_trace_row &q) {
                                     return p.mutation_index < q.mutation_index;
                                 });
            }
        }
    }
};

} // namespace orc

// ---- C ABI -----------------------------------------------------------------------
namespace {
void copy_err(char *err, int errlen, const char *msg) {
    if (!err || errlen <= 0)
        return;
    std::strncpy(err, msg, static_cast<size_t>(errlen) - 1);
    err[errlen - 1] = '\0';
}
} // namespace

extern "C" {

// Same contract as ref_render (oracle/ref_harness.cpp).
int oracle_render(const char *scene_text, const oracle_config *c, oracle_stats *st, oracle_log *lg,
                  oracle_outputs *out, char *err, int errlen) {
    try {
        orc::Scene s = orc::parse(scene_text);
        s.cam.configure(c->width, c->height);
        orc::Render r(s, *c, lg);
        r.run();
            r.dump_partition();
        const orc::Out &o = r.out;
        if (st) {
            std::memset(st, 0, sizeof(*st));
            st->b = o.b;
            st->b_stderr = o.b_se;
            st->b_samples = o.b_n;
            st->total_mutations = o.done;
            st->perturbation_proposals = o.npert;
            st->large_step_proposals = o.nlarge;
            st->mean_acceptance = o.mean_acc;
            st->film_luminance = o.film_lum;
            st->identity_residual = o.identity;
            st->region_count = o.regions;
            st->loop_time_s = o.loop_s;
            st->rays_closest = o.rays_c;
            st->rays_visibility = o.rays_v;
            st->n_tallies = o.tallies.size();
            st->n_trace = o.trace.size();
            st->n_metrics = o.metrics.size();
        }
        if (out) {
            double scale = o.done > 0 ? o.b / static_cast<double>(o.done) : 0.0;
            if (out->image)
                for (size_t i = 0; i < o.film.size(); ++i)
                    out->image[i] = static_cast<float>(o.film[i] * scale);
            if (out->film)
                std::memcpy(out->film, o.film.data(), o.film.size() * sizeof(double));
            for (size_t i = 0; i < o.tallies.size() && i < out->cap_tallies; ++i) {
                if (out->tally_accept)
                    out->tally_accept[i] = o.tallies[i].first;
                if (out->tally_visits)
                    out->tally_visits[i] = o.tallies[i].second;
            }
            for (size_t i = 0; i < o.trace.size() && i < out->cap_trace && out->trace; ++i)
                out->trace[i] = o.trace[i];
            if (out->dump && out->cap_dump > 0) {
                std::strncpy(out->dump, o.dump.c_str(), out->cap_dump - 1);
                out->dump[out->cap_dump - 1] = '\0';
            }
            for (size_t i = 0; i < o.metrics.size() && i < out->cap_metrics && out->metrics; ++i)
                for (int k = 0; k < 4; ++k)
                    out->metrics[i * 4 + k] = o.metrics[i][k];
        }
        if (lg) {
            size_t chains = static_cast<size_t>(c->chains);
            std::memset(lg->flags, 0, chains * lg->steps);
            for (size_t i = 0; i < chains * lg->steps; ++i)
                lg->a[i] = 0.0;
            for (size_t ci = 0; ci < chains; ++ci)
                for (size_t j = 0; j < r.logs[ci].size(); ++j) {
                    lg->a[ci * lg->steps + j] = r.logs[ci][j].first;
                    lg->flags[ci * lg->steps + j] = r.logs[ci][j].second;
                }
        }
        return 0;
    } catch (const std::invalid_argument &e) {
        copy_err(err, errlen, e.what());
        return 3;
    } catch (const std::logic_error &e) {
        copy_err(err, errlen, e.what());
        return 2;
    } catch (const std::runtime_error &e) {
        copy_err(err, errlen, e.what());
        return 1;
    } catch (const std::exception &e) {
        copy_err(err, errlen, e.what());
        return 4;
    }
}

// Per-substream b partial sums (sum, sum of squares) for substreams
// [begin, end): the sharded form of estimate_b used by multi-GPU runs.
int orc_b_partials(const char *scene_text, const oracle_config *c, uint64_t begin, uint64_t end,
                   double *out) {
    try {
        orc::Scene s = orc::parse(scene_text);
        s.cam.configure(c->width, c->height);
        uint64_t S = std::min<uint64_t>(c->b_samples, orc::B_SUBSTREAMS);
        for (uint64_t sub = begin; sub < end && sub < S; ++sub) {
            orc::Rng rng;
            rng.kind = c->rng;
            rng.reseed(c->seed, orc::STREAM_B + 2 * sub);
            double sum = 0.0, sq = 0.0;
            for (uint64_t j = sub; j < c->b_samples; j += S) {
                double v = orc::b_sample(s, rng, c->max_vertices);
                sum += v;
                sq += v * v;
            }
            out[2 * (sub - begin)] = sum;
            out[2 * (sub - begin) + 1] = sq;
        }
        return 0;
    } catch (...) {
        return 4;
    }
}

// Function-level exports mirroring the ref_* pins in ref_harness.cpp.
double orc_normal_quantile(double p) { return orc::nquantile(p); }
int orc_angular_pdf(double sigma, double theta, double *pdf, double *pdf_sa) {
    try {
        orc::Kern k(sigma);
        *pdf = k.pdf(theta);
        *pdf_sa = k.pdf_sa(theta);
        return 0;
    } catch (...) {
        return 3;
    }
}
int orc_angular_sample(double sigma, uint64_t seed, uint64_t stream, uint64_t n, double *out,
                       int rng_kind) {
    try {
        orc::Kern k(sigma);
        orc::Rng rng;
        rng.kind = rng_kind;
        rng.reseed(seed, stream);
        for (uint64_t i = 0; i < n; ++i)
            out[i] = k.sample(rng);
        return 0;
    } catch (...) {
        return 3;
    }
}
void orc_rng_u32(uint64_t seed, uint64_t stream, uint64_t n, uint32_t *out, int rng_kind) {
    orc::Rng rng;
    rng.kind = rng_kind;
    rng.reseed(seed, stream);
    for (uint64_t i = 0; i < n; ++i)
        out[i] = rng.next_u32();
}
void orc_philox_block(const uint32_t *ctr, const uint32_t *key, uint32_t *out) {
    orc::Rng::philox(ctr, key[0], key[1], out);
}
void orc_perturb_direction(const double *omega, double sigma, uint64_t seed, uint64_t stream,
                           uint64_t n, double *out) {
    orc::Kern k(sigma);
    orc::Rng rng;
    rng.reseed(seed, stream);
    orc::V3 w = {omega[0], omega[1], omega[2]};
    for (uint64_t i = 0; i < n; ++i) {
        orc::V3 r = orc::perturb_dir(w, k, rng);
        out[3 * i + 0] = r.x;
        out[3 * i + 1] = r.y;
        out[3 * i + 2] = r.z;
    }
}
void orc_cylindrical(const double *omega, double *uv) {
    orc::cyl({omega[0], omega[1], omega[2]}, &uv[0], &uv[1]);
}
double orc_update_lambda(double lambda, double ah, uint64_t n, double target, double lmin) {
    orc::Adapt a;
    a.target = target;
    a.lmin = lmin;
    return orc::lambda_next(lambda, ah, n, a);
}
int orc_grid_cell(int n, double u, double v) { return orc::grid_cell(n, u, v); }
double orc_mh_accept(double pc, double pp, double tf, double tr, double sf, double sr, int *status) {
    try {
        *status = 0;
        return orc::mh(pc, pp, tf, tr, sf, sr);
    } catch (...) {
        *status = 3;
        return 0.0;
    }
}
double orc_fresnel(double c, double ior) { return orc::fresnel(c, ior); }
int orc_camera(const double *cam, int w, int h, double u, double v, double *dir3, double *uv2,
               double *importance, double *dir_pdf) {
    try {
        orc::Cam c;
        c.init({cam[0], cam[1], cam[2]}, {cam[3], cam[4], cam[5]}, {cam[6], cam[7], cam[8]}, cam[9]);
        c.configure(w, h);
        orc::V3 d = c.primary(u, v);
        dir3[0] = d.x;
        dir3[1] = d.y;
        dir3[2] = d.z;
        double ru = -1.0, rv = -1.0;
        c.raster(d, &ru, &rv);
        uv2[0] = ru;
        uv2[1] = rv;
        *importance = c.importance(d);
        *dir_pdf = c.dir_pdf(d);
        return 0;
    } catch (...) {
        return 3;
    }
}

// Analytic-target harness (oracle_abi.h oracle_mix_config): 0 ok, else the
// ref_render status convention with err = what().
int oracle_mix_run(const oracle_mix_config *c, oracle_mix_out *o, char *err, int errlen) {
    try {
        orc::MixRun m(*c);
        m.run();
        const int C = m.C, D = m.D;
        if (o->x)
            std::memcpy(o->x, m.x.data(), sizeof(double) * static_cast<size_t>(C) * D);
        if (o->log_pi)
            std::memcpy(o->log_pi, m.lp.data(), sizeof(double) * C);
        if (o->log_a && c->log_steps)
            std::memcpy(o->log_a, m.log_a.data(), sizeof(double) * m.log_a.size());
        if (o->log_f && c->log_steps)
            std::memcpy(o->log_f, m.log_f.data(), m.log_f.size());
        o->n_regions = static_cast<uint64_t>(m.nreg);
        for (uint64_t r = 0; r < std::min<uint64_t>(o->cap_regions, m.nreg); ++r) {
            if (o->lambda)
                o->lambda[r] = m.reg[r].lambda;
            if (o->n)
                o->n[r] = m.reg[r].n;
            if (o->tally_accept)
                o->tally_accept[r] = c->adapt_mode == 0 ? m.reg[r].tot_acc
                                                        : static_cast<double>(m.reg[r].tot_fx) / 16777216.0;
            if (o->tally_visits)
                o->tally_visits[r] = m.reg[r].tot_vis;
        }
        o->n_trace = m.trace.size();
        for (uint64_t i = 0; i < std::min<uint64_t>(o->cap_trace, m.trace.size()); ++i)
            o->trace[i] = m.trace[i];
        o->accepted = 0;
        o->acceptance_sum = 0.0;
        for (int i = 0; i < C; ++i) {
            o->accepted += m.nacc[i];
            o->acceptance_sum += m.asum[i];
        }
        return 0;
    } catch (const std::invalid_argument &e) {
        copy_err(err, errlen, e.what());
        return 3;
    } catch (const std::logic_error &e) {
        copy_err(err, errlen, e.what());
        return 2;
    } catch (const std::runtime_error &e) {
        copy_err(err, errlen, e.what());
        return 1;
    } catch (const std::exception &e) {
        copy_err(err, errlen, e.what());
        return 4;
    }
}

} // extern "C"
