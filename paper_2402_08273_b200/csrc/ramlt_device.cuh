// ramlt_device.cuh -- device-side building blocks of the MLT chain step.
//
// Everything is templated on the arithmetic type R:
//   R = double : the parity build.  Compiled with -fmad=false; every expression
//                keeps the reference's evaluation order, so +,-,*,/,sqrt round
//                exactly as the reference's x86-64 SSE2 doubles do.  Only the
//                libm transcendentals (exp, log, erfc, atan2, sin, cos, pow)
//                differ from glibc by ulps.
//   R = float  : the production build (FMA contraction allowed).
// Reference citations: core/X:N = /root/reference/proj/src/core/X line N.
#pragma once

#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>

namespace rd {

constexpr int kMaxV = 24;              // compile-time path capacity (max_vertices <= kMaxV)
constexpr double kPiD = 3.14159265358979323846;
constexpr double kTwoPiD = 2.0 * 3.14159265358979323846;
constexpr double kInvPiD = 0.318309886183790671538;
constexpr double kEpsD = 1e-4;          // core/scene.hpp:13
constexpr uint64_t kStreamB = 0x4000000000000000ULL;     // core/driver.cpp:20
constexpr uint64_t kStreamInit = 0x4000000000000001ULL;  // core/driver.cpp:21

// ---- math traits --------------------------------------------------------------
template <class R> struct M;
template <> struct M<double> {
    static __device__ __forceinline__ double exp(double x) { return ::exp(x); }
    static __device__ __forceinline__ double log(double x) { return ::log(x); }
    static __device__ __forceinline__ double sqrt(double x) { return ::sqrt(x); }
    static __device__ __forceinline__ double erfc(double x) { return ::erfc(x); }
    static __device__ __forceinline__ double atan2(double y, double x) { return ::atan2(y, x); }
    static __device__ __forceinline__ double sin(double x) { return ::sin(x); }
    static __device__ __forceinline__ double cos(double x) { return ::cos(x); }
    static __device__ __forceinline__ double pow(double x, double y) { return ::pow(x, y); }
    static __device__ __forceinline__ double abs(double x) { return ::fabs(x); }
    static __device__ __forceinline__ double copysign(double x, double y) { return ::copysign(x, y); }
    static __device__ __forceinline__ double ldexp(double x, int e) { return ::ldexp(x, e); }
    static __device__ __forceinline__ bool finite(double x) { return ::isfinite(x); }
    static __device__ __forceinline__ bool isnan(double x) { return ::isnan(x); }
    static __device__ __forceinline__ double rcp(double x) { return 1.0 / x; }
    static __device__ __forceinline__ double fma(double a, double b, double c) { return ::fma(a, b, c); }
    static __device__ __forceinline__ double inf() { return __longlong_as_double(0x7ff0000000000000LL); }
};
template <> struct M<float> {
    static __device__ __forceinline__ float exp(float x) { return ::expf(x); }
    static __device__ __forceinline__ float log(float x) { return ::logf(x); }
    static __device__ __forceinline__ float sqrt(float x) { return ::sqrtf(x); }
    static __device__ __forceinline__ float erfc(float x) { return ::erfcf(x); }
    static __device__ __forceinline__ float atan2(float y, float x) { return ::atan2f(y, x); }
    static __device__ __forceinline__ float sin(float x) { return ::sinf(x); }
    static __device__ __forceinline__ float cos(float x) { return ::cosf(x); }
    static __device__ __forceinline__ float pow(float x, float y) { return ::powf(x, y); }
    static __device__ __forceinline__ float abs(float x) { return ::fabsf(x); }
    static __device__ __forceinline__ float copysign(float x, float y) { return ::copysignf(x, y); }
    static __device__ __forceinline__ float ldexp(float x, int e) { return ::ldexpf(x, e); }
    static __device__ __forceinline__ bool finite(float x) { return ::isfinite(x); }
    static __device__ __forceinline__ bool isnan(float x) { return ::isnan(x); }
    static __device__ __forceinline__ float rcp(float x) { return 1.0f / x; }
    static __device__ __forceinline__ float fma(float a, float b, float c) { return ::fmaf(a, b, c); }
    static __device__ __forceinline__ float inf() { return __int_as_float(0x7f800000); }
};

// ---- vectors (core/vec.hpp:9-53, same evaluation order) -----------------------
template <class R> struct V3 {
    R x, y, z;
};
template <class R> __device__ __forceinline__ V3<R> mk(R x, R y, R z) { return {x, y, z}; }
template <class R> __device__ __forceinline__ V3<R> add(V3<R> a, V3<R> b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
template <class R> __device__ __forceinline__ V3<R> sub(V3<R> a, V3<R> b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
template <class R> __device__ __forceinline__ V3<R> mul(V3<R> a, V3<R> b) { return {a.x * b.x, a.y * b.y, a.z * b.z}; }
template <class R> __device__ __forceinline__ V3<R> scl(V3<R> a, R s) { return {a.x * s, a.y * s, a.z * s}; }
template <class R> __device__ __forceinline__ V3<R> dvs(V3<R> a, R s) { return {a.x / s, a.y / s, a.z / s}; }
template <class R> __device__ __forceinline__ V3<R> neg(V3<R> a) { return {-a.x, -a.y, -a.z}; }
template <class R> __device__ __forceinline__ R dot(V3<R> a, V3<R> b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
template <class R> __device__ __forceinline__ V3<R> cross(V3<R> a, V3<R> b) {
    return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
template <class R> __device__ __forceinline__ R len(V3<R> a) { return M<R>::sqrt(dot(a, a)); }
template <class R> __device__ __forceinline__ V3<R> unit(V3<R> a) { return dvs(a, len(a)); }
template <class R> __device__ __forceinline__ V3<R> reflect(V3<R> w, V3<R> n) { return sub(scl(n, R(2) * dot(w, n)), w); }
template <class R> __device__ __forceinline__ R lum(V3<R> c) {
    return R(0.2126) * c.x + R(0.7152) * c.y + R(0.0722) * c.z;
}
template <class R> __device__ __forceinline__ bool zero3(V3<R> a) { return a.x == R(0) && a.y == R(0) && a.z == R(0); }

// ---- random sequences ------------------------------------------------------------
// RNG_PCG: core/rng.hpp:11-50 bit for bit (same seeds and streams as the
// reference driver, core/driver.cpp:223-225).
// RNG_PHILOX: Philox4x32-10, key = seed, counter = (block lo, block hi, stream
// lo, stream hi); next_u32 consumes one word of each 4-word block in order.
enum { RNG_PCG = 0, RNG_PHILOX = 1 };

template <int KIND> struct Rng;

template <> struct Rng<RNG_PCG> {
    uint64_t state, inc;
    __device__ __forceinline__ uint32_t next_u32() {
        uint64_t old = state;
        state = old * 6364136223846793005ULL + inc;
        uint32_t xs = static_cast<uint32_t>(((old >> 18u) ^ old) >> 27u);
        uint32_t rot = static_cast<uint32_t>(old >> 59u);
        return __funnelshift_r(xs, xs, rot);
    }
    __device__ __forceinline__ void reseed(uint64_t seed, uint64_t stream) {
        state = 0u;
        inc = (stream << 1u) | 1u;
        next_u32();
        state += seed;
        next_u32();
    }
};

__device__ __forceinline__ void philox10(uint32_t &c0, uint32_t &c1, uint32_t &c2, uint32_t &c3,
                                         uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
        uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        c0 = n0;
        c1 = lo1;
        c2 = n2;
        c3 = lo0;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
}

template <> struct Rng<RNG_PHILOX> {
    uint64_t key, stream, draw;
    uint32_t b0, b1, b2, b3;
    uint64_t bid;
    __device__ __forceinline__ void reseed(uint64_t seed, uint64_t strm) {
        key = seed;
        stream = strm;
        draw = 0;
        bid = ~0ULL;
    }
    // The 10-round block computation is out of line: the refill runs once per
    // four words.  (Passing the state by value instead, which lets the
    // coroutine state leave local memory, measured slower: c4 62 -> 52 M
    // mutations/s from register spills at the 64-register budget.)
    __device__ __noinline__ void refill(uint64_t b) {
        b0 = static_cast<uint32_t>(b);
        b1 = static_cast<uint32_t>(b >> 32);
        b2 = static_cast<uint32_t>(stream);
        b3 = static_cast<uint32_t>(stream >> 32);
        philox10(b0, b1, b2, b3, static_cast<uint32_t>(key), static_cast<uint32_t>(key >> 32));
        bid = b;
    }
    __device__ __forceinline__ uint32_t next_u32() {
        uint64_t b = draw >> 2;
        if (b != bid)
            refill(b);
        uint32_t w = draw & 3;
        ++draw;
        return w == 0 ? b0 : (w == 1 ? b1 : (w == 2 ? b2 : b3));
    }
};

// Uniform in [0,1): next_double (core/rng.hpp:32-40) for R = double; the same
// two words truncated to 24 bits for R = float (identical consumption).
// The Philox uniform draw is out of line: one copy per kernel instead of an
// expansion at each of the ~20 draw sites of the chain step (a smaller
// instruction footprint for the divergent coroutine; c4 +4 %).
#ifndef RAMLT_DRAW_INLINE
#define RAMLT_DRAW_INLINE __noinline__
#endif
// Philox: a uniform is always the word pair (2i, 2i+1) of one block when the
// draw counter is even (every draw in the hot path is a next_double), so one
// block check and one select replace two next_u32 expansions per draw site.
__device__ __forceinline__ bool philox_pair(Rng<RNG_PHILOX> &g, uint32_t &hi, uint32_t &lo) {
    if (g.draw & 1ull)
        return false;
    uint64_t b = g.draw >> 2;
    if (b != g.bid)
        g.refill(b);
    const bool second = (g.draw & 2ull) != 0;
    hi = second ? g.b2 : g.b0;
    lo = second ? g.b3 : g.b1;
    g.draw += 2;
    return true;
}

template <class R> struct Unit;
template <> struct Unit<double> {
    static __device__ RAMLT_DRAW_INLINE double draw(Rng<RNG_PHILOX> &g) {
        uint32_t h, l;
        if (!philox_pair(g, h, l)) {
            h = g.next_u32();
            l = g.next_u32();
        }
        return static_cast<double>(((static_cast<uint64_t>(h) << 32) | l) >> 11) * 0x1.0p-53;
    }
    template <class G> static __device__ __forceinline__ double draw(G &g) {
        uint64_t hi = g.next_u32();
        uint64_t lo = g.next_u32();
        return static_cast<double>(((hi << 32) | lo) >> 11) * 0x1.0p-53;
    }
};
template <> struct Unit<float> {
    static __device__ RAMLT_DRAW_INLINE float draw(Rng<RNG_PHILOX> &g) {
        uint32_t h, l;
        if (!philox_pair(g, h, l)) {
            h = g.next_u32();
            (void)g.next_u32();
        }
        return static_cast<float>(h >> 8) * 0x1.0p-24f;
    }
    template <class G> static __device__ __forceinline__ float draw(G &g) {
        uint32_t hi = g.next_u32();
        (void)g.next_u32();
        return static_cast<float>(hi >> 8) * 0x1.0p-24f;
    }
};

// ---- scene --------------------------------------------------------------------------
enum { MAT_DIFFUSE = 0, MAT_MIRROR = 1, MAT_DIELECTRIC = 2, MAT_GLOSSY = 3 };
enum { EV_NONE = 0, EV_REFLECT = 1, EV_TRANSMIT = 2 };

template <class R> struct TriD {   // a, e1 = b - a, e2 = c - a, n = normalize(cross(e1, e2))
    V3<R> a, e1, e2, n;
    int mat, emi;
    int orig;   // index in the scene's triangle order (BVH leaves are reordered)
    int pad_;
};

// ---- BVH record formats -------------------------------------------------------------
// One array of fixed-size units holds the whole BVH: internal nodes (one unit)
// and, in place of each leaf, its triangles' leaf-test records (TU units
// each).  The two children of a node are stored back to back at `base`:
// child 0 at base, child 1 right after it (1 unit for an internal node,
// cnt * TU units for a leaf of cnt triangles).  Traversal is bound by the
// L1 data pipe -- one wavefront per 32 B sector a lane touches (k_trace_bench:
// l1tex data-pipe wavefronts 93 % of peak, profiles/r02h) -- so records are
// sized in sectors: a quantised node is one 32 B sector (RAMLT_QNODE=1), a
// leaf triangle two (two 256-bit loads instead of three 16 B loads).
#ifndef RAMLT_QNODE
#define RAMLT_QNODE 0
#endif
// Leaf-test record: what Moeller-Trumbore reads plus the triangle's index in
// the scene (tie-break) and its position in the BVH-ordered TriD array (hit
// record: normal, material, emitter).  64 B in fp32, 128 B in fp64.
template <class R> struct alignas(sizeof(R) == 4 ? 64 : 128) TriT {
    R a[3], e1[3], e2[3];
    int orig, pos;
};
// Quantised node (RAMLT_QNODE=1): the children's boxes as 8-bit offsets on a
// per-axis power-of-two grid anchored at `org` (rounded outward at build
// time, so the decoded box contains the padded exact box).  32 B in fp32.
//   ex[k]: biased exponent of the grid step 2^(ex[k] - 127)
//   meta: cnt0 | cnt1 << 4 (0: internal child)
//   q: lo0 xyz, hi0 xyz, lo1 xyz, hi1 xyz
template <class R> struct alignas(sizeof(R) == 4 ? 32 : 64) QNode {
    R org[3];
    uint8_t ex[3], meta;
    uint8_t q[12];
    int32_t base;
};
// Plain node (RAMLT_QNODE=0): both children's boxes in R, same child rule.
template <class R> struct alignas(sizeof(R) == 4 ? 64 : 128) PNode {
    R lo0[3], hi0[3], lo1[3], hi1[3];
    int32_t base, meta;
};
template <class R> struct BvhFmt {
    using Node = typename std::conditional<RAMLT_QNODE != 0, QNode<R>, PNode<R>>::type;
    static constexpr int U = static_cast<int>(sizeof(Node));              // unit bytes
    static constexpr int TU = static_cast<int>(sizeof(TriT<R>)) / U;      // units per triangle
};
static_assert(sizeof(QNode<float>) == 32 && sizeof(TriT<float>) == 64, "fp32 records are 1 and 2 sectors");
static_assert(sizeof(TriT<double>) % sizeof(QNode<double>) == 0 && sizeof(TriT<double>) % sizeof(PNode<double>) == 0,
              "triangle records are whole units");
static_assert(sizeof(TriT<float>) % sizeof(PNode<float>) == 0, "triangle records are whole units");
template <class R> struct SphD {
    V3<R> c;
    R r;
    int mat, emi;
};
template <class R> struct MatD {
    int kind;
    V3<R> albedo;
    R ior, expo;
};
template <class R> struct CamD {   // core/camera.hpp:44-52 (basis computed on the host in fp64)
    V3<R> pos, right, up, fwd;
    R tanh, aspect, area, sensor;
};

template <class R> struct SceneView {
    const TriD<R> *tri;
    const SphD<R> *sph;
    const MatD<R> *mat;
    const V3<R> *emit;
    int ntri, nsph;
    CamD<R> cam;
    const unsigned char *bvh;   // BVH units (nodes + leaf triangles); null: brute force over smem-staged triangles
};

template <class R> struct Hit {
    V3<R> p, n;
    int mat, emi;
    R t;
};

// Cooperative lane groups: G lanes share one chain; G = 1 is one chain per
// thread.  G = 0 is the BVH instantiation: one chain per thread, triangles
// traversed through the BVH (a compile-time choice, so the brute-force kernels
// carry no traversal code or stack).
template <int G> struct Lanes {
    static constexpr int n = G == 0 ? 1 : G;
};
template <int G> struct Group {
    unsigned mask;
    int lane;
    __device__ __forceinline__ Group() {
        constexpr int N = Lanes<G>::n;
        int wl = threadIdx.x & 31;
        lane = wl & (N - 1);
        mask = N == 32 ? 0xffffffffu : (((1u << N) - 1u) << (wl & ~(N - 1)));
    }
};

// core/scene.cpp:15-29
template <class R>
__device__ __forceinline__ bool hit_sphere(const SphD<R> &s, V3<R> o, V3<R> d, R &t) {
    V3<R> oc = sub(o, s.c);
    R b = dot(oc, d);
    R c = dot(oc, oc) - s.r * s.r;
    R disc = b * b - c;
    if (disc < R(0))
        return false;
    R sq = M<R>::sqrt(disc);
    R tt = -b - sq;
    if (tt > R(kEpsD)) {
        t = tt;
        return true;
    }
    tt = -b + sq;
    if (tt > R(kEpsD)) {
        t = tt;
        return true;
    }
    return false;
}

// core/scene.cpp:31-52 (Moeller-Trumbore with the stored edges)
template <class R>
__device__ __forceinline__ bool hit_tri(const TriD<R> &tr, V3<R> o, V3<R> d, R &t) {
    V3<R> p = cross(d, tr.e2);
    R det = dot(tr.e1, p);
    if (M<R>::abs(det) < R(1e-14))
        return false;
    R inv = R(1) / det;
    V3<R> tv = sub(o, tr.a);
    R u = dot(tv, p) * inv;
    if (u < R(0) || u > R(1))
        return false;
    V3<R> q = cross(tv, tr.e1);
    R v = dot(d, q) * inv;
    if (v < R(0) || u + v > R(1))
        return false;
    R tt = dot(tr.e2, q) * inv;
    if (tt > R(kEpsD)) {
        t = tt;
        return true;
    }
    return false;
}

// Two triangles at a time for the brute-force scans: the determinant and u
// test of both are computed back to back (independent chains: ILP), the rest
// only when either passed -- the same operations and order per triangle as
// hit_tri, so the same results; a miss returns +inf.  The scans stay in index
// order with strict '<' (the linear scan's first minimum).
template <class R>
__device__ __forceinline__ void hit_tri2(const TriD<R> &ta, const TriD<R> &tb, V3<R> o, V3<R> d, R &xa, R &xb) {
    const V3<R> pa = cross(d, ta.e2), pb = cross(d, tb.e2);
    const R deta = dot(ta.e1, pa), detb = dot(tb.e1, pb);
    const R inva = R(1) / deta, invb = R(1) / detb;
    const V3<R> tva = sub(o, ta.a), tvb = sub(o, tb.a);
    const R ua = dot(tva, pa) * inva, ub = dot(tvb, pb) * invb;
    const bool oka = !(M<R>::abs(deta) < R(1e-14)) && !(ua < R(0) || ua > R(1));
    const bool okb = !(M<R>::abs(detb) < R(1e-14)) && !(ub < R(0) || ub > R(1));
    xa = xb = M<R>::inf();
    if (oka || okb) {
        const V3<R> qa = cross(tva, ta.e1), qb = cross(tvb, tb.e1);
        const R va = dot(d, qa) * inva, vb = dot(d, qb) * invb;
        const R tta = dot(ta.e2, qa) * inva, ttb = dot(tb.e2, qb) * invb;
        if (oka && !(va < R(0) || ua + va > R(1)) && tta > R(kEpsD))
            xa = tta;
        if (okb && !(vb < R(0) || ub + vb > R(1)) && ttb > R(kEpsD))
            xb = ttb;
    }
}

#ifndef RAMLT_SCAN2
#define RAMLT_SCAN2 1
#endif
// Closest hit over triangles first, first + step, ... < n (index order, strict '<').
template <class R>
__device__ __forceinline__ void scan_tris(const TriD<R> *tri, int first, int n, int step, V3<R> o, V3<R> d,
                                          R &best, int &bi, int base) {
    int j = first;
#if RAMLT_SCAN2
    for (; j + step < n; j += 2 * step) {
        R xa, xb;
        hit_tri2(tri[j], tri[j + step], o, d, xa, xb);
        if (xa < best) {
            best = xa;
            bi = base + j;
        }
        if (xb < best) {
            best = xb;
            bi = base + j + step;
        }
    }
#endif
    for (; j < n; j += step) {
        R t;
        if (hit_tri(tri[j], o, d, t) && t < best) {
            best = t;
            bi = base + j;
        }
    }
}

// Any triangle of first, first + step, ... < n with a root below lim.
template <class R>
__device__ __forceinline__ bool any_tri(const TriD<R> *tri, int first, int n, int step, V3<R> o, V3<R> d, R lim) {
    int j = first;
#if RAMLT_SCAN2
    for (; j + step < n; j += 2 * step) {
        R xa, xb;
        hit_tri2(tri[j], tri[j + step], o, d, xa, xb);
        if (xa < lim || xb < lim)
            return true;
    }
#endif
    for (; j < n; j += step) {
        R t;
        if (hit_tri(tri[j], o, d, t) && t < lim)
            return true;
    }
    return false;
}

// ---- BVH record loads -------------------------------------------------------------------
// sm_100 256-bit loads (LDG.E.ENL2.256): one 32 B sector per request.
__device__ __forceinline__ void ldg256(const void *p, float4 &a, float4 &b) {
    asm("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w), "=f"(b.x), "=f"(b.y), "=f"(b.z), "=f"(b.w)
        : "l"(p));
}

// Leaf-test record of the triangle at BVH unit address p (two sectors in fp32).
template <class R> __device__ __forceinline__ TriT<R> ld_trit(const unsigned char *p) {
    return *reinterpret_cast<const TriT<R> *>(p);
}
template <> __device__ __forceinline__ TriT<float> ld_trit<float>(const unsigned char *p) {
    float4 a, b;
    ldg256(p, a, b);
    const float4 c = __ldg(reinterpret_cast<const float4 *>(p + 32));
    TriT<float> t;
    t.a[0] = a.x, t.a[1] = a.y, t.a[2] = a.z, t.e1[0] = a.w;
    t.e1[1] = b.x, t.e1[2] = b.y, t.e2[0] = b.z, t.e2[1] = b.w;
    t.e2[2] = c.x;
    t.orig = __float_as_int(c.y);
    t.pos = __float_as_int(c.z);
    return t;
}

// Moeller-Trumbore on the compact record: identical arithmetic to hit_tri.
template <class R>
__device__ __forceinline__ bool hit_tri_t(const TriT<R> &tr, V3<R> o, V3<R> d, R &t) {
    const V3<R> a = mk(tr.a[0], tr.a[1], tr.a[2]);
    const V3<R> e1 = mk(tr.e1[0], tr.e1[1], tr.e1[2]);
    const V3<R> e2 = mk(tr.e2[0], tr.e2[1], tr.e2[2]);
    V3<R> p = cross(d, e2);
    R det = dot(e1, p);
    if (M<R>::abs(det) < R(1e-14))
        return false;
    R inv = R(1) / det;
    V3<R> tv = sub(o, a);
    R u = dot(tv, p) * inv;
    if (u < R(0) || u > R(1))
        return false;
    V3<R> q = cross(tv, e1);
    R v = dot(d, q) * inv;
    if (v < R(0) || u + v > R(1))
        return false;
    R tt = dot(e2, q) * inv;
    if (tt > R(kEpsD)) {
        t = tt;
        return true;
    }
    return false;
}

// ---- BVH traversal ------------------------------------------------------------------
// The result equals the reference's linear scan (core/scene.cpp:57-92): the
// winner is the lexicographic minimum of (t, original primitive index) over all
// hits below `lim`, and padded boxes plus a relative slack on the slab test
// never cull a primitive the exact test accepts.
template <class R> struct Slack;
template <> struct Slack<float> {
    static __device__ __forceinline__ float v() { return 1.0f + 2e-6f; }
};
template <> struct Slack<double> {
    static __device__ __forceinline__ double v() { return 1.0 + 1e-13; }
};

// Slab test on the six plane parameters of one box.
template <class R>
__device__ __forceinline__ bool slab_t(R tx0, R tx1, R ty0, R ty1, R tz0, R tz1, R tcap, R &tnear) {
    R tmin = fmax(fmax(fmin(tx0, tx1), fmin(ty0, ty1)), fmin(tz0, tz1));
    R tmax = fmin(fmin(fmax(tx0, tx1), fmax(ty0, ty1)), fmax(tz0, tz1));
    tmax = tmax * Slack<R>::v();
    tnear = tmin;
    return tmax >= tmin && tmax >= R(0) && tmin <= tcap * Slack<R>::v();
}

template <class R> __device__ __forceinline__ V3<R> safe_inv(V3<R> d) {
    const R tiny = sizeof(R) == 8 ? R(1e-300) : R(1e-30);
    R x = M<R>::abs(d.x) < tiny ? M<R>::copysign(tiny, d.x) : d.x;
    R y = M<R>::abs(d.y) < tiny ? M<R>::copysign(tiny, d.y) : d.y;
    R z = M<R>::abs(d.z) < tiny ? M<R>::copysign(tiny, d.z) : d.z;
    return mk(R(1) / x, R(1) / y, R(1) / z);
}

// Child references: >= 0 internal node (unit index), < 0 leaf ~((unit << 4) | cnt).
__device__ __forceinline__ void child_refs(int base, unsigned meta, int tu, int &c0, int &c1) {
    const int n0 = static_cast<int>(meta & 15u), n1 = static_cast<int>((meta >> 4) & 15u);
    const int b1 = base + (n0 ? n0 * tu : 1);
    c0 = n0 ? ~((base << 4) | n0) : base;
    c1 = n1 ? ~((b1 << 4) | n1) : b1;
}

template <class R> struct NodeHit {
    R t0, t1;
    int c0, c1;
    bool h0, h1;
};

// Quantised planes: plane = org + q * 2^e, so t = (plane - o) / d = q * A + B
// with A = 2^e * inv (exact: a power-of-two scaling) and B = org * inv - o * inv
// (one FMA per axis and node), then one FMA per plane as for unquantised boxes.
__device__ __forceinline__ float qbyte(unsigned w, unsigned i) {
    // 2^23 + byte as a float bit pattern (one PRMT), minus 2^23: exact
    return __uint_as_float(__byte_perm(w, 0x4B000000u, 0x7540u | i)) - 8388608.0f;
}

template <class R>
__device__ __forceinline__ NodeHit<R> visit_node(const unsigned char *__restrict__ bvh, int node, V3<R> inv,
                                                 V3<R> oinv, R tcap) {
    NodeHit<R> r;
    if constexpr (RAMLT_QNODE != 0) {
        const QNode<R> n = *reinterpret_cast<const QNode<R> *>(bvh + static_cast<size_t>(node) * BvhFmt<R>::U);
        auto scale = [](uint8_t e) {
            return sizeof(R) == 4 ? R(__uint_as_float(static_cast<unsigned>(e) << 23))
                                  : R(__longlong_as_double(static_cast<long long>(e - 127 + 1023) << 52));
        };
        const V3<R> A = mk(scale(n.ex[0]) * inv.x, scale(n.ex[1]) * inv.y, scale(n.ex[2]) * inv.z);
        const V3<R> B = mk(M<R>::fma(n.org[0], inv.x, -oinv.x), M<R>::fma(n.org[1], inv.y, -oinv.y),
                           M<R>::fma(n.org[2], inv.z, -oinv.z));
        R t[12];
#pragma unroll
        for (int k = 0; k < 12; ++k) {
            const int ax = k % 3;
            t[k] = M<R>::fma(R(n.q[k]), ax == 0 ? A.x : (ax == 1 ? A.y : A.z), ax == 0 ? B.x : (ax == 1 ? B.y : B.z));
        }
        r.h0 = slab_t(t[0], t[3], t[1], t[4], t[2], t[5], tcap, r.t0);
        r.h1 = slab_t(t[6], t[9], t[7], t[10], t[8], t[11], tcap, r.t1);
        child_refs(n.base, n.meta, BvhFmt<R>::TU, r.c0, r.c1);
    } else {
        const PNode<R> n = *reinterpret_cast<const PNode<R> *>(bvh + static_cast<size_t>(node) * BvhFmt<R>::U);
        r.h0 = slab_t(M<R>::fma(n.lo0[0], inv.x, -oinv.x), M<R>::fma(n.hi0[0], inv.x, -oinv.x),
                      M<R>::fma(n.lo0[1], inv.y, -oinv.y), M<R>::fma(n.hi0[1], inv.y, -oinv.y),
                      M<R>::fma(n.lo0[2], inv.z, -oinv.z), M<R>::fma(n.hi0[2], inv.z, -oinv.z), tcap, r.t0);
        r.h1 = slab_t(M<R>::fma(n.lo1[0], inv.x, -oinv.x), M<R>::fma(n.hi1[0], inv.x, -oinv.x),
                      M<R>::fma(n.lo1[1], inv.y, -oinv.y), M<R>::fma(n.hi1[1], inv.y, -oinv.y),
                      M<R>::fma(n.lo1[2], inv.z, -oinv.z), M<R>::fma(n.hi1[2], inv.z, -oinv.z), tcap, r.t1);
        child_refs(n.base, static_cast<unsigned>(n.meta), BvhFmt<R>::TU, r.c0, r.c1);
    }
    return r;
}

// fp32: one 256-bit load per node (quantised) or two (plain).
template <>
__device__ __forceinline__ NodeHit<float> visit_node<float>(const unsigned char *__restrict__ bvh, int node,
                                                            V3<float> inv, V3<float> oinv, float tcap) {
    NodeHit<float> r;
    const unsigned char *p = bvh + static_cast<size_t>(node) * BvhFmt<float>::U;
    float4 a, b;
    ldg256(p, a, b);
#if RAMLT_QNODE
    // a = org xyz, (ex0 ex1 ex2 meta); b = q[0..3], q[4..7], q[8..11], base
    const unsigned w3 = __float_as_uint(a.w), w4 = __float_as_uint(b.x), w5 = __float_as_uint(b.y),
                   w6 = __float_as_uint(b.z);
    const float Ax = __uint_as_float((w3 & 0xFFu) << 23) * inv.x;
    const float Ay = __uint_as_float(((w3 >> 8) & 0xFFu) << 23) * inv.y;
    const float Az = __uint_as_float(((w3 >> 16) & 0xFFu) << 23) * inv.z;
    const float Bx = fmaf(a.x, inv.x, -oinv.x), By = fmaf(a.y, inv.y, -oinv.y), Bz = fmaf(a.z, inv.z, -oinv.z);
    r.h0 = slab_t(fmaf(qbyte(w4, 0), Ax, Bx), fmaf(qbyte(w4, 3), Ax, Bx), fmaf(qbyte(w4, 1), Ay, By),
                  fmaf(qbyte(w5, 0), Ay, By), fmaf(qbyte(w4, 2), Az, Bz), fmaf(qbyte(w5, 1), Az, Bz), tcap, r.t0);
    r.h1 = slab_t(fmaf(qbyte(w5, 2), Ax, Bx), fmaf(qbyte(w6, 1), Ax, Bx), fmaf(qbyte(w5, 3), Ay, By),
                  fmaf(qbyte(w6, 2), Ay, By), fmaf(qbyte(w6, 0), Az, Bz), fmaf(qbyte(w6, 3), Az, Bz), tcap, r.t1);
    child_refs(__float_as_int(b.w), w3 >> 24, BvhFmt<float>::TU, r.c0, r.c1);
#else
    float4 c, e;
    ldg256(p + 32, c, e);
    // lo0 xyz hi0 x | hi0 yz lo1 xy | lo1 z hi1 xyz | base meta
    r.h0 = slab_t(fmaf(a.x, inv.x, -oinv.x), fmaf(a.w, inv.x, -oinv.x), fmaf(a.y, inv.y, -oinv.y),
                  fmaf(b.x, inv.y, -oinv.y), fmaf(a.z, inv.z, -oinv.z), fmaf(b.y, inv.z, -oinv.z), tcap, r.t0);
    r.h1 = slab_t(fmaf(b.z, inv.x, -oinv.x), fmaf(c.y, inv.x, -oinv.x), fmaf(b.w, inv.y, -oinv.y),
                  fmaf(c.z, inv.y, -oinv.y), fmaf(c.x, inv.z, -oinv.z), fmaf(c.w, inv.z, -oinv.z), tcap, r.t1);
    child_refs(__float_as_int(e.x), __float_as_uint(e.y), BvhFmt<float>::TU, r.c0, r.c1);
#endif
    return r;
}

// Triangle record k of the leaf that starts at unit `first`.
template <class R> __device__ __forceinline__ const unsigned char *leaf_tri(const unsigned char *bvh, int first, int k) {
    return bvh + static_cast<size_t>(first + k * BvhFmt<R>::TU) * BvhFmt<R>::U;
}

// BVH2 traversal state of one ray for the coroutine kernel (bvh_trace below is
// the run-to-completion form used by the megakernel); same visit order, so
// the same hits.
//
// `step` runs one "while-while" round (Aila & Laine 2009): descend internal
// nodes until every still-traversing lane of the warp holds a leaf (one leaf
// postponed per lane), then test the leaves with the lanes converged.  It
// returns true when the ray is done.  The coroutine kernel interleaves rounds
// with handing finished lanes a new ray (dynamic ray fetch) instead of idling
// them until the warp's longest traversal ends.
template <class R> struct BvhTrav {
    static constexpr int DONE = 0x7fffffff;
    static constexpr int STACK = 64;   // BVH2 depth <= 62 (checked at build)
    V3<R> o, d, inv, oinv;
    R best;
    int key, pos, spos, node, leaf, sp;
    bool any;
    // The lane's stack: the first SSTACK entries in shared memory at stride
    // 128 (one bank per lane: conflict-free whatever each lane's depth), the
    // rest in local memory.  Scattered per-lane depths made a local-only stack
    // the top L1 miss / long-scoreboard stall.
#ifndef RAMLT_SSTACK
#define RAMLT_SSTACK 16
#endif
    static constexpr int SSTACK = RAMLT_SSTACK;
    int *ss;    // shared: entry i at ss[i * 128]
    int *sl;    // local: entry i >= SSTACK at sl[i - SSTACK]

    __device__ __forceinline__ void push(int v) {
        if (sp < SSTACK)
            ss[sp * 128] = v;
        else
            sl[sp - SSTACK] = v;
        ++sp;
    }

    // Spheres first (linear scan, strict '<'), then the BVH below `best`.
    __device__ __forceinline__ void begin(const SceneView<R> &s, V3<R> o_, V3<R> d_, R lim, bool any_hit) {
        o = o_;
        d = d_;
        any = any_hit;
        best = lim;
        key = -1;   // no winner yet: a hit at exactly t == lim loses the tie (reference: visible iff t >= dist - eps)
        spos = -1;
        pos = -1;
        for (int i = 0; i < s.nsph; ++i) {
            R t;
            if (hit_sphere(s.sph[i], o, d, t) && t < best) {
                best = t;
                key = i;
                spos = i;
            }
        }
        inv = safe_inv(d);
        oinv = mul(o, inv);
        sp = 0;
        leaf = 0;
        node = (any && spos >= 0) ? DONE : 0;
    }

    __device__ __forceinline__ int pop() {
        if (sp == 0)
            return DONE;
        --sp;
        return sp < SSTACK ? ss[sp * 128] : sl[sp - SSTACK];
    }

    // The BVH base is passed from the kernel parameters (constant bank) rather
    // than read through a SceneView the register allocator may have spilled:
    // that reload sat on every node fetch's dependency chain.
    __device__ __forceinline__ bool step(const SceneView<R> &s) { return step(s.bvh, s.nsph); }
    __device__ __forceinline__ bool step(const unsigned char *__restrict__ bvh, int nsph) {
        while (node >= 0 && node != DONE) {
            const NodeHit<R> n = visit_node<R>(bvh, node, inv, oinv, best);
            if (n.h0 && n.h1) {
                bool near0 = n.t0 <= n.t1;
                push(near0 ? n.c1 : n.c0);
                node = near0 ? n.c0 : n.c1;
            } else if (n.h0) {
                node = n.c0;
            } else if (n.h1) {
                node = n.c1;
            } else {
                node = pop();
            }
            if (node < 0) {   // reached a leaf
                if (leaf != 0)
                    break;    // slot busy: test the postponed leaf first
                leaf = node;
                node = pop();
            }
            if (__all_sync(__activemask(), leaf != 0))
                break;
        }
        while (leaf < 0) {
            int code = ~leaf;
            int first = code >> 4, cnt = code & 15;
            for (int k = 0; k < cnt; ++k) {
                const TriT<R> tr = ld_trit<R>(leaf_tri<R>(bvh, first, k));
                R t;
                if (!hit_tri_t(tr, o, d, t))
                    continue;
                int kk = nsph + tr.orig;
                if (t < best || (t == best && kk < key)) {
                    best = t;
                    key = kk;
                    pos = tr.pos;
                    if (any) {
                        node = DONE;
                        leaf = 0;
                        return true;
                    }
                }
            }
            leaf = 0;
            if (node < 0) {   // the next popped entry was a leaf too
                leaf = node;
                node = pop();
            }
        }
        return node == DONE;
    }

    // Hit primitive index (spheres first, triangles by BVH position) or -1.
    __device__ __forceinline__ int prim(const SceneView<R> &s) const {
        return pos >= 0 ? s.nsph + pos : spos;
    }
};

// Returns the winner's position in s.tri (BVH order) or -1; `key` carries the
// combined original index (spheres first) used for ties.  With any_hit, stops
// at the first primitive below lim (visibility).
//
// "While-while" traversal with one postponed leaf (Aila & Laine 2009): lanes
// descend internal nodes until every still-traversing lane holds a leaf, then
// all of them test their leaf's triangles together, so the slab tests and the
// triangle tests each run with the warp's lanes converged.  Every box that
// overlaps [0, best] is still visited, so the result is exactly the linear
// scan's.
template <class R>
__device__ int bvh_trace(const SceneView<R> &s, V3<R> o, V3<R> d, R lim, R &best, int &key, bool any_hit) {
    constexpr int DONE = 0x7fffffff;
    V3<R> inv = safe_inv(d);
    V3<R> oinv = mul(o, inv);
    (void)lim;
    int pos = -1;
    int stack[64];
    int sp = 0;
    int node = 0;    // >= 0 internal node, < 0 leaf code, DONE
    int leaf = 0;    // postponed leaf code (< 0) or 0
    for (;;) {
        while (node >= 0 && node != DONE) {
            const NodeHit<R> n = visit_node<R>(s.bvh, node, inv, oinv, best);
            if (n.h0 && n.h1) {
                bool near0 = n.t0 <= n.t1;
                stack[sp++] = near0 ? n.c1 : n.c0;
                node = near0 ? n.c0 : n.c1;
            } else if (n.h0) {
                node = n.c0;
            } else if (n.h1) {
                node = n.c1;
            } else {
                node = sp ? stack[--sp] : DONE;
            }
            if (node < 0) {   // reached a leaf
                if (leaf != 0)
                    break;    // slot busy: test the postponed leaf first
                leaf = node;
                node = sp ? stack[--sp] : DONE;
            }
            if (__all_sync(__activemask(), leaf != 0))
                break;
        }
        while (leaf < 0) {
            int code = ~leaf;
            int first = code >> 4, cnt = code & 15;
            for (int k = 0; k < cnt; ++k) {
                const TriT<R> tr = ld_trit<R>(leaf_tri<R>(s.bvh, first, k));
                R t;
                if (!hit_tri_t(tr, o, d, t))
                    continue;
                int kk = s.nsph + tr.orig;
                if (t < best || (t == best && kk < key)) {
                    best = t;
                    key = kk;
                    pos = tr.pos;
                    if (any_hit)
                        return pos;
                }
            }
            leaf = 0;
            if (node < 0) {   // the next popped entry was a leaf too
                leaf = node;
                node = sp ? stack[--sp] : DONE;
            }
        }
        if (node == DONE)
            break;
    }
    return pos;
}

// Closest hit (core/scene.cpp:57-92).  Primitive order = spheres then
// triangles; each lane scans its stride-G subset in increasing order with
// strict '<', and the (t, index) lexicographic minimum across lanes is the
// reference's first-minimum winner.
template <class R, int G>
__device__ __forceinline__ bool intersect(const SceneView<R> &s, V3<R> o, V3<R> d, Hit<R> &h,
                                          const Group<G> &g) {
    if constexpr (G == 0) {
        // every lane of a group traverses the same ray: identical results, no reduction
        R best = M<R>::inf();
        int key = -1, spos = -1;
        for (int i = 0; i < s.nsph; ++i) {
            R t;
            if (hit_sphere(s.sph[i], o, d, t) && t < best) {
                best = t;
                key = i;
                spos = i;
            }
        }
        int tpos = bvh_trace(s, o, d, best, best, key, false);
        if (tpos < 0 && spos < 0)
            return false;
        h.t = best;
        h.p = add(o, scl(d, best));
        if (tpos < 0) {
            const SphD<R> &sp = s.sph[spos];
            h.n = unit(sub(h.p, sp.c));
            h.mat = sp.mat;
            h.emi = sp.emi;
        } else {
            const TriD<R> &tr = s.tri[tpos];
            h.n = tr.n;
            h.mat = tr.mat;
            h.emi = tr.emi;
        }
        return true;
    } else {
    R best = M<R>::inf();
    int bi = 0x7fffffff;
    for (int i = g.lane; i < s.nsph; i += G) {
        R t;
        if (hit_sphere(s.sph[i], o, d, t) && t < best) {
            best = t;
            bi = i;
        }
    }
    scan_tris(s.tri, g.lane, s.ntri, G, o, d, best, bi, s.nsph);
    if (G > 1) {
#pragma unroll
        for (int off = G / 2; off > 0; off >>= 1) {
            R ot = __shfl_xor_sync(g.mask, best, off, G);
            int oi = __shfl_xor_sync(g.mask, bi, off, G);
            if (ot < best || (ot == best && oi < bi)) {
                best = ot;
                bi = oi;
            }
        }
    }
    if (bi == 0x7fffffff)
        return false;
    h.t = best;
    h.p = add(o, scl(d, best));
    if (bi < s.nsph) {
        const SphD<R> &sp = s.sph[bi];
        h.n = unit(sub(h.p, sp.c));
        h.mat = sp.mat;
        h.emi = sp.emi;
    } else {
        const TriD<R> &tr = s.tri[bi - s.nsph];
        h.n = tr.n;
        h.mat = tr.mat;
        h.emi = tr.emi;
    }
    return true;
    }
}

// visible (core/scene.cpp:94-102) as an any-hit query: the reference's
// "closest t >= dist - eps" is "no primitive's first root lies in (eps, dist - eps)".
template <class R, int G>
__device__ __forceinline__ bool visible(const SceneView<R> &s, V3<R> a, V3<R> b, const Group<G> &g) {
    V3<R> d = sub(b, a);
    R dist = len(d);
    if (dist <= R(2) * R(kEpsD))
        return false;
    d = dvs(d, dist);
    R lim = dist - R(kEpsD);
    bool occ = false;
    if constexpr (G == 0) {
        for (int i = 0; i < s.nsph && !occ; ++i) {
            R t;
            if (hit_sphere(s.sph[i], a, d, t) && t < lim)
                occ = true;
        }
        if (!occ) {
            R best = lim;
            int key = -1;   // strict t < lim occludes, as the brute-force scan
            occ = bvh_trace(s, a, d, lim, best, key, true) >= 0;
        }
        return !occ;
    } else {
    for (int i = g.lane; i < s.nsph && !occ; i += G) {
        R t;
        if (hit_sphere(s.sph[i], a, d, t) && t < lim)
            occ = true;
    }
    if (!occ)
        occ = any_tri(s.tri, g.lane, s.ntri, G, a, d, lim);
    if (G > 1)
        occ = __any_sync(g.mask, occ);
    return !occ;
    }
}

// ---- camera (core/camera.cpp:32-64) ---------------------------------------------------
template <class R> __device__ __forceinline__ V3<R> cam_primary(const CamD<R> &c, R u, R v) {
    R px = (R(2) * u - R(1)) * c.tanh * c.aspect;
    R py = (R(2) * v - R(1)) * c.tanh;
    return unit(add(add(scl(c.right, px), scl(c.up, py)), c.fwd));
}
template <class R> __device__ __forceinline__ bool cam_raster(const CamD<R> &c, V3<R> w, R &u, R &v) {
    R ct = dot(w, c.fwd);
    if (ct <= R(0))
        return false;
    R px = dot(w, c.right) / ct;
    R py = dot(w, c.up) / ct;
    R uu = R(0.5) * (px / (c.tanh * c.aspect) + R(1));
    R vv = R(0.5) * (py / c.tanh + R(1));
    if (uu < R(0) || uu > R(1) || vv < R(0) || vv > R(1))
        return false;
    u = uu;
    v = vv;
    return true;
}
template <class R> __device__ __forceinline__ R cam_importance(const CamD<R> &c, V3<R> w) {
    R u, v;
    if (!cam_raster(c, w, u, v))
        return R(0);
    R ct = dot(w, c.fwd);
    R c2 = ct * ct;
    return c.sensor / (c2 * c2);
}
template <class R> __device__ __forceinline__ R cam_dir_pdf(const CamD<R> &c, V3<R> w) {
    R u, v;
    if (!cam_raster(c, w, u, v))
        return R(0);
    R ct = dot(w, c.fwd);
    return R(1) / (c.area * ct * ct * ct);
}

// ---- sampling core (core/sampling.cpp) -------------------------------------------------
template <class R> __device__ __forceinline__ R npdf(R x) {
    return M<R>::exp(R(-0.5) * x * x) / M<R>::sqrt(R(kTwoPiD));
}
template <class R> __device__ __forceinline__ R ncdf(R x) {
    return R(0.5) * M<R>::erfc(-x / R(1.41421356237309504880));
}

// Acklam + one Halley step (core/sampling.cpp:19-60).
template <class R> __device__ __forceinline__ R nquantile(R p) {
    const R a0 = R(-3.969683028665376e+01), a1 = R(2.209460984245205e+02),
            a2 = R(-2.759285104469687e+02), a3 = R(1.383577518672690e+02),
            a4 = R(-3.066479806614716e+01), a5 = R(2.506628277459239e+00);
    const R b0 = R(-5.447609879822406e+01), b1 = R(1.615858368580409e+02),
            b2 = R(-1.556989798598866e+02), b3 = R(6.680131188771972e+01),
            b4 = R(-1.328068155288572e+01);
    const R c0 = R(-7.784894002430293e-03), c1 = R(-3.223964580411365e-01),
            c2 = R(-2.400758277161838e+00), c3 = R(-2.549732539343734e+00),
            c4 = R(4.374664141464968e+00), c5 = R(2.938163982698783e+00);
    const R d0 = R(7.784695709041462e-03), d1 = R(3.224671290700398e-01),
            d2 = R(2.445134137142996e+00), d3 = R(3.754408661907416e+00);
    // Branch-free over the three regions (warps almost always hold lanes of
    // more than one): select the region's coefficients and evaluate one
    // rational function.  Same operations in the same order as the branchy
    // form (the tail denominator's missing leading term enters as 0 * t + d0
    // = d0, the tail numerator's sign as an exact +-1 factor), so fp64 results
    // are bit-identical to it.
    const bool lo = p < R(0.02425), hi = p > R(1) - R(0.02425), mid = !lo && !hi;
    const R qc = p - R(0.5);
    const R qt = M<R>::sqrt(R(-2) * M<R>::log(hi ? R(1) - p : p));
    const R t = mid ? qc * qc : qt;
    const R n = (((((mid ? a0 : c0) * t + (mid ? a1 : c1)) * t + (mid ? a2 : c2)) * t + (mid ? a3 : c3)) * t +
                 (mid ? a4 : c4)) * t + (mid ? a5 : c5);
    const R d = (((((mid ? b0 : R(0)) * t + (mid ? b1 : d0)) * t + (mid ? b2 : d1)) * t + (mid ? b3 : d2)) * t +
                 (mid ? b4 : d3)) * t + R(1);
    R x = n * (mid ? qc : (hi ? R(-1) : R(1))) / d;
    if (sizeof(R) == 8) {   // the Halley refinement only pays at fp64 precision
        R e = ncdf(x) - p;
        R u = e * M<R>::sqrt(R(kTwoPiD)) * M<R>::exp(R(0.5) * x * x);
        x = x - u / (R(1) + R(0.5) * x * u);
    }
    return x;
}

// Truncated normal on [-pi, pi] (core/sampling.cpp:62-92).  The (sigma,
// cdf_lo, mass) triple is a pure function of sigma; the engine caches it per
// region (KernTab) so a proposal never re-evaluates erfc.
template <class R> struct Kern {
    R sigma, lo, mass;
};
template <class R> __device__ __forceinline__ Kern<R> make_kern(R sigma) {
    Kern<R> k;
    k.sigma = sigma;
    R t = R(kPiD) / sigma;
    k.lo = ncdf(-t);
    k.mass = ncdf(t) - k.lo;
    return k;
}
template <class R, class G> __device__ __forceinline__ R kern_sample(const Kern<R> &k, G &rng) {
    R u = Unit<R>::draw(rng);
    R p = k.lo + u * k.mass;
    if (p <= R(0))
        return R(-kPiD);
    if (p >= R(1))
        return R(kPiD);
    R th = k.sigma * nquantile(p);
    return th < R(-kPiD) ? R(-kPiD) : (th > R(kPiD) ? R(kPiD) : th);
}
template <class R> __device__ __forceinline__ R kern_pdf(const Kern<R> &k, R th) {
    if (M<R>::abs(th) > R(kPiD))
        return R(0);
    return npdf(th / k.sigma) / (k.sigma * k.mass);
}
template <class R> __device__ __forceinline__ R kern_pdf_sa(const Kern<R> &k, R alpha) {
    R s = M<R>::sin(alpha);
    // fp32: pdf <= 0.4 / sigma <= 1.4e6 for sigma >= e^-15, so 1e-30 keeps the
    // quotient finite when a direction did not move in fp32 (alpha = 0).
    const R floor_ = sizeof(R) == 8 ? R(1e-300) : R(1e-30);
    s = s > floor_ ? s : floor_;
    return kern_pdf(k, alpha) / (R(kPiD) * s);
}

// Duff et al. frame (core/sampling.cpp:94-101), to_world (sampling.hpp:49-51).
template <class R> __device__ __forceinline__ V3<R> to_world(V3<R> n, V3<R> l) {
    R sign = M<R>::copysign(R(1), n.z);
    R a = R(-1) / (sign + n.z);
    R b = n.x * n.y * a;
    V3<R> t = mk(R(1) + sign * n.x * n.x * a, sign * b, -sign * n.x);
    V3<R> bt = mk(b, sign + n.y * n.y * a, -n.y);
    return add(add(scl(t, l.x), scl(bt, l.y)), scl(n, l.z));
}

// core/sampling.cpp:103-110
template <class R, class G>
__device__ __forceinline__ V3<R> perturb_dir(V3<R> w, const Kern<R> &k, G &rng) {
    R th = kern_sample(k, rng);
    R ph = R(kTwoPiD) * Unit<R>::draw(rng);
    R st = M<R>::sin(th);
    V3<R> l = mk(st * M<R>::cos(ph), st * M<R>::sin(ph), M<R>::cos(th));
    return unit(to_world(w, l));
}

// core/sampling.cpp:112-121
template <class R> __device__ __forceinline__ void cylindrical(V3<R> w, R &u, R &v) {
    R ph = M<R>::atan2(w.y, w.x);
    if (ph < R(0))
        ph += R(kTwoPiD);
    R uu = ph / R(kTwoPiD);
    if (uu >= R(1))
        uu = R(0);
    R vv = R(0.5) * (w.z + R(1));
    u = uu;
    v = vv < R(0) ? R(0) : (vv > R(1) ? R(1) : vv);
}

// ---- BSDFs (core/scene.cpp:245-414) ---------------------------------------------------
template <class R> __device__ __forceinline__ V3<R> facing(V3<R> n, V3<R> wi) { return dot(n, wi) >= R(0) ? n : neg(n); }

template <class R> __device__ __forceinline__ R fresnel(R cos_i, R ior) {
    R ei = R(1), et = ior, ci = cos_i;
    if (ci < R(0)) {
        R tmp = ei;
        ei = et;
        et = tmp;
        ci = -ci;
    }
    R s2 = (ei / et) * (ei / et) * (R(1) - ci * ci);
    if (s2 >= R(1))
        return R(1);
    R ct = M<R>::sqrt(R(1) - s2);
    R rpa = (et * ci - ei * ct) / (et * ci + ei * ct);
    R rpe = (ei * ci - et * ct) / (ei * ci + et * ct);
    return R(0.5) * (rpa * rpa + rpe * rpe);
}

template <class R> __device__ __forceinline__ V3<R> bsdf_f(const MatD<R> &m, V3<R> wi, V3<R> wo, V3<R> n) {
    if (m.kind == MAT_DIFFUSE) {
        V3<R> ns = facing(n, wi);
        if (dot(ns, wo) <= R(0))
            return mk(R(0), R(0), R(0));
        return scl(m.albedo, R(kInvPiD));
    }
    if (m.kind == MAT_GLOSSY) {
        V3<R> ns = facing(n, wi);
        if (dot(ns, wo) <= R(0))
            return mk(R(0), R(0), R(0));
        R ca = dot(reflect(wi, ns), wo);
        if (ca <= R(0))
            return mk(R(0), R(0), R(0));
        R norm = (m.expo + R(1)) / R(kTwoPiD);
        return scl(m.albedo, norm * M<R>::pow(ca, m.expo));
    }
    return mk(R(0), R(0), R(0));
}

template <class R> __device__ __forceinline__ R bsdf_pdf(const MatD<R> &m, V3<R> wi, V3<R> wo, V3<R> n) {
    if (m.kind == MAT_DIFFUSE) {
        V3<R> ns = facing(n, wi);
        R c = dot(ns, wo);
        return c > R(0) ? c * R(kInvPiD) : R(0);
    }
    if (m.kind == MAT_GLOSSY) {
        V3<R> ns = facing(n, wi);
        R ca = dot(reflect(wi, ns), wo);
        if (ca <= R(0))
            return R(0);
        return (m.expo + R(1)) / R(kTwoPiD) * M<R>::pow(ca, m.expo);
    }
    return R(0);
}

template <class R>
__device__ __forceinline__ bool spec_cont(const MatD<R> &m, V3<R> wi, V3<R> n, int ev, V3<R> &out) {
    if (m.kind == MAT_MIRROR) {
        if (ev != EV_REFLECT)
            return false;
        out = unit(reflect(wi, facing(n, wi)));
        return true;
    }
    if (m.kind != MAT_DIELECTRIC)
        return false;
    R cos_i = dot(n, wi);
    if (ev == EV_REFLECT) {
        out = unit(reflect(wi, facing(n, wi)));
        return true;
    }
    R eta = cos_i > R(0) ? R(1) / m.ior : m.ior;
    V3<R> ns = facing(n, wi);
    R ci = dot(ns, wi);
    R s2 = eta * eta * (R(1) - ci * ci);
    if (s2 >= R(1))
        return false;
    R ct = M<R>::sqrt(R(1) - s2);
    out = unit(add(scl(wi, -eta), scl(ns, eta * ci - ct)));
    return true;
}

template <class R> __device__ __forceinline__ V3<R> spec_weight(const MatD<R> &m, V3<R> wi, V3<R> n, int ev) {
    if (m.kind == MAT_MIRROR)
        return ev == EV_REFLECT ? m.albedo : mk(R(0), R(0), R(0));
    if (m.kind == MAT_DIELECTRIC) {
        R f = fresnel(dot(n, wi), m.ior);
        if (ev == EV_REFLECT)
            return scl(m.albedo, f);
        if (ev == EV_TRANSMIT)
            return scl(m.albedo, R(1) - f);
    }
    return mk(R(0), R(0), R(0));
}

template <class R> __device__ __forceinline__ R spec_prob(const MatD<R> &m, V3<R> wi, V3<R> n, int ev) {
    if (m.kind == MAT_MIRROR)
        return ev == EV_REFLECT ? R(1) : R(0);
    if (m.kind == MAT_DIELECTRIC) {
        R f = fresnel(dot(n, wi), m.ior);
        return ev == EV_REFLECT ? f : R(1) - f;
    }
    return R(0);
}

template <class R> struct BS {
    V3<R> dir;
    R pdf;
    bool zero_thr;
    bool delta;
    int ev;
};

// core/scene.cpp:323-367 (only what the tracer consumes: direction, pdf,
// whether the throughput is zero, delta flag and event).
template <class R, class G>
__device__ __forceinline__ bool bsdf_sample(const MatD<R> &m, V3<R> wi, V3<R> n, G &rng, BS<R> &bs) {
    if (m.kind == MAT_DIFFUSE) {
        V3<R> ns = facing(n, wi);
        R u1 = Unit<R>::draw(rng);
        R u2 = Unit<R>::draw(rng);
        R r = M<R>::sqrt(u1);
        R ph = R(kTwoPiD) * u2;
        R z = R(1) - u1;
        V3<R> l = mk(r * M<R>::cos(ph), r * M<R>::sin(ph), M<R>::sqrt(z > R(0) ? z : R(0)));
        V3<R> wo = to_world(ns, l);
        R c = dot(ns, wo);
        R pdf = (c > R(0) ? c : R(0)) * R(kInvPiD);
        if (pdf <= R(0))
            return false;
        bs.dir = wo;
        bs.pdf = pdf;
        bs.zero_thr = zero3(m.albedo);
        bs.delta = false;
        bs.ev = EV_NONE;
        return true;
    }
    if (m.kind == MAT_GLOSSY) {
        V3<R> ns = facing(n, wi);
        V3<R> axis = reflect(wi, ns);
        R u1 = Unit<R>::draw(rng);
        R u2 = Unit<R>::draw(rng);
        R ca = M<R>::pow(u1, R(1) / (m.expo + R(1)));
        R z = R(1) - ca * ca;
        R sa = M<R>::sqrt(z > R(0) ? z : R(0));
        R ph = R(kTwoPiD) * u2;
        V3<R> l = mk(sa * M<R>::cos(ph), sa * M<R>::sin(ph), ca);
        V3<R> wo = unit(to_world(axis, l));
        R pdf = (m.expo + R(1)) / R(kTwoPiD) * M<R>::pow(ca, m.expo);
        R co = dot(ns, wo);
        bs.dir = wo;
        bs.pdf = pdf;
        bs.zero_thr = !(co > R(0)) || zero3(scl(m.albedo, co));
        bs.delta = false;
        bs.ev = EV_NONE;
        return true;
    }
    if (m.kind == MAT_MIRROR) {
        V3<R> ns = facing(n, wi);
        bs.dir = unit(reflect(wi, ns));
        bs.pdf = R(1);
        bs.zero_thr = zero3(m.albedo);
        bs.delta = true;
        bs.ev = EV_REFLECT;
        return true;
    }
    R f = fresnel(dot(n, wi), m.ior);
    int ev = Unit<R>::draw(rng) < f ? EV_REFLECT : EV_TRANSMIT;
    V3<R> wo;
    if (!spec_cont(m, wi, n, ev, wo))
        return false;
    R q = ev == EV_REFLECT ? f : R(1) - f;
    bs.dir = wo;
    bs.pdf = q;
    bs.zero_thr = zero3(dvs(spec_weight(m, wi, n, ev), q));
    bs.delta = true;
    bs.ev = ev;
    return true;
}

// ---- path vertices ----------------------------------------------------------------------
// Register/local form.  Vertex 0 of every chain path is the camera vertex
// (core/path.cpp:88-92): position = camera position, normal = forward.
template <class R> struct Vx {
    V3<R> p, n;
    int mat, emi;
    bool spec;
    int ev;
};

// Global SoA record [vertex][chain]; meta packs material+1 (16 bits),
// emitter+1 (12 bits), specular (1 bit), event (2 bits).
template <class R> struct alignas(16) GV;
template <> struct alignas(16) GV<float> {
    float4 a, b;   // (px py pz nx) (ny nz meta 0)
};
template <> struct alignas(16) GV<double> {
    double2 a, b, c;   // (px py) (pz nx) (ny nz)
    long long meta, pad;
};

__device__ __forceinline__ uint32_t pack_meta(int mat, int emi, bool spec, int ev) {
    return static_cast<uint32_t>(mat + 1) | (static_cast<uint32_t>(emi + 1) << 16) |
           (spec ? (1u << 28) : 0u) | (static_cast<uint32_t>(ev) << 29);
}
template <class R> __device__ __forceinline__ void unpack_meta(uint32_t m, Vx<R> &v) {
    v.mat = static_cast<int>(m & 0xffffu) - 1;
    v.emi = static_cast<int>((m >> 16) & 0xfffu) - 1;
    v.spec = (m >> 28) & 1u;
    v.ev = static_cast<int>((m >> 29) & 3u);
}

__device__ __forceinline__ Vx<float> load_gv(const GV<float> *p) {
    GV<float> g;
    g.a = p->a;
    g.b = p->b;
    Vx<float> v;
    v.p = mk(g.a.x, g.a.y, g.a.z);
    v.n = mk(g.a.w, g.b.x, g.b.y);
    unpack_meta(__float_as_uint(g.b.z), v);
    return v;
}
__device__ __forceinline__ void store_gv(GV<float> *p, const Vx<float> &v) {
    float4 a = make_float4(v.p.x, v.p.y, v.p.z, v.n.x);
    float4 b = make_float4(v.n.y, v.n.z, __uint_as_float(pack_meta(v.mat, v.emi, v.spec, v.ev)), 0.f);
    p->a = a;
    p->b = b;
}
__device__ __forceinline__ Vx<double> load_gv(const GV<double> *p) {
    double2 a = p->a, b = p->b, c = p->c;
    long long m = p->meta;
    Vx<double> v;
    v.p = mk(a.x, a.y, b.x);
    v.n = mk(b.y, c.x, c.y);
    unpack_meta(static_cast<uint32_t>(m), v);
    return v;
}
__device__ __forceinline__ void store_gv(GV<double> *p, const Vx<double> &v) {
    p->a = make_double2(v.p.x, v.p.y);
    p->b = make_double2(v.p.z, v.n.x);
    p->c = make_double2(v.n.y, v.n.z);
    p->meta = static_cast<long long>(pack_meta(v.mat, v.emi, v.spec, v.ev));
}

}  // namespace rd
