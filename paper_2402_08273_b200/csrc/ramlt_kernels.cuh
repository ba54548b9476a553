// ramlt_kernels.cuh -- sm_100a kernels of the MLT hot path.
//
//   k_step      the persistent chain-step megakernel: one chain per thread (or
//               per G-lane group), chain state SoA in HBM, proposal path in
//               per-thread local memory, scene primitives staged in shared
//               memory, splat fused as vector float4 atomics (fp32) or fp64
//               atomics (parity build).  Replaces run_chain_span
//               (core/driver.cpp:109-173) and everything below it.
//   k_init      chain initialisation (core/driver.cpp:219-242).
//   k_bsub      estimate_b substream sums (core/driver.cpp:31-57).
//   k_adapt_*   shared adaptation statistics (KernelController::record_acceptance,
//               core/adaptation.cpp:60-92) after each lockstep step.
//   k_refine_*  quadtree refinement at barriers (core/partition.cpp:68-100,
//               217-227; core/adaptation.cpp:34-42).
#pragma once

#include "ramlt_device.cuh"

#include <cub/block/block_radix_sort.cuh>
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>
#include <cub/device/device_radix_sort.cuh>

namespace rd {

// ---- engine-side device structures -------------------------------------------------
template <class R> struct KernTab {   // per region: kernels for sigma1 and sigma2
    Kern<R> k1, k2;
};

struct NodeD {   // quadtree node (core/partition.hpp:92-101)
    int level, ix, iy, child, region, tree;
};

struct PartView {
    int kind;   // 0 none, 1 lens grid, 2 lens quadtree, 3 mc grid, 4 mc quadtree
    int ntop, nbot;
    const NodeD *nodes;
    const int *roots;
    unsigned long long *visits;   // per region (record_visit)
};

struct RegionArrays {   // KernelController regions (adaptation.hpp:35-46)
    double *lambda;
    unsigned long long *n;        // n_k
    unsigned int *pend_n;         // i_k
    double *pend_sum;             // A_k (literal)
    unsigned long long *pend_fx;  // A_k (pooled, 2^-24 fixed point)
    unsigned long long *tot_vis;
    double *tot_acc;              // literal
    unsigned long long *tot_fx;   // pooled
    // pooled per-exchange accumulators
    unsigned long long *x_cnt, *x_fx, *x_last;
    unsigned int *x_touched;
    unsigned int *touched_list;
    unsigned int *n_touched;
};

struct TraceBuf {
    unsigned long long *count;
    unsigned long long cap;
    unsigned long long *index;
    long long *region;
    unsigned long long *n;
    double *lambda, *alpha;
};

struct AdaptCfg {
    int L;
    double gmax, gscale, target, lmin, ratio;
    int trace;
};

template <class R> struct ChainArrays {
    GV<R> *verts;   // vertex v >= 1 of chain c at verts[(v-1)*C + c]
    int *klen;
    unsigned int *smask;
    R *cf;          // [4][C]: f.x f.y f.z pi
    R *cr;          // [2][C]: raster u v
    double *eyeden; // cached eye_path_density(current), NaN = unknown
    unsigned long long *rng0, *rng1;
    double *acc, *iacc, *lum;
    unsigned long long *npert, *nlarge, *ipert, *nsteps;
    double *log_a;
    unsigned char *log_f;
    unsigned int log_K;
    int *vreg;
    double *va;
    int *err;
    unsigned long long *rays;   // [2]
};

template <class R> struct StepParams {
    SceneView<R> scene;   // tri/sph point to global; staged into smem by the kernel
    int C;                // chains in this handle
    long long C_total, chain_off;
    int maxv, pk, ctl;    // perturbation kind, controller (0 fixed 1 global 2 regional)
    int W, H;
    unsigned long long seed;
    ChainArrays<R> ch;
    PartView part;
    const KernTab<R> *ktab;
    double *film64;   // parity build: RGB fp64
    float4 *film32;   // production build: RGBA fp32 staging
    // span
    unsigned long long span_start, per, rem;
    int j0, j1;
    int record_visits;   // write vreg/va (adaptive)
    int steal;           // k_step_co: 1 = warp-aggregated work stealing, 0 = one chain per lane
    int refill;          // k_step_co (BVH): idle lanes that end a traversal round
    unsigned long long init_attempts;   // k_step_co<INIT>: attempts per chain before giving up
    GV<R> *pv_scratch;   // k_step_co: proposal vertices in global memory (nullptr: smem)
    unsigned co_stack_off;   // k_step_co (BVH): byte offset of the shared traversal stacks
    int ktab_l2;         // region kernel tables change inside this launch (cooperative): read via L2
    int pooled;          // fuse pooled accumulation into the step
    RegionArrays reg;
};

// Region kernel tables are rewritten between lockstep steps of one cooperative
// launch: read them through L2 (never a stale L1 line).
template <class R> __device__ __forceinline__ KernTab<R> ld_ktab(const KernTab<R> *p, int via_l2) {
    if (!via_l2)
        return *p;
    const R *q = reinterpret_cast<const R *>(p);
    KernTab<R> t;
    t.k1.sigma = __ldcg(q + 0);
    t.k1.lo = __ldcg(q + 1);
    t.k1.mass = __ldcg(q + 2);
    t.k2.sigma = __ldcg(q + 3);
    t.k2.lo = __ldcg(q + 4);
    t.k2.mass = __ldcg(q + 5);
    return t;
}

// ---- path accessors --------------------------------------------------------------------
template <class R> struct CurPath {
    const GV<R> *verts;
    int C, c;
    const CamD<R> *cam;
    __device__ __forceinline__ Vx<R> get(int i) const {
        if (i == 0) {
            Vx<R> v;
            v.p = cam->pos;
            v.n = cam->fwd;
            v.mat = -1;
            v.emi = -1;
            v.spec = false;
            v.ev = EV_NONE;
            return v;
        }
        return load_gv(&verts[static_cast<size_t>(i - 1) * C + c]);
    }
};

// The coroutine kernel's form: the camera vertex by value.  A pointer into
// its block-staged SceneView would take the view's address and pin it -- every
// scene pointer the step reads -- to local memory (c4 -3 %); the megakernel's
// view is in local memory anyway and keeps the pointer (c3 -4 % by value).
template <class R> struct CurPathV {
    const GV<R> *verts;
    int C, c;
    V3<R> cam_pos, cam_fwd;
    __device__ __forceinline__ Vx<R> get(int i) const {
        if (i == 0) {
            Vx<R> v;
            v.p = cam_pos;
            v.n = cam_fwd;
            v.mat = -1;
            v.emi = -1;
            v.spec = false;
            v.ev = EV_NONE;
            return v;
        }
        return load_gv(&verts[static_cast<size_t>(i - 1) * C + c]);
    }
};

template <class R> struct PropPath {
    const Vx<R> *pv;
    int head_end;
    const CurPath<R> *cur;
    __device__ __forceinline__ Vx<R> get(int i) const { return i <= head_end ? pv[i] : cur->get(i); }
};

template <class R, class P> __device__ __forceinline__ V3<R> pdir(const P &path, int i) {
    return unit(sub(path.get(i + 1).p, path.get(i).p));
}

struct RayCount {
    unsigned long long c = 0, v = 0;
};

// core/path.cpp:7-17
template <class R, int G>
__device__ __forceinline__ R geom_term(const SceneView<R> &S, const Vx<R> &a, const Vx<R> &b,
                                       const Group<G> &g, RayCount &rc, bool known_visible = false) {
    V3<R> d = sub(b.p, a.p);
    R d2 = dot(d, d);
    if (d2 <= R(0))
        return R(0);
    V3<R> dir = dvs(d, M<R>::sqrt(d2));
    R gt = M<R>::abs(dot(a.n, dir)) * M<R>::abs(dot(b.n, dir)) / d2;
    if (gt <= R(0))
        return R(0);
    if (known_visible)
        return gt;
    ++rc.v;
    return visible(S, a.p, b.p, g) ? gt : R(0);
}

// core/path.cpp:19-29
template <class R, int G>
__device__ __forceinline__ R area_conv(const SceneView<R> &S, V3<R> from, const Vx<R> &b,
                                       const Group<G> &g, RayCount &rc, bool known_visible = false) {
    V3<R> d = sub(b.p, from);
    R d2 = dot(d, d);
    if (d2 <= R(0))
        return R(0);
    V3<R> dir = dvs(d, M<R>::sqrt(d2));
    R c = M<R>::abs(dot(b.n, dir)) / d2;
    if (c <= R(0))
        return R(0);
    if (known_visible)
        return c;
    ++rc.v;
    return visible(S, from, b.p, g) ? c : R(0);
}

template <class R> struct Contrib {
    V3<R> f;
    R pi, u, v;
};

// eval_contribution (core/path.cpp:40-82)
// vis_from: segments (i, i+1) with i >= vis_from are segments of the chain's
// current path (bit-identical vertices).  That path has pi > 0, so their
// visibility test already passed: the ray is skipped, the value is unchanged.
template <class R, int G, class P>
__device__ Contrib<R> evaluate(const SceneView<R> &S, const P &path, int k, const Group<G> &g,
                               RayCount &rc, int vis_from = 0x7fffffff) {
    Contrib<R> z;
    z.f = mk(R(0), R(0), R(0));
    z.pi = R(0);
    z.u = R(0);
    z.v = R(0);
    if (k < 2)
        return z;
    Vx<R> last = path.get(k - 1);
    if (last.emi < 0)
        return z;
    V3<R> w0 = pdir<R>(path, 0);
    R ru, rv;
    if (!cam_raster(S.cam, w0, ru, rv))
        return z;
    R imp = cam_importance(S.cam, w0);
    V3<R> f = mk(imp, imp, imp);
    Vx<R> prev = path.get(0);
    Vx<R> a = prev;
    for (int i = 0; i + 1 < k; ++i) {
        Vx<R> b = path.get(i + 1);
        if (i > 0 && a.emi >= 0)
            return z;
        R seg = a.spec ? area_conv(S, a.p, b, g, rc, i >= vis_from) : geom_term(S, a, b, g, rc, i >= vis_from);
        if (seg <= R(0))
            return z;
        f = scl(f, seg);
        if (i > 0) {
            const MatD<R> m = S.mat[a.mat];
            V3<R> wi = unit(sub(prev.p, a.p));
            V3<R> wo = unit(sub(b.p, a.p));
            V3<R> bf = a.spec ? spec_weight(m, wi, a.n, a.ev) : bsdf_f(m, wi, wo, a.n);
            if (zero3(bf))
                return z;
            f = mul(f, bf);
        }
        prev = a;
        a = b;
    }
    // a == last, prev == path[k-2]
    V3<R> toward = unit(sub(prev.p, last.p));
    if (dot(last.n, toward) <= R(0))
        return z;
    V3<R> le = S.emit[last.emi];
    if (zero3(le))
        return z;
    f = mul(f, le);
    R pi = lum(f);
    if (!(pi > R(0)) || !M<R>::finite(pi))
        return z;
    z.f = f;
    z.pi = pi;
    z.u = ru;
    z.v = rv;
    return z;
}

// trace_eye_subpath (core/path.cpp:84-142) into pv[0..k-1]; tf = prod of
// dir_pdf * area_conv (large_step t_forward, mutations.cpp:63-66).
// Transition densities and the Metropolis ratio are carried in fp64 in every
// build (as in the reference): products of up to 16 area conversions and the
// truncated-normal pdf at tiny sigma overflow fp32.
template <class R, int G, class RNG>
__device__ bool trace_eye(const SceneView<R> &S, RNG &rng, int maxv, Vx<R> *pv, int &k,
                          unsigned &sm, double &tf, const Group<G> &g, RayCount &rc) {
    Vx<R> cv;
    cv.p = S.cam.pos;
    cv.n = S.cam.fwd;
    cv.mat = -1;
    cv.emi = -1;
    cv.spec = false;
    cv.ev = EV_NONE;
    pv[0] = cv;
    k = 1;
    sm = 0;
    tf = 1.0;
    if (maxv < 2)
        return false;
    R u = Unit<R>::draw(rng);
    R v = Unit<R>::draw(rng);
    V3<R> dir = cam_primary(S.cam, u, v);
    R dpdf = cam_dir_pdf(S.cam, dir);
    V3<R> o = S.cam.pos;
    while (k < maxv) {
        Hit<R> h;
        ++rc.c;
        if (!intersect(S, o, dir, h, g))
            return false;
        Vx<R> x;
        x.p = h.p;
        x.n = h.n;
        x.mat = h.mat;
        x.emi = h.emi;
        const MatD<R> m = S.mat[h.mat];
        x.spec = h.emi < 0 && (m.kind == MAT_MIRROR || m.kind == MAT_DIELECTRIC);
        x.ev = EV_NONE;
        tf *= static_cast<double>(dpdf * (M<R>::abs(dot(h.n, dir)) / (h.t * h.t)));
        pv[k] = x;
        if (x.spec)
            sm |= 1u << k;
        ++k;
        if (h.emi >= 0)
            return true;
        if (k >= maxv)
            return false;
        BS<R> bs;
        if (!bsdf_sample(m, neg(dir), h.n, rng, bs) || bs.zero_thr)
            return false;
        pv[k - 1].ev = bs.ev;
        o = h.p;
        dir = bs.dir;
        dpdf = bs.pdf;
    }
    return false;
}

// eye_path_density (core/path.cpp:144-170)
template <class R, int G, class P>
__device__ double eye_density(const SceneView<R> &S, const P &path, int k, const Group<G> &g, RayCount &rc) {
    if (k < 2)
        return 0.0;
    if (path.get(k - 1).emi < 0)
        return 0.0;
    double p = static_cast<double>(cam_dir_pdf(S.cam, pdir<R>(path, 0)));
    if (p <= 0.0)
        return 0.0;
    Vx<R> prev = path.get(0);
    Vx<R> a = path.get(1);
    p *= static_cast<double>(area_conv(S, prev.p, a, g, rc));
    for (int i = 1; i + 1 < k; ++i) {
        if (a.emi >= 0)
            return 0.0;
        Vx<R> b = path.get(i + 1);
        const MatD<R> m = S.mat[a.mat];
        V3<R> wi = unit(sub(prev.p, a.p));
        V3<R> wo = unit(sub(b.p, a.p));
        R q = a.spec ? spec_prob(m, wi, a.n, a.ev) : bsdf_pdf(m, wi, wo, a.n);
        if (q <= R(0))
            return 0.0;
        p *= static_cast<double>(q * area_conv(S, a.p, b, g, rc));
        if (p <= 0.0)
            return 0.0;
        prev = a;
        a = b;
    }
    return p;
}

// ---- mutation structure from (k, specular mask) -------------------------------------------
// lens_eligibility (core/mutations.cpp:9-21): endpoint or -1
__device__ __forceinline__ int lens_endpoint(int k, unsigned sm) {
    if (k < 2)
        return -1;
    int s = 1;
    while (s < k - 1 && ((sm >> s) & 1u))
        ++s;
    if (s == k - 1)
        return s;
    if (!((sm >> (s + 1)) & 1u))
        return s;
    return -1;
}

// multichain_eligibility (core/mutations.cpp:23-45): returns false when
// ineligible; first = first non-specular after the camera; pmask = perturbed set.
__device__ __forceinline__ bool mc_structure(int k, unsigned sm, int &first, int &endpoint,
                                             unsigned &pmask) {
    if (k < 3)
        return false;
    int f = 1;
    while (f < k - 1 && ((sm >> f) & 1u))
        ++f;
    if (f == k - 1)
        return false;
    int e = -1;
    for (int i = f + 1; i < k; ++i) {
        if (i == k - 1 || (!((sm >> i) & 1u) && !((sm >> (i + 1)) & 1u))) {
            e = i;
            break;
        }
    }
    first = f;
    endpoint = e;
    unsigned below = e >= 32 ? 0xffffffffu : ((1u << e) - 1u);
    pmask = ~sm & below;
    return true;
}

__device__ __forceinline__ float suit_of(int pk, int k, unsigned sm) {
    if (pk == 0)
        return lens_endpoint(k, sm) >= 0 ? 0.5f : 0.0f;
    int f, e;
    unsigned pm;
    return mc_structure(k, sm, f, e, pm) ? 0.5f : 0.0f;
}

// retrace_chain (core/mutations.cpp:78-110): pv[start+1..end] re-traced from o along d.
template <class R, int G>
__device__ bool retrace(const SceneView<R> &S, const CurPath<R> &ref, int kref, int start, int end,
                        V3<R> o, V3<R> d, Vx<R> *pv, const Group<G> &g, RayCount &rc) {
    for (int i = start + 1; i <= end; ++i) {
        Hit<R> h;
        ++rc.c;
        if (!intersect(S, o, d, h, g))
            return false;
        Vx<R> r = ref.get(i);
        const MatD<R> m = S.mat[h.mat];
        bool he = h.emi >= 0;
        bool hs = !he && (m.kind == MAT_MIRROR || m.kind == MAT_DIELECTRIC);
        if (he != (r.emi >= 0) || hs != r.spec)
            return false;
        Vx<R> x;
        x.p = h.p;
        x.n = h.n;
        x.mat = h.mat;
        x.emi = h.emi;
        x.spec = hs;
        x.ev = r.ev;
        pv[i] = x;
        if (i == end)
            break;
        V3<R> c;
        if (!spec_cont(m, neg(d), h.n, r.ev, c))
            return false;
        o = h.p;
        d = c;
    }
    (void)kref;
    return true;
}

// perturbation_density (core/mutations.cpp:176-196)
template <class R> __device__ __forceinline__ Kern<double> kern_d(const Kern<R> &k) {
    return Kern<double>{static_cast<double>(k.sigma), static_cast<double>(k.lo), static_cast<double>(k.mass)};
}

template <class R, class PF, class PT>
__device__ __noinline__ double pert_density(const PF &from, const PT &to, unsigned pmask, int endpoint,
                          const Kern<R> &k1, const Kern<R> &k2) {
    double q = 1.0;
    unsigned m = pmask;
    while (m) {
        int idx = __ffs(m) - 1;
        m &= m - 1;
        V3<R> a = pdir<R>(from, idx);
        V3<R> b = pdir<R>(to, idx);
        R alpha = M<R>::atan2(len(cross(a, b)), dot(a, b));
        q *= static_cast<double>(kern_pdf_sa(idx == 0 ? k1 : k2, alpha));
    }
    Vx<R> p0 = to.get(0);
    for (int i = 0; i < endpoint; ++i) {
        Vx<R> p1 = to.get(i + 1);
        V3<R> d = sub(p1.p, p0.p);
        R d2 = dot(d, d);
        if (d2 <= R(0))
            return 0.0;
        q *= static_cast<double>(M<R>::abs(dot(p1.n, d)) / (d2 * M<R>::sqrt(d2)));
        p0 = p1;
    }
    return q;
}

// mh_accept (core/mutations.cpp:198-208); pi_current > 0 holds for every chain.
__device__ __forceinline__ double mh_accept(double pc, double pp, double tf, double tr, double sf, double sr) {
    if (!(pp > 0.0) || !(tf > 0.0) || !(sf > 0.0))
        return 0.0;
    double r = (pp * tr * sr) / (pc * tf * sf);
    if (::isnan(r))
        return 0.0;
    return r < 1.0 ? r : 1.0;
}

// ---- partitions (core/partition.cpp) --------------------------------------------------------
template <class R> __device__ __forceinline__ int grid_cell(int n, R u, R v) {
    int ix = min(static_cast<int>(u * R(n)), n - 1);
    int iy = min(static_cast<int>(v * R(n)), n - 1);
    return iy * n + ix;
}

template <class R> __device__ __forceinline__ int descend(const NodeD *nodes, int root, R u, R v) {
    NodeD nd = nodes[root];
    while (nd.child >= 0) {
        R sc = M<R>::ldexp(R(1), -nd.level);
        R mu = (R(nd.ix) + R(0.5)) * sc;
        R mv = (R(nd.iy) + R(0.5)) * sc;
        int q = (u >= mu ? 1 : 0) + (v >= mv ? 2 : 0);
        nd = nodes[nd.child + q];
    }
    return nd.region;
}

template <class R> __device__ __forceinline__ int classify(const PartView &p, R ru, R rv, R cu, R cv) {
    switch (p.kind) {
    case 1: return grid_cell(p.ntop, ru, rv);
    case 2: return descend(p.nodes, 0, ru, rv);
    case 3: return grid_cell(p.ntop, ru, rv) * (p.nbot * p.nbot) + grid_cell(p.nbot, cu, cv);
    case 4: return descend(p.nodes, p.roots[grid_cell(p.ntop, ru, rv)], cu, cv);
    }
    return 0;
}

// ---- splat (core/driver.cpp:59-64; core/film.cpp:12-20) ------------------------------------
template <class R>
__device__ __forceinline__ void film_add(const StepParams<R> &P, R u, R v, V3<R> val, double &lum_acc);

template <>
__device__ __forceinline__ void film_add<double>(const StepParams<double> &P, double u, double v,
                                                 V3<double> val, double &lum_acc) {
    int x = min(static_cast<int>(u * P.W), P.W - 1);
    int row = P.H - 1 - min(static_cast<int>(v * P.H), P.H - 1);
    double *px = &P.film64[(static_cast<size_t>(row) * P.W + x) * 3];
    atomicAdd(px + 0, val.x);
    atomicAdd(px + 1, val.y);
    atomicAdd(px + 2, val.z);
    lum_acc += lum(val);
}

template <>
__device__ __forceinline__ void film_add<float>(const StepParams<float> &P, float u, float v,
                                                V3<float> val, double &lum_acc) {
    int x = min(static_cast<int>(u * P.W), P.W - 1);
    int row = P.H - 1 - min(static_cast<int>(v * P.H), P.H - 1);
    atomicAdd(&P.film32[static_cast<size_t>(row) * P.W + x], make_float4(val.x, val.y, val.z, 0.f));
    lum_acc += static_cast<double>(lum(val));
}

// ---- scene staging ------------------------------------------------------------------------
template <class R> __device__ __forceinline__ size_t stage_bytes_sph(int nsph) {
    return (static_cast<size_t>(nsph) * sizeof(SphD<R>) + 15) & ~size_t(15);
}

template <class R> __device__ SceneView<R> stage_scene(const SceneView<R> &g, char *smem) {
    SceneView<R> s = g;
    size_t bs = static_cast<size_t>(g.nsph) * sizeof(SphD<R>);
    size_t bt = g.bvh ? 0 : static_cast<size_t>(g.ntri) * sizeof(TriD<R>);   // BVH: triangles stay in L2
    size_t off = stage_bytes_sph<R>(g.nsph);
    const unsigned *src_s = reinterpret_cast<const unsigned *>(g.sph);
    const unsigned *src_t = reinterpret_cast<const unsigned *>(g.tri);
    unsigned *dst_s = reinterpret_cast<unsigned *>(smem);
    unsigned *dst_t = reinterpret_cast<unsigned *>(smem + off);
    for (size_t i = threadIdx.x; i < bs / 4; i += blockDim.x)
        dst_s[i] = __ldg(src_s + i);
    for (size_t i = threadIdx.x; i < bt / 4; i += blockDim.x)
        dst_t[i] = __ldg(src_t + i);
    __syncthreads();
    s.sph = reinterpret_cast<const SphD<R> *>(smem);
    if (!g.bvh)
        s.tri = reinterpret_cast<const TriD<R> *>(smem + off);
    return s;
}

// ---- the chain-step megakernel --------------------------------------------------------------
template <class R> struct ChainRegs {
    int k;
    unsigned sm;
    V3<R> f;
    R pi, ru, rv;
    double eyeden;
    double acc, iacc, lum;
    unsigned long long npert, nlarge, ipert, nsteps;
};

template <int RK> struct RngIO;
template <> struct RngIO<RNG_PCG> {
    static __device__ __forceinline__ void load(Rng<RNG_PCG> &r, const unsigned long long *a,
                                                const unsigned long long *b, int c, unsigned long long,
                                                unsigned long long) {
        r.state = a[c];
        r.inc = b[c];
    }
    static __device__ __forceinline__ void store(const Rng<RNG_PCG> &r, unsigned long long *a,
                                                 unsigned long long *b, int c) {
        a[c] = r.state;
        b[c] = r.inc;
    }
};
template <> struct RngIO<RNG_PHILOX> {
    static __device__ __forceinline__ void load(Rng<RNG_PHILOX> &r, const unsigned long long *a,
                                                const unsigned long long *, int c, unsigned long long seed,
                                                unsigned long long stream) {
        r.reseed(seed, stream);
        r.draw = a[c];
    }
    static __device__ __forceinline__ void store(const Rng<RNG_PHILOX> &r, unsigned long long *a,
                                                 unsigned long long *, int c) {
        a[c] = r.draw;
    }
};

// One mutation of one chain: core/driver.cpp:113-171.
template <class R, int RK, int G>
__device__ void mutate(const StepParams<R> &P, const SceneView<R> &S, int c, long long gc,
                       unsigned long long index, ChainRegs<R> &cs, Rng<RK> &rng, const Group<G> &g,
                       RayCount &rc) {
    CurPath<R> cur{P.ch.verts, P.C, c, &S.cam};
    Vx<R> pv[kMaxV];
    int head_end = 0;
    int kp = cs.k;
    unsigned smp = cs.sm;
    double tf = 0.0, tr = 0.0;
    const int pk = P.pk;

    // suitability (core/mutations.cpp:47-56)
    int e_lens = -1, first = 0, endpoint = 0;
    unsigned pmask = 0;
    bool elig;
    if (pk == 0) {
        e_lens = lens_endpoint(cs.k, cs.sm);
        elig = e_lens >= 0;
        endpoint = e_lens;
        pmask = 1u;
    } else {
        elig = mc_structure(cs.k, cs.sm, first, endpoint, pmask);
    }
    const R s_pert = elig ? R(0.5) : R(0);
    const bool choose = elig && Unit<R>::draw(rng) < s_pert;

    double a = 0.0;
    Contrib<R> pc;
    pc.pi = R(0);
    int region = -1;

    if (choose) {
        // classify_path (core/driver.cpp:95-107)
        R cu = R(0), cv = R(0);
        if (P.ctl == 2 && pk == 1)
            cylindrical(pdir<R>(cur, first), cu, cv);
        region = P.ctl == 2 ? classify(P.part, cs.ru, cs.rv, cu, cv) : 0;
        const KernTab<R> kt = ld_ktab(P.ktab + region, P.ktab_l2);
        // lens_perturb / multichain_perturb (core/mutations.cpp:122-174)
        Vx<R> cam0 = cur.get(0);
        pv[0] = cam0;
        bool ok = true;
        unsigned m = pmask;
        while (m) {
            int idx = __ffs(m) - 1;
            m &= m - 1;
            int next = m ? (__ffs(m) - 1) : endpoint;
            V3<R> nd = perturb_dir(pdir<R>(cur, idx), idx == 0 ? kt.k1 : kt.k2, rng);
            if (!retrace(S, cur, cs.k, idx, next, pv[idx].p, nd, pv, g, rc)) {
                ok = false;
                break;
            }
        }
        if (ok) {
            head_end = endpoint;
            PropPath<R> prop{pv, head_end, &cur};
            tf = pert_density(cur, prop, pmask, endpoint, kt.k1, kt.k2);
            tr = pert_density(prop, cur, pmask, endpoint, kt.k1, kt.k2);
            pc = evaluate(S, prop, cs.k, g, rc, endpoint + 1);
            if (pc.pi > R(0)) {
                if (P.ctl == 2) {
                    R pu = R(0), pv_ = R(0);
                    if (pk == 1)
                        cylindrical(pdir<R>(prop, first), pu, pv_);
                    int preg = classify(P.part, pc.u, pc.v, pu, pv_);
                    const KernTab<R> kr = ld_ktab(P.ktab + preg, P.ktab_l2);
                    tr = pert_density(prop, cur, pmask, endpoint, kr.k1, kr.k2);
                }
                a = mh_accept(cs.pi, pc.pi, tf, tr, s_pert, s_pert);
            }
        }
        if (g.lane == 0 && P.ctl == 2)
            atomicAdd(&P.part.visits[region], 1ull);
        cs.acc += a;
        cs.iacc += a;
        ++cs.npert;
        ++cs.ipert;
    } else {
        ++cs.nlarge;
        // large_step (core/mutations.cpp:58-71)
        if (trace_eye(S, rng, P.maxv, pv, kp, smp, tf, g, rc)) {
            head_end = kp - 1;
            PropPath<R> prop{pv, head_end, &cur};
            pc = evaluate(S, prop, kp, g, rc);
            if (pc.pi > R(0)) {
                if (!(cs.eyeden == cs.eyeden))   // NaN: not cached yet
                    cs.eyeden = eye_density(S, cur, cs.k, g, rc);
                tr = cs.eyeden;
                R sx = R(1) - s_pert;
                R sy = R(1) - R(suit_of(pk, kp, smp));
                a = mh_accept(cs.pi, pc.pi, tf, tr, sx, sy);
            }
        }
    }

    // splat (core/driver.cpp:59-64) -- the group leader writes
    if (g.lane == 0) {
        const R ar = static_cast<R>(a);
        if (a < 1.0 && cs.pi > R(0))
            film_add(P, cs.ru, cs.rv, scl(cs.f, (R(1) - ar) / cs.pi), cs.lum);
        if (pc.pi > R(0) && a > 0.0)
            film_add(P, pc.u, pc.v, scl(pc.f, ar / pc.pi), cs.lum);
    } else {
        // keep the lum accumulator identical on all lanes (leader's value is stored)
    }

    // accept / commit (core/driver.cpp:168-171)
    bool accepted = false;
    if (a > 0.0 && static_cast<double>(Unit<R>::draw(rng)) < a) {
        accepted = true;
        if (g.lane == 0)
            for (int i = 1; i <= head_end; ++i)
                store_gv(&P.ch.verts[static_cast<size_t>(i - 1) * P.C + c], pv[i]);
        cs.k = kp;
        cs.sm = choose ? cs.sm : smp;
        cs.f = pc.f;
        cs.pi = pc.pi;
        cs.ru = pc.u;
        cs.rv = pc.v;
        cs.eyeden = __longlong_as_double(0x7ff8000000000000LL);   // NaN
    }

    if (g.lane == 0) {
        if (cs.nsteps < P.ch.log_K) {
            size_t o = static_cast<size_t>(cs.nsteps) * P.C + c;
            P.ch.log_a[o] = a;
            P.ch.log_f[o] = static_cast<unsigned char>((accepted ? 1 : 0) | (choose ? 2 : 0) | 4);
        }
        if (P.record_visits) {
            P.ch.vreg[c] = (choose && P.ctl != 0) ? region : -1;
            P.ch.va[c] = a;
        }
    }
    ++cs.nsteps;
    (void)gc;
    (void)index;
}

#ifndef RAMLT_BVH_MINBLOCKS
#define RAMLT_BVH_MINBLOCKS 10
#endif
#ifndef RAMLT_LANES_MINBLOCKS
#define RAMLT_LANES_MINBLOCKS 4
#endif
// fp32 k_step trades registers for resident warps.  The BVH instantiation
// (G == 0) is memory-latency bound -- c4 (fixed) at 1/5/6/7/8/10/12/16 blocks
// per SM: 35.4/39.1/42.6/45.2/46.8/48.3/48.0/37.5 M mut/s; the lane-group
// instantiations gain ~5% at 4 blocks (128 registers) on c5.
template <class R, int RK, int G>
__global__ void __launch_bounds__(128, sizeof(R) == 8 ? 1 : G == 0 ? RAMLT_BVH_MINBLOCKS : RAMLT_LANES_MINBLOCKS)
k_step(StepParams<R> P) {
    extern __shared__ __align__(16) char smem[];
    SceneView<R> S = stage_scene(P.scene, smem);
    Group<G> g;
    const int c = static_cast<int>((static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) / Lanes<G>::n);
    if (c >= P.C)
        return;
    const long long gc = P.chain_off + c;
    const unsigned long long my_steps = P.per + (static_cast<unsigned long long>(gc) < P.rem ? 1ull : 0ull);

    ChainRegs<R> cs;
    cs.k = P.ch.klen[c];
    cs.sm = P.ch.smask[c];
    cs.f = mk(P.ch.cf[c], P.ch.cf[P.C + c], P.ch.cf[2 * P.C + c]);
    cs.pi = P.ch.cf[3 * P.C + c];
    cs.ru = P.ch.cr[c];
    cs.rv = P.ch.cr[P.C + c];
    cs.eyeden = P.ch.eyeden[c];
    cs.acc = P.ch.acc[c];
    cs.iacc = P.ch.iacc[c];
    cs.lum = P.ch.lum[c];
    cs.npert = P.ch.npert[c];
    cs.nlarge = P.ch.nlarge[c];
    cs.ipert = P.ch.ipert[c];
    cs.nsteps = P.ch.nsteps[c];
    Rng<RK> rng;
    RngIO<RK>::load(rng, P.ch.rng0, P.ch.rng1, c, P.seed, static_cast<unsigned long long>(gc));
    RayCount rc;

    for (int j = P.j0; j < P.j1; ++j) {
        if (static_cast<unsigned long long>(j) >= my_steps) {
            if (P.record_visits && g.lane == 0)
                P.ch.vreg[c] = -1;
            break;
        }
        unsigned long long index = P.span_start + static_cast<unsigned long long>(j) * P.C_total + gc;
        mutate<R, RK, G>(P, S, c, gc, index, cs, rng, g, rc);
    }

    if (g.lane == 0) {
        P.ch.klen[c] = cs.k;
        P.ch.smask[c] = cs.sm;
        P.ch.cf[c] = cs.f.x;
        P.ch.cf[P.C + c] = cs.f.y;
        P.ch.cf[2 * P.C + c] = cs.f.z;
        P.ch.cf[3 * P.C + c] = cs.pi;
        P.ch.cr[c] = cs.ru;
        P.ch.cr[P.C + c] = cs.rv;
        P.ch.eyeden[c] = cs.eyeden;
        P.ch.acc[c] = cs.acc;
        P.ch.iacc[c] = cs.iacc;
        P.ch.lum[c] = cs.lum;
        P.ch.npert[c] = cs.npert;
        P.ch.nlarge[c] = cs.nlarge;
        P.ch.ipert[c] = cs.ipert;
        P.ch.nsteps[c] = cs.nsteps;
        RngIO<RK>::store(rng, P.ch.rng0, P.ch.rng1, c);
        // warp-aggregated ray counters
    }
    // ray counters: one atomic per converged lane set (any subset mask is safe
    // for __reduce_add_sync; per-launch per-thread counts fit 32 bits)
    unsigned rcc = g.lane == 0 ? static_cast<unsigned>(rc.c) : 0u;
    unsigned rcv = g.lane == 0 ? static_cast<unsigned>(rc.v) : 0u;
    unsigned act = __activemask();
    unsigned sc = __reduce_add_sync(act, rcc);
    unsigned sv = __reduce_add_sync(act, rcv);
    if ((threadIdx.x & 31) == __ffs(act) - 1) {
        atomicAdd(&P.ch.rays[0], static_cast<unsigned long long>(sc));
        atomicAdd(&P.ch.rays[1], static_cast<unsigned long long>(sv));
    }
}

// ---- chain initialisation (core/driver.cpp:219-242) -----------------------------------------
template <class R, int RK, int G>
__device__ void init_chain(const StepParams<R> &P, const SceneView<R> &S, int c, unsigned long long max_attempts,
                           RayCount &rc) {
    Group<G> g;
    const long long gc = P.chain_off + c;
    Rng<RK> init;
    init.reseed(P.seed, kStreamInit + static_cast<unsigned long long>(gc) * 2ull);
    Vx<R> pv[kMaxV];
    bool ok = false;
    for (unsigned long long t = 0; t < max_attempts; ++t) {
        int k;
        unsigned sm;
        double tf;
        if (!trace_eye(S, init, P.maxv, pv, k, sm, tf, g, rc))
            continue;
        CurPath<R> dummy{P.ch.verts, P.C, c, &S.cam};
        PropPath<R> path{pv, k - 1, &dummy};
        Contrib<R> con = evaluate(S, path, k, g, rc);
        if (con.pi > R(0)) {
            for (int i = 1; i < k; ++i)
                store_gv(&P.ch.verts[static_cast<size_t>(i - 1) * P.C + c], pv[i]);
            P.ch.klen[c] = k;
            P.ch.smask[c] = sm;
            P.ch.cf[c] = con.f.x;
            P.ch.cf[P.C + c] = con.f.y;
            P.ch.cf[2 * P.C + c] = con.f.z;
            P.ch.cf[3 * P.C + c] = con.pi;
            P.ch.cr[c] = con.u;
            P.ch.cr[P.C + c] = con.v;
            ok = true;
            break;
        }
    }
    if (!ok)
        atomicExch(P.ch.err, 1);
    P.ch.eyeden[c] = __longlong_as_double(0x7ff8000000000000LL);
    P.ch.acc[c] = 0.0;
    P.ch.iacc[c] = 0.0;
    P.ch.lum[c] = 0.0;
    P.ch.npert[c] = 0;
    P.ch.nlarge[c] = 0;
    P.ch.ipert[c] = 0;
    P.ch.nsteps[c] = 0;
    Rng<RK> rng;
    rng.reseed(P.seed, static_cast<unsigned long long>(gc));
    RngIO<RK>::store(rng, P.ch.rng0, P.ch.rng1, c);
}

// Persistent, work-stealing chain initialisation: the number of attempts per
// chain is geometric, so a lane that finishes takes the next chain instead of
// idling until the warp's unluckiest chain is done.  `work` is zeroed.
template <class R, int RK, int G>
__global__ void __launch_bounds__(128, sizeof(R) == 4 && G == 0 ? RAMLT_BVH_MINBLOCKS : 1)
k_init(StepParams<R> P, unsigned long long max_attempts, unsigned int *work) {
    extern __shared__ __align__(16) char smem[];
    SceneView<R> S = stage_scene(P.scene, smem);
    RayCount rc;
    for (;;) {
        unsigned c = atomicAdd(work, 1u);
        if (c >= static_cast<unsigned>(P.C))
            break;
        init_chain<R, RK, G>(P, S, static_cast<int>(c), max_attempts, rc);
    }
}

// ---- estimate_b substreams (core/driver.cpp:31-57) --------------------------------------------
template <class R, int RK, int G>
__global__ void __launch_bounds__(128) k_bsub(StepParams<R> P, unsigned long long n_samples,
                                              unsigned long long S_total, unsigned long long s_begin,
                                              unsigned long long s_end, double *partials) {
    extern __shared__ __align__(16) char smem[];
    SceneView<R> S = stage_scene(P.scene, smem);
    Group<G> g;
    unsigned long long s = s_begin + blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x;
    if (s >= s_end)
        return;
    Rng<RK> rng;
    rng.reseed(P.seed, kStreamB + 2ull * s);
    Vx<R> pv[kMaxV];
    RayCount rc;
    double sum = 0.0, sq = 0.0;
    for (unsigned long long j = s; j < n_samples; j += S_total) {
        int k;
        unsigned sm;
        double tf;
        double v = 0.0;
        if (trace_eye(S, rng, P.maxv, pv, k, sm, tf, g, rc)) {
            CurPath<R> dummy{P.ch.verts, P.C, 0, &S.cam};
            PropPath<R> path{pv, k - 1, &dummy};
            Contrib<R> con = evaluate(S, path, k, g, rc);
            if (con.pi > R(0)) {
                if (tf > 0.0)
                    v = static_cast<double>(con.pi) / tf;
            }
        }
        sum += v;
        sq += v * v;
    }
    partials[2 * (s - s_begin)] = sum;
    partials[2 * (s - s_begin) + 1] = sq;
}

// ---- adaptation ------------------------------------------------------------------------------
// step_size / update_lambda (core/adaptation.cpp:10-20)
__device__ __forceinline__ double lambda_next(double lam, double ah, unsigned long long n, const AdaptCfg &c) {
    double gs = c.gscale / ::sqrt(static_cast<double>(n));
    double gm = c.gmax < gs ? c.gmax : gs;
    double diff = ah - c.target;
    double sg = diff > 0.0 ? 1.0 : (diff < 0.0 ? -1.0 : 0.0);
    double nl = lam + gm * sg;
    return c.lmin > nl ? c.lmin : nl;
}

template <class R> __device__ __forceinline__ void set_ktab(KernTab<R> *kt, double lambda, double ratio) {
    // sigma_for (core/adaptation.cpp:44-50) + AngularKernel ctor in fp64, stored as R
    double s = ::exp(0.5 * lambda);
    Kern<double> a = make_kern<double>(s);
    Kern<double> b = make_kern<double>(ratio * s);
    KernTab<R> t;
    t.k1.sigma = static_cast<R>(a.sigma);
    t.k1.lo = static_cast<R>(a.lo);
    t.k1.mass = static_cast<R>(a.mass);
    t.k2.sigma = static_cast<R>(b.sigma);
    t.k2.lo = static_cast<R>(b.lo);
    t.k2.mass = static_cast<R>(b.mass);
    *kt = t;
}

template <class R>
__global__ void k_ktab_init(KernTab<R> *kt, const double *lambda, int n, double ratio) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n)
        set_ktab(&kt[i], lambda[i], ratio);
}

__device__ __forceinline__ void trace_push(const TraceBuf &tb, unsigned long long index, int region,
                                           unsigned long long n, double lam, double ah) {
    unsigned long long slot = atomicAdd(tb.count, 1ull);
    if (slot < tb.cap) {
        tb.index[slot] = index;
        tb.region[slot] = region;
        tb.n[slot] = n;
        tb.lambda[slot] = lam;
        tb.alpha[slot] = ah;
    }
}

// Literal rule: record_acceptance in canonical (lockstep step, chain) order.
// One block; tiles of 1024 chains in order; each tile stable-sorted by region
// so every region's visits form a run processed sequentially by one thread.
template <class R>
__global__ void __launch_bounds__(1024) k_adapt_literal(const int *vreg, const double *va, int C,
                                                        long long chain_off, long long C_total,
                                                        unsigned long long span_start, int j,
                                                        RegionArrays ra, KernTab<R> *ktab, AdaptCfg cfg,
                                                        TraceBuf tb) {
    typedef cub::BlockRadixSort<int, 1024, 1, int> Sort;
    __shared__ union {
        typename Sort::TempStorage tmp;
        struct {
            int k[1024];
            int v[1024];
            double a[1024];
        } d;
    } sm;
    int *keys_s = sm.d.k;
    int *vals_s = sm.d.v;
    double *a_s = sm.d.a;
    for (int base = 0; base < C; base += 1024) {
        int t = threadIdx.x;
        int cidx = base + t;
        int key[1], val[1];
        key[0] = (cidx < C && vreg[cidx] >= 0) ? vreg[cidx] : 0x7fffffff;
        val[0] = cidx;
        Sort(sm.tmp).Sort(key, val);
        __syncthreads();   // temp storage is aliased by the run arrays below
        // BlockRadixSort with 1 item/thread leaves thread t holding rank t
        keys_s[t] = key[0];
        vals_s[t] = val[0];
        a_s[t] = key[0] != 0x7fffffff ? va[val[0]] : 0.0;
        __syncthreads();
        int r = keys_s[t];
        bool head = r != 0x7fffffff && (t == 0 || keys_s[t - 1] != r);
        if (head) {
            double lam = ra.lambda[r];
            unsigned long long n = ra.n[r];
            unsigned int pn = ra.pend_n[r];
            double ps = ra.pend_sum[r];
            unsigned long long tv = ra.tot_vis[r];
            double ta = ra.tot_acc[r];
            bool changed = false;
            for (int q = t; q < 1024 && keys_s[q] == r; ++q) {
                int ci = vals_s[q];
                double a = a_s[q];
                ta += a;
                tv += 1;
                ps += a;
                pn += 1;
                if (pn < static_cast<unsigned int>(cfg.L))
                    continue;
                double ah = ps / pn;
                ah = ah < 0.0 ? 0.0 : (ah > 1.0 ? 1.0 : ah);
                unsigned long long n0 = n;
                lam = lambda_next(lam, ah, n0, cfg);
                n = n0 + 1;
                pn = 0;
                ps = 0.0;
                changed = true;
                if (cfg.trace)
                    trace_push(tb, span_start + static_cast<unsigned long long>(j) * C_total + chain_off + ci,
                               r, n0, lam, ah);
            }
            ra.lambda[r] = lam;
            ra.n[r] = n;
            ra.pend_n[r] = pn;
            ra.pend_sum[r] = ps;
            ra.tot_vis[r] = tv;
            ra.tot_acc[r] = ta;
            if (changed)
                set_ktab(&ktab[r], lam, cfg.ratio);
        }
        __syncthreads();
    }
}

// Pooled rule, phase 1: per-region visit counts / fixed-point sums / last
// index, warp-aggregated over lanes that share a region.
__device__ __forceinline__ unsigned long long to_fx(double a) {
    return static_cast<unsigned long long>(a * 16777216.0 + 0.5);   // 2^-24 resolution
}

__global__ void k_adapt_pool_accum(const int *vreg, const double *va, int C, long long chain_off,
                                   long long C_total, unsigned long long span_start, int j, RegionArrays ra) {
    int c = blockIdx.x * blockDim.x + threadIdx.x;
    int r = (c < C) ? vreg[c] : -1;
    unsigned act = __ballot_sync(0xffffffffu, r >= 0);
    if (r < 0)
        return;
    unsigned peers = __match_any_sync(act, r);
    unsigned long long fx = to_fx(va[c]);
    unsigned long long idx = span_start + static_cast<unsigned long long>(j) * C_total + chain_off + c;
    // reduce over peers
    unsigned fx32 = static_cast<unsigned>(fx);   // <= 2^24, 32 lanes <= 2^29
    unsigned s = __reduce_add_sync(peers, fx32);
    unsigned cnt = __popc(peers);
    int leader = __ffs(peers) - 1;
    int hi = 31 - __clz(peers);
    unsigned long long last = __shfl_sync(peers, idx, hi);
    if ((threadIdx.x & 31) == leader) {
        atomicAdd(&ra.x_cnt[r], static_cast<unsigned long long>(cnt));
        atomicAdd(&ra.x_fx[r], static_cast<unsigned long long>(s));
        atomicMax(&ra.x_last[r], last);
        if (atomicExch(&ra.x_touched[r], 1u) == 0u) {
            unsigned slot = atomicAdd(ra.n_touched, 1u);
            ra.touched_list[slot] = static_cast<unsigned>(r);
        }
    }
}

// Pooled rule, phase 2: one update per touched region.
// n_scan > 0 (sharded runs, after the SUM/SUM/MAX all-reduce of x_cnt/x_fx/x_last):
// every region in [0, n_scan) with pooled visits is updated, not only the ones
// this rank's chains touched -- a region visited only on another rank must take
// the same lambda step here, and its exchanged counts must be consumed.
template <class R>
__global__ void k_adapt_pool_apply(RegionArrays ra, KernTab<R> *ktab, AdaptCfg cfg, TraceBuf tb, int n_scan) {
    unsigned nt = n_scan > 0 ? static_cast<unsigned>(n_scan) : *ra.n_touched;
    for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < nt; i += gridDim.x * blockDim.x) {
        int r = n_scan > 0 ? static_cast<int>(i) : static_cast<int>(ra.touched_list[i]);
        unsigned long long cnt = ra.x_cnt[r], fx = ra.x_fx[r], last = ra.x_last[r];
        if (n_scan > 0 && cnt == 0)
            continue;
        ra.x_cnt[r] = 0;
        ra.x_fx[r] = 0;
        ra.x_last[r] = 0;
        ra.x_touched[r] = 0;
        ra.tot_vis[r] += cnt;
        ra.tot_fx[r] += fx;
        unsigned long long pn = ra.pend_n[r] + cnt;
        unsigned long long pf = ra.pend_fx[r] + fx;
        if (pn < static_cast<unsigned long long>(cfg.L)) {
            ra.pend_n[r] = static_cast<unsigned>(pn);
            ra.pend_fx[r] = pf;
            continue;
        }
        double ah = static_cast<double>(pf) / 16777216.0 / static_cast<double>(pn);
        ah = ah < 0.0 ? 0.0 : (ah > 1.0 ? 1.0 : ah);
        unsigned long long n0 = ra.n[r];
        double lam = lambda_next(ra.lambda[r], ah, n0, cfg);
        ra.lambda[r] = lam;
        ra.n[r] = n0 + 1;
        ra.pend_n[r] = 0;
        ra.pend_fx[r] = 0;
        set_ktab(&ktab[r], lam, cfg.ratio);
        if (cfg.trace)
            trace_push(tb, last, r, n0, lam, ah);
    }
}

__global__ void k_reset_touched(unsigned *n_touched) { *n_touched = 0; }

// ---- quadtree refinement (core/partition.cpp:68-100, 217-227; core/adaptation.cpp:34-42) --------
// Snapshot the leaves, split those with visits >= M_split; children get ids in
// tree-then-leaf order.  Data-parallel with the exact id order preserved:
//   k_refine_keys   candidate leaves of the snapshot [0, n0): key = tree, others
//                   key = n_trees (sorted last); counts the candidates
//   (host)          cub::DeviceRadixSort::SortPairs (stable LSD) -> candidates in
//                   tree-major, node-index order = the reference's visiting order
//   k_refine_apply  split s gets nodes n0 + 4s.. and regions nreg0 + 4s..,
//                   children LL, LR, UL, UR, lambda copied, n = max(1, n / 4)
//   k_refine_finish node / region counts
__global__ void k_refine_keys(const NodeD *nodes, int n0, int n_trees, const unsigned long long *visits,
                              unsigned long long m_split, int *key, int *val, int *count) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    bool cand = false;
    if (i < n0) {
        NodeD nd = nodes[i];
        cand = nd.child < 0 && nd.level < 16 && visits[nd.region] >= m_split;
        key[i] = cand ? nd.tree : n_trees;
        val[i] = i;
    }
    unsigned b = __ballot_sync(0xffffffffu, cand);
    if ((threadIdx.x & 31) == 0 && b)
        atomicAdd(count, __popc(b));
}

template <class R>
__global__ void k_refine_apply(NodeD *nodes, int n0, int cap_nodes, const int *order, const int *count,
                               RegionArrays ra, KernTab<R> *ktab, unsigned long long *visits, const int *n_regions,
                               int cap_regions, int *err) {
    int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= *count)
        return;
    const int nn = n0 + 4 * s, nr = *n_regions + 4 * s;
    if (nn + 4 > cap_nodes || nr + 4 > cap_regions) {
        *err = 2;
        return;
    }
    int idx = order[s];
    NodeD nd = nodes[idx];
    unsigned long long np = ra.n[nd.region];
    double lam = ra.lambda[nd.region];
    unsigned long long nc = np / 4 > 1 ? np / 4 : 1;
    KernTab<R> kt = ktab[nd.region];
    for (int q = 0; q < 4; ++q) {
        NodeD ch;
        ch.level = nd.level + 1;
        ch.ix = nd.ix * 2 + (q & 1);
        ch.iy = nd.iy * 2 + (q >> 1);
        ch.child = -1;
        ch.tree = nd.tree;
        ch.region = nr + q;
        ra.lambda[nr + q] = lam;
        ra.n[nr + q] = nc;
        ra.pend_n[nr + q] = 0;
        ra.pend_sum[nr + q] = 0.0;
        ra.pend_fx[nr + q] = 0;
        ra.tot_vis[nr + q] = 0;
        ra.tot_acc[nr + q] = 0.0;
        ra.tot_fx[nr + q] = 0;
        visits[nr + q] = 0;
        ktab[nr + q] = kt;
        nodes[nn + q] = ch;
    }
    nodes[idx].child = nn;
    visits[nd.region] = 0;
}

__global__ void k_refine_finish(int n0, const int *count, int *n_nodes, int *n_regions, int *splits_out) {
    int m = *count;
    *n_nodes = n0 + 4 * m;
    *n_regions += 4 * m;
    *splits_out = m;
}

// ---- reductions & film ---------------------------------------------------------------------
// Fixed-order two-level reduction of per-chain tallies: block b sums chains
// [b*256, (b+1)*256) by a shared-memory tree; the host-side caller finishes
// in block order.  out[b*6 + 0..5] = acc, iacc, lum, npert, nlarge, ipert.
__global__ void k_reduce_chains(const double *acc, double *iacc, const double *lum,
                                const unsigned long long *npert, const unsigned long long *nlarge,
                                unsigned long long *ipert, int C, int reset_interval, double *out) {
    __shared__ double s[6][256];
    int c = blockIdx.x * 256 + threadIdx.x;
    bool in = c < C;
    s[0][threadIdx.x] = in ? acc[c] : 0.0;
    s[1][threadIdx.x] = in ? iacc[c] : 0.0;
    s[2][threadIdx.x] = in ? lum[c] : 0.0;
    s[3][threadIdx.x] = in ? static_cast<double>(npert[c]) : 0.0;
    s[4][threadIdx.x] = in ? static_cast<double>(nlarge[c]) : 0.0;
    s[5][threadIdx.x] = in ? static_cast<double>(ipert[c]) : 0.0;
    if (in && reset_interval) {
        iacc[c] = 0.0;
        ipert[c] = 0;
    }
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if (threadIdx.x < w)
            for (int q = 0; q < 6; ++q)
                s[q][threadIdx.x] += s[q][threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x < 6)
        out[blockIdx.x * 6 + threadIdx.x] = s[threadIdx.x][0];
}

__global__ void k_fold_film(float4 *stage, double *master, int npix) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= npix)
        return;
    float4 v = stage[i];
    master[3 * i + 0] += static_cast<double>(v.x);
    master[3 * i + 1] += static_cast<double>(v.y);
    master[3 * i + 2] += static_cast<double>(v.z);
    stage[i] = make_float4(0.f, 0.f, 0.f, 0.f);
}

__global__ void k_to_image(const double *film, float *img, int n, double scale) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n)
        img[i] = static_cast<float>(film[i] * scale);
}

// error_report(image, reference, eps, rgb = false) (core/diagnostics.cpp:11-38)
// on the image to_image(scale) would produce: per pixel e = |lum(a) - lum(b)| /
// (lum(b) + eps) with lum in fp64 of the fp32 pixels; per-block sums of e^2 in
// a fixed-order tree, finished on the host in block order.
__global__ void k_rrmse_partial(const double *film, const float *ref, int npix, double scale, double eps,
                                double *out) {
    __shared__ double s[256];
    int i = blockIdx.x * 256 + threadIdx.x;
    double e2 = 0.0;
    if (i < npix) {
        double a0 = static_cast<float>(film[3 * i] * scale), a1 = static_cast<float>(film[3 * i + 1] * scale),
               a2 = static_cast<float>(film[3 * i + 2] * scale);
        double b0 = ref[3 * i], b1 = ref[3 * i + 1], b2 = ref[3 * i + 2];
        double la = 0.2126 * a0 + 0.7152 * a1 + 0.0722 * a2;
        double lb = 0.2126 * b0 + 0.7152 * b1 + 0.0722 * b2;
        double e = ::fabs(la - lb) / (lb + eps);
        e2 = e * e;
    }
    s[threadIdx.x] = e2;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if (static_cast<int>(threadIdx.x) < w)
            s[threadIdx.x] += s[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0)
        out[blockIdx.x] = s[0];
}

}  // namespace rd

// ---- cooperative persistent step kernel (adaptive strategies, small chain counts) ----------
#include <cooperative_groups.h>

namespace rd {

// Literal adaptation for one lockstep step by one 128-thread block: tiles of
// 1024 chains in order (core/adaptation.cpp:60-92 applied in canonical order).
//  * single-region tiles (Global, or a quadtree before its first split): the
//    visits are compacted in chain order by a block scan; complete batches of L
//    are summed in parallel (each sequentially, the first continuing from the
//    pending sum); one thread runs the lambda recurrence over the batches while
//    another accumulates the lifetime tally sequentially;
//  * multi-region tiles: stable radix sort by region over just the key bits in
//    use, then each region's run is processed sequentially by its head thread.
struct LiteralSmem {
    typedef cub::BlockRadixSort<int, 128, 8, int> Sort;
    typedef cub::BlockScan<int, 128> Scan;
    typedef cub::BlockReduce<int, 128> Reduce;
    union {
        typename Sort::TempStorage tmp;
        typename Scan::TempStorage scan;
        typename Reduce::TempStorage red;
        struct {
            int k[1024];
            int v[1024];
            double a[1024];
        } d;
    };
    double bsum[1024 / 1 + 1];
    double bstep[1024 / 1 + 1];   // gamma(n + b) * sgn(alpha_hat_b - target) per complete batch
    double bah[1024 / 1 + 1];
    int rmin, rmax, cnt;
};

template <class R>
__device__ void adapt_literal_block(LiteralSmem &sm, const int *vreg, const double *va, int C, long long chain_off,
                                    long long C_total, unsigned long long span_start, int j, RegionArrays ra,
                                    KernTab<R> *ktab, const AdaptCfg &cfg, const TraceBuf &tb, int key_bits) {
    const int t = threadIdx.x;
    for (int base = 0; base < C; base += 1024) {
        int key[8], val[8], flag[8];
        int lo = 0x7fffffff, hi = -1, nv = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            int ci = base + t * 8 + q;
            int r = (ci < C) ? __ldcg(&vreg[ci]) : -1;
            key[q] = r;
            val[q] = ci;
            flag[q] = r >= 0;
            if (r >= 0) {
                lo = min(lo, r);
                hi = max(hi, r);
                ++nv;
            }
        }
        int blo = LiteralSmem::Reduce(sm.red).Reduce(lo, cub::Min());
        __syncthreads();
        int bhi = LiteralSmem::Reduce(sm.red).Reduce(hi, cub::Max());
        __syncthreads();
        if (t == 0) {
            sm.rmin = blo;
            sm.rmax = bhi;
        }
        __syncthreads();
        if (sm.rmax < 0) {   // no visits in this tile
            __syncthreads();
            continue;
        }
        if (sm.rmin == sm.rmax) {
            // ---- single region: compact in chain order ----
            const int r = sm.rmin;
            int pos[8];
            int total;
            LiteralSmem::Scan(sm.scan).ExclusiveSum(flag, pos, total);
            __syncthreads();
#pragma unroll
            for (int q = 0; q < 8; ++q)
                if (flag[q]) {
                    sm.d.a[pos[q]] = __ldcg(&va[val[q]]);
                    sm.d.v[pos[q]] = val[q];
                }
            if (t == 0)
                sm.cnt = total;
            __syncthreads();
            const int m = sm.cnt;
            const int L = cfg.L;
            const unsigned pn0 = ra.pend_n[r];
            const double ps0 = ra.pend_sum[r];
            const int first_len = L - static_cast<int>(pn0);   // visits that complete batch 0
            const int nb = m >= first_len ? 1 + (m - first_len) / L : 0;   // complete batches
            // batch b covers [s_b, e_b): s_0 = 0, e_0 = first_len, then L each
            for (int b = t; b <= nb; b += 128) {
                int sb = b == 0 ? 0 : first_len + (b - 1) * L;
                int eb = b == 0 ? min(m, first_len) : min(m, sb + L);
                double acc = b == 0 ? ps0 : 0.0;
                for (int q = sb; q < eb; ++q)
                    acc += sm.d.a[q];
                sm.bsum[b] = acc;
                if (b < nb) {
                    // the lambda-independent half of update_lambda (adaptation.cpp:15-20)
                    double ah = acc / static_cast<unsigned>(L);
                    ah = ah < 0.0 ? 0.0 : (ah > 1.0 ? 1.0 : ah);
                    double gs = cfg.gscale / ::sqrt(static_cast<double>(ra.n[r] + static_cast<unsigned long long>(b)));
                    double gm = cfg.gmax < gs ? cfg.gmax : gs;
                    double diff = ah - cfg.target;
                    double sg = diff > 0.0 ? 1.0 : (diff < 0.0 ? -1.0 : 0.0);
                    sm.bstep[b] = gm * sg;   // exact: sg is -1, 0 or 1
                    sm.bah[b] = ah;
                }
            }
            __syncthreads();
            if (t == 0) {
                double lam = ra.lambda[r];
                unsigned long long n = ra.n[r];
                for (int b = 0; b < nb; ++b) {
                    double ah = sm.bah[b];
                    unsigned long long n0 = n;
                    double nl = lam + sm.bstep[b];
                    lam = cfg.lmin > nl ? cfg.lmin : nl;
                    n = n0 + 1;
                    if (cfg.trace) {
                        int last = first_len + b * L - 1;
                        trace_push(tb, span_start + static_cast<unsigned long long>(j) * C_total + chain_off +
                                           sm.d.v[last], r, n0, lam, ah);
                    }
                }
                // leftover partial batch (sequential partial sum of batch nb)
                int lead = nb == 0 ? m : m - (first_len + (nb - 1) * L);
                ra.pend_n[r] = nb == 0 ? pn0 + static_cast<unsigned>(m) : static_cast<unsigned>(lead);
                ra.pend_sum[r] = sm.bsum[nb];
                if (nb > 0) {
                    ra.lambda[r] = lam;
                    ra.n[r] = n;
                    set_ktab(&ktab[r], lam, cfg.ratio);
                }
            } else if (t == 32) {
                double ta = ra.tot_acc[r];
                for (int q = 0; q < m; ++q)
                    ta += sm.d.a[q];
                ra.tot_acc[r] = ta;
                ra.tot_vis[r] += static_cast<unsigned long long>(m);
            }
            __syncthreads();
            continue;
        }
        // ---- several regions: stable sort over the bits in use ----
#pragma unroll
        for (int q = 0; q < 8; ++q)
            key[q] = key[q] >= 0 ? key[q] : ((1 << key_bits) - 1);
        LiteralSmem::Sort(sm.tmp).Sort(key, val, 0, key_bits);
        __syncthreads();
        const int none = (1 << key_bits) - 1;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            sm.d.k[t * 8 + q] = key[q];
            sm.d.v[t * 8 + q] = val[q];
            sm.d.a[t * 8 + q] = key[q] != none ? __ldcg(&va[val[q]]) : 0.0;
        }
        __syncthreads();
        for (int p = t; p < 1024; p += 128) {
            int r = sm.d.k[p];
            if (r == none || (p > 0 && sm.d.k[p - 1] == r))
                continue;
            double lam = ra.lambda[r];
            unsigned long long n = ra.n[r];
            unsigned int pn = ra.pend_n[r];
            double ps = ra.pend_sum[r];
            unsigned long long tv = ra.tot_vis[r];
            double ta = ra.tot_acc[r];
            bool changed = false;
            for (int q = p; q < 1024 && sm.d.k[q] == r; ++q) {
                double a = sm.d.a[q];
                ta += a;
                tv += 1;
                ps += a;
                pn += 1;
                if (pn < static_cast<unsigned int>(cfg.L))
                    continue;
                double ah = ps / pn;
                ah = ah < 0.0 ? 0.0 : (ah > 1.0 ? 1.0 : ah);
                unsigned long long n0 = n;
                lam = lambda_next(lam, ah, n0, cfg);
                n = n0 + 1;
                pn = 0;
                ps = 0.0;
                changed = true;
                if (cfg.trace)
                    trace_push(tb, span_start + static_cast<unsigned long long>(j) * C_total + chain_off + sm.d.v[q], r,
                               n0, lam, ah);
            }
            ra.lambda[r] = lam;
            ra.n[r] = n;
            ra.pend_n[r] = pn;
            ra.pend_sum[r] = ps;
            ra.tot_vis[r] = tv;
            ra.tot_acc[r] = ta;
            if (changed)
                set_ktab(&ktab[r], lam, cfg.ratio);
        }
        __syncthreads();
        (void)nv;
    }
}

template <class R> struct CoopArgs {
    KernTab<R> *ktab;   // writable view of P.ktab
    AdaptCfg cfg;
    TraceBuf tb;
    int pooled;
    int key_bits;       // radix-sort bits covering region ids + one sentinel
};

// All lockstep steps [j0, j1) of a span in one cooperative launch: every group
// keeps its chain in registers; after each step a grid-wide barrier, the
// adaptation update (block 0 for the literal rule, the whole grid for the
// pooled rule), another barrier.  Same semantics as k_step + k_adapt_* per step.
template <class R, int RK, int G>
__global__ void __launch_bounds__(128) k_step_coop(StepParams<R> P, CoopArgs<R> A) {
    namespace cg = cooperative_groups;
    extern __shared__ __align__(16) char smem[];
    __shared__ LiteralSmem lit;
    cg::grid_group grid = cg::this_grid();
    SceneView<R> S = stage_scene(P.scene, smem);
    Group<G> g;
    const long long tid = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int c = static_cast<int>(tid / Lanes<G>::n);
    const bool active = c < P.C;
    const long long gc = P.chain_off + c;
    const unsigned long long my_steps = P.per + (static_cast<unsigned long long>(gc) < P.rem ? 1ull : 0ull);

    ChainRegs<R> cs;
    Rng<RK> rng;
    RayCount rc;
    if (active) {
        cs.k = P.ch.klen[c];
        cs.sm = P.ch.smask[c];
        cs.f = mk(P.ch.cf[c], P.ch.cf[P.C + c], P.ch.cf[2 * P.C + c]);
        cs.pi = P.ch.cf[3 * P.C + c];
        cs.ru = P.ch.cr[c];
        cs.rv = P.ch.cr[P.C + c];
        cs.eyeden = P.ch.eyeden[c];
        cs.acc = P.ch.acc[c];
        cs.iacc = P.ch.iacc[c];
        cs.lum = P.ch.lum[c];
        cs.npert = P.ch.npert[c];
        cs.nlarge = P.ch.nlarge[c];
        cs.ipert = P.ch.ipert[c];
        cs.nsteps = P.ch.nsteps[c];
        RngIO<RK>::load(rng, P.ch.rng0, P.ch.rng1, c, P.seed, static_cast<unsigned long long>(gc));
    }
    for (int j = P.j0; j < P.j1; ++j) {
        if (active) {
            if (static_cast<unsigned long long>(j) < my_steps) {
                unsigned long long index = P.span_start + static_cast<unsigned long long>(j) * P.C_total + gc;
                mutate<R, RK, G>(P, S, c, gc, index, cs, rng, g, rc);
            } else if (g.lane == 0) {
                P.ch.vreg[c] = -1;
            }
        }
        grid.sync();
        if (!A.pooled) {
            if (blockIdx.x == 0)
                adapt_literal_block<R>(lit, P.ch.vreg, P.ch.va, P.C, P.chain_off, P.C_total, P.span_start, j, P.reg,
                                       A.ktab, A.cfg, A.tb, A.key_bits);
            grid.sync();
        } else {
            // pooled: accumulate (one thread per chain) ...
            if (tid < P.C) {
                int r = __ldcg(&P.ch.vreg[tid]);
                if (r >= 0) {
                    unsigned long long fx = to_fx(__ldcg(&P.ch.va[tid]));
                    unsigned long long idx =
                        P.span_start + static_cast<unsigned long long>(j) * P.C_total + P.chain_off + tid;
                    atomicAdd(&P.reg.x_cnt[r], 1ull);
                    atomicAdd(&P.reg.x_fx[r], fx);
                    atomicMax(&P.reg.x_last[r], idx);
                    if (atomicExch(&P.reg.x_touched[r], 1u) == 0u) {
                        unsigned slot = atomicAdd(P.reg.n_touched, 1u);
                        P.reg.touched_list[slot] = static_cast<unsigned>(r);
                    }
                }
            }
            grid.sync();
            // ... then one update per touched region
            unsigned nt = __ldcg(P.reg.n_touched);
            for (unsigned i = static_cast<unsigned>(tid); i < nt; i += gridDim.x * blockDim.x) {
                RegionArrays ra = P.reg;
                int r = static_cast<int>(ra.touched_list[i]);
                unsigned long long cnt = ra.x_cnt[r], fx = ra.x_fx[r], last = ra.x_last[r];
                ra.x_cnt[r] = 0;
                ra.x_fx[r] = 0;
                ra.x_last[r] = 0;
                ra.x_touched[r] = 0;
                ra.tot_vis[r] += cnt;
                ra.tot_fx[r] += fx;
                unsigned long long pn = ra.pend_n[r] + cnt;
                unsigned long long pf = ra.pend_fx[r] + fx;
                if (pn < static_cast<unsigned long long>(A.cfg.L)) {
                    ra.pend_n[r] = static_cast<unsigned>(pn);
                    ra.pend_fx[r] = pf;
                    continue;
                }
                double ah = static_cast<double>(pf) / 16777216.0 / static_cast<double>(pn);
                ah = ah < 0.0 ? 0.0 : (ah > 1.0 ? 1.0 : ah);
                unsigned long long n0 = ra.n[r];
                double lam = lambda_next(ra.lambda[r], ah, n0, A.cfg);
                ra.lambda[r] = lam;
                ra.n[r] = n0 + 1;
                ra.pend_n[r] = 0;
                ra.pend_fx[r] = 0;
                set_ktab(&A.ktab[r], lam, A.cfg.ratio);
                if (A.cfg.trace)
                    trace_push(A.tb, last, r, n0, lam, ah);
            }
            grid.sync();
            if (tid == 0)
                *P.reg.n_touched = 0;
        }
    }
    if (active && g.lane == 0) {
        P.ch.klen[c] = cs.k;
        P.ch.smask[c] = cs.sm;
        P.ch.cf[c] = cs.f.x;
        P.ch.cf[P.C + c] = cs.f.y;
        P.ch.cf[2 * P.C + c] = cs.f.z;
        P.ch.cf[3 * P.C + c] = cs.pi;
        P.ch.cr[c] = cs.ru;
        P.ch.cr[P.C + c] = cs.rv;
        P.ch.eyeden[c] = cs.eyeden;
        P.ch.acc[c] = cs.acc;
        P.ch.iacc[c] = cs.iacc;
        P.ch.lum[c] = cs.lum;
        P.ch.npert[c] = cs.npert;
        P.ch.nlarge[c] = cs.nlarge;
        P.ch.ipert[c] = cs.ipert;
        P.ch.nsteps[c] = cs.nsteps;
        RngIO<RK>::store(rng, P.ch.rng0, P.ch.rng1, c);
    }
    unsigned act = __activemask();
    unsigned sc = __reduce_add_sync(act, g.lane == 0 ? static_cast<unsigned>(rc.c) : 0u);
    unsigned sv = __reduce_add_sync(act, g.lane == 0 ? static_cast<unsigned>(rc.v) : 0u);
    if ((threadIdx.x & 31) == __ffs(act) - 1) {
        atomicAdd(&P.ch.rays[0], static_cast<unsigned long long>(sc));
        atomicAdd(&P.ch.rays[1], static_cast<unsigned long long>(sv));
    }
}

}  // namespace rd
