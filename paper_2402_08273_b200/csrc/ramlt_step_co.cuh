// ramlt_step_co.cuh -- the divergence-free chain-step kernel (one chain per lane).
//
// The reference's mutation (core/driver.cpp:113-171) is written as a
// resumable coroutine (protothread style: every variable that lives across a
// ray cast is a member, and `CO_RAY` returns to the caller with a pending ray
// and resumes at the same point).  The kernel loop then alternates
//   (1) converged:  warp-aggregated work stealing -- idle lanes take the next
//                   chain from a global counter (one atomic per warp),
//   (2) divergent:  every lane advances its coroutine until its next ray cast
//                   (or the end of its chain's steps),
//   (3) converged:  every lane with a pending ray traces it with the uniform
//                   smem-broadcast primitive loop -- the expensive part, now
//                   executed by (nearly) full warps whatever phase each chain is
//                   in (perturbation replay, large-step bounce, visibility).
// Arithmetic and RNG consumption are identical to `mutate` (ramlt_kernels.cuh),
// so the fp64/PCG build stays bit-exact with the reference.
#pragma once

#include "ramlt_kernels.cuh"

namespace rd {

template <class R> struct RayReq {
    V3<R> o, d;
    R lim;   // +inf: closest hit; dist - eps: visibility (occluded iff some t < lim)
};

// Closest hit below `lim` over spheres then triangles (core/scene.cpp:57-92);
// ties resolved to the lowest primitive index exactly as the reference loop.
template <class R, bool BVH>
__device__ __forceinline__ int trace_ray(const SceneView<R> &s, const RayReq<R> &r, R &t_out) {
    if constexpr (BVH) {
        R best = r.lim;
        int key = -1, spos = -1;   // a hit at exactly t == lim is not below lim
        for (int i = 0; i < s.nsph; ++i) {
            R t;
            if (hit_sphere(s.sph[i], r.o, r.d, t) && t < best) {
                best = t;
                key = i;
                spos = i;
            }
        }
        int tpos = bvh_trace(s, r.o, r.d, best, best, key, false);
        t_out = best;
        return tpos >= 0 ? s.nsph + tpos : spos;   // hit_record indexes s.tri by position
    } else {
    R best = r.lim;
    int bi = -1;
    for (int i = 0; i < s.nsph; ++i) {
        R t;
        if (hit_sphere(s.sph[i], r.o, r.d, t) && t < best) {
            best = t;
            bi = i;
        }
    }
    scan_tris(s.tri, 0, s.ntri, 1, r.o, r.d, best, bi, s.nsph);
    t_out = best;
    return bi;
    }
}

template <class R> __device__ __forceinline__ void hit_record(const SceneView<R> &s, const RayReq<R> &r, int prim,
                                                             R t, Hit<R> &h) {
    h.t = t;
    h.p = add(r.o, scl(r.d, t));
    if (prim < s.nsph) {
        const SphD<R> &sp = s.sph[prim];
        h.n = unit(sub(h.p, sp.c));
        h.mat = sp.mat;
        h.emi = sp.emi;
    } else {
        const TriD<R> &tr = s.tri[prim - s.nsph];
        h.n = tr.n;
        h.mat = tr.mat;
        h.emi = tr.emi;
    }
}

// Proposal path storage in shared memory: vertex i of lane t at pv[i*B + t].
template <class R> struct PvSmem {
    GV<R> *base;
    int stride;
    __device__ __forceinline__ Vx<R> get(int i) const;
    __device__ __forceinline__ void set(int i, const Vx<R> &v) const;
};
template <> __device__ __forceinline__ Vx<float> PvSmem<float>::get(int i) const {
    GV<float> g = base[i * stride];
    Vx<float> v;
    v.p = mk(g.a.x, g.a.y, g.a.z);
    v.n = mk(g.a.w, g.b.x, g.b.y);
    unpack_meta(__float_as_uint(g.b.z), v);
    return v;
}
template <> __device__ __forceinline__ void PvSmem<float>::set(int i, const Vx<float> &v) const {
    GV<float> g;
    g.a = make_float4(v.p.x, v.p.y, v.p.z, v.n.x);
    g.b = make_float4(v.n.y, v.n.z, __uint_as_float(pack_meta(v.mat, v.emi, v.spec, v.ev)), 0.f);
    base[i * stride] = g;
}
template <> __device__ __forceinline__ Vx<double> PvSmem<double>::get(int i) const {
    const GV<double> &g = base[i * stride];
    Vx<double> v;
    v.p = mk(g.a.x, g.a.y, g.b.x);
    v.n = mk(g.b.y, g.c.x, g.c.y);
    unpack_meta(static_cast<uint32_t>(g.meta), v);
    return v;
}
template <> __device__ __forceinline__ void PvSmem<double>::set(int i, const Vx<double> &v) const {
    GV<double> &g = base[i * stride];
    g.a = make_double2(v.p.x, v.p.y);
    g.b = make_double2(v.p.z, v.n.x);
    g.c = make_double2(v.n.y, v.n.z);
    g.meta = static_cast<long long>(pack_meta(v.mat, v.emi, v.spec, v.ev));
}

// Proposal = smem head [0..head_end] + current-path tail.
template <class R> struct PropS {
    PvSmem<R> pv;
    int head_end;
    const CurPathV<R> *cur;
    __device__ __forceinline__ Vx<R> get(int i) const { return i <= head_end ? pv.get(i) : cur->get(i); }
};

enum { CO_RAY_PENDING = 1, CO_STEP_DONE = 2 };

// Where a coroutine's rays go.  NoSink: one pending ray at a time in `ray`, traced by
// the caller (k_step_co).  A batching sink (ramlt_wavefront.cuh, BATCH = true) takes
// the rays itself -- reserve(n) slots, put(slot, o, d, lim, k) -- so the independent
// visibility rays of eval_contribution / eye_path_density leave in ONE yield
// (ordinal k, answered by occluded(k)) instead of one yield per segment.
struct NoSink {
    static constexpr bool BATCH = false;
    // never called (BATCH is false); present so both arms of `if (Sink::BATCH)` compile
    // -- a case label may not sit inside an `if constexpr` block
    __device__ __forceinline__ unsigned reserve(unsigned) const { return 0u; }
    template <class V, class T> __device__ __forceinline__ void put(unsigned, V, V, T, int) const {}
    __device__ __forceinline__ void null(unsigned) const {}
    __device__ __forceinline__ void begin_batch() const {}
    __device__ __forceinline__ bool occluded(int) const { return false; }
    __device__ __forceinline__ void cold() const {}
};

#define CO_RAY(O, D, LIM, N)                                                                       \
    do {                                                                                           \
        ray.o = (O);                                                                               \
        ray.d = (D);                                                                               \
        ray.lim = (LIM);                                                                           \
        pc = (N);                                                                                  \
        if constexpr (Sink::BATCH)                                                                 \
            sink.put(sink.reserve(1u), ray.o, ray.d, ray.lim, 0);                                  \
        return CO_RAY_PENDING;                                                                     \
    case (N):;                                                                                     \
    } while (0)

// One iteration of trace_eye_subpath's loop (path.cpp:84-142) once the closest hit of the
// pending ray is known: record the vertex, extend the transition density, sample the
// continuation.  Returns true when the path continues with the ray (o, d); false when the
// loop ends (miss, emitter reached -- ok --, path capacity, no continuation).  Shared by the
// coroutine (StepCo::advance) and the wavefront's bounce kernel (k_wf_bounce).
template <class R, int RK>
__device__ __forceinline__ bool bounce_body(const StepParams<R> &P, const SceneView<R> &S, const PvSmem<R> &pv,
                                            const RayReq<R> &ray, int res_prim, R res_t, Rng<RK> &rng, R &dpdf,
                                            int &kp, unsigned &smp, double &tf, bool &ok, V3<R> &o, V3<R> &d) {
    d = ray.d;
    if (res_prim < 0)
        return false;
    Hit<R> h;
    hit_record(S, ray, res_prim, res_t, h);
    const MatD<R> mt = S.mat[h.mat];
    Vx<R> x;
    x.p = h.p;
    x.n = h.n;
    x.mat = h.mat;
    x.emi = h.emi;
    x.spec = h.emi < 0 && (mt.kind == MAT_MIRROR || mt.kind == MAT_DIELECTRIC);
    x.ev = EV_NONE;
    tf *= static_cast<double>(dpdf * (M<R>::abs(dot(h.n, d)) / (h.t * h.t)));
    if (x.spec)
        smp |= 1u << kp;
    if (h.emi >= 0) {
        pv.set(kp, x);
        ++kp;
        ok = true;
        return false;
    }
    if (kp + 1 >= P.maxv) {
        pv.set(kp, x);
        ++kp;
        return false;
    }
    BS<R> bs;
    if (!bsdf_sample(mt, neg(d), h.n, rng, bs) || bs.zero_thr) {
        pv.set(kp, x);
        ++kp;
        return false;
    }
    x.ev = bs.ev;
    pv.set(kp, x);
    ++kp;
    o = h.p;
    d = bs.dir;
    dpdf = bs.pdf;
    return true;
}

// INIT: the same coroutine runs chain initialisation (core/driver.cpp:219-242):
// large-step eye paths from the chain's init stream until one has a nonzero
// contribution, then the chain's state is written (as init_chain does).
// The chain's persistent state the coroutine carries (ChainRegs without the
// per-chain tallies: those are read-modify-written in HBM at the step's end,
// which keeps the local-memory coroutine state 56 B smaller).
template <class R> struct ChainCo {
    int k;
    unsigned sm;
    V3<R> f;
    R pi, ru, rv;
    double eyeden;
};

template <class R, int RK, bool INIT = false> struct StepCo {
    // ---- hot: everything the large-step bounce loop (yield point 2) reads or writes.
    // The wavefront step (ramlt_wavefront.cuh) moves only these leading sectors for a
    // chain resumed in that loop and fetches the rest when the chain leaves it.
    int c;
    int pc;
    int wf_j, wf_jend;              // wavefront: the chain's step cursor within the launch
    Rng<RK> rng;
    RayReq<R> ray;
    int res_prim;   // -1 miss / visible
    R res_t;
    R dpdf;
    int kp;
    unsigned smp;
    double tf;                      // transition densities and acceptance: fp64 in every build
    bool choose, ok, accepted, pert_rec;
    unsigned attempts;              // INIT (init_attempts < 2^32)
    // ---- cold (32-byte aligned: no sector holds both hot and cold fields) ----
    alignas(32) ChainCo<R> cs;      // chain state that persists over the chain's steps
    R s_pert;
    double tr, a;
    int endpoint, first, idx, next, i, region, head_end;
    unsigned pmask, m;
    V3<R> o, d;
    Contrib<R> pcb;
    // evaluate / eye density sub-state
    V3<R> ef;
    double ep;
    R eseg;
    int ek, ei;

    template <class Sink = NoSink>
    __device__ __forceinline__ int advance(const StepParams<R> &P, const SceneView<R> &S, const PvSmem<R> &pv,
                                           RayCount &rc, unsigned long long index, Sink sink = Sink{});

    // Batching sinks: every visibility ray eval_contribution can ask for (segments
    // 0..endpoint of a perturbation, all segments of a large step), in segment order;
    // stops at the first segment whose geometry ends the evaluation.  Returns the
    // slots reserved (unused ones are null rays).
    template <class Sink>
    __device__ __forceinline__ int emit_eval_rays(const CurPathV<R> &cur, const PvSmem<R> &pv, Sink &sink) const {
        const int nseg = ek - 1;
        const int nmax = choose ? min(nseg, endpoint + 1) : nseg;
        if (nmax <= 0)
            return 0;
        const unsigned base = sink.reserve(static_cast<unsigned>(nmax));
        sink.begin_batch();
        PropS<R> prop{pv, head_end, &cur};
        int nb = 0;
        for (int e = 0; e < nmax; ++e) {
            Vx<R> av = prop.get(e);
            Vx<R> bv = prop.get(e + 1);
            if (e > 0 && av.emi >= 0)
                break;
            V3<R> dd = sub(bv.p, av.p);
            R d2 = dot(dd, dd);
            if (d2 <= R(0))
                break;
            V3<R> dir = dvs(dd, M<R>::sqrt(d2));
            R sg = av.spec ? M<R>::abs(dot(bv.n, dir)) / d2
                           : M<R>::abs(dot(av.n, dir)) * M<R>::abs(dot(bv.n, dir)) / d2;
            if (sg <= R(0))
                break;
            R dist = len(dd);
            if (dist <= R(2) * R(kEpsD))
                break;
            sink.put(base + static_cast<unsigned>(nb), av.p, dvs(dd, dist), dist - R(kEpsD), nb);
            ++nb;
        }
        for (int q = nb; q < nmax; ++q)
            sink.null(base + static_cast<unsigned>(q));
        return nmax;
    }
    // The visibility rays of eye_path_density(current path), in segment order.
    template <class Sink>
    __device__ __forceinline__ int emit_eyeden_rays(const CurPathV<R> &cur, Sink &sink) const {
        const int nseg = cs.k - 1;
        if (nseg <= 0)
            return 0;
        const unsigned base = sink.reserve(static_cast<unsigned>(nseg));
        sink.begin_batch();
        int nb = 0;
        for (int e = 0; e < nseg; ++e) {
            Vx<R> av = cur.get(e);
            Vx<R> bv = cur.get(e + 1);
            if (e > 0 && av.emi >= 0)
                break;
            V3<R> dd = sub(bv.p, av.p);
            R d2 = dot(dd, dd);
            R cval = R(0);
            if (d2 > R(0)) {
                V3<R> dir = dvs(dd, M<R>::sqrt(d2));
                cval = M<R>::abs(dot(bv.n, dir)) / d2;
            }
            if (cval <= R(0))
                break;
            R dist = len(dd);
            if (dist <= R(2) * R(kEpsD))
                break;
            sink.put(base + static_cast<unsigned>(nb), av.p, dvs(dd, dist), dist - R(kEpsD), nb);
            ++nb;
        }
        for (int q = nb; q < nseg; ++q)
            sink.null(base + static_cast<unsigned>(q));
        return nseg;
    }

    // INIT: write the found path (vertices 1..kp-1, contribution) and the
    // chain's fresh counters and step stream -- what init_chain stores.
    __device__ __forceinline__ void init_commit(const StepParams<R> &P, const PvSmem<R> &pv) {
        if (pcb.pi > R(0)) {
            for (int q = 1; q < kp; ++q)
                store_gv(&P.ch.verts[static_cast<size_t>(q - 1) * P.C + c], pv.get(q));
            P.ch.klen[c] = kp;
            P.ch.smask[c] = smp;
            P.ch.cf[c] = pcb.f.x;
            P.ch.cf[P.C + c] = pcb.f.y;
            P.ch.cf[2 * P.C + c] = pcb.f.z;
            P.ch.cf[3 * P.C + c] = pcb.pi;
            P.ch.cr[c] = pcb.u;
            P.ch.cr[P.C + c] = pcb.v;
        }
        P.ch.eyeden[c] = __longlong_as_double(0x7ff8000000000000LL);
        P.ch.acc[c] = 0.0;
        P.ch.iacc[c] = 0.0;
        P.ch.lum[c] = 0.0;
        P.ch.npert[c] = 0;
        P.ch.nlarge[c] = 0;
        P.ch.ipert[c] = 0;
        P.ch.nsteps[c] = 0;
        Rng<RK> fresh;
        fresh.reseed(P.seed, static_cast<unsigned long long>(P.chain_off + c));
        RngIO<RK>::store(fresh, P.ch.rng0, P.ch.rng1, c);
    }
};

template <class R, int RK, bool INIT>
template <class Sink>
__device__ __forceinline__ int StepCo<R, RK, INIT>::advance(const StepParams<R> &P, const SceneView<R> &S,
                                                      const PvSmem<R> &pv, RayCount &rc,
                                                      unsigned long long index, Sink sink) {
    CurPathV<R> cur{P.ch.verts, P.C, c, S.cam.pos, S.cam.fwd};
    switch (pc) {
    case 0: {
        if constexpr (INIT) {
            choose = false;
            s_pert = R(0);
            a = 0.0;
            region = -1;
            head_end = 0;
            goto init_attempt;
        }
        {
            // suitability (core/mutations.cpp:47-56) and strategy selection (driver.cpp:115-116)
            bool elig;
            if (P.pk == 0) {
                endpoint = lens_endpoint(cs.k, cs.sm);
                elig = endpoint >= 0;
                pmask = 1u;
                first = 0;
            } else {
                elig = mc_structure(cs.k, cs.sm, first, endpoint, pmask);
            }
            s_pert = elig ? R(0.5) : R(0);
            choose = elig && Unit<R>::draw(rng) < s_pert;
        }
        a = 0.0;
        pcb.pi = R(0);
        region = -1;
        ok = false;
        pert_rec = false;
        kp = cs.k;
        smp = cs.sm;
        head_end = 0;
        if (!choose)
            goto large_step;
        {
            // classify_path (driver.cpp:95-107)
            R cu = R(0), cv = R(0);
            if (P.ctl == 2 && P.pk == 1)
                cylindrical(pdir<R>(cur, first), cu, cv);
            region = P.ctl == 2 ? classify(P.part, cs.ru, cs.rv, cu, cv) : 0;
            pv.set(0, cur.get(0));
        }
        // lens_perturb / multichain_perturb (mutations.cpp:122-174)
        m = pmask;
        ok = true;
        while (m) {
            idx = __ffs(m) - 1;
            m &= m - 1;
            next = m ? (__ffs(m) - 1) : endpoint;
            {
                const KernTab<R> kt = P.ktab[region];
                d = perturb_dir(pdir<R>(cur, idx), idx == 0 ? kt.k1 : kt.k2, rng);
                o = pv.get(idx).p;
            }
            // retrace_chain (mutations.cpp:78-110)
            for (i = idx + 1; i <= next; ++i) {
                ++rc.c;
                CO_RAY(o, d, M<R>::inf(), 1);
                {
                    if (res_prim < 0) {
                        ok = false;
                        break;
                    }
                    Hit<R> h;
                    hit_record(S, ray, res_prim, res_t, h);
                    Vx<R> r = cur.get(i);
                    const MatD<R> mt = S.mat[h.mat];
                    bool he = h.emi >= 0;
                    bool hs = !he && (mt.kind == MAT_MIRROR || mt.kind == MAT_DIELECTRIC);
                    if (he != (r.emi >= 0) || hs != r.spec) {
                        ok = false;
                        break;
                    }
                    Vx<R> x;
                    x.p = h.p;
                    x.n = h.n;
                    x.mat = h.mat;
                    x.emi = h.emi;
                    x.spec = hs;
                    x.ev = r.ev;
                    pv.set(i, x);
                    if (i == next)
                        break;
                    V3<R> cn;
                    if (!spec_cont(mt, neg(d), h.n, r.ev, cn)) {
                        ok = false;
                        break;
                    }
                    o = h.p;
                    d = cn;
                }
            }
            if (!ok)
                break;
        }
        if (!ok)
            goto pert_record;
        head_end = endpoint;
        {
            const KernTab<R> kt = P.ktab[region];
            PropS<R> prop{pv, head_end, &cur};
            tf = pert_density(cur, prop, pmask, endpoint, kt.k1, kt.k2);
            tr = pert_density(prop, cur, pmask, endpoint, kt.k1, kt.k2);
        }
        ek = cs.k;
        goto eval_start;

    large_step:
    init_attempt:
        pcb.pi = R(0);
        // trace_eye_subpath (path.cpp:84-142) -- large_step (mutations.cpp:58-71)
        {
            Vx<R> cv;
            cv.p = S.cam.pos;
            cv.n = S.cam.fwd;
            cv.mat = -1;
            cv.emi = -1;
            cv.spec = false;
            cv.ev = EV_NONE;
            pv.set(0, cv);
            kp = 1;
            smp = 0;
            tf = 1.0;
            ok = false;
            if (P.maxv < 2)
                goto finish;
            R u = Unit<R>::draw(rng);
            R v = Unit<R>::draw(rng);
            d = cam_primary(S.cam, u, v);
            dpdf = cam_dir_pdf(S.cam, d);
            o = S.cam.pos;
        }
        while (kp < P.maxv) {
            ++rc.c;
            CO_RAY(o, d, M<R>::inf(), 2);
            // (o, d are cold: a chain resumed here may hold the hot fields only; the body
            // takes the incoming direction from the ray)
            if (!bounce_body<R, RK>(P, S, pv, ray, res_prim, res_t, rng, dpdf, kp, smp, tf, ok, o, d))
                break;
        }
    case 7:   // wavefront: the loop ran in k_wf_bounce, the chain resumes behind it
        sink.cold();   // leaving the bounce loop: the rest of the state is needed from here on
        if (!ok)
            goto finish;
        head_end = kp - 1;
        ek = kp;

    eval_start:
        // eval_contribution (path.cpp:40-82) over the proposal
        {
            PropS<R> prop{pv, head_end, &cur};
            pcb.pi = R(0);
            Vx<R> last = prop.get(ek - 1);
            if (ek < 2 || last.emi < 0)
                goto eval_done;
            V3<R> w0 = pdir<R>(prop, 0);
            R ru, rv;
            if (!cam_raster(S.cam, w0, ru, rv))
                goto eval_done;
            pcb.u = ru;
            pcb.v = rv;
            R imp = cam_importance(S.cam, w0);
            ef = mk(imp, imp, imp);
        }
        if (Sink::BATCH) {   // all the segments' visibility rays in one yield
            if (emit_eval_rays(cur, pv, sink) > 0) {
                pc = 5;
                return CO_RAY_PENDING;
            }
        case 5:
            i = 0;   // ordinal of the next answer
        }
        for (ei = 0; ei + 1 < ek; ++ei) {
            {
                PropS<R> prop{pv, head_end, &cur};
                Vx<R> av = prop.get(ei);
                Vx<R> bv = prop.get(ei + 1);
                if (ei > 0 && av.emi >= 0)
                    goto eval_fail;
                // geometry_term / area_conversion (path.cpp:7-29) up to the visibility test
                V3<R> dd = sub(bv.p, av.p);
                R d2 = dot(dd, dd);
                if (d2 <= R(0))
                    goto eval_fail;
                V3<R> dir = dvs(dd, M<R>::sqrt(d2));
                eseg = av.spec ? M<R>::abs(dot(bv.n, dir)) / d2
                               : M<R>::abs(dot(av.n, dir)) * M<R>::abs(dot(bv.n, dir)) / d2;
                if (eseg <= R(0))
                    goto eval_fail;
                // unchanged tail segment of a perturbation: visibility already held
                // for the current path (pi > 0), so no ray (see evaluate)
                if (choose && ei > endpoint)
                    goto eval_seg_visible;
                ++rc.v;
                // visible(a, b) (scene.cpp:94-102)
                R dist = len(dd);
                if (dist <= R(2) * R(kEpsD))
                    goto eval_fail;
                o = av.p;
                d = dvs(dd, dist);
                ray.lim = dist - R(kEpsD);
            }
            if (Sink::BATCH) {
                if (sink.occluded(i++))
                    goto eval_fail;
            } else {
                CO_RAY(o, d, ray.lim, 3);
                if (res_prim >= 0)
                    goto eval_fail;
            }
        eval_seg_visible:
            {
                ef = scl(ef, eseg);
                if (ei > 0) {
                    PropS<R> prop{pv, head_end, &cur};
                    Vx<R> pr = prop.get(ei - 1);
                    Vx<R> av = prop.get(ei);
                    Vx<R> bv = prop.get(ei + 1);
                    const MatD<R> mt = S.mat[av.mat];
                    V3<R> wi = unit(sub(pr.p, av.p));
                    V3<R> wo = unit(sub(bv.p, av.p));
                    V3<R> bf = av.spec ? spec_weight(mt, wi, av.n, av.ev) : bsdf_f(mt, wi, wo, av.n);
                    if (zero3(bf))
                        goto eval_fail;
                    ef = mul(ef, bf);
                }
            }
        }
        {
            PropS<R> prop{pv, head_end, &cur};
            Vx<R> last = prop.get(ek - 1);
            Vx<R> pr = prop.get(ek - 2);
            V3<R> toward = unit(sub(pr.p, last.p));
            if (dot(last.n, toward) <= R(0))
                goto eval_fail;
            V3<R> le = S.emit[last.emi];
            if (zero3(le))
                goto eval_fail;
            V3<R> f = mul(ef, le);
            R pi = lum(f);
            if (!(pi > R(0)) || !M<R>::finite(pi))
                goto eval_fail;
            pcb.f = f;
            pcb.pi = pi;
        }
        goto eval_done;
    eval_fail:
        pcb.pi = R(0);
    eval_done:
        if constexpr (INIT) {
            if (pcb.pi > R(0)) {
                init_commit(P, pv);
                pc = 0;
                return CO_STEP_DONE;
            }
            goto finish;
        }
        if (choose) {
            if (pcb.pi > R(0)) {
                if (P.ctl == 2) {
                    PropS<R> prop{pv, head_end, &cur};
                    R pu = R(0), pvv = R(0);
                    if (P.pk == 1)
                        cylindrical(pdir<R>(prop, first), pu, pvv);
                    int preg = classify(P.part, pcb.u, pcb.v, pu, pvv);
                    const KernTab<R> kr = P.ktab[preg];
                    tr = pert_density(prop, cur, pmask, endpoint, kr.k1, kr.k2);
                }
                a = mh_accept(cs.pi, pcb.pi, tf, tr, s_pert, s_pert);
            }
            goto pert_record;
        }
        if (!(pcb.pi > R(0)))
            goto finish;
        if (cs.eyeden == cs.eyeden)   // cached eye_path_density(current)
            goto large_accept;
        // eye_path_density (path.cpp:144-170) of the current path
        ep = 0.0;
        {
            if (cs.k < 2 || cur.get(cs.k - 1).emi < 0)
                goto ed_done;
            R p0 = cam_dir_pdf(S.cam, pdir<R>(cur, 0));
            if (p0 <= R(0))
                goto ed_done;
            ep = static_cast<double>(p0);
        }
        if (Sink::BATCH) {
            if (emit_eyeden_rays(cur, sink) > 0) {
                pc = 6;
                return CO_RAY_PENDING;
            }
        case 6:
            i = 0;
        }
        for (ei = 0; ei + 1 < cs.k; ++ei) {
            {
                Vx<R> av = cur.get(ei);
                Vx<R> bv = cur.get(ei + 1);
                if (ei > 0) {
                    if (av.emi >= 0) {
                        ep = 0.0;
                        goto ed_done;
                    }
                    Vx<R> pr = cur.get(ei - 1);
                    const MatD<R> mt = S.mat[av.mat];
                    V3<R> wi = unit(sub(pr.p, av.p));
                    V3<R> wo = unit(sub(bv.p, av.p));
                    eseg = av.spec ? spec_prob(mt, wi, av.n, av.ev) : bsdf_pdf(mt, wi, wo, av.n);
                    if (eseg <= R(0)) {
                        ep = 0.0;
                        goto ed_done;
                    }
                }
                // area_conversion(a.p, b) (path.cpp:19-29)
                V3<R> dd = sub(bv.p, av.p);
                R d2 = dot(dd, dd);
                R cval = R(0);
                if (d2 > R(0)) {
                    V3<R> dir = dvs(dd, M<R>::sqrt(d2));
                    cval = M<R>::abs(dot(bv.n, dir)) / d2;
                }
                if (cval <= R(0)) {
                    ef.x = R(0);
                } else {
                    ef.x = cval;
                    ++rc.v;
                    R dist = len(dd);
                    if (dist <= R(2) * R(kEpsD)) {
                        ef.x = R(0);
                    } else {
                        o = av.p;
                        d = dvs(dd, dist);
                        ef.y = dist - R(kEpsD);
                        goto ed_ray;
                    }
                }
                goto ed_apply;
            }
        ed_ray:
            if (Sink::BATCH) {
                if (sink.occluded(i++))
                    ef.x = R(0);
            } else {
                CO_RAY(o, d, ef.y, 4);
                if (res_prim >= 0)
                    ef.x = R(0);
            }
        ed_apply:
            if (ei == 0)
                ep *= static_cast<double>(ef.x);          // p *= area_conversion(path[0], path[1])
            else
                ep *= static_cast<double>(eseg * ef.x);   // p *= q * area_conversion(...)
            if (ep <= 0.0) {
                ep = 0.0;
                goto ed_done;
            }
        }
    ed_done:
        cs.eyeden = ep;
    large_accept:
        tr = cs.eyeden;
        {
            R sx = R(1) - s_pert;
            R sy = R(1) - R(suit_of(P.pk, kp, smp));
            a = mh_accept(cs.pi, pcb.pi, tf, tr, sx, sy);
        }
        goto finish;

    pert_record:
        if (P.ctl == 2)
            atomicAdd(&P.part.visits[region], 1ull);
        pert_rec = true;

    finish:
        if constexpr (INIT) {   // failed attempt: the next one continues the init stream
            if (++attempts < P.init_attempts)
                goto init_attempt;
            atomicExch(P.ch.err, 1);
            init_commit(P, pv);
            pc = 0;
            return CO_STEP_DONE;
        }
        // splat (driver.cpp:59-64)
        {
            // per-chain tallies read-modify-written in HBM, in the reference's order
            double lum = P.ch.lum[c];
            if (a < 1.0 && cs.pi > R(0))
                film_add(P, cs.ru, cs.rv, scl(cs.f, (R(1) - static_cast<R>(a)) / cs.pi), lum);
            if (pcb.pi > R(0) && a > 0.0)
                film_add(P, pcb.u, pcb.v, scl(pcb.f, static_cast<R>(a) / pcb.pi), lum);
            P.ch.lum[c] = lum;
            if (pert_rec) {
                P.ch.acc[c] += a;
                P.ch.iacc[c] += a;
                P.ch.npert[c] += 1;
                P.ch.ipert[c] += 1;
            } else {
                P.ch.nlarge[c] += 1;
            }
        }
        // accept / commit (driver.cpp:168-171)
        accepted = false;
        if (a > 0.0 && static_cast<double>(Unit<R>::draw(rng)) < a) {
            accepted = true;
            for (int q = 1; q <= head_end; ++q)
                store_gv(&P.ch.verts[static_cast<size_t>(q - 1) * P.C + c], pv.get(q));
            cs.k = kp;
            cs.sm = choose ? cs.sm : smp;
            cs.f = pcb.f;
            cs.pi = pcb.pi;
            cs.ru = pcb.u;
            cs.rv = pcb.v;
            cs.eyeden = __longlong_as_double(0x7ff8000000000000LL);
        }
        const unsigned long long nst = P.ch.nsteps[c];
        if (nst < P.ch.log_K) {
            size_t ofs = static_cast<size_t>(nst) * P.C + c;
            P.ch.log_a[ofs] = a;
            P.ch.log_f[ofs] = static_cast<unsigned char>((accepted ? 1 : 0) | (choose ? 2 : 0) | 4);
        }
        if (P.record_visits) {
            P.ch.vreg[c] = (choose && P.ctl != 0) ? region : -1;
            P.ch.va[c] = a;
        }
        P.ch.nsteps[c] = nst + 1;
        (void)index;
        pc = 0;
        return CO_STEP_DONE;
    }
    default:
        break;
    }
    pc = 0;
    return CO_STEP_DONE;
}

#undef CO_RAY

template <class R, int RK, bool I>
__device__ __forceinline__ void co_load(StepCo<R, RK, I> &co, const StepParams<R> &P, int c) {
    co.c = c;
    ChainCo<R> &cs = co.cs;
    cs.k = P.ch.klen[c];
    cs.sm = P.ch.smask[c];
    cs.f = mk(P.ch.cf[c], P.ch.cf[P.C + c], P.ch.cf[2 * P.C + c]);
    cs.pi = P.ch.cf[3 * P.C + c];
    cs.ru = P.ch.cr[c];
    cs.rv = P.ch.cr[P.C + c];
    cs.eyeden = P.ch.eyeden[c];
    RngIO<RK>::load(co.rng, P.ch.rng0, P.ch.rng1, c, P.seed, static_cast<unsigned long long>(P.chain_off + c));
    co.pc = 0;
}

template <class R, int RK, bool I>
__device__ __forceinline__ void co_store(const StepCo<R, RK, I> &co, const StepParams<R> &P) {
    const int c = co.c;
    const ChainCo<R> &cs = co.cs;
    P.ch.klen[c] = cs.k;
    P.ch.smask[c] = cs.sm;
    P.ch.cf[c] = cs.f.x;
    P.ch.cf[P.C + c] = cs.f.y;
    P.ch.cf[2 * P.C + c] = cs.f.z;
    P.ch.cf[3 * P.C + c] = cs.pi;
    P.ch.cr[c] = cs.ru;
    P.ch.cr[P.C + c] = cs.rv;
    P.ch.eyeden[c] = cs.eyeden;
    RngIO<RK>::store(co.rng, P.ch.rng0, P.ch.rng1, c);
}

// fp32 BVH: 64 registers for 8 resident blocks -- c4 at 4/8/10/12 blocks per
// SM: 46.8/54.9/54.4/46.4 M mut/s (Fixed strategy).
#ifndef RAMLT_CO_MINBLOCKS
#define RAMLT_CO_MINBLOCKS 8
#endif
// Persistent, work-stealing chain-step kernel.  `work` is a zeroed counter.
// INIT: chain initialisation instead of steps (k_init's job, same results).
template <class R, int RK, bool BVH, bool INIT = false>
__global__ void __launch_bounds__(128, BVH && sizeof(R) == 4 ? RAMLT_CO_MINBLOCKS : 1)
k_step_co(StepParams<R> P, unsigned int *work) {
    extern __shared__ __align__(16) char smem[];
    SceneView<R> S = stage_scene(P.scene, smem);
    size_t scene_bytes = stage_bytes_sph<R>(P.scene.nsph) +
                         (P.scene.bvh ? 0 : static_cast<size_t>(P.scene.ntri) * sizeof(TriD<R>));
    scene_bytes = (scene_bytes + 15) & ~size_t(15);
    PvSmem<R> pv = P.pv_scratch
                       ? PvSmem<R>{P.pv_scratch + blockIdx.x * blockDim.x + threadIdx.x,
                                   static_cast<int>(gridDim.x * blockDim.x)}
                       : PvSmem<R>{reinterpret_cast<GV<R> *>(smem + scene_bytes) + threadIdx.x,
                                   static_cast<int>(blockDim.x)};
    const unsigned lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;

    StepCo<R, RK, INIT> co;
    RayCount rc;
    BvhTrav<R> tv;   // BVH: resumable traversal of this lane's pending ray
    int tv_sl[BvhTrav<R>::STACK - BvhTrav<R>::SSTACK];
    tv.sl = tv_sl;
    tv.ss = reinterpret_cast<int *>(smem + P.co_stack_off) + threadIdx.x;
    bool have = false, exhausted = false, want = false;
    int j = 0, jend = 0;
    bool first_grab = true;
    for (;;) {
        // (1) converged: idle lanes take chains (one atomic per warp), or --
        // without stealing -- each lane takes its own chain once
        unsigned need = __ballot_sync(0xffffffffu, !have && !exhausted);
        if (need) {
            unsigned base = 0;
            int leader = __ffs(need) - 1;
            if (P.steal) {
                if (static_cast<int>(lane) == leader)
                    base = atomicAdd(work, static_cast<unsigned>(__popc(need)));
                base = __shfl_sync(0xffffffffu, base, leader);
            }
            if (!have && !exhausted) {
                unsigned mine = base + __popc(need & lt);
                if (!P.steal) {
                    mine = first_grab ? blockIdx.x * blockDim.x + threadIdx.x : 0xffffffffu;
                    first_grab = false;
                }
                if (INIT && mine < static_cast<unsigned>(P.C)) {
                    co.c = static_cast<int>(mine);
                    co.rng.reseed(P.seed, kStreamInit + static_cast<unsigned long long>(P.chain_off + co.c) * 2ull);
                    co.pc = 0;
                    co.attempts = 0;
                    have = true;
                } else if (mine < static_cast<unsigned>(P.C)) {
                    co_load(co, P, static_cast<int>(mine));
                    const unsigned long long my_steps =
                        P.per + (static_cast<unsigned long long>(P.chain_off + co.c) < P.rem ? 1ull : 0ull);
                    j = P.j0;
                    jend = static_cast<int>(min(static_cast<unsigned long long>(P.j1), my_steps));
                    have = true;
                    if (j >= jend) {   // inactive for this launch
                        if (P.record_visits)
                            P.ch.vreg[co.c] = -1;
                        have = false;
                    }
                } else {
                    exhausted = true;
                }
            }
        }
        // (2) divergent: advance to the next ray cast
        while (have && !want) {
            unsigned long long index = P.span_start + static_cast<unsigned long long>(j) * P.C_total + P.chain_off + co.c;
            int st = co.advance(P, S, pv, rc, index);
            if (st == CO_RAY_PENDING) {
                want = true;
                if constexpr (BVH)
                    tv.begin(S, co.ray.o, co.ray.d, co.ray.lim, co.ray.lim < M<R>::inf());
            } else if (INIT) {
                have = false;   // the coroutine stored the chain
            } else if (++j >= jend) {
                co_store(co, P);
                have = false;
            }
        }
        // (3) converged: trace every pending ray
        __syncwarp();
        if (!__any_sync(0xffffffffu, want || !exhausted))
            break;
        if constexpr (BVH) {
            // while-while rounds until the warp is done or enough lanes can
            // take a new ray (their chains' next ray, or a new chain)
            for (;;) {
                unsigned busy = __ballot_sync(0xffffffffu, want);
                unsigned idle = __ballot_sync(0xffffffffu, !want && (have || !exhausted));
                if (!busy || __popc(idle) >= P.refill)
                    break;
                if (want && tv.step(P.scene.bvh, P.scene.nsph)) {
                    co.res_prim = tv.prim(S);
                    co.res_t = tv.best;
                    want = false;
                }
            }
        } else if (want) {
            R t;
            co.res_prim = trace_ray<R, BVH>(S, co.ray, t);
            co.res_t = t;
            want = false;
        }
    }
    if (INIT)   // ray statistics cover mutations only (as with k_init)
        return;
    unsigned act = __activemask();
    unsigned sc = __reduce_add_sync(act, static_cast<unsigned>(rc.c));
    unsigned sv = __reduce_add_sync(act, static_cast<unsigned>(rc.v));
    if (lane == static_cast<unsigned>(__ffs(act) - 1)) {
        atomicAdd(&P.ch.rays[0], static_cast<unsigned long long>(sc));
        atomicAdd(&P.ch.rays[1], static_cast<unsigned long long>(sv));
    }
}

// ---- traversal-only throughput probe (ramlt_gpu_trace_benchmark) ------------------------------
__device__ __forceinline__ uint32_t tb_hash(uint32_t x) {
    x ^= x >> 16;
    x *= 0x7feb352dU;
    x ^= x >> 15;
    x *= 0x846ca68bU;
    x ^= x >> 16;
    return x;
}

// The coroutine kernel's traversal loop (while-while rounds, dynamic ray
// fetch with the same refill rule) on synthetic incoherent rays.
template <class R>
__global__ void __launch_bounds__(128, sizeof(R) == 4 ? RAMLT_CO_MINBLOCKS : 1)
k_trace_bench(StepParams<R> P, unsigned long long n, unsigned *work, unsigned long long *hits, V3<R> lo, V3<R> ext,
              int cells) {
    extern __shared__ __align__(16) char smem[];
    SceneView<R> S = stage_scene(P.scene, smem);
    const unsigned lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    BvhTrav<R> tv;
    int tv_sl[BvhTrav<R>::STACK - BvhTrav<R>::SSTACK];
    tv.sl = tv_sl;
    tv.ss = reinterpret_cast<int *>(smem + P.co_stack_off) + threadIdx.x;
    bool want = false, exhausted = false;
    unsigned h = 0;
    for (;;) {
        unsigned need = __ballot_sync(0xffffffffu, !want && !exhausted);
        if (need) {
            int leader = __ffs(need) - 1;
            unsigned base = 0;
            if (static_cast<int>(lane) == leader)
                base = atomicAdd(work, static_cast<unsigned>(__popc(need)));
            base = __shfl_sync(0xffffffffu, base, leader);
            if (!want && !exhausted) {
                unsigned mine = base + __popc(need & lt);
                if (mine < n) {
                    uint32_t a = tb_hash(mine * 5u + 1u), b = tb_hash(mine * 5u + 2u), c = tb_hash(mine * 5u + 3u);
                    uint32_t e = tb_hash(mine * 5u + 4u), f = tb_hash(mine * 5u + 5u);
                    const R k = R(1) / R(4294967296.0);
                    V3<R> o = mk(lo.x + ext.x * (R(a) * k), lo.y + ext.y * (R(b) * k), lo.z + ext.z * (R(c) * k));
                    R z = R(1) - R(2) * (R(e) * k), ph = R(kTwoPiD) * (R(f) * k);
                    R r = M<R>::sqrt(fmax(R(0), R(1) - z * z));
                    V3<R> dir = mk(r * M<R>::cos(ph), r * M<R>::sin(ph), z);
                    if (cells > 0) {
                        // the same ray population in bucket order (origin cell, direction octant):
                        // what a queue sorted by (cell, octant) would hand to neighbouring lanes
                        const unsigned long long nb = static_cast<unsigned long long>(cells) * cells * cells * 8ull;
                        const unsigned long long bkt = static_cast<unsigned long long>(mine) * nb / n;
                        const unsigned cell = static_cast<unsigned>(bkt >> 3), oct = static_cast<unsigned>(bkt & 7u);
                        const R inv = R(1) / R(cells);
                        o = mk(lo.x + ext.x * (R(cell % cells) + R(a) * k) * inv,
                               lo.y + ext.y * (R((cell / cells) % cells) + R(b) * k) * inv,
                               lo.z + ext.z * (R(cell / (cells * cells)) + R(c) * k) * inv);
                        dir = mk((oct & 1u) ? -M<R>::abs(dir.x) : M<R>::abs(dir.x),
                                 (oct & 2u) ? -M<R>::abs(dir.y) : M<R>::abs(dir.y),
                                 (oct & 4u) ? -M<R>::abs(dir.z) : M<R>::abs(dir.z));
                    }
                    tv.begin(S, o, dir, M<R>::inf(), false);
                    want = true;
                } else {
                    exhausted = true;
                }
            }
        }
        if (!__any_sync(0xffffffffu, want))
            break;
        for (;;) {
            unsigned busy = __ballot_sync(0xffffffffu, want);
            unsigned idle = __ballot_sync(0xffffffffu, !want && !exhausted);
            if (!busy || __popc(idle) >= P.refill)
                break;
            if (want && tv.step(P.scene.bvh, P.scene.nsph)) {
                h += tv.pos >= 0 ? 1u : 0u;
                want = false;
            }
        }
    }
    unsigned s = __reduce_add_sync(0xffffffffu, h);
    if (lane == 0)
        atomicAdd(hits, static_cast<unsigned long long>(s));
}

}  // namespace rd

