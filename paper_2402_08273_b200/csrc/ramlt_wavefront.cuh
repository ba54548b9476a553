// ramlt_wavefront.cuh -- the chain step as a wavefront (the default for BVH scenes).
//
// The mutation of core/driver.cpp:113-171 is the resumable coroutine StepCo
// (ramlt_step_co.cuh).  Instead of tracing inside the coroutine kernel, a
// lockstep step alternates kernels until no chain has a ray pending:
//
//   k_wf_logic  one thread per chain that yielded: resume the coroutine with
//               its answer, advance it to its next yield (or the end of its
//               step); its rays go into the round's ray queue and the chain
//               into the next round's chain queue, with warp-aggregated
//               atomics.  A yield is one closest-hit ray (retrace, large-step
//               bounce) or ALL the visibility rays of eval_contribution /
//               eye_path_density at once (they do not depend on each other),
//               so a mutation takes ~closest-hit rays + 2 rounds.  Chains are
//               queued per yield point and every queue is resumed from a warp
//               boundary: a warp's lanes resume at the same point;
//   k_wf_bounce (RAMLT_WF_BOUNCE=1) the large-step bounce loop -- half of all
//               mutations, ~11 rounds each -- resumed by a small kernel from
//               the chain's compact image (bounce_body, the coroutine's own
//               loop body);
//   k_wf_trace  persistent, one ray per lane, dynamic ray fetch and
//               while-while BVH rounds over the queue, writing (t, prim) by
//               chain for closest hits and OR-ing bit k of the chain's
//               occlusion mask for an occluded visibility ray k
//               (k_wf_trace_brute: the shared-memory linear scan instead).
//
// Between rounds the coroutine state lives in HBM as whole 32-byte sectors
// indexed [sector][chain] (256-bit evict-first loads / stores); a chain inside
// the bounce loop moves only a compact image of the loop's live values (2
// sectors in fp32 / Philox) and fetches the cold sectors when it leaves the
// loop.  The proposal vertices live in a [vertex][chain] array.  The trace
// kernel carries no mutation state, so it runs with far fewer registers and
// more warps than the fused coroutine kernel, and every warp of it holds rays,
// whatever phase each chain is in.  Arithmetic and RNG consumption are the
// coroutine's, so the results equal k_step_co's (and the fp64/PCG build the
// reference's).
#pragma once

#include "ramlt_step_co.cuh"

namespace rd {

// Pending ray: 32 B in fp32 (one sector).  `ck` = chain | ordinal << 27: ordinal 0
// for a closest-hit ray (answer in hits[chain]); ordinal k of a visibility batch
// sets bit k of occ[chain] when occluded.  lim <= 0 marks an unused slot.
constexpr int kWfChainBits = 27;
template <class R> struct alignas(sizeof(R) * 8) WfRay {
    R o[3], lim;
    R d[3];
    int ck;
};
template <class R> struct alignas(sizeof(R) * 2) WfHit {
    R t;
    int prim;
};

// Coroutine state carried between rounds.
template <class R, int RK, bool INIT = false> struct alignas(32) WfState {
    StepCo<R, RK, INIT> co;   // its step cursor: co.wf_j, co.wf_jend
    // Sectors [0, HOT) hold the fields the large-step bounce loop uses (StepCo's
    // leading members); a chain resumed in that loop moves only those.
    static constexpr int HOT = static_cast<int>((__builtin_offsetof(StepCo<R, RK, INIT>, cs) + 31) / 32);
};

// Chain queues are kept per yield point (kWfQueues sub-queues of capacity C each:
// retrace ray, large-step bounce, eval_contribution batch, eye_path_density batch),
// and a round resumes them queue by queue with every queue's segment starting on a
// warp boundary: the lanes of a warp resume at the same point of the coroutine
// instead of at four different ones.
// A fifth queue holds the chains k_wf_bounce took out of the bounce loop: k_wf_logic resumes
// them behind the loop (yield point 7) in the next round.
constexpr int kWfQueues = 5;
__device__ __forceinline__ int wf_queue_of(int pc) {
    return pc == 1 ? 0 : (pc == 2 ? 1 : (pc == 5 ? 2 : (pc == 6 ? 3 : 4)));
}

template <class R> struct WfParams {
    unsigned c0, cn;           // this pipeline's chain range [c0, c0 + cn) (round 0)
    int bounce_sep;            // != 0: the bounce queue (1) belongs to k_wf_bounce, not to k_wf_logic
    const int *cq_in;          // chains resumed this round (round > 0): sub-queue q at cq_in + q * C
    const unsigned *n_in;      // [kWfQueues]
    int *cq_out;               // chains that yielded this round, by yield point
    unsigned *n_out;           // [kWfQueues]
    WfRay<R> *rays;            // this round's ray queue
    unsigned *n_rays;
    unsigned *trace_work;      // zeroed here for the following k_wf_trace
    const WfHit<R> *hits;      // closest-hit answers, by chain
    unsigned *occ;             // visibility-batch answers, by chain (bit k = ray k occluded)
    uint4 *state;              // WfState as 16 B chunks: chunk k of chain c at state[k * C + c]
    GV<R> *pv;                 // proposal vertices, vertex i of chain c at pv[i * C + c]
};

// The coroutine's rays go straight into the round's ray queue (StepCo::advance, BATCH).
template <class R> struct WfSink {
    static constexpr bool BATCH = true;
    WfRay<R> *rays;
    unsigned *n_rays;
    unsigned *occ_g;
    int c;
    unsigned occ;   // answers of the batch this chain is resumed from
    // hot/cold state: where the chain's cold sectors are and whether they are resident
    const uint4 *state;
    size_t C;
    char *resident;      // the thread's coroutine state (shared memory)
    int *full;           // != 0: every sector is resident
    int hot, total;      // sectors
    __device__ __forceinline__ void cold() const;
    // n slots per calling lane: one atomic for the lanes converged here
    __device__ __forceinline__ unsigned reserve(unsigned n) const {
        const unsigned act = __activemask();
        const unsigned lane = threadIdx.x & 31;
        const unsigned lt = (1u << lane) - 1u;
        unsigned pre = 0, tot = 0;
#pragma unroll
        for (int b = 0; b < 5; ++b) {   // n < 32
            const unsigned mb = __ballot_sync(act, (n >> b) & 1u);
            pre += static_cast<unsigned>(__popc(mb & lt)) << b;
            tot += static_cast<unsigned>(__popc(mb)) << b;
        }
        const int leader = __ffs(act) - 1;
        unsigned base = 0;
        if (static_cast<int>(lane) == leader)
            base = atomicAdd(n_rays, tot);
        base = __shfl_sync(act, base, leader);
        return base + pre;
    }
    __device__ __forceinline__ void put(unsigned slot, V3<R> o, V3<R> d, R lim, int k) const {
        WfRay<R> r;
        r.o[0] = o.x, r.o[1] = o.y, r.o[2] = o.z;
        r.lim = lim;
        r.d[0] = d.x, r.d[1] = d.y, r.d[2] = d.z;
        r.ck = c | (k << kWfChainBits);
        rays[slot] = r;
    }
    __device__ __forceinline__ void null(unsigned slot) const {
        WfRay<R> r;
        r.o[0] = r.o[1] = r.o[2] = r.lim = R(0);
        r.d[0] = R(1), r.d[1] = r.d[2] = R(0);
        r.ck = c;
        rays[slot] = r;
    }
    __device__ __forceinline__ void begin_batch() const { occ_g[c] = 0u; }
    __device__ __forceinline__ bool occluded(int k) const { return (occ >> k) & 1u; }
};

// RAMLT_WF_HOTCOLD=1 (default): chains resumed in the large-step bounce loop -- half of
// all mutations, ~11 rounds each, nearly all of them ending without a contribution --
// load and store only the hot sectors of their state (4 of 10 in fp32).
#ifndef RAMLT_WF_HOTCOLD
#define RAMLT_WF_HOTCOLD 1
#endif

// State chunks are whole 32 B sectors moved with 256-bit evict-first loads / stores
// (LDG/STG.E.EF.ENL2.256): a chain's chunk never shares a sector with its neighbour's,
// so a queue that no longer holds consecutive chains costs no half-used sectors.
// RAMLT_WF_CHUNK32=0: 16 B chunks (the first wavefront build), kept for A/B runs.
#ifndef RAMLT_WF_CHUNK32
#define RAMLT_WF_CHUNK32 1
#endif
// RAMLT_WF_SMEM=1 (default): the resumed coroutine lives in shared memory (one
// WfState per thread, 5 blocks per SM) instead of the thread's local memory, whose
// lines the streaming state traffic kept evicting to L2 / HBM.  c5, one box:
// 16 B chunks + local 86.4, 32 B chunks + local 100.8, 32 B chunks + smem 105.8 M
// mutations/s.
#ifndef RAMLT_WF_SMEM
#define RAMLT_WF_SMEM 1
#endif
struct __align__(32) Sector {
    unsigned w[8];
};
__device__ __forceinline__ Sector ld_sector_cs(const void *p) {
    Sector r;
    asm volatile("ld.global.cs.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r.w[0]), "=r"(r.w[1]), "=r"(r.w[2]), "=r"(r.w[3]), "=r"(r.w[4]), "=r"(r.w[5]),
                   "=r"(r.w[6]), "=r"(r.w[7])
                 : "l"(p));
    return r;
}
__device__ __forceinline__ void st_sector_cs(void *p, const Sector &r) {
    asm volatile("st.global.cs.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(r.w[0]), "r"(r.w[1]),
                 "r"(r.w[2]), "r"(r.w[3]), "r"(r.w[4]), "r"(r.w[5]), "r"(r.w[6]), "r"(r.w[7])
                 : "memory");
}

template <class T> struct Chunks {
#if RAMLT_WF_CHUNK32
    static constexpr int K = 2 * static_cast<int>((sizeof(T) + 31) / 32);   // in uint4 units
    Sector w[K / 2];
#else
    static constexpr int K = static_cast<int>((sizeof(T) + 15) / 16);
    uint4 w[K];
#endif
};

template <class T> __device__ __forceinline__ void ld_state(T &v, const uint4 *__restrict__ base, size_t C, int c) {
    Chunks<T> b;
#if RAMLT_WF_CHUNK32
    const Sector *p = reinterpret_cast<const Sector *>(base);
#pragma unroll
    for (int k = 0; k < Chunks<T>::K / 2; ++k)
        b.w[k] = ld_sector_cs(p + static_cast<size_t>(k) * C + c);
#else
#pragma unroll
    for (int k = 0; k < Chunks<T>::K; ++k)
        b.w[k] = __ldcs(base + static_cast<size_t>(k) * C + c);
#endif
    memcpy(&v, &b, sizeof(T));
}
template <class T> __device__ __forceinline__ void st_state(const T &v, uint4 *__restrict__ base, size_t C, int c) {
    Chunks<T> b;
    memcpy(&b, &v, sizeof(T));
#if RAMLT_WF_CHUNK32
    Sector *p = reinterpret_cast<Sector *>(base);
#pragma unroll
    for (int k = 0; k < Chunks<T>::K / 2; ++k)
        st_sector_cs(p + static_cast<size_t>(k) * C + c, b.w[k]);
#else
#pragma unroll
    for (int k = 0; k < Chunks<T>::K; ++k)
        __stcs(base + static_cast<size_t>(k) * C + c, b.w[k]);
#endif
}

// Sectors [k0, k1) of a state image (32 B aligned, a whole number of sectors long).
__device__ __forceinline__ void ld_sectors(char *dst, const uint4 *__restrict__ base, size_t C, int c, int k0, int k1) {
    const Sector *p = reinterpret_cast<const Sector *>(base);
    for (int k = k0; k < k1; ++k)
        *reinterpret_cast<Sector *>(dst + 32 * k) = ld_sector_cs(p + static_cast<size_t>(k) * C + c);
}
__device__ __forceinline__ void st_sectors(const char *src, uint4 *__restrict__ base, size_t C, int c, int k0, int k1) {
    Sector *p = reinterpret_cast<Sector *>(base);
    for (int k = k0; k < k1; ++k)
        st_sector_cs(p + static_cast<size_t>(k) * C + c, *reinterpret_cast<const Sector *>(src + 32 * k));
}
template <class R> __device__ __forceinline__ void WfSink<R>::cold() const {
    if (!*full) {
        ld_sectors(resident, state, C, c, hot, total);
        *full = 1;
    }
}

// Compact image of a chain inside the large-step bounce loop (steps and INIT): the
// loop's live values in 2 sectors (fp32 / Philox) instead of the 4 hot ones -- the pending ray (its lim is
// +inf), the Philox draw counter (key and stream follow from the seed and the chain id; the
// cached block is recomputed from the counter, the same words), tf, dpdf, the specular mask,
// kp, the four flags and the step cursor.  It lives in sectors 0-1 of the chain's state; the
// cold sectors keep their place.  RAMLT_WF_COMPACT=0: the 4 raw hot sectors.
#ifndef RAMLT_WF_COMPACT
#define RAMLT_WF_COMPACT 1
#endif
template <int RK> struct WfRngSave;
template <> struct WfRngSave<RNG_PHILOX> {
    unsigned long long draw;
    __device__ __forceinline__ void save(const Rng<RNG_PHILOX> &r) { draw = r.draw; }
    template <bool INIT, class R>
    __device__ __forceinline__ void restore(Rng<RNG_PHILOX> &r, const StepParams<R> &P, int c) const {
        const unsigned long long gc = static_cast<unsigned long long>(P.chain_off + c);
        r.reseed(P.seed, INIT ? kStreamInit + gc * 2ull : gc);   // the chain's init / step stream
        r.draw = draw;
    }
};
template <> struct WfRngSave<RNG_PCG> {
    unsigned long long state, inc;
    __device__ __forceinline__ void save(const Rng<RNG_PCG> &r) { state = r.state, inc = r.inc; }
    template <bool INIT, class R>
    __device__ __forceinline__ void restore(Rng<RNG_PCG> &r, const StepParams<R> &, int) const {
        r.state = state, r.inc = inc;
    }
};
// The image: 64 B (2 sectors) in fp32 / Philox, 72 B (3) in fp32 / PCG, 96-104 B (3-4) in fp64.
template <class R, int RK> struct WfBounceImage {
    double tf;
    WfRngSave<RK> rng;
    R o[3], d[3];
    R dpdf;
    unsigned smp;
    unsigned kp_flags;   // kp | choose << 8 | ok << 9 | accepted << 10 | pert_rec << 11
    int j, jend;
    unsigned attempts;   // INIT
};
// The members of StepCo the image restores, for k_wf_bounce (no cold part, no coroutine).
template <class R, int RK> struct WfBounceRegs {
    int c, pc, wf_j, wf_jend;
    Rng<RK> rng;
    RayReq<R> ray;
    R dpdf;
    int kp;
    unsigned smp;
    double tf;
    bool choose, ok, accepted, pert_rec;
    unsigned attempts;
};
template <class R, int RK, bool INIT> struct WfCompact {
    static constexpr bool OK = RAMLT_WF_COMPACT && RAMLT_WF_HOTCOLD && RAMLT_WF_CHUNK32;
    using Img = WfBounceImage<R, RK>;
    static constexpr int N = static_cast<int>((sizeof(Img) + 31) / 32);   // sectors
    struct alignas(32) Buf {
        Sector w[N];
    };
    template <class CoT> static __device__ __forceinline__ void pack(const CoT &co, Buf &buf) {
        Img im;
        im.tf = co.tf;
        im.rng.save(co.rng);
        im.o[0] = co.ray.o.x, im.o[1] = co.ray.o.y, im.o[2] = co.ray.o.z;
        im.d[0] = co.ray.d.x, im.d[1] = co.ray.d.y, im.d[2] = co.ray.d.z;
        im.dpdf = co.dpdf;
        im.smp = co.smp;
        im.kp_flags = static_cast<unsigned>(co.kp) | (co.choose ? 0x100u : 0u) | (co.ok ? 0x200u : 0u) |
                      (co.accepted ? 0x400u : 0u) | (co.pert_rec ? 0x800u : 0u);
        im.j = co.wf_j;
        im.jend = co.wf_jend;
        im.attempts = co.attempts;
        memcpy(&buf, &im, sizeof(Img));
    }
    template <class CoT>
    static __device__ __forceinline__ void unpack(CoT &co, const Buf &buf, int c, const StepParams<R> &P) {
        Img im;
        memcpy(&im, &buf, sizeof(Img));
        co.c = c;
        co.pc = 2;
        co.ray.o = mk(im.o[0], im.o[1], im.o[2]);
        co.ray.d = mk(im.d[0], im.d[1], im.d[2]);
        co.ray.lim = M<R>::inf();
        im.rng.template restore<INIT>(co.rng, P, c);
        co.tf = im.tf;
        co.dpdf = im.dpdf;
        co.smp = im.smp;
        co.kp = static_cast<int>(im.kp_flags & 0xffu);
        co.choose = (im.kp_flags & 0x100u) != 0;
        co.ok = (im.kp_flags & 0x200u) != 0;
        co.accepted = (im.kp_flags & 0x400u) != 0;
        co.pert_rec = (im.kp_flags & 0x800u) != 0;
        co.wf_j = im.j;
        co.wf_jend = im.jend;
        co.attempts = im.attempts;
    }
    static __device__ __forceinline__ void load(Buf &buf, const uint4 *__restrict__ state, size_t C, int c) {
        const Sector *sp = reinterpret_cast<const Sector *>(state);
#pragma unroll
        for (int k = 0; k < N; ++k)
            buf.w[k] = ld_sector_cs(sp + static_cast<size_t>(k) * C + c);
    }
    static __device__ __forceinline__ void store(const Buf &buf, uint4 *__restrict__ state, size_t C, int c) {
        Sector *sp = reinterpret_cast<Sector *>(state);
#pragma unroll
        for (int k = 0; k < N; ++k)
            st_sector_cs(sp + static_cast<size_t>(k) * C + c, buf.w[k]);
    }
};

// INIT: chain initialisation (core/driver.cpp:219-242) instead of a step -- the
// coroutine draws large-step eye paths from the chain's init stream until one
// contributes and stores the chain itself; rounds run until every chain has one.
template <class R, int RK, bool INIT = false>
__global__ void __launch_bounds__(128, RAMLT_WF_SMEM && sizeof(R) == 4 ? 5 : 1) k_wf_logic(StepParams<R> P, WfParams<R> W, int round0) {
    extern __shared__ __align__(32) char smem[];
    SceneView<R> S = stage_scene(P.scene, smem);
    if (blockIdx.x == 0 && threadIdx.x == 0)
        *W.trace_work = 0;
    // round > 0: index space = the sub-queues back to back, each padded to whole warps
    unsigned qn[kWfQueues], qstart[kWfQueues + 1];
    qstart[0] = 0;
#pragma unroll
    for (int q = 0; q < kWfQueues; ++q) {
        qn[q] = (round0 || (q == 1 && W.bounce_sep)) ? 0u : W.n_in[q];
        qstart[q + 1] = qstart[q] + ((qn[q] + 31u) & ~31u);
    }
    const unsigned n = round0 ? W.cn : qstart[kWfQueues];
    RayCount rc;
    const unsigned stride = gridDim.x * blockDim.x;
    for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
#if RAMLT_WF_SMEM
        WfState<R, RK, INIT> &s = reinterpret_cast<WfState<R, RK, INIT> *>(smem + P.co_stack_off)[threadIdx.x];
#else
        WfState<R, RK, INIT> s;
#endif
        using St = WfState<R, RK, INIT>;
        constexpr int TOTAL = static_cast<int>(sizeof(St) / 32);
        static_assert(WfCompact<R, RK, INIT>::N <= St::HOT, "the compact image must not reach the cold sectors");
        int full = 1;   // every sector of the state is resident
        WfSink<R> sink{W.rays, W.n_rays, W.occ, 0, 0u, W.state, static_cast<size_t>(P.C),
                       reinterpret_cast<char *>(&s), &full, St::HOT, TOTAL};
        int c;
        if (round0 && INIT) {
            c = static_cast<int>(W.c0 + i);
            s.co.c = c;
            s.co.rng.reseed(P.seed, kStreamInit + static_cast<unsigned long long>(P.chain_off + c) * 2ull);
            s.co.pc = 0;
            s.co.attempts = 0;
            s.co.wf_j = 0;
            s.co.wf_jend = 1;
        } else if (round0) {
            c = static_cast<int>(W.c0 + i);
            co_load(s.co, P, c);
            const unsigned long long my_steps =
                P.per + (static_cast<unsigned long long>(P.chain_off + c) < P.rem ? 1ull : 0ull);
            s.co.wf_j = P.j0;
            s.co.wf_jend = static_cast<int>(min(static_cast<unsigned long long>(P.j1), my_steps));
            if (s.co.wf_j >= s.co.wf_jend) {   // inactive for this launch
                if (P.record_visits)
                    P.ch.vreg[c] = -1;
                continue;
            }
        } else {
            int q = 0;
#pragma unroll
            for (int k = 1; k < kWfQueues; ++k)
                q += i >= qstart[k] ? 1 : 0;
            const unsigned k = i - qstart[q];
            if (k >= qn[q])   // padding of this queue's last warp
                continue;
            c = W.cq_in[static_cast<size_t>(q) * P.C + k];
#if RAMLT_WF_HOTCOLD && RAMLT_WF_CHUNK32
            if ((q == 1 || q == 4) && WfCompact<R, RK, INIT>::OK) {   // in (4: just behind) the large-step bounce loop: the compact image
                typename WfCompact<R, RK, INIT>::Buf buf;
                WfCompact<R, RK, INIT>::load(buf, W.state, static_cast<size_t>(P.C), c);
                WfCompact<R, RK, INIT>::unpack(s.co, buf, c, P);
                if (q == 4)
                    s.co.pc = 7;
                full = 0;
            } else if (q == 1) {   // ... or the hot sectors only
                ld_sectors(reinterpret_cast<char *>(&s), W.state, static_cast<size_t>(P.C), c, 0, St::HOT);
                full = 0;
            } else {
                ld_sectors(reinterpret_cast<char *>(&s), W.state, static_cast<size_t>(P.C), c, 0, TOTAL);
            }
#else
            ld_state(s, W.state, static_cast<size_t>(P.C), c);
#endif
            if (q < 2) {   // a closest-hit yield: its answer
                const WfHit<R> h = W.hits[c];
                s.co.res_prim = h.prim;
                s.co.res_t = h.t;
            }
            sink.occ = q >= 2 ? W.occ[c] : 0u;   // only the batch yields have occlusion answers
        }
        sink.c = c;
        const PvSmem<R> pv{W.pv + c, P.C};
        for (;;) {
            const unsigned long long index =
                P.span_start + static_cast<unsigned long long>(s.co.wf_j) * P.C_total + P.chain_off + c;
            if (s.co.advance(P, S, pv, rc, index, sink) == CO_RAY_PENDING) {
                const unsigned act = __activemask();
                const int q = wf_queue_of(s.co.pc);
                const unsigned grp = __match_any_sync(act, q);   // the lanes yielding at the same point
                const int leader = __ffs(grp) - 1;
                unsigned base = 0;
                if (static_cast<int>(threadIdx.x & 31) == leader)
                    base = atomicAdd(W.n_out + q, static_cast<unsigned>(__popc(grp)));
                base = __shfl_sync(grp, base, leader);
                W.cq_out[static_cast<size_t>(q) * P.C + base + __popc(grp & ((1u << (threadIdx.x & 31)) - 1u))] = c;
#if RAMLT_WF_HOTCOLD && RAMLT_WF_CHUNK32
                // still in the bounce loop it was resumed in: the cold sectors in HBM are current
                if (q == 1 && WfCompact<R, RK, INIT>::OK) {
                    // entering the loop (full): the cold sectors too; the raw hot sectors are never read back
                    typename WfCompact<R, RK, INIT>::Buf buf;
                    WfCompact<R, RK, INIT>::pack(s.co, buf);
                    WfCompact<R, RK, INIT>::store(buf, W.state, static_cast<size_t>(P.C), c);
                    if (full)
                        st_sectors(reinterpret_cast<const char *>(&s), W.state, static_cast<size_t>(P.C), c, St::HOT,
                                   TOTAL);
                } else {
                    st_sectors(reinterpret_cast<const char *>(&s), W.state, static_cast<size_t>(P.C), c, 0,
                               full ? TOTAL : St::HOT);
                }
#else
                st_state(s, W.state, static_cast<size_t>(P.C), c);
#endif
                break;
            }
            if (INIT)   // the coroutine stored the chain
                break;
            if (++s.co.wf_j >= s.co.wf_jend) {
                co_store(s.co, P);
                break;
            }
        }
    }
    unsigned act = __activemask();
    unsigned sc = __reduce_add_sync(act, static_cast<unsigned>(rc.c));
    unsigned sv = __reduce_add_sync(act, static_cast<unsigned>(rc.v));
    if ((sc | sv) && (threadIdx.x & 31) == static_cast<unsigned>(__ffs(act) - 1)) {
        atomicAdd(&P.ch.rays[0], static_cast<unsigned long long>(sc));
        atomicAdd(&P.ch.rays[1], static_cast<unsigned long long>(sv));
    }
}

// The large-step bounce loop as its own kernel: half of all mutations spend ~11 rounds in
// it and its live state is the compact image, so those resumes run here -- a few dozen
// registers, no shared-memory coroutine, a small instruction footprint -- instead of in
// k_wf_logic.  One thread per chain of the bounce queue: unpack, bounce_body (the
// coroutine's own loop body), then either the next ray and the bounce queue again, or the
// post-loop queue, from which k_wf_logic resumes the chain behind the loop next round.
template <class R, int RK, bool INIT = false>
__global__ void __launch_bounds__(128, sizeof(R) == 4 ? 8 : 1) k_wf_bounce(StepParams<R> P, WfParams<R> W) {
    extern __shared__ __align__(32) char smem[];
    SceneView<R> S = stage_scene(P.scene, smem);
    using Cp = WfCompact<R, RK, INIT>;
    const unsigned n = W.n_in[1];
    const unsigned stride = gridDim.x * blockDim.x;
    unsigned cast = 0;
    for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < ((n + 31u) & ~31u); i += stride) {
        const bool live = i < n;
        bool cont = false;
        int c = 0;
        WfBounceRegs<R, RK> co;
        V3<R> o, d;
        if (live) {
            c = W.cq_in[static_cast<size_t>(P.C) + i];
            typename Cp::Buf buf;
            Cp::load(buf, W.state, static_cast<size_t>(P.C), c);
            Cp::unpack(co, buf, c, P);
            const WfHit<R> h = W.hits[c];
            const PvSmem<R> pv{W.pv + c, P.C};
            cont = bounce_body<R, RK>(P, S, pv, co.ray, h.prim, h.t, co.rng, co.dpdf, co.kp, co.smp, co.tf, co.ok, o, d);
        }
        // warp-aggregated appends: continuing chains -> a ray and the bounce queue, the others -> post-loop queue
        const unsigned lane = threadIdx.x & 31;
        const unsigned lt = (1u << lane) - 1u;
        const unsigned mc = __ballot_sync(0xffffffffu, live && cont);
        const unsigned me = __ballot_sync(0xffffffffu, live && !cont);
        unsigned base_c = 0, base_r = 0, base_e = 0;
        if (lane == 0) {
            if (mc) {
                base_c = atomicAdd(W.n_out + 1, static_cast<unsigned>(__popc(mc)));
                base_r = atomicAdd(W.n_rays, static_cast<unsigned>(__popc(mc)));
            }
            if (me)
                base_e = atomicAdd(W.n_out + 4, static_cast<unsigned>(__popc(me)));
        }
        base_c = __shfl_sync(0xffffffffu, base_c, 0);
        base_r = __shfl_sync(0xffffffffu, base_r, 0);
        base_e = __shfl_sync(0xffffffffu, base_e, 0);
        if (live) {
            if (cont) {
                co.ray.o = o;
                co.ray.d = d;
                ++cast;
                const unsigned k = static_cast<unsigned>(__popc(mc & lt));
                WfRay<R> r;
                r.o[0] = o.x, r.o[1] = o.y, r.o[2] = o.z;
                r.lim = M<R>::inf();
                r.d[0] = d.x, r.d[1] = d.y, r.d[2] = d.z;
                r.ck = c;
                W.rays[base_r + k] = r;
                W.cq_out[static_cast<size_t>(P.C) + base_c + k] = c;
            } else {
                W.cq_out[static_cast<size_t>(4) * P.C + base_e + __popc(me & lt)] = c;
            }
            typename Cp::Buf buf;
            Cp::pack(co, buf);
            Cp::store(buf, W.state, static_cast<size_t>(P.C), c);
        }
    }
    cast = __reduce_add_sync(0xffffffffu, cast);
    if (cast && (threadIdx.x & 31) == 0)
        atomicAdd(&P.ch.rays[0], static_cast<unsigned long long>(cast));
}

template <class R> __device__ __forceinline__ WfRay<R> ld_ray(const WfRay<R> *p) { return *p; }
template <> __device__ __forceinline__ WfRay<float> ld_ray<float>(const WfRay<float> *p) {
    float4 a, b;
    ldg256(p, a, b);
    WfRay<float> r;
    r.o[0] = a.x, r.o[1] = a.y, r.o[2] = a.z, r.lim = a.w;
    r.d[0] = b.x, r.d[1] = b.y, r.d[2] = b.z, r.ck = __float_as_int(b.w);
    return r;
}

// c5 (tools/ab.py, one box): 12 / 10 / 8 resident blocks per SM (40 / 48 / 55
// registers) -> 75.2 / 79.7 / 80.5 M mutations/s.
#ifndef RAMLT_WF_MINBLOCKS
#define RAMLT_WF_MINBLOCKS 8
#endif
// Persistent closest-hit / any-hit tracer over the queue (the while-while
// rounds and refill rule of k_trace_bench).  `zero_a`, `zero_b` are the
// counters the next round's k_wf_logic appends to.
template <class R>
__global__ void __launch_bounds__(128, sizeof(R) == 4 ? RAMLT_WF_MINBLOCKS : 1)
k_wf_trace(StepParams<R> P, const WfRay<R> *__restrict__ rays, WfHit<R> *__restrict__ hits,
           unsigned *__restrict__ occ, const unsigned *n_ptr, unsigned *work, unsigned *zero_a, unsigned *zero_b) {
    extern __shared__ __align__(16) char smem[];
    SceneView<R> S = stage_scene(P.scene, smem);
    if (blockIdx.x == 0 && threadIdx.x < kWfQueues)   // the next round's chain-queue lengths ...
        zero_a[threadIdx.x] = 0;
    if (blockIdx.x == 0 && threadIdx.x == 0)           // ... and its ray-queue length
        *zero_b = 0;
    const unsigned n = *n_ptr;
    const unsigned lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    BvhTrav<R> tv;
    int tv_sl[BvhTrav<R>::STACK - BvhTrav<R>::SSTACK];
    tv.sl = tv_sl;
    tv.ss = reinterpret_cast<int *>(smem + P.co_stack_off) + threadIdx.x;
    bool want = false, exhausted = n == 0, any = false;
    int ck = 0;
    for (;;) {
        const unsigned need = __ballot_sync(0xffffffffu, !want && !exhausted);
        if (need) {
            const int leader = __ffs(need) - 1;
            unsigned base = 0;
            if (static_cast<int>(lane) == leader)
                base = atomicAdd(work, static_cast<unsigned>(__popc(need)));
            base = __shfl_sync(0xffffffffu, base, leader);
            if (!want && !exhausted) {
                const unsigned mine = base + __popc(need & lt);
                if (mine < n) {
                    const WfRay<R> r = ld_ray(rays + mine);
                    if (r.lim > R(0)) {   // lim <= 0: unused slot of a batch
                        any = r.lim < M<R>::inf();
                        tv.begin(S, mk(r.o[0], r.o[1], r.o[2]), mk(r.d[0], r.d[1], r.d[2]), r.lim, any);
                        ck = r.ck;
                        want = true;
                    }
                } else {
                    exhausted = true;
                }
            }
        }
        if (!__any_sync(0xffffffffu, want || !exhausted))
            break;
        for (;;) {
            const unsigned busy = __ballot_sync(0xffffffffu, want);
            const unsigned idle = __ballot_sync(0xffffffffu, !want && !exhausted);
            if (!busy || __popc(idle) >= P.refill)
                break;
            if (want && tv.step(P.scene.bvh, P.scene.nsph)) {
                const int prim = tv.prim(S);
                const int c = ck & ((1 << kWfChainBits) - 1);
                if (any) {
                    if (prim >= 0)
                        atomicOr(occ + c, 1u << (static_cast<unsigned>(ck) >> kWfChainBits));
                } else {
                    WfHit<R> h;
                    h.t = tv.best;
                    h.prim = prim;
                    hits[c] = h;
                }
                want = false;
            }
        }
    }
}

// Brute-force scenes (primitives staged in shared memory, <= 128 triangles): the
// same queue traced with the linear scan of core/scene.cpp:57-92 -- one ray per
// lane, every lane of a warp in the same primitive loop (no per-lane mutation
// state, so the scan runs at full warp width whatever phase each chain is in).
template <class R>
__global__ void __launch_bounds__(128)
k_wf_trace_brute(StepParams<R> P, const WfRay<R> *__restrict__ rays, WfHit<R> *__restrict__ hits,
                 unsigned *__restrict__ occ, const unsigned *n_ptr, unsigned *zero_a, unsigned *zero_b) {
    extern __shared__ __align__(16) char smem[];
    SceneView<R> S = stage_scene(P.scene, smem);
    if (blockIdx.x == 0 && threadIdx.x < kWfQueues)   // the next round's chain-queue lengths ...
        zero_a[threadIdx.x] = 0;
    if (blockIdx.x == 0 && threadIdx.x == 0)           // ... and its ray-queue length
        *zero_b = 0;
    const unsigned n = *n_ptr;
    const unsigned stride = gridDim.x * blockDim.x;
    for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const WfRay<R> r = ld_ray(rays + i);
        if (!(r.lim > R(0)))   // unused slot of a batch
            continue;
        RayReq<R> q;
        q.o = mk(r.o[0], r.o[1], r.o[2]);
        q.d = mk(r.d[0], r.d[1], r.d[2]);
        q.lim = r.lim;
        R t;
        const int prim = trace_ray<R, false>(S, q, t);
        const int c = r.ck & ((1 << kWfChainBits) - 1);
        if (r.lim < M<R>::inf()) {
            if (prim >= 0)
                atomicOr(occ + c, 1u << (static_cast<unsigned>(r.ck) >> kWfChainBits));
        } else {
            WfHit<R> h;
            h.t = t;
            h.prim = prim;
            hits[c] = h;
        }
    }
}

}  // namespace rd
