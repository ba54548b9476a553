// ramlt_wavefront.cuh -- the chain step as a wavefront (BVH scenes).
//
// The mutation of core/driver.cpp:113-171 is the resumable coroutine StepCo
// (ramlt_step_co.cuh).  Instead of tracing inside the coroutine kernel, a
// lockstep step alternates two kernels until no chain has a ray pending:
//
//   k_wf_logic  one thread per chain with a pending ray (compacted queue):
//               resume the coroutine with its hit, advance it to its next ray
//               cast (or the end of its step), append the ray to the next
//               queue with a warp-aggregated atomic;
//   k_wf_trace  persistent, one ray per lane, dynamic ray fetch and
//               while-while BVH rounds over the queue, writing (t, prim).
//
// Between rounds the coroutine state lives in HBM as 16-byte chunks indexed
// [chunk][chain] (coalesced vectorised loads/stores); the proposal vertices
// live in a [vertex][chain] array.  The trace kernel carries no mutation
// state, so it runs with far fewer registers and more warps than the fused
// coroutine kernel, and every warp of it holds rays, whatever phase each
// chain is in.  Arithmetic and RNG consumption are the coroutine's, so the
// results equal k_step_co's (and the fp64/PCG build the reference's).
#pragma once

#include "ramlt_step_co.cuh"

namespace rd {

// Pending ray of chain c: 32 B in fp32 (one sector).
template <class R> struct alignas(sizeof(R) * 8) WfRay {
    R o[3], lim;
    R d[3];
    int c;
};
template <class R> struct alignas(sizeof(R) * 2) WfHit {
    R t;
    int prim;
};

// Coroutine state carried between rounds.
template <class R, int RK> struct WfState {
    StepCo<R, RK, false> co;
    int j, jend;
};

template <class R> struct WfParams {
    const WfRay<R> *rays_in;   // previous round's queue (round > 0)
    const WfHit<R> *hits_in;
    const unsigned *n_in;
    WfRay<R> *rays_out;        // this round's queue
    unsigned *n_out;
    unsigned *trace_work;      // zeroed here for the following k_wf_trace
    uint4 *state;              // WfState as 16 B chunks: chunk k of chain c at state[k * C + c]
    GV<R> *pv;                 // proposal vertices, vertex i of chain c at pv[i * C + c]
};

template <class T> struct Chunks {
    static constexpr int K = static_cast<int>((sizeof(T) + 15) / 16);
    uint4 w[K];
};

template <class T> __device__ __forceinline__ void ld_state(T &v, const uint4 *__restrict__ base, size_t C, int c) {
    Chunks<T> b;
#pragma unroll
    for (int k = 0; k < Chunks<T>::K; ++k)
        b.w[k] = __ldcs(base + static_cast<size_t>(k) * C + c);
    memcpy(&v, &b, sizeof(T));
}
template <class T> __device__ __forceinline__ void st_state(const T &v, uint4 *__restrict__ base, size_t C, int c) {
    Chunks<T> b;
    memcpy(&b, &v, sizeof(T));
#pragma unroll
    for (int k = 0; k < Chunks<T>::K; ++k)
        __stcs(base + static_cast<size_t>(k) * C + c, b.w[k]);
}

template <class R, int RK>
__global__ void __launch_bounds__(128) k_wf_logic(StepParams<R> P, WfParams<R> W, int round0) {
    extern __shared__ __align__(16) char smem[];
    SceneView<R> S = stage_scene(P.scene, smem);
    if (blockIdx.x == 0 && threadIdx.x == 0)
        *W.trace_work = 0;
    const unsigned n = round0 ? static_cast<unsigned>(P.C) : *W.n_in;
    RayCount rc;
    const unsigned stride = gridDim.x * blockDim.x;
    for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        WfState<R, RK> s;
        int c;
        if (round0) {
            c = static_cast<int>(i);
            co_load(s.co, P, c);
            const unsigned long long my_steps =
                P.per + (static_cast<unsigned long long>(P.chain_off + c) < P.rem ? 1ull : 0ull);
            s.j = P.j0;
            s.jend = static_cast<int>(min(static_cast<unsigned long long>(P.j1), my_steps));
            if (s.j >= s.jend) {   // inactive for this launch
                if (P.record_visits)
                    P.ch.vreg[c] = -1;
                continue;
            }
        } else {
            c = W.rays_in[i].c;
            ld_state(s, W.state, static_cast<size_t>(P.C), c);
            const WfHit<R> h = W.hits_in[i];
            s.co.res_prim = h.prim;
            s.co.res_t = h.t;
        }
        const PvSmem<R> pv{W.pv + c, P.C};
        for (;;) {
            const unsigned long long index =
                P.span_start + static_cast<unsigned long long>(s.j) * P.C_total + P.chain_off + c;
            if (s.co.advance(P, S, pv, rc, index) == CO_RAY_PENDING) {
                const unsigned act = __activemask();
                const int leader = __ffs(act) - 1;
                unsigned base = 0;
                if (static_cast<int>(threadIdx.x & 31) == leader)
                    base = atomicAdd(W.n_out, static_cast<unsigned>(__popc(act)));
                base = __shfl_sync(act, base, leader);
                const unsigned slot = base + __popc(act & ((1u << (threadIdx.x & 31)) - 1u));
                WfRay<R> r;
                r.o[0] = s.co.ray.o.x, r.o[1] = s.co.ray.o.y, r.o[2] = s.co.ray.o.z;
                r.lim = s.co.ray.lim;
                r.d[0] = s.co.ray.d.x, r.d[1] = s.co.ray.d.y, r.d[2] = s.co.ray.d.z;
                r.c = c;
                W.rays_out[slot] = r;
                st_state(s, W.state, static_cast<size_t>(P.C), c);
                break;
            }
            if (++s.j >= s.jend) {
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

template <class R> __device__ __forceinline__ WfRay<R> ld_ray(const WfRay<R> *p) { return *p; }
template <> __device__ __forceinline__ WfRay<float> ld_ray<float>(const WfRay<float> *p) {
    float4 a, b;
    ldg256(p, a, b);
    WfRay<float> r;
    r.o[0] = a.x, r.o[1] = a.y, r.o[2] = a.z, r.lim = a.w;
    r.d[0] = b.x, r.d[1] = b.y, r.d[2] = b.z, r.c = __float_as_int(b.w);
    return r;
}

// c5 (tools/ab.py, one box): 12 / 10 / 8 resident blocks per SM (40 / 48 / 55
// registers) -> 75.2 / 79.7 / 80.5 M mutations/s.
#ifndef RAMLT_WF_MINBLOCKS
#define RAMLT_WF_MINBLOCKS 8
#endif
// Persistent closest-hit / any-hit tracer over the queue (the while-while
// rounds and refill rule of k_trace_bench).  `zero_next` is the counter the
// next round's k_wf_logic appends to.
template <class R>
__global__ void __launch_bounds__(128, sizeof(R) == 4 ? RAMLT_WF_MINBLOCKS : 1)
k_wf_trace(StepParams<R> P, const WfRay<R> *__restrict__ rays, WfHit<R> *__restrict__ hits,
           const unsigned *n_ptr, unsigned *work, unsigned *zero_next) {
    extern __shared__ __align__(16) char smem[];
    SceneView<R> S = stage_scene(P.scene, smem);
    if (blockIdx.x == 0 && threadIdx.x == 0)
        *zero_next = 0;
    const unsigned n = *n_ptr;
    const unsigned lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    BvhTrav<R> tv;
    int tv_sl[BvhTrav<R>::STACK - BvhTrav<R>::SSTACK];
    tv.sl = tv_sl;
    tv.ss = reinterpret_cast<int *>(smem + P.co_stack_off) + threadIdx.x;
    bool want = false, exhausted = n == 0;
    unsigned cur = 0;
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
                    tv.begin(S, mk(r.o[0], r.o[1], r.o[2]), mk(r.d[0], r.d[1], r.d[2]), r.lim,
                             r.lim < M<R>::inf());
                    cur = mine;
                    want = true;
                } else {
                    exhausted = true;
                }
            }
        }
        if (!__any_sync(0xffffffffu, want))
            break;
        for (;;) {
            const unsigned busy = __ballot_sync(0xffffffffu, want);
            const unsigned idle = __ballot_sync(0xffffffffu, !want && !exhausted);
            if (!busy || __popc(idle) >= P.refill)
                break;
            if (want && tv.step(P.scene.bvh, P.scene.nsph)) {
                WfHit<R> h;
                h.t = tv.best;
                h.prim = tv.prim(S);
                hits[cur] = h;
                want = false;
            }
        }
    }
}

}  // namespace rd
