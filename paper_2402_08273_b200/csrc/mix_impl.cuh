// mix_impl.cuh -- sm_100a kernels and host engine of the analytic-target
// adaptive MCMC harness (include/ramlt_mix.h, BASELINE.json configs[1]).
//
// The chain step is run_chain_span's (core/driver.cpp:113-171) with the light
// path replaced by a point of [0,1]^D:
//   region   r = Grid2D::cell_of(x0, x1) for RA-grid, else 0   (core/partition.cpp:16-20)
//   sigma    = exp(lambda_r / 2)                                (core/adaptation.cpp:44-50)
//   propose  y_d = x_d + sigma * normal_quantile(next_double()), d = 0..D-1
//            (core/sampling.cpp:20-60, core/rng.hpp:32-40)
//   a        = mh_accept(pi(x), pi(y), 1, 1, 1, 1) evaluated as min(1, exp(log pi(y) - log pi(x)))
//            and 0 outside the cube                         (core/mutations.cpp:198-208)
//   accept   iff a > 0 && next_double() < a                     (core/driver.cpp:168-171)
//   record_acceptance(r, a)                                     (core/adaptation.cpp:60-92)
//
// Layout: chain c's coordinate d at x[d*C + c] (coalesced SoA), log pi at
// lp[c], RNG position in rng0/rng1 (Philox draw counter | PCG state, inc).
// The target (whitening matrices, means, log normalisers) travels in the
// kernel parameter block: every thread reads the same element at the same
// time, so the constant bank broadcasts it straight into the FFMA operands.
//
// Kernels:
//   k_mix_init   x_0 ~ U[0,1]^D from stream kStreamInit + 2*id (core/driver.cpp:223)
//   k_mix_fixed  Fixed strategy: every step of a chain in registers, no sync
//   k_mix_coop   adaptive: persistent cooperative kernel, chains in registers,
//                per lockstep step a warp-shuffle / block reduction of the
//                pooled (count, fixed-point sum) and one grid barrier (Global),
//                or region-keyed warp aggregation + apply (RA-grid, literal)
//   k_mix_step + k_mix_apply_*  the same step from HBM state, one launch per
//                step (non-resident chain counts, sharded exchange)
#pragma once

#include "mix.h"
#include "ramlt_device.cuh"

#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

// back-off of the configs[1] grid barrier's spin (ns; 0 = busy spin)
#ifndef RAMLT_MIX_SPIN_NS
#define RAMLT_MIX_SPIN_NS 32
#endif

namespace rdm {
using namespace rd;

constexpr int kDMax = RAMLT_MIX_MAX_DIM;
constexpr int kKMax = RAMLT_MIX_MAX_COMP;
constexpr int kTri = kDMax * (kDMax + 1) / 2;

template <class R> struct MixTgt {
    int D, K;
    R ell[kKMax];
    R mu[kKMax][kDMax];
    R W[kKMax][kTri];   // packed lower-triangular rows: W_ij at i(i+1)/2 + j
};

template <class R> struct MixP {
    MixTgt<R> T;
    int C;                  // chains of this handle
    long long C_total, off; // sharding
    int grid_n;             // > 0: RA-grid over (x0, x1)
    int nreg;
    int L;                  // batch_size
    double gmax, gscale, target, lmin;
    unsigned long long seed;
    int trace;
    unsigned K_log;
    unsigned T_series;      // record a scalar per chain for the first T_series steps
    int series_dim;         // -1: log pi(x), else coordinate x_d
    double *series;         // [T_series][C], fp64
    // chain SoA
    R *x;                   // [D][C]
    R *lp;                  // [C]
    unsigned long long *rng0, *rng1;
    double *asum;           // [C]
    unsigned *nacc;         // [C]
    double *log_a;          // [K_log][C]
    unsigned char *log_f;   // [K_log][C]
    int *vreg;              // literal: the step's (region, a) per chain
    double *va;
    // regions
    R *sig;                 // sigma_for(r), stored as R
    double *lambda;
    unsigned long long *n;
    unsigned long long *pend_n;
    double *pend_sum;       // literal A_k
    unsigned long long *pend_fx;   // pooled A_k (2^-24 fixed point)
    double *tot_acc;        // literal lifetime tally
    unsigned long long *tot_fx, *tot_vis;
    unsigned long long *x_cnt, *x_fx, *x_last;   // pooled per-step exchange
    unsigned long long *gbuf;      // Global fast path: [3] rotating fixed-point sums
    // trace
    unsigned long long *tr_count, tr_cap, *tr_index, *tr_n;
    long long *tr_region;
    double *tr_lambda, *tr_alpha;
    int *err;
};

__device__ __forceinline__ unsigned long long mix_fx(double a) {
    return static_cast<unsigned long long>(a * 16777216.0 + 0.5);   // 2^-24 resolution
}

__device__ __forceinline__ double mix_lambda_next(double lam, double ah, unsigned long long n, double gmax,
                                                  double gscale, double target, double lmin) {
    // step_size + update_lambda (core/adaptation.cpp:10-20)
    double gs = gscale / ::sqrt(static_cast<double>(n));
    double gm = gmax < gs ? gmax : gs;
    double diff = ah - target;
    double sg = diff > 0.0 ? 1.0 : (diff < 0.0 ? -1.0 : 0.0);
    double nl = lam + gm * sg;
    return lmin > nl ? lmin : nl;
}

template <class R>
__device__ __forceinline__ void mix_trace(const MixP<R> &P, unsigned long long idx, int r, unsigned long long n0,
                                          double lam, double ah) {
    unsigned long long slot = atomicAdd(P.tr_count, 1ull);
    if (slot < P.tr_cap) {
        P.tr_index[slot] = idx;
        P.tr_region[slot] = r;
        P.tr_n[slot] = n0;
        P.tr_lambda[slot] = lam;
        P.tr_alpha[slot] = ah;
    }
}

// log pi(x) = logsumexp_k (ell_k - |W_k (x - mu_k)|^2 / 2); DT / KT > 0 fix
// D / K at compile time (configs[1]: D = 8, K = 4), 0 reads them from T.
template <class R, int DT, int KT>
__device__ __forceinline__ R log_target(const MixTgt<R> &T, const R *x) {
    constexpr int KN = KT ? KT : kKMax;
    constexpr int DN = DT ? DT : kDMax;
    const int D = DT ? DT : T.D;
    const int K = KT ? KT : T.K;
    R e[KN];
    R m = -M<R>::inf();
#pragma unroll
    for (int k = 0; k < KN; ++k) {
        if (k >= K)
            break;
        R dif[DN];
#pragma unroll
        for (int j = 0; j < DN; ++j)
            if (j < D)
                dif[j] = x[j] - T.mu[k][j];
        R s = R(0);
#pragma unroll
        for (int i = 0; i < DN; ++i) {
            if (i >= D)
                break;
            R z = R(0);
#pragma unroll
            for (int j = 0; j <= i; ++j)
                z = z + T.W[k][i * (i + 1) / 2 + j] * dif[j];
            s = s + z * z;
        }
        e[k] = T.ell[k] - R(0.5) * s;
        m = e[k] > m ? e[k] : m;
    }
    R acc = R(0);
#pragma unroll
    for (int k = 0; k < KN; ++k) {
        if (k >= K)
            break;
        acc = acc + M<R>::exp(e[k] - m);
    }
    return m + M<R>::log(acc);
}

template <class R, int DT> struct MixRegs {
    static constexpr int DN = DT ? DT : kDMax;
    R x[DN];
    R lp;
    double asum;
    unsigned nacc;
};

template <int RK> struct MixRngIO;
template <> struct MixRngIO<RNG_PCG> {
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
template <> struct MixRngIO<RNG_PHILOX> {
    static __device__ __forceinline__ void load(Rng<RNG_PHILOX> &r, const unsigned long long *a,
                                                const unsigned long long *, int c, unsigned long long seed,
                                                unsigned long long stream) {
        r.key = seed;
        r.draw = a[c];
        r.stream = stream;
        r.bid = ~0ULL;
    }
    static __device__ __forceinline__ void store(const Rng<RNG_PHILOX> &r, unsigned long long *a,
                                                 unsigned long long *, int c) {
        a[c] = r.draw;
    }
};

template <class R, int RK, int DT>
__device__ __forceinline__ void load_chain(const MixP<R> &P, int c, MixRegs<R, DT> &cs, Rng<RK> &rng) {
    const int D = DT ? DT : P.T.D;
#pragma unroll
    for (int d = 0; d < MixRegs<R, DT>::DN; ++d)
        if (d < D)
            cs.x[d] = P.x[static_cast<size_t>(d) * P.C + c];
    cs.lp = P.lp[c];
    cs.asum = P.asum[c];
    cs.nacc = P.nacc[c];
    MixRngIO<RK>::load(rng, P.rng0, P.rng1, c, P.seed, static_cast<unsigned long long>(P.off + c));
}

template <class R, int RK, int DT>
__device__ __forceinline__ void store_chain(const MixP<R> &P, int c, const MixRegs<R, DT> &cs, const Rng<RK> &rng) {
    const int D = DT ? DT : P.T.D;
#pragma unroll
    for (int d = 0; d < MixRegs<R, DT>::DN; ++d)
        if (d < D)
            P.x[static_cast<size_t>(d) * P.C + c] = cs.x[d];
    P.lp[c] = cs.lp;
    P.asum[c] = cs.asum;
    P.nacc[c] = cs.nacc;
    MixRngIO<RK>::store(rng, P.rng0, P.rng1, c);
}

template <class R, int DT>
__device__ __forceinline__ int mix_region(const MixP<R> &P, const MixRegs<R, DT> &cs) {
    if (P.grid_n <= 0)
        return 0;
    int ix = min(static_cast<int>(cs.x[0] * R(P.grid_n)), P.grid_n - 1);
    int iy = min(static_cast<int>(cs.x[1] * R(P.grid_n)), P.grid_n - 1);
    return iy * P.grid_n + ix;
}

// One step of one chain with kernel scale sigma; returns a, updates the chain.
template <class R, int RK, int DT, int KT>
__device__ __forceinline__ double mix_step(const MixP<R> &P, R sigma, MixRegs<R, DT> &cs, Rng<RK> &rng,
                                           bool &accepted) {
    constexpr int DN = MixRegs<R, DT>::DN;
    const int D = DT ? DT : P.T.D;
    R y[DN];
    bool in = true;
#pragma unroll
    for (int d = 0; d < DN; ++d) {
        if (d < D) {
            R u = Unit<R>::draw(rng);
            y[d] = cs.x[d] + sigma * nquantile<R>(u);
            in = in && (y[d] >= R(0) && y[d] <= R(1));
        }
    }
    double a = 0.0;
    R lpy = R(0);
    if (in) {
        lpy = log_target<R, DT, KT>(P.T, y);
        R rr = M<R>::exp(lpy - cs.lp);
        a = rr > R(0) ? (rr < R(1) ? static_cast<double>(rr) : 1.0) : 0.0;
    }
    accepted = false;
    if (a > 0.0) {
        R u = Unit<R>::draw(rng);
        if (u < static_cast<R>(a)) {
            accepted = true;
#pragma unroll
            for (int d = 0; d < DN; ++d)
                if (d < D)
                    cs.x[d] = y[d];
            cs.lp = lpy;
        }
    }
    cs.asum += a;
    cs.nacc += accepted ? 1u : 0u;
    return a;
}

// Uniform from the two words of one next_double (hi first): Unit<R> without the generator.
template <class R> __device__ __forceinline__ R mix_unit(uint32_t hi, uint32_t lo);
template <> __device__ __forceinline__ double mix_unit<double>(uint32_t hi, uint32_t lo) {
    return static_cast<double>(((static_cast<unsigned long long>(hi) << 32) | lo) >> 11) * 0x1.0p-53;
}
template <> __device__ __forceinline__ float mix_unit<float>(uint32_t hi, uint32_t) {
    return static_cast<float>(hi >> 8) * 0x1.0p-24f;
}

// mix_step for Philox at D = 8 (configs[1]): a step consumes words
// [c0, c0 + 16) for the 8 proposal draws and [c0 + 16, c0 + 18) for the accept
// draw, i.e. at most Philox blocks c0/4 .. c0/4 + 4 (draws come in pairs, so
// c0 % 4 is 0 or 2).  The five blocks are computed up front as five
// independent Philox chains (instruction-level parallelism instead of five
// serial out-of-line refills) and the words are picked from registers.  Same
// words, same order, same arithmetic as mix_step.
// The draw half of a configs[1] step (Philox, D = 8): every word the step can
// consume is known from the draw counter alone -- [c0, c0+16) for the
// proposal, [c0+16, c0+18) for the accept draw -- so the five Philox blocks,
// the eight normal quantiles and the accept uniform can be computed before
// sigma (the pending lambda update) is known.  k_mix_coop computes them while
// its grid barrier completes.  ok = false: odd counter alignment (generic path).
template <class R> struct Px8Pre {
    R z[8];
    R ua;
    bool ok;
};

template <class R>
__device__ __forceinline__ void px8_pre(const Rng<RNG_PHILOX> &rng, Px8Pre<R> &pre) {
    const unsigned long long c0 = rng.draw;
    const unsigned off = static_cast<unsigned>(c0 & 3ull);
    pre.ok = !(off & 1u);
    if (!pre.ok)
        return;
    const unsigned long long b = c0 >> 2;
    const uint32_t k0 = static_cast<uint32_t>(rng.key), k1 = static_cast<uint32_t>(rng.key >> 32);
    const uint32_t s0 = static_cast<uint32_t>(rng.stream), s1 = static_cast<uint32_t>(rng.stream >> 32);
    uint32_t w[20];
#pragma unroll
    for (int q = 0; q < 5; ++q) {
        uint32_t x0 = static_cast<uint32_t>(b + q), x1 = static_cast<uint32_t>((b + q) >> 32), x2 = s0, x3 = s1;
        philox10(x0, x1, x2, x3, k0, k1);
        w[4 * q] = x0;
        w[4 * q + 1] = x1;
        w[4 * q + 2] = x2;
        w[4 * q + 3] = x3;
    }
    uint32_t u[18];
#pragma unroll
    for (int i = 0; i < 18; ++i)
        u[i] = off ? w[i + 2] : w[i];
#pragma unroll
    for (int d = 0; d < 8; ++d)
        pre.z[d] = nquantile<R>(mix_unit<R>(u[2 * d], u[2 * d + 1]));
    pre.ua = mix_unit<R>(u[16], u[17]);
}

// The rest of the step once sigma is known: propose, evaluate, accept.
template <class R, int KT>
__device__ __forceinline__ double px8_finish(const MixP<R> &P, R sigma, MixRegs<R, 8> &cs, Rng<RNG_PHILOX> &rng,
                                             const Px8Pre<R> &pre, bool &accepted) {
    const unsigned long long c0 = rng.draw;
    R y[8];
    bool in = true;
#pragma unroll
    for (int d = 0; d < 8; ++d) {
        y[d] = cs.x[d] + sigma * pre.z[d];
        in = in && (y[d] >= R(0) && y[d] <= R(1));
    }
    double a = 0.0;
    R lpy = R(0);
    if (in) {
        lpy = log_target<R, 8, KT>(P.T, y);
        R rr = M<R>::exp(lpy - cs.lp);
        a = rr > R(0) ? (rr < R(1) ? static_cast<double>(rr) : 1.0) : 0.0;
    }
    accepted = false;
    if (a > 0.0 && pre.ua < static_cast<R>(a)) {
        accepted = true;
#pragma unroll
        for (int d = 0; d < 8; ++d)
            cs.x[d] = y[d];
        cs.lp = lpy;
    }
    rng.draw = c0 + (a > 0.0 ? 18ull : 16ull);
    rng.bid = ~0ULL;
    cs.asum += a;
    cs.nacc += accepted ? 1u : 0u;
    return a;
}

// configs[1] path (Philox, D = 8): the step's words are computed up front as
// independent Philox blocks (ILP) instead of serial out-of-line refills.
template <class R, int KT>
__device__ __forceinline__ double mix_step_px8(const MixP<R> &P, R sigma, MixRegs<R, 8> &cs, Rng<RNG_PHILOX> &rng,
                                               bool &accepted) {
    Px8Pre<R> pre;
    px8_pre<R>(rng, pre);
    if (!pre.ok)
        return mix_step<R, RNG_PHILOX, 8, KT>(P, sigma, cs, rng, accepted);
    return px8_finish<R, KT>(P, sigma, cs, rng, pre, accepted);
}

// Dispatch: the batched-draw form where it applies.
template <class R, int RK, int DT, int KT>
__device__ __forceinline__ double mix_step_any(const MixP<R> &P, R sigma, MixRegs<R, DT> &cs, Rng<RK> &rng,
                                               bool &accepted) {
    if constexpr (RK == RNG_PHILOX && DT == 8)
        return mix_step_px8<R, KT>(P, sigma, cs, rng, accepted);
    else
        return mix_step<R, RK, DT, KT>(P, sigma, cs, rng, accepted);
}

template <class R>
__device__ __forceinline__ void mix_log(const MixP<R> &P, int c, unsigned long long j, double a, bool acc) {
    if (j < P.K_log) {
        P.log_a[j * P.C + c] = a;
        P.log_f[j * P.C + c] = static_cast<unsigned char>((acc ? 1 : 0) | 2 | 4);
    }
}

// The chain's scalar series for autocorrelation_time (core/diagnostics.cpp:87-127):
// the state after step j.
template <class R, int DT>
__device__ __forceinline__ void mix_record(const MixP<R> &P, int c, unsigned long long j, const MixRegs<R, DT> &cs) {
    if (j < P.T_series) {
        R v = cs.lp;
#pragma unroll
        for (int d = 0; d < MixRegs<R, DT>::DN; ++d)
            if (d == P.series_dim)
                v = cs.x[d];
        P.series[j * P.C + c] = static_cast<double>(v);
    }
}

// ---- initialisation --------------------------------------------------------------------
template <class R, int RK, int DT, int KT>
__global__ void __launch_bounds__(128) k_mix_init(MixP<R> P) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= P.C)
        return;
    const int D = DT ? DT : P.T.D;
    const unsigned long long g = static_cast<unsigned long long>(P.off + c);
    MixRegs<R, DT> cs;
    Rng<RK> init;
    init.reseed(P.seed, kStreamInit + 2ull * g);
    bool ok = false;
    for (int attempt = 0; attempt < 1000 && !ok; ++attempt) {
#pragma unroll
        for (int d = 0; d < MixRegs<R, DT>::DN; ++d)
            if (d < D)
                cs.x[d] = Unit<R>::draw(init);
        cs.lp = log_target<R, DT, KT>(P.T, cs.x);
        ok = M<R>::finite(cs.lp);
    }
    if (!ok)
        atomicExch(P.err, 1);
    cs.asum = 0.0;
    cs.nacc = 0;
    Rng<RK> rng;
    rng.reseed(P.seed, g);
    store_chain<R, RK, DT>(P, c, cs, rng);
}

// ---- Fixed strategy: no shared state, every step in registers ----------------------------
template <class R, int RK, int DT, int KT>
__global__ void __launch_bounds__(128) k_mix_fixed(MixP<R> P, unsigned long long j0, unsigned long long j1) {
    const R sigma = P.sig[0];
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < P.C; c += gridDim.x * blockDim.x) {
        MixRegs<R, DT> cs;
        Rng<RK> rng;
        load_chain<R, RK, DT>(P, c, cs, rng);
        for (unsigned long long j = j0; j < j1; ++j) {
            bool acc;
            double a = mix_step_any<R, RK, DT, KT>(P, sigma, cs, rng, acc);
            mix_log(P, c, j, a, acc);
            mix_record(P, c, j, cs);
        }
        store_chain<R, RK, DT>(P, c, cs, rng);
    }
}

// ---- adaptation: literal rule (canonical chain order, batches of exactly L) -------------
template <class R>
__device__ void mix_apply_literal(const MixP<R> &P, unsigned long long j) {
    for (int ci = 0; ci < P.C; ++ci) {
        int r = __ldcg(&P.vreg[ci]);
        double a = __ldcg(&P.va[ci]);
        P.tot_acc[r] += a;
        P.tot_vis[r] += 1;
        double ps = P.pend_sum[r] + a;
        unsigned long long pn = P.pend_n[r] + 1;
        if (pn >= static_cast<unsigned long long>(P.L)) {
            double ah = ps / static_cast<double>(pn);
            ah = ah < 0.0 ? 0.0 : (ah > 1.0 ? 1.0 : ah);
            unsigned long long n0 = P.n[r];
            double lam = mix_lambda_next(P.lambda[r], ah, n0, P.gmax, P.gscale, P.target, P.lmin);
            P.lambda[r] = lam;
            P.n[r] = n0 + 1;
            P.sig[r] = static_cast<R>(::exp(0.5 * lam));
            if (P.trace)
                mix_trace(P, j * static_cast<unsigned long long>(P.C_total) + P.off + ci, r, n0, lam, ah);
            ps = 0.0;
            pn = 0;
        }
        P.pend_sum[r] = ps;
        P.pend_n[r] = pn;
    }
}

// ---- adaptation: pooled rule, region-keyed warp aggregation --------------------------------
template <class R>
__device__ __forceinline__ void mix_accum_pooled(const MixP<R> &P, int r, double a, unsigned long long idx) {
    unsigned peers = __match_any_sync(0xffffffffu, r);
    if (r < 0)
        return;
    unsigned fx = static_cast<unsigned>(mix_fx(a));            // <= 2^24; 32 lanes <= 2^29
    unsigned s = __reduce_add_sync(peers, fx);
    int hi = 31 - __clz(peers);
    unsigned long long last = __shfl_sync(peers, idx, hi);   // the group's highest chain = last visit
    if ((threadIdx.x & 31) == __ffs(peers) - 1) {
        atomicAdd(&P.x_cnt[r], static_cast<unsigned long long>(__popc(peers)));
        atomicAdd(&P.x_fx[r], static_cast<unsigned long long>(s));
        atomicMax(&P.x_last[r], last);
    }
}

template <class R>
__device__ __forceinline__ void mix_apply_pooled_region(const MixP<R> &P, int r) {
    unsigned long long cnt = __ldcg(&P.x_cnt[r]);
    if (cnt == 0)
        return;
    unsigned long long fx = __ldcg(&P.x_fx[r]), last = __ldcg(&P.x_last[r]);
    P.x_cnt[r] = 0;
    P.x_fx[r] = 0;
    P.x_last[r] = 0;
    P.tot_vis[r] += cnt;
    P.tot_fx[r] += fx;
    unsigned long long pn = P.pend_n[r] + cnt;
    unsigned long long pf = P.pend_fx[r] + fx;
    if (pn < static_cast<unsigned long long>(P.L)) {
        P.pend_n[r] = pn;
        P.pend_fx[r] = pf;
        return;
    }
    double ah = static_cast<double>(pf) / 16777216.0 / static_cast<double>(pn);
    ah = ah < 0.0 ? 0.0 : (ah > 1.0 ? 1.0 : ah);
    unsigned long long n0 = P.n[r];
    double lam = mix_lambda_next(P.lambda[r], ah, n0, P.gmax, P.gscale, P.target, P.lmin);
    P.lambda[r] = lam;
    P.n[r] = n0 + 1;
    P.pend_n[r] = 0;
    P.pend_fx[r] = 0;
    P.sig[r] = static_cast<R>(::exp(0.5 * lam));
    if (P.trace)
        mix_trace(P, last, r, n0, lam, ah);
}

// ---- one step from HBM state (non-resident / sharded) --------------------------------------
template <class R, int RK, int DT, int KT>
__global__ void __launch_bounds__(128) k_mix_step(MixP<R> P, unsigned long long j, int pooled) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    const bool active = c < P.C;
    int r = -1;
    double a = 0.0;
    if (active) {
        MixRegs<R, DT> cs;
        Rng<RK> rng;
        load_chain<R, RK, DT>(P, c, cs, rng);
        r = mix_region(P, cs);
        bool acc;
        a = mix_step_any<R, RK, DT, KT>(P, __ldcg(&P.sig[r]), cs, rng, acc);
        mix_log(P, c, j, a, acc);
        mix_record(P, c, j, cs);
        store_chain<R, RK, DT>(P, c, cs, rng);
        if (!pooled) {
            P.vreg[c] = r;
            P.va[c] = a;
        }
    }
    if (pooled)
        mix_accum_pooled(P, r, a, j * static_cast<unsigned long long>(P.C_total) + P.off + c);
}

template <class R> __global__ void k_mix_apply_pooled(MixP<R> P) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < P.nreg; r += gridDim.x * blockDim.x)
        mix_apply_pooled_region(P, r);
}

template <class R> __global__ void k_mix_apply_literal(MixP<R> P, unsigned long long j) {
    if (blockIdx.x == 0 && threadIdx.x == 0)
        mix_apply_literal(P, j);
}

// ---- persistent cooperative kernel (adaptive strategies) -----------------------------------
// mode 0: Global + pooled -- the region state is replicated in every thread's
//         registers; per step one block-reduced 64-bit atomic per block into a
//         rotating 3-slot buffer that doubles as the grid barrier (arrival
//         count in the high bits, no cooperative-groups barrier); every thread
//         then applies the identical update (slot j+2 is cleared by thread 0:
//         its last readers arrived at step j, its next writers wait for step j+1).
// mode 1: pooled, any partition: region-keyed warp aggregation, barrier,
//         grid-stride apply, barrier.
// mode 2: literal: per-chain (region, a) to HBM, barrier, canonical-order
//         sequential apply by one thread, barrier.
template <class R, int RK, int DT, int KT>
__global__ void __launch_bounds__(512) k_mix_coop(MixP<R> P, unsigned long long j0, unsigned long long j1, int mode) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    __shared__ unsigned long long wsum[8];
    __shared__ R wsig;
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    const bool active = c < P.C;
    MixRegs<R, DT> cs;
    Rng<RK> rng;
    if (active)
        load_chain<R, RK, DT>(P, c, cs, rng);
    // Global fast-path replica of region 0
    double lam = P.lambda[0];
    unsigned long long n = P.n[0], pn = P.pend_n[0], pf = P.pend_fx[0];
    unsigned long long tfx = 0, tvis = 0;
    R sigma = P.sig[0];
    // mode 0 with Philox and D = 8: the next step's draws are computed between
    // the barrier arrival and the wait (split-phase barrier), hiding the wait
    constexpr bool kPre = RK == RNG_PHILOX && DT == 8;
    Px8Pre<R> pre;
    bool have_pre = false;
    for (unsigned long long j = j0; j < j1; ++j) {
        int r = -1;
        double a = 0.0;
        if (active) {
            r = mix_region(P, cs);
            bool acc;
            if constexpr (kPre) {
                if (mode == 0 && have_pre && pre.ok)
                    a = px8_finish<R, KT>(P, sigma, *reinterpret_cast<MixRegs<R, 8> *>(&cs), rng, pre, acc);
                else
                    a = mix_step_any<R, RK, DT, KT>(P, mode == 0 ? sigma : __ldcg(&P.sig[r]), cs, rng, acc);
            } else {
                a = mix_step_any<R, RK, DT, KT>(P, mode == 0 ? sigma : __ldcg(&P.sig[r]), cs, rng, acc);
            }
            have_pre = false;
            mix_log(P, c, j, a, acc);
            mix_record(P, c, j, cs);
        }
        const unsigned long long idx0 = j * static_cast<unsigned long long>(P.C_total) + P.off;
        if (mode == 0) {
            // One 64-bit atomic per block is both the data and the barrier
            // arrival: bits 48.. count arrived blocks, bits 0..47 carry the
            // fixed-point sum (<= 65,536 chains x 2^24 < 2^41).  Thread 0 spins
            // until every block arrived, then the block reads the total.
            unsigned fx = active ? static_cast<unsigned>(mix_fx(a)) : 0u;
            unsigned ws = __reduce_add_sync(0xffffffffu, fx);
            if ((threadIdx.x & 31) == 0)
                wsum[threadIdx.x >> 5] = ws;
            __syncthreads();
            unsigned long long v = 0;
            if (threadIdx.x == 0) {   // arrive
                unsigned long long b = 1ull << 48;
                for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w)
                    b += wsum[w];
                v = atomicAdd(&P.gbuf[j % 3], b) + b;
            }
            if constexpr (kPre) {   // overlap: the next step's words do not depend on sigma
                if (active && j + 1 < j1) {
                    px8_pre<R>(*reinterpret_cast<Rng<RNG_PHILOX> *>(&rng), pre);
                    have_pre = true;
                }
            }
            if (threadIdx.x == 0) {   // wait
                const unsigned long long want = static_cast<unsigned long long>(gridDim.x);
                while ((v >> 48) < want) {
                    if (RAMLT_MIX_SPIN_NS > 0)
                        __nanosleep(RAMLT_MIX_SPIN_NS);
                    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(&P.gbuf[j % 3]) : "memory");
                }
                // the region update once per block (thread 0 holds the replica)
                unsigned long long fxs = v & ((1ull << 48) - 1);
                unsigned long long cnt = static_cast<unsigned long long>(P.C);
                tfx += fxs;
                tvis += cnt;
                pn += cnt;
                pf += fxs;
                if (pn >= static_cast<unsigned long long>(P.L)) {
                    double ah = static_cast<double>(pf) / 16777216.0 / static_cast<double>(pn);
                    ah = ah < 0.0 ? 0.0 : (ah > 1.0 ? 1.0 : ah);
                    unsigned long long n0 = n;
                    lam = mix_lambda_next(lam, ah, n0, P.gmax, P.gscale, P.target, P.lmin);
                    n = n0 + 1;
                    pn = 0;
                    pf = 0;
                    sigma = static_cast<R>(::exp(0.5 * lam));
                    if (c == 0 && P.trace)
                        mix_trace(P, idx0 + P.C - 1, 0, n0, lam, ah);
                }
                wsig = sigma;
                if (c == 0) {
                    P.gbuf[(j + 2) % 3] = 0;   // its readers all arrived at step j; next written after step j+1
                    __threadfence();
                }
            }
            __syncthreads();
            sigma = wsig;
        } else if (mode == 1) {
            mix_accum_pooled(P, r, a, idx0 + c);
            grid.sync();
            for (int rr = c; rr < P.nreg; rr += gridDim.x * blockDim.x)
                mix_apply_pooled_region(P, rr);
            grid.sync();
        } else {
            if (active) {
                P.vreg[c] = r;
                P.va[c] = a;
            }
            grid.sync();
            if (c == 0)
                mix_apply_literal(P, j);
            grid.sync();
        }
    }
    if (active)
        store_chain<R, RK, DT>(P, c, cs, rng);
    if (mode == 0 && c == 0) {
        P.lambda[0] = lam;
        P.n[0] = n;
        P.pend_n[0] = pn;
        P.pend_fx[0] = pf;
        P.tot_fx[0] += tfx;
        P.tot_vis[0] += tvis;
        P.sig[0] = sigma;
    }
}

// ---- autocorrelation_time (core/diagnostics.cpp:87-127) on device -------------------------
// One block per selected chain: the series (stride C in the [T][C] record) is
// staged in shared memory, mean / variance / rho(k) are block reductions in a
// fixed order, and thread 0 runs Geyer's initial positive sequence exactly as
// the reference (pairs rho(2m) + rho(2m+1) while positive, up to lag n/2).
// status: 0 ok, 3 series shorter than 1000 or without variance (the reference
// throws std::invalid_argument).
__device__ __forceinline__ double block_sum(double v, double *red) {
    red[threadIdx.x] = v;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
        if (static_cast<int>(threadIdx.x) < w)
            red[threadIdx.x] += red[threadIdx.x + w];
        __syncthreads();
    }
    double r = red[0];
    __syncthreads();
    return r;
}

__global__ void __launch_bounds__(256) k_autocorr(const double *series, int C, int n, int first, double *tau,
                                                  double *n_eff, double *sigma2, int *status) {
    extern __shared__ double sm[];   // n series values + 256 reduction slots
    double *sv = sm, *red = sm + n;
    const int c = first + blockIdx.x;
    for (int i = threadIdx.x; i < n; i += blockDim.x)
        sv[i] = series[static_cast<size_t>(i) * C + c];
    __syncthreads();
    double part = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x)
        part += sv[i];
    const double mean = block_sum(part, red) / static_cast<double>(n);
    part = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x)
        part += (sv[i] - mean) * (sv[i] - mean);
    const double var = block_sum(part, red) / static_cast<double>(n);
    if (n < 1000 || !(var > 0.0)) {
        if (threadIdx.x == 0) {
            status[blockIdx.x] = 3;
            tau[blockIdx.x] = n_eff[blockIdx.x] = sigma2[blockIdx.x] = 0.0;
        }
        return;
    }
    for (int i = threadIdx.x; i < n; i += blockDim.x)
        sv[i] -= mean;
    __syncthreads();
    double t = -1.0;
    const int max_lag = n / 2;
    for (int m = 0;; ++m) {
        const int k0 = 2 * m, k1 = 2 * m + 1;
        if (k1 > max_lag)
            break;
        double p0 = 0.0, p1 = 0.0;
        for (int i = threadIdx.x; i + k0 < n; i += blockDim.x) {
            p0 += sv[i] * sv[i + k0];
            if (i + k1 < n)
                p1 += sv[i] * sv[i + k1];
        }
        const double r0 = block_sum(p0, red) / (static_cast<double>(n) * var);
        const double r1 = block_sum(p1, red) / (static_cast<double>(n) * var);
        const double gamma = r0 + r1;
        if (gamma <= 0.0)
            break;
        t += 2.0 * gamma;
    }
    t = t > 1e-3 ? t : 1e-3;
    if (threadIdx.x == 0) {
        status[blockIdx.x] = 0;
        tau[blockIdx.x] = t;
        n_eff[blockIdx.x] = static_cast<double>(n) / t;
        sigma2[blockIdx.x] = t / static_cast<double>(n) * var;
    }
}

}  // namespace rdm

namespace ramlt_b200 {

#define RAMLT_MCUDA(x)                                                                             \
    do {                                                                                           \
        cudaError_t e_ = (x);                                                                      \
        if (e_ != cudaSuccess)                                                                     \
            throw CudaError(std::string("cuda: ") + cudaGetErrorString(e_) + " at " #x);           \
    } while (0)

template <class T> struct MBuf {
    T *p = nullptr;
    size_t n = 0;
    void alloc(size_t count) {
        free();
        n = count;
        if (count)
            RAMLT_MCUDA(cudaMalloc(&p, count * sizeof(T)));
    }
    void zero(cudaStream_t s) {
        if (n)
            RAMLT_MCUDA(cudaMemsetAsync(p, 0, n * sizeof(T), s));
    }
    void up(const T *h, size_t count) {
        RAMLT_MCUDA(cudaMemcpy(p, h, count * sizeof(T), cudaMemcpyHostToDevice));
    }
    void down(T *h, size_t count) const {
        RAMLT_MCUDA(cudaMemcpy(h, p, count * sizeof(T), cudaMemcpyDeviceToHost));
    }
    void free() {
        if (p)
            cudaFree(p);
        p = nullptr;
        n = 0;
    }
    ~MBuf() { free(); }
};

template <class R> class MixEngineT final : public MixEngineBase {
public:
    MixEngineT(const MixHostTarget &t, const ramlt_mix_desc &d);
    ~MixEngineT() override;
    void init_chains() override;
    void run(uint64_t steps) override;
    void synchronize() override { RAMLT_MCUDA(cudaStreamSynchronize(stream_)); }
    void set_stream(void *s) override {
        if (own_stream_ && stream_)
            cudaStreamDestroy(stream_);
        stream_ = static_cast<cudaStream_t>(s);
        own_stream_ = false;
    }
    void read_stats(ramlt_mix_stats *out) override;
    void read_state(double *x, double *lp) override;
    void read_chain_tallies(double *asum, uint64_t *nacc) override;
    uint64_t read_regions(double *lambda, uint64_t *n, double *acc, uint64_t *vis, uint64_t cap) override;
    uint64_t read_trace(ramlt_trace_row *rows, uint64_t cap) override;
    void read_decisions(uint32_t K, double *a, uint8_t *flags) override;
    void read_series(double *out) override;
    void autocorrelation(int first, int count, double *tau, double *n_eff, double *sigma2, int32_t *status) override;
    void adapt_exchange(uint64_t **cnt, uint64_t **fx, uint64_t **last, uint64_t *n) override {
        *cnt = reinterpret_cast<uint64_t *>(x_cnt_.p);
        *fx = reinterpret_cast<uint64_t *>(x_fx_.p);
        *last = reinterpret_cast<uint64_t *>(x_last_.p);
        *n = static_cast<uint64_t>(nreg_);
    }
    void adapt_apply() override;
    void set_external(bool on) override {
        if (on && adapt_ == 0 && ctl_ != 0)
            throw std::logic_error("external adaptation needs the pooled rule");
        external_ = on;
    }

private:
    rdm::MixP<R> params() const;
    template <int RK, int DT, int KT> void launch_run(uint64_t steps);
    void check_err(const char *what);
    void drain_events();

    ramlt_mix_desc d_;
    MixHostTarget ht_;
    rdm::MixTgt<R> tgt_{};
    int C_, D_, K_, nreg_;
    long long Ctot_, off_;
    int ctl_;        // 0 fixed, 1 global, 2 ra-grid
    int adapt_;      // 0 literal, 1 pooled
    bool external_ = false;
    bool ready_ = false;
    cudaStream_t stream_ = nullptr;
    bool own_stream_ = true;
    int coop_blocks_ = -1;   // resident capacity of k_mix_coop in blocks (-1 unknown)
    int coop_threads_ = 0;   // 0: SM-balanced blocks; RAMLT_MIX_COOP_THREADS: a fixed block size (multiple of 32)
    uint64_t steps_ = 0, launches_ = 0;
    MBuf<R> x_, lp_, sig_;
    MBuf<unsigned long long> rng0_, rng1_;
    MBuf<double> asum_;
    MBuf<unsigned> nacc_;
    MBuf<double> log_a_;
    MBuf<unsigned char> log_f_;
    MBuf<double> series_;
    MBuf<int> vreg_, err_;
    MBuf<double> va_, lambda_, pend_sum_, tot_acc_;
    MBuf<unsigned long long> n_, pend_n_, pend_fx_, tot_fx_, tot_vis_, x_cnt_, x_fx_, x_last_, gbuf_;
    MBuf<unsigned long long> tr_count_, tr_index_, tr_n_;
    MBuf<long long> tr_region_;
    MBuf<double> tr_lambda_, tr_alpha_;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_;
    double step_ms_ = 0.0;
    uint64_t step_launches_ = 0;
};

template <class R>
MixEngineT<R>::MixEngineT(const MixHostTarget &t, const ramlt_mix_desc &d) : d_(d), ht_(t) {
    if (d.chains < 1)
        throw std::logic_error("need at least one chain");
    if (d.batch_size < 1)
        throw std::logic_error("batch_size must be >= 1");
    if (d.strategy != RAMLT_FIXED && d.strategy != RAMLT_GLOBAL && d.strategy != RAMLT_RA_GRID)
        throw std::invalid_argument("mix: strategy must be fixed, global or ra-grid");
    if (d.strategy == RAMLT_RA_GRID && (d.grid_n < 1 || t.D < 2))
        throw std::logic_error("grid size must be >= 1 and the target at least 2-D");
    if (d.rng != RAMLT_RNG_PCG32 && d.rng != RAMLT_RNG_PHILOX)
        throw std::invalid_argument("mix: unknown rng");
    if (d.device >= 0)
        RAMLT_MCUDA(cudaSetDevice(d.device));
    RAMLT_MCUDA(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
    if (const char *v = std::getenv("RAMLT_MIX_COOP_THREADS"))
        coop_threads_ = std::max(0, std::min(512, std::atoi(v) / 32 * 32));
    C_ = d.chains;
    D_ = t.D;
    K_ = t.K;
    Ctot_ = d.chains_total > 0 ? d.chains_total : d.chains;
    off_ = d.chain_offset;
    if (off_ < 0 || off_ + C_ > Ctot_)
        throw std::logic_error("chain shard outside [0, chains_total)");
    ctl_ = d.strategy == RAMLT_FIXED ? 0 : (d.strategy == RAMLT_GLOBAL ? 1 : 2);
    nreg_ = ctl_ == 2 ? d.grid_n * d.grid_n : 1;
    adapt_ = d.adapt_mode;
    if (adapt_ < 0)
        adapt_ = Ctot_ <= 4096 ? 0 : 1;
    if (Ctot_ != C_ && ctl_ != 0)
        adapt_ = 1;   // sharded adaptive runs use the pooled rule (G-invariant)

    tgt_.D = D_;
    tgt_.K = K_;
    for (int k = 0; k < K_; ++k) {
        tgt_.ell[k] = static_cast<R>(t.ell[k]);
        for (int j = 0; j < D_; ++j)
            tgt_.mu[k][j] = static_cast<R>(t.mu[static_cast<size_t>(k) * D_ + j]);
        for (int i = 0; i < D_; ++i)
            for (int j = 0; j <= i; ++j)
                tgt_.W[k][i * (i + 1) / 2 + j] = static_cast<R>(t.W[(static_cast<size_t>(k) * D_ + i) * D_ + j]);
    }

    x_.alloc(static_cast<size_t>(D_) * C_);
    lp_.alloc(C_);
    rng0_.alloc(C_);
    rng1_.alloc(C_);
    asum_.alloc(C_);
    nacc_.alloc(C_);
    vreg_.alloc(C_);
    va_.alloc(C_);
    err_.alloc(1);
    if (d.series_dim < -1 || d.series_dim >= t.D)
        throw std::invalid_argument("mix: series_dim must be -1 (log pi) or a coordinate index");
    if (d.series_steps)
        series_.alloc(static_cast<size_t>(d.series_steps) * C_);
    if (d.log_steps) {
        log_a_.alloc(static_cast<size_t>(d.log_steps) * C_);
        log_f_.alloc(static_cast<size_t>(d.log_steps) * C_);
    }
    sig_.alloc(nreg_);
    lambda_.alloc(nreg_);
    pend_sum_.alloc(nreg_);
    tot_acc_.alloc(nreg_);
    n_.alloc(nreg_);
    pend_n_.alloc(nreg_);
    pend_fx_.alloc(nreg_);
    tot_fx_.alloc(nreg_);
    tot_vis_.alloc(nreg_);
    x_cnt_.alloc(nreg_);
    x_fx_.alloc(nreg_);
    x_last_.alloc(nreg_);
    gbuf_.alloc(3);
    size_t tcap = d.trace_enabled ? (d.trace_capacity ? d.trace_capacity : (1u << 20)) : 1;
    tr_count_.alloc(1);
    tr_index_.alloc(tcap);
    tr_n_.alloc(tcap);
    tr_region_.alloc(tcap);
    tr_lambda_.alloc(tcap);
    tr_alpha_.alloc(tcap);
    // regions: lambda_init, n = 1 (RegionState, adaptation.hpp:35-44)
    std::vector<double> lam(nreg_, d.lambda_init);
    std::vector<unsigned long long> ones(nreg_, 1ull);
    std::vector<R> sg(nreg_, static_cast<R>(std::exp(0.5 * d.lambda_init)));
    lambda_.up(lam.data(), nreg_);
    n_.up(ones.data(), nreg_);
    sig_.up(sg.data(), nreg_);
    for (auto *b : {&pend_n_, &pend_fx_, &tot_fx_, &tot_vis_, &x_cnt_, &x_fx_, &x_last_, &gbuf_, &tr_count_})
        RAMLT_MCUDA(cudaMemset(b->p, 0, b->n * sizeof(unsigned long long)));
    RAMLT_MCUDA(cudaMemset(pend_sum_.p, 0, nreg_ * sizeof(double)));
    RAMLT_MCUDA(cudaMemset(tot_acc_.p, 0, nreg_ * sizeof(double)));
    RAMLT_MCUDA(cudaMemset(err_.p, 0, sizeof(int)));
}

template <class R> MixEngineT<R>::~MixEngineT() {
    for (auto &e : ev_) {
        cudaEventDestroy(e.first);
        cudaEventDestroy(e.second);
    }
    if (own_stream_ && stream_)
        cudaStreamDestroy(stream_);
}

template <class R> rdm::MixP<R> MixEngineT<R>::params() const {
    rdm::MixP<R> P;
    std::memset(&P, 0, sizeof(P));
    P.T = tgt_;
    P.C = C_;
    P.C_total = Ctot_;
    P.off = off_;
    P.grid_n = ctl_ == 2 ? d_.grid_n : 0;
    P.nreg = nreg_;
    P.L = d_.batch_size;
    P.gmax = d_.gamma_max;
    P.gscale = d_.gamma_scale;
    P.target = d_.target_acceptance;
    P.lmin = d_.lambda_min;
    P.seed = d_.seed;
    P.trace = d_.trace_enabled;
    P.K_log = d_.log_steps;
    P.T_series = d_.series_steps;
    P.series_dim = d_.series_dim;
    P.series = series_.p;
    P.x = x_.p;
    P.lp = lp_.p;
    P.rng0 = rng0_.p;
    P.rng1 = rng1_.p;
    P.asum = asum_.p;
    P.nacc = nacc_.p;
    P.log_a = log_a_.p;
    P.log_f = log_f_.p;
    P.vreg = vreg_.p;
    P.va = va_.p;
    P.sig = sig_.p;
    P.lambda = lambda_.p;
    P.n = n_.p;
    P.pend_n = pend_n_.p;
    P.pend_sum = pend_sum_.p;
    P.pend_fx = pend_fx_.p;
    P.tot_acc = tot_acc_.p;
    P.tot_fx = tot_fx_.p;
    P.tot_vis = tot_vis_.p;
    P.x_cnt = x_cnt_.p;
    P.x_fx = x_fx_.p;
    P.x_last = x_last_.p;
    P.gbuf = gbuf_.p;
    P.tr_count = tr_count_.p;
    P.tr_cap = tr_index_.n;
    P.tr_index = tr_index_.p;
    P.tr_n = tr_n_.p;
    P.tr_region = tr_region_.p;
    P.tr_lambda = tr_lambda_.p;
    P.tr_alpha = tr_alpha_.p;
    P.err = err_.p;
    return P;
}

template <class R> void MixEngineT<R>::check_err(const char *what) {
    int e = 0;
    RAMLT_MCUDA(cudaMemcpyAsync(&e, err_.p, sizeof(int), cudaMemcpyDeviceToHost, stream_));
    RAMLT_MCUDA(cudaStreamSynchronize(stream_));
    if (e)
        throw std::runtime_error(std::string("mix: ") + what);
}

template <class R, int RK, int DT, int KT> static void mix_init_launch(const rdm::MixP<R> &P, cudaStream_t s) {
    rdm::k_mix_init<R, RK, DT, KT><<<(P.C + 127) / 128, 128, 0, s>>>(P);
}

template <class R> void MixEngineT<R>::init_chains() {
    using namespace rd;
    rdm::MixP<R> P = params();
#define RAMLT_MIX_INIT(RK, DT, KT) mix_init_launch<R, RK, DT, KT>(P, stream_)
    if (d_.rng == RAMLT_RNG_PHILOX) {
        if (D_ == 8 && K_ == 4) RAMLT_MIX_INIT(RNG_PHILOX, 8, 4); else RAMLT_MIX_INIT(RNG_PHILOX, 0, 0);
    } else {
        if (D_ == 8 && K_ == 4) RAMLT_MIX_INIT(RNG_PCG, 8, 4); else RAMLT_MIX_INIT(RNG_PCG, 0, 0);
    }
#undef RAMLT_MIX_INIT
    RAMLT_MCUDA(cudaGetLastError());
    ++launches_;
    check_err("chain initialisation found no state with finite log density");
    ready_ = true;
}

template <class R> void MixEngineT<R>::drain_events() {
    for (auto &e : ev_) {
        float ms = 0.f;
        RAMLT_MCUDA(cudaEventSynchronize(e.second));
        RAMLT_MCUDA(cudaEventElapsedTime(&ms, e.first, e.second));
        step_ms_ += ms;
        ++step_launches_;
        cudaEventDestroy(e.first);
        cudaEventDestroy(e.second);
    }
    ev_.clear();
}

template <class R>
template <int RK, int DT, int KT>
void MixEngineT<R>::launch_run(uint64_t steps) {
    rdm::MixP<R> P = params();
    const int threads = 128;
    const int blocks = (C_ + threads - 1) / threads;
    // cooperative kernel: 256-thread blocks halve the barrier arrivals; the
    // busiest SM holds the same number of chains as with 128-thread blocks
    // cooperative kernel: every SM gets the same number of chains (k blocks per
    // SM of ceil(C / (k SMs)) threads rounded up to a warp, <= 256): fixed
    // 256-thread blocks made 256 blocks for 65,536 chains on 148 SMs, so the
    // barrier waited every step for the SMs holding two blocks.
    int cthreads = coop_threads_;
    if (cthreads <= 0) {
        int dev = 0, nsm = 148;
        RAMLT_MCUDA(cudaGetDevice(&dev));
        RAMLT_MCUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
        const int per_block = 256;
        const int k = std::max(1, (C_ + nsm * per_block - 1) / (nsm * per_block));
        const int nb = nsm * k;
        cthreads = std::min(per_block, std::max(32, ((C_ + nb - 1) / nb + 31) / 32 * 32));
    }
    const int cblocks = (C_ + cthreads - 1) / cthreads;
    auto ev_begin = [&]() -> std::pair<cudaEvent_t, cudaEvent_t> {
        std::pair<cudaEvent_t, cudaEvent_t> e{nullptr, nullptr};
        if (d_.profile_kernels) {
            RAMLT_MCUDA(cudaEventCreate(&e.first));
            RAMLT_MCUDA(cudaEventCreate(&e.second));
            RAMLT_MCUDA(cudaEventRecord(e.first, stream_));
        }
        return e;
    };
    auto ev_end = [&](std::pair<cudaEvent_t, cudaEvent_t> e) {
        if (d_.profile_kernels) {
            RAMLT_MCUDA(cudaEventRecord(e.second, stream_));
            ev_.push_back(e);
        }
    };
    unsigned long long j0 = steps_, j1 = steps_ + steps;
    if (ctl_ == 0) {
        // Fixed: one launch, grid sized to the chains (no shared state)
        auto e = ev_begin();
        rdm::k_mix_fixed<R, RK, DT, KT><<<blocks, threads, 0, stream_>>>(P, j0, j1);
        RAMLT_MCUDA(cudaGetLastError());
        ev_end(e);
        ++launches_;
        return;
    }
    if (coop_blocks_ < 0) {
        int dev = 0, nsm = 0, per = 0, coop = 0;
        RAMLT_MCUDA(cudaGetDevice(&dev));
        RAMLT_MCUDA(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev));
        RAMLT_MCUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
        RAMLT_MCUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, rdm::k_mix_coop<R, RK, DT, KT>, cthreads, 0));
        coop_blocks_ = coop ? per * nsm : 0;
    }
    const bool coop = !external_ && d_.cooperative && cblocks <= coop_blocks_;
    if (coop) {
        int mode = adapt_ == 0 ? 2 : (ctl_ == 1 ? 0 : 1);
        const uint64_t chunk = 1024;   // bound one launch's duration
        for (unsigned long long a = j0; a < j1; a += chunk) {
            unsigned long long b = std::min<unsigned long long>(j1, a + chunk);
            void *args[] = {&P, &a, &b, &mode};
            auto e = ev_begin();
            RAMLT_MCUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void *>(rdm::k_mix_coop<R, RK, DT, KT>),
                                                    dim3(cblocks), dim3(cthreads), args, 0, stream_));
            ev_end(e);
            ++launches_;
        }
        return;
    }
    if (external_ && steps != 1)
        throw std::logic_error("external adaptation advances one lockstep step per run()");
    const int pooled = adapt_ == 1 ? 1 : 0;
    for (unsigned long long j = j0; j < j1; ++j) {
        auto e = ev_begin();
        rdm::k_mix_step<R, RK, DT, KT><<<blocks, threads, 0, stream_>>>(P, j, pooled);
        RAMLT_MCUDA(cudaGetLastError());
        ev_end(e);
        ++launches_;
        if (external_)
            break;   // the caller exchanges and calls adapt_apply
        if (pooled)
            rdm::k_mix_apply_pooled<R><<<(nreg_ + 127) / 128, 128, 0, stream_>>>(P);
        else
            rdm::k_mix_apply_literal<R><<<1, 32, 0, stream_>>>(P, j);
        RAMLT_MCUDA(cudaGetLastError());
        ++launches_;
    }
}

template <class R> void MixEngineT<R>::run(uint64_t steps) {
    using namespace rd;
    if (!ready_)
        throw std::logic_error("mix: init_chains() must run before run()");
    if (steps == 0)
        return;
    if (d_.rng == RAMLT_RNG_PHILOX) {
        if (D_ == 8 && K_ == 4) launch_run<RNG_PHILOX, 8, 4>(steps); else launch_run<RNG_PHILOX, 0, 0>(steps);
    } else {
        if (D_ == 8 && K_ == 4) launch_run<RNG_PCG, 8, 4>(steps); else launch_run<RNG_PCG, 0, 0>(steps);
    }
    steps_ += steps;
}

template <class R> void MixEngineT<R>::adapt_apply() {
    rdm::MixP<R> P = params();
    rdm::k_mix_apply_pooled<R><<<(nreg_ + 127) / 128, 128, 0, stream_>>>(P);
    RAMLT_MCUDA(cudaGetLastError());
    ++launches_;
}

template <class R> void MixEngineT<R>::read_stats(ramlt_mix_stats *out) {
    synchronize();
    drain_events();
    std::vector<double> as(C_);
    std::vector<unsigned> na(C_);
    asum_.down(as.data(), C_);
    nacc_.down(na.data(), C_);
    double s = 0.0;
    uint64_t acc = 0;
    for (int c = 0; c < C_; ++c) {
        s += as[c];
        acc += na[c];
    }
    unsigned long long nt = 0;
    tr_count_.down(&nt, 1);
    std::memset(out, 0, sizeof(*out));
    out->steps = steps_;
    out->proposals = steps_ * static_cast<uint64_t>(C_);
    out->accepted = acc;
    out->acceptance_sum = s;
    out->mean_acceptance = out->proposals ? s / static_cast<double>(out->proposals) : 0.0;
    out->region_count = static_cast<uint64_t>(nreg_);
    out->n_trace = std::min<unsigned long long>(nt, tr_index_.n);
    out->kernel_launches = launches_;
    out->step_kernel_ms = step_ms_;
    out->step_kernel_launches = step_launches_;
}

template <class R> void MixEngineT<R>::read_state(double *x, double *lp) {
    synchronize();
    std::vector<R> hx(static_cast<size_t>(D_) * C_), hl(C_);
    x_.down(hx.data(), hx.size());
    lp_.down(hl.data(), C_);
    for (int c = 0; c < C_; ++c) {
        for (int d = 0; d < D_; ++d)
            x[static_cast<size_t>(c) * D_ + d] = static_cast<double>(hx[static_cast<size_t>(d) * C_ + c]);
        if (lp)
            lp[c] = static_cast<double>(hl[c]);
    }
}

template <class R> void MixEngineT<R>::read_chain_tallies(double *asum, uint64_t *nacc) {
    synchronize();
    if (asum)
        asum_.down(asum, C_);
    if (nacc) {
        std::vector<unsigned> na(C_);
        nacc_.down(na.data(), C_);
        for (int c = 0; c < C_; ++c)
            nacc[c] = na[c];
    }
}

template <class R>
uint64_t MixEngineT<R>::read_regions(double *lambda, uint64_t *n, double *acc, uint64_t *vis, uint64_t cap) {
    synchronize();
    uint64_t m = std::min<uint64_t>(cap, static_cast<uint64_t>(nreg_));
    std::vector<double> l(nreg_), ta(nreg_);
    std::vector<unsigned long long> nn(nreg_), tf(nreg_), tv(nreg_);
    lambda_.down(l.data(), nreg_);
    n_.down(nn.data(), nreg_);
    tot_acc_.down(ta.data(), nreg_);
    tot_fx_.down(tf.data(), nreg_);
    tot_vis_.down(tv.data(), nreg_);
    for (uint64_t i = 0; i < m; ++i) {
        if (lambda)
            lambda[i] = l[i];
        if (n)
            n[i] = nn[i];
        if (acc)
            acc[i] = adapt_ == 0 ? ta[i] : static_cast<double>(tf[i]) / 16777216.0;
        if (vis)
            vis[i] = tv[i];
    }
    return static_cast<uint64_t>(nreg_);
}

template <class R> uint64_t MixEngineT<R>::read_trace(ramlt_trace_row *rows, uint64_t cap) {
    synchronize();
    unsigned long long nt = 0;
    tr_count_.down(&nt, 1);
    uint64_t m = std::min<uint64_t>(std::min<unsigned long long>(nt, tr_index_.n), cap);
    std::vector<unsigned long long> idx(m), nn(m);
    std::vector<long long> rg(m);
    std::vector<double> l(m), a(m);
    if (m) {
        tr_index_.down(idx.data(), m);
        tr_n_.down(nn.data(), m);
        tr_region_.down(rg.data(), m);
        tr_lambda_.down(l.data(), m);
        tr_alpha_.down(a.data(), m);
    }
    // canonical order: by mutation index (the pooled/literal rules push in that order
    // within a step; one step's regions may interleave)
    std::vector<size_t> ord(m);
    for (size_t i = 0; i < m; ++i)
        ord[i] = i;
    std::stable_sort(ord.begin(), ord.end(), [&](size_t p, size_t q) {
        return idx[p] != idx[q] ? idx[p] < idx[q] : rg[p] < rg[q];
    });
    for (uint64_t i = 0; i < m; ++i) {
        size_t s = ord[i];
        rows[i].mutation_index = idx[s];
        rows[i].region = rg[s];
        rows[i].n = nn[s];
        rows[i].lambda = l[s];
        rows[i].alpha_hat = a[s];
    }
    return std::min<unsigned long long>(nt, tr_index_.n);
}

template <class R> void MixEngineT<R>::read_decisions(uint32_t K, double *a, uint8_t *flags) {
    synchronize();
    uint32_t kk = std::min<uint32_t>(K, d_.log_steps);
    std::vector<double> la(static_cast<size_t>(d_.log_steps) * C_);
    std::vector<unsigned char> lf(la.size());
    if (!la.empty()) {
        log_a_.down(la.data(), la.size());
        log_f_.down(lf.data(), lf.size());
    }
    uint64_t logged = std::min<uint64_t>(steps_, kk);
    for (int c = 0; c < C_; ++c)
        for (uint32_t j = 0; j < K; ++j) {
            bool have = j < logged;
            a[static_cast<size_t>(c) * K + j] = have ? la[static_cast<size_t>(j) * C_ + c] : 0.0;
            flags[static_cast<size_t>(c) * K + j] = have ? lf[static_cast<size_t>(j) * C_ + c] : 0;
        }
}

template <class R> void MixEngineT<R>::read_series(double *out) {
    synchronize();
    const uint64_t T = std::min<uint64_t>(steps_, d_.series_steps);
    std::vector<double> h(static_cast<size_t>(d_.series_steps) * C_);
    if (!h.empty())
        series_.down(h.data(), h.size());
    for (int c = 0; c < C_; ++c)
        for (uint64_t j = 0; j < d_.series_steps; ++j)
            out[static_cast<size_t>(c) * d_.series_steps + j] = j < T ? h[j * C_ + c] : 0.0;
}

template <class R>
void MixEngineT<R>::autocorrelation(int first, int count, double *tau, double *n_eff, double *sigma2,
                                    int32_t *status) {
    if (first < 0 || count < 0 || first + count > C_)
        throw std::logic_error("mix: autocorrelation chain range outside the handle");
    const uint64_t n = std::min<uint64_t>(steps_, d_.series_steps);
    if (count == 0)
        return;
    size_t smem = (static_cast<size_t>(n) + 256) * sizeof(double);
    if (smem > 227 * 1024)
        throw std::invalid_argument("mix: series too long for the on-chip autocorrelation (<= 28,800 steps)");
    MBuf<double> t, e, s2;
    MBuf<int> st;
    t.alloc(count);
    e.alloc(count);
    s2.alloc(count);
    st.alloc(count);
    RAMLT_MCUDA(cudaFuncSetAttribute(rdm::k_autocorr, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    rdm::k_autocorr<<<count, 256, smem, stream_>>>(series_.p, C_, static_cast<int>(n), first, t.p, e.p, s2.p, st.p);
    RAMLT_MCUDA(cudaGetLastError());
    ++launches_;
    synchronize();
    t.down(tau, count);
    e.down(n_eff, count);
    s2.down(sigma2, count);
    st.down(status, count);
}

}  // namespace ramlt_b200
