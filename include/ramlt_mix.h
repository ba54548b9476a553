/*
 * ramlt_mix.h -- C-ABI of the analytic-target adaptive MCMC harness
 * (BASELINE.json configs[1]; SURVEY.md §8 column C2), exported by
 * libramlt_gpu.so next to ramlt_gpu.h.
 *
 * What it is: the reference's chain loop (run_chain_span, core/driver.cpp:109-173)
 * with the light-transport proposal replaced by an isotropic Gaussian random
 * walk in [0,1]^D and the path contribution replaced by an analytic target
 * (a mixture of K anisotropic Gaussians, zero outside the cube).  Everything
 * else is the reference's: the kernel scale sigma_for = exp(lambda/2)
 * (core/adaptation.cpp:44-50), the Gaussian draws through normal_quantile of
 * next_double (core/sampling.cpp:20-60, core/rng.hpp:32-40), mh_accept
 * (core/mutations.cpp:198-208), the "u only if a > 0" accept draw
 * (core/driver.cpp:168-171), record_acceptance / update_lambda batching
 * (core/adaptation.cpp:10-20, 60-92), the RA-grid cell rule over (x0, x1)
 * (core/partition.cpp:16-20) and the chain / init RNG streams
 * (core/driver.cpp:20-21, 223-225).  The target density and the random-walk
 * proposal have no reference implementation: SURVEY.md §8(c) pins this config
 * at the controller / accept boundary only.
 *
 * Conventions are those of ramlt_gpu.h (RAMLT_OK / RAMLT_E_*; the handle is
 * single-host-thread; the caller owns every descriptor and output buffer).
 */
#ifndef RAMLT_MIX_H
#define RAMLT_MIX_H

#include "ramlt_gpu.h"

#ifdef __cplusplus
extern "C" {
#endif

#define RAMLT_MIX_MAX_DIM 16
#define RAMLT_MIX_MAX_COMP 8

/* pi(x) = sum_k w_k N(x; mu_k, Sigma_k) on [0,1]^D, 0 outside.  Arrays are
 * row-major fp64: weights[K], means[K*D], covariances[K*D*D] (SPD). */
typedef struct ramlt_mix_target {
    int32_t dim;
    int32_t n_comp;
    const double *weights;
    const double *means;
    const double *covariances;
} ramlt_mix_target;

/* Chain-loop configuration: AdaptationConfig (adaptation.hpp:14-22) field for
 * field plus the B200 engine knobs of ramlt_render_desc. */
typedef struct ramlt_mix_desc {
    int32_t strategy;          /* RAMLT_FIXED | RAMLT_GLOBAL | RAMLT_RA_GRID (grid over x0, x1) */
    int32_t grid_n;            /* RA-grid resolution (cells per axis) */
    int32_t chains;
    int32_t batch_size;        /* L */
    double gamma_max;
    double gamma_scale;
    double target_acceptance;
    double lambda_init;
    double lambda_min;
    uint64_t seed;
    int32_t precision;         /* RAMLT_F32 | RAMLT_F64 */
    int32_t rng;               /* RAMLT_RNG_PCG32 | RAMLT_RNG_PHILOX */
    int32_t adapt_mode;        /* RAMLT_ADAPT_* (auto: literal <= 4096 chains, else pooled) */
    int32_t device;            /* CUDA device ordinal, -1 = current */
    int64_t chains_total;      /* sharding: global chain count (0 = chains) */
    int64_t chain_offset;      /* sharding: first global chain id of this handle */
    uint32_t log_steps;        /* K: per-chain decision log depth (0 = off) */
    int32_t trace_enabled;
    uint64_t trace_capacity;   /* update-event rows kept on the device */
    int32_t profile_kernels;   /* CUDA events around every step launch */
    int32_t cooperative;       /* 1 (default): persistent cooperative kernel when resident */
    uint32_t series_steps;     /* record one scalar per chain for the first T steps (0 = off) */
    int32_t series_dim;        /* -1: log pi(x); d >= 0: coordinate x_d */
} ramlt_mix_desc;

typedef struct ramlt_mix_stats {
    uint64_t steps;            /* lockstep steps per chain run so far */
    uint64_t proposals;        /* = steps * chains */
    uint64_t accepted;
    double acceptance_sum;     /* sum of a over all proposals */
    double mean_acceptance;
    uint64_t region_count;
    uint64_t n_trace;
    uint64_t kernel_launches;
    double step_kernel_ms;     /* summed event time of the step launches (profile_kernels) */
    uint64_t step_kernel_launches;
} ramlt_mix_stats;

typedef struct ramlt_mix ramlt_mix;

RAMLT_API void ramlt_mix_default_desc(ramlt_mix_desc *desc);
/* Validates the target (Cholesky of every Sigma_k, w_k > 0) and the config,
 * uploads the whitened target, allocates the chain state. */
RAMLT_API int ramlt_mix_create(const ramlt_mix_target *target, const ramlt_mix_desc *desc, ramlt_mix **out);
RAMLT_API const char *ramlt_mix_last_create_error(void);
RAMLT_API const char *ramlt_mix_last_error(ramlt_mix *h);
RAMLT_API void ramlt_mix_destroy(ramlt_mix *h);
RAMLT_API int ramlt_mix_set_stream(ramlt_mix *h, void *cuda_stream);

/* Start states x_0 ~ U[0,1]^D from stream kStreamInit + 2*id (driver.cpp:223). */
RAMLT_API int ramlt_mix_init_chains(ramlt_mix *h);
/* Advance every chain by `steps` lockstep steps. */
RAMLT_API int ramlt_mix_run(ramlt_mix *h, uint64_t steps);
RAMLT_API int ramlt_mix_synchronize(ramlt_mix *h);

RAMLT_API int ramlt_mix_read_stats(ramlt_mix *h, ramlt_mix_stats *out);
/* Current states (chains x D, fp64) and log pi(x) (chains). */
RAMLT_API int ramlt_mix_read_state(ramlt_mix *h, double *x, double *log_pi);
/* Per-chain (acceptance sum, accepted count). */
RAMLT_API int ramlt_mix_read_chain_tallies(ramlt_mix *h, double *accept_sum, uint64_t *accepted);
/* Region lambda / n / lifetime tallies (KernelController::lambda_of, updates_of, tallies). */
RAMLT_API int ramlt_mix_read_regions(ramlt_mix *h, double *lambda, uint64_t *n, double *accept_sum,
                                     uint64_t *visits, uint64_t cap, uint64_t *count);
RAMLT_API int ramlt_mix_read_trace(ramlt_mix *h, ramlt_trace_row *rows, uint64_t cap, uint64_t *n);
/* First K steps per chain: a[chain*K + step], flags bit0 accepted, bit1 proposal, bit2 logged. */
RAMLT_API int ramlt_mix_read_decisions(ramlt_mix *h, uint32_t K, double *a, uint8_t *flags);

/* The recorded series, chain-major (chains x series_steps; steps not yet run are 0). */
RAMLT_API int ramlt_mix_read_series(ramlt_mix *h, double *out);
/* autocorrelation_time (core/diagnostics.cpp:87-127: Geyer initial positive
 * sequence, tau >= 1e-3, n_eff = n / tau, sigma2 = tau / n * var) of the
 * recorded series of chains [first, first + count), on the device.  status[i]
 * = RAMLT_E_INVALID where the reference throws (fewer than 1000 steps or no
 * variance), else 0. */
RAMLT_API int ramlt_mix_autocorrelation(ramlt_mix *h, int32_t first, int32_t count, double *tau,
                                        double *n_eff, double *sigma2, int32_t *status);

/* Sharded pooled adaptation (as ramlt_gpu_adapt_exchange / _apply): after a
 * run() step the handle holds per-region (count, fixed-point sum, last index)
 * device arrays; SUM/SUM/MAX them across ranks, then apply. */
RAMLT_API int ramlt_mix_adapt_exchange(ramlt_mix *h, uint64_t **cnt, uint64_t **fx, uint64_t **last, uint64_t *n);
RAMLT_API int ramlt_mix_adapt_apply(ramlt_mix *h);
/* 1: run() stops after each step with the exchange arrays filled (sharded use). */
RAMLT_API int ramlt_mix_set_external_adaptation(ramlt_mix *h, int enabled);

#ifdef __cplusplus
}
#endif

#endif /* RAMLT_MIX_H */
