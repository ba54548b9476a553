/*
 * oracle_abi.h -- C layouts shared by the two CPU checkers under oracle/.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product package may include,
 * link or call anything under oracle/; only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs do.
 *
 *   libramlt_ref*.so   -- the UNMODIFIED reference (/root/reference/proj/src/core)
 *                         compiled by oracle/Makefile, driven by ref_harness.cpp.
 *   libramlt_oracle.so -- ramlt_oracle.cpp, an independent restatement of the
 *                         reference hot path with the lockstep semantics of the
 *                         GPU engine and a selectable RNG (PCG32 / Philox4x32-10).
 *
 * The config struct mirrors ramlt::RenderConfig (core/driver.hpp:19-39) and
 * ramlt::AdaptationConfig (core/adaptation.hpp:14-22) field for field.
 */
#ifndef RAMLT_ORACLE_ABI_H
#define RAMLT_ORACLE_ABI_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct oracle_config {
    int32_t strategy;      /* 0 fixed, 1 global, 2 ra-grid, 3 ra-quadtree (core/driver.hpp:15) */
    int32_t perturbation;  /* 0 lens, 1 multi-chain (core/driver.hpp:17) */
    uint64_t mutations;
    int32_t chains;
    int32_t batch_size;    /* L */
    double gamma_max;
    double gamma_scale;
    double target_acceptance;
    double lambda_init;
    double lambda_min;
    double sigma2_ratio;
    int32_t n_top;
    int32_t n_bottom;
    uint64_t m_split;
    uint64_t m_refine;
    uint64_t b_samples;
    uint64_t seed;
    int32_t width;
    int32_t height;
    int32_t max_vertices;
    int32_t trace_enabled;
    uint64_t metrics_interval;
    /* restatement-only knobs (ignored by the reference harness) */
    int32_t rng;           /* 0 pcg32 (reference), 1 philox4x32-10 */
    int32_t adapt_mode;    /* 0 literal (canonical lockstep order), 1 pooled */
    double b_override;     /* > 0: skip estimate_b and use this b */
    int64_t chain_offset;  /* sharding: this run simulates global chains */
    int64_t chains_total;  /* [chain_offset, chain_offset + chains) of chains_total (0 = chains) */
} oracle_config;

typedef struct oracle_stats {
    double b;
    double b_stderr;
    uint64_t b_samples;
    uint64_t total_mutations;
    uint64_t perturbation_proposals;
    uint64_t large_step_proposals;
    double mean_acceptance;
    double film_luminance;
    double identity_residual;
    uint64_t region_count;
    double loop_time_s;
    uint64_t rays_closest;      /* closest-hit casts inside the mutation loop */
    uint64_t rays_visibility;   /* visibility casts inside the mutation loop */
    uint64_t n_tallies;         /* regions with tallies (controller order) */
    uint64_t n_trace;           /* adaptation trace rows */
    uint64_t n_metrics;
} oracle_stats;

/* Per-chain decision log, first K steps: a (acceptance probability) and
 * flags: bit0 accepted, bit1 perturbation proposal, bit2 step was logged. */
typedef struct oracle_log {
    uint32_t steps;     /* K */
    double *a;          /* chains * K */
    uint8_t *flags;     /* chains * K */
} oracle_log;

/* Adaptation trace row (core/driver.hpp:59-62 + core/adaptation.hpp:51-56). */
typedef struct oracle_trace_row {
    uint64_t mutation_index;
    int64_t region;
    uint64_t n;
    double lambda;
    double alpha_hat;
} oracle_trace_row;

typedef struct oracle_outputs {
    float *image;               /* W*H*3, row 0 at the top (core/film.hpp:8-21) */
    double *tally_accept;       /* cap_tallies */
    uint64_t *tally_visits;     /* cap_tallies */
    uint64_t cap_tallies;
    oracle_trace_row *trace;    /* cap_trace */
    uint64_t cap_trace;
    char *dump;                 /* partition dump text, cap_dump bytes */
    uint64_t cap_dump;
    double *metrics;            /* cap_metrics * 4: time_s, mutations, rrmse, mean_acc */
    uint64_t cap_metrics;
    double *film;               /* optional raw fp64 film W*H*3 (restatement only) */
} oracle_outputs;


/* Analytic-target adaptive MCMC (BASELINE.json configs[1]; include/ramlt_mix.h).
 * The chain loop of core/driver.cpp:113-171 with a Gaussian random-walk
 * proposal on [0,1]^D and a Gaussian-mixture target; the controller, accept
 * rule, quantile and RNG are the reference's (oracle_mix_run restates them,
 * ref_mix_run calls them). */
typedef struct oracle_mix_config {
    int32_t strategy;      /* 0 fixed, 1 global, 2 ra-grid over (x0, x1) */
    int32_t grid_n;
    int32_t chains;
    int32_t batch_size;
    double gamma_max;
    double gamma_scale;
    double target_acceptance;
    double lambda_init;
    double lambda_min;
    uint64_t seed;
    uint64_t steps;        /* lockstep steps per chain */
    int32_t rng;           /* restatement only: 0 pcg32, 1 philox */
    int32_t adapt_mode;    /* restatement only: 0 literal, 1 pooled */
    int64_t chain_offset;
    int64_t chains_total;
    uint32_t log_steps;
    int32_t dim;
    int32_t n_comp;
    int32_t pad_;
    const double *weights;      /* n_comp */
    const double *means;        /* n_comp * dim */
    const double *covariances;  /* n_comp * dim * dim */
} oracle_mix_config;

typedef struct oracle_mix_out {
    double *x;                  /* chains * dim final states, or NULL */
    double *log_pi;             /* chains, or NULL */
    double *log_a;              /* chains * log_steps, or NULL */
    uint8_t *log_f;             /* chains * log_steps, or NULL */
    double *lambda;             /* cap_regions */
    uint64_t *n;
    double *tally_accept;
    uint64_t *tally_visits;
    uint64_t cap_regions;
    oracle_trace_row *trace;    /* cap_trace */
    uint64_t cap_trace;
    uint64_t n_trace;           /* out */
    uint64_t n_regions;         /* out */
    uint64_t accepted;          /* out */
    double acceptance_sum;      /* out */
} oracle_mix_out;

#ifdef __cplusplus
}
#endif
#endif
