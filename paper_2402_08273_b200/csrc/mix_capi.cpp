// mix_capi.cpp -- C-ABI of the analytic-target adaptive MCMC harness
// (include/ramlt_mix.h) and the host preparation of the target (Cholesky,
// whitening, log normalisers) in fp64 without FMA contraction.
#include "mix.h"

#include <cmath>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>

struct ramlt_mix {
    std::unique_ptr<ramlt_b200::MixEngineBase> eng;
    std::string err;
};

namespace ramlt_b200 {

MixHostTarget prepare_mix_target(const ramlt_mix_target &t) {
    if (t.dim < 1 || t.dim > RAMLT_MIX_MAX_DIM)
        throw std::invalid_argument("mix: dim must be in [1, " + std::to_string(RAMLT_MIX_MAX_DIM) + "]");
    if (t.n_comp < 1 || t.n_comp > RAMLT_MIX_MAX_COMP)
        throw std::invalid_argument("mix: n_comp must be in [1, " + std::to_string(RAMLT_MIX_MAX_COMP) + "]");
    if (!t.weights || !t.means || !t.covariances)
        throw std::logic_error("mix: null target array");
    const int D = t.dim, K = t.n_comp;
    MixHostTarget h;
    h.D = D;
    h.K = K;
    h.W.assign(static_cast<size_t>(K) * D * D, 0.0);
    h.mu.assign(t.means, t.means + static_cast<size_t>(K) * D);
    h.ell.assign(K, 0.0);
    const double half_log_2pi = 0.5 * std::log(2.0 * 3.14159265358979323846);
    for (int k = 0; k < K; ++k) {
        if (!(t.weights[k] > 0.0) || !std::isfinite(t.weights[k]))
            throw std::invalid_argument("mix: component weights must be positive and finite");
        const double *S = t.covariances + static_cast<size_t>(k) * D * D;
        for (int i = 0; i < D; ++i)
            for (int j = 0; j < i; ++j)
                if (S[i * D + j] != S[j * D + i])
                    throw std::invalid_argument("mix: covariance " + std::to_string(k) + " is not symmetric");
        // Cholesky-Banachiewicz: Sigma = L L^T, row by row
        std::vector<double> L(static_cast<size_t>(D) * D, 0.0);
        for (int i = 0; i < D; ++i)
            for (int j = 0; j <= i; ++j) {
                double s = S[i * D + j];
                for (int q = 0; q < j; ++q)
                    s = s - L[i * D + q] * L[j * D + q];
                if (i == j) {
                    if (!(s > 0.0))
                        throw std::invalid_argument("mix: covariance " + std::to_string(k) +
                                                    " is not positive definite");
                    L[i * D + i] = std::sqrt(s);
                } else {
                    L[i * D + j] = s / L[j * D + j];
                }
            }
        // W = L^{-1} by forward substitution, column by column
        double *W = h.W.data() + static_cast<size_t>(k) * D * D;
        for (int j = 0; j < D; ++j) {
            W[j * D + j] = 1.0 / L[j * D + j];
            for (int i = j + 1; i < D; ++i) {
                double s = 0.0;
                for (int q = j; q < i; ++q)
                    s = s + L[i * D + q] * W[q * D + j];
                W[i * D + j] = -s / L[i * D + i];
            }
        }
        double ell = std::log(t.weights[k]);
        for (int i = 0; i < D; ++i)
            ell = ell - std::log(L[i * D + i]);
        h.ell[k] = ell - static_cast<double>(D) * half_log_2pi;
    }
    return h;
}

}  // namespace ramlt_b200

namespace {

thread_local std::string g_mix_create_err;

template <class F> int mguard(std::string &err, F &&f) {
    try {
        f();
        return RAMLT_OK;
    } catch (const ramlt_b200::CudaError &e) {
        err = e.what();
        return RAMLT_E_CUDA;
    } catch (const std::invalid_argument &e) {
        err = e.what();
        return RAMLT_E_INVALID;
    } catch (const std::logic_error &e) {
        err = e.what();
        return RAMLT_E_LOGIC;
    } catch (const std::runtime_error &e) {
        err = e.what();
        return RAMLT_E_RUNTIME;
    } catch (const std::exception &e) {
        err = e.what();
        return RAMLT_E_OTHER;
    }
}

}  // namespace

extern "C" {

void ramlt_mix_default_desc(ramlt_mix_desc *d) {
    std::memset(d, 0, sizeof(*d));
    // AdaptationConfig defaults (core/adaptation.hpp:14-22)
    d->strategy = RAMLT_GLOBAL;
    d->grid_n = 4;
    d->chains = 1;
    d->batch_size = 10;
    d->gamma_max = 1.0;
    d->gamma_scale = 5.0;
    d->target_acceptance = 0.5;
    d->lambda_init = 1.0;
    d->lambda_min = -30.0;
    d->seed = 1;
    d->precision = RAMLT_F32;
    d->rng = RAMLT_RNG_PHILOX;
    d->adapt_mode = RAMLT_ADAPT_AUTO;
    d->device = -1;
    d->cooperative = 1;
    d->series_steps = 0;
    d->series_dim = -1;
}

int ramlt_mix_create(const ramlt_mix_target *target, const ramlt_mix_desc *desc, ramlt_mix **out) {
    return mguard(g_mix_create_err, [&] {
        if (!target || !desc || !out)
            throw std::logic_error("mix: null argument");
        ramlt_b200::MixHostTarget ht = ramlt_b200::prepare_mix_target(*target);
        auto h = std::make_unique<ramlt_mix>();
        if (desc->precision == RAMLT_F64)
            h->eng.reset(ramlt_b200::make_mix_engine_f64(ht, *desc));
        else if (desc->precision == RAMLT_F32)
            h->eng.reset(ramlt_b200::make_mix_engine_f32(ht, *desc));
        else
            throw std::invalid_argument("precision must be RAMLT_F32 or RAMLT_F64");
        *out = h.release();
    });
}

const char *ramlt_mix_last_create_error(void) { return g_mix_create_err.c_str(); }
const char *ramlt_mix_last_error(ramlt_mix *h) { return h ? h->err.c_str() : "null handle"; }
void ramlt_mix_destroy(ramlt_mix *h) { delete h; }

#define RAMLT_MH(body)                                                                             \
    do {                                                                                           \
        if (!h)                                                                                    \
            return RAMLT_E_LOGIC;                                                                  \
        return mguard(h->err, [&] { body; });                                                      \
    } while (0)

int ramlt_mix_set_stream(ramlt_mix *h, void *s) { RAMLT_MH(h->eng->set_stream(s)); }
int ramlt_mix_init_chains(ramlt_mix *h) { RAMLT_MH(h->eng->init_chains()); }
int ramlt_mix_run(ramlt_mix *h, uint64_t steps) { RAMLT_MH(h->eng->run(steps)); }
int ramlt_mix_synchronize(ramlt_mix *h) { RAMLT_MH(h->eng->synchronize()); }
int ramlt_mix_read_stats(ramlt_mix *h, ramlt_mix_stats *o) { RAMLT_MH(h->eng->read_stats(o)); }
int ramlt_mix_read_state(ramlt_mix *h, double *x, double *lp) { RAMLT_MH(h->eng->read_state(x, lp)); }
int ramlt_mix_read_chain_tallies(ramlt_mix *h, double *a, uint64_t *n) {
    RAMLT_MH(h->eng->read_chain_tallies(a, n));
}
int ramlt_mix_read_regions(ramlt_mix *h, double *lambda, uint64_t *n, double *acc, uint64_t *vis, uint64_t cap,
                           uint64_t *count) {
    RAMLT_MH(uint64_t c = h->eng->read_regions(lambda, n, acc, vis, cap); if (count) *count = c);
}
int ramlt_mix_read_trace(ramlt_mix *h, ramlt_trace_row *rows, uint64_t cap, uint64_t *n) {
    RAMLT_MH(uint64_t c = h->eng->read_trace(rows, cap); if (n) *n = c);
}
int ramlt_mix_read_decisions(ramlt_mix *h, uint32_t K, double *a, uint8_t *f) {
    RAMLT_MH(h->eng->read_decisions(K, a, f));
}
int ramlt_mix_read_series(ramlt_mix *h, double *out) { RAMLT_MH(h->eng->read_series(out)); }
int ramlt_mix_autocorrelation(ramlt_mix *h, int32_t first, int32_t count, double *tau, double *n_eff,
                              double *sigma2, int32_t *status) {
    RAMLT_MH(h->eng->autocorrelation(first, count, tau, n_eff, sigma2, status));
}
int ramlt_mix_adapt_exchange(ramlt_mix *h, uint64_t **cnt, uint64_t **fx, uint64_t **last, uint64_t *n) {
    RAMLT_MH(h->eng->adapt_exchange(cnt, fx, last, n));
}
int ramlt_mix_adapt_apply(ramlt_mix *h) { RAMLT_MH(h->eng->adapt_apply()); }
int ramlt_mix_set_external_adaptation(ramlt_mix *h, int on) { RAMLT_MH(h->eng->set_external(on != 0)); }

}  // extern "C"
