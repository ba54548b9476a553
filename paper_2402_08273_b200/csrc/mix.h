// mix.h -- host interface of the analytic-target adaptive MCMC harness
// (include/ramlt_mix.h; BASELINE.json configs[1]).
#pragma once

#include "../../include/ramlt_mix.h"
#include "engine.h"

#include <string>
#include <vector>

namespace ramlt_b200 {

// The target after host preparation (fp64): per component k the whitening
// matrix W_k = L_k^{-1} (Sigma_k = L_k L_k^T, lower triangular, full D x D
// row-major with zeros above the diagonal), the mean, and the log normaliser
// ell_k = log w_k - sum_i log L_k,ii - D/2 log(2 pi), so that
//   log pi(x) = logsumexp_k (ell_k - |W_k (x - mu_k)|^2 / 2).
struct MixHostTarget {
    int D = 0, K = 0;
    std::vector<double> W, mu, ell;
};

// Validates and prepares (throws std::invalid_argument with the reason).
MixHostTarget prepare_mix_target(const ramlt_mix_target &t);

class MixEngineBase {
public:
    virtual ~MixEngineBase() = default;
    virtual void init_chains() = 0;
    virtual void run(uint64_t steps) = 0;
    virtual void synchronize() = 0;
    virtual void set_stream(void *stream) = 0;
    virtual void read_stats(ramlt_mix_stats *out) = 0;
    virtual void read_state(double *x, double *lp) = 0;
    virtual void read_chain_tallies(double *asum, uint64_t *nacc) = 0;
    virtual uint64_t read_regions(double *lambda, uint64_t *n, double *acc, uint64_t *vis, uint64_t cap) = 0;
    virtual uint64_t read_trace(ramlt_trace_row *rows, uint64_t cap) = 0;
    virtual void read_decisions(uint32_t K, double *a, uint8_t *flags) = 0;
    virtual void read_series(double *out) = 0;
    virtual void autocorrelation(int first, int count, double *tau, double *n_eff, double *sigma2,
                                 int32_t *status) = 0;
    virtual void adapt_exchange(uint64_t **cnt, uint64_t **fx, uint64_t **last, uint64_t *n) = 0;
    virtual void adapt_apply() = 0;
    virtual void set_external(bool on) = 0;
    std::string last_error;
};

MixEngineBase *make_mix_engine_f32(const MixHostTarget &t, const ramlt_mix_desc &d);
MixEngineBase *make_mix_engine_f64(const MixHostTarget &t, const ramlt_mix_desc &d);

}  // namespace ramlt_b200
