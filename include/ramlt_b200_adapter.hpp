// ramlt_b200_adapter.hpp -- reference-side binding of the B200 engine.
//
// A maintainer of the reference library (namespace ramlt, /proj/src/core)
// includes this header next to driver.hpp and links libramlt_gpu.so to route
// run_render (core/driver.hpp:80) through the sm_100a kernels:
//
//     #include "driver.hpp"
//     #include "ramlt_b200_adapter.hpp"
//     ramlt::RenderResult r = ramlt_b200::run_render<ramlt::RenderResult>(scene_text, cfg);
//
// It converts the reference's own types (RenderConfig, SceneModel, Image,
// RenderResult, MetricsRow, TraceRow, Tally) to and from the C-ABI in
// ramlt_gpu.h and rethrows the reference's exception types.  Header-only; no
// torch, no CUDA headers.
#pragma once

#include "ramlt_gpu.h"

#include <stdexcept>
#include <string>
#include <vector>

namespace ramlt_b200 {

struct Options {
    int precision = RAMLT_F32;      // RAMLT_F64 for the parity build
    int rng = RAMLT_RNG_PHILOX;     // RAMLT_RNG_PCG32 reproduces the reference's streams
    int device = -1;
    unsigned log_steps = 0;
    // Several GPUs of this process (e.g. {0,...,7}): one handle over all of them
    // (ramlt_gpu_create_multi), chains sharded by global id -- the drop-in for the
    // reference's thread-per-chain loop (core/driver.cpp:282-297) on 1..8 B200s.
    std::vector<int> devices;
    unsigned film_sync_steps = 4096;   // configs[4]: film merged every 2^12 lockstep steps
};

inline void rethrow(int rc, const char *msg) {
    switch (rc) {
    case RAMLT_OK: return;
    case RAMLT_E_RUNTIME: throw std::runtime_error(msg);
    case RAMLT_E_LOGIC: throw std::logic_error(msg);
    case RAMLT_E_INVALID: throw std::invalid_argument(msg);
    default: throw std::runtime_error(std::string("ramlt_gpu: ") + msg);
    }
}

// ramlt::RenderConfig (core/driver.hpp:19-39) -> ramlt_render_desc
template <class RenderConfig>
inline ramlt_render_desc to_desc(const RenderConfig &cfg, const Options &opt) {
    ramlt_render_desc d;
    ramlt_gpu_default_desc(&d);
    d.strategy = static_cast<int32_t>(cfg.strategy);          // Fixed, Global, RaGrid, RaQuadtree
    d.perturbation = static_cast<int32_t>(cfg.perturbation);  // Lens, MultiChain
    d.mutations = cfg.mutations;
    d.time_budget_s = cfg.time_budget_s;
    d.chains = cfg.chains;
    d.batch_size = cfg.adaptation.batch_size;
    d.gamma_max = cfg.adaptation.gamma_max;
    d.gamma_scale = cfg.adaptation.gamma_scale;
    d.target_acceptance = cfg.adaptation.target_acceptance;
    d.lambda_init = cfg.adaptation.lambda_init;
    d.lambda_min = cfg.adaptation.lambda_min;
    d.sigma2_ratio = cfg.adaptation.sigma2_ratio;
    d.n_top = cfg.n_top;
    d.n_bottom = cfg.n_bottom;
    d.m_split = cfg.m_split;
    d.m_refine = cfg.m_refine;
    d.b_samples = cfg.b_samples;
    d.seed = cfg.seed;
    d.width = cfg.width;
    d.height = cfg.height;
    d.max_vertices = cfg.max_vertices;
    d.trace_enabled = cfg.trace_enabled ? 1 : 0;
    d.metrics_interval = cfg.metrics_interval;
    d.dump_partition = cfg.dump_partition ? 1 : 0;
    d.precision = opt.precision;
    d.rng = opt.rng;
    d.device = opt.device;
    d.log_steps = opt.log_steps;
    return d;
}

// Fills a ramlt::RenderResult (core/driver.hpp:64-78) from a finished handle.
template <class RenderResult>
inline void fill_result(ramlt_gpu *h, int width, int height, RenderResult &r) {
    ramlt_stats s;
    rethrow(ramlt_gpu_read_stats(h, &s), ramlt_gpu_last_error(h));
    r.image.width = width;
    r.image.height = height;
    r.image.data.assign(static_cast<size_t>(width) * height * 3, 0.0f);
    rethrow(ramlt_gpu_read_image(h, r.image.data.data()), ramlt_gpu_last_error(h));
    r.b.b = s.b;
    r.b.stderr_ = s.b_stderr;
    r.b.samples = s.b_samples;
    r.total_mutations = s.total_mutations;
    r.perturbation_proposals = s.perturbation_proposals;
    r.large_step_proposals = s.large_step_proposals;
    r.mean_acceptance = s.mean_acceptance;
    r.film_luminance = s.film_luminance;
    r.identity_residual = s.identity_residual;
    r.region_count = s.region_count;
    std::vector<double> m(4 * s.n_metrics);
    uint64_t nm = 0;
    rethrow(ramlt_gpu_read_metrics(h, m.data(), s.n_metrics, &nm), ramlt_gpu_last_error(h));
    r.metrics.resize(nm);
    for (uint64_t i = 0; i < nm; ++i) {
        r.metrics[i].time_s = m[4 * i];
        r.metrics[i].mutations = static_cast<uint64_t>(m[4 * i + 1]);
        r.metrics[i].rrmse = m[4 * i + 2];
        r.metrics[i].mean_acceptance = m[4 * i + 3];
    }
    std::vector<ramlt_trace_row> tr(s.n_trace);
    uint64_t nt = 0;
    rethrow(ramlt_gpu_read_trace(h, tr.data(), tr.size(), &nt), ramlt_gpu_last_error(h));
    r.trace.resize(tr.size());
    for (size_t i = 0; i < tr.size(); ++i) {
        r.trace[i].mutation_index = tr[i].mutation_index;
        r.trace[i].event.region = static_cast<int>(tr[i].region);
        r.trace[i].event.n = tr[i].n;
        r.trace[i].event.lambda = tr[i].lambda;
        r.trace[i].event.alpha_hat = tr[i].alpha_hat;
    }
    uint64_t n = 0;
    rethrow(ramlt_gpu_read_tallies(h, nullptr, nullptr, 0, &n), ramlt_gpu_last_error(h));
    std::vector<double> acc(n);
    std::vector<uint64_t> vis(n);
    rethrow(ramlt_gpu_read_tallies(h, acc.data(), vis.data(), n, &n), ramlt_gpu_last_error(h));
    r.tallies.resize(n);
    for (uint64_t i = 0; i < n; ++i) {
        r.tallies[i].accept_sum = acc[i];
        r.tallies[i].visits = vis[i];
    }
}

// run_render over the reference's scene text (the input of parse_scene /
// load_scene, core/scene.hpp:77-78):
//     auto r = ramlt_b200::run_render<ramlt::RenderResult>(text, cfg);
template <class RenderResult, class RenderConfig>
inline RenderResult run_render(const std::string &scene_text, const RenderConfig &cfg,
                               const Options &opt = {}) {
    ramlt_render_desc d = to_desc(cfg, opt);
    ramlt_gpu *h = nullptr;
    if (opt.devices.size() > 1) {
        std::vector<int32_t> devs(opt.devices.begin(), opt.devices.end());
        rethrow(ramlt_gpu_create_multi_from_text(scene_text.c_str(), "<scene>", &d, static_cast<int32_t>(devs.size()),
                                                 devs.data(), opt.film_sync_steps, &h),
                ramlt_gpu_last_create_error());
    } else {
        if (opt.devices.size() == 1)
            d.device = opt.devices[0];
        rethrow(ramlt_gpu_create_from_text(scene_text.c_str(), "<scene>", &d, &h), ramlt_gpu_last_create_error());
    }
    RenderResult r;
    try {
        // RenderConfig::reference (core/driver.hpp:38): metrics rows carry the rRMSE
        // of the running image against it (core/driver.cpp:265-272)
        if (cfg.reference)
            rethrow(ramlt_gpu_set_reference(h, cfg.reference->data.data(), cfg.reference->width,
                                            cfg.reference->height),
                    ramlt_gpu_last_error(h));
        rethrow(ramlt_gpu_render(h), ramlt_gpu_last_error(h));
        fill_result(h, cfg.width, cfg.height, r);
        if (cfg.dump_partition) {
            std::vector<char> buf(1 << 24);
            rethrow(ramlt_gpu_read_partition(h, buf.data(), buf.size()), ramlt_gpu_last_error(h));
            r.partition_dump = buf.data();
        }
    } catch (...) {
        ramlt_gpu_destroy(h);
        throw;
    }
    ramlt_gpu_destroy(h);
    return r;
}

}  // namespace ramlt_b200
