// ref_harness.cpp -- drives the UNMODIFIED reference library as a checker.
//
// TEST INFRASTRUCTURE ONLY (see oracle_abi.h).  This file is compiled by
// oracle/Makefile together with the reference sources *where they lie* under
// /root/reference/proj/src/core (nothing is copied into this repo) into
// oracle/_ref/libramlt_ref.so (timing build) and libramlt_ref_log.so (decision
// logging build).
//
// The logging build observes the reference's own hot loop, run_chain_span
// (core/driver.cpp:109-173), without modifying it: the linker redirects the
// cross-object calls driver.o makes (suitability, mh_accept, lens_perturb,
// multichain_perturb, large_step, KernelController::tallies) and the ray casts
// path.o / mutations.o make (SceneModel::intersect / visible) to __wrap_*
// shims below (-Wl,--wrap=<mangled name>).
//
//  * A step starts when suitability() is called on the chain's own path
//    (core/driver.cpp:115).  The first suitability() call a worker thread makes
//    is always that one, so its argument address identifies the chain.
//  * a = the value the step's mh_accept() returned (core/driver.cpp:138, 161),
//    0 when mh_accept was not reached.
//  * accepted <=> chain.path's vertex buffer changed between two step starts
//    (core/driver.cpp:169 moves the proposal's buffer into chain.path).
//  * Chains are std::vector<ChainState> elements (core/driver.cpp:220), so the
//    address order of &chain.path is the chain index order.
#include "driver.hpp"
#include "sampling.hpp"
#include "scene.hpp"
#include "camera.hpp"
#include "adaptation.hpp"
#include "partition.hpp"
#include "diagnostics.hpp"
#include "film.hpp"
#include "image_io.hpp"

#include "oracle_abi.h"

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <limits>
#include <map>
#include <memory>
#include <mutex>
#include <span>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

namespace {

void copy_err(char *err, int errlen, const char *msg) {
    if (!err || errlen <= 0)
        return;
    std::strncpy(err, msg, static_cast<size_t>(errlen) - 1);
    err[errlen - 1] = '\0';
}

ramlt::RenderConfig to_config(const oracle_config *c) {
    ramlt::RenderConfig cfg;
    static const ramlt::StrategyVariant kStrat[] = {
        ramlt::StrategyVariant::Fixed, ramlt::StrategyVariant::Global,
        ramlt::StrategyVariant::RaGrid, ramlt::StrategyVariant::RaQuadtree};
    if (c->strategy < 0 || c->strategy > 3)
        throw std::invalid_argument("harness: bad strategy");
    cfg.strategy = kStrat[c->strategy];
    cfg.perturbation = c->perturbation == 0 ? ramlt::PerturbationKind::Lens
                                            : ramlt::PerturbationKind::MultiChain;
    cfg.mutations = c->mutations;
    cfg.chains = c->chains;
    cfg.adaptation.batch_size = c->batch_size;
    cfg.adaptation.gamma_max = c->gamma_max;
    cfg.adaptation.gamma_scale = c->gamma_scale;
    cfg.adaptation.target_acceptance = c->target_acceptance;
    cfg.adaptation.lambda_init = c->lambda_init;
    cfg.adaptation.lambda_min = c->lambda_min;
    cfg.adaptation.sigma2_ratio = c->sigma2_ratio;
    cfg.n_top = c->n_top;
    cfg.n_bottom = c->n_bottom;
    cfg.m_split = c->m_split;
    cfg.m_refine = c->m_refine;
    cfg.b_samples = c->b_samples;
    cfg.seed = c->seed;
    cfg.width = c->width;
    cfg.height = c->height;
    cfg.max_vertices = c->max_vertices;
    cfg.metrics_interval = c->metrics_interval;
    cfg.trace_enabled = c->trace_enabled != 0;
    return cfg;
}

#ifdef RAMLT_REF_LOG
struct ChainLog {
    std::vector<double> a;
    std::vector<uint8_t> flags;
};

std::mutex g_mu;
std::map<const void *, ChainLog *> g_logs;
std::atomic<bool> g_enabled{false};
std::atomic<uint64_t> g_rays_closest{0}, g_rays_vis{0};
uint32_t g_max_steps = 0;

struct ThreadState {
    const ramlt::Path *chain_path = nullptr;
    ChainLog *log = nullptr;
    const void *prev_data = nullptr;
    bool in_step = false;
    double a = 0.0;
    uint8_t kind = 0;
    uint64_t rays_c = 0, rays_v = 0;

    void finalize() {
        if (in_step && log) {
            bool accepted = static_cast<const void *>(chain_path->vertices.data()) != prev_data;
            if (log->a.size() < g_max_steps) {
                log->a.push_back(a);
                log->flags.push_back(static_cast<uint8_t>((accepted ? 1 : 0) | (kind ? 2 : 0) | 4));
            }
        }
        in_step = false;
        g_rays_closest.fetch_add(rays_c);
        g_rays_vis.fetch_add(rays_v);
        rays_c = rays_v = 0;
    }
    void reset() {
        chain_path = nullptr;
        log = nullptr;
        in_step = false;
        rays_c = rays_v = 0;
    }
    ~ThreadState() {
        if (g_enabled.load())
            finalize();
    }
};
thread_local ThreadState tls;
#endif

} // namespace

#ifdef RAMLT_REF_LOG
extern "C" {
double __real__ZN5ramlt9mh_acceptEdddddd(double, double, double, double, double, double);
double __wrap__ZN5ramlt9mh_acceptEdddddd(double pc, double pp, double tf, double tr, double sf,
                                         double sr) {
    double a = __real__ZN5ramlt9mh_acceptEdddddd(pc, pp, tf, tr, sf, sr);
    tls.a = a;
    return a;
}

double __real__ZN5ramlt11suitabilityERKNS_4PathENS_8StrategyE(const ramlt::Path &, ramlt::Strategy);
double __wrap__ZN5ramlt11suitabilityERKNS_4PathENS_8StrategyE(const ramlt::Path &p,
                                                               ramlt::Strategy s) {
    if (g_enabled.load(std::memory_order_relaxed)) {
        if (!tls.chain_path) {
            tls.chain_path = &p;
            std::lock_guard<std::mutex> lock(g_mu);
            auto it = g_logs.find(&p);
            if (it == g_logs.end())
                it = g_logs.emplace(&p, new ChainLog()).first;
            tls.log = it->second;
        }
        if (&p == tls.chain_path) {
            if (tls.in_step) {
                bool accepted = static_cast<const void *>(p.vertices.data()) != tls.prev_data;
                if (tls.log->a.size() < g_max_steps) {
                    tls.log->a.push_back(tls.a);
                    tls.log->flags.push_back(
                        static_cast<uint8_t>((accepted ? 1 : 0) | (tls.kind ? 2 : 0) | 4));
                }
            }
            tls.prev_data = p.vertices.data();
            tls.a = 0.0;
            tls.kind = 0;
            tls.in_step = true;
        }
    }
    return __real__ZN5ramlt11suitabilityERKNS_4PathENS_8StrategyE(p, s);
}

std::optional<ramlt::Proposal> __real__ZN5ramlt12lens_perturbERKNS_10SceneModelERKNS_4PathERKNS_9SigmaPairERNS_14RandomSequenceE(
    const ramlt::SceneModel &, const ramlt::Path &, const ramlt::SigmaPair &, ramlt::RandomSequence &);
std::optional<ramlt::Proposal> __wrap__ZN5ramlt12lens_perturbERKNS_10SceneModelERKNS_4PathERKNS_9SigmaPairERNS_14RandomSequenceE(
    const ramlt::SceneModel &sc, const ramlt::Path &p, const ramlt::SigmaPair &s, ramlt::RandomSequence &r) {
    tls.kind = 1;
    return __real__ZN5ramlt12lens_perturbERKNS_10SceneModelERKNS_4PathERKNS_9SigmaPairERNS_14RandomSequenceE(sc, p, s, r);
}

std::optional<ramlt::Proposal> __real__ZN5ramlt18multichain_perturbERKNS_10SceneModelERKNS_4PathERKNS_9SigmaPairERNS_14RandomSequenceE(
    const ramlt::SceneModel &, const ramlt::Path &, const ramlt::SigmaPair &, ramlt::RandomSequence &);
std::optional<ramlt::Proposal> __wrap__ZN5ramlt18multichain_perturbERKNS_10SceneModelERKNS_4PathERKNS_9SigmaPairERNS_14RandomSequenceE(
    const ramlt::SceneModel &sc, const ramlt::Path &p, const ramlt::SigmaPair &s, ramlt::RandomSequence &r) {
    tls.kind = 1;
    return __real__ZN5ramlt18multichain_perturbERKNS_10SceneModelERKNS_4PathERKNS_9SigmaPairERNS_14RandomSequenceE(sc, p, s, r);
}

std::optional<ramlt::Intersection> __real__ZNK5ramlt10SceneModel9intersectERKNS_4Vec3ES3_(
    const ramlt::SceneModel *, const ramlt::Vec3 &, const ramlt::Vec3 &);
std::optional<ramlt::Intersection> __wrap__ZNK5ramlt10SceneModel9intersectERKNS_4Vec3ES3_(
    const ramlt::SceneModel *self, const ramlt::Vec3 &o, const ramlt::Vec3 &d) {
    if (tls.in_step)
        ++tls.rays_c;
    return __real__ZNK5ramlt10SceneModel9intersectERKNS_4Vec3ES3_(self, o, d);
}

bool __real__ZNK5ramlt10SceneModel7visibleERKNS_4Vec3ES3_(const ramlt::SceneModel *,
                                                          const ramlt::Vec3 &, const ramlt::Vec3 &);
bool __wrap__ZNK5ramlt10SceneModel7visibleERKNS_4Vec3ES3_(const ramlt::SceneModel *self,
                                                          const ramlt::Vec3 &a, const ramlt::Vec3 &b) {
    if (tls.in_step)
        ++tls.rays_v;
    return __real__ZNK5ramlt10SceneModel7visibleERKNS_4Vec3ES3_(self, a, b);
}

std::vector<ramlt::KernelController::Tally> __real__ZNK5ramlt16KernelController7talliesEv(
    const ramlt::KernelController *);
std::vector<ramlt::KernelController::Tally> __wrap__ZNK5ramlt16KernelController7talliesEv(
    const ramlt::KernelController *self) {
    // Called once after the span loop (core/driver.cpp:332): the 1-chain run's
    // last step is still open in this (main) thread and chain.path is alive.
    if (g_enabled.load())
        tls.finalize();
    return __real__ZNK5ramlt16KernelController7talliesEv(self);
}
} // extern "C"
#endif

extern "C" {

int ref_has_log(void) {
#ifdef RAMLT_REF_LOG
    return 1;
#else
    return 0;
#endif
}

// RenderConfig::reference for the next ref_render calls (w = 0 clears it).
ramlt::Image g_reference;
void ref_set_reference(const float *rgb, int w, int h) {
    g_reference = ramlt::Image();
    if (w > 0 && h > 0) {
        g_reference = ramlt::Image(w, h);
        std::memcpy(g_reference.data.data(), rgb, sizeof(float) * 3 * static_cast<size_t>(w) * h);
    }
}

// autocorrelation_time (core/diagnostics.cpp:87-127) on one series.
int ref_autocorrelation_time(const double *series, uint64_t n, double *tau, double *n_eff, double *sigma2) {
    try {
        ramlt::ChainDiagnostics d = ramlt::autocorrelation_time(std::span<const double>(series, n));
        *tau = d.tau;
        *n_eff = d.n_eff;
        *sigma2 = d.sigma2;
        return 0;
    } catch (const std::invalid_argument &) {
        return 3;
    }
}

// write_pfm / read_pfm (core/image_io.cpp:15-56).
int ref_write_pfm(const float *rgb, int w, int h, const char *path) {
    try {
        ramlt::Image img(w, h);
        std::memcpy(img.data.data(), rgb, sizeof(float) * 3 * static_cast<size_t>(w) * h);
        ramlt::write_pfm(img, path);
        return 0;
    } catch (...) {
        return 1;
    }
}
int ref_read_pfm(const char *path, float *rgb, int cap_pixels, int *w, int *h, char *err, int errlen) {
    try {
        ramlt::Image img = ramlt::read_pfm(path);
        *w = img.width;
        *h = img.height;
        if (static_cast<long long>(img.width) * img.height <= cap_pixels)
            std::memcpy(rgb, img.data.data(), img.data.size() * sizeof(float));
        return 0;
    } catch (const std::exception &e) {
        copy_err(err, errlen, e.what());
        return 1;
    }
}

// error_report (core/diagnostics.cpp:11-38) on two W x H RGB images.
int ref_error_report(const float *img, const float *ref, int w, int h, double eps, int rgb, double *rrmse) {
    try {
        ramlt::Image a(w, h), b(w, h);
        std::memcpy(a.data.data(), img, sizeof(float) * 3 * static_cast<size_t>(w) * h);
        std::memcpy(b.data.data(), ref, sizeof(float) * 3 * static_cast<size_t>(w) * h);
        *rrmse = ramlt::error_report(a, b, eps, rgb != 0).rrmse;
        return 0;
    } catch (...) {
        return 3;
    }
}

// run_render through the reference's public API (core/driver.hpp:80).
// Returns 0 on success; 1 runtime_error, 2 logic_error, 3 invalid_argument,
// 4 other exception.  err receives e.what().
int ref_render(const char *scene_text, const oracle_config *c, oracle_stats *st, oracle_log *lg,
               oracle_outputs *out, char *err, int errlen) {
    try {
        ramlt::SceneModel scene = ramlt::parse_scene(scene_text, "<scene>");
        ramlt::RenderConfig cfg = to_config(c);
        cfg.dump_partition = out && out->dump && out->cap_dump > 0;
        if (g_reference.width > 0)
            cfg.reference = &g_reference;   // RenderConfig::reference (driver.hpp:38)
#ifdef RAMLT_REF_LOG
        for (auto &kv : g_logs)
            delete kv.second;
        g_logs.clear();
        tls.reset();
        g_rays_closest = 0;
        g_rays_vis = 0;
        g_max_steps = lg ? lg->steps : 0;
        g_enabled = lg != nullptr;
#endif
        ramlt::RenderResult r = ramlt::run_render(scene, cfg);
#ifdef RAMLT_REF_LOG
        g_enabled = false;
#endif
        if (st) {
            std::memset(st, 0, sizeof(*st));
            st->b = r.b.b;
            st->b_stderr = r.b.stderr_;
            st->b_samples = r.b.samples;
            st->total_mutations = r.total_mutations;
            st->perturbation_proposals = r.perturbation_proposals;
            st->large_step_proposals = r.large_step_proposals;
            st->mean_acceptance = r.mean_acceptance;
            st->film_luminance = r.film_luminance;
            st->identity_residual = r.identity_residual;
            st->region_count = r.region_count;
            st->loop_time_s = r.metrics.empty() ? 0.0 : r.metrics.back().time_s;
#ifdef RAMLT_REF_LOG
            st->rays_closest = g_rays_closest.load();
            st->rays_visibility = g_rays_vis.load();
#endif
            st->n_tallies = r.tallies.size();
            st->n_trace = r.trace.size();
            st->n_metrics = r.metrics.size();
        }
        if (out) {
            if (out->image)
                std::memcpy(out->image, r.image.data.data(), r.image.data.size() * sizeof(float));
            for (size_t i = 0; i < r.tallies.size() && i < out->cap_tallies; ++i) {
                if (out->tally_accept)
                    out->tally_accept[i] = r.tallies[i].accept_sum;
                if (out->tally_visits)
                    out->tally_visits[i] = r.tallies[i].visits;
            }
            for (size_t i = 0; i < r.trace.size() && i < out->cap_trace && out->trace; ++i) {
                out->trace[i].mutation_index = r.trace[i].mutation_index;
                out->trace[i].region = r.trace[i].event.region;
                out->trace[i].n = r.trace[i].event.n;
                out->trace[i].lambda = r.trace[i].event.lambda;
                out->trace[i].alpha_hat = r.trace[i].event.alpha_hat;
            }
            if (out->dump && out->cap_dump > 0) {
                std::strncpy(out->dump, r.partition_dump.c_str(), out->cap_dump - 1);
                out->dump[out->cap_dump - 1] = '\0';
            }
            for (size_t i = 0; i < r.metrics.size() && i < out->cap_metrics && out->metrics; ++i) {
                out->metrics[i * 4 + 0] = r.metrics[i].time_s;
                out->metrics[i * 4 + 1] = static_cast<double>(r.metrics[i].mutations);
                out->metrics[i * 4 + 2] = r.metrics[i].rrmse;
                out->metrics[i * 4 + 3] = r.metrics[i].mean_acceptance;
            }
        }
#ifdef RAMLT_REF_LOG
        if (lg) {
            std::vector<const void *> keys;
            for (auto &kv : g_logs)
                keys.push_back(kv.first);
            std::sort(keys.begin(), keys.end());
            size_t chains = static_cast<size_t>(c->chains);
            std::memset(lg->flags, 0, chains * lg->steps);
            for (size_t i = 0; i < chains * lg->steps; ++i)
                lg->a[i] = 0.0;
            for (size_t ci = 0; ci < keys.size() && ci < chains; ++ci) {
                ChainLog *l = g_logs[keys[ci]];
                for (size_t j = 0; j < l->a.size() && j < lg->steps; ++j) {
                    lg->a[ci * lg->steps + j] = l->a[j];
                    lg->flags[ci * lg->steps + j] = l->flags[j];
                }
            }
        }
#endif
        return 0;
    } catch (const std::invalid_argument &e) {
        copy_err(err, errlen, e.what());
        return 3;
    } catch (const std::logic_error &e) {
        copy_err(err, errlen, e.what());
        return 2;
    } catch (const std::runtime_error &e) {
        copy_err(err, errlen, e.what());
        return 1;
    } catch (const std::exception &e) {
        copy_err(err, errlen, e.what());
        return 4;
    }
}

// ---- reference primitives, exported for function-level pinning --------------

double ref_normal_quantile(double p) { return ramlt::normal_quantile(p); }
double ref_normal_cdf(double x) { return ramlt::normal_cdf(x); }

// AngularKernel (core/sampling.cpp:62-92): pdf and pdf_solid_angle.
int ref_angular_pdf(double sigma, double theta, double *pdf, double *pdf_sa) {
    try {
        ramlt::AngularKernel k(sigma);
        *pdf = k.pdf(theta);
        *pdf_sa = k.pdf_solid_angle(theta);
        return 0;
    } catch (...) {
        return 3;
    }
}

// n draws of AngularKernel::sample from RandomSequence(seed, stream).
int ref_angular_sample(double sigma, uint64_t seed, uint64_t stream, uint64_t n, double *out) {
    try {
        ramlt::AngularKernel k(sigma);
        ramlt::RandomSequence rng(seed, stream);
        for (uint64_t i = 0; i < n; ++i)
            out[i] = k.sample(rng);
        return 0;
    } catch (...) {
        return 3;
    }
}

void ref_rng_u32(uint64_t seed, uint64_t stream, uint64_t n, uint32_t *out) {
    ramlt::RandomSequence rng(seed, stream);
    for (uint64_t i = 0; i < n; ++i)
        out[i] = rng.next_u32();
}

void ref_perturb_direction(const double *omega, double sigma, uint64_t seed, uint64_t stream,
                           uint64_t n, double *out) {
    ramlt::AngularKernel k(sigma);
    ramlt::RandomSequence rng(seed, stream);
    ramlt::Vec3 w(omega[0], omega[1], omega[2]);
    for (uint64_t i = 0; i < n; ++i) {
        ramlt::Vec3 r = ramlt::perturb_direction(w, k, rng);
        out[3 * i + 0] = r.x;
        out[3 * i + 1] = r.y;
        out[3 * i + 2] = r.z;
    }
}

void ref_cylindrical(const double *omega, double *uv) {
    auto p = ramlt::cylindrical_coords(ramlt::Vec3(omega[0], omega[1], omega[2]));
    uv[0] = p.u;
    uv[1] = p.v;
}

double ref_step_size(double gamma_max, double gamma_scale, uint64_t n) {
    ramlt::AdaptationConfig cfg;
    cfg.gamma_max = gamma_max;
    cfg.gamma_scale = gamma_scale;
    return ramlt::step_size(cfg, n);
}

double ref_update_lambda(double lambda, double alpha_hat, uint64_t n, double target,
                         double lambda_min) {
    ramlt::AdaptationConfig cfg;
    cfg.target_acceptance = target;
    cfg.lambda_min = lambda_min;
    return ramlt::update_lambda(lambda, alpha_hat, n, cfg);
}

// sigma_for of a Global controller after feeding `n` acceptances.
double ref_controller_feed(const double *a, uint64_t n, int *updates_out) {
    ramlt::AdaptationConfig cfg;
    ramlt::KernelController ctl(ramlt::ControllerKind::Global, cfg);
    int updates = 0;
    for (uint64_t i = 0; i < n; ++i)
        if (ctl.record_acceptance(0, a[i]))
            ++updates;
    if (updates_out)
        *updates_out = updates;
    return ctl.lambda_of(0);
}

int ref_grid_cell(int n, double u, double v) {
    ramlt::Grid2D g(n);
    return g.cell_of({u, v});
}

double ref_mh_accept(double pc, double pp, double tf, double tr, double sf, double sr, int *status) {
    try {
        *status = 0;
        return ramlt::mh_accept(pc, pp, tf, tr, sf, sr);
    } catch (...) {
        *status = 3;
        return 0.0;
    }
}

double ref_fresnel(double cos_i, double ior) { return ramlt::fresnel_dielectric(cos_i, ior); }

// Camera round trip rp(primary(u,v)) (core/camera.cpp:32-49) and pdfs.
int ref_camera(const double *cam /*pos3 look3 up3 fov*/, int w, int h, double u, double v,
               double *dir3, double *uv2, double *importance, double *dir_pdf) {
    try {
        ramlt::Camera c(ramlt::Vec3(cam[0], cam[1], cam[2]), ramlt::Vec3(cam[3], cam[4], cam[5]),
                        ramlt::Vec3(cam[6], cam[7], cam[8]), cam[9]);
        c.configure_image(w, h);
        ramlt::Vec3 d = c.primary_direction(u, v);
        dir3[0] = d.x;
        dir3[1] = d.y;
        dir3[2] = d.z;
        auto rp = c.raster_position(d);
        uv2[0] = rp ? rp->u : -1.0;
        uv2[1] = rp ? rp->v : -1.0;
        *importance = c.importance(d);
        *dir_pdf = c.direction_pdf(d);
        return 0;
    } catch (...) {
        return 3;
    }
}

// parse_scene (core/scene.cpp:114-234): 0 ok, 1 runtime_error (message in err).
int ref_parse(const char *text, int *counts /* materials spheres triangles emitters */, char *err,
              int errlen) {
    try {
        ramlt::SceneModel s = ramlt::parse_scene(text, "<scene>");
        counts[0] = static_cast<int>(s.materials.size());
        counts[1] = static_cast<int>(s.spheres.size());
        counts[2] = static_cast<int>(s.triangles.size());
        counts[3] = static_cast<int>(s.emitters.size());
        return 0;
    } catch (const std::runtime_error &e) {
        copy_err(err, errlen, e.what());
        return 1;
    } catch (const std::exception &e) {
        copy_err(err, errlen, e.what());
        return 4;
    }
}

// Quadtree::refine (core/partition.cpp:68-100): visit a point list, refine,
// and return the leaf list (region u0 v0 u1 v1 visits) as text.
int ref_quadtree(const double *uv, uint64_t n, uint64_t m_split, int rounds, char *out, int cap) {
    ramlt::AdaptationConfig cfg;
    ramlt::KernelController ctl(ramlt::ControllerKind::Regional, cfg);
    ramlt::Quadtree tree(ctl);
    int splits = 0;
    for (int r = 0; r < rounds; ++r) {
        for (uint64_t i = 0; i < n; ++i)
            tree.record_visit(tree.classify({uv[2 * i], uv[2 * i + 1]}));
        splits += tree.refine(m_split);
    }
    std::ostringstream os;
    for (const auto &leaf : tree.leaves())
        os << leaf.region << " " << leaf.u0 << " " << leaf.v0 << " " << leaf.u1 << " " << leaf.v1
           << " " << leaf.visits << "\n";
    std::string s = os.str();
    std::strncpy(out, s.c_str(), static_cast<size_t>(cap) - 1);
    out[cap - 1] = '\0';
    return splits;
}

// Analytic-target harness (BASELINE.json configs[1]) composed from the
// UNMODIFIED reference's own pieces: RandomSequence (core/rng.hpp),
// normal_quantile (core/sampling.cpp:20-60), mh_accept (core/mutations.cpp:198-208),
// KernelController::sigma_for / record_acceptance (core/adaptation.cpp:44-92),
// Grid2D::cell_of (core/partition.cpp:16-20) and the chain / init stream ids
// (core/driver.cpp:20-21, 223-225), driven in lockstep exactly as
// run_chain_span drives one step (core/driver.cpp:113-171).  Only the target
// density and the random-walk proposal are harness code (no reference
// counterpart exists); they are written out here and in
// oracle_mix_run independently with the same evaluation order.
namespace {
struct RefMixTarget {
    int D = 0, K = 0;
    std::vector<double> W, mu, ell;
};

RefMixTarget ref_mix_prepare(const oracle_mix_config *c) {
    RefMixTarget t;
    const int D = c->dim, K = c->n_comp;
    t.D = D;
    t.K = K;
    t.W.assign(static_cast<size_t>(K) * D * D, 0.0);
    t.mu.assign(c->means, c->means + static_cast<size_t>(K) * D);
    t.ell.assign(K, 0.0);
    const double half_log_2pi = 0.5 * std::log(2.0 * 3.14159265358979323846);
    for (int k = 0; k < K; ++k) {
        const double *S = c->covariances + static_cast<size_t>(k) * D * D;
        std::vector<double> L(static_cast<size_t>(D) * D, 0.0);
        for (int i = 0; i < D; ++i)
            for (int j = 0; j <= i; ++j) {
                double s = S[i * D + j];
                for (int q = 0; q < j; ++q)
                    s = s - L[i * D + q] * L[j * D + q];
                if (i == j) {
                    if (!(s > 0.0))
                        throw std::invalid_argument("mix: covariance is not positive definite");
                    L[i * D + i] = std::sqrt(s);
                } else {
                    L[i * D + j] = s / L[j * D + j];
                }
            }
        double *Wk = t.W.data() + static_cast<size_t>(k) * D * D;
        for (int j = 0; j < D; ++j) {
            Wk[j * D + j] = 1.0 / L[j * D + j];
            for (int i = j + 1; i < D; ++i) {
                double s = 0.0;
                for (int q = j; q < i; ++q)
                    s = s + L[i * D + q] * Wk[q * D + j];
                Wk[i * D + j] = -s / L[i * D + i];
            }
        }
        double e = std::log(c->weights[k]);
        for (int i = 0; i < D; ++i)
            e = e - std::log(L[i * D + i]);
        t.ell[k] = e - static_cast<double>(D) * half_log_2pi;
    }
    return t;
}

double ref_mix_log_target(const RefMixTarget &t, const double *x) {
    const int D = t.D;
    std::vector<double> e(t.K), dif(D);
    double m = -std::numeric_limits<double>::infinity();
    for (int k = 0; k < t.K; ++k) {
        const double *Wk = t.W.data() + static_cast<size_t>(k) * D * D;
        for (int j = 0; j < D; ++j)
            dif[j] = x[j] - t.mu[static_cast<size_t>(k) * D + j];
        double s = 0.0;
        for (int i = 0; i < D; ++i) {
            double z = 0.0;
            for (int j = 0; j <= i; ++j)
                z = z + Wk[i * D + j] * dif[j];
            s = s + z * z;
        }
        e[k] = t.ell[k] - 0.5 * s;
        m = e[k] > m ? e[k] : m;
    }
    double acc = 0.0;
    for (int k = 0; k < t.K; ++k)
        acc = acc + std::exp(e[k] - m);
    return m + std::log(acc);
}
} // namespace

int ref_mix_run(const oracle_mix_config *c, oracle_mix_out *o, char *err, int errlen) {
    try {
        if (c->chains < 1)
            throw std::logic_error("need at least one chain");
        constexpr uint64_t kStreamInit = 0x4000000000000001ULL;   // core/driver.cpp:21
        RefMixTarget t = ref_mix_prepare(c);
        const int C = c->chains, D = c->dim;
        ramlt::AdaptationConfig ac;
        ac.batch_size = c->batch_size;
        ac.gamma_max = c->gamma_max;
        ac.gamma_scale = c->gamma_scale;
        ac.target_acceptance = c->target_acceptance;
        ac.lambda_init = c->lambda_init;
        ac.lambda_min = c->lambda_min;
        ramlt::ControllerKind kind = c->strategy == 0   ? ramlt::ControllerKind::Fixed
                                     : c->strategy == 1 ? ramlt::ControllerKind::Global
                                                        : ramlt::ControllerKind::Regional;
        ramlt::KernelController ctl(kind, ac);
        std::unique_ptr<ramlt::Grid2D> grid;
        if (c->strategy == 2) {
            grid = std::make_unique<ramlt::Grid2D>(c->grid_n);
            for (int r = 0; r < grid->cell_count(); ++r)
                ctl.allocate_region();
        }
        std::vector<double> x(static_cast<size_t>(C) * D), lp(C), asum(C, 0.0);
        std::vector<uint64_t> nacc(C, 0);
        std::vector<ramlt::RandomSequence> rng;
        rng.reserve(C);
        for (int i = 0; i < C; ++i) {
            uint64_t g = static_cast<uint64_t>(c->chain_offset + i);
            ramlt::RandomSequence init(c->seed, kStreamInit + g * 2);
            bool ok = false;
            for (int attempt = 0; attempt < 1000 && !ok; ++attempt) {
                for (int d = 0; d < D; ++d)
                    x[static_cast<size_t>(i) * D + d] = init.next_double();
                lp[i] = ref_mix_log_target(t, &x[static_cast<size_t>(i) * D]);
                ok = std::isfinite(lp[i]);
            }
            if (!ok)
                throw std::runtime_error("mix: chain initialisation found no state with finite log density");
            rng.emplace_back(c->seed, g);
        }
        const uint64_t Ctot = c->chains_total > 0 ? static_cast<uint64_t>(c->chains_total) : C;
        std::vector<oracle_trace_row> trace;
        std::vector<ramlt::SigmaPair> sig(C);
        std::vector<int> reg(C);
        std::vector<double> y(D);
        for (uint64_t j = 0; j < c->steps; ++j) {
            // lockstep: the whole step reads the controller before any record
            for (int i = 0; i < C; ++i) {
                const double *xi = &x[static_cast<size_t>(i) * D];
                reg[i] = grid ? grid->cell_of(ramlt::CanonicalPoint2{xi[0], xi[1]}) : 0;
                sig[i] = ctl.sigma_for(reg[i]);
            }
            for (int i = 0; i < C; ++i) {
                double *xi = &x[static_cast<size_t>(i) * D];
                bool in = true;
                for (int d = 0; d < D; ++d) {
                    double u = rng[i].next_double();
                    y[d] = xi[d] + sig[i].primary * ramlt::normal_quantile(u);
                    in = in && (y[d] >= 0.0 && y[d] <= 1.0);
                }
                double a = 0.0, lpy = 0.0;
                if (in) {
                    lpy = ref_mix_log_target(t, y.data());
                    a = ramlt::mh_accept(1.0, std::exp(lpy - lp[i]), 1.0, 1.0, 1.0, 1.0);
                }
                if (auto ev = ctl.record_acceptance(reg[i], a))
                    trace.push_back({j * Ctot + static_cast<uint64_t>(c->chain_offset) + i, ev->region, ev->n,
                                     ev->lambda, ev->alpha_hat});
                bool acc = a > 0.0 && rng[i].next_double() < a;
                if (acc) {
                    for (int d = 0; d < D; ++d)
                        xi[d] = y[d];
                    lp[i] = lpy;
                }
                asum[i] += a;
                nacc[i] += acc ? 1 : 0;
                if (j < c->log_steps) {
                    if (o->log_a)
                        o->log_a[static_cast<size_t>(i) * c->log_steps + j] = a;
                    if (o->log_f)
                        o->log_f[static_cast<size_t>(i) * c->log_steps + j] =
                            static_cast<uint8_t>((acc ? 1 : 0) | 2 | 4);
                }
            }
        }
        if (o->x)
            std::memcpy(o->x, x.data(), sizeof(double) * x.size());
        if (o->log_pi)
            std::memcpy(o->log_pi, lp.data(), sizeof(double) * C);
        auto tal = ctl.tallies();
        o->n_regions = ctl.region_count();
        for (uint64_t r = 0; r < std::min<uint64_t>(o->cap_regions, ctl.region_count()); ++r) {
            if (o->lambda)
                o->lambda[r] = ctl.lambda_of(static_cast<int>(r));
            if (o->n)
                o->n[r] = ctl.updates_of(static_cast<int>(r));
            if (o->tally_accept)
                o->tally_accept[r] = tal[r].accept_sum;
            if (o->tally_visits)
                o->tally_visits[r] = tal[r].visits;
        }
        o->n_trace = trace.size();
        for (uint64_t i = 0; i < std::min<uint64_t>(o->cap_trace, trace.size()); ++i)
            o->trace[i] = trace[i];
        o->accepted = 0;
        o->acceptance_sum = 0.0;
        for (int i = 0; i < C; ++i) {
            o->accepted += nacc[i];
            o->acceptance_sum += asum[i];
        }
        return 0;
    } catch (const std::runtime_error &e) {
        copy_err(err, errlen, e.what());
        return 1;
    } catch (const std::invalid_argument &e) {
        copy_err(err, errlen, e.what());
        return 3;
    } catch (const std::logic_error &e) {
        copy_err(err, errlen, e.what());
        return 2;
    } catch (const std::exception &e) {
        copy_err(err, errlen, e.what());
        return 4;
    }
}

} // extern "C"
