// engine.h -- precision-agnostic interface of the B200 engine (host side).
#pragma once

#include "../../include/ramlt_gpu.h"

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace ramlt_b200 {

// Exceptions mapped to the C-ABI status codes (ramlt_gpu.h).
struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

struct HostScene {
    double cam[10];   // position, look_at, up, fov
    std::vector<ramlt_material> mats;
    std::vector<ramlt_sphere> sph;
    std::vector<ramlt_triangle> tri;
    std::vector<double> emit;   // 3 per emitter
};

// Camera basis exactly as the reference builds it (core/camera.cpp:8-30).
struct CameraBasis {
    double pos[3], right[3], up[3], fwd[3];
    double tanh, aspect, area, sensor;
};
CameraBasis make_camera(const double cam[10], int width, int height);

class EngineBase {
public:
    virtual ~EngineBase() = default;
    virtual void estimate_b(double *b, double *se) = 0;
    virtual void estimate_b_partials(uint64_t begin, uint64_t end, double *out) = 0;
    virtual void reduce_b(const double *partials, uint64_t n, double *b, double *se) = 0;
    virtual void set_b(double b) = 0;
    virtual void init_chains() = 0;
    virtual void run(uint64_t mutations) = 0;
    virtual uint64_t run_steps(uint32_t n, uint32_t *executed) = 0;
    virtual void render() = 0;
    virtual void synchronize() = 0;
    virtual void read_stats(ramlt_stats *out) = 0;
    virtual void read_film(double *rgb, double *lum) = 0;
    virtual void read_image(float *rgb) = 0;
    virtual uint64_t read_tallies(double *acc, uint64_t *vis, uint64_t cap) = 0;
    virtual uint64_t read_regions(double *lambda, uint64_t *n, uint64_t cap) = 0;
    virtual uint64_t read_trace(ramlt_trace_row *rows, uint64_t cap) = 0;
    virtual uint64_t read_metrics(double *rows, uint64_t cap) = 0;
    virtual void read_decisions(uint32_t K, double *a, uint8_t *flags) = 0;
    virtual void read_chain_lengths(int32_t *k) = 0;
    virtual std::string read_partition() = 0;
    // the dump with caller-supplied per-region visit counts (sharded runs: the SUM over shards)
    virtual std::string read_partition_visits(const uint64_t *visits, uint64_t n) = 0;
    virtual void set_stream(void *stream) = 0;
    virtual void film_device(double **film, uint64_t *n) = 0;
    virtual void adapt_exchange(uint64_t **cnt, uint64_t **fx, uint64_t **last, uint64_t *n) = 0;
    virtual void adapt_apply() = 0;
    virtual void set_exchange_interval(uint32_t steps) = 0;
    virtual void visits_device(uint64_t **visits, uint64_t *n) = 0;
    virtual bool refine_pending() = 0;
    virtual void refine_now(bool keep_counts) = 0;
    virtual void trace_benchmark(uint64_t n_rays, double *ms, uint64_t *hits) = 0;
    virtual void set_reference(const float *rgb, int width, int height) = 0;
    // multi-device handle (multi.cu) plumbing
    virtual void *stream_handle() = 0;
    virtual double rrmse(uint64_t at) = 0;   // error_report rRMSE of this handle's film; NaN without a reference
    // interval acceptance sums (accepted, proposals) of the metrics row flushed at `at`
    virtual bool metrics_sums(uint64_t at, double *num, double *den) = 0;

    std::string last_error;
};

EngineBase *make_engine_f32(const HostScene &scene, const ramlt_render_desc &desc);
EngineBase *make_engine_f64(const HostScene &scene, const ramlt_render_desc &desc);
// One handle over several devices (chains sharded by global id, pooled adaptation
// and quadtree visits exchanged every lockstep step, film every film_sync steps).
EngineBase *make_engine_multi(const HostScene &scene, const ramlt_render_desc &desc, int n_dev, const int *devs,
                              uint32_t film_sync_steps);

}  // namespace ramlt_b200
