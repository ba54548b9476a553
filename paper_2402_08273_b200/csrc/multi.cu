// multi.cu -- one ramlt_gpu handle over several devices of one process
// (create(..., n_dev, devs); §8(e): chains shard by global id).
//
// The reference runs every chain of run_render on host threads of one process
// (core/driver.cpp:282-297) and merges the per-chain films at the end
// (core/film.cpp:22-27; core/driver.cpp:315-330).  Here each device holds a
// contiguous shard of global chain ids in its own EngineT; the exchanges are
// the method's only shared state, done device-to-device over peer memory
// (NVLink / NVSwitch when the devices differ, a plain D2D copy when a test puts
// two shards on one device), fully stream-ordered with events, no host sync:
//
//   * pooled adaptation after every lockstep step: SUM visit counts and
//     fixed-point acceptance sums, MAX last mutation index per region, gathered
//     on the root device, reduced, broadcast; every shard then applies the
//     identical update (ramlt_kernels.cuh k_adapt_pool_apply, scan mode);
//   * quadtree visits at every m_refine barrier: SUM, then every shard runs the
//     identical deterministic refine (only shard 0 keeps the carried counts);
//   * film every `film_sync_steps` lockstep steps (configs[4]: 2^12) and at
//     metrics rows / reads: delta all-reduce (every shard's film becomes the
//     global film, so the normalised image and the rRMSE are global);
//   * b: substream partials computed per shard, concatenated in substream
//     order and reduced identically on every shard (bit-identical to 1 device).
//
// Chain c keeps its global id (RNG stream, decision order), so Fixed runs are
// identical to the single-device handle, and pooled adaptive runs are too
// (integer sums do not depend on the partition).
#include "engine.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <limits>
#include <memory>
#include <string>
#include <thread>
#include <vector>

namespace ramlt_b200 {

#define RAMLT_MCUDA(x)                                                                             \
    do {                                                                                           \
        cudaError_t e_ = (x);                                                                      \
        if (e_ != cudaSuccess)                                                                     \
            throw CudaError(std::string("cuda: ") + cudaGetErrorString(e_) + " at " #x);           \
    } while (0)

namespace {

// stage: [other shard][3][n] -- x_cnt, x_fx (SUM), x_last (MAX)
__global__ void k_x_reduce(unsigned long long *cnt, unsigned long long *fx, unsigned long long *last,
                           const unsigned long long *stage, int n_other, size_t n) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        unsigned long long c = cnt[i], f = fx[i], l = last[i];
        for (int s = 0; s < n_other; ++s) {
            const unsigned long long *b = stage + static_cast<size_t>(s) * 3 * n;
            c += b[i];
            f += b[n + i];
            l = max(l, b[2 * n + i]);
        }
        cnt[i] = c;
        fx[i] = f;
        last[i] = l;
    }
}

__global__ void k_u64_sum(unsigned long long *dst, const unsigned long long *stage, int n_other, size_t n) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        unsigned long long v = dst[i];
        for (int s = 0; s < n_other; ++s)
            v += stage[static_cast<size_t>(s) * n + i];
        dst[i] = v;
    }
}

// acc = root film - synced (first) / acc += other film - synced
__global__ void k_film_delta(double *acc, const double *film, const double *synced, size_t n, int first) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        double d = film[i] - synced[i];
        acc[i] = first ? d : acc[i] + d;
    }
}

__global__ void k_film_finish(double *root_film, double *synced, const double *acc, size_t n) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        double v = synced[i] + acc[i];
        root_film[i] = v;
        synced[i] = v;
    }
}

template <class T> struct DevBuf {
    T *p = nullptr;
    size_t n = 0;
    int dev = 0;
    void ensure(size_t count, int device) {
        if (count <= n)
            return;
        release();
        dev = device;
        RAMLT_MCUDA(cudaSetDevice(device));
        RAMLT_MCUDA(cudaMalloc(&p, count * sizeof(T)));
        n = count;
    }
    void release() {
        if (p) {
            cudaSetDevice(dev);
            cudaFree(p);
        }
        p = nullptr;
        n = 0;
    }
    ~DevBuf() { release(); }
};

}  // namespace

class MultiEngine final : public EngineBase {
public:
    MultiEngine(const HostScene &scene, const ramlt_render_desc &d, int n_dev, const int *devs, uint32_t film_sync)
        : d_(d), film_sync_(film_sync) {
        if (n_dev < 2)
            throw std::logic_error("multi-device handle needs at least two devices");
        if (d.chains < n_dev)
            throw std::logic_error("need at least one chain per device");
        if (d.chains_total > 0 && d.chains_total != d.chains)
            throw std::logic_error("a multi-device handle owns every chain (chains_total must be 0 or chains)");
        int count = 0;
        RAMLT_MCUDA(cudaGetDeviceCount(&count));
        for (int i = 0; i < n_dev; ++i)
            if (devs[i] < 0 || devs[i] >= count)
                throw std::invalid_argument("device ordinal out of range");
        adaptive_ = d.strategy != RAMLT_FIXED;
        quadtree_ = d.strategy == RAMLT_RA_QUADTREE;
        const long long C = d.chains;
        for (int i = 0; i < n_dev; ++i) {
            ramlt_render_desc di = d;
            long long off = i * C / n_dev, end = (i + 1) * C / n_dev;
            di.chains = static_cast<int32_t>(end - off);
            di.chains_total = C;
            di.chain_offset = off;
            di.device = devs[i];
            dev_.push_back(devs[i]);
            off_.push_back(off);
            RAMLT_MCUDA(cudaSetDevice(devs[i]));
            sh_.emplace_back(d.precision == RAMLT_F64 ? make_engine_f64(scene, di) : make_engine_f32(scene, di));
            if (adaptive_)
                sh_.back()->set_exchange_interval(1);
        }
        for (int i = 1; i < n_dev; ++i) {   // NVLink peer access root <-> shard (ignored when unavailable)
            if (dev_[i] == dev_[0])
                continue;
            int ok = 0;
            cudaDeviceCanAccessPeer(&ok, dev_[0], dev_[i]);
            if (ok) {
                cudaSetDevice(dev_[0]);
                if (cudaDeviceEnablePeerAccess(dev_[i], 0) != cudaSuccess)
                    cudaGetLastError();
                cudaSetDevice(dev_[i]);
                if (cudaDeviceEnablePeerAccess(dev_[0], 0) != cudaSuccess)
                    cudaGetLastError();
            }
        }
        ev_.resize(n_dev);
        for (int i = 0; i < n_dev; ++i) {
            RAMLT_MCUDA(cudaSetDevice(dev_[i]));
            RAMLT_MCUDA(cudaEventCreateWithFlags(&ev_[i], cudaEventDisableTiming));
        }
        next_metrics_ = d.metrics_interval;
        RAMLT_MCUDA(cudaSetDevice(dev_[0]));
    }

    ~MultiEngine() override {
        for (size_t i = 0; i < ev_.size(); ++i) {
            cudaSetDevice(dev_[i]);
            cudaEventDestroy(ev_[i]);
        }
        for (size_t i = 0; i < sh_.size(); ++i) {
            cudaSetDevice(dev_[i]);
            sh_[i].reset();
        }
    }

    // ---- b (core/driver.cpp:219-242): substreams split across devices -----------------
    void estimate_b(double *b, double *se) override {
        const uint64_t S = std::min<uint64_t>(d_.b_samples, d_.b_substreams ? d_.b_substreams : 65536);
        std::vector<double> part(2 * S);
        const int n = static_cast<int>(sh_.size());
        for_each_parallel([&](int i) {
            uint64_t b0 = static_cast<uint64_t>(i) * S / n, b1 = static_cast<uint64_t>(i + 1) * S / n;
            sh_[i]->estimate_b_partials(b0, b1, part.data() + 2 * b0);
        });
        reduce_b(part.data(), S, b, se);
    }
    void estimate_b_partials(uint64_t begin, uint64_t end, double *out) override {
        on(0);
        sh_[0]->estimate_b_partials(begin, end, out);
    }
    void reduce_b(const double *partials, uint64_t n, double *b, double *se) override {
        for (size_t i = 0; i < sh_.size(); ++i) {
            on(static_cast<int>(i));
            sh_[i]->reduce_b(partials, n, i == 0 ? b : nullptr, i == 0 ? se : nullptr);
        }
        b_set_ = true;
    }
    void set_b(double b) override {
        for (size_t i = 0; i < sh_.size(); ++i) {
            on(static_cast<int>(i));
            sh_[i]->set_b(b);
        }
        b_set_ = true;
    }
    void init_chains() override {
        for_each_parallel([&](int i) { sh_[i]->init_chains(); });
        chains_ready_ = true;
    }

    // ---- the span loop with the exchanges ------------------------------------------------
    // Every shard advances the same canonical lockstep steps (EngineT::run_steps),
    // then the exchanges run; adaptive strategies exchange after every step.
    uint64_t run_steps(uint32_t n, uint32_t *executed) override {
        if (!chains_ready_)
            throw std::logic_error("run before init_chains");
        if (!t0_set_) {
            synchronize();
            t0_ = std::chrono::steady_clock::now();
            t0_set_ = true;
        }
        uint32_t total = 0;
        while (total < n) {
            uint32_t k = adaptive_ ? 1u : n - total;
            if (film_sync_)
                k = std::min<uint32_t>(k, film_sync_ - static_cast<uint32_t>(steps_ % film_sync_));
            uint64_t reached = done_;
            uint32_t ex = 0;
            for (size_t i = 0; i < sh_.size(); ++i) {
                on(static_cast<int>(i));
                reached = sh_[i]->run_steps(k, &ex);   // identical on every shard
            }
            done_ = reached;
            steps_ += ex;
            total += ex;
            if (ex) {
                film_dirty_ = true;
                if (adaptive_)
                    exchange_adaptation();
            }
            bool refined = false;
            if (quadtree_) {
                on(0);
                if (sh_[0]->refine_pending()) {
                    exchange_refine();
                    refined = true;
                }
            }
            if (film_sync_ && ex && steps_ % film_sync_ == 0)
                sync_film();
            if (done_ == next_metrics_ || (done_ == d_.mutations && last_row_ != done_)) {
                push_row();
                next_metrics_ = done_ + d_.metrics_interval;
            }
            if (!ex && !refined)
                break;
        }
        if (executed)
            *executed = total;
        return done_;
    }

    // run(m): whole lockstep steps until m more mutations are done (exact when
    // the target is a span boundary, e.g. the configured total; otherwise the
    // last step may pass it by less than one lockstep step).
    void run(uint64_t mutations) override {
        const uint64_t C = static_cast<uint64_t>(d_.chains);
        const uint64_t target = done_ + mutations;
        while (done_ < target) {
            uint64_t need = std::max<uint64_t>(1, (target - done_) / C);
            uint32_t ex = 0;
            run_steps(static_cast<uint32_t>(std::min<uint64_t>(need, 1u << 20)), &ex);
            if (!ex)
                throw std::logic_error("multi-device run made no progress");
        }
    }

    void render() override {
        if (!b_set_)
            estimate_b(nullptr, nullptr);
        if (!chains_ready_)
            init_chains();
        if (d_.time_budget_s > 0.0) {
            if (!t0_set_) {
                synchronize();
                t0_ = std::chrono::steady_clock::now();
                t0_set_ = true;
            }
            for (;;) {
                run(std::min<uint64_t>(d_.metrics_interval, next_metrics_ - done_));
                synchronize();
                double t = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0_).count();
                if (t >= d_.time_budget_s)
                    break;
            }
        } else {
            run(d_.mutations - std::min(d_.mutations, done_));
        }
        if (last_row_ != done_)
            push_row();
        sync_film();
    }

    void synchronize() override {
        for (size_t i = 0; i < sh_.size(); ++i) {
            on(static_cast<int>(i));
            sh_[i]->synchronize();
        }
    }

    // ---- outputs: shard 0 holds the global adaptation state and (after a sync) film -----
    void read_stats(ramlt_stats *out) override {
        ramlt_stats s{};
        double acc_sum = 0.0, lum = 0.0;
        for (size_t i = 0; i < sh_.size(); ++i) {
            on(static_cast<int>(i));
            ramlt_stats si;
            sh_[i]->read_stats(&si);
            if (i == 0)
                s = si;
            else {
                s.perturbation_proposals += si.perturbation_proposals;
                s.large_step_proposals += si.large_step_proposals;
                s.rays_closest += si.rays_closest;
                s.rays_visibility += si.rays_visibility;
                s.kernel_launches += si.kernel_launches;
                s.step_kernel_ms = std::max(s.step_kernel_ms, si.step_kernel_ms);
                s.step_kernel_launches += si.step_kernel_launches;
                s.trace_kernel_ms = std::max(s.trace_kernel_ms, si.trace_kernel_ms);
                s.trace_kernel_launches += si.trace_kernel_launches;
                s.wavefront_rounds = std::max(s.wavefront_rounds, si.wavefront_rounds);
            }
            acc_sum += si.mean_acceptance * static_cast<double>(si.perturbation_proposals);
            lum += si.film_luminance;
        }
        s.total_mutations = done_;
        s.mean_acceptance = s.perturbation_proposals ? acc_sum / static_cast<double>(s.perturbation_proposals) : 0.0;
        s.film_luminance = lum;
        s.n_metrics = rows_.size();
        s.loop_time_s = rows_.empty() ? 0.0 : rows_.back()[0];
        s.kernel_launches += launches_;
        *out = s;
    }
    void read_film(double *rgb, double *lum) override {
        if (film_dirty_)
            sync_film();
        on(0);
        sh_[0]->read_film(rgb, nullptr);
        if (lum) {
            double t = 0.0;
            for (size_t i = 0; i < sh_.size(); ++i) {
                on(static_cast<int>(i));
                double l = 0.0;
                sh_[i]->read_film(nullptr, &l);
                t += l;
            }
            *lum = t;
        }
    }
    void read_image(float *rgb) override {
        if (film_dirty_)
            sync_film();
        on(0);
        sh_[0]->read_image(rgb);
    }
    uint64_t read_tallies(double *acc, uint64_t *vis, uint64_t cap) override {
        on(0);
        return sh_[0]->read_tallies(acc, vis, cap);
    }
    uint64_t read_regions(double *lambda, uint64_t *n, uint64_t cap) override {
        on(0);
        return sh_[0]->read_regions(lambda, n, cap);
    }
    uint64_t read_trace(ramlt_trace_row *rows, uint64_t cap) override {
        on(0);
        return sh_[0]->read_trace(rows, cap);
    }
    uint64_t read_metrics(double *rows, uint64_t cap) override {
        uint64_t m = std::min<uint64_t>(rows_.size(), cap);
        for (uint64_t i = 0; i < m; ++i)
            for (int q = 0; q < 4; ++q)
                rows[4 * i + q] = rows_[i][q];
        return rows_.size();
    }
    void read_decisions(uint32_t K, double *a, uint8_t *flags) override {
        for (size_t i = 0; i < sh_.size(); ++i) {
            on(static_cast<int>(i));
            size_t o = static_cast<size_t>(off_[i]) * K;
            sh_[i]->read_decisions(K, a ? a + o : nullptr, flags ? flags + o : nullptr);
        }
    }
    void read_chain_lengths(int32_t *k) override {
        for (size_t i = 0; i < sh_.size(); ++i) {
            on(static_cast<int>(i));
            sh_[i]->read_chain_lengths(k + off_[i]);
        }
    }
    std::string read_partition() override {
        // leaf visit counts live split over the shards between refines: dump their SUM
        std::vector<uint64_t> tot, part;
        for (size_t i = 0; i < sh_.size(); ++i) {
            on(static_cast<int>(i));
            uint64_t *v = nullptr, n = 0;
            sh_[i]->visits_device(&v, &n);
            sh_[i]->synchronize();
            part.assign(n, 0);
            if (n)
                RAMLT_MCUDA(cudaMemcpy(part.data(), v, n * sizeof(uint64_t), cudaMemcpyDeviceToHost));
            if (i == 0)
                tot = part;
            else
                for (uint64_t q = 0; q < n && q < tot.size(); ++q)
                    tot[q] += part[q];
        }
        on(0);
        return sh_[0]->read_partition_visits(tot.data(), tot.size());
    }
    std::string read_partition_visits(const uint64_t *visits, uint64_t n) override {
        on(0);
        return sh_[0]->read_partition_visits(visits, n);
    }
    void set_reference(const float *rgb, int width, int height) override {
        on(0);
        sh_[0]->set_reference(rgb, width, height);
        has_ref_ = true;
    }
    void trace_benchmark(uint64_t n_rays, double *ms, uint64_t *hits) override {
        on(0);
        sh_[0]->trace_benchmark(n_rays, ms, hits);
    }
    void *stream_handle() override { return sh_[0]->stream_handle(); }
    double rrmse(uint64_t at) override {
        if (film_dirty_)
            sync_film();
        on(0);
        return sh_[0]->rrmse(at);
    }
    bool metrics_sums(uint64_t, double *, double *) override { return false; }

    // per-shard plumbing is internal to this handle
    [[noreturn]] static void shard_only(const char *what) {
        throw std::logic_error(std::string(what) + " is not available on a multi-device handle");
    }
    void set_stream(void *) override { shard_only("set_stream"); }
    void film_device(double **, uint64_t *) override { shard_only("film_device"); }
    void adapt_exchange(uint64_t **, uint64_t **, uint64_t **, uint64_t *) override { shard_only("adapt_exchange"); }
    void adapt_apply() override { shard_only("adapt_apply"); }
    void set_exchange_interval(uint32_t) override { shard_only("set_exchange_interval"); }
    void visits_device(uint64_t **, uint64_t *) override { shard_only("visits_device"); }
    bool refine_pending() override { return false; }
    void refine_now(bool) override { shard_only("refine"); }

private:
    void on(int i) const { RAMLT_MCUDA(cudaSetDevice(dev_[i])); }
    cudaStream_t st(int i) const { return static_cast<cudaStream_t>(sh_[i]->stream_handle()); }

    template <class F> void for_each_parallel(F &&f) {
        const int n = static_cast<int>(sh_.size());
        std::vector<std::string> err(n);
        std::vector<int> code(n, 0);
        std::vector<std::thread> th;
        for (int i = 0; i < n; ++i)
            th.emplace_back([&, i] {
                try {
                    on(i);
                    f(i);
                } catch (const CudaError &e) {
                    err[i] = e.what(), code[i] = 5;
                } catch (const std::invalid_argument &e) {
                    err[i] = e.what(), code[i] = 3;
                } catch (const std::logic_error &e) {
                    err[i] = e.what(), code[i] = 2;
                } catch (const std::runtime_error &e) {
                    err[i] = e.what(), code[i] = 1;
                } catch (const std::exception &e) {
                    err[i] = e.what(), code[i] = 4;
                }
            });
        for (auto &t : th)
            t.join();
        for (int i = 0; i < n; ++i)
            switch (code[i]) {   // rethrow the first shard's failure with its type
            case 0: break;
            case 5: throw CudaError(err[i]);
            case 3: throw std::invalid_argument(err[i]);
            case 2: throw std::logic_error(err[i]);
            case 1: throw std::runtime_error(err[i]);
            default: throw std::runtime_error(err[i]);
            }
        on(0);
    }

    // gather `arrays` (k per shard, n u64 each) of shards 1.. into the root's stage
    // buffer on the root stream, after each shard's last enqueued work
    void gather(const std::vector<std::vector<unsigned long long *>> &arrays, size_t n, DevBuf<unsigned long long> &stage) {
        const int ns = static_cast<int>(sh_.size());
        const size_t k = arrays[0].size();
        stage.ensure(static_cast<size_t>(ns - 1) * k * n, dev_[0]);
        for (int i = 1; i < ns; ++i) {
            on(i);
            RAMLT_MCUDA(cudaEventRecord(ev_[i], st(i)));
        }
        on(0);
        for (int i = 1; i < ns; ++i) {
            RAMLT_MCUDA(cudaStreamWaitEvent(st(0), ev_[i], 0));
            for (size_t q = 0; q < k; ++q)
                RAMLT_MCUDA(cudaMemcpyPeerAsync(stage.p + (static_cast<size_t>(i - 1) * k + q) * n, dev_[0],
                                                arrays[i][q], dev_[i], n * sizeof(unsigned long long), st(0)));
        }
    }
    // broadcast the root's arrays to every shard, after the root's reduction; the
    // root stream then waits for every copy, so the root's next writes (apply,
    // refine, splats) cannot race with a peer still reading its buffers
    void broadcast(const std::vector<std::vector<unsigned long long *>> &arrays, size_t bytes_each) {
        const int ns = static_cast<int>(sh_.size());
        on(0);
        RAMLT_MCUDA(cudaEventRecord(ev_[0], st(0)));
        for (int i = 1; i < ns; ++i) {
            on(i);
            RAMLT_MCUDA(cudaStreamWaitEvent(st(i), ev_[0], 0));
            for (size_t q = 0; q < arrays[0].size(); ++q)
                RAMLT_MCUDA(cudaMemcpyPeerAsync(arrays[i][q], dev_[i], arrays[0][q], dev_[0], bytes_each, st(i)));
        }
        join_root();
    }
    void join_root() {
        const int ns = static_cast<int>(sh_.size());
        for (int i = 1; i < ns; ++i) {
            on(i);
            RAMLT_MCUDA(cudaEventRecord(ev_[i], st(i)));
        }
        on(0);
        for (int i = 1; i < ns; ++i)
            RAMLT_MCUDA(cudaStreamWaitEvent(st(0), ev_[i], 0));
    }
    unsigned grid(size_t n) const { return static_cast<unsigned>(std::min<size_t>((n + 255) / 256, 148 * 8)); }

    void exchange_adaptation() {
        const int ns = static_cast<int>(sh_.size());
        std::vector<std::vector<unsigned long long *>> arr(ns);
        uint64_t n = 0;
        for (int i = 0; i < ns; ++i) {
            uint64_t *c, *f, *l;
            on(i);
            sh_[i]->adapt_exchange(&c, &f, &l, &n);
            arr[i] = {reinterpret_cast<unsigned long long *>(c), reinterpret_cast<unsigned long long *>(f),
                      reinterpret_cast<unsigned long long *>(l)};
        }
        if (n) {
            gather(arr, n, xstage_);
            k_x_reduce<<<grid(n), 256, 0, st(0)>>>(arr[0][0], arr[0][1], arr[0][2], xstage_.p, ns - 1, n);
            RAMLT_MCUDA(cudaGetLastError());
            ++launches_;
            broadcast(arr, n * sizeof(unsigned long long));
        }
        for (int i = 0; i < ns; ++i) {
            on(i);
            sh_[i]->adapt_apply();
        }
    }

    void exchange_refine() {
        const int ns = static_cast<int>(sh_.size());
        std::vector<std::vector<unsigned long long *>> arr(ns);
        uint64_t n = 0;
        for (int i = 0; i < ns; ++i) {
            uint64_t *v;
            on(i);
            sh_[i]->visits_device(&v, &n);
            arr[i] = {reinterpret_cast<unsigned long long *>(v)};
        }
        if (n) {
            gather(arr, n, xstage_);
            k_u64_sum<<<grid(n), 256, 0, st(0)>>>(arr[0][0], xstage_.p, ns - 1, n);
            RAMLT_MCUDA(cudaGetLastError());
            ++launches_;
            broadcast(arr, n * sizeof(unsigned long long));
        }
        for (int i = 0; i < ns; ++i) {
            on(i);
            sh_[i]->refine_now(i == 0);   // the carried counts stay on one shard only
        }
    }

    // Delta all-reduce of the fp64 films: every shard's film becomes the global
    // film (core/film.cpp:22-27 merge), exactly once per contribution.
    void sync_film() {
        const int ns = static_cast<int>(sh_.size());
        std::vector<double *> film(ns);
        uint64_t n = 0;
        for (int i = 0; i < ns; ++i) {
            on(i);
            sh_[i]->film_device(&film[i], &n);   // folds the fp32 staging film first
        }
        if (!synced_.p) {
            synced_.ensure(n, dev_[0]);
            on(0);
            RAMLT_MCUDA(cudaMemsetAsync(synced_.p, 0, n * sizeof(double), st(0)));
        }
        acc_.ensure(n, dev_[0]);
        fstage_.ensure(n, dev_[0]);
        on(0);
        k_film_delta<<<grid(n), 256, 0, st(0)>>>(acc_.p, film[0], synced_.p, n, 1);
        ++launches_;
        for (int i = 1; i < ns; ++i) {
            on(i);
            RAMLT_MCUDA(cudaEventRecord(ev_[i], st(i)));
            on(0);
            RAMLT_MCUDA(cudaStreamWaitEvent(st(0), ev_[i], 0));
            RAMLT_MCUDA(cudaMemcpyPeerAsync(fstage_.p, dev_[0], film[i], dev_[i], n * sizeof(double), st(0)));
            k_film_delta<<<grid(n), 256, 0, st(0)>>>(acc_.p, fstage_.p, synced_.p, n, 0);
            ++launches_;
        }
        k_film_finish<<<grid(n), 256, 0, st(0)>>>(film[0], synced_.p, acc_.p, n);
        ++launches_;
        RAMLT_MCUDA(cudaGetLastError());
        RAMLT_MCUDA(cudaEventRecord(ev_[0], st(0)));
        for (int i = 1; i < ns; ++i) {
            on(i);
            RAMLT_MCUDA(cudaStreamWaitEvent(st(i), ev_[0], 0));
            RAMLT_MCUDA(cudaMemcpyPeerAsync(film[i], dev_[i], film[0], dev_[0], n * sizeof(double), st(i)));
        }
        join_root();
        film_dirty_ = false;
    }

    // MetricsRow (core/driver.hpp:50-55): wall time, mutations, rRMSE of the
    // global image (NaN without a reference), interval acceptance over all shards
    void push_row() {
        double num = 0.0, den = 0.0;
        for (size_t i = 0; i < sh_.size(); ++i) {
            double a = 0.0, b = 0.0;
            on(static_cast<int>(i));
            sh_[i]->synchronize();
            if (sh_[i]->metrics_sums(done_, &a, &b)) {
                num += a;
                den += b;
            }
        }
        double rr = std::numeric_limits<double>::quiet_NaN();
        if (has_ref_)
            rr = rrmse(done_);
        double t = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0_).count();
        rows_.push_back({t, static_cast<double>(done_), rr, den > 0 ? num / den : 0.0});
        last_row_ = done_;
    }

    ramlt_render_desc d_;
    uint32_t film_sync_;
    std::vector<std::unique_ptr<EngineBase>> sh_;
    std::vector<int> dev_;
    std::vector<long long> off_;
    std::vector<cudaEvent_t> ev_;
    bool adaptive_ = false, quadtree_ = false, has_ref_ = false;
    bool b_set_ = false, chains_ready_ = false, film_dirty_ = false, t0_set_ = false;
    uint64_t done_ = 0, next_metrics_ = 0, steps_ = 0, launches_ = 0;
    uint64_t last_row_ = std::numeric_limits<uint64_t>::max();
    std::chrono::steady_clock::time_point t0_;
    std::vector<std::array<double, 4>> rows_;
    DevBuf<unsigned long long> xstage_;
    DevBuf<double> synced_, acc_, fstage_;
};

EngineBase *make_engine_multi(const HostScene &scene, const ramlt_render_desc &desc, int n_dev, const int *devs,
                              uint32_t film_sync_steps) {
    if (n_dev < 1 || !devs)
        throw std::logic_error("need at least one device");
    if (n_dev == 1) {
        ramlt_render_desc d = desc;
        d.device = devs[0];
        return d.precision == RAMLT_F64 ? make_engine_f64(scene, d) : make_engine_f32(scene, d);
    }
    return new MultiEngine(scene, desc, n_dev, devs, film_sync_steps);
}

}  // namespace ramlt_b200
