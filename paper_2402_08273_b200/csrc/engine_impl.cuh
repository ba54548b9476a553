// engine_impl.cuh -- EngineT<R>: device memory, the span loop and the
// barriers of run_render (core/driver.cpp:177-342) around the sm_100a kernels.
#pragma once

#include "bvh.h"
#include "engine.h"
#include "ramlt_kernels.cuh"
#include "ramlt_step_co.cuh"
#include "ramlt_wavefront.cuh"
#include "bvh_layout.h"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <sstream>
#include <vector>

namespace ramlt_b200 {

#define RAMLT_CUDA(x)                                                                              \
    do {                                                                                           \
        cudaError_t e_ = (x);                                                                      \
        if (e_ != cudaSuccess) {                                                                   \
            cudaGetLastError(); /* a failed launch must not resurface at the next check */         \
            throw CudaError(std::string("cuda: ") + cudaGetErrorString(e_) + " at " #x);           \
        }                                                                                          \
    } while (0)

template <class T> struct DBuf {
    T *p = nullptr;
    size_t n = 0;
    void alloc(size_t count) {
        free();
        n = count;
        if (count)
            RAMLT_CUDA(cudaMalloc(&p, count * sizeof(T)));
    }
    void zero(cudaStream_t s) {
        if (n)
            RAMLT_CUDA(cudaMemsetAsync(p, 0, n * sizeof(T), s));
    }
    void free() {
        if (p)
            cudaFree(p);
        p = nullptr;
        n = 0;
    }
    ~DBuf() { free(); }
};

template <class R> class EngineT final : public EngineBase {
public:
    EngineT(const HostScene &scene, const ramlt_render_desc &d);
    ~EngineT() override;

    void estimate_b(double *b, double *se) override;
    void estimate_b_partials(uint64_t begin, uint64_t end, double *out) override;
    void reduce_b(const double *partials, uint64_t n, double *b, double *se) override;
    void set_b(double b) override {
        b_ = b;
        b_set_ = true;
    }
    void init_chains() override;
    void run(uint64_t mutations) override;
    uint64_t run_steps(uint32_t n, uint32_t *executed) override;
    void render() override;
    void synchronize() override { RAMLT_CUDA(cudaStreamSynchronize(stream_)); }
    void read_stats(ramlt_stats *out) override;
    void read_film(double *rgb, double *lum) override;
    void read_image(float *rgb) override;
    uint64_t read_tallies(double *acc, uint64_t *vis, uint64_t cap) override;
    uint64_t read_regions(double *lambda, uint64_t *n, uint64_t cap) override;
    uint64_t read_trace(ramlt_trace_row *rows, uint64_t cap) override;
    uint64_t read_metrics(double *rows, uint64_t cap) override;
    void read_decisions(uint32_t K, double *a, uint8_t *flags) override;
    void read_chain_lengths(int32_t *k) override {
        RAMLT_CUDA(cudaStreamSynchronize(stream_));
        RAMLT_CUDA(cudaMemcpy(k, klen_.p, static_cast<size_t>(C_) * sizeof(int), cudaMemcpyDeviceToHost));
    }
    std::string read_partition() override { return read_partition_visits(nullptr, 0); }
    std::string read_partition_visits(const uint64_t *visits, uint64_t n) override;
    void set_stream(void *stream) override {
        stream_ = static_cast<cudaStream_t>(stream);
        own_stream_ = false;
    }
    void film_device(double **film, uint64_t *n) override {
        fold();
        *film = film64_.p;
        *n = film64_.n;
    }
    void adapt_exchange(uint64_t **cnt, uint64_t **fx, uint64_t **last, uint64_t *n) override {
        *cnt = reinterpret_cast<uint64_t *>(x_cnt_.p);
        *fx = reinterpret_cast<uint64_t *>(x_fx_.p);
        *last = reinterpret_cast<uint64_t *>(x_last_.p);
        *n = static_cast<uint64_t>(n_regions_host_);
    }
    void adapt_apply() override;
    void set_exchange_interval(uint32_t steps) override { exchange_interval_ = steps; }
    void visits_device(uint64_t **visits, uint64_t *n) override {
        *visits = reinterpret_cast<uint64_t *>(visits_.p);
        *n = static_cast<uint64_t>(n_regions_host_);
    }
    bool refine_pending() override { return refine_pending_; }
    void trace_benchmark(uint64_t n_rays, double *ms, uint64_t *hits) override;
    void set_reference(const float *rgb, int width, int height) override;
    double rrmse_now(uint64_t at);
    void *stream_handle() override { return stream_; }
    double rrmse(uint64_t at) override {
        return ref_img_.p && at > 0 ? rrmse_now(at) : std::numeric_limits<double>::quiet_NaN();
    }
    bool metrics_sums(uint64_t at, double *num, double *den) override {
        for (auto it = metrics_.rbegin(); it != metrics_.rend(); ++it)
            if (static_cast<uint64_t>((*it)[1]) == at) {
                *num = (*it)[4];
                *den = (*it)[5];
                return true;
            }
        return false;
    }
    DBuf<float> ref_img_;      // RenderConfig::reference (driver.hpp:38) for the metrics rRMSE
    DBuf<double> rrmse_part_;
    void refine_now(bool keep_counts) override {
        if (!refine_pending_)
            return;
        refine_pending_ = false;
        refine();
        if (!keep_counts)
            RAMLT_CUDA(cudaMemsetAsync(visits_.p, 0, static_cast<size_t>(n_regions_host_) * sizeof(unsigned long long),
                                       stream_));
    }

private:
    rd::StepParams<R> params() const;
    rd::RegionArrays regions() const;
    rd::TraceBuf tracebuf() const;
    rd::AdaptCfg adaptcfg() const;
    void launch_step(int j0, int j1, unsigned long long span_start, unsigned long long per,
                     unsigned long long rem, bool record);
    void adapt_after_step(int j, unsigned long long span_start);
    template <bool INIT = false> void launch_step_co(const rd::StepParams<R> &P);
    template <int RK, bool INIT = false> void launch_step_wf(rd::StepParams<R> P);
    bool launch_coop(int j0, int j1, unsigned long long span_start, unsigned long long per,
                     unsigned long long rem);
    int coop_state_ = -1;   // -1 unknown, 0 unavailable, 1 usable
    void refine();
    void fold();
    void flush_metrics(uint64_t at);
    void check_err(const char *what);
    void alloc_regions(size_t cap);
    void grow_regions(size_t cap);
    void reduce_chains(bool reset_interval, double out[6]);
    void finalize_stats();

    ramlt_render_desc d_;
    HostScene hs_;
    CameraBasis cb_;
    int C_;
    long long Ctot_, off_;
    int G_;
    int ctl_;      // 0 fixed, 1 global, 2 regional
    int pkind_;    // partition kind (PartView::kind)
    int adapt_;    // 0 literal, 1 pooled
    size_t smem_;
    cudaStream_t stream_ = nullptr;
    bool own_stream_ = true;
    uint32_t exchange_interval_ = 0;
    bool refine_pending_ = false;   // sharded runs: refine after the visit all-reduce

    // scene
    DBuf<rd::TriD<R>> tri_;
    DBuf<rd::SphD<R>> sph_;
    DBuf<rd::MatD<R>> mat_;
    DBuf<rd::V3<R>> emit_;
    DBuf<unsigned char> bvh_;   // BVH units: nodes + leaf triangle records (bvh_layout.h)
    bool use_bvh_ = false;
    int bvh_depth_ = 0;
    // chains
    DBuf<rd::GV<R>> verts_;
    DBuf<rd::GV<R>> pv_scratch_;   // k_step_co proposal vertices in global memory (L1/L2-cached)
    bool co_pv_global_ = true;     // RAMLT_CO_PV=smem: in shared memory (caps occupancy)
    DBuf<int> klen_;
    DBuf<unsigned> smask_;
    DBuf<R> cf_, cr_;
    DBuf<double> eyeden_;
    DBuf<unsigned long long> rng0_, rng1_;
    DBuf<double> acc_, iacc_, lum_;
    DBuf<unsigned long long> npert_, nlarge_, ipert_, nsteps_;
    DBuf<double> log_a_;
    DBuf<unsigned char> log_f_;
    DBuf<int> vreg_;
    DBuf<double> va_;
    DBuf<int> err_;
    DBuf<unsigned long long> rays_;
    DBuf<unsigned> work_;     // work-stealing counter of k_step_co
    bool use_co_ = false;     // G == 1: the coroutine kernel (default with a BVH)
    bool use_co_init_ = false;  // chain initialisation with the coroutine kernel (default with a BVH)
    int steal_ = 1;           // RAMLT_STEP_KERNEL=co_static: one chain per lane, no stealing
    int init_refill_ = 8;     // the same for chain initialisation (RAMLT_CO_INIT_REFILL; c4 init 8/16/24/32: 0.81/0.84/0.85/0.95 s)
    int refill_ = 24;         // k_step_co (BVH): RAMLT_CO_REFILL idle lanes end a traversal round (c4: 4/8/16/24/28/32 -> 62.3/65.8/70.0/71.8/72.2/71.3 M)
    int co_carveout_ = -1;    // k_step_co: RAMLT_CO_CARVEOUT percent (-1: driver default)
    // wavefront step (BVH scenes, ramlt_wavefront.cuh): RAMLT_STEP_KERNEL=wf (default) | co
    bool use_wf_ = false;
    bool use_wf_init_ = false;   // chain initialisation as wavefront rounds (RAMLT_INIT_KERNEL=wf)
    int wf_refill_ = 8;       // k_wf_trace: RAMLT_WF_REFILL idle lanes end a traversal round
    int wf_check_ = 4;        // rounds between host checks of the queue length (RAMLT_WF_CHECK)
    bool wf_log_ = false;     // RAMLT_WF_LOG=1
    bool wf_bounce_ = true;   // RAMLT_WF_BOUNCE=0: the large-step bounce loop resumed by k_wf_logic instead of k_wf_bounce
    int wf_pipes_ = 1;        // RAMLT_WF_PIPES: chain ranges stepped as concurrent wavefront pipelines
    size_t wf_pipes_min_ = size_t(1) << 18;   // RAMLT_WF_PIPES_MIN: fewest chains split into pipelines
    int wf_lblk_ = 0, wf_tblk_ = 0;   // RAMLT_WF_LBLK / RAMLT_WF_TBLK: resident blocks per SM of a pipeline's kernels
    cudaStream_t wf_stream2_ = nullptr;
    cudaEvent_t wf_ev_[3] = {nullptr, nullptr, nullptr};
    bool wf_poll_ = false;    // RAMLT_WF_POLL=1: poll the queue length every wf_check_ rounds even for one-step launches
    DBuf<uint4> wf_state_;
    DBuf<rd::GV<R>> wf_pv_;
    DBuf<rd::WfRay<R>> wf_rays_;   // one round's rays: up to max_vertices - 1 per chain (a visibility batch)
    DBuf<rd::WfHit<R>> wf_hits_;   // closest-hit answers by chain
    DBuf<unsigned> wf_occ_;        // visibility-batch answers by chain (bit k: ray k occluded)
    DBuf<int> wf_cq_[2];           // chain queues (ping-pong)
    DBuf<unsigned> wf_cnt_;        // chain-queue lengths (ping-pong x yield point), trace work counter, ray-queue lengths
    unsigned *wf_host_ = nullptr;   // pinned: queue length read back every wf_check_ rounds
    uint64_t wf_rounds_ = 0;
    // film
    DBuf<double> film64_;
    DBuf<float4> film32_;
    // adaptation / partition
    size_t reg_cap_ = 0;
    int n_regions_host_ = 0;
    int n_nodes_host_ = 0;
    int n_trees_ = 0;
    DBuf<rd::KernTab<R>> ktab_;
    DBuf<double> lambda_, pend_sum_, tot_acc_;
    DBuf<unsigned long long> n_, pend_fx_, tot_vis_, tot_fx_, x_cnt_, x_fx_, x_last_, visits_;
    DBuf<unsigned> pend_n_, x_touched_, touched_list_, n_touched_;
    DBuf<rd::NodeD> nodes_;
    DBuf<int> roots_, n_nodes_, n_regions_, scratch_cnt_, scratch_list_, splits_;
    DBuf<int> rf_key_[2], rf_val_[2], rf_count_;   // parallel refine: sort keys / node ids
    DBuf<unsigned char> rf_tmp_;
    DBuf<unsigned long long> trace_count_, trace_index_, trace_n_;
    DBuf<long long> trace_region_;
    DBuf<double> trace_lambda_, trace_alpha_;
    DBuf<double> red_;
    // host state
    double b_ = 0.0, b_se_ = 0.0;
    uint64_t b_n_ = 0;
    bool b_set_ = false, chains_ready_ = false;
    uint64_t done_ = 0, next_refine_, next_metrics_;
    // run_steps: the open span of the canonical span loop (boundaries at the
    // configured total, refine and metrics barriers -- what run(d.mutations) uses)
    bool span_open_ = false;
    uint64_t sp_start_ = 0, sp_end_ = 0;
    unsigned long long sp_per_ = 0, sp_rem_ = 0;
    int sp_steps_ = 0, sp_j_ = 0;
    void span_boundary();
    std::vector<std::array<double, 6>> metrics_;   // time, at, rrmse, acceptance, accepted sum, proposals
    std::chrono::steady_clock::time_point t0_;
    bool t0_set_ = false;
    uint64_t launches_ = 0;
    uint64_t steps_since_fold_ = 0;
    ramlt_stats final_{};
    bool finalized_ = false;
    // live kernel timing (profile_kernels): event pairs around chain-step launches
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_, ev_trace_;
    double step_ms_ = 0.0, trace_ms_ = 0.0;
    uint64_t step_launches_ = 0, trace_launches_ = 0;
    void drain_events();
    // launch configuration cache: the dynamic-smem attribute is set and the
    // occupancy queried once per (kernel, smem) instead of on every launch
    // (per-step launches of small-chain runs are host-bound)
    struct LaunchCfg {
        const void *kern;
        size_t smem;
        int per_sm;
    };
    std::vector<LaunchCfg> lcfg_;
    int sms_ = 0;
    int prepare(const void *kern, size_t smem, int carveout = -1);
};

// ---------------------------------------------------------------------------------------
template <class R> static rd::V3<R> v3c(const double *p) {
    return rd::V3<R>{static_cast<R>(p[0]), static_cast<R>(p[1]), static_cast<R>(p[2])};
}

template <class R>
EngineT<R>::EngineT(const HostScene &scene, const ramlt_render_desc &d) : d_(d), hs_(scene) {
    if (d.chains < 1)
        throw std::logic_error("need at least one chain");
    if (d.width < 1 || d.height < 1)
        throw std::logic_error("resolution must be positive");
    if (d.max_vertices < 2)
        throw std::logic_error("max_vertices must be at least 2");
    if (d.max_vertices > rd::kMaxV)
        throw std::invalid_argument("max_vertices exceeds the engine's path capacity (" +
                                    std::to_string(rd::kMaxV) + ")");
    if (d.batch_size < 1)
        throw std::logic_error("batch_size must be >= 1");
    if (hs_.emit.size() / 3 >= 4095 || hs_.mats.size() >= 65535)
        throw std::invalid_argument("too many emitters or materials for the vertex encoding");
    if (d.device >= 0)
        RAMLT_CUDA(cudaSetDevice(d.device));
    RAMLT_CUDA(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));

    C_ = d.chains;
    Ctot_ = d.chains_total > 0 ? d.chains_total : d.chains;
    off_ = d.chain_offset;
    if (off_ < 0 || off_ + C_ > Ctot_)
        throw std::logic_error("chain shard outside [0, chains_total)");
    G_ = d.lanes_per_chain;
    if (G_ <= 0)
        G_ = C_ <= 8192 ? 32 : 1;
    if (G_ != 1 && G_ != 2 && G_ != 4 && G_ != 8 && G_ != 16 && G_ != 32)
        throw std::invalid_argument("lanes_per_chain must be a power of two <= 32");
    if (d.accel == RAMLT_ACCEL_BVH || (d.accel == RAMLT_ACCEL_AUTO && scene.tri.size() > 128))
        G_ = 1;   // BVH traversal is per thread (lanes_per_chain applies to the brute-force path)
    if (const char *v = std::getenv("RAMLT_ACCEL"))
        if (std::string(v) == "bvh")
            G_ = 1;
    ctl_ = d.strategy == RAMLT_FIXED ? 0 : (d.strategy == RAMLT_GLOBAL ? 1 : 2);
    pkind_ = 0;
    if (ctl_ == 2)
        pkind_ = d.strategy == RAMLT_RA_GRID ? (d.perturbation == RAMLT_LENS ? 1 : 3)
                                             : (d.perturbation == RAMLT_LENS ? 2 : 4);
    adapt_ = d.adapt_mode;
    if (adapt_ < 0)
        adapt_ = Ctot_ <= 4096 ? 0 : 1;
    if (Ctot_ != C_ && ctl_ != 0)
        adapt_ = 1;   // sharded adaptive runs use the pooled rule (G-invariant)
    next_refine_ = d.m_refine;
    next_metrics_ = d.metrics_interval;

    // camera (core/driver.cpp:181 -> camera.cpp:22-30)
    cb_ = make_camera(hs_.cam, d.width, d.height);

    // scene upload
    std::vector<rd::TriD<R>> tris(hs_.tri.size());
    for (size_t i = 0; i < hs_.tri.size(); ++i) {
        const ramlt_triangle &t = hs_.tri[i];
        double e1[3] = {t.b[0] - t.a[0], t.b[1] - t.a[1], t.b[2] - t.a[2]};
        double e2[3] = {t.c[0] - t.a[0], t.c[1] - t.a[1], t.c[2] - t.a[2]};
        double cr[3] = {e1[1] * e2[2] - e1[2] * e2[1], e1[2] * e2[0] - e1[0] * e2[2],
                        e1[0] * e2[1] - e1[1] * e2[0]};
        double l = std::sqrt(cr[0] * cr[0] + cr[1] * cr[1] + cr[2] * cr[2]);
        double n[3] = {cr[0] / l, cr[1] / l, cr[2] / l};
        tris[i].a = v3c<R>(t.a);
        tris[i].e1 = v3c<R>(e1);
        tris[i].e2 = v3c<R>(e2);
        tris[i].n = v3c<R>(n);
        tris[i].mat = t.material;
        tris[i].emi = t.emitter;
        tris[i].orig = static_cast<int>(i);
        tris[i].pad_ = 0;
    }
    // triangle accelerator: brute force from shared memory for small scenes,
    // SAH BVH2 from L2/HBM above 128 triangles (identical results, see bvh.h)
    {
        int accel = d.accel;
        if (const char *v = std::getenv("RAMLT_ACCEL"))
            accel = std::string(v) == "bvh" ? RAMLT_ACCEL_BVH : (std::string(v) == "brute" ? RAMLT_ACCEL_BRUTE : accel);
        use_bvh_ = !tris.empty() && (accel == RAMLT_ACCEL_BVH || (accel == RAMLT_ACCEL_AUTO && tris.size() > 128));
    }
    if (use_bvh_) {
        std::vector<double> coords(9 * hs_.tri.size());
        for (size_t i = 0; i < hs_.tri.size(); ++i) {
            std::memcpy(&coords[9 * i + 0], hs_.tri[i].a, 3 * sizeof(double));
            std::memcpy(&coords[9 * i + 3], hs_.tri[i].b, 3 * sizeof(double));
            std::memcpy(&coords[9 * i + 6], hs_.tri[i].c, 3 * sizeof(double));
        }
        // leaves of at most 2 triangles: c5 on the wavefront build 121.2 (4) / 124.4 (3) / 125.1 (2) /
        // 117.5 (6) M mutations/s (profiles/r03a): 66 vs 59 node visits but 13 vs 27 triangle tests per ray
        int leaf_max = 2;
        if (const char *v = std::getenv("RAMLT_BVH_LEAF"))
            leaf_max = std::max(1, std::min(15, std::atoi(v)));
        BvhBuild bb = build_bvh(coords.data(), hs_.tri.size(), leaf_max);
        bvh_depth_ = bb.depth;
        if (bb.depth > 62)
            throw std::runtime_error("BVH deeper than the traversal stack");
        std::vector<rd::TriD<R>> ordered(tris.size());
        for (size_t i = 0; i < tris.size(); ++i)
            ordered[i] = tris[static_cast<size_t>(bb.order[i])];
        tris.swap(ordered);
        std::vector<unsigned char> units = layout_bvh<R>(bb, tris);
        bvh_.alloc(units.size());
        RAMLT_CUDA(cudaMemcpy(bvh_.p, units.data(), units.size(), cudaMemcpyHostToDevice));
    }
    std::vector<rd::SphD<R>> sphs(hs_.sph.size());
    for (size_t i = 0; i < hs_.sph.size(); ++i) {
        sphs[i].c = v3c<R>(hs_.sph[i].center);
        sphs[i].r = static_cast<R>(hs_.sph[i].radius);
        sphs[i].mat = hs_.sph[i].material;
        sphs[i].emi = hs_.sph[i].emitter;
    }
    std::vector<rd::MatD<R>> mats(hs_.mats.size());
    for (size_t i = 0; i < hs_.mats.size(); ++i) {
        mats[i].kind = hs_.mats[i].kind;
        mats[i].albedo = v3c<R>(hs_.mats[i].albedo);
        mats[i].ior = static_cast<R>(hs_.mats[i].ior);
        mats[i].expo = static_cast<R>(hs_.mats[i].exponent);
    }
    std::vector<rd::V3<R>> emit(hs_.emit.size() / 3);
    for (size_t i = 0; i < emit.size(); ++i)
        emit[i] = v3c<R>(&hs_.emit[3 * i]);
    tri_.alloc(std::max<size_t>(tris.size(), 1));
    sph_.alloc(std::max<size_t>(sphs.size(), 1));
    mat_.alloc(std::max<size_t>(mats.size(), 1));
    emit_.alloc(std::max<size_t>(emit.size(), 1));
    if (!tris.empty())
        RAMLT_CUDA(cudaMemcpy(tri_.p, tris.data(), tris.size() * sizeof(tris[0]), cudaMemcpyHostToDevice));
    if (!sphs.empty())
        RAMLT_CUDA(cudaMemcpy(sph_.p, sphs.data(), sphs.size() * sizeof(sphs[0]), cudaMemcpyHostToDevice));
    if (!mats.empty())
        RAMLT_CUDA(cudaMemcpy(mat_.p, mats.data(), mats.size() * sizeof(mats[0]), cudaMemcpyHostToDevice));
    if (!emit.empty())
        RAMLT_CUDA(cudaMemcpy(emit_.p, emit.data(), emit.size() * sizeof(emit[0]), cudaMemcpyHostToDevice));
    smem_ = ((sphs.size() * sizeof(rd::SphD<R>) + 15) & ~size_t(15)) +
            (use_bvh_ ? 0 : tris.size() * sizeof(rd::TriD<R>));
    if (smem_ > 200 * 1024)
        throw std::invalid_argument("scene too large for the shared-memory primitive path (" +
                                    std::to_string(hs_.tri.size()) + " triangles)");

    // chain state
    size_t C = static_cast<size_t>(C_);
    verts_.alloc(C * static_cast<size_t>(d.max_vertices - 1));
    klen_.alloc(C);
    smask_.alloc(C);
    cf_.alloc(4 * C);
    cr_.alloc(2 * C);
    eyeden_.alloc(C);
    rng0_.alloc(C);
    rng1_.alloc(C);
    acc_.alloc(C);
    iacc_.alloc(C);
    lum_.alloc(C);
    npert_.alloc(C);
    nlarge_.alloc(C);
    ipert_.alloc(C);
    nsteps_.alloc(C);
    if (d.log_steps) {
        log_a_.alloc(C * d.log_steps);
        log_f_.alloc(C * d.log_steps);
        log_a_.zero(stream_);
        log_f_.zero(stream_);
    }
    vreg_.alloc(C);
    va_.alloc(C);
    err_.alloc(4);
    err_.zero(stream_);
    rays_.alloc(2);
    rays_.zero(stream_);
    work_.alloc(1);
    // BVH scenes step with the coroutine kernel (dynamic ray fetch), brute-force
    // scenes with the lane-group megakernel; RAMLT_STEP_KERNEL=mega|co|co_static overrides.
    use_co_ = use_bvh_;
    use_co_init_ = use_bvh_;
    use_wf_ = use_bvh_;
    if (const char *v = std::getenv("RAMLT_INIT_KERNEL")) {
        use_co_init_ = std::string(v) == "co" || std::string(v) == "wf";
        use_wf_init_ = std::string(v) == "wf";
    }
    if (const char *v = std::getenv("RAMLT_STEP_KERNEL")) {
        use_co_ = std::string(v) == "co" || std::string(v) == "co_static" || std::string(v) == "wf";
        steal_ = std::string(v) == "co_static" ? 0 : 1;
        use_wf_ = std::string(v) == "wf";   // brute-force scenes too (k_wf_trace_brute), G == 1
    }
    // ray records carry (chain, batch ordinal) in 27 + 5 bits
    if (static_cast<unsigned long long>(C_) >= (1ull << rd::kWfChainBits) || d.max_vertices > 32)
        use_wf_ = false;
    // Chain initialisation stays with the fused kernel by default: nearly every attempt of a
    // chain fails (c4/c5: ~37 attempts of ~11 rays before a path reaches a light), so as
    // wavefront rounds every chain's state makes thousands of HBM round trips -- c5 init
    // 7.4 s (wf) vs 4.5 s (co), c4 1.86 s vs 0.75 s (profiles/r02t); 5.7 s vs 4.5 s with the compact
    // image and k_wf_bounce<INIT> (profiles/r02z: the ~7,000 nearly empty rounds of the unluckiest
    // chains).  RAMLT_INIT_KERNEL=wf keeps the wavefront form for the parity tests.
    if (static_cast<unsigned long long>(C_) >= (1ull << rd::kWfChainBits) || d.max_vertices > 32)
        use_wf_init_ = false;
    if (const char *v = std::getenv("RAMLT_WF_REFILL"))
        wf_refill_ = std::min(32, std::max(1, std::atoi(v)));
    if (const char *v = std::getenv("RAMLT_WF_LOG"))
        wf_log_ = std::string(v) == "1";
    if (const char *v = std::getenv("RAMLT_WF_BOUNCE"))
        wf_bounce_ = std::string(v) == "1";
    if (const char *v = std::getenv("RAMLT_WF_PIPES"))
        wf_pipes_ = std::min(2, std::max(1, std::atoi(v)));
    if (const char *v = std::getenv("RAMLT_WF_PIPES_MIN"))
        wf_pipes_min_ = static_cast<size_t>(std::max(256, std::atoi(v)));
    if (const char *v = std::getenv("RAMLT_WF_LBLK"))
        wf_lblk_ = std::min(8, std::max(0, std::atoi(v)));
    if (const char *v = std::getenv("RAMLT_WF_TBLK"))
        wf_tblk_ = std::min(16, std::max(0, std::atoi(v)));
    if (wf_pipes_ > 1) {
        RAMLT_CUDA(cudaStreamCreateWithFlags(&wf_stream2_, cudaStreamNonBlocking));
        for (cudaEvent_t &e : wf_ev_)
            RAMLT_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    if (const char *v = std::getenv("RAMLT_WF_POLL"))
        wf_poll_ = std::string(v) == "1";
    if (const char *v = std::getenv("RAMLT_WF_CHECK"))
        wf_check_ = std::min(64, std::max(1, std::atoi(v)));
    if (const char *v = std::getenv("RAMLT_CO_PV"))
        co_pv_global_ = std::string(v) != "smem";
    if (const char *v = std::getenv("RAMLT_CO_CARVEOUT"))
        co_carveout_ = std::min(100, std::max(0, std::atoi(v)));
    if (const char *v = std::getenv("RAMLT_CO_REFILL"))
        refill_ = std::min(32, std::max(1, std::atoi(v)));
    if (const char *v = std::getenv("RAMLT_CO_INIT_REFILL"))
        init_refill_ = std::min(32, std::max(1, std::atoi(v)));
    size_t npix = static_cast<size_t>(d.width) * d.height;
    film64_.alloc(npix * 3);
    film64_.zero(stream_);
    if (sizeof(R) == 4) {
        film32_.alloc(npix);
        film32_.zero(stream_);
    }
    red_.alloc(6 * ((C + 255) / 256));

    // controller + partition (core/driver.cpp:190-212)
    size_t initial = 1;
    if (pkind_ == 1)
        initial = static_cast<size_t>(d.n_top) * d.n_top;
    else if (pkind_ == 3)
        initial = static_cast<size_t>(d.n_top) * d.n_top * d.n_bottom * d.n_bottom;
    else if (pkind_ == 4)
        initial = static_cast<size_t>(d.n_top) * d.n_top;
    size_t cap = initial;
    if (pkind_ == 2 || pkind_ == 4) {
        // Every split consumes >= m_split visits, so the run can create at most
        // 4 * mutations / m_split regions: reserve that up front (bounded) so
        // the quadtree never reallocates (a device-wide sync) inside the span loop.
        size_t bound = initial + 4 * static_cast<size_t>(d.mutations / std::max<uint64_t>(d.m_split, 1)) + 64;
        size_t autocap = std::max<size_t>(4096, std::min<size_t>(bound, size_t(1) << 24));
        cap = std::max<size_t>(d.region_capacity ? d.region_capacity : autocap, initial * 8);
    }
    alloc_regions(cap);
    n_regions_host_ = static_cast<int>(initial);
    {
        std::vector<double> lam(initial, d.lambda_init);
        std::vector<unsigned long long> one(initial, 1ull);
        RAMLT_CUDA(cudaMemcpy(lambda_.p, lam.data(), initial * sizeof(double), cudaMemcpyHostToDevice));
        RAMLT_CUDA(cudaMemcpy(n_.p, one.data(), initial * sizeof(unsigned long long), cudaMemcpyHostToDevice));
        rd::k_ktab_init<R><<<static_cast<unsigned>((initial + 255) / 256), 256, 0, stream_>>>(
            ktab_.p, lambda_.p, static_cast<int>(initial), d.sigma2_ratio);
        ++launches_;
        RAMLT_CUDA(cudaGetLastError());
    }
    if (pkind_ == 2 || pkind_ == 4) {
        n_trees_ = pkind_ == 2 ? 1 : d.n_top * d.n_top;
        std::vector<rd::NodeD> nodes(n_trees_);
        std::vector<int> roots(n_trees_);
        for (int t = 0; t < n_trees_; ++t) {
            nodes[t] = rd::NodeD{0, 0, 0, -1, t, t};
            roots[t] = t;
        }
        RAMLT_CUDA(cudaMemcpy(nodes_.p, nodes.data(), nodes.size() * sizeof(rd::NodeD), cudaMemcpyHostToDevice));
        roots_.alloc(n_trees_);
        RAMLT_CUDA(cudaMemcpy(roots_.p, roots.data(), roots.size() * sizeof(int), cudaMemcpyHostToDevice));
        n_nodes_host_ = n_trees_;
        n_nodes_.alloc(1);
        n_regions_.alloc(1);
        RAMLT_CUDA(cudaMemcpy(n_nodes_.p, &n_nodes_host_, sizeof(int), cudaMemcpyHostToDevice));
        RAMLT_CUDA(cudaMemcpy(n_regions_.p, &n_regions_host_, sizeof(int), cudaMemcpyHostToDevice));
        scratch_cnt_.alloc(n_trees_);
        splits_.alloc(1);
    }
    size_t tcap = d.trace_enabled ? (d.trace_capacity ? d.trace_capacity : (1u << 20)) : 0;
    trace_count_.alloc(1);
    trace_count_.zero(stream_);
    if (tcap) {
        trace_index_.alloc(tcap);
        trace_n_.alloc(tcap);
        trace_region_.alloc(tcap);
        trace_lambda_.alloc(tcap);
        trace_alpha_.alloc(tcap);
    }
    RAMLT_CUDA(cudaStreamSynchronize(stream_));
}

template <class R> int EngineT<R>::prepare(const void *kern, size_t smem, int carveout) {
    for (const LaunchCfg &c : lcfg_)
        if (c.kern == kern && c.smem == smem)
            return c.per_sm;
    RAMLT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    if (carveout >= 0)   // RAMLT_CO_CARVEOUT: shared-memory share of the L1/smem pool (percent)
        RAMLT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, carveout));
    int per_sm = 0;
    RAMLT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 128, smem));
    if (!sms_) {
        int dev = 0;
        RAMLT_CUDA(cudaGetDevice(&dev));
        RAMLT_CUDA(cudaDeviceGetAttribute(&sms_, cudaDevAttrMultiProcessorCount, dev));
    }
    lcfg_.push_back({kern, smem, per_sm});
    return per_sm;
}

template <class R> void EngineT<R>::drain_events() {
    for (auto &e : ev_) {
        RAMLT_CUDA(cudaEventSynchronize(e.second));
        float ms = 0.f;
        RAMLT_CUDA(cudaEventElapsedTime(&ms, e.first, e.second));
        step_ms_ += ms;
        ++step_launches_;
        cudaEventDestroy(e.first);
        cudaEventDestroy(e.second);
    }
    ev_.clear();
    for (auto &e : ev_trace_) {
        RAMLT_CUDA(cudaEventSynchronize(e.second));
        float ms = 0.f;
        RAMLT_CUDA(cudaEventElapsedTime(&ms, e.first, e.second));
        trace_ms_ += ms;
        ++trace_launches_;
        cudaEventDestroy(e.first);
        cudaEventDestroy(e.second);
    }
    ev_trace_.clear();
}

template <class R> EngineT<R>::~EngineT() {
    if (wf_host_)
        cudaFreeHost(wf_host_);
    if (wf_stream2_)
        cudaStreamDestroy(wf_stream2_);
    for (cudaEvent_t e : wf_ev_)
        if (e)
            cudaEventDestroy(e);
    for (auto &e : ev_trace_) {
        cudaEventDestroy(e.first);
        cudaEventDestroy(e.second);
    }
    for (auto &e : ev_) {
        cudaEventDestroy(e.first);
        cudaEventDestroy(e.second);
    }
    if (stream_ && own_stream_) {
        cudaStreamSynchronize(stream_);
        cudaStreamDestroy(stream_);
    }
}

template <class R> void EngineT<R>::alloc_regions(size_t cap) {
    reg_cap_ = cap;
    ktab_.alloc(cap);
    lambda_.alloc(cap);
    pend_sum_.alloc(cap);
    tot_acc_.alloc(cap);
    n_.alloc(cap);
    pend_fx_.alloc(cap);
    tot_vis_.alloc(cap);
    tot_fx_.alloc(cap);
    x_cnt_.alloc(cap);
    x_fx_.alloc(cap);
    x_last_.alloc(cap);
    visits_.alloc(cap);
    pend_n_.alloc(cap);
    x_touched_.alloc(cap);
    touched_list_.alloc(cap);
    n_touched_.alloc(1);
    for (auto *b : {&pend_sum_, &tot_acc_})
        b->zero(stream_);
    for (auto *b : {&pend_fx_, &tot_vis_, &tot_fx_, &x_cnt_, &x_fx_, &x_last_, &visits_})
        b->zero(stream_);
    pend_n_.zero(stream_);
    x_touched_.zero(stream_);
    n_touched_.zero(stream_);
    if (pkind_ == 2 || pkind_ == 4) {
        nodes_.alloc(cap + 4);
        scratch_list_.alloc(cap + 4);
    }
}

template <class T> static void grow_buf(DBuf<T> &b, size_t cap, size_t used, cudaStream_t s) {
    DBuf<T> nb;
    nb.alloc(cap);
    nb.zero(s);
    if (used)
        RAMLT_CUDA(cudaMemcpyAsync(nb.p, b.p, used * sizeof(T), cudaMemcpyDeviceToDevice, s));
    RAMLT_CUDA(cudaStreamSynchronize(s));
    b.free();
    b.p = nb.p;
    b.n = nb.n;
    nb.p = nullptr;
    nb.n = 0;
}

template <class R> void EngineT<R>::grow_regions(size_t cap) {
    size_t used = static_cast<size_t>(n_regions_host_);
    grow_buf(ktab_, cap, used, stream_);
    grow_buf(lambda_, cap, used, stream_);
    grow_buf(pend_sum_, cap, used, stream_);
    grow_buf(tot_acc_, cap, used, stream_);
    grow_buf(n_, cap, used, stream_);
    grow_buf(pend_fx_, cap, used, stream_);
    grow_buf(tot_vis_, cap, used, stream_);
    grow_buf(tot_fx_, cap, used, stream_);
    grow_buf(x_cnt_, cap, used, stream_);
    grow_buf(x_fx_, cap, used, stream_);
    grow_buf(x_last_, cap, used, stream_);
    grow_buf(visits_, cap, used, stream_);
    grow_buf(pend_n_, cap, used, stream_);
    grow_buf(x_touched_, cap, used, stream_);
    grow_buf(touched_list_, cap, 0, stream_);
    grow_buf(nodes_, cap + 4, static_cast<size_t>(n_nodes_host_), stream_);
    grow_buf(scratch_list_, cap + 4, 0, stream_);
    reg_cap_ = cap;
}

template <class R> rd::StepParams<R> EngineT<R>::params() const {
    rd::StepParams<R> P{};
    P.scene.tri = tri_.p;
    P.scene.sph = sph_.p;
    P.scene.mat = mat_.p;
    P.scene.emit = emit_.p;
    P.scene.ntri = static_cast<int>(hs_.tri.size());
    P.scene.nsph = static_cast<int>(hs_.sph.size());
    P.scene.cam.pos = v3c<R>(cb_.pos);
    P.scene.cam.right = v3c<R>(cb_.right);
    P.scene.cam.up = v3c<R>(cb_.up);
    P.scene.cam.fwd = v3c<R>(cb_.fwd);
    P.scene.cam.tanh = static_cast<R>(cb_.tanh);
    P.scene.cam.aspect = static_cast<R>(cb_.aspect);
    P.scene.cam.area = static_cast<R>(cb_.area);
    P.scene.cam.sensor = static_cast<R>(cb_.sensor);
    P.scene.bvh = use_bvh_ ? bvh_.p : nullptr;
    P.C = C_;
    P.C_total = Ctot_;
    P.chain_off = off_;
    P.maxv = d_.max_vertices;
    P.pk = d_.perturbation;
    P.ctl = ctl_;
    P.W = d_.width;
    P.H = d_.height;
    P.seed = d_.seed;
    P.ch.verts = verts_.p;
    P.ch.klen = klen_.p;
    P.ch.smask = smask_.p;
    P.ch.cf = cf_.p;
    P.ch.cr = cr_.p;
    P.ch.eyeden = eyeden_.p;
    P.ch.rng0 = rng0_.p;
    P.ch.rng1 = rng1_.p;
    P.ch.acc = acc_.p;
    P.ch.iacc = iacc_.p;
    P.ch.lum = lum_.p;
    P.ch.npert = npert_.p;
    P.ch.nlarge = nlarge_.p;
    P.ch.ipert = ipert_.p;
    P.ch.nsteps = nsteps_.p;
    P.ch.log_a = log_a_.p;
    P.ch.log_f = log_f_.p;
    P.ch.log_K = d_.log_steps;
    P.ch.vreg = vreg_.p;
    P.ch.va = va_.p;
    P.ch.err = err_.p;
    P.ch.rays = rays_.p;
    P.part.kind = pkind_;
    P.part.ntop = d_.n_top;
    P.part.nbot = d_.n_bottom;
    P.part.nodes = nodes_.p;
    P.part.roots = roots_.p;
    P.part.visits = visits_.p;
    P.ktab = ktab_.p;
    P.film64 = film64_.p;
    P.film32 = film32_.p;
    P.reg = regions();
    return P;
}

template <class R> rd::RegionArrays EngineT<R>::regions() const {
    rd::RegionArrays ra;
    ra.lambda = lambda_.p;
    ra.n = n_.p;
    ra.pend_n = pend_n_.p;
    ra.pend_sum = pend_sum_.p;
    ra.pend_fx = pend_fx_.p;
    ra.tot_vis = tot_vis_.p;
    ra.tot_acc = tot_acc_.p;
    ra.tot_fx = tot_fx_.p;
    ra.x_cnt = x_cnt_.p;
    ra.x_fx = x_fx_.p;
    ra.x_last = x_last_.p;
    ra.x_touched = x_touched_.p;
    ra.touched_list = touched_list_.p;
    ra.n_touched = n_touched_.p;
    return ra;
}

template <class R> rd::TraceBuf EngineT<R>::tracebuf() const {
    rd::TraceBuf t;
    t.count = trace_count_.p;
    t.cap = trace_index_.n;
    t.index = trace_index_.p;
    t.region = trace_region_.p;
    t.n = trace_n_.p;
    t.lambda = trace_lambda_.p;
    t.alpha = trace_alpha_.p;
    return t;
}

template <class R> rd::AdaptCfg EngineT<R>::adaptcfg() const {
    rd::AdaptCfg a;
    a.L = d_.batch_size;
    a.gmax = d_.gamma_max;
    a.gscale = d_.gamma_scale;
    a.target = d_.target_acceptance;
    a.lmin = d_.lambda_min;
    a.ratio = d_.sigma2_ratio;
    a.trace = d_.trace_enabled && trace_index_.n > 0;
    return a;
}

template <class R> void EngineT<R>::check_err(const char *what) {
    int e[4];
    RAMLT_CUDA(cudaMemcpyAsync(e, err_.p, sizeof(e), cudaMemcpyDeviceToHost, stream_));
    RAMLT_CUDA(cudaStreamSynchronize(stream_));
    if (e[0] == 1)
        throw std::runtime_error("black-scene: could not find an initial path");
    if (e[0] == 2)
        throw std::runtime_error(std::string("region capacity exceeded in ") + what);
}

template <class R> void EngineT<R>::estimate_b_partials(uint64_t begin, uint64_t end, double *out) {
    if (d_.b_samples < 1)
        throw std::logic_error("estimate_b needs at least one sample");
    uint64_t S = std::min<uint64_t>(d_.b_samples, d_.b_substreams ? d_.b_substreams : 65536);
    if (end > S || begin > end)
        throw std::logic_error("substream range outside [0, b_substreams)");
    DBuf<double> part;
    part.alloc(2 * std::max<uint64_t>(end - begin, 1));
    rd::StepParams<R> P = params();
    unsigned blocks = static_cast<unsigned>((end - begin + 127) / 128);
    if (end > begin) {
        auto kern = d_.rng == RAMLT_RNG_PHILOX
                        ? (use_bvh_ ? rd::k_bsub<R, rd::RNG_PHILOX, 0> : rd::k_bsub<R, rd::RNG_PHILOX, 1>)
                        : (use_bvh_ ? rd::k_bsub<R, rd::RNG_PCG, 0> : rd::k_bsub<R, rd::RNG_PCG, 1>);
        RAMLT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem_)));
        kern<<<blocks, 128, smem_, stream_>>>(P, d_.b_samples, S, begin, end, part.p);
        ++launches_;
        RAMLT_CUDA(cudaGetLastError());
        RAMLT_CUDA(cudaMemcpyAsync(out, part.p, 2 * (end - begin) * sizeof(double), cudaMemcpyDeviceToHost, stream_));
    }
    RAMLT_CUDA(cudaStreamSynchronize(stream_));
}

template <class R> void EngineT<R>::reduce_b(const double *partials, uint64_t n, double *b, double *se) {
    // fixed substream order (oracle/ramlt_oracle.cpp mirrors it)
    double sum = 0.0, sq = 0.0;
    for (uint64_t s = 0; s < n; ++s) {
        sum += partials[2 * s];
        sq += partials[2 * s + 1];
    }
    double nn = static_cast<double>(d_.b_samples);
    double mean = sum / nn;
    if (mean <= 0.0)
        throw std::runtime_error("black-scene: no sample carried any contribution");
    double var = d_.b_samples > 1 ? std::max(0.0, (sq - nn * mean * mean) / (nn - 1.0)) : 0.0;
    b_ = mean;
    b_se_ = std::sqrt(var / nn);
    b_n_ = d_.b_samples;
    b_set_ = true;
    if (b)
        *b = b_;
    if (se)
        *se = b_se_;
}

template <class R> void EngineT<R>::estimate_b(double *b, double *se) {
    uint64_t S = std::min<uint64_t>(d_.b_samples, d_.b_substreams ? d_.b_substreams : 65536);
    std::vector<double> part(2 * S);
    estimate_b_partials(0, S, part.data());
    reduce_b(part.data(), S, b, se);
}

template <class R> void EngineT<R>::init_chains() {
    rd::StepParams<R> P = params();
    if (use_co_init_) {   // BVH scenes: the coroutine, as wavefront rounds or the fused kernel
        P.steal = 1;
        P.refill = init_refill_;
        P.init_attempts = 50000000ull;
        if (use_wf_init_) {
            P.refill = wf_refill_;
            P.j0 = 0;
            P.j1 = 1;
            if (d_.rng == RAMLT_RNG_PHILOX)
                launch_step_wf<rd::RNG_PHILOX, true>(P);
            else
                launch_step_wf<rd::RNG_PCG, true>(P);
        } else {
            launch_step_co<true>(P);
        }
        check_err("init");
        chains_ready_ = true;
        return;
    }
    auto kern = d_.rng == RAMLT_RNG_PHILOX
                    ? (use_bvh_ ? rd::k_init<R, rd::RNG_PHILOX, 0> : rd::k_init<R, rd::RNG_PHILOX, 1>)
                    : (use_bvh_ ? rd::k_init<R, rd::RNG_PCG, 0> : rd::k_init<R, rd::RNG_PCG, 1>);
    RAMLT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem_)));
    int per_sm = 0, dev = 0, sms = 148;
    RAMLT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 128, smem_));
    RAMLT_CUDA(cudaGetDevice(&dev));
    RAMLT_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    unsigned blocks = std::min<unsigned>(static_cast<unsigned>((C_ + 127) / 128),
                                         static_cast<unsigned>(std::max(per_sm, 1) * sms));
    RAMLT_CUDA(cudaMemsetAsync(work_.p, 0, sizeof(unsigned), stream_));
    kern<<<blocks, 128, smem_, stream_>>>(P, 50000000ull, work_.p);
    ++launches_;
    RAMLT_CUDA(cudaGetLastError());
    check_err("init");
    chains_ready_ = true;
}

template <class R> void EngineT<R>::trace_benchmark(uint64_t n_rays, double *ms, uint64_t *hits) {
    if (!use_bvh_)
        throw std::logic_error("trace_benchmark needs the BVH accelerator (accel=bvh or > 128 triangles)");
    if (n_rays >= 0xffffffffull)
        throw std::invalid_argument("trace_benchmark: n_rays must fit 32 bits");
    // scene bounds from the triangles, shrunk by 10 % on every side
    double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
    for (const ramlt_triangle &t : hs_.tri)
        for (const double *v : {t.a, t.b, t.c})
            for (int k = 0; k < 3; ++k) {
                lo[k] = std::min(lo[k], v[k]);
                hi[k] = std::max(hi[k], v[k]);
            }
    rd::V3<R> l, e;
    l.x = static_cast<R>(lo[0] + 0.1 * (hi[0] - lo[0]));
    l.y = static_cast<R>(lo[1] + 0.1 * (hi[1] - lo[1]));
    l.z = static_cast<R>(lo[2] + 0.1 * (hi[2] - lo[2]));
    e.x = static_cast<R>(0.8 * (hi[0] - lo[0]));
    e.y = static_cast<R>(0.8 * (hi[1] - lo[1]));
    e.z = static_cast<R>(0.8 * (hi[2] - lo[2]));
    rd::StepParams<R> P = params();
    P.refill = refill_;
    size_t smem = (smem_ + 15) & ~size_t(15);
    P.co_stack_off = static_cast<unsigned>(smem);
    smem += static_cast<size_t>(128) * rd::BvhTrav<R>::SSTACK * sizeof(int);
    int cells = 0;   // RAMLT_TB_CELLS=n: rays in (origin cell of an n^3 grid, direction octant) order
    if (const char *v = std::getenv("RAMLT_TB_CELLS"))
        cells = std::max(0, std::atoi(v));
    auto kern = rd::k_trace_bench<R>;
    RAMLT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    int per_sm = 0, dev = 0, sms = 148;
    RAMLT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 128, smem));
    RAMLT_CUDA(cudaGetDevice(&dev));
    RAMLT_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    DBuf<unsigned long long> h;
    h.alloc(1);
    h.zero(stream_);
    RAMLT_CUDA(cudaMemsetAsync(work_.p, 0, sizeof(unsigned), stream_));
    cudaEvent_t e0, e1;
    RAMLT_CUDA(cudaEventCreate(&e0));
    RAMLT_CUDA(cudaEventCreate(&e1));
    RAMLT_CUDA(cudaEventRecord(e0, stream_));
    kern<<<static_cast<unsigned>(std::max(per_sm, 1) * sms), 128, smem, stream_>>>(P, n_rays, work_.p, h.p, l, e, cells);
    RAMLT_CUDA(cudaGetLastError());
    RAMLT_CUDA(cudaEventRecord(e1, stream_));
    RAMLT_CUDA(cudaEventSynchronize(e1));
    float t = 0.f;
    RAMLT_CUDA(cudaEventElapsedTime(&t, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    ++launches_;
    *ms = t;
    unsigned long long hh = 0;
    RAMLT_CUDA(cudaMemcpy(&hh, h.p, sizeof(hh), cudaMemcpyDeviceToHost));
    *hits = hh;
}

template <class R>
void EngineT<R>::launch_step(int j0, int j1, unsigned long long span_start, unsigned long long per,
                             unsigned long long rem, bool record) {
    rd::StepParams<R> P = params();
    P.span_start = span_start;
    P.per = per;
    P.rem = rem;
    P.j0 = j0;
    P.j1 = j1;
    P.record_visits = record ? 1 : 0;
    if (G_ == 1 && use_co_) {
        P.steal = steal_;
        P.refill = refill_;
        if (use_wf_) {
            P.refill = wf_refill_;
            if (d_.rng == RAMLT_RNG_PHILOX)
                launch_step_wf<rd::RNG_PHILOX>(P);
            else
                launch_step_wf<rd::RNG_PCG>(P);
        } else {
            launch_step_co(P);
        }
        return;
    }
    const long long threads = static_cast<long long>(C_) * G_;
    const unsigned blocks = static_cast<unsigned>((threads + 127) / 128);
    void (*kern)(rd::StepParams<R>) = nullptr;
#define RAMLT_PICK(RK)                                                                              \
    switch (use_bvh_ ? 0 : G_) {                                                                    \
    case 0: kern = rd::k_step<R, RK, 0>; break;                                                     \
    case 1: kern = rd::k_step<R, RK, 1>; break;                                                     \
    case 2: kern = rd::k_step<R, RK, 2>; break;                                                     \
    case 4: kern = rd::k_step<R, RK, 4>; break;                                                     \
    case 8: kern = rd::k_step<R, RK, 8>; break;                                                     \
    case 16: kern = rd::k_step<R, RK, 16>; break;                                                   \
    default: kern = rd::k_step<R, RK, 32>; break;                                                   \
    }
    if (d_.rng == RAMLT_RNG_PHILOX) {
        RAMLT_PICK(rd::RNG_PHILOX)
    } else {
        RAMLT_PICK(rd::RNG_PCG)
    }
#undef RAMLT_PICK
    prepare(reinterpret_cast<const void *>(kern), smem_);
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (d_.profile_kernels) {
        if (ev_.size() + ev_trace_.size() >= 4096)
            drain_events();
        RAMLT_CUDA(cudaEventCreate(&e0));
        RAMLT_CUDA(cudaEventCreate(&e1));
        RAMLT_CUDA(cudaEventRecord(e0, stream_));
    }
    kern<<<blocks, 128, smem_, stream_>>>(P);
    ++launches_;
    RAMLT_CUDA(cudaGetLastError());
    if (d_.profile_kernels) {
        RAMLT_CUDA(cudaEventRecord(e1, stream_));
        ev_.emplace_back(e0, e1);
    }
}

template <class R>
template <bool INIT>
void EngineT<R>::launch_step_co(const rd::StepParams<R> &P0) {
    rd::StepParams<R> P = P0;
    auto kern = d_.rng == RAMLT_RNG_PHILOX
                    ? (use_bvh_ ? rd::k_step_co<R, rd::RNG_PHILOX, true, INIT>
                                : rd::k_step_co<R, rd::RNG_PHILOX, false, INIT>)
                    : (use_bvh_ ? rd::k_step_co<R, rd::RNG_PCG, true, INIT> : rd::k_step_co<R, rd::RNG_PCG, false, INIT>);
    size_t scene = (smem_ + 15) & ~size_t(15);
    size_t smem = scene + (co_pv_global_ ? 0 : static_cast<size_t>(128) * d_.max_vertices * sizeof(rd::GV<R>));
    P.co_stack_off = static_cast<unsigned>(smem);
    if (use_bvh_)
        smem += static_cast<size_t>(128) * rd::BvhTrav<R>::SSTACK * sizeof(int);
    const int per_sm = prepare(reinterpret_cast<const void *>(kern), smem, co_carveout_);
    const int sms = sms_;
    unsigned want = static_cast<unsigned>((C_ + 127) / 128);
    unsigned blocks = P.steal ? std::min<unsigned>(want, static_cast<unsigned>(std::max(per_sm, 1) * sms)) : want;
    P.pv_scratch = nullptr;
    if (co_pv_global_) {
        size_t need = static_cast<size_t>(blocks) * 128 * d_.max_vertices;
        if (pv_scratch_.n < need)
            pv_scratch_.alloc(need);
        P.pv_scratch = pv_scratch_.p;
    }
    RAMLT_CUDA(cudaMemsetAsync(work_.p, 0, sizeof(unsigned), stream_));
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (d_.profile_kernels && !INIT) {
        if (ev_.size() + ev_trace_.size() >= 4096)
            drain_events();
        RAMLT_CUDA(cudaEventCreate(&e0));
        RAMLT_CUDA(cudaEventCreate(&e1));
        RAMLT_CUDA(cudaEventRecord(e0, stream_));
    }
    kern<<<blocks, 128, smem, stream_>>>(P, work_.p);
    ++launches_;
    RAMLT_CUDA(cudaGetLastError());
    if (d_.profile_kernels && !INIT) {
        RAMLT_CUDA(cudaEventRecord(e1, stream_));
        ev_.emplace_back(e0, e1);
    }
}

// Wavefront lockstep step (ramlt_wavefront.cuh): k_wf_logic / k_wf_trace rounds
// until no chain has a ray pending.  The queue length is read back every
// wf_check_ rounds; the rounds launched past the last ray find empty queues
// and exit at once.
template <class R>
template <int RK, bool INIT>
void EngineT<R>::launch_step_wf(rd::StepParams<R> P) {
    const size_t C = static_cast<size_t>(C_);
    constexpr int K = rd::Chunks<rd::WfState<R, RK, INIT>>::K;
    const size_t per_chain = static_cast<size_t>(std::max<int>(1, static_cast<int>(d_.max_vertices) - 1));
    if (wf_state_.n < K * C) {
        wf_state_.alloc(K * C);
        wf_pv_.alloc(static_cast<size_t>(d_.max_vertices) * C);
        wf_rays_.alloc(C * per_chain);
        wf_hits_.alloc(C);
        wf_occ_.alloc(C);
        for (int q = 0; q < 2; ++q)
            wf_cq_[q].alloc(rd::kWfQueues * C);
        wf_cnt_.alloc(32);
        if (!wf_host_)
            RAMLT_CUDA(cudaMallocHost(&wf_host_, rd::kWfQueues * sizeof(unsigned)));
    }
    auto logic = rd::k_wf_logic<R, RK, INIT>;
    auto trace = rd::k_wf_trace<R>;
    auto trace_brute = rd::k_wf_trace_brute<R>;
    size_t lsmem = smem_;
    size_t tsmem = (smem_ + 31) & ~size_t(31);   // the coroutine states are moved as 32 B sectors
    rd::StepParams<R> PL = P;   // k_wf_logic's parameters: co_stack_off = its shared-memory coroutine states
#if RAMLT_WF_SMEM
    PL.co_stack_off = static_cast<unsigned>(tsmem);
    lsmem = tsmem + static_cast<size_t>(128) * sizeof(rd::WfState<R, RK, INIT>);
#endif
    P.co_stack_off = static_cast<unsigned>(tsmem);
    tsmem += static_cast<size_t>(128) * rd::BvhTrav<R>::SSTACK * sizeof(int);
    const int lper = prepare(reinterpret_cast<const void *>(logic), lsmem);
    const int tper = use_bvh_ ? prepare(reinterpret_cast<const void *>(trace), tsmem)
                              : prepare(reinterpret_cast<const void *>(trace_brute), tsmem);
    // chain initialisation runs until every chain found a contributing path: polled
    const bool poll = INIT || P.j1 - P.j0 > 1 || wf_poll_;
    // default (RAMLT_WF_BOUNCE=0 turns it off): the bounce queue is resumed by k_wf_bounce (one more round: the
    // chains it takes out of the loop pass through the post-loop queue)
    const bool bounce_sep = wf_bounce_ && rd::WfCompact<R, RK, INIT>::OK;
    const int planned = poll ? 0 : static_cast<int>(d_.max_vertices) + 2 + (bounce_sep ? 1 : 0);
    // Pipelines: the chains of a one-step launch are cut into wf_pipes_ contiguous ranges,
    // each with its own queues and counters, and the ranges' rounds are enqueued on
    // separate streams.  k_wf_trace is bound by instruction issue and k_wf_logic by
    // memory latency, so a range in its trace kernel and another in its logic kernel
    // share the SMs instead of taking turns; the second range starts one logic kernel
    // late so that the two stay out of phase.  Each range's kernels get 1 / wf_pipes_
    // of the resident blocks.  Results do not depend on the split (per-chain state;
    // pooled adaptation and the film are order-independent sums / atomics).
    const int npipe = (!poll && !wf_log_ && wf_pipes_ > 1 && C >= wf_pipes_min_) ? 2 : 1;
    constexpr int NQ = rd::kWfQueues;
    struct Pipe {
        size_t c0, cn;
        cudaStream_t st;
        unsigned *cnt;   // chain-queue lengths [0..3] / [4..7] (ping-pong, one per yield point), trace
                         // work counter [8], ray-queue lengths [9] / [10]
        unsigned lblocks, tblocks, bblocks;
    } pipe[2];
    const size_t bsmem = (smem_ + 31) & ~size_t(31);
    int bper = 1;
    if (bounce_sep)
        bper = prepare(reinterpret_cast<const void *>(rd::k_wf_bounce<R, RK, INIT>), bsmem);
    for (int p = 0; p < npipe; ++p) {
        Pipe &pp = pipe[p];
        pp.c0 = npipe == 1 ? 0 : (p == 0 ? 0 : ((C / 2 + 127) & ~size_t(127)));
        pp.cn = npipe == 1 ? C : (p == 0 ? ((C / 2 + 127) & ~size_t(127)) : C - ((C / 2 + 127) & ~size_t(127)));
        pp.st = p == 0 ? stream_ : wf_stream2_;
        pp.cnt = wf_cnt_.p + 16 * p;
        const int lb = npipe == 1 ? std::max(lper, 1) : std::max(1, wf_lblk_ > 0 ? wf_lblk_ : lper / 2);
        const int tb = npipe == 1 ? std::max(tper, 1) : std::max(1, wf_tblk_ > 0 ? wf_tblk_ : tper / 2);
        pp.lblocks = std::min<unsigned>(static_cast<unsigned>((pp.cn + 127) / 128), static_cast<unsigned>(lb * sms_));
        pp.tblocks = static_cast<unsigned>(tb * sms_);
        pp.bblocks = std::min<unsigned>(static_cast<unsigned>((pp.cn + 127) / 128),
                                        static_cast<unsigned>(std::max(1, npipe == 1 ? bper : bper / 2) * sms_));
    }
    RAMLT_CUDA(cudaMemsetAsync(wf_cnt_.p, 0, 32 * sizeof(unsigned), stream_));
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    const bool prof = d_.profile_kernels && !INIT;
    if (prof) {
        if (ev_.size() + ev_trace_.size() >= 4096)
            drain_events();
        RAMLT_CUDA(cudaEventCreate(&e0));
        RAMLT_CUDA(cudaEventCreate(&e1));
        RAMLT_CUDA(cudaEventRecord(e0, stream_));
    }
    auto fork = [&] {
        if (npipe > 1) {
            RAMLT_CUDA(cudaEventRecord(wf_ev_[0], stream_));
            RAMLT_CUDA(cudaStreamWaitEvent(wf_stream2_, wf_ev_[0], 0));
        }
    };
    auto join = [&] {
        if (npipe > 1) {
            RAMLT_CUDA(cudaEventRecord(wf_ev_[1], wf_stream2_));
            RAMLT_CUDA(cudaStreamWaitEvent(stream_, wf_ev_[1], 0));
        }
    };
    fork();
    for (int r = 0;; ++r) {
        const int a = r & 1;
        for (int p = 0; p < npipe; ++p) {
            const Pipe &pp = pipe[p];
            unsigned *cnt = pp.cnt;
            rd::WfParams<R> W;
            W.bounce_sep = bounce_sep ? 1 : 0;
            W.c0 = static_cast<unsigned>(pp.c0);
            W.cn = static_cast<unsigned>(pp.cn);
            W.trace_work = cnt + 2 * NQ;
            W.rays = wf_rays_.p + pp.c0 * per_chain;
            W.hits = wf_hits_.p;
            W.occ = wf_occ_.p;
            W.state = wf_state_.p;
            W.pv = wf_pv_.p;
            W.cq_in = wf_cq_[a ^ 1].p + pp.c0;
            W.n_in = cnt + NQ * (a ^ 1);
            W.cq_out = wf_cq_[a].p + pp.c0;
            W.n_out = cnt + NQ * a;
            W.n_rays = cnt + 2 * NQ + 1 + a;
            if (r == 0 && p == 1)   // out of phase: the second range starts after the first's first logic kernel
                RAMLT_CUDA(cudaStreamWaitEvent(pp.st, wf_ev_[2], 0));
            logic<<<pp.lblocks, 128, lsmem, pp.st>>>(PL, W, r == 0 ? 1 : 0);
            if (bounce_sep && r > 0) {
                rd::k_wf_bounce<R, RK, INIT><<<pp.bblocks, 128, bsmem, pp.st>>>(P, W);
                ++launches_;
            }
            if (r == 0 && p == 0 && npipe > 1)
                RAMLT_CUDA(cudaEventRecord(wf_ev_[2], pp.st));
            cudaEvent_t t0 = nullptr, t1 = nullptr;
            if (prof) {
                RAMLT_CUDA(cudaEventCreate(&t0));
                RAMLT_CUDA(cudaEventCreate(&t1));
                RAMLT_CUDA(cudaEventRecord(t0, pp.st));
            }
            // traces this round's rays; zeroes the counters the next round's logic appends to
            if (use_bvh_)
                trace<<<pp.tblocks, 128, tsmem, pp.st>>>(P, W.rays, wf_hits_.p, wf_occ_.p, cnt + 2 * NQ + 1 + a,
                                                          cnt + 2 * NQ, cnt + NQ * (a ^ 1), cnt + 2 * NQ + 1 + (a ^ 1));
            else
                trace_brute<<<pp.tblocks, 128, tsmem, pp.st>>>(P, W.rays, wf_hits_.p, wf_occ_.p,
                                                                cnt + 2 * NQ + 1 + a, cnt + NQ * (a ^ 1),
                                                                cnt + 2 * NQ + 1 + (a ^ 1));
            if (prof) {
                RAMLT_CUDA(cudaEventRecord(t1, pp.st));
                ev_trace_.emplace_back(t0, t1);
            }
            launches_ += 2;
        }
        ++wf_rounds_;
        RAMLT_CUDA(cudaGetLastError());
        if (wf_log_) {   // RAMLT_WF_LOG=1: the round's queue lengths (ties an ncu launch to its ray count)
            unsigned hq[16];
            RAMLT_CUDA(cudaMemcpyAsync(hq, wf_cnt_.p, sizeof(hq), cudaMemcpyDeviceToHost, stream_));
            RAMLT_CUDA(cudaStreamSynchronize(stream_));
            std::fprintf(stderr, "wf %s round %d: rays %u, chains yielded %u %u %u %u %u\n", INIT ? "init" : "step", r,
                         hq[2 * NQ + 1 + a], hq[NQ * a], hq[NQ * a + 1], hq[NQ * a + 2], hq[NQ * a + 3], hq[NQ * a + 4]);
        }
        // A mutation yields at most max_vertices + 1 times (max_vertices - 1 closest-hit
        // rays, the eval_contribution batch, the eye_path_density batch), so a
        // one-step launch needs max_vertices + 2 logic rounds: they are enqueued
        // without a host round trip and the queue length is read back once, after
        // the last (a nonzero length -- never seen -- just continues the loop).
        // Multi-step launches (Fixed strategy) and chain initialisation poll every
        // wf_check_ rounds instead.
        const bool last_planned = !poll && r + 1 >= planned;
        const int check = INIT ? 8 * wf_check_ : wf_check_;   // initialisation runs thousands of short rounds
        if (last_planned || (poll && r % check == check - 1)) {
            join();
            unsigned left = 0;
            for (int p = 0; p < npipe; ++p) {
                RAMLT_CUDA(cudaMemcpyAsync(wf_host_, pipe[p].cnt + NQ * a, NQ * sizeof(unsigned),
                                           cudaMemcpyDeviceToHost, stream_));
                RAMLT_CUDA(cudaStreamSynchronize(stream_));
                for (int q = 0; q < NQ; ++q)
                    left += wf_host_[q];
            }
            if (left == 0)
                break;
            fork();
        }
    }
    if (prof) {
        RAMLT_CUDA(cudaEventRecord(e1, stream_));
        ev_.emplace_back(e0, e1);
    }
}

// All steps of a span in one cooperative launch when every chain group fits
// on the GPU at once (small chain counts, where per-step launches dominate).
template <class R>
bool EngineT<R>::launch_coop(int j0, int j1, unsigned long long span_start, unsigned long long per,
                             unsigned long long rem) {
    if (coop_state_ == 0 || j1 <= j0)
        return coop_state_ != 0 && j1 <= j0;
    if (const char *v = std::getenv("RAMLT_COOP"))
        if (std::string(v) == "0") {
            coop_state_ = 0;
            return false;
        }
    void (*kern)(rd::StepParams<R>, rd::CoopArgs<R>) = nullptr;
#define RAMLT_PICK(RK)                                                                              \
    switch (use_bvh_ ? 0 : G_) {                                                                    \
    case 0: kern = rd::k_step_coop<R, RK, 0>; break;                                                \
    case 1: kern = rd::k_step_coop<R, RK, 1>; break;                                                \
    case 2: kern = rd::k_step_coop<R, RK, 2>; break;                                                \
    case 4: kern = rd::k_step_coop<R, RK, 4>; break;                                                \
    case 8: kern = rd::k_step_coop<R, RK, 8>; break;                                                \
    case 16: kern = rd::k_step_coop<R, RK, 16>; break;                                              \
    default: kern = rd::k_step_coop<R, RK, 32>; break;                                              \
    }
    if (d_.rng == RAMLT_RNG_PHILOX) {
        RAMLT_PICK(rd::RNG_PHILOX)
    } else {
        RAMLT_PICK(rd::RNG_PCG)
    }
#undef RAMLT_PICK
    const long long threads = static_cast<long long>(C_) * G_;
    const unsigned blocks = static_cast<unsigned>((threads + 127) / 128);
    if (coop_state_ < 0) {
        int dev = 0, sms = 0, coop = 0, per_sm = 0;
        RAMLT_CUDA(cudaGetDevice(&dev));
        RAMLT_CUDA(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev));
        RAMLT_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        RAMLT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem_)));
        RAMLT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 128, smem_));
        coop_state_ = (coop && static_cast<long long>(per_sm) * sms >= blocks) ? 1 : 0;
        if (!coop_state_)
            return false;
    }
    rd::StepParams<R> P = params();
    P.span_start = span_start;
    P.per = per;
    P.rem = rem;
    P.j0 = j0;
    P.j1 = j1;
    P.record_visits = 1;
    P.ktab_l2 = 1;
    rd::CoopArgs<R> A;
    A.ktab = ktab_.p;
    A.cfg = adaptcfg();
    A.tb = tracebuf();
    A.pooled = adapt_ == 1 ? 1 : 0;
    A.key_bits = 1;
    while ((1ll << A.key_bits) - 1 < static_cast<long long>(n_regions_host_) + 0)
        ++A.key_bits;
    if ((1ll << A.key_bits) - 1 <= n_regions_host_ - 1)
        ++A.key_bits;
    void *args[] = {&P, &A};
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (d_.profile_kernels) {
        if (ev_.size() + ev_trace_.size() >= 4096)
            drain_events();
        RAMLT_CUDA(cudaEventCreate(&e0));
        RAMLT_CUDA(cudaEventCreate(&e1));
        RAMLT_CUDA(cudaEventRecord(e0, stream_));
    }
    RAMLT_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void *>(kern), dim3(blocks), dim3(128), args, smem_,
                                           stream_));
    ++launches_;
    if (d_.profile_kernels) {
        RAMLT_CUDA(cudaEventRecord(e1, stream_));
        ev_.emplace_back(e0, e1);
    }
    return true;
}

template <class R> void EngineT<R>::adapt_after_step(int j, unsigned long long span_start) {
    if (ctl_ == 0)
        return;
    rd::RegionArrays ra = regions();
    if (adapt_ == 0) {
        rd::k_adapt_literal<R><<<1, 1024, 0, stream_>>>(vreg_.p, va_.p, C_, off_, Ctot_, span_start, j, ra,
                                                         ktab_.p, adaptcfg(), tracebuf());
        ++launches_;
    } else {
        rd::k_adapt_pool_accum<<<static_cast<unsigned>((C_ + 255) / 256), 256, 0, stream_>>>(
            vreg_.p, va_.p, C_, off_, Ctot_, span_start, j, ra);
        ++launches_;
        if (!exchange_interval_)
            adapt_apply();
    }
    RAMLT_CUDA(cudaGetLastError());
}

template <class R> void EngineT<R>::adapt_apply() {
    if (ctl_ == 0 || adapt_ != 1)
        return;
    rd::RegionArrays ra = regions();
    rd::k_adapt_pool_apply<R><<<148, 256, 0, stream_>>>(ra, ktab_.p, adaptcfg(), tracebuf(),
                                                        exchange_interval_ ? n_regions_host_ : 0);
    rd::k_reset_touched<<<1, 1, 0, stream_>>>(n_touched_.p);
    launches_ += 2;
    RAMLT_CUDA(cudaGetLastError());
}

template <class R> void EngineT<R>::refine() {
    if (pkind_ != 2 && pkind_ != 4)
        return;
    // worst case every current region splits: keep capacity ahead of it
    size_t need = static_cast<size_t>(n_regions_host_) * 5 + 8;
    if (need > reg_cap_)
        grow_regions(std::max(need, reg_cap_ * 2));
    rd::RegionArrays ra = regions();
    const int n0 = n_nodes_host_;
    if (rf_key_[0].n < static_cast<size_t>(n0)) {
        size_t cap = std::max<size_t>(static_cast<size_t>(n0) * 2, 1024);
        for (int q = 0; q < 2; ++q) {
            rf_key_[q].alloc(cap);
            rf_val_[q].alloc(cap);
        }
        size_t tmp = 0;
        RAMLT_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, rf_key_[0].p, rf_key_[1].p, rf_val_[0].p,
                                                   rf_val_[1].p, static_cast<int>(cap)));
        rf_tmp_.alloc(tmp);
        rf_count_.alloc(1);
    }
    RAMLT_CUDA(cudaMemsetAsync(rf_count_.p, 0, sizeof(int), stream_));
    const unsigned nb = static_cast<unsigned>((n0 + 255) / 256);
    rd::k_refine_keys<<<nb, 256, 0, stream_>>>(nodes_.p, n0, n_trees_, visits_.p, d_.m_split, rf_key_[0].p,
                                                rf_val_[0].p, rf_count_.p);
    RAMLT_CUDA(cudaGetLastError());
    int end_bit = 1;
    while ((1 << end_bit) <= n_trees_)
        ++end_bit;
    size_t tmp = rf_tmp_.n;
    RAMLT_CUDA(cub::DeviceRadixSort::SortPairs(rf_tmp_.p, tmp, rf_key_[0].p, rf_key_[1].p, rf_val_[0].p,
                                               rf_val_[1].p, n0, 0, end_bit, stream_));
    rd::k_refine_apply<R><<<nb, 256, 0, stream_>>>(nodes_.p, n0, static_cast<int>(reg_cap_ + 4), rf_val_[1].p,
                                                   rf_count_.p, ra, ktab_.p, visits_.p, n_regions_.p,
                                                   static_cast<int>(reg_cap_), err_.p);
    RAMLT_CUDA(cudaGetLastError());
    rd::k_refine_finish<<<1, 1, 0, stream_>>>(n0, rf_count_.p, n_nodes_.p, n_regions_.p, splits_.p);
    launches_ += 4;
    RAMLT_CUDA(cudaGetLastError());
    RAMLT_CUDA(cudaMemcpyAsync(&n_regions_host_, n_regions_.p, sizeof(int), cudaMemcpyDeviceToHost, stream_));
    RAMLT_CUDA(cudaMemcpyAsync(&n_nodes_host_, n_nodes_.p, sizeof(int), cudaMemcpyDeviceToHost, stream_));
    check_err("refine");
}

template <class R> void EngineT<R>::fold() {
    if (sizeof(R) != 4)
        return;
    int npix = d_.width * d_.height;
    rd::k_fold_film<<<static_cast<unsigned>((npix + 255) / 256), 256, 0, stream_>>>(film32_.p, film64_.p, npix);
    ++launches_;
    RAMLT_CUDA(cudaGetLastError());
    steps_since_fold_ = 0;
}

template <class R> void EngineT<R>::reduce_chains(bool reset_interval, double out[6]) {
    unsigned blocks = static_cast<unsigned>((C_ + 255) / 256);
    rd::k_reduce_chains<<<blocks, 256, 0, stream_>>>(acc_.p, iacc_.p, lum_.p, npert_.p, nlarge_.p, ipert_.p, C_,
                                                     reset_interval ? 1 : 0, red_.p);
    ++launches_;
    RAMLT_CUDA(cudaGetLastError());
    std::vector<double> h(6 * blocks);
    RAMLT_CUDA(cudaMemcpyAsync(h.data(), red_.p, h.size() * sizeof(double), cudaMemcpyDeviceToHost, stream_));
    RAMLT_CUDA(cudaStreamSynchronize(stream_));
    for (int q = 0; q < 6; ++q)
        out[q] = 0.0;
    for (unsigned b = 0; b < blocks; ++b)
        for (int q = 0; q < 6; ++q)
            out[q] += h[6 * b + q];
}

template <class R> void EngineT<R>::flush_metrics(uint64_t at) {
    double r[6];
    reduce_chains(true, r);
    double t = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0_).count();
    // row.rrmse (core/driver.cpp:265-272): NaN unless a reference image is set;
    // a sharded handle holds a partial film, so its rows stay NaN
    double rr = (ref_img_.p && Ctot_ == C_) ? rrmse_now(at) : std::numeric_limits<double>::quiet_NaN();
    metrics_.push_back({t, static_cast<double>(at), rr, r[5] > 0 ? r[1] / r[5] : 0.0, r[1], r[5]});
}

template <class R> void EngineT<R>::set_reference(const float *rgb, int width, int height) {
    if (width != d_.width || height != d_.height)
        throw std::invalid_argument("error_report: image dimensions differ");
    size_t n = static_cast<size_t>(width) * height * 3;
    ref_img_.alloc(n);
    RAMLT_CUDA(cudaMemcpy(ref_img_.p, rgb, n * sizeof(float), cudaMemcpyHostToDevice));
}

// error_report(to_image(b / at), reference, kDefaultRrmseEpsilon = 1e-2, luminance).rrmse
template <class R> double EngineT<R>::rrmse_now(uint64_t at) {
    fold();
    const int npix = d_.width * d_.height;
    const unsigned blocks = static_cast<unsigned>((npix + 255) / 256);
    if (rrmse_part_.n < blocks)
        rrmse_part_.alloc(blocks);
    rd::k_rrmse_partial<<<blocks, 256, 0, stream_>>>(film64_.p, ref_img_.p, npix, b_ / static_cast<double>(at),
                                                      1e-2, rrmse_part_.p);
    ++launches_;
    RAMLT_CUDA(cudaGetLastError());
    std::vector<double> h(blocks);
    RAMLT_CUDA(cudaMemcpyAsync(h.data(), rrmse_part_.p, blocks * sizeof(double), cudaMemcpyDeviceToHost, stream_));
    RAMLT_CUDA(cudaStreamSynchronize(stream_));
    double sum = 0.0;
    for (double v : h)
        sum += v;
    return std::sqrt(sum / static_cast<double>(npix));
}

template <class R> void EngineT<R>::run(uint64_t mutations) {
    if (!chains_ready_)
        throw std::logic_error("run before init_chains");
    if (span_open_)
        throw std::logic_error("run() inside a span opened by run_steps(): finish it with run_steps");
    if (!t0_set_) {
        RAMLT_CUDA(cudaStreamSynchronize(stream_));
        t0_ = std::chrono::steady_clock::now();
        t0_set_ = true;
    }
    finalized_ = false;
    const uint64_t target = done_ + mutations;
    // Sharded quadtree runs defer the refine to the caller (visit all-reduce,
    // then ramlt_gpu_refine): a run must end at the refine boundary, never step
    // past it on the old partition (distributed.py chunks its runs this way).
    if (exchange_interval_ && (pkind_ == 2 || pkind_ == 4)) {
        if (refine_pending_ && mutations > 0)
            throw std::logic_error("sharded run: refine pending (all-reduce visits and call ramlt_gpu_refine first)");
        if (target > next_refine_)
            throw std::logic_error("sharded run crosses a refine boundary: end run() at multiples of m_refine");
    }
    const uint32_t fuse = d_.steps_per_launch ? d_.steps_per_launch : 256;
    while (done_ < target) {
        uint64_t boundary = std::min({target, next_refine_, next_metrics_});
        uint64_t span = boundary - done_;
        unsigned long long per = span / static_cast<uint64_t>(Ctot_);
        unsigned long long rem = span % static_cast<uint64_t>(Ctot_);
        int steps = static_cast<int>(per + (rem ? 1 : 0));
        if (ctl_ == 0) {
            for (int j = 0; j < steps; j += static_cast<int>(fuse)) {
                int j1 = std::min(steps, j + static_cast<int>(fuse));
                launch_step(j, j1, done_, per, rem, false);
                steps_since_fold_ += static_cast<uint64_t>(j1 - j);
                if (sizeof(R) == 4 && steps_since_fold_ >= 4096)
                    fold();
            }
        } else if (!exchange_interval_ && launch_coop(0, steps, done_, per, rem)) {
            steps_since_fold_ += static_cast<uint64_t>(steps);
        } else {
            for (int j = 0; j < steps; ++j) {
                launch_step(j, j + 1, done_, per, rem, true);
                adapt_after_step(j, done_);
                if (sizeof(R) == 4 && ++steps_since_fold_ >= 4096)
                    fold();
            }
        }
        done_ += span;
        span_boundary();
    }
    fold();
}

// Barrier work at the end of a span (core/driver.cpp:298-312): refine, metrics row.
template <class R> void EngineT<R>::span_boundary() {
    if (done_ == next_refine_) {
        if (exchange_interval_ && (pkind_ == 2 || pkind_ == 4))
            refine_pending_ = true;   // caller all-reduces visits, then ramlt_gpu_refine
        else
            refine();
        next_refine_ += d_.m_refine;
    }
    if (done_ == next_metrics_ || done_ == d_.mutations) {
        flush_metrics(done_);
        next_metrics_ = done_ + d_.metrics_interval;
    }
}

// Advance up to n lockstep steps of the canonical span loop -- the spans
// run(d.mutations) would use, so per-chain step counts (span % chains extra
// steps to the first chains, core/driver.cpp:283-291) do not depend on how
// often the caller stops -- returning early at the end of the current span
// (a barrier: refine / metrics row / total).  Sharded callers exchange between
// calls; with a refine pending (quadtree, exchange mode) no step runs until the
// caller has all-reduced the visits and called ramlt_gpu_refine.  Returns the
// global mutation count reached; *executed = lockstep steps run.
template <class R> uint64_t EngineT<R>::run_steps(uint32_t n, uint32_t *executed) {
    if (!chains_ready_)
        throw std::logic_error("run before init_chains");
    if (!t0_set_) {
        RAMLT_CUDA(cudaStreamSynchronize(stream_));
        t0_ = std::chrono::steady_clock::now();
        t0_set_ = true;
    }
    finalized_ = false;
    if (executed)
        *executed = 0;
    if (n == 0 || (!span_open_ && refine_pending_))
        return done_;
    const uint32_t fuse = d_.steps_per_launch ? d_.steps_per_launch : 256;
    if (!span_open_) {
        uint64_t end = done_ < d_.mutations ? d_.mutations : std::numeric_limits<uint64_t>::max();
        end = std::min({end, next_refine_, next_metrics_});
        const uint64_t span = end - done_;
        sp_start_ = done_;
        sp_end_ = end;
        sp_per_ = span / static_cast<uint64_t>(Ctot_);
        sp_rem_ = span % static_cast<uint64_t>(Ctot_);
        sp_steps_ = static_cast<int>(sp_per_ + (sp_rem_ ? 1 : 0));
        sp_j_ = 0;
        span_open_ = true;
    }
    const int j1 = static_cast<int>(std::min<uint64_t>(static_cast<uint64_t>(sp_steps_),
                                                        static_cast<uint64_t>(sp_j_) + n));
    if (ctl_ == 0) {
        for (int j = sp_j_; j < j1; j += static_cast<int>(fuse)) {
            int je = std::min(j1, j + static_cast<int>(fuse));
            launch_step(j, je, sp_start_, sp_per_, sp_rem_, false);
            steps_since_fold_ += static_cast<uint64_t>(je - j);
            if (sizeof(R) == 4 && steps_since_fold_ >= 4096)
                fold();
        }
    } else {
        for (int j = sp_j_; j < j1; ++j) {
            launch_step(j, j + 1, sp_start_, sp_per_, sp_rem_, true);
            adapt_after_step(j, sp_start_);
            if (sizeof(R) == 4 && ++steps_since_fold_ >= 4096)
                fold();
        }
    }
    if (executed)
        *executed = static_cast<uint32_t>(j1 - sp_j_);
    sp_j_ = j1;
    fold();
    if (sp_j_ == sp_steps_) {
        span_open_ = false;
        done_ = sp_end_;
        span_boundary();
        return done_;
    }
    const uint64_t j = static_cast<uint64_t>(sp_j_);
    return sp_start_ + (j <= sp_per_ ? j * static_cast<uint64_t>(Ctot_)
                                     : sp_per_ * static_cast<uint64_t>(Ctot_) + sp_rem_);
}

template <class R> void EngineT<R>::render() {
    if (!b_set_)
        estimate_b(nullptr, nullptr);
    if (!chains_ready_)
        init_chains();
    if (d_.time_budget_s > 0.0) {
        if (!t0_set_) {
            RAMLT_CUDA(cudaStreamSynchronize(stream_));
            t0_ = std::chrono::steady_clock::now();
            t0_set_ = true;
        }
        for (;;) {
            run(std::min<uint64_t>(d_.metrics_interval, next_metrics_ - done_));
            RAMLT_CUDA(cudaStreamSynchronize(stream_));
            double t = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0_).count();
            if (t >= d_.time_budget_s)
                break;
        }
    } else {
        run(d_.mutations - std::min(d_.mutations, done_));
    }
    finalize_stats();
}

template <class R> void EngineT<R>::finalize_stats() {
    if (metrics_.empty() || static_cast<uint64_t>(metrics_.back()[1]) != done_) {
        if (!t0_set_) {
            t0_ = std::chrono::steady_clock::now();
            t0_set_ = true;
        }
        flush_metrics(done_);
    }
    double r[6];
    reduce_chains(false, r);
    ramlt_stats s{};
    s.b = b_;
    s.b_stderr = b_se_;
    s.b_samples = b_n_;
    s.total_mutations = done_;
    s.perturbation_proposals = static_cast<uint64_t>(r[3]);
    s.large_step_proposals = static_cast<uint64_t>(r[4]);
    s.mean_acceptance = r[3] > 0 ? r[0] / r[3] : 0.0;
    s.film_luminance = r[2];
    s.loop_time_s = metrics_.empty() ? 0.0 : metrics_.back()[0];
    final_ = s;
    finalized_ = true;
}

template <class R> void EngineT<R>::read_stats(ramlt_stats *out) {
    if (!finalized_)
        finalize_stats();
    ramlt_stats s = final_;
    unsigned long long rays[2];
    RAMLT_CUDA(cudaMemcpyAsync(rays, rays_.p, sizeof(rays), cudaMemcpyDeviceToHost, stream_));
    RAMLT_CUDA(cudaStreamSynchronize(stream_));
    s.rays_closest = rays[0];
    s.rays_visibility = rays[1];
    std::vector<double> acc(n_regions_host_);
    std::vector<uint64_t> vis(n_regions_host_);
    uint64_t nt = read_tallies(acc.data(), vis.data(), acc.size());
    // global_acceptance_identity (core/adaptation.cpp:103-125)
    double tot = 0.0, comp = 0.0;
    uint64_t tv = 0;
    for (uint64_t i = 0; i < nt; ++i) {
        double y = acc[i] - comp;
        double sm = tot + y;
        comp = (sm - tot) - y;
        tot = sm;
        tv += vis[i];
    }
    s.identity_residual = 0.0;
    if (tv > 0) {
        double pooled = tot / static_cast<double>(tv);
        double w = 0.0;
        for (uint64_t i = 0; i < nt; ++i) {
            if (!vis[i])
                continue;
            w += (static_cast<double>(vis[i]) / static_cast<double>(tv)) * (acc[i] / static_cast<double>(vis[i]));
        }
        s.identity_residual = std::abs(pooled - w);
    }
    s.n_tallies = nt;
    // region_count: partition leaves (partition.hpp:33) or controller regions
    if (pkind_ == 2 || pkind_ == 4) {
        std::vector<rd::NodeD> nodes(n_nodes_host_);
        RAMLT_CUDA(cudaMemcpy(nodes.data(), nodes_.p, nodes.size() * sizeof(rd::NodeD), cudaMemcpyDeviceToHost));
        uint64_t leaves = 0;
        for (auto &nd : nodes)
            leaves += nd.child < 0;
        s.region_count = leaves;
    } else {
        s.region_count = static_cast<uint64_t>(n_regions_host_);
    }
    unsigned long long tc = 0;
    RAMLT_CUDA(cudaMemcpy(&tc, trace_count_.p, sizeof(tc), cudaMemcpyDeviceToHost));
    s.n_trace = std::min<uint64_t>(tc, trace_index_.n);
    s.n_metrics = metrics_.size();
    s.kernel_launches = launches_;
    drain_events();
    s.step_kernel_ms = step_ms_;
    s.step_kernel_launches = step_launches_;
    s.trace_kernel_ms = trace_ms_;
    s.trace_kernel_launches = trace_launches_;
    s.wavefront_rounds = wf_rounds_;
    *out = s;
}

template <class R> void EngineT<R>::read_film(double *rgb, double *lum) {
    fold();
    if (rgb)
        RAMLT_CUDA(cudaMemcpyAsync(rgb, film64_.p, film64_.n * sizeof(double), cudaMemcpyDeviceToHost, stream_));
    RAMLT_CUDA(cudaStreamSynchronize(stream_));
    if (lum) {
        double r[6];
        reduce_chains(false, r);
        *lum = r[2];
    }
}

template <class R> void EngineT<R>::read_image(float *rgb) {
    fold();
    DBuf<float> img;
    img.alloc(film64_.n);
    double scale = done_ > 0 ? b_ / static_cast<double>(done_) : 0.0;
    rd::k_to_image<<<static_cast<unsigned>((film64_.n + 255) / 256), 256, 0, stream_>>>(
        film64_.p, img.p, static_cast<int>(film64_.n), scale);
    ++launches_;
    RAMLT_CUDA(cudaGetLastError());
    RAMLT_CUDA(cudaMemcpyAsync(rgb, img.p, film64_.n * sizeof(float), cudaMemcpyDeviceToHost, stream_));
    RAMLT_CUDA(cudaStreamSynchronize(stream_));
}

template <class R> uint64_t EngineT<R>::read_tallies(double *acc, uint64_t *vis, uint64_t cap) {
    // Fixed controllers never record (adaptation.cpp:63-64): one all-zero tally.
    uint64_t n = static_cast<uint64_t>(n_regions_host_);
    uint64_t m = std::min(n, cap);
    std::vector<double> ta(n);
    std::vector<unsigned long long> tv(n), tf(n);
    RAMLT_CUDA(cudaStreamSynchronize(stream_));
    RAMLT_CUDA(cudaMemcpy(ta.data(), tot_acc_.p, n * sizeof(double), cudaMemcpyDeviceToHost));
    RAMLT_CUDA(cudaMemcpy(tv.data(), tot_vis_.p, n * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
    RAMLT_CUDA(cudaMemcpy(tf.data(), tot_fx_.p, n * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
    for (uint64_t i = 0; i < m; ++i) {
        if (acc)
            acc[i] = adapt_ == 1 ? static_cast<double>(tf[i]) / 16777216.0 : ta[i];
        if (vis)
            vis[i] = tv[i];
    }
    return n;
}

template <class R> uint64_t EngineT<R>::read_regions(double *lambda, uint64_t *n, uint64_t cap) {
    uint64_t cnt = static_cast<uint64_t>(n_regions_host_);
    uint64_t m = std::min(cnt, cap);
    RAMLT_CUDA(cudaStreamSynchronize(stream_));
    if (lambda && m)
        RAMLT_CUDA(cudaMemcpy(lambda, lambda_.p, m * sizeof(double), cudaMemcpyDeviceToHost));
    if (n && m)
        RAMLT_CUDA(cudaMemcpy(n, n_.p, m * sizeof(uint64_t), cudaMemcpyDeviceToHost));
    return cnt;
}

template <class R> uint64_t EngineT<R>::read_trace(ramlt_trace_row *rows, uint64_t cap) {
    unsigned long long tc = 0;
    RAMLT_CUDA(cudaStreamSynchronize(stream_));
    RAMLT_CUDA(cudaMemcpy(&tc, trace_count_.p, sizeof(tc), cudaMemcpyDeviceToHost));
    uint64_t n = std::min<uint64_t>(tc, trace_index_.n);
    std::vector<unsigned long long> idx(n), nn(n);
    std::vector<long long> reg(n);
    std::vector<double> lam(n), al(n);
    if (n) {
        RAMLT_CUDA(cudaMemcpy(idx.data(), trace_index_.p, n * 8, cudaMemcpyDeviceToHost));
        RAMLT_CUDA(cudaMemcpy(nn.data(), trace_n_.p, n * 8, cudaMemcpyDeviceToHost));
        RAMLT_CUDA(cudaMemcpy(reg.data(), trace_region_.p, n * 8, cudaMemcpyDeviceToHost));
        RAMLT_CUDA(cudaMemcpy(lam.data(), trace_lambda_.p, n * 8, cudaMemcpyDeviceToHost));
        RAMLT_CUDA(cudaMemcpy(al.data(), trace_alpha_.p, n * 8, cudaMemcpyDeviceToHost));
    }
    // device appends are unordered across regions: restore (index, region, n) order
    std::vector<size_t> ord(n);
    for (size_t i = 0; i < n; ++i)
        ord[i] = i;
    std::sort(ord.begin(), ord.end(), [&](size_t a, size_t b) {
        if (idx[a] != idx[b])
            return idx[a] < idx[b];
        if (reg[a] != reg[b])
            return reg[a] < reg[b];
        return nn[a] < nn[b];
    });
    uint64_t m = std::min(n, cap);
    for (uint64_t i = 0; i < m && rows; ++i) {
        size_t o = ord[i];
        rows[i].mutation_index = idx[o];
        rows[i].region = reg[o];
        rows[i].n = nn[o];
        rows[i].lambda = lam[o];
        rows[i].alpha_hat = al[o];
    }
    return n;
}

template <class R> uint64_t EngineT<R>::read_metrics(double *rows, uint64_t cap) {
    uint64_t m = std::min<uint64_t>(metrics_.size(), cap);
    for (uint64_t i = 0; i < m; ++i)
        for (int q = 0; q < 4; ++q)
            rows[4 * i + q] = metrics_[i][q];
    return metrics_.size();
}

template <class R> void EngineT<R>::read_decisions(uint32_t K, double *a, uint8_t *flags) {
    uint32_t Kd = d_.log_steps;
    size_t C = static_cast<size_t>(C_);
    std::vector<double> ha(C * Kd);
    std::vector<unsigned char> hf(C * Kd);
    RAMLT_CUDA(cudaStreamSynchronize(stream_));
    if (Kd) {
        RAMLT_CUDA(cudaMemcpy(ha.data(), log_a_.p, ha.size() * sizeof(double), cudaMemcpyDeviceToHost));
        RAMLT_CUDA(cudaMemcpy(hf.data(), log_f_.p, hf.size(), cudaMemcpyDeviceToHost));
    }
    for (size_t c = 0; c < C; ++c)
        for (uint32_t k = 0; k < K; ++k) {
            bool in = k < Kd;
            if (a)
                a[c * K + k] = in ? ha[static_cast<size_t>(k) * C + c] : 0.0;
            if (flags)
                flags[c * K + k] = in ? hf[static_cast<size_t>(k) * C + c] : 0;
        }
}

template <class R> std::string EngineT<R>::read_partition_visits(const uint64_t *ext, uint64_t n_ext) {
    // PartitionIndex::dump formats (core/partition.cpp:104-121, 138-147, 175-190, 229-245)
    uint64_t n = static_cast<uint64_t>(n_regions_host_);
    std::vector<double> lam(n);
    std::vector<uint64_t> nn(n);
    read_regions(lam.data(), nn.data(), n);
    std::vector<unsigned long long> vis(n);
    if (ext) {
        if (n_ext != n)
            throw std::invalid_argument("partition dump: visit array length differs from the region count");
        for (uint64_t i = 0; i < n; ++i)
            vis[i] = ext[i];
    } else {
        RAMLT_CUDA(cudaMemcpy(vis.data(), visits_.p, n * 8, cudaMemcpyDeviceToHost));
    }
    std::ostringstream os;
    auto leaf_line = [&](int region, double u0, double v0, double u1, double v1) {
        double l = ctl_ == 0 ? d_.lambda_init : lam[region];
        os << "leaf " << region << " " << u0 << " " << v0 << " " << u1 << " " << v1 << " " << l << " "
           << nn[region] << " " << vis[region] << "\n";
    };
    auto cell_b = [](int g, int cell, double *b) {
        int iy = cell / g, ix = cell % g;
        double inv = 1.0 / g;
        b[0] = ix * inv;
        b[1] = iy * inv;
        b[2] = (ix + 1) * inv;
        b[3] = (iy + 1) * inv;
    };
    std::vector<rd::NodeD> nodes(n_nodes_host_);
    if (n_nodes_host_)
        RAMLT_CUDA(cudaMemcpy(nodes.data(), nodes_.p, nodes.size() * sizeof(rd::NodeD), cudaMemcpyDeviceToHost));
    auto tree_leaves = [&](int tree) {
        for (const rd::NodeD &nd : nodes) {
            if (nd.tree != tree || nd.child >= 0)
                continue;
            double sc = std::ldexp(1.0, -nd.level);
            leaf_line(nd.region, nd.ix * sc, nd.iy * sc, (nd.ix + 1) * sc, (nd.iy + 1) * sc);
        }
    };
    double b[4];
    if (pkind_ == 1) {
        for (int c = 0; c < d_.n_top * d_.n_top; ++c) {
            cell_b(d_.n_top, c, b);
            leaf_line(c, b[0], b[1], b[2], b[3]);
        }
    } else if (pkind_ == 2) {
        tree_leaves(0);
    } else if (pkind_ == 3 || pkind_ == 4) {
        for (int c = 0; c < d_.n_top * d_.n_top; ++c) {
            cell_b(d_.n_top, c, b);
            os << "# cell " << c << " " << b[0] << " " << b[1] << " " << b[2] << " " << b[3] << "\n";
            if (pkind_ == 4) {
                tree_leaves(c);
            } else {
                int nb2 = d_.n_bottom * d_.n_bottom;
                for (int sb = 0; sb < nb2; ++sb) {
                    double bb[4];
                    cell_b(d_.n_bottom, sb, bb);
                    leaf_line(c * nb2 + sb, bb[0], bb[1], bb[2], bb[3]);
                }
            }
        }
    }
    return os.str();
}

}  // namespace ramlt_b200
