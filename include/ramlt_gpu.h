/*
 * ramlt_gpu.h -- C-ABI of the B200 MLT engine (libramlt_gpu.so).
 *
 * This is the drop-in boundary for the reference's renderer entry point
 *     ramlt::RenderResult ramlt::run_render(SceneModel, const RenderConfig&)
 *         (reference: proj/src/core/driver.hpp:80, driver.cpp:177-342)
 * whose file-local integrator run_chain_span (driver.cpp:109-173) is what the
 * sm_100a kernels replace.  Plain C types only: no torch, no C++ in the
 * signatures.  Every entry point names the reference interface it replaces.
 *
 * Conventions (mirroring the reference's error behaviour):
 *   return value 0 = success; otherwise one of RAMLT_E_* and
 *   ramlt_gpu_last_error(h) (or ramlt_gpu_last_create_error() when no handle
 *   exists) holds the reference-style message, e.g. "black-scene: ...".
 *   RAMLT_E_RUNTIME  <-> std::runtime_error   (driver.cpp:54, 241; scene parse)
 *   RAMLT_E_LOGIC    <-> std::logic_error     (RAMLT_CHECK, check.hpp:15-19)
 *   RAMLT_E_INVALID  <-> std::invalid_argument (sampling.cpp:63; camera.cpp:10-24;
 *                                              mutations.cpp:200)
 *   RAMLT_E_CUDA     a CUDA/driver failure (no reference counterpart)
 * A handle is single-host-thread and not re-entrant.  The caller owns every
 * descriptor and output buffer; create() copies the scene to the device.
 */
#ifndef RAMLT_GPU_H
#define RAMLT_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RAMLT_GPU_ABI_VERSION 2

#if defined(__GNUC__)
#define RAMLT_API __attribute__((visibility("default")))
#else
#define RAMLT_API
#endif

enum {
    RAMLT_OK = 0,
    RAMLT_E_RUNTIME = 1,
    RAMLT_E_LOGIC = 2,
    RAMLT_E_INVALID = 3,
    RAMLT_E_OTHER = 4,
    RAMLT_E_CUDA = 5
};

/* StrategyVariant (driver.hpp:15), PerturbationKind (driver.hpp:17) */
enum { RAMLT_FIXED = 0, RAMLT_GLOBAL = 1, RAMLT_RA_GRID = 2, RAMLT_RA_QUADTREE = 3 };
enum { RAMLT_LENS = 0, RAMLT_MULTI_CHAIN = 1 };
/* MaterialKind (scene.hpp:18) */
enum { RAMLT_DIFFUSE = 0, RAMLT_MIRROR = 1, RAMLT_DIELECTRIC = 2, RAMLT_GLOSSY = 3 };
/* engine knobs */
enum { RAMLT_F32 = 0, RAMLT_F64 = 1 };
enum { RAMLT_RNG_PCG32 = 0, RAMLT_RNG_PHILOX = 1 };
enum { RAMLT_ADAPT_AUTO = -1, RAMLT_ADAPT_LITERAL = 0, RAMLT_ADAPT_POOLED = 1 };
/* auto: BVH above 128 triangles; brute: smem-staged linear scan; bvh: SAH BVH2 */
enum { RAMLT_ACCEL_AUTO = 0, RAMLT_ACCEL_BRUTE = 1, RAMLT_ACCEL_BVH = 2 };

/* Material (scene.hpp:20-31) */
typedef struct ramlt_material {
    int32_t kind;
    int32_t pad_;
    double albedo[3];
    double ior;
    double exponent;
} ramlt_material;

/* Sphere / Triangle (scene.hpp:44-53) with the per-primitive emitter id that
 * SceneModel::sphere_emitter / triangle_emitter hold (scene.hpp:69-70). */
typedef struct ramlt_sphere {
    double center[3];
    double radius;
    int32_t material;
    int32_t emitter;
} ramlt_sphere;

typedef struct ramlt_triangle {
    double a[3], b[3], c[3];
    int32_t material;
    int32_t emitter;
} ramlt_triangle;

/* SceneModel (scene.hpp:60-75).  The camera is given by its constructor
 * arguments (camera.hpp:17); the engine rebuilds the basis with the
 * reference's formulas (camera.cpp:8-30) in fp64 on the host. */
typedef struct ramlt_scene_desc {
    double cam_position[3];
    double cam_look_at[3];
    double cam_up[3];
    double cam_fov_deg;
    int32_t n_materials, n_spheres, n_triangles, n_emitters;
    const ramlt_material *materials;
    const ramlt_sphere *spheres;
    const ramlt_triangle *triangles;
    const double *emitter_radiance; /* n_emitters * 3 (Emitter::radiance, scene.hpp:55-58) */
} ramlt_scene_desc;

/* RenderConfig (driver.hpp:19-39) + AdaptationConfig (adaptation.hpp:14-22)
 * field for field, then the B200 engine knobs.  ramlt_gpu_default_desc()
 * fills the reference defaults (§8.1). */
typedef struct ramlt_render_desc {
    int32_t strategy;
    int32_t perturbation;
    uint64_t mutations;
    double time_budget_s;
    int32_t chains;
    int32_t batch_size;
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
    int32_t dump_partition;
    /* ---- B200 engine knobs ---- */
    int32_t precision;        /* RAMLT_F32 (production) | RAMLT_F64 (parity) */
    int32_t rng;              /* RAMLT_RNG_PCG32 (reference streams) | RAMLT_RNG_PHILOX */
    int32_t adapt_mode;       /* RAMLT_ADAPT_* (auto: literal <= 4096 chains, else pooled) */
    int32_t lanes_per_chain;  /* 0 = auto, else 1,2,4,8,16,32 lanes cooperate on a chain */
    int32_t device;           /* CUDA device ordinal, -1 = current */
    int32_t pad_;
    int64_t chains_total;     /* sharding: global chain count (0 = chains) */
    int64_t chain_offset;     /* sharding: first global chain id of this handle */
    uint32_t log_steps;       /* K: per-chain decision log depth (0 = off) */
    uint32_t steps_per_launch;/* Fixed strategy: lockstep steps fused per launch (0 = auto) */
    uint64_t trace_capacity;  /* adaptation trace rows kept on the device */
    uint64_t region_capacity; /* initial region/node capacity (0 = auto; grows at barriers) */
    uint64_t b_substreams;    /* parallel b-estimate substreams (0 = 65536) */
    int32_t profile_kernels;  /* record CUDA events around every chain-step launch */
    int32_t accel;            /* RAMLT_ACCEL_*: triangle intersection structure */
} ramlt_render_desc;

/* RenderResult scalars (driver.hpp:64-78) + device counters. */
typedef struct ramlt_stats {
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
    double loop_time_s;          /* metrics.back().time_s equivalent */
    uint64_t rays_closest;       /* device closest-hit casts in the mutation loop */
    uint64_t rays_visibility;    /* device visibility casts in the mutation loop */
    uint64_t n_tallies;
    uint64_t n_trace;
    uint64_t n_metrics;
    uint64_t kernel_launches;    /* engine kernels launched so far */
    double step_kernel_ms;       /* summed event time of chain-step launches (profile_kernels) */
    uint64_t step_kernel_launches;
    double trace_kernel_ms;      /* wavefront steps: summed event time of the k_wf_trace launches */
    uint64_t trace_kernel_launches;
    uint64_t wavefront_rounds;   /* wavefront steps: logic/trace rounds launched */
} ramlt_stats;

/* UpdateEvent trace row (driver.hpp:59-62, adaptation.hpp:51-56). */
typedef struct ramlt_trace_row {
    uint64_t mutation_index;
    int64_t region;
    uint64_t n;
    double lambda;
    double alpha_hat;
} ramlt_trace_row;

RAMLT_API int ramlt_gpu_abi_version(void);
RAMLT_API void ramlt_gpu_default_desc(ramlt_render_desc *desc);

/* parse_scene (scene.hpp:77-78, scene.cpp:114-234): text -> descriptor
 * arrays owned by the returned opaque scene; ramlt_scene_free releases it. */
typedef struct ramlt_scene ramlt_scene;
RAMLT_API int ramlt_scene_parse(const char *text, const char *origin, ramlt_scene **out);
RAMLT_API const ramlt_scene_desc *ramlt_scene_get_desc(const ramlt_scene *scene);
RAMLT_API void ramlt_scene_free(ramlt_scene *scene);

typedef struct ramlt_gpu ramlt_gpu;

/* Validates the config (RAMLT_CHECKs of driver.cpp:178-180), configures the
 * camera (driver.cpp:181), uploads the scene, allocates chain state and builds
 * the controller/partition (driver.cpp:190-212). */
RAMLT_API int ramlt_gpu_create(const ramlt_scene_desc *scene, const ramlt_render_desc *desc, ramlt_gpu **out);
RAMLT_API int ramlt_gpu_create_from_text(const char *scene_text, const char *origin,
                               const ramlt_render_desc *desc, ramlt_gpu **out);
RAMLT_API const char *ramlt_gpu_last_create_error(void);

/* create() over several devices of this process (n_dev, devs):
 * one handle, chains sharded by global id in contiguous blocks (device i owns
 * [i*C/n, (i+1)*C/n)), so it is a drop-in for run_render's thread-per-chain
 * loop (core/driver.cpp:282-297) at 1..8 GPUs.  Exchanges are device to device
 * over peer memory (NVLink/NVSwitch), stream-ordered: pooled adaptation after
 * every lockstep step, quadtree visits at every m_refine barrier, b partials
 * once, and the film every film_sync_steps lockstep steps (configs[4]: 4096;
 * 0 = only at metrics rows and reads) -- film merge of core/film.cpp:22-27.
 * Fixed runs are identical to the single-device handle; adaptive runs use the
 * pooled rule (RAMLT_ADAPT_POOLED), also identical to one device.  Devices may
 * repeat (two shards on one GPU: a functional test of the same path).
 * n_dev == 1 returns a plain single-device handle on devs[0].  The per-shard
 * plumbing calls (set_stream, film_device, adapt_*, visits_device, refine)
 * return RAMLT_E_LOGIC on a multi-device handle. */
RAMLT_API int ramlt_gpu_create_multi(const ramlt_scene_desc *scene, const ramlt_render_desc *desc, int32_t n_dev,
                                     const int32_t *devs, uint32_t film_sync_steps, ramlt_gpu **out);
RAMLT_API int ramlt_gpu_create_multi_from_text(const char *scene_text, const char *origin,
                                               const ramlt_render_desc *desc, int32_t n_dev, const int32_t *devs,
                                               uint32_t film_sync_steps, ramlt_gpu **out);

/* estimate_b (driver.hpp:49, driver.cpp:31-57) over desc.b_samples samples
 * split into b_substreams independent substreams. */
RAMLT_API int ramlt_gpu_estimate_b(ramlt_gpu *h, double *b, double *stderr_);
/* Partial sums of substreams [begin, end) for sharded estimation: out receives
 * (end-begin)*2 doubles (sum, sum of squares) in substream order. */
RAMLT_API int ramlt_gpu_estimate_b_partials(ramlt_gpu *h, uint64_t begin, uint64_t end, double *out);
/* Reduce gathered partials (all substreams, in order) exactly like
 * ramlt_gpu_estimate_b and install the result. */
RAMLT_API int ramlt_gpu_reduce_b(ramlt_gpu *h, const double *partials, uint64_t n_substreams,
                       double *b, double *stderr_);
RAMLT_API int ramlt_gpu_set_b(ramlt_gpu *h, double b);

/* Chain initialisation (driver.cpp:219-242): per chain, eye paths from stream
 * kStreamInit + 2*id until pi > 0. */
RAMLT_API int ramlt_gpu_init_chains(ramlt_gpu *h);

/* The span loop (driver.cpp:276-311): advances by `mutations` global
 * mutations, splitting at m_refine / metrics_interval boundaries exactly as
 * the reference does (per-chain steps = span / chains, +1 for the first
 * span % chains chains), refining and flushing metrics at the barriers. */
RAMLT_API int ramlt_gpu_run(ramlt_gpu *h, uint64_t mutations);
/* The span loop of run_render (core/driver.cpp:282-312) one piece at a time,
 * for sharded callers that exchange state between lockstep steps: runs up to
 * n lockstep steps of the CANONICAL spans (boundaries at the configured total
 * and the m_refine / metrics_interval barriers -- exactly the spans of
 * ramlt_gpu_run(desc.mutations), so every chain's step count and decisions
 * are independent of n), returning early at the end of a span.  *done = the
 * global mutation count reached, *executed = lockstep steps run (0 while a
 * sharded quadtree refine is pending).  Do not mix with ramlt_gpu_run inside
 * an open span (RAMLT_E_LOGIC). */
RAMLT_API int ramlt_gpu_run_steps(ramlt_gpu *h, uint32_t n, uint64_t *done, uint32_t *executed);

/* run_render in one call: estimate_b (unless set), init, run(desc.mutations)
 * or the wall-clock budget, finalise.  Synchronous. */
RAMLT_API int ramlt_gpu_render(ramlt_gpu *h);

/* Blocks until all queued device work of the handle is done. */
RAMLT_API int ramlt_gpu_synchronize(ramlt_gpu *h);

/* Outputs (RenderResult fields). */
RAMLT_API int ramlt_gpu_read_stats(ramlt_gpu *h, ramlt_stats *out);
/* Unscaled film (Film::accum_, film.hpp:41), rows top to bottom, RGB fp64. */
RAMLT_API int ramlt_gpu_read_film(ramlt_gpu *h, double *rgb, double *total_luminance);
/* Film::to_image(b / total_mutations) (film.cpp:29-34, driver.cpp:325). */
RAMLT_API int ramlt_gpu_read_image(ramlt_gpu *h, float *rgb);
/* KernelController::tallies (adaptation.hpp:84-88). */
RAMLT_API int ramlt_gpu_read_tallies(ramlt_gpu *h, double *accept_sum, uint64_t *visits, uint64_t cap,
                           uint64_t *n);
/* Region lambda / update counts (KernelController::lambda_of / updates_of). */
RAMLT_API int ramlt_gpu_read_regions(ramlt_gpu *h, double *lambda, uint64_t *n, uint64_t cap, uint64_t *count);
RAMLT_API int ramlt_gpu_read_trace(ramlt_gpu *h, ramlt_trace_row *rows, uint64_t cap, uint64_t *n);
/* MetricsRow (driver.hpp:52-57): cap rows of (time_s, mutations, rrmse, mean_acceptance);
 * rrmse is NaN unless a reference image was set (driver.cpp:265-272). */
RAMLT_API int ramlt_gpu_read_metrics(ramlt_gpu *h, double *rows, uint64_t cap, uint64_t *n);
/* Per-chain decision log of the first K steps: a[K][chains] and flags
 * (bit0 accepted, bit1 perturbation, bit2 logged), chain-major copy out:
 * a[chain*K + step]. */
RAMLT_API int ramlt_gpu_read_decisions(ramlt_gpu *h, uint32_t K, double *a, uint8_t *flags);
/* PartitionIndex::dump text (partition.hpp:30, partition.cpp:104-245). */
RAMLT_API int ramlt_gpu_read_partition(ramlt_gpu *h, char *buf, uint64_t cap);
/* The same dump with caller-supplied per-region visit counts (n = region
 * count): a sharded caller (one process per GPU) passes the SUM over ranks of
 * ramlt_gpu_visits_device, since leaf visits are split over the shards between
 * refine barriers. */
RAMLT_API int ramlt_gpu_read_partition_visits(ramlt_gpu *h, const uint64_t *visits, uint64_t n, char *buf,
                                              uint64_t cap);
/* Current path length k (vertices, camera included; Path::vertices.size(),
 * core/path.hpp:28-35) of every chain of the handle, in chain order. */
RAMLT_API int ramlt_gpu_read_chain_lengths(ramlt_gpu *h, int32_t *k);

/* ---- multi-GPU plumbing (chains shard across ranks) ----
 * The caller (e.g. torch.distributed over NCCL) owns the collective; the
 * engine works on the caller's CUDA stream so stream order is shared. */
RAMLT_API int ramlt_gpu_set_stream(ramlt_gpu *h, void *cuda_stream);
/* Device pointer + element count of the fp64 film (W*H*3) for an all-reduce. */
RAMLT_API int ramlt_gpu_film_device(ramlt_gpu *h, double **film, uint64_t *n);
/* Pooled adaptation exchange: device arrays of per-region (visit count u64,
 * fixed-point acceptance sum u64, last mutation index u64) accumulated since
 * the last apply, for a SUM/SUM/MAX all-reduce; then apply on every rank. */
RAMLT_API int ramlt_gpu_adapt_exchange(ramlt_gpu *h, uint64_t **counts, uint64_t **fx_sums,
                             uint64_t **last_index, uint64_t *n_regions);
RAMLT_API int ramlt_gpu_adapt_apply(ramlt_gpu *h);
/* Split a run into externally synchronised chunks: the engine pauses for an
 * exchange every `steps` lockstep steps (0 = never).  In this mode quadtree
 * refinement at m_refine barriers is deferred: the caller SUM-all-reduces the
 * per-region visit counts (ramlt_gpu_visits_device) and calls
 * ramlt_gpu_refine on every rank (identical partitions); keep_counts = 0 on all
 * ranks but one so carried-over counts are summed once. */
RAMLT_API int ramlt_gpu_set_exchange_interval(ramlt_gpu *h, uint32_t steps);
RAMLT_API int ramlt_gpu_visits_device(ramlt_gpu *h, uint64_t **visits, uint64_t *n_regions);
RAMLT_API int ramlt_gpu_refine_pending(ramlt_gpu *h, int32_t *pending);
RAMLT_API int ramlt_gpu_refine(ramlt_gpu *h, int32_t keep_counts);

/* RenderConfig::reference (driver.hpp:38): a W*H*3 fp32 image (rows top to
 * bottom, as read_image) copied to the device; every metrics row then carries
 * error_report(image, reference, 1e-2, luminance).rrmse (diagnostics.cpp:11-38).
 * Dimensions must match the render (std::invalid_argument otherwise). */
RAMLT_API int ramlt_gpu_set_reference(ramlt_gpu *h, const float *rgb, int32_t width, int32_t height);
/* error_report(to_image(b / at), reference, 1e-2, luminance).rrmse
 * (core/diagnostics.cpp:11-38, the MetricsRow.rrmse of core/driver.cpp:265-272)
 * of the handle's current film; NaN without a reference.  On a sharded handle
 * (chains_total > chains) call it after the film all-reduce. */
RAMLT_API int ramlt_gpu_rrmse(ramlt_gpu *h, uint64_t at, double *out);

/* Diagnostic (no reference counterpart): closest-hit throughput of the scene's
 * triangle accelerator alone, for the roofline discussion in DESIGN.md.
 * n_rays seeded incoherent rays (origins uniform in the scene bounds shrunk by
 * 10 %, directions uniform on the sphere) traced by the coroutine kernel's
 * traversal loop with dynamic ray fetch; returns the kernel time (CUDA events)
 * and the number of rays that hit a triangle. */
RAMLT_API int ramlt_gpu_trace_benchmark(ramlt_gpu *h, uint64_t n_rays, double *ms, uint64_t *hits);

RAMLT_API const char *ramlt_gpu_last_error(ramlt_gpu *h);
RAMLT_API void ramlt_gpu_destroy(ramlt_gpu *h);

#ifdef __cplusplus
}
#endif
#endif /* RAMLT_GPU_H */
