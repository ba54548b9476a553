// capi.cpp -- the C-ABI of libramlt_gpu.so (include/ramlt_gpu.h), the host
// mirror of the reference's scene parser (core/scene.cpp:104-243) and camera
// construction (core/camera.cpp:8-30).  Host code only; compiled without FMA
// contraction so the camera basis rounds exactly like the reference's.
#include "engine.h"

#include <charconv>
#include <cmath>
#include <cstring>
#include <map>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <string>
#include <thread>
#include <utility>

using ramlt_b200::EngineBase;
using ramlt_b200::HostScene;

struct ramlt_gpu {
    std::unique_ptr<EngineBase> eng;
    std::string err;
};

struct ramlt_scene {
    HostScene hs;
    ramlt_scene_desc desc;
};

namespace ramlt_b200 {

namespace {
inline void sub3(const double *a, const double *b, double *o) {
    o[0] = a[0] - b[0];
    o[1] = a[1] - b[1];
    o[2] = a[2] - b[2];
}
inline double dot3(const double *a, const double *b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }
inline void cross3(const double *a, const double *b, double *o) {
    o[0] = a[1] * b[2] - a[2] * b[1];
    o[1] = a[2] * b[0] - a[0] * b[2];
    o[2] = a[0] * b[1] - a[1] * b[0];
}
inline void unit3(const double *a, double *o) {
    double l = std::sqrt(dot3(a, a));
    o[0] = a[0] / l;
    o[1] = a[1] / l;
    o[2] = a[2] / l;
}
}  // namespace

CameraBasis make_camera(const double cam[10], int width, int height) {
    // Camera::Camera (core/camera.cpp:8-20)
    double fov = cam[9];
    if (!(fov > 0.0 && fov < 180.0))
        throw std::invalid_argument("camera: fov must be in (0, 180) degrees");
    CameraBasis c;
    double d[3], r[3];
    std::memcpy(c.pos, cam, sizeof(c.pos));
    sub3(cam + 3, cam, d);
    unit3(d, c.fwd);
    cross3(c.fwd, cam + 6, r);
    if (std::sqrt(dot3(r, r)) < 1e-12)
        throw std::invalid_argument("camera: up vector is parallel to the view direction");
    unit3(r, c.right);
    cross3(c.right, c.fwd, c.up);
    c.tanh = std::tan(0.5 * fov * 3.14159265358979323846 / 180.0);
    // configure_image (core/camera.cpp:22-30)
    if (width < 1 || height < 1)
        throw std::invalid_argument("camera: resolution must be positive");
    c.aspect = static_cast<double>(width) / static_cast<double>(height);
    c.area = 4.0 * c.tanh * c.tanh * c.aspect;
    c.sensor = static_cast<double>(width) * static_cast<double>(height) / c.area;
    return c;
}

// Fast path for the bulk records ("tri", "sphere"): whitespace-separated
// tokens with std::from_chars, which rounds exactly like the stream's strtod.
// Anything unusual (a '+' sign, a token from_chars does not consume whole,
// out-of-range values, missing tokens) returns false and the line goes
// through the istringstream path, so results and errors match the reference.
namespace {
inline bool is_ws(char c) { return c == ' ' || c == '\t' || c == '\n' || c == '\v' || c == '\f' || c == '\r'; }
struct Tok {
    const char *p, *e;
    bool next(const char *&b, const char *&t) {
        while (p < e && is_ws(*p))
            ++p;
        if (p == e)
            return false;
        b = p;
        while (p < e && !is_ws(*p))
            ++p;
        t = p;
        return true;
    }
    bool num(double &x) {
        const char *b, *t;
        if (!next(b, t) || *b == '+')
            return false;
        for (const char *c = b; c < t; ++c)   // plain decimal only (no inf/nan/hex)
            if (!((*c >= '0' && *c <= '9') || *c == '.' || *c == 'e' || *c == 'E' || *c == '-' || *c == '+'))
                return false;
        auto r = std::from_chars(b, t, x);
        return r.ec == std::errc() && r.ptr == t;
    }
};
}  // namespace

// Bulk records pre-parsed per text chunk (phase 1, one thread per chunk): the
// numbers of every "tri" / "sphere" line the fast path accepts, the span of its
// material token, and every other non-blank line as a `slow` record.  Phase 2
// walks the records in file order on one thread -- material ids, emitter order
// and error line numbers depend on everything before a line -- and sends slow
// records through the istringstream path.
namespace {
struct PreRec {
    const char *lb, *eol;    // the line
    const char *mb, *me;     // material token (kind 1, 2)
    int ln;                  // line number within the chunk (1-based)
    int kind;                // 0 slow, 1 tri, 2 sphere
    double v[9];
};
struct PreChunk {
    std::vector<PreRec> recs;
    int lines = 0;
};
void pre_parse(const char *cur, const char *end, PreChunk &out) {
    int ln = 0;
    while (cur < end) {
        const char *eol = static_cast<const char *>(std::memchr(cur, '\n', static_cast<size_t>(end - cur)));
        if (!eol)
            eol = end;
        const char *lb = cur;
        cur = eol < end ? eol + 1 : end;
        ++ln;
        const char *q = lb;
        while (q < eol && (*q == ' ' || *q == '\t' || *q == '\r'))
            ++q;
        if (q == eol || *q == '#')
            continue;
        PreRec r;
        r.lb = lb, r.eol = eol, r.mb = r.me = nullptr, r.ln = ln, r.kind = 0;
        Tok tk{q, eol};
        const char *tb = q, *te = q;
        tk.next(tb, te);
        std::string_view tg(tb, static_cast<size_t>(te - tb));
        if (tg == "tri") {
            bool ok = true;
            for (int k = 0; k < 9; ++k)
                ok = ok && tk.num(r.v[k]);
            if (ok && tk.next(r.mb, r.me))
                r.kind = 1;
        } else if (tg == "sphere") {
            bool ok = tk.num(r.v[0]) && tk.num(r.v[1]) && tk.num(r.v[2]) && tk.num(r.v[3]);
            if (ok && r.v[3] > 0.0 && tk.next(r.mb, r.me))
                r.kind = 2;
        }
        out.recs.push_back(r);
    }
    out.lines = ln;
}
}  // namespace

// parse_scene mirror (core/scene.cpp:104-234): same grammar, same messages.
static HostScene parse_scene(const std::string &text, const std::string &origin) {
    HostScene s;
    std::map<std::string, int> ids;
    bool have_camera = false;
    std::vector<std::pair<bool, int>> order;
    std::string line;
    auto fail = [&](int l, const std::string &msg) {
        throw std::runtime_error(origin + ":" + std::to_string(l) + ": " + msg);
    };
    // phase 1: chunks cut at line ends, pre-parsed in parallel above 4 MB of text
    const char *t0 = text.data(), *t1 = text.data() + text.size();
    unsigned nchunk = 1;
    if (text.size() >= (size_t(4) << 20))
        nchunk = std::min(64u, std::max(1u, std::thread::hardware_concurrency()));
    std::vector<const char *> cut(nchunk + 1, t1);
    cut[0] = t0;
    for (unsigned i = 1; i < nchunk; ++i) {
        const char *p = t0 + text.size() / nchunk * i;
        if (p < cut[i - 1])
            p = cut[i - 1];
        const char *nl = static_cast<const char *>(std::memchr(p, '\n', static_cast<size_t>(t1 - p)));
        cut[i] = nl ? nl + 1 : t1;
    }
    std::vector<PreChunk> chunks(nchunk);
    if (nchunk == 1) {
        pre_parse(cut[0], cut[1], chunks[0]);
    } else {
        std::vector<std::thread> pool;
        for (unsigned i = 0; i < nchunk; ++i)
            pool.emplace_back([&, i] {
                chunks[i].recs.reserve(static_cast<size_t>(cut[i + 1] - cut[i]) / 64 + 16);
                pre_parse(cut[i], cut[i + 1], chunks[i]);
            });
        for (auto &th : pool)
            th.join();
    }
    size_t nrec = 0;
    for (const PreChunk &ch : chunks)
        nrec += ch.recs.size();
    s.tri.reserve(nrec);
    order.reserve(nrec);
    // phase 2: file order
    std::string_view last_name;   // the previous bulk record's material (names never rebind)
    int last_id = -1;
    auto lookup = [&](const char *mb, const char *me) {
        std::string_view nm(mb, static_cast<size_t>(me - mb));
        if (last_id >= 0 && nm == last_name)
            return last_id;
        auto it = ids.find(std::string(nm));
        if (it == ids.end())
            return -1;
        last_name = nm;
        last_id = it->second;
        return last_id;
    };
    int ln_base = 0;
    for (const PreChunk &ch : chunks) {
      for (const PreRec &r : ch.recs) {
        const int ln = ln_base + r.ln;
        const char *lb = r.lb, *eol = r.eol;
        if (r.kind == 1) {
            const int id = lookup(r.mb, r.me);
            if (id >= 0) {
                ramlt_triangle t{};
                std::memcpy(t.a, r.v, 3 * sizeof(double));
                std::memcpy(t.b, r.v + 3, 3 * sizeof(double));
                std::memcpy(t.c, r.v + 6, 3 * sizeof(double));
                t.material = id;
                t.emitter = -1;
                order.emplace_back(false, static_cast<int>(s.tri.size()));
                s.tri.push_back(t);
                continue;
            }
        } else if (r.kind == 2) {
            const int id = lookup(r.mb, r.me);
            if (id >= 0) {
                ramlt_sphere sp{};
                std::memcpy(sp.center, r.v, 3 * sizeof(double));
                sp.radius = r.v[3];
                sp.material = id;
                sp.emitter = -1;
                order.emplace_back(true, static_cast<int>(s.sph.size()));
                s.sph.push_back(sp);
                continue;
            }
        }
        line.assign(lb, static_cast<size_t>(eol - lb));
        std::istringstream ls(line);
        std::string tag;
        ls >> tag;
        auto check = [&] {
            if (ls.fail())
                fail(ln, "malformed '" + tag + "' record");
        };
        auto mat_id = [&](const std::string &name) {
            auto it = ids.find(name);
            if (it == ids.end())
                fail(ln, "unknown material '" + name + "'");
            return it->second;
        };
        if (tag == "camera") {
            double v[10];
            for (double &x : v)
                ls >> x;
            check();
            try {
                make_camera(v, 1, 1);
            } catch (const std::exception &e) {
                fail(ln, e.what());
            }
            std::memcpy(s.cam, v, sizeof(v));
            have_camera = true;
        } else if (tag == "material") {
            std::string name, kind;
            ls >> name >> kind;
            check();
            ramlt_material m{};
            m.albedo[0] = m.albedo[1] = m.albedo[2] = 0.5;
            m.ior = 1.5;
            m.exponent = 32.0;
            if (kind == "diffuse") {
                m.kind = RAMLT_DIFFUSE;
                ls >> m.albedo[0] >> m.albedo[1] >> m.albedo[2];
                check();
            } else if (kind == "mirror") {
                m.kind = RAMLT_MIRROR;
                ls >> m.albedo[0] >> m.albedo[1] >> m.albedo[2];
                check();
            } else if (kind == "dielectric") {
                m.kind = RAMLT_DIELECTRIC;
                ls >> m.ior >> m.albedo[0] >> m.albedo[1] >> m.albedo[2];
                check();
                if (m.ior <= 1.0)
                    fail(ln, "dielectric ior must be > 1");
            } else if (kind == "glossy") {
                m.kind = RAMLT_GLOSSY;
                ls >> m.albedo[0] >> m.albedo[1] >> m.albedo[2] >> m.exponent;
                check();
                if (m.exponent <= 0.0)
                    fail(ln, "glossy exponent must be > 0");
            } else {
                fail(ln, "unknown material kind '" + kind + "'");
            }
            if (m.kind != RAMLT_DIELECTRIC)
                for (int c = 0; c < 3; ++c)
                    if (m.albedo[c] < 0.0 || m.albedo[c] > 1.0)
                        fail(ln, "albedo components must be in [0,1]");
            if (ids.count(name))
                fail(ln, "duplicate material '" + name + "'");
            ids[name] = static_cast<int>(s.mats.size());
            s.mats.push_back(m);
        } else if (tag == "sphere") {
            ramlt_sphere sp{};
            std::string mat;
            ls >> sp.center[0] >> sp.center[1] >> sp.center[2] >> sp.radius >> mat;
            check();
            if (sp.radius <= 0.0)
                fail(ln, "sphere radius must be > 0");
            sp.material = mat_id(mat);
            sp.emitter = -1;
            order.emplace_back(true, static_cast<int>(s.sph.size()));
            s.sph.push_back(sp);
        } else if (tag == "tri") {
            ramlt_triangle t{};
            std::string mat;
            ls >> t.a[0] >> t.a[1] >> t.a[2] >> t.b[0] >> t.b[1] >> t.b[2] >> t.c[0] >> t.c[1] >> t.c[2] >> mat;
            check();
            t.material = mat_id(mat);
            t.emitter = -1;
            order.emplace_back(false, static_cast<int>(s.tri.size()));
            s.tri.push_back(t);
        } else if (tag == "emitter") {
            int index;
            double r[3];
            ls >> index >> r[0] >> r[1] >> r[2];
            check();
            if (index < 0 || index >= static_cast<int>(order.size()))
                fail(ln, "emitter geometry index out of range");
            if (r[0] < 0.0 || r[1] < 0.0 || r[2] < 0.0)
                fail(ln, "emitted radiance must be non-negative");
            int e = static_cast<int>(s.emit.size() / 3);
            s.emit.insert(s.emit.end(), r, r + 3);
            auto [is_sphere, gi] = order[index];
            if (is_sphere)
                s.sph[gi].emitter = e;
            else
                s.tri[gi].emitter = e;
        } else {
            fail(ln, "unknown record '" + tag + "'");
        }
      }
      ln_base += ch.lines;
    }
    if (!have_camera)
        throw std::runtime_error(origin + ": scene has no camera");
    if (s.emit.empty())
        throw std::runtime_error(origin + ": scene has no emitter");
    return s;
}

static HostScene from_desc(const ramlt_scene_desc *d) {
    HostScene s;
    std::memcpy(s.cam, d->cam_position, 3 * sizeof(double));
    std::memcpy(s.cam + 3, d->cam_look_at, 3 * sizeof(double));
    std::memcpy(s.cam + 6, d->cam_up, 3 * sizeof(double));
    s.cam[9] = d->cam_fov_deg;
    s.mats.assign(d->materials, d->materials + d->n_materials);
    s.sph.assign(d->spheres, d->spheres + d->n_spheres);
    s.tri.assign(d->triangles, d->triangles + d->n_triangles);
    s.emit.assign(d->emitter_radiance, d->emitter_radiance + 3 * d->n_emitters);
    if (s.emit.empty())
        throw std::runtime_error("scene has no emitter");
    for (auto &t : s.tri)
        if (t.material < 0 || t.material >= d->n_materials || t.emitter >= d->n_emitters)
            throw std::invalid_argument("triangle references an unknown material or emitter");
    for (auto &sp : s.sph)
        if (sp.material < 0 || sp.material >= d->n_materials || sp.emitter >= d->n_emitters)
            throw std::invalid_argument("sphere references an unknown material or emitter");
    return s;
}

}  // namespace ramlt_b200

namespace {

thread_local std::string g_create_err;

template <class F> int guard(std::string &err, F &&f) {
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

ramlt_b200::EngineBase *make(const HostScene &hs, const ramlt_render_desc *d) {
    if (!d)
        throw std::logic_error("null render descriptor");
    if (d->precision == RAMLT_F64)
        return ramlt_b200::make_engine_f64(hs, *d);
    if (d->precision == RAMLT_F32)
        return ramlt_b200::make_engine_f32(hs, *d);
    throw std::invalid_argument("precision must be RAMLT_F32 or RAMLT_F64");
}

}  // namespace

extern "C" {

int ramlt_gpu_abi_version(void) { return RAMLT_GPU_ABI_VERSION; }

void ramlt_gpu_default_desc(ramlt_render_desc *d) {
    std::memset(d, 0, sizeof(*d));
    // RenderConfig defaults (core/driver.hpp:19-39), AdaptationConfig (adaptation.hpp:14-22)
    d->strategy = RAMLT_RA_QUADTREE;
    d->perturbation = RAMLT_LENS;
    d->mutations = 1000000;
    d->time_budget_s = 0.0;
    d->chains = 1;
    d->batch_size = 10;
    d->gamma_max = 1.0;
    d->gamma_scale = 5.0;
    d->target_acceptance = 0.5;
    d->lambda_init = 1.0;
    d->lambda_min = -30.0;
    d->sigma2_ratio = 1.0;
    d->n_top = 20;
    d->n_bottom = 50;
    d->m_split = 5000;
    d->m_refine = 10000000;
    d->b_samples = 1000000;
    d->seed = 1;
    d->width = 256;
    d->height = 256;
    d->max_vertices = 20;
    d->metrics_interval = 1000000;
    d->precision = RAMLT_F32;
    d->rng = RAMLT_RNG_PHILOX;
    d->adapt_mode = RAMLT_ADAPT_AUTO;
    d->lanes_per_chain = 0;
    d->device = -1;
}

int ramlt_scene_parse(const char *text, const char *origin, ramlt_scene **out) {
    return guard(g_create_err, [&] {
        auto sc = std::make_unique<ramlt_scene>();
        sc->hs = ramlt_b200::parse_scene(text ? text : "", origin ? origin : "<string>");
        ramlt_scene_desc &d = sc->desc;
        std::memset(&d, 0, sizeof(d));
        std::memcpy(d.cam_position, sc->hs.cam, 3 * sizeof(double));
        std::memcpy(d.cam_look_at, sc->hs.cam + 3, 3 * sizeof(double));
        std::memcpy(d.cam_up, sc->hs.cam + 6, 3 * sizeof(double));
        d.cam_fov_deg = sc->hs.cam[9];
        d.n_materials = static_cast<int32_t>(sc->hs.mats.size());
        d.n_spheres = static_cast<int32_t>(sc->hs.sph.size());
        d.n_triangles = static_cast<int32_t>(sc->hs.tri.size());
        d.n_emitters = static_cast<int32_t>(sc->hs.emit.size() / 3);
        d.materials = sc->hs.mats.data();
        d.spheres = sc->hs.sph.data();
        d.triangles = sc->hs.tri.data();
        d.emitter_radiance = sc->hs.emit.data();
        *out = sc.release();
    });
}

const ramlt_scene_desc *ramlt_scene_get_desc(const ramlt_scene *s) { return s ? &s->desc : nullptr; }
void ramlt_scene_free(ramlt_scene *s) { delete s; }

int ramlt_gpu_create(const ramlt_scene_desc *scene, const ramlt_render_desc *desc, ramlt_gpu **out) {
    return guard(g_create_err, [&] {
        if (!scene)
            throw std::logic_error("null scene descriptor");
        HostScene hs = ramlt_b200::from_desc(scene);
        auto h = std::make_unique<ramlt_gpu>();
        h->eng.reset(make(hs, desc));
        *out = h.release();
    });
}

int ramlt_gpu_create_from_text(const char *text, const char *origin, const ramlt_render_desc *desc,
                               ramlt_gpu **out) {
    return guard(g_create_err, [&] {
        HostScene hs = ramlt_b200::parse_scene(text ? text : "", origin ? origin : "<string>");
        auto h = std::make_unique<ramlt_gpu>();
        h->eng.reset(make(hs, desc));
        *out = h.release();
    });
}

int ramlt_gpu_create_multi(const ramlt_scene_desc *scene, const ramlt_render_desc *desc, int32_t n_dev,
                           const int32_t *devs, uint32_t film_sync_steps, ramlt_gpu **out) {
    return guard(g_create_err, [&] {
        if (!scene || !desc)
            throw std::logic_error("null scene or render descriptor");
        HostScene hs = ramlt_b200::from_desc(scene);
        auto h = std::make_unique<ramlt_gpu>();
        h->eng.reset(ramlt_b200::make_engine_multi(hs, *desc, n_dev, devs, film_sync_steps));
        *out = h.release();
    });
}

int ramlt_gpu_create_multi_from_text(const char *text, const char *origin, const ramlt_render_desc *desc,
                                     int32_t n_dev, const int32_t *devs, uint32_t film_sync_steps, ramlt_gpu **out) {
    return guard(g_create_err, [&] {
        if (!desc)
            throw std::logic_error("null render descriptor");
        HostScene hs = ramlt_b200::parse_scene(text ? text : "", origin ? origin : "<string>");
        auto h = std::make_unique<ramlt_gpu>();
        h->eng.reset(ramlt_b200::make_engine_multi(hs, *desc, n_dev, devs, film_sync_steps));
        *out = h.release();
    });
}

const char *ramlt_gpu_last_create_error(void) { return g_create_err.c_str(); }

#define RAMLT_H(body)                                                                              \
    do {                                                                                           \
        if (!h)                                                                                    \
            return RAMLT_E_LOGIC;                                                                  \
        return guard(h->err, [&] { body; });                                                       \
    } while (0)

int ramlt_gpu_estimate_b(ramlt_gpu *h, double *b, double *se) { RAMLT_H(h->eng->estimate_b(b, se)); }
int ramlt_gpu_estimate_b_partials(ramlt_gpu *h, uint64_t begin, uint64_t end, double *out) {
    RAMLT_H(h->eng->estimate_b_partials(begin, end, out));
}
int ramlt_gpu_reduce_b(ramlt_gpu *h, const double *p, uint64_t n, double *b, double *se) {
    RAMLT_H(h->eng->reduce_b(p, n, b, se));
}
int ramlt_gpu_set_b(ramlt_gpu *h, double b) { RAMLT_H(h->eng->set_b(b)); }
int ramlt_gpu_init_chains(ramlt_gpu *h) { RAMLT_H(h->eng->init_chains()); }
int ramlt_gpu_run(ramlt_gpu *h, uint64_t m) { RAMLT_H(h->eng->run(m)); }
int ramlt_gpu_run_steps(ramlt_gpu *h, uint32_t n, uint64_t *done, uint32_t *executed) {
    RAMLT_H(uint64_t d = h->eng->run_steps(n, executed); if (done) *done = d);
}
int ramlt_gpu_render(ramlt_gpu *h) { RAMLT_H(h->eng->render()); }
int ramlt_gpu_synchronize(ramlt_gpu *h) { RAMLT_H(h->eng->synchronize()); }
int ramlt_gpu_read_stats(ramlt_gpu *h, ramlt_stats *o) { RAMLT_H(h->eng->read_stats(o)); }
int ramlt_gpu_read_film(ramlt_gpu *h, double *rgb, double *lum) { RAMLT_H(h->eng->read_film(rgb, lum)); }
int ramlt_gpu_read_image(ramlt_gpu *h, float *rgb) { RAMLT_H(h->eng->read_image(rgb)); }
int ramlt_gpu_read_tallies(ramlt_gpu *h, double *a, uint64_t *v, uint64_t cap, uint64_t *n) {
    RAMLT_H(uint64_t m = h->eng->read_tallies(a, v, cap); if (n) *n = m);
}
int ramlt_gpu_read_regions(ramlt_gpu *h, double *l, uint64_t *nn, uint64_t cap, uint64_t *count) {
    RAMLT_H(uint64_t m = h->eng->read_regions(l, nn, cap); if (count) *count = m);
}
int ramlt_gpu_read_trace(ramlt_gpu *h, ramlt_trace_row *rows, uint64_t cap, uint64_t *n) {
    RAMLT_H(uint64_t m = h->eng->read_trace(rows, cap); if (n) *n = m);
}
int ramlt_gpu_read_metrics(ramlt_gpu *h, double *rows, uint64_t cap, uint64_t *n) {
    RAMLT_H(uint64_t m = h->eng->read_metrics(rows, cap); if (n) *n = m);
}
int ramlt_gpu_read_decisions(ramlt_gpu *h, uint32_t K, double *a, uint8_t *f) {
    RAMLT_H(h->eng->read_decisions(K, a, f));
}
int ramlt_gpu_read_chain_lengths(ramlt_gpu *h, int32_t *k) { RAMLT_H(h->eng->read_chain_lengths(k)); }
int ramlt_gpu_read_partition_visits(ramlt_gpu *h, const uint64_t *visits, uint64_t n, char *buf, uint64_t cap) {
    RAMLT_H(std::string s = h->eng->read_partition_visits(visits, n); if (buf && cap) {
        std::strncpy(buf, s.c_str(), cap - 1);
        buf[cap - 1] = '\0';
    });
}
int ramlt_gpu_read_partition(ramlt_gpu *h, char *buf, uint64_t cap) {
    RAMLT_H(std::string s = h->eng->read_partition(); if (buf && cap) {
        std::strncpy(buf, s.c_str(), cap - 1);
        buf[cap - 1] = '\0';
    });
}
int ramlt_gpu_set_stream(ramlt_gpu *h, void *stream) { RAMLT_H(h->eng->set_stream(stream)); }
int ramlt_gpu_film_device(ramlt_gpu *h, double **film, uint64_t *n) { RAMLT_H(h->eng->film_device(film, n)); }
int ramlt_gpu_adapt_exchange(ramlt_gpu *h, uint64_t **c, uint64_t **fx, uint64_t **last, uint64_t *n) {
    RAMLT_H(h->eng->adapt_exchange(c, fx, last, n));
}
int ramlt_gpu_adapt_apply(ramlt_gpu *h) { RAMLT_H(h->eng->adapt_apply()); }
int ramlt_gpu_set_exchange_interval(ramlt_gpu *h, uint32_t s) { RAMLT_H(h->eng->set_exchange_interval(s)); }
int ramlt_gpu_visits_device(ramlt_gpu *h, uint64_t **v, uint64_t *n) { RAMLT_H(h->eng->visits_device(v, n)); }
int ramlt_gpu_refine_pending(ramlt_gpu *h, int32_t *p) { RAMLT_H(*p = h->eng->refine_pending() ? 1 : 0); }
int ramlt_gpu_refine(ramlt_gpu *h, int32_t keep) { RAMLT_H(h->eng->refine_now(keep != 0)); }
int ramlt_gpu_set_reference(ramlt_gpu *h, const float *rgb, int32_t w, int32_t ht) {
    RAMLT_H(h->eng->set_reference(rgb, w, ht));
}
int ramlt_gpu_rrmse(ramlt_gpu *h, uint64_t at, double *out) { RAMLT_H(*out = h->eng->rrmse(at)); }
int ramlt_gpu_trace_benchmark(ramlt_gpu *h, uint64_t n, double *ms, uint64_t *hits) {
    RAMLT_H(h->eng->trace_benchmark(n, ms, hits));
}

const char *ramlt_gpu_last_error(ramlt_gpu *h) { return h ? h->err.c_str() : g_create_err.c_str(); }
void ramlt_gpu_destroy(ramlt_gpu *h) { delete h; }

}  // extern "C"
