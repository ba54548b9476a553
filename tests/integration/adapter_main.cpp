// Compile/link check of include/ramlt_b200_adapter.hpp inside the reference's
// include tree: the reference's own types flow through the C-ABI.
#include "driver.hpp"
#include "scene.hpp"
#include "ramlt_b200_adapter.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <fstream>
#include <sstream>

int main(int argc, char **argv) {
    if (argc < 2)
        return 2;
    std::ifstream f(argv[1]);
    std::stringstream ss;
    ss << f.rdbuf();
    ramlt::RenderConfig cfg;
    cfg.strategy = ramlt::StrategyVariant::Fixed;
    cfg.chains = 16;
    cfg.mutations = 16 * 64;
    cfg.width = cfg.height = 32;
    cfg.max_vertices = 9;
    cfg.b_samples = 4096;
    ramlt_b200::Options opt;
    opt.precision = RAMLT_F64;
    opt.rng = RAMLT_RNG_PCG32;
    ramlt::RenderResult gpu = ramlt_b200::run_render<ramlt::RenderResult>(ss.str(), cfg, opt);
    ramlt::RenderResult cpu = ramlt::run_render(ramlt::parse_scene(ss.str()), cfg);
    std::printf("gpu acc=%.6f lum=%.3f  cpu acc=%.6f lum=%.3f  b gpu=%.4f cpu=%.4f\n", gpu.mean_acceptance,
                gpu.film_luminance, cpu.mean_acceptance, cpu.film_luminance, gpu.b.b, cpu.b.b);
    // Fixed strategy, reference PCG streams, fp64: identical decisions; only the
    // cross-chain summation order of the mean differs.
    double rel = std::abs(gpu.mean_acceptance - cpu.mean_acceptance) / std::max(cpu.mean_acceptance, 1e-300);
    bool ok = rel < 1e-12 && gpu.total_mutations == cpu.total_mutations;
    // the same call over two shards of one handle (Options::devices; two shards on
    // device 0 stand in for two GPUs) with RenderConfig::reference set: identical
    // decisions, and every metrics row carries the rRMSE against the reference image
    ramlt::RenderConfig cfg2 = cfg;
    cfg2.metrics_interval = 16 * 16;
    cfg2.reference = &cpu.image;
    ramlt_b200::Options opt2 = opt;
    opt2.devices = {0, 0};
    ramlt::RenderResult multi = ramlt_b200::run_render<ramlt::RenderResult>(ss.str(), cfg2, opt2);
    double rel2 = std::abs(multi.mean_acceptance - cpu.mean_acceptance) / std::max(cpu.mean_acceptance, 1e-300);
    bool rows = !multi.metrics.empty();
    for (const auto &m : multi.metrics)
        rows = rows && std::isfinite(m.rrmse);
    std::printf("multi-device acc=%.6f rows=%zu last rrmse=%.4f\n", multi.mean_acceptance, multi.metrics.size(),
                multi.metrics.empty() ? -1.0 : multi.metrics.back().rrmse);
    ok = ok && rel2 < 1e-12 && multi.total_mutations == cpu.total_mutations && rows;
    return ok ? 0 : 1;
}
