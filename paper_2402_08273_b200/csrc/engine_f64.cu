// Parity build: fp64 arithmetic, compiled with -fmad=false so every
// expression rounds exactly like the reference's x86-64 doubles.
#include <array>
#include "engine_impl.cuh"

namespace ramlt_b200 {
EngineBase *make_engine_f64(const HostScene &scene, const ramlt_render_desc &desc) {
    return new EngineT<double>(scene, desc);
}
}  // namespace ramlt_b200
