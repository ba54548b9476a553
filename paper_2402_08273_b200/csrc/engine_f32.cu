// Production build: fp32 arithmetic (FMA contraction on), fp64 lambda / film master.
#include <array>
#include "engine_impl.cuh"

namespace ramlt_b200 {
EngineBase *make_engine_f32(const HostScene &scene, const ramlt_render_desc &desc) {
    return new EngineT<float>(scene, desc);
}
}  // namespace ramlt_b200
