// Production build of the analytic-target harness: fp32 arithmetic, fp64 lambda.
#include "mix_impl.cuh"

namespace ramlt_b200 {
MixEngineBase *make_mix_engine_f32(const MixHostTarget &t, const ramlt_mix_desc &d) {
    return new MixEngineT<float>(t, d);
}
}  // namespace ramlt_b200
