// Parity build of the analytic-target harness: fp64, -fmad=false (see engine_f64.cu).
#include "mix_impl.cuh"

namespace ramlt_b200 {
MixEngineBase *make_mix_engine_f64(const MixHostTarget &t, const ramlt_mix_desc &d) {
    return new MixEngineT<double>(t, d);
}
}  // namespace ramlt_b200
