// fo_step_sgd_extra.cu -- the sgd step's optional-layout and device-scalar
// (capturable) kernel instances (fo_step_impl.cuh, FO_DEFINE_EXTRA), in their
// own translation unit so they compile in parallel with fo_step_sgd.cu.
#define FO_DEFINE_EXTRA
#include "fo_step_impl.cuh"

namespace fo {

FO_INSTANTIATE_EXTRA(FO_OPT_SGD)

}  // namespace fo
