// fo_step_sgd.cu -- instantiates the fused sgd step (fo_step_impl.cuh).
#include "fo_step_impl.cuh"

namespace fo {

int step_sgd(const fo_tensor* ts, int32_t nt, const fo_hparams* hps, int32_t nhp, int grad_dtype, int rho_bits,
             int32_t G, int var_scheme, uint32_t* d_err, cudaStream_t s, const DevScalars* dev) {
  return grad_dtype == FO_GRAD_BF16
             ? step_mt_typed<FO_OPT_SGD, __nv_bfloat16>(ts, nt, hps, nhp, rho_bits, G, var_scheme, d_err, s, dev)
             : step_mt_typed<FO_OPT_SGD, float>(ts, nt, hps, nhp, rho_bits, G, var_scheme, d_err, s, dev);
}

}  // namespace fo
