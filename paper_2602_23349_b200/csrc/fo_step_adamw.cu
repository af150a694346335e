// fo_step_adamw.cu -- instantiates the fused adamw step (fo_step_impl.cuh).
#include "fo_step_impl.cuh"

namespace fo {

int step_adamw(const fo_tensor* ts, int32_t nt, const fo_hparams* hps, int32_t nhp, int grad_dtype, int rho_bits,
             int32_t G, int var_scheme, uint32_t* d_err, cudaStream_t s, const DevScalars* dev) {
  return grad_dtype == FO_GRAD_BF16
             ? step_mt_typed<FO_OPT_ADAMW, __nv_bfloat16>(ts, nt, hps, nhp, rho_bits, G, var_scheme, d_err, s, dev)
             : step_mt_typed<FO_OPT_ADAMW, float>(ts, nt, hps, nhp, rho_bits, G, var_scheme, d_err, s, dev);
}

int64_t fused_tile_elems() { return WS_CT; }

// Bitmap words one fused launch (per FO_MT_MAX_TENSORS block) needs: the
// launcher's 2^fix_shift words for its slice count.
int64_t fix_words_for(const fo_tensor* ts, int32_t nt) {
  int64_t words = 1;
  for (int32_t off = 0; off < nt; off += FO_MT_MAX_TENSORS) {
    uint64_t slices = 0;
    for (int32_t q = off; q < std::min<int32_t>(nt, off + FO_MT_MAX_TENSORS); ++q)
      slices += (uint64_t)((ts[q].n + WS_CT - 1) / WS_CT) * WS_NCW;
    int64_t w = 1;
    while ((uint64_t)(32 * w) < slices) w <<= 1;
    words = std::max(words, w);
  }
  return words;
}

}  // namespace fo
