// fo_api.cu -- the extern "C" boundary (include/flashoptim_b200.h).
// Argument validation happens here, synchronously, before anything is
// enqueued; everything else is stream-ordered on the caller's stream.
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>

#include "fo_internal.h"

namespace {

cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

const char* kMsg[8] = {
    "gradient-nonfinite: gradient contains NaN/Inf",                 // optim.py:183
    "invalid-correction-code: asymmetric minimum is forbidden",      // formats.py:271
    "split-nonfinite: cannot split NaN/Inf master weights",          // formats.py:243
    "quantize-nonfinite: state buffer contains NaN/Inf",             // quantize.py:69
    "scale-overflow: group absmax exceeds FP16 range",               // quantize.py:85
    "quantize-nonfinite: state buffer contains NaN/Inf",             // quantize.py:69
    "negative-variance: variance entries must be >= 0",              // quantize.py:144
    "scale-overflow: group absmax exceeds FP16 range",               // quantize.py:85
};

int check_opt(int opt) { return (opt == FO_OPT_SGD || opt == FO_OPT_ADAMW || opt == FO_OPT_LION) ? 0 : FO_EINVAL; }

}  // namespace

extern "C" {

uint32_t fo_abi_version(void) { return FO_ABI_VERSION; }

const char* fo_status_string(int status) {
  switch (status) {
    case FO_OK: return "ok";
    case FO_EINVAL: return "invalid argument";
    case FO_EUNSUPPORTED: return "unsupported layout";
    case FO_ETOOMANY: return "too many hyper-parameter sets";
    default: return status > 0 ? cudaGetErrorString((cudaError_t)status) : "unknown status";
  }
}

const char* fo_error_message(uint32_t mask, int optimizer) {
  // Program order of each reference step: the first failing stage raises.
  static const uint32_t adamw[] = {FO_ERR_GRAD_NONFINITE, FO_ERR_RHO_INVALID, FO_ERR_SPLIT_NONFINITE,
                                   FO_ERR_M_NONFINITE,    FO_ERR_M_OVERFLOW,  FO_ERR_V_NONFINITE,
                                   FO_ERR_V_NEGATIVE,     FO_ERR_V_OVERFLOW};
  static const uint32_t sgd[] = {FO_ERR_GRAD_NONFINITE, FO_ERR_M_NONFINITE, FO_ERR_M_OVERFLOW, FO_ERR_RHO_INVALID,
                                 FO_ERR_SPLIT_NONFINITE};
  static const uint32_t lion[] = {FO_ERR_GRAD_NONFINITE, FO_ERR_RHO_INVALID, FO_ERR_SPLIT_NONFINITE,
                                  FO_ERR_M_NONFINITE, FO_ERR_M_OVERFLOW};
  const uint32_t* order = adamw;
  int count = 8;
  if (optimizer == FO_OPT_SGD) order = sgd, count = 5;
  if (optimizer == FO_OPT_LION) order = lion, count = 5;
  for (int i = 0; i < count; ++i)
    if (mask & order[i]) return kMsg[__builtin_ctz(order[i])];
  for (int b = 0; b < 8; ++b)
    if (mask & (1u << b)) return kMsg[b];
  return "";
}

void fo_make_hparams(int optimizer, double lr, double beta1, double beta2, double eps, double weight_decay,
                     double momentum, int64_t t, fo_hparams* out) {
  (void)optimizer;
  out->lr = (float)lr;
  out->wd = (float)weight_decay;
  out->eps = (float)eps;
  out->b1 = (float)beta1;
  out->omb1 = (float)(1.0 - beta1);
  out->b2 = (float)beta2;
  out->omb2 = (float)(1.0 - beta2);
  out->mu = (float)momentum;
  out->bc1 = (float)(1.0 - std::pow(beta1, (double)t));  // optim.py:212
  out->bc2 = (float)(1.0 - std::pow(beta2, (double)t));  // optim.py:213
  volatile float one = 1.0f;                                // f32 division: RN(1/bc)
  out->rbc1 = one / out->bc1;
  out->rbc2 = one / out->bc2;
}

int fo_step_mt(int optimizer, const fo_tensor* tensors, int32_t n_tensors, const fo_hparams* hparams,
               int32_t n_hparams, int grad_dtype, int rho_bits, int32_t group_size, int variance_scheme,
               uint32_t* d_err, void* stream) {
  if (check_opt(optimizer) || n_tensors < 0 || (n_tensors && !tensors) || !hparams || n_hparams < 1)
    return FO_EINVAL;
  if (n_hparams > FO_MAX_HPARAMS) return FO_ETOOMANY;
  if (grad_dtype != FO_GRAD_BF16 && grad_dtype != FO_GRAD_F32) return FO_EINVAL;
  if (rho_bits != 8 && rho_bits != 16) return FO_EINVAL;
  if (group_size < 1) return FO_EINVAL;
  if (variance_scheme != FO_VAR_COMPANDED && variance_scheme != FO_VAR_LINEAR) return FO_EINVAL;
  for (int32_t i = 0; i < n_tensors; ++i) {
    const fo_tensor& t = tensors[i];
    if (t.n < 0 || t.hp_index < 0 || t.hp_index >= n_hparams) return FO_EINVAL;
    if (t.n == 0) continue;
    if (!t.lp || !t.rho || !t.m_codes || !t.m_scales || !t.grad) return FO_EINVAL;
    if (optimizer == FO_OPT_ADAMW && (!t.v_codes || !t.v_scales)) return FO_EINVAL;
  }
  return fo::step_mt(optimizer, tensors, n_tensors, hparams, n_hparams, grad_dtype, rho_bits, group_size,
                     variance_scheme, d_err, as_stream(stream));
}

int fo_step_mt_dev(int optimizer, const fo_tensor* tensors, int32_t n_tensors, const fo_hparams* hparams,
                   const fo_dev_scalars* dev, int grad_dtype, uint32_t* d_err, void* stream) {
  if (!dev || !dev->step || dev->bc_len < 0 || (dev->bc_len > 0 && !dev->bc_table)) return FO_EINVAL;
  if (optimizer == FO_OPT_ADAMW && dev->bc_len < 2) return FO_EINVAL;
  for (int32_t i = 0; i < n_tensors; ++i)
    if (tensors && tensors[i].hp_index != 0) return FO_EINVAL;
  if (check_opt(optimizer) || n_tensors < 0 || (n_tensors && !tensors) || !hparams) return FO_EINVAL;
  if (grad_dtype != FO_GRAD_BF16 && grad_dtype != FO_GRAD_F32) return FO_EINVAL;
  for (int32_t i = 0; i < n_tensors; ++i) {
    const fo_tensor& t = tensors[i];
    if (t.n < 0) return FO_EINVAL;
    if (t.n == 0) continue;
    if (!t.lp || !t.rho || !t.m_codes || !t.m_scales || !t.grad) return FO_EINVAL;
    if (optimizer == FO_OPT_ADAMW && (!t.v_codes || !t.v_scales)) return FO_EINVAL;
  }
  // the fused tile's hyper-parameter ranges are checked on the first
  // (smallest) bias corrections of the run, t = 1
  // (bc at t = 1 is f32(1 - beta) = omb, fo_make_hparams; nothing is read
  // back from the device, so the call stays capturable)
  fo_hparams h = *hparams;
  if (optimizer == FO_OPT_ADAMW) {
    volatile float one = 1.0f;
    h.bc1 = h.omb1;
    h.bc2 = h.omb2;
    h.rbc1 = one / h.bc1;
    h.rbc2 = one / h.bc2;
  }
  if (!dev->fix_bits || dev->fix_words < fo::fix_words_for(tensors, n_tensors)) return FO_EINVAL;
  const fo::DevScalars ds{dev->step, dev->lr, dev->bc_table, dev->bc_len, dev->fix_bits, dev->fix_words,
                          dev->fix_count};
  return fo::step_mt(optimizer, tensors, n_tensors, &h, 1, grad_dtype, 8, 32, FO_VAR_COMPANDED, d_err,
                     as_stream(stream), &ds);
}

int fo_step_mt_peers(int optimizer, const fo_tensor* tensors, int32_t n_tensors, const fo_hparams* hparams,
                     int grad_dtype, const int64_t* peer_delta, int32_t n_peers, uint32_t* d_err, void* stream) {
  if (check_opt(optimizer) || n_tensors < 0 || (n_tensors && !tensors) || !hparams) return FO_EINVAL;
  if (n_peers < 0 || n_peers > FO_MAX_PEERS || (n_peers && !peer_delta)) return FO_EINVAL;
  if (grad_dtype != FO_GRAD_BF16 && grad_dtype != FO_GRAD_F32) return FO_EINVAL;
  for (int32_t i = 0; i < n_tensors; ++i) {
    const fo_tensor& t = tensors[i];
    if (t.n < 0 || t.hp_index != 0) return FO_EINVAL;
    if (t.n == 0) continue;
    if (!t.lp || !t.rho || !t.m_codes || !t.m_scales || !t.grad) return FO_EINVAL;
    if (optimizer == FO_OPT_ADAMW && (!t.v_codes || !t.v_scales)) return FO_EINVAL;
  }
  fo::DevScalars ds{};
  ds.npeers = n_peers;
  ds.peer_delta = peer_delta;
  return fo::step_mt(optimizer, tensors, n_tensors, hparams, 1, grad_dtype, 8, 32, FO_VAR_COMPANDED, d_err,
                     as_stream(stream), n_peers ? &ds : nullptr);
}

int fo_ipc_export(const void* ptr, void* handle64, int64_t* offset) {
  if (!ptr || !handle64 || !offset) return FO_EINVAL;
  // the allocation's base: cuMemGetAddressRange through the runtime's
  // driver entry point (no libcuda link)
  typedef int (*GetRange)(uintptr_t*, size_t*, uintptr_t);
  static GetRange get_range = nullptr;
  if (!get_range) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn)
      return (int)cudaErrorNotSupported;
    get_range = reinterpret_cast<GetRange>(fn);
  }
  uintptr_t base = 0;
  size_t size = 0;
  if (get_range(&base, &size, reinterpret_cast<uintptr_t>(ptr)) != 0) return (int)cudaErrorInvalidValue;
  cudaIpcMemHandle_t h;
  const cudaError_t rc = cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base));
  if (rc != cudaSuccess) return (int)rc;
  std::memcpy(handle64, &h, sizeof(h));
  *offset = (int64_t)(reinterpret_cast<uintptr_t>(ptr) - base);
  return 0;
}

int fo_ipc_open(const void* handle64, int64_t offset, void** ptr) {
  if (!handle64 || !ptr || offset < 0) return FO_EINVAL;
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle64, sizeof(h));
  void* base = nullptr;
  const cudaError_t rc = cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess);
  if (rc != cudaSuccess) return (int)rc;
  *ptr = static_cast<char*>(base) + offset;
  return 0;
}

int fo_ipc_close(void* ptr, int64_t offset) {
  if (!ptr || offset < 0) return FO_EINVAL;
  return (int)cudaIpcCloseMemHandle(static_cast<char*>(ptr) - offset);
}

int fo_bias_table(double beta1, double beta2, int32_t max_len, float* out, int32_t* len) {
  if (!len || max_len < 2 || !(beta1 >= 0.0 && beta1 < 1.0) || !(beta2 >= 0.0 && beta2 < 1.0)) return FO_EINVAL;
  int32_t n = 0;
  for (int64_t t = 0;; ++t) {
    if (t >= max_len) return FO_ETOOMANY;
    fo_hparams h;
    fo_make_hparams(FO_OPT_ADAMW, 1.0, beta1, beta2, 1.0, 0.0, 0.0, t, &h);
    if (out) {
      out[4 * t] = h.bc1;
      out[4 * t + 1] = h.rbc1;
      out[4 * t + 2] = h.bc2;
      out[4 * t + 3] = h.rbc2;
    }
    n = (int32_t)t + 1;
    if (t >= 1 && h.bc1 == 1.0f && h.bc2 == 1.0f) break;
  }
  *len = n;
  return 0;
}

int64_t fo_fused_tile_elems(void) { return fo::fused_tile_elems(); }

int64_t fo_fix_words(const fo_tensor* tensors, int32_t n_tensors) {
  if (n_tensors < 0 || (n_tensors && !tensors)) return FO_EINVAL;
  return fo::fix_words_for(tensors, n_tensors);
}

int fo_step_host(int optimizer, const fo_tensor* tensors, int32_t n_tensors, const fo_hparams* hparams,
                 int32_t n_hparams, int grad_dtype, int rho_bits, int32_t group_size, int variance_scheme,
                 int64_t chunk_elems, uint32_t* h_err) {
  if (check_opt(optimizer) || n_tensors < 0 || (n_tensors && !tensors) || !hparams || n_hparams < 1)
    return FO_EINVAL;
  if (n_hparams > FO_MAX_HPARAMS) return FO_ETOOMANY;
  if ((grad_dtype != FO_GRAD_BF16 && grad_dtype != FO_GRAD_F32) || (rho_bits != 8 && rho_bits != 16) ||
      group_size < 1 || (variance_scheme != FO_VAR_COMPANDED && variance_scheme != FO_VAR_LINEAR) || chunk_elems < 0)
    return FO_EINVAL;
  for (int32_t i = 0; i < n_tensors; ++i) {
    const fo_tensor& t = tensors[i];
    if (t.n < 0 || t.hp_index < 0 || t.hp_index >= n_hparams) return FO_EINVAL;
    if (t.n == 0) continue;
    if (!t.lp || !t.rho || !t.m_codes || !t.m_scales || !t.grad) return FO_EINVAL;
    if (optimizer == FO_OPT_ADAMW && (!t.v_codes || !t.v_scales)) return FO_EINVAL;
  }
  return fo::step_host(optimizer, tensors, n_tensors, hparams, n_hparams, grad_dtype, rho_bits, group_size,
                       variance_scheme, chunk_elems, h_err);
}

void fo_host_release(void) { fo::host_release(); }

int fo_fixup_stats(void* stream, uint64_t* flagged, uint64_t* slices, int reset) {
  return fo::fix_stats(as_stream(stream), flagged, slices, reset);
}

int fo_reserve(void* stream, int64_t max_elems) {
  if (max_elems < 0) return FO_EINVAL;
  return fo::fix_reserve(as_stream(stream), max_elems);
}

int fo_adamw_step(uint16_t* lp, int8_t* rho, int8_t* m_codes, uint16_t* m_scales, uint8_t* v_codes,
                  uint16_t* v_scales, const void* grad, int grad_dtype, int64_t n, const fo_hparams* hp,
                  uint32_t* d_err, void* stream) {
  fo_tensor t{lp, rho, m_codes, m_scales, v_codes, v_scales, grad, n, 0, 0};
  return fo_step_mt(FO_OPT_ADAMW, &t, 1, hp, 1, grad_dtype, 8, 32, FO_VAR_COMPANDED, d_err, stream);
}

int fo_sgd_step(uint16_t* lp, int8_t* rho, int8_t* m_codes, uint16_t* m_scales, const void* grad, int grad_dtype,
                int64_t n, const fo_hparams* hp, uint32_t* d_err, void* stream) {
  fo_tensor t{lp, rho, m_codes, m_scales, nullptr, nullptr, grad, n, 0, 0};
  return fo_step_mt(FO_OPT_SGD, &t, 1, hp, 1, grad_dtype, 8, 32, FO_VAR_COMPANDED, d_err, stream);
}

int fo_lion_step(uint16_t* lp, int8_t* rho, int8_t* m_codes, uint16_t* m_scales, const void* grad, int grad_dtype,
                 int64_t n, const fo_hparams* hp, uint32_t* d_err, void* stream) {
  fo_tensor t{lp, rho, m_codes, m_scales, nullptr, nullptr, grad, n, 0, 0};
  return fo_step_mt(FO_OPT_LION, &t, 1, hp, 1, grad_dtype, 8, 32, FO_VAR_COMPANDED, d_err, stream);
}

int fo_split(const float* theta, int64_t n, uint16_t* lp, void* rho, int rho_bits, uint32_t* d_err, void* stream) {
  if (n < 0 || (n && (!theta || !lp || !rho)) || (rho_bits != 8 && rho_bits != 16)) return FO_EINVAL;
  return fo::split(theta, n, lp, rho, rho_bits, d_err, as_stream(stream));
}

int fo_reconstruct(const uint16_t* lp, const void* rho, int rho_bits, int64_t n, float* out, uint32_t* d_err,
                   void* stream) {
  if (n < 0 || (n && (!lp || !rho || !out)) || (rho_bits != 8 && rho_bits != 16)) return FO_EINVAL;
  return fo::reconstruct(lp, rho, rho_bits, n, out, d_err, as_stream(stream));
}

int fo_quantize_momentum(const float* m, int64_t n, int32_t group_size, int8_t* codes, uint16_t* scales,
                         uint32_t* d_err, void* stream) {
  if (n < 0 || group_size < 1 || (n && (!m || !codes || !scales))) return FO_EINVAL;
  return fo::quantize(false, m, n, group_size, codes, scales, d_err, as_stream(stream));
}

int fo_dequantize_momentum(const int8_t* codes, const uint16_t* scales, int64_t n, int32_t group_size, float* out,
                           void* stream) {
  if (n < 0 || group_size < 1 || (n && (!codes || !scales || !out))) return FO_EINVAL;
  return fo::dequantize(false, codes, scales, n, group_size, out, as_stream(stream));
}

int fo_quantize_variance(const float* v, int64_t n, int32_t group_size, uint8_t* codes, uint16_t* scales,
                         uint32_t* d_err, void* stream) {
  if (n < 0 || group_size < 1 || (n && (!v || !codes || !scales))) return FO_EINVAL;
  return fo::quantize(true, v, n, group_size, codes, scales, d_err, as_stream(stream));
}

int fo_dequantize_variance(const uint8_t* codes, const uint16_t* scales, int64_t n, int32_t group_size, float* out,
                           void* stream) {
  if (n < 0 || group_size < 1 || (n && (!codes || !scales || !out))) return FO_EINVAL;
  return fo::dequantize(true, codes, scales, n, group_size, out, as_stream(stream));
}

int fo_selftest(int mode, uint64_t begin, uint64_t count, uint64_t* d_out, void* stream) {
  if (!d_out) return FO_EINVAL;
  return fo::selftest(mode, begin, count, reinterpret_cast<unsigned long long*>(d_out), as_stream(stream));
}

int fo_sweep(int block0, int nblocks, uint32_t scheme_mask, uint64_t* d_out, void* stream) {
  return fo::sweep(block0, nblocks, scheme_mask, d_out, as_stream(stream));
}

}  // extern "C"
