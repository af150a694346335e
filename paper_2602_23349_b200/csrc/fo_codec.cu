// fo_codec.cu -- standalone device codecs: split / reconstruct
// (formats.py:232-276) and group-wise momentum / variance (de)quantization
// (quantize.py:109-158).  Used by init_flash_state (fp32 master weights ->
// bf16 + rho), state export (dequantized fp32 moments for inspection) and
// the exhaustive codec tests.  Grid-stride, one element (or one group) per
// thread; these run once per training job, not per step.
#include <cuda_runtime.h>

#include <algorithm>

#include "fo_internal.h"
#include "fo_math.cuh"

namespace fo {

static int blocks_for(int64_t work, int threads) {
  int64_t b = (work + threads - 1) / threads;
  return (int)std::max<int64_t>(1, std::min<int64_t>(b, 148 * 32));
}

template <int NCORR>
__global__ void split_kernel(const float* __restrict__ theta, int64_t n, uint16_t* __restrict__ lp, void* rho_,
                             uint32_t* err_out) {
  typedef typename std::conditional<NCORR == 127, int8_t, int16_t>::type RhoT;
  RhoT* rho = reinterpret_cast<RhoT*>(rho_);
  uint32_t err = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float x = theta[i];
    uint32_t code;
    int r;
    if (!finite(x)) {  // formats.py:242-243
      err |= FO_ERR_SPLIT_NONFINITE;
      code = (x != x) ? 0x7FC0u : bf16_rne(x);
      r = 0;
    } else {
      split1<NCORR>(x, code, r);
    }
    lp[i] = (uint16_t)code;
    rho[i] = (RhoT)r;
  }
  err = __reduce_or_sync(__activemask(), err);
  if (err && err_out) atomicOr(err_out, err);
}

template <int NCORR>
__global__ void reconstruct_kernel(const uint16_t* __restrict__ lp, const void* rho_, int64_t n,
                                   float* __restrict__ out, uint32_t* err_out) {
  typedef typename std::conditional<NCORR == 127, int8_t, int16_t>::type RhoT;
  const RhoT* rho = reinterpret_cast<const RhoT*>(rho_);
  uint32_t err = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)rho[i];
    if (r < -NCORR) err |= FO_ERR_RHO_INVALID;  // formats.py:270-271
    out[i] = reconstruct1(lp[i], r, __fdiv_rn((float)r, (float)NCORR));
  }
  err = __reduce_or_sync(__activemask(), err);
  if (err && err_out) atomicOr(err_out, err);
}

// quantize.py:109-122 (momentum) and :134-149 (variance), one group per thread.
template <bool VARIANCE>
__global__ void quantize_kernel(const float* __restrict__ x, int64_t n, int64_t G, void* codes_,
                                uint16_t* __restrict__ scales, uint32_t* err_out) {
  const int64_t ng = (n + G - 1) / G;
  uint32_t err = 0;
  const uint32_t nonfinite = VARIANCE ? FO_ERR_V_NONFINITE : FO_ERR_M_NONFINITE;
  const uint32_t overflow = VARIANCE ? FO_ERR_V_OVERFLOW : FO_ERR_M_OVERFLOW;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < ng; k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = k * G, e = min(n, b + G);
    float gmax = 0.0f;
    for (int64_t i = b; i < e; ++i) {
      float v = x[i];
      if (!finite(v)) err |= nonfinite;
      if (VARIANCE) {
        if (v < 0.0f) err |= FO_ERR_V_NEGATIVE;
        gmax = fmaxf(gmax, __fsqrt_rn(v));
      } else {
        gmax = fmaxf(gmax, fabsf(v));
      }
    }
    const uint32_t sb = scale_ru(gmax, err, overflow);
    const float s = half_bits_to_float(sb);
    const float den = s == 0.0f ? 1.0f : s;
    for (int64_t i = b; i < e; ++i) {
      if (VARIANCE)
        reinterpret_cast<uint8_t*>(codes_)[i] = (uint8_t)variance_code(__fdiv_rn(__fsqrt_rn(x[i]), den));
      else
        reinterpret_cast<int8_t*>(codes_)[i] = (int8_t)momentum_code(__fdiv_rn(x[i], den));
    }
    scales[k] = (uint16_t)sb;
  }
  err = __reduce_or_sync(__activemask(), err);
  if (err && err_out) atomicOr(err_out, err);
}

template <bool VARIANCE>
__global__ void dequantize_kernel(const void* codes_, const uint16_t* __restrict__ scales, int64_t n, int64_t G,
                                  float* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float s = half_bits_to_float(scales[i / G]);
    if (VARIANCE) {
      float r = __fmul_rn(variance_unit(reinterpret_cast<const uint8_t*>(codes_)[i]), s);  // quantize.py:156-157
      out[i] = __fmul_rn(r, r);                                                            // :158
    } else {
      out[i] = __fmul_rn(momentum_unit(reinterpret_cast<const int8_t*>(codes_)[i]), s);    // :129-131
    }
  }
}

int split(const float* theta, int64_t n, uint16_t* lp, void* rho, int rho_bits, uint32_t* d_err, cudaStream_t s) {
  if (n == 0) return 0;
  if (rho_bits == 8)
    split_kernel<127><<<blocks_for(n, 256), 256, 0, s>>>(theta, n, lp, rho, d_err);
  else
    split_kernel<32767><<<blocks_for(n, 256), 256, 0, s>>>(theta, n, lp, rho, d_err);
  return (int)cudaGetLastError();
}

int reconstruct(const uint16_t* lp, const void* rho, int rho_bits, int64_t n, float* out, uint32_t* d_err,
                cudaStream_t s) {
  if (n == 0) return 0;
  if (rho_bits == 8)
    reconstruct_kernel<127><<<blocks_for(n, 256), 256, 0, s>>>(lp, rho, n, out, d_err);
  else
    reconstruct_kernel<32767><<<blocks_for(n, 256), 256, 0, s>>>(lp, rho, n, out, d_err);
  return (int)cudaGetLastError();
}

int quantize(bool variance, const float* x, int64_t n, int64_t G, void* codes, uint16_t* scales, uint32_t* d_err,
             cudaStream_t s) {
  if (n == 0) return 0;
  const int64_t ng = (n + G - 1) / G;
  if (variance)
    quantize_kernel<true><<<blocks_for(ng, 128), 128, 0, s>>>(x, n, G, codes, scales, d_err);
  else
    quantize_kernel<false><<<blocks_for(ng, 128), 128, 0, s>>>(x, n, G, codes, scales, d_err);
  return (int)cudaGetLastError();
}

int dequantize(bool variance, const void* codes, const uint16_t* scales, int64_t n, int64_t G, float* out,
               cudaStream_t s) {
  if (n == 0) return 0;
  if (variance)
    dequantize_kernel<true><<<blocks_for(n, 256), 256, 0, s>>>(codes, scales, n, G, out);
  else
    dequantize_kernel<false><<<blocks_for(n, 256), 256, 0, s>>>(codes, scales, n, G, out);
  return (int)cudaGetLastError();
}

}  // namespace fo
