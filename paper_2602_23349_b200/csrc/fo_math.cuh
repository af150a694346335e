// fo_math.cuh -- bit-exact device restatement of the FlashOptim codecs.
//
// Every function names the reference line it reproduces
// (/root/reference/pkg/src/flashopt/...).  All arithmetic goes through the
// explicit IEEE round-to-nearest intrinsics (__fmul_rn, __fadd_rn, ...) so
// no FMA contraction can change a rounding; the library is additionally
// compiled with -fmad=false -ftz=false -prec-div=true -prec-sqrt=true.
#pragma once

#include <cuda_fp16.h>
#include <stdint.h>

#include "flashoptim_b200.h"

namespace fo {

// ---------------------------------------------------------------------------
// bf16 / fp16 helpers
// ---------------------------------------------------------------------------

// formats.py:165-171: RNE downcast of a finite f32 to bf16 bits (overflow
// saturates to inf through the carry).  NaN never reaches here (split
// rejects it first, formats.py:242).
__device__ __forceinline__ uint32_t bf16_rne(float x) {
  uint32_t u = __float_as_uint(x);
  return (u + 0x7FFFu + ((u >> 16) & 1u)) >> 16;
}

// formats.py:183-187
__device__ __forceinline__ float bf16_up(uint32_t code) { return __uint_as_float(code << 16); }

// formats.py:114-116 (_pow2_normal): 2^k for -126 <= k <= 127.
__device__ __forceinline__ float pow2i(int k) { return __uint_as_float((uint32_t)(k + 127) << 23); }

// formats.py:127-154 (_ulp_exponent_scale) for BF16 with the binade-bottom
// refinement: ell = max(expf,1) - 135, minus one when the code's mantissa
// is zero, expf >= 2 and the residual points toward zero.
__device__ __forceinline__ int ulp_exp(uint32_t code, bool residual_negative) {
  int expf = (code >> 7) & 0xFF;
  int ell = max(expf, 1) - 135;
  bool toward_zero = residual_negative != ((code & 0x8000u) != 0);
  bool at_bottom = ((code & 0x7Fu) == 0) && (expf >= 2);
  return ell - ((at_bottom && toward_zero) ? 1 : 0);
}

// formats.py:248-276 reconstruct: lp + RN(rho/N)*2^h*2^(ell-h) with a single
// rounding (the float64 sum in the reference is exact, so fmaf matches).
// rho_over_n is RN(rho/N), supplied by the caller (exact LUT or division).
__device__ __forceinline__ float reconstruct1(uint32_t code, int rho, float rho_over_n) {
  int ell = ulp_exp(code, rho < 0);
  int half = ell >> 1;  // floor(ell/2), formats.py:273
  float scaled = __fmul_rn(rho_over_n, pow2i(half));
  return __fmaf_rn(scaled, pow2i(ell - half), bf16_up(code));
}

// formats.py:205-229 encode_correction + downcast: finite theta -> (code, rho).
template <int NCORR>
__device__ __forceinline__ void split1(float theta, uint32_t& code, int& rho) {
  code = bf16_rne(theta);
  float e = __fsub_rn(theta, bf16_up(code));           // :220 (exact)
  int ell = ulp_exp(code, e < 0.0f);                   // :221
  int half = (-ell) >> 1;                              // :222 floor(-ell/2)
  float en = __fmul_rn(__fmul_rn(e, pow2i(half)), pow2i(-ell - half));  // :223
  en = fminf(fmaxf(en, -1.0f), 1.0f);                  // :224
  int r = __float2int_rn(__fmul_rn(en, (float)NCORR)); // :225 rint, ties-to-even
  rho = (((code >> 7) & 0xFF) == 0xFF) ? 0 : r;        // :226-228 saturated lanes
}

// quantize.py:82-93: non-negative group max -> fp16 scale rounded up.
// Returns the fp16 bits and raises `bit` in err when the max exceeds 65504.
__device__ __forceinline__ uint32_t scale_ru(float gmax, uint32_t& err, uint32_t bit) {
  if (gmax > 65504.0f) {
    err |= bit;
    return 0x7BFFu;
  }
  return (uint32_t)__half_as_ushort(__float2half_ru(gmax));
}

__device__ __forceinline__ float half_bits_to_float(uint32_t h) {
  return __half2float(__ushort_as_half((unsigned short)h));
}

// quantize.py:125-131 dequantize_momentum: z = c/127, m' = z/(2-|z|).
// Depends on the code only; evaluated once per code into a LUT.
__device__ __forceinline__ float momentum_unit(int c) {
  float z = __fdiv_rn((float)c, 127.0f);
  return __fdiv_rn(z, __fsub_rn(2.0f, fabsf(z)));
}

// quantize.py:156: z = c/255.
__device__ __forceinline__ float variance_unit(int c) { return __fdiv_rn((float)c, 255.0f); }

// quantize.py:119-121: one normalised momentum value -> code.
__device__ __forceinline__ int momentum_code(float mn) {
  float z = __fdiv_rn(__fmul_rn(2.0f, mn), __fadd_rn(1.0f, fabsf(mn)));
  float q = rintf(__fmul_rn(z, 127.0f));
  q = fminf(fmaxf(q, -127.0f), 127.0f);
  return (int)q;
}

// quantize.py:147-148: one normalised root -> code.
__device__ __forceinline__ int variance_code(float vn) {
  float q = rintf(__fmul_rn(vn, 255.0f));
  q = fminf(fmaxf(q, 0.0f), 255.0f);
  return (int)q;
}

__device__ __forceinline__ bool finite(float x) { return (__float_as_uint(x) & 0x7F800000u) != 0x7F800000u; }

}  // namespace fo
