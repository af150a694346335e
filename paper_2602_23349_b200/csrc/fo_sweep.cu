// fo_sweep.cu -- exhaustive FP32 reconstruction sweep on the GPU
// (reference: flashopt/sweep.py).
//
// Every finite FP32 bit pattern of the requested (sign, exponent-field)
// blocks goes through one weight-compression scheme -- bf16 + int8 ULP
// correction ("ulp8"), bf16 + int16 ("ulp16"), plain bf16 ("none") or bf16 +
// bf16 residual ("baseline") -- using the same device codec as the generic
// step kernel (fo_math.cuh), and is compared with the original.  Per block
// and scheme the kernel accumulates exactly what sweep.py's _sweep_block
// does: valid count, bitwise-exact count, sum (float64) and max of the
// float32 relative error, overflow count (downcast to inf), and the +-0
// lane separately.  Counts and maxima are order-independent and match the
// reference exactly; the float64 sums differ only in summation order.
#include <cuda_runtime.h>

#include "fo_internal.h"
#include "fo_math.cuh"

namespace fo {

namespace {

constexpr int kSchemes = 4;  // 0 ulp8, 1 ulp16, 2 none, 3 baseline (sweep.py SCHEMES order)
constexpr uint32_t kChunk = 1u << 16;

__device__ __forceinline__ float rec_scheme(int s, float theta, uint32_t code) {
  if (s == 2) return bf16_up(code);
  if (s == 3) {  // sweep.py:150-156: lp + upcast(downcast(theta - lp))
    const float lp = bf16_up(code);
    const uint32_t r = bf16_rne(__fsub_rn(theta, lp));
    return __fadd_rn(lp, bf16_up(r));
  }
  uint32_t c;
  int rho;
  if (s == 0) {
    split1<127>(theta, c, rho);
    return reconstruct1(code, rho, __fdiv_rn((float)rho, 127.0f));
  }
  split1<32767>(theta, c, rho);
  return reconstruct1(code, rho, __fdiv_rn((float)rho, 32767.0f));
}

// out layout per (block, scheme): u64[5] {count, exact, overflow, zero, zero_exact},
// then double relsum, then u32 relmax bits (stored in a u64 slot).
struct Acc {  // FO_SWEEP_RECORD_U64 = 8 words
  unsigned long long n[5];
  double relsum;
  unsigned long long relmax;
  unsigned long long unused;
};
static_assert(sizeof(Acc) == 8 * FO_SWEEP_RECORD_U64, "record layout is part of the C ABI");

__global__ void sweep_kernel(int block0, int nblocks, uint32_t scheme_mask, Acc* out) {
  const int b = block0 + (int)(blockIdx.x / (((1u << 23) / kChunk)));
  const uint32_t chunk = blockIdx.x % ((1u << 23) / kChunk);
  const uint32_t sign = (uint32_t)b / 255u, expf = (uint32_t)b % 255u;
  const uint32_t base = (sign << 31) | (expf << 23) | (chunk * kChunk);
  uint32_t cnt[kSchemes] = {0, 0, 0, 0}, ex[kSchemes] = {0, 0, 0, 0}, relmax[kSchemes] = {0, 0, 0, 0};
  double rs[kSchemes] = {0.0, 0.0, 0.0, 0.0};
  uint32_t ovf = 0, zc = 0, zex[kSchemes] = {0, 0, 0, 0};
  for (uint32_t i = threadIdx.x; i < kChunk; i += blockDim.x) {
    const uint32_t u = base + i;
    const float theta = __uint_as_float(u);
    const uint32_t code = bf16_rne(theta);
    if ((code & 0x7F80u) == 0x7F80u) {  // downcast overflows (sweep.py:186-189)
      ++ovf;
      continue;
    }
    const bool zero_lane = (u & 0x7FFFFFFFu) == 0;
    if (zero_lane) ++zc;
    const float at = fabsf(theta);
#pragma unroll
    for (int s = 0; s < kSchemes; ++s) {
      if (!((scheme_mask >> s) & 1u)) continue;
      const float rec = rec_scheme(s, theta, code);
      const bool exact = __float_as_uint(rec) == u;
      if (zero_lane) {
        zex[s] += exact;
        continue;
      }
      const float rel = __fdiv_rn(fabsf(__fsub_rn(rec, theta)), at);
      ++cnt[s];
      ex[s] += exact;
      rs[s] += (double)rel;
      relmax[s] = max(relmax[s], __float_as_uint(rel));
    }
  }
  // warp reduce, then one atomic per warp
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ovf += __shfl_xor_sync(0xffffffffu, ovf, o);
    zc += __shfl_xor_sync(0xffffffffu, zc, o);
#pragma unroll
    for (int s = 0; s < kSchemes; ++s) {
      cnt[s] += __shfl_xor_sync(0xffffffffu, cnt[s], o);
      ex[s] += __shfl_xor_sync(0xffffffffu, ex[s], o);
      zex[s] += __shfl_xor_sync(0xffffffffu, zex[s], o);
      rs[s] += __shfl_xor_sync(0xffffffffu, rs[s], o);
      relmax[s] = max(relmax[s], __shfl_xor_sync(0xffffffffu, relmax[s], o));
    }
  }
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < kSchemes; ++s) {
      if (!((scheme_mask >> s) & 1u)) continue;
      Acc* a = out + (size_t)(b - block0) * kSchemes + s;
      atomicAdd(&a->n[0], (unsigned long long)cnt[s]);
      atomicAdd(&a->n[1], (unsigned long long)ex[s]);
      atomicAdd(&a->n[2], (unsigned long long)ovf);
      atomicAdd(&a->n[3], (unsigned long long)zc);
      atomicAdd(&a->n[4], (unsigned long long)zex[s]);
      atomicAdd(&a->relsum, rs[s]);
      atomicMax(&a->relmax, (unsigned long long)relmax[s]);
    }
  }
}

}  // namespace

// Sweep blocks [block0, block0 + nblocks) of the 510 (sign, exponent-field)
// blocks; `out` holds nblocks * 4 records of 8 u64 (see Acc), zeroed by the
// caller.  bf16 only.
int sweep(int block0, int nblocks, uint32_t scheme_mask, void* out, cudaStream_t s) {
  if (block0 < 0 || nblocks <= 0 || block0 + nblocks > 510 || !out || (scheme_mask & ~0xFu)) return FO_EINVAL;
  const unsigned grid = (unsigned)nblocks * ((1u << 23) / kChunk);
  sweep_kernel<<<grid, 256, 0, s>>>(block0, nblocks, scheme_mask, static_cast<Acc*>(out));
  return (int)cudaGetLastError();
}

}  // namespace fo
