// Pipe-throughput microbenchmark: cycles per warp-instruction per SMSP for
// the FP32x2 / FP32 / integer forms the fused step uses (sm_100a).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define N_ITER 256
template <int MODE>
__global__ void kern(float* out, unsigned long long* cyc, float a0, float b0) {
  float2 x[8], y = make_float2(a0, b0), z = make_float2(b0, a0);
  uint32_t u[8];
  for (int i = 0; i < 8; ++i) { x[i] = make_float2(a0 + i, b0 - i); u[i] = threadIdx.x * (i + 3); }
  float s = a0;
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int it = 0; it < N_ITER; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) x[i] = __ffma2_rn(x[i], y, z);                       // FFMA2 3 pairs
      if (MODE == 1) x[i] = __ffma2_rn(x[i], make_float2(s, s), z);       // FFMA2 scalar-broadcast operand
      if (MODE == 2) x[i] = __fmul2_rn(x[i], y);                          // FMUL2
      if (MODE == 3) x[i] = __fadd2_rn(x[i], y);                          // FADD2
      if (MODE == 4) { x[i].x = __fmaf_rn(x[i].x, y.x, z.x); }            // FFMA scalar 3 regs
      if (MODE == 5) { x[i].x = __fmaf_rn(x[i].x, 1.0001f, 0.5f); }       // FFMA imm
      if (MODE == 6) { u[i] = u[i] * 0x10001u + 7u; }                     // IMAD
      if (MODE == 7) { u[i] = (u[i] ^ 0x1234u) + (u[i] >> 3); }           // ALU LOP3/SHF/IADD
      if (MODE == 8) { x[i] = __ffma2_rn(x[i], y, z); u[i] = (u[i] << 3) ^ 0x55u; }   // FFMA2 + 2 ALU
      if (MODE == 9) { x[i].x = __fmaf_rn(x[i].x, y.x, z.x); x[i].y = __fmaf_rn(x[i].y, y.y, z.y); }  // 2 scalar FFMA
      if (MODE == 10) { x[i] = __ffma2_rn(x[i], y, make_float2(-0.0f, -0.0f)); }  // FFMA2 with -0 const addend
    }
  }
  unsigned long long t1 = clock64();
  float acc = 0;
  for (int i = 0; i < 8; ++i) acc += x[i].x + x[i].y + (float)u[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int MODE>
void run(const char* name, int warps_per_sm, int ninst_per_iter) {
  float* out; unsigned long long* cyc;
  int blocks = 148;
  cudaMalloc(&out, sizeof(float) * blocks * 32 * warps_per_sm);
  cudaMalloc(&cyc, sizeof(unsigned long long) * blocks);
  kern<MODE><<<blocks, 32 * warps_per_sm>>>(out, cyc, 1.0f, 2.0f);
  kern<MODE><<<blocks, 32 * warps_per_sm>>>(out, cyc, 1.0f, 2.0f);
  cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double c = 0; for (int i = 0; i < blocks; ++i) c += h[i]; c /= blocks;
  double inst = (double)N_ITER * 8 * ninst_per_iter * warps_per_sm / 4.0;  // per SMSP
  printf("%-34s warps/SM=%2d  cycles/warp-inst/SMSP = %.3f\n", name, warps_per_sm, c / inst);
  cudaFree(out); cudaFree(cyc);
}

int main() {
  for (int w : {16, 32}) {
    run<0>("FFMA2 r,r,r", w, 1);
    run<1>("FFMA2 r,bcast,r", w, 1);
    run<10>("FFMA2 r,r,-0const", w, 1);
    run<2>("FMUL2 r,r", w, 1);
    run<3>("FADD2 r,r", w, 1);
    run<4>("FFMA r,r,r", w, 1);
    run<9>("2x FFMA r,r,r", w, 2);
    run<5>("FFMA r,imm,imm", w, 1);
    run<6>("IMAD", w, 1);
    run<7>("ALU (3 ops)", w, 3);
    run<8>("FFMA2 + 2 ALU (per 3 inst)", w, 3);
  }
  return 0;
}
