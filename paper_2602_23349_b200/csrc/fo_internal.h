// fo_internal.h -- shared declarations between the .cu translation units.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>
#include <vector>

#include "flashoptim_b200.h"

// Max tensors per fused launch: the whole table travels as one
// __grid_constant__ kernel parameter block (< 32 KB, CUDA >= 12.1).
#define FO_MT_MAX_TENSORS 384

namespace fo {

// Device-resident step scalars (fo_step_mt_dev): NULL `step` = host scalars.
struct DevScalars {
  const int32_t* step;
  const float* lr;
  const float* bc;  // 4 floats per t
  int32_t bc_len;
  uint32_t* fix_bits;  // caller-owned fix-up bitmap (no allocation on the launch path)
  int64_t fix_words;
  unsigned long long* fix_count;
  // fo_step_mt_peers: mirror every updated weights.lp to these byte deltas
  int32_t npeers;
  const int64_t* peer_delta;
};
int64_t fix_words_for(const fo_tensor* ts, int32_t nt);  // fo_step_adamw.cu

int step_mt(int opt, const fo_tensor* ts, int32_t nt, const fo_hparams* hps, int32_t nhp, int grad_dtype,
            int rho_bits, int32_t G, int var_scheme, uint32_t* d_err, cudaStream_t s,
            const DevScalars* dev = nullptr);
int split(const float* theta, int64_t n, uint16_t* lp, void* rho, int rho_bits, uint32_t* d_err, cudaStream_t s);
int reconstruct(const uint16_t* lp, const void* rho, int rho_bits, int64_t n, float* out, uint32_t* d_err,
                cudaStream_t s);
int quantize(bool variance, const float* x, int64_t n, int64_t G, void* codes, uint16_t* scales, uint32_t* d_err,
             cudaStream_t s);
int step_host(int opt, const fo_tensor* ts, int32_t nt, const fo_hparams* hps, int32_t nhp, int grad_dtype,
              int rho_bits, int32_t G, int var_scheme, int64_t chunk_elems, uint32_t* h_err);
void host_release();

// Fix-up bitmap of one (device, stream): one bit per 512-element slice of a
// fused launch whose guards tripped, plus a device counter of the slices the
// fix-up launches re-ran.  Shared by the three optimizer translation units
// (fo_step.cu).  `bits` is NULL when allocation failed.
struct FixBuf {
  uint32_t* bits;
  unsigned long long* count;
};
FixBuf fix_buffer(cudaStream_t s, size_t words);
void fix_account(cudaStream_t s, uint64_t slices);  // host-side count of fast-tile slices launched
int fix_stats(cudaStream_t s, uint64_t* flagged, uint64_t* slices, int reset);
int fix_reserve(cudaStream_t s, int64_t elems);
int64_t fused_tile_elems();  // fo_step_adamw.cu (WS_CT)
// Persistent-grid size of `kernel` on the current device (cached per kernel and device).
int grid_cap_for(const void* kernel, int threads, int smem);
int selftest(int mode, uint64_t begin, uint64_t count, unsigned long long* d_out, cudaStream_t s);
int sweep(int block0, int nblocks, uint32_t scheme_mask, void* out, cudaStream_t s);
int dequantize(bool variance, const void* codes, const uint16_t* scales, int64_t n, int64_t G, float* out,
               cudaStream_t s);

}  // namespace fo
