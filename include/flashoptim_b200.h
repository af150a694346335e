/*
 * flashoptim_b200.h -- C ABI of the B200 (sm_100a) FlashOptim step library
 * (libflashoptim_b200.so).
 *
 * Plain pointers and sizes only; no torch types.  Every device pointer is a
 * CUDA global-memory address; `stream` is a cudaStream_t passed as void*.
 * Each entry point names the reference function it replaces
 * (/root/reference/pkg/src/flashopt/<file>:<line>).  The reference API is a
 * set of pure NumPy functions; the C ABI is the in-place, stream-ordered
 * device form of the same contract:
 *
 *   reference                                  C ABI
 *   optim.adamw_step(state, grad, hp)  :208    fo_adamw_step / fo_step_mt(FO_OPT_ADAMW)
 *   optim.sgd_step(state, grad, hp)    :187    fo_sgd_step   / fo_step_mt(FO_OPT_SGD)
 *   optim.lion_step(state, grad, hp)   :238    fo_lion_step  / fo_step_mt(FO_OPT_LION)
 *   optim.STEP_FUNCTIONS               :261    fo_step_mt's `optimizer` argument
 *   optim.init_flash_state             :143    fo_split + zeroed codes/scales
 *   formats.split                      :232    fo_split
 *   formats.reconstruct                :248    fo_reconstruct
 *   quantize.quantize_momentum         :109    fo_quantize_momentum
 *   quantize.dequantize_momentum       :125    fo_dequantize_momentum
 *   quantize.quantize_variance         :134    fo_quantize_variance
 *   quantize.dequantize_variance       :152    fo_dequantize_variance
 *
 * Error behaviour.  The reference raises ValueError before producing any
 * output.  Device kernels cannot raise: each launch ORs FO_ERR_* bits into
 * the caller-owned device word `d_err` (may be NULL to skip reporting) and
 * the buffers are updated regardless.  fo_error_message() maps a mask to the
 * message the reference would have raised first.  Host-side argument errors
 * (bad sizes, unsupported layouts) are returned synchronously as FO_E*.
 */
#ifndef FLASHOPTIM_B200_H
#define FLASHOPTIM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FO_ABI_VERSION 2

/* Return codes (>0 values are cudaError_t). */
#define FO_OK 0
#define FO_EINVAL (-1)       /* bad argument (null pointer, size, unknown enum) */
#define FO_EUNSUPPORTED (-2) /* layout the library does not implement */
#define FO_ETOOMANY (-3)     /* hyper-parameter table larger than FO_MAX_HPARAMS */

/* Device error bits, one per reference ValueError class and buffer. */
#define FO_ERR_GRAD_NONFINITE 0x01u  /* optim.py:183 "gradient-nonfinite" */
#define FO_ERR_RHO_INVALID 0x02u     /* formats.py:271 "invalid-correction-code" */
#define FO_ERR_SPLIT_NONFINITE 0x04u /* formats.py:243 "split-nonfinite" */
#define FO_ERR_M_NONFINITE 0x08u     /* quantize.py:69 "quantize-nonfinite" (momentum) */
#define FO_ERR_M_OVERFLOW 0x10u      /* quantize.py:85,92 "scale-overflow" (momentum) */
#define FO_ERR_V_NONFINITE 0x20u     /* quantize.py:69 "quantize-nonfinite" (variance) */
#define FO_ERR_V_NEGATIVE 0x40u      /* quantize.py:144 "negative-variance" */
#define FO_ERR_V_OVERFLOW 0x80u      /* quantize.py:85,92 "scale-overflow" (variance) */

/* Optimizer tags = FLOP v1 header tags (checkpoint.py:54). */
#define FO_OPT_SGD 0
#define FO_OPT_ADAMW 1
#define FO_OPT_LION 2

/* Gradient element types.  The reference upcasts any grad to f32
 * (optim.py:179); bf16 is the training-time layout, f32 the exact one. */
#define FO_GRAD_BF16 0
#define FO_GRAD_F32 1

/* Variance storage schemes (optim.py:164-175). */
#define FO_VAR_COMPANDED 0
#define FO_VAR_LINEAR 1

#define FO_MAX_HPARAMS 16
#define FO_MAX_PEERS 7 /* peer mirrors per fo_step_mt_peers call (8 GPUs) */

/* Per-step float32 scalars, formed on the host exactly as the reference
 * forms them: Python floats rounded once to f32 (NEP 50), 1-beta and the
 * bias corrections 1-beta**t evaluated in float64 then rounded once
 * (optim.py:212-213, 220-221, 247-248).  Fill with fo_make_hparams(). */
typedef struct fo_hparams {
  float lr, wd, eps;
  float b1, omb1; /* beta1 and f32(1-beta1)          (AdamW, Lion) */
  float b2, omb2; /* beta2 and f32(1-beta2)          (AdamW, Lion) */
  float mu;       /* SGD momentum                    (SGD)         */
  float bc1, bc2; /* f32(1-beta1**t), f32(1-beta2**t) (AdamW)      */
  float rbc1, rbc2; /* RN(1/bc1), RN(1/bc2) (f32 division; used for exact Markstein quotients) */
} fo_hparams;

/* One flat parameter tensor's state (FLOP v1 record names,
 * checkpoint.py:111-123).  All element pointers cover `n` elements; scale
 * pointers cover ceil(n / group_size) fp16 values.  v_* are NULL for
 * SGD/Lion.  `hp_index` selects the fo_hparams entry (param group). */
typedef struct fo_tensor {
  void *lp;        /* "weights.lp"      bf16 bits, u16[n], in/out  */
  void *rho;       /* "weights.rho"     i8[n] (or i16[n]), in/out  */
  void *m_codes;   /* "momentum.codes"  i8[n], in/out              */
  void *m_scales;  /* "momentum.scales" f16[ceil(n/G)], in/out     */
  void *v_codes;   /* "variance.codes"  u8[n], in/out (AdamW)      */
  void *v_scales;  /* "variance.scales" f16[ceil(n/G)], in/out     */
  const void *grad;/* bf16[n] or f32[n], read only                 */
  int64_t n;
  int32_t hp_index;
  int32_t reserved;
} fo_tensor;

/* Library / device queries. */
uint32_t fo_abi_version(void);
const char *fo_status_string(int status);
/* Message of the reference ValueError that `mask` corresponds to for
 * `optimizer` (first in the reference's program order), or "" if mask==0.
 * Precedence: optim.py:208-235 (AdamW), :187-205 (SGD), :238-258 (Lion). */
const char *fo_error_message(uint32_t mask, int optimizer);

/* Host helper: the reference's per-step f32 scalars (optim.py:210-226). */
void fo_make_hparams(int optimizer, double lr, double beta1, double beta2, double eps, double weight_decay,
                     double momentum, int64_t t, fo_hparams *out);

/* Multi-tensor fused step: the whole parameter list in as few launches as
 * possible (one per FO_MT_MAX_TENSORS tensors), stream-ordered on `stream`.
 * Replaces a Python loop of STEP_FUNCTIONS[opt](state, grad, hp) calls
 * (training.py:219-226).  `tensors` and `hparams` are HOST arrays, read
 * before return.  rho_bits 8|16, group_size >= 1 (32 is the fused fast
 * path), variance_scheme FO_VAR_*. */
int fo_step_mt(int optimizer, const fo_tensor *tensors, int32_t n_tensors, const fo_hparams *hparams,
               int32_t n_hparams, int grad_dtype, int rho_bits, int32_t group_size, int variance_scheme,
               uint32_t *d_err, void *stream);

/* Host-resident state (the reference's calling convention: NumPy arrays in
 * host memory, optim.py:187-261).  Every pointer in `tensors` is a HOST
 * pointer (pinned for full PCIe bandwidth; pageable works).  The list is cut
 * into group-aligned pieces that stream through `chunk_elems`-element device
 * slots (0 = 64M): H2D copy, fused step, D2H copy on three rotating slots
 * and streams.  Any group_size >= 1 (quantize.py:33-44); every piece keeps
 * its own 16-byte aligned run of scales in the slot.  Synchronous; the error
 * mask is written to *h_err.  Reentrant: each call leases its own slots and
 * streams from a pool of per-device contexts, so concurrent calls from
 * several host threads neither share buffers nor serialise. */
int fo_step_host(int optimizer, const fo_tensor *tensors, int32_t n_tensors, const fo_hparams *hparams,
                 int32_t n_hparams, int grad_dtype, int rho_bits, int32_t group_size, int variance_scheme,
                 int64_t chunk_elems, uint32_t *h_err);
/* Free the idle contexts (device slots and streams) fo_step_host keeps
 * between calls. */
void fo_host_release(void);

/* Fast-path accounting of the fused launches on `stream` (current device).
 * The fused kernel computes every 512-element slice with exact shortcuts
 * whose preconditions it checks per slice; a slice whose check trips stores
 * nothing and is re-run by the fix-up launch that follows on the same stream
 * (DESIGN.md §3.2).  *flagged = slices re-run by fix-up launches, *slices =
 * slices the fused launches covered, both since the last reset.  Synchronises
 * `stream`.  No reference counterpart (test and bench support). */
int fo_fixup_stats(void *stream, uint64_t *flagged, uint64_t *slices, int reset);
/* Pre-size the fix-up bitmap of `stream` for launches of up to `max_elems`
 * elements, so that a CUDA-graph capture of fo_step_mt on that stream
 * allocates nothing.  Optional. */
int fo_reserve(void *stream, int64_t max_elems);
/* Elements per CTA tile of the fused kernel: every tensor of a launch is
 * padded to a multiple of it in the fix-up bitmap, so fo_reserve(stream,
 * sum of round_up(n_i, fo_fused_tile_elems())) covers any list. */
int64_t fo_fused_tile_elems(void);

/* Device-resident step scalars for CUDA-graph capture (the role of torch's
 * `capturable=True`): a captured fo_step_mt_dev reads, every time the graph
 * runs, the step counter t from device memory and takes (bc1, RN(1/bc1),
 * bc2, RN(1/bc2)) from a table built by fo_bias_table (entry min(t,
 * bc_len-1)), and the learning rate from `lr` when it is not NULL.  The
 * caller advances *step before each step (optim.py:211: t = state.t + 1),
 * e.g. with a captured device increment. */
typedef struct fo_dev_scalars {
  const int32_t *step;   /* device int32: t of the step being taken          */
  const float *lr;       /* device f32 learning rate, or NULL (hparams->lr)  */
  const float *bc_table; /* device f32[4 * bc_len] from fo_bias_table        */
  int32_t bc_len;        /* 0 for SGD / Lion (no bias correction)            */
  int32_t reserved;
  /* The caller's fix-up bitmap (zeroed once; every launch leaves it zero):
   * at least fo_fix_words(tensors) words.  The library allocates nothing. */
  uint32_t *fix_bits;
  int64_t fix_words;
  unsigned long long *fix_count; /* device counter of re-run slices, or NULL */
} fo_dev_scalars;

/* Words of fix-up bitmap a fused launch over `tensors` needs (a power of two). */
int64_t fo_fix_words(const fo_tensor *tensors, int32_t n_tensors);

/* fo_step_mt with one hyper-parameter set whose t-dependent fields come from
 * `dev` (hparams->bc1 ... are ignored).  The default layout only (int8
 * corrections, companded variance, group size 32, 16-byte aligned views,
 * hyper-parameters inside the fused tile's ranges): anything else returns
 * FO_EUNSUPPORTED.  Allocates nothing once fo_reserve has sized the stream's
 * fix-up bitmap, so it can be captured into a CUDA graph. */
int fo_step_mt_dev(int optimizer, const fo_tensor *tensors, int32_t n_tensors, const fo_hparams *hparams,
                   const fo_dev_scalars *dev, int grad_dtype, uint32_t *d_err, void *stream);

/* Fused step + all-gather over peer memory (ZeRO-1, zero.py): fo_step_mt
 * whose kernels also store every updated weights.lp value at
 * (char *)lp + peer_delta[r] for r < n_peers (<= FO_MAX_PEERS) -- the same
 * flat offset in each peer's parameter buffer, mapped into this process with
 * fo_ipc_open -- so the all-gather of the bf16 weights happens inside the
 * step, tile by tile, over NVLink.  One hyper-parameter set, the default
 * layout (int8 corrections, companded variance, group size 32, 16-byte
 * aligned views; FO_EUNSUPPORTED otherwise).  The caller orders the peers'
 * next reads after every rank's step (a cross-rank barrier on the stream). */
int fo_step_mt_peers(int optimizer, const fo_tensor *tensors, int32_t n_tensors, const fo_hparams *hparams,
                     int grad_dtype, const int64_t *peer_delta, int32_t n_peers, uint32_t *d_err, void *stream);

/* CUDA IPC for the peer mirrors.  fo_ipc_export: a 64-byte handle of the
 * allocation holding `ptr` and ptr's byte offset in it.  fo_ipc_open (in
 * another process): the mapped address of that byte; fo_ipc_close unmaps
 * (pass the address and offset fo_ipc_open took). */
int fo_ipc_export(const void *ptr, void *handle64, int64_t *offset);
int fo_ipc_open(const void *handle64, int64_t offset, void **ptr);
int fo_ipc_close(void *ptr, int64_t offset);

/* Host table for fo_dev_scalars: out[4t .. 4t+3] = (bc1, RN(1/bc1), bc2,
 * RN(1/bc2)) of fo_make_hparams at step t, for t = 0 .. *len-1, where *len-1
 * is the first t >= 1 at which both corrections are 1.0f (every later t has
 * the same entry; optim.py:212-213).  out may be NULL to query *len.
 * FO_ETOOMANY if that needs more than max_len entries. */
int fo_bias_table(double beta1, double beta2, int32_t max_len, float *out, int32_t *len);

/* Single-tensor steps, in place (optim.py:208, :187, :238). */
int fo_adamw_step(uint16_t *lp, int8_t *rho, int8_t *m_codes, uint16_t *m_scales, uint8_t *v_codes,
                  uint16_t *v_scales, const void *grad, int grad_dtype, int64_t n, const fo_hparams *hp,
                  uint32_t *d_err, void *stream);
int fo_sgd_step(uint16_t *lp, int8_t *rho, int8_t *m_codes, uint16_t *m_scales, const void *grad, int grad_dtype,
                int64_t n, const fo_hparams *hp, uint32_t *d_err, void *stream);
int fo_lion_step(uint16_t *lp, int8_t *rho, int8_t *m_codes, uint16_t *m_scales, const void *grad, int grad_dtype,
                 int64_t n, const fo_hparams *hp, uint32_t *d_err, void *stream);

/* Codecs (formats.py:232-276, quantize.py:109-158), device buffers. */
int fo_split(const float *theta, int64_t n, uint16_t *lp, void *rho, int rho_bits, uint32_t *d_err, void *stream);
int fo_reconstruct(const uint16_t *lp, const void *rho, int rho_bits, int64_t n, float *out, uint32_t *d_err,
                   void *stream);
int fo_quantize_momentum(const float *m, int64_t n, int32_t group_size, int8_t *codes, uint16_t *scales,
                         uint32_t *d_err, void *stream);
int fo_dequantize_momentum(const int8_t *codes, const uint16_t *scales, int64_t n, int32_t group_size, float *out,
                           void *stream);
int fo_quantize_variance(const float *v, int64_t n, int32_t group_size, uint8_t *codes, uint16_t *scales,
                         uint32_t *d_err, void *stream);
int fo_dequantize_variance(const uint8_t *codes, const uint16_t *scales, int64_t n, int32_t group_size, float *out,
                           void *stream);

/* Device self-check of the fast exact primitives against the IEEE
 * intrinsics (no reference counterpart; test support).  mode 0: sqrt over
 * f32 bit patterns [begin, begin+count); 1: reciprocal of every fp16 value;
 * 2/3/4: hash-sampled quotients (per-element, per-group-scale and
 * bias-correction divisors); 6: the fused tile's integer reconstruct over
 * every (bf16 code, rho); 7: the wide-range sqrt over f32 bit patterns
 * [begin, begin+count) below 2^64.  d_out[0] += mismatches, d_out[1] = min failing
 * index (initialise to 0 and UINT64_MAX); mode 5 writes raw sqrt results to
 * d_out[2..] (debug). */
int fo_selftest(int mode, uint64_t begin, uint64_t count, uint64_t *d_out, void *stream);

/* Exhaustive FP32 reconstruction sweep (replaces sweep.py:166-218
 * _sweep_block / :231 exhaustive_sweep_multi for the BF16 format).  Sweeps
 * the (sign, exponent-field) blocks [block0, block0 + nblocks) of the 510
 * finite ones; scheme_mask bit s selects sweep.SCHEMES[s] (ulp8, ulp16,
 * none, baseline).  d_out: nblocks * 4 records of 8 uint64 each, zeroed by
 * the caller: {count, exact, overflow, zero, zero_exact, (double) relsum,
 * (float bits) relmax, unused}, the per-block tuple _sweep_block returns. */
#define FO_SWEEP_RECORD_U64 8
int fo_sweep(int block0, int nblocks, uint32_t scheme_mask, uint64_t *d_out, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* FLASHOPTIM_B200_H */
