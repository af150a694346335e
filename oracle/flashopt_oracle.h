/*
 * flashopt_oracle.h -- CPU restatement of the reference FlashOptim path.
 * TEST INFRASTRUCTURE ONLY (see flashopt_oracle.c header).
 */
#ifndef FLASHOPT_ORACLE_H
#define FLASHOPT_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Error bits: one per reference ValueError class and buffer.  Same values as
 * include/flashoptim_b200.h so tests can compare masks directly. */
#define FO_ERR_GRAD_NONFINITE 0x01u  /* optim.py:183 "gradient-nonfinite" */
#define FO_ERR_RHO_INVALID 0x02u     /* formats.py:271 "invalid-correction-code" */
#define FO_ERR_SPLIT_NONFINITE 0x04u /* formats.py:243 "split-nonfinite" */
#define FO_ERR_M_NONFINITE 0x08u     /* quantize.py:69 "quantize-nonfinite" (momentum) */
#define FO_ERR_M_OVERFLOW 0x10u      /* quantize.py:85,92 "scale-overflow" (momentum) */
#define FO_ERR_V_NONFINITE 0x20u     /* quantize.py:69 (variance) */
#define FO_ERR_V_NEGATIVE 0x40u      /* quantize.py:144 "negative-variance" */
#define FO_ERR_V_OVERFLOW 0x80u      /* quantize.py:85,92 (variance) */

#define FO_OPT_SGD 0   /* checkpoint.py:54 tags */
#define FO_OPT_ADAMW 1
#define FO_OPT_LION 2

typedef struct {
  float lr, wd, eps, b1, omb1, b2, omb2, mu, bc1, bc2;
} fo_oracle_scalars;

uint16_t fo_oracle_downcast_bf16(float x);
int fo_oracle_ulp_exponent(uint16_t code, int residual_negative);
uint32_t fo_oracle_split(const float *theta, int64_t n, int width_bits, uint16_t *lp, void *rho);
uint32_t fo_oracle_reconstruct(const uint16_t *lp, const void *rho, int64_t n, int width_bits, float *out);
uint32_t fo_oracle_quantize_momentum(const float *m, int64_t n, int64_t G, int8_t *codes, uint16_t *scales);
void fo_oracle_dequantize_momentum(const int8_t *codes, const uint16_t *scales, int64_t n, int64_t G, float *out);
uint32_t fo_oracle_quantize_variance(const float *v, int64_t n, int64_t G, uint8_t *codes, uint16_t *scales);
void fo_oracle_dequantize_variance(const uint8_t *codes, const uint16_t *scales, int64_t n, int64_t G, float *out);
uint32_t fo_oracle_quantize_linear(const float *x, int64_t n, int64_t G, int is_signed, void *codes, uint16_t *scales);
void fo_oracle_dequantize_linear(const void *codes, const uint16_t *scales, int64_t n, int64_t G, int is_signed,
                                 float *out);
void fo_oracle_make_scalars(int opt, double lr, double b1, double b2, double eps, double wd, double mu, int64_t t,
                            fo_oracle_scalars *s);
uint32_t fo_oracle_step(int opt, uint16_t *lp, void *rho, int width_bits, int8_t *mq, uint16_t *ms, void *vq,
                        uint16_t *vs, int variance_scheme, const float *grad, int64_t n, int64_t G,
                        const fo_oracle_scalars *s, int nthreads);
int fo_oracle_max_threads(void);

#ifdef __cplusplus
}
#endif
#endif
