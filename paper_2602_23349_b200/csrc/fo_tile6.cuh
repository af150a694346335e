// fo_tile6.cuh -- the fused step's per-tile arithmetic (warp-specialised
// kernel), included by fo_step_impl.cuh.
//
// Bit-identical to process_tile_exact (and therefore to the reference,
// optim.py:187-261) whenever no guard trips; a tripped guard anywhere in the
// warp sends the whole tile to process_tile_exact before anything is
// stored.  Differences from compute_tile (the older kernels' tile):
//
//  * integer reconstruct (formats.py:248-276).  theta = RN(lp + RN(rho/127)
//    * 2^ell) is lp's f32 bit pattern plus R(rho) = rint_even(RN(|rho|/127)
//    * 2^15) ulps, moving away from zero when rho has lp's sign and toward
//    zero otherwise.  lp has 16 zero low mantissa bits, so the tie parity
//    is R's; 2^ell is exactly 2^15 f32 ulps of lp's binade, and at a binade
//    bottom with rho pointing toward zero (the formats.py:147-154
//    refinement) 2^(ell-1) is 2^15 ulps of the binade below, which integer
//    subtraction on the bit pattern steps into.  Checked for every finite
//    bf16 code x every rho (tests/test_gpu_primitives.py, test_tile6_
//    reconstruct): the only mismatches are lp = +-0 with rho of the other
//    sign (theta comes out NaN -> guard) and (-0, rho = 0) (theta comes out
//    -0 where the reference has +0 -> guard on a -0 / zero update).
//  * guards on the packed inputs with 16x2 SIMD min/max, and on the
//    updated weights with float min/max of |theta_new|;
//  * gradients stay packed bf16 words until the update.
#pragma once
// (textually included inside namespace fo)

#ifndef FO_VG
#define FO_VG 1
#endif
// Steady state (f32 bias corrections == 1): the variance root is taken with
// fast::sqrt_rn2_wide, exact for every v < 2^64, so the v operand guard goes.
#ifndef FO_SQRT_WIDE
#define FO_SQRT_WIDE 1
#endif
// Split code from a K * 2^-13 made by one LOP3 (1 instead of 2 integer ops
// per element); 0: K = 127 * 2^-ell by LOP3 + IADD3.
// FO_MQ_APPROX=1: momentum codes from an approximate quotient with an
// exactness check on the rounding distance (exact fallback per lane).
#ifndef FO_MQ_APPROX
#define FO_MQ_APPROX 1
#endif
// FO_PROBE (energy measurements only, results NOT exact): 1 momentum
// quotients -> one multiply, 2 variance quotient -> one multiply, 3 the
// update's division -> a multiply, 4 no range guards, 5 no moment LUT lookups.
#ifndef FO_PROBE
#define FO_PROBE 0
#endif
#ifndef FO_SPLIT_K13
#define FO_SPLIT_K13 1
#endif
// Steady-state AdamW keeps the variance roots scaled by 2^30 (one FMUL2 per
// pair fewer); 0: unscaled roots.
#ifndef FO_ROOT_SCALED
#define FO_ROOT_SCALED 1
#endif

struct Luts6 {
  int r[256];    // R(rho) by byte, signed; 0 for the invalid code -128 (caught by the rho guard)
  float m[256];  // quantize.py:129-130, z/(2-|z|) for every int8 code (by byte)
  float v[256];  // quantize.py:156, c/255
};

__device__ __forceinline__ void init_luts6(Luts6& L) {
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    const int rho = (int)(int8_t)i;
    L.r[i] = rho == -128 ? 0 : fast::recon_r(rho);
    L.m[i] = momentum_unit(rho);
    L.v[i] = variance_unit(i);
  }
}

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
  return r;
}

// Peer mirrors of the bf16 weights (the fused step + all-gather): every
// updated weights.lp value is also stored at its address + delta[r] (bytes)
// for r < n -- the same flat offset in peer r's parameter buffer, mapped
// into this process with CUDA IPC (zero.py, fused_allgather).
struct PeerSet {
  const int64_t* delta;
  int n;
  template <typename T>
  __device__ __forceinline__ T* at(T* p, int r) const {
    return reinterpret_cast<T*>(reinterpret_cast<char*>(p) + delta[r]);
  }
};

// (~t & 0x7F800000) | 0x007E0000 as one LOP3 (left to itself ptxas emits a
// mask and an XOR): K * 2^-13 of the split, see compute_tile6.
__device__ __forceinline__ uint32_t k13_bits(uint32_t t) {
  uint32_t r;
  asm("lop3.b32 %0, %1, %2, %3, 0xAE;" : "=r"(r) : "r"(t), "r"(0x7F800000u), "r"(0x007E0000u));
  return r;
}

// (~t & 0x7F800000) | 0x007FFE00: K * 2^-21 of the int16 split.
__device__ __forceinline__ uint32_t k16_bits(uint32_t t) {
  uint32_t r;
  asm("lop3.b32 %0, %1, %2, %3, 0xAE;" : "=r"(r) : "r"(t), "r"(0x7F800000u), "r"(0x007FFE00u));
  return r;
}

// Compact LUTs (3 KB): index = code byte, one PRMT + one LEA per lookup.
struct NarrowLut {
  const Luts6& L;
  __device__ __forceinline__ int r(uint32_t w, int j) const { return L.r[prmt(w, 0, 0x4440u + j)]; }
  __device__ __forceinline__ float m(uint32_t w, int j) const { return L.m[prmt(w, 0, 0x4440u + j)]; }
  __device__ __forceinline__ float v(uint32_t w, int j) const { return L.v[prmt(w, 0, 0x4440u + j)]; }
};

// No table: the SAFE re-run computes the dequantisation units directly.
struct NoLut {
  __device__ __forceinline__ int r(uint32_t w, int j) const { return fast::recon_r((int)(int8_t)(w >> (8 * j))); }
  __device__ __forceinline__ float m(uint32_t w, int j) const { return momentum_unit((int)(int8_t)(w >> (8 * j))); }
  __device__ __forceinline__ float v(uint32_t w, int j) const { return variance_unit((int)((w >> (8 * j)) & 0xFFu)); }
};

// Wide LUTs (64 KB at shared-window address 0x20000): row b (256 bytes)
// holds 21 copies of each table, so the shared address
// 0x20000 + 256*b + 4*(21*t + lane%21) is ONE PRMT of the code word with a
// per-lane register holding 0x00020000 | offset (code byte -> byte 1,
// offset -> byte 0, 0x02 -> byte 2): no address arithmetic at all, and the
// lanes of a warp hit distinct banks except l and l+21 (at most 2-way
// conflicts, against ~3.5-way for random indices into a compact table).
// FO_R_LUT=0: R(rho) is computed (see compute_tile6) and the wide LUT holds
// only the two moment tables, 32 copies each: lane l reads word l of its
// table's half row, so every lookup is conflict-free.
#ifndef FO_R_LUT
#define FO_R_LUT 1
#endif
constexpr int WIDE_COPIES = FO_R_LUT ? 21 : 32;
constexpr int WIDE_TABLES = FO_R_LUT ? 3 : 2;
constexpr uint32_t WIDE_LUT_ADDR = 0x20000u;
constexpr uint32_t WIDE_LUT_BYTES = 256u * 256u;
struct WideLut {
  uint32_t o_r, o_m, o_v;  // 0x20000 | 4*(21*t + lane%21), t = 0, 1, 2
  __device__ __forceinline__ static uint32_t ld(uint32_t a) {
    uint32_t v;
    asm("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
  }
  __device__ __forceinline__ int r(uint32_t w, int j) const { return (int)ld(prmt(w, o_r, 0x7604u | ((uint32_t)j << 4))); }
  __device__ __forceinline__ float m(uint32_t w, int j) const {
    return __uint_as_float(ld(prmt(w, o_m, 0x7604u | ((uint32_t)j << 4))));
  }
  __device__ __forceinline__ float v(uint32_t w, int j) const {
    return __uint_as_float(ld(prmt(w, o_v, 0x7604u | ((uint32_t)j << 4))));
  }
};

// `dsm`: the CTA's dynamic shared memory, at least WIDE_LUT_ADDR +
// WIDE_LUT_BYTES - (its shared address) bytes long.  The 768 distinct
// values are computed once into `Ls` (the narrow tables) and then
// replicated, so the prologue costs a few hundred stores per thread
// instead of ~30 IEEE quotients.  Contains a __syncthreads.
__device__ __forceinline__ WideLut init_wide_lut(uint8_t* dsm, Luts6& Ls) {
  uint8_t* base = dsm + (WIDE_LUT_ADDR - (uint32_t)__cvta_generic_to_shared(dsm));
  init_luts6(Ls);
  __syncthreads();
  for (int i = threadIdx.x; i < 256 * WIDE_TABLES * WIDE_COPIES; i += blockDim.x) {
    const int b = i / (WIDE_TABLES * WIDE_COPIES), w = i % (WIDE_TABLES * WIDE_COPIES), t = w / WIDE_COPIES + (3 - WIDE_TABLES);
    const uint32_t val = t == 0 ? (uint32_t)Ls.r[b] : __float_as_uint(t == 1 ? Ls.m[b] : Ls.v[b]);
    reinterpret_cast<uint32_t*>(base + b * 256)[w] = val;
  }
  const uint32_t c = (threadIdx.x & 31) % WIDE_COPIES;
  if (WIDE_TABLES == 2) return WideLut{0u, WIDE_LUT_ADDR | (4u * c), WIDE_LUT_ADDR | (4u * (WIDE_COPIES + c))};
  return WideLut{WIDE_LUT_ADDR | (4u * c), WIDE_LUT_ADDR | (4u * (WIDE_COPIES + c)),
                 WIDE_LUT_ADDR | (4u * (2 * WIDE_COPIES + c))};
}

// RB: bytes per correction code (1: int8, N = 127; 2: int16, N = 32767).
template <int NCORR>
struct Corr {
  static constexpr int RB = NCORR == 127 ? 1 : 2;
  typedef typename std::conditional<NCORR == 127, int8_t, int16_t>::type T;
};

template <typename GradT, int NCORR = 127>
struct TileIn6 {
  static constexpr int E = FEPL, NW = FEPL / 2, NB = FEPL / 4;
  static constexpr int NG = sizeof(GradT) == 2 ? NW : E;  // grad words
  static constexpr int NR = NB * Corr<NCORR>::RB;        // correction words
  uint32_t lw[NW], rw[NR], mw[NB], vw[NB], gw[NG];
  uint32_t msb, vsb;
};

// Partial (or unaligned) tile straight from global memory; elements past n
// read as zero state with zero gradient.
template <int OPT, typename GradT, int NCORR = 127>
__device__ __forceinline__ void load6_global(const TArg& T, int64_t base, int lane, TileIn6<GradT, NCORR>& in) {
  constexpr bool ADAM = (OPT == FO_OPT_ADAMW);
  constexpr int E = FEPL, NW = E / 2, NB = E / 4, NG = TileIn6<GradT, NCORR>::NG, NR = TileIn6<GradT, NCORR>::NR;
  const int64_t n = T.n;
  const int64_t e0 = base + (int64_t)lane * E;
  if (e0 + E <= n) {
    // a lane whose 16 elements are all inside the tensor: 128-bit loads (the
    // fused paths take 16-byte aligned views only, and e0 is a multiple of 16)
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const uint4 a = ldcs4(T.lp + e0 + 8 * c);
      in.lw[4 * c] = a.x; in.lw[4 * c + 1] = a.y; in.lw[4 * c + 2] = a.z; in.lw[4 * c + 3] = a.w;
    }
#pragma unroll
    for (int c = 0; c < NG / 4; ++c) {
      const uint4 a = ldcs4(reinterpret_cast<const GradT*>(T.g) + e0 + (16 / sizeof(GradT)) * c);
      in.gw[4 * c] = a.x; in.gw[4 * c + 1] = a.y; in.gw[4 * c + 2] = a.z; in.gw[4 * c + 3] = a.w;
    }
    if (NCORR == 127) {
      load_bytes<4>(T.rho + e0, in.rw);
    } else {
      load_bytes<4>(reinterpret_cast<const int16_t*>(T.rho) + e0, in.rw);
      load_bytes<4>(reinterpret_cast<const int16_t*>(T.rho) + e0 + 8, in.rw + 4);
    }
    load_bytes<4>(T.mq + e0, in.mw);
    if (ADAM) load_bytes<4>(T.vq + e0, in.vw);
    else {
#pragma unroll
      for (int q = 0; q < NB; ++q) in.vw[q] = 0;
    }
    in.msb = T.ms[e0 >> 5];
    in.vsb = ADAM ? (uint32_t)T.vs[e0 >> 5] : 0u;
    return;
  }
  // elements past n: weight 1.0 (0x3F80), zero correction, codes, scales
  // and gradient -- their m and v are 0 (no effect on a group maximum) and
  // their updated weight stays near 1, so they trip no guard; they are
  // never stored
#pragma unroll
  for (int q = 0; q < NW; ++q) in.lw[q] = 0x3F803F80u;
#pragma unroll
  for (int q = 0; q < NG; ++q) in.gw[q] = 0;
#pragma unroll
  for (int q = 0; q < NB; ++q) in.mw[q] = in.vw[q] = 0;
#pragma unroll
  for (int q = 0; q < NR; ++q) in.rw[q] = 0;
#pragma unroll
  for (int j = 0; j < E; ++j) {
    const int64_t i = e0 + j;
    if (i < n) {
      in.lw[j >> 1] = (in.lw[j >> 1] & (0xFFFF0000u >> (16 * (j & 1)))) | ((uint32_t)T.lp[i] << (16 * (j & 1)));
      if (NCORR == 127) in.rw[j >> 2] |= (uint32_t)(uint8_t)T.rho[i] << (8 * (j & 3));
      else in.rw[j >> 1] |= (uint32_t)reinterpret_cast<const uint16_t*>(T.rho)[i] << (16 * (j & 1));
      in.mw[j >> 2] |= (uint32_t)(uint8_t)T.mq[i] << (8 * (j & 3));
      if (ADAM) in.vw[j >> 2] |= (uint32_t)T.vq[i] << (8 * (j & 3));
      if (sizeof(GradT) == 2)
        in.gw[j >> 1] |= (uint32_t)reinterpret_cast<const uint16_t*>(T.g)[i] << (16 * (j & 1));
      else
        in.gw[j] = reinterpret_cast<const uint32_t*>(T.g)[i];
    }
  }
  in.msb = e0 < n ? (uint32_t)T.ms[e0 >> 5] : 0u;
  in.vsb = (ADAM && e0 < n) ? (uint32_t)T.vs[e0 >> 5] : 0u;
}

// Sources of one lane's 16 elements, read half (8 elements) at a time so
// only half of the packed inputs is live at once.
template <int OPT, typename GradT, int NCORR = 127>
struct SmemSrc {  // a full tile in the stage ring (read in place)
  static constexpr int NGH = TileIn6<GradT, NCORR>::NG / 2;
  const uint8_t *lp, *g, *rho, *mq, *vq;
  uint32_t msb, vsb;
  uint32_t release_bar;  // mbarrier to arrive on once the second half is read (0: none)
  __device__ __forceinline__ void half(int h, uint32_t* lw, uint32_t* gw, uint32_t* rw, uint32_t* mw,
                                       uint32_t* vw) const {
    const uint4 a = *reinterpret_cast<const uint4*>(lp + 16 * h);
    lw[0] = a.x; lw[1] = a.y; lw[2] = a.z; lw[3] = a.w;
#pragma unroll
    for (int c = 0; c < NGH / 4; ++c) {
      const uint4 b = *reinterpret_cast<const uint4*>(g + 4 * NGH * h + 16 * c);
      gw[4 * c] = b.x; gw[4 * c + 1] = b.y; gw[4 * c + 2] = b.z; gw[4 * c + 3] = b.w;
    }
    if (NCORR == 127) {
      const uint2 r = *reinterpret_cast<const uint2*>(rho + 8 * h);
      rw[0] = r.x; rw[1] = r.y;
    } else {
      const uint4 r = *reinterpret_cast<const uint4*>(rho + 16 * h);
      rw[0] = r.x; rw[1] = r.y; rw[2] = r.z; rw[3] = r.w;
    }
    const uint2 m = *reinterpret_cast<const uint2*>(mq + 8 * h);
    mw[0] = m.x; mw[1] = m.y;
    if (OPT == FO_OPT_ADAMW) {
      const uint2 v = *reinterpret_cast<const uint2*>(vq + 8 * h);
      vw[0] = v.x; vw[1] = v.y;
    }
    if (h == 1 && release_bar) {
      // the warp's last reads of this stage are issued: release it now (the
      // arrive's release semantics order the reads before the producer's
      // next bulk copy into the stage), half a tile before the compute ends
      __syncwarp();
      if ((threadIdx.x & 31) == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(release_bar) : "memory");
    }
  }
};

template <typename GradT, int NCORR = 127>
struct RegSrc {  // a partial tile already gathered into registers
  static constexpr int NGH = TileIn6<GradT, NCORR>::NG / 2;
  static constexpr int NRH = TileIn6<GradT, NCORR>::NR / 2;
  const TileIn6<GradT, NCORR>& in;
  uint32_t msb, vsb;
  __device__ __forceinline__ void half(int h, uint32_t* lw, uint32_t* gw, uint32_t* rw, uint32_t* mw,
                                       uint32_t* vw) const {
#pragma unroll
    for (int q = 0; q < 4; ++q) lw[q] = in.lw[4 * h + q];
#pragma unroll
    for (int q = 0; q < NGH; ++q) gw[q] = in.gw[NGH * h + q];
#pragma unroll
    for (int q = 0; q < NRH; ++q) rw[q] = in.rw[NRH * h + q];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      mw[q] = in.mw[2 * h + q];
      vw[q] = in.vw[2 * h + q];
    }
  }
};

// A tripped guard does not recompute in place: lane 0 sets bit `fix_idx` of
// `fix` and the tile stores nothing, so its inputs stay intact in global
// memory for the fix-up launch that follows every fused launch
// (step_fixup_kernel: process_tile_exact on the flagged slices, which also
// sets the reference's error bits).  The fast kernel carries no fallback code.
// Primitives of the fast tile and their IEEE forms (SAFE re-run, fix-up launch).
template <bool SAFE>
__device__ __forceinline__ float2 quot_y(float2 a, float b, float y) {  // a / b, y = RN(1/b)
  if (SAFE) return make_float2(__fdiv_rn(a.x, b), __fdiv_rn(a.y, b));
  return fast::div_y(a, fast::dup(b), fast::dup(y));
}
template <bool SAFE>
__device__ __forceinline__ float2 quot(float2 a, float2 b) {
  if (SAFE) return make_float2(__fdiv_rn(a.x, b.x), __fdiv_rn(a.y, b.y));
  return fast::div_rn2(a, b);
}
template <bool SAFE>
__device__ __forceinline__ float2 root2(float2 x) {
  if (SAFE) return make_float2(__fsqrt_rn(x.x), __fsqrt_rn(x.y));
  return fast::sqrt_rn2(x);
}

// SAFE = true (the fix-up launch only): the same tile with IEEE division /
// square root and the exact reconstruct / split of fo_math.cuh, so only the
// reference's error conditions (non-finite values, rho = -128, scale
// overflow) remain; those go to process_tile_exact, which reports them.
template <int OPT, typename GradT, int BC, class Src, class Lut, bool SAFE = false, int NCORR = 127,
          bool LINEAR = false, bool PEER = false>
__device__ __forceinline__ void compute_tile6(const TArg& T, const fo_hparams& h, int64_t base, int lane,
                                              uint32_t& err, const Lut& L, float negzero, uint32_t* fix,
                                              uint32_t fix_idx, bool full, const Src& in,
                                              const PeerSet& peers = PeerSet{nullptr, 0}) {
  using namespace fast;
  constexpr bool ADAM = (OPT == FO_OPT_ADAMW);
  constexpr int E = FEPL, NW = E / 2, NB = E / 4, LPG = GROUP / E;
  // Every product that feeds an addition is an FFMA2 with this run-time -0:
  // RN(a*b + -0) == RN(a*b) bit for bit, and ptxas cannot contract it into
  // the following add (it does contract plain f32x2 mul+add, .rn or not).
  const float2 Z = dup(negzero);
  const int64_t n = T.n;
  const int64_t e0 = base + (int64_t)lane * E;
  // steady-state AdamW keeps the variance roots scaled by 2^30 (RSCALED):
  // every use of them is a max, a quotient by the group scale or the sum
  // with eps, and all three take the exact power-of-two scaling for free
  constexpr bool RSCALED = FO_ROOT_SCALED && ADAM && FO_SQRT_WIDE && (BC & 2) && !SAFE;
  // ... which the variance epilogue sees only when it quantises the roots
  // (companded); the linear ablation quantises v itself
  constexpr bool QSCALED = RSCALED && !LINEAR;
  constexpr float RS = QSCALED ? 0x1p30f : 1.0f;
  // int16 corrections (formats.py:94-95): no R(rho) table; the reconstruct
  // and the split compute with N = 32767 (see below)
  constexpr bool C16 = NCORR != 127;
  static_assert(!SAFE || (!C16 && !LINEAR), "the SAFE tile is the int8 / companded layout's");
  constexpr int RB = Corr<NCORR>::RB;
#ifdef FO_COPY_ONLY
  // bandwidth/power experiment: same loads and stores, no arithmetic
  if (!C16 && full) {
    uint32_t hl[4], hg[TileIn6<GradT>::NG / 2], hr[2], hm[2], hv[2], a[8], b[4], c[4], d[4];
    for (int hh = 0; hh < 2; ++hh) {
      in.half(hh, hl, hg, hr, hm, hv);
      for (int q = 0; q < 4; ++q) a[4 * hh + q] = hl[q] ^ hg[q & (TileIn6<GradT>::NG / 2 - 1)];
      b[2 * hh] = hr[0]; b[2 * hh + 1] = hr[1];
      c[2 * hh] = hm[0]; c[2 * hh + 1] = hm[1];
      d[2 * hh] = hv[0]; d[2 * hh + 1] = hv[1];
    }
    stcs4(T.lp + e0, make_uint4(a[0], a[1], a[2], a[3]));
    stcs4(T.lp + e0 + 8, make_uint4(a[4], a[5], a[6], a[7]));
    store_bytes<4>(T.rho + e0, b);
    store_bytes<4>(T.mq + e0, c);
    if (ADAM) store_bytes<4>(T.vq + e0, d);
    if ((lane & 1) == 0) {
      T.ms[e0 >> 5] = (uint16_t)in.msb;
      if (ADAM) T.vs[e0 >> 5] = (uint16_t)in.vsb;
    }
    return;
  }
#endif

  // ---- input guards (accumulated over the packed inputs in the loop) ----
  // The fast divisions / square roots need their operands away from the
  // underflow range.  FO_VG (default): guard the operands themselves --
  // AdamW: every nonzero |m| >= 2^-84 and v >= 2^-94;
  // SGD / Lion divide m only to quantise it, where a tiny m gives code 0
  // either way, so they need no guard.  FO_VG=0: the older, stronger
  // condition on the inputs, 0 < |g| < 2^-35 trips.  rho == -128
  // (formats.py:270-271): as signed 16-bit lanes, a word whose high byte is
  // 0x80 is below -32512, and the shifted copy covers the low bytes.
  constexpr bool VG = FO_VG != 0;
  bool bad = false;
  uint32_t gmin = 0xFFFFFFFFu, rmin = 0x7FFF7FFFu, gnf = 0;
  // min over 2 * (bits of |m|, v) - 2: the sign bit shifts out, +-0 maps to the top
  uint32_t mlo = 0xFFFFFFFFu, vlo = 0xFFFFFFFFu;
  // A non-finite input scale makes every dequantised value of its group
  // non-finite (quantize.py:131,157): exact path.
  bad |= (in.msb & 0x7C00u) == 0x7C00u;
  if (ADAM) bad |= (in.vsb & 0x7C00u) == 0x7C00u;

  // ---- per pair: reconstruct, dequantise, update, split ----
  // One pass per pair keeps only m, the variance root and the packed
  // outputs live across the tile (the group maxima need all 16 elements).
  const float msf = half_bits_to_float(in.msb);
  const float vsf = half_bits_to_float(in.vsb);
  float m[E], root[E];
  uint32_t cw[NW], ro[NB * RB];
  float tmin = 3.0e38f, tmax = 0.0f;
  constexpr int NGH = TileIn6<GradT>::NG / 2;
  uint32_t hl[4], hg[NGH], hr[2 * RB], hm[2], hv[2];
#pragma unroll
  for (int k = 0; k < NW; ++k) {
    const int j = 2 * k;
    if ((k & 3) == 0) {
      in.half(k >> 2, hl, hg, hr, hm, hv);
      if (SAFE) {  // only non-finite gradients matter here (optim.py:182-183)
        if (sizeof(GradT) == 2) {
#pragma unroll
          for (int q = 0; q < NGH; ++q) gnf |= __vcmpeq2(hg[q] & 0x7F807F80u, 0x7F807F80u);
        } else {
#pragma unroll
          for (int q = 0; q < NGH; ++q) gnf |= (hg[q] & 0x7F800000u) == 0x7F800000u;
        }
      } else if (VG) {
      } else if (sizeof(GradT) == 2) {
#pragma unroll
        for (int q = 0; q < NGH; ++q) gmin = __vminu2(gmin, __vsub2(hg[q] & 0x7FFF7FFFu, 0x00010001u));
      } else {
#pragma unroll
        for (int q = 0; q < NGH; ++q) gmin = min(gmin, hg[q] * 2u - 1u);
      }
      if (C16) {  // rho == -32768 (formats.py:270-271)
#pragma unroll
        for (int q = 0; q < 4; ++q) rmin = __vmins2(rmin, hr[q]);
      } else {
#pragma unroll
        for (int q = 0; q < 2; ++q) if (FO_PROBE != 4) rmin = __vmins2(rmin, __vmins2(hr[q], hr[q] << 8));
      }
    }
    const uint32_t w = hl[k & 3];
    const uint32_t rwd = C16 ? hr[k & 3] : hr[(j >> 2) & 1], mwd = hm[(j >> 2) & 1], vwd = hv[(j >> 2) & 1];
    // reconstruct (formats.py:248-276), see the header comment
    // lp +- R as one IMAD (fast::recon_bits)
    float2 th2;
    if (SAFE) {  // formats.py:248-276 restated (fo_math.cuh)
      const int ql = (int)(int8_t)(rwd >> (8 * (j & 3))), qh = (int)(int8_t)(rwd >> (8 * ((j & 3) + 1)));
      th2 = make_float2(reconstruct1(w & 0xFFFFu, ql, __fdiv_rn((float)ql, 127.0f)),
                        reconstruct1(w >> 16, qh, __fdiv_rn((float)qh, 127.0f)));
    } else if (C16) {
      // R(rho) = rint_even(RN(rho/32767) * 2^15) computed: the Markstein
      // quotient with RN(1/32767) is exact for every int16 code
      // (tests/test_gpu_g32.py::test_int16_every_code), * 2^15 is exact, and
      // the magic add rounds half-even; |R| <= 2^15 < 2^16 keeps lp + R
      // inside lp's binade exactly as for int8
      const float2 q2 = div_y(make_float2((float)(int)(int16_t)(rwd & 0xFFFFu), (float)((int)rwd >> 16)),
                              dup(32767.0f), dup(0x1.0002p-15f));
      const float2 t2 = fma2(q2, dup(32768.0f), dup(12582912.0f));
      const int rl = (int)(__float_as_uint(t2.x) - 0x4B400000u), rh = (int)(__float_as_uint(t2.y) - 0x4B400000u);
      th2 = make_float2(__uint_as_float(recon_bits(w << 16, rl)), __uint_as_float(recon_bits(w & 0xFFFF0000u, rh)));
    } else if (!FO_R_LUT) {
      // R(rho) = rint(rho * RN(32768/127)) in one FFMA2: rho * 32768/127 is
      // at least 0.5/127 away from any half-integer and RN(32768/127) moves
      // rho * it by < 0.002, so this equals rint_even(RN(rho/127) * 2^15)
      // for every int8 code (tests/test_reconstruct_int.py).  float(rho)
      // exactly: bytes (rho + 128) | 0x4B000000 = 2^23 + rho + 128.
      const uint32_t wx = rwd ^ 0x80808080u;
      const float2 fx = make_float2(__uint_as_float(prmt(wx, 0x4B000000u, 0x7440u + (j & 3))),
                                    __uint_as_float(prmt(wx, 0x4B000000u, 0x7441u + (j & 3))));
      const float2 t2 = fma2(add2(fx, dup(-8388736.0f)), dup(32768.0f / 127.0f), dup(12582912.0f));
      const int rl = (int)(__float_as_uint(t2.x) - 0x4B400000u), rh = (int)(__float_as_uint(t2.y) - 0x4B400000u);
      th2 = make_float2(__uint_as_float(recon_bits(w << 16, rl)), __uint_as_float(recon_bits(w & 0xFFFF0000u, rh)));
    } else {
      const int rl = L.r(rwd, j & 3);
      const int rh = L.r(rwd, (j & 3) + 1);
      th2 = make_float2(__uint_as_float(recon_bits(w << 16, rl)), __uint_as_float(recon_bits(w & 0xFFFF0000u, rh)));
    }
    // dequantise (quantize.py:125-131, :152-158)
#if FO_PROBE == 5  // energy probe (not exact): no moment LUT lookups
    const float2 u2 = make_float2(__uint_as_float(0x3F000000u | ((mwd >> (8 * (j & 3))) & 0xFFu)),
                                  __uint_as_float(0x3F000000u | (mwd & 0xFF00u)));
#else
    const float2 u2 = make_float2(L.m(mwd, j & 3), L.m(mwd, (j & 3) + 1));
#endif
    const float2 mp2 = fma2(u2, dup(msf), Z);
    float2 g2;
    if (sizeof(GradT) == 2) {
      const uint32_t gwd = hg[k & 3];
      g2 = make_float2(__uint_as_float(gwd << 16), __uint_as_float(gwd & 0xFFFF0000u));
    } else {
      g2 = make_float2(__uint_as_float(hg[j & 7]), __uint_as_float(hg[(j & 7) + 1]));
    }
    // update (optim.py:195-198, :220-226, :247-249)
    float2 m2, tn2;
    if (OPT == FO_OPT_ADAMW) {
#if FO_PROBE == 5
      const float2 z2 = make_float2(__uint_as_float(0x3F000000u | ((vwd >> (8 * (j & 3))) & 0xFFu)),
                                    __uint_as_float(0x3F000000u | (vwd & 0xFF00u)));
#else
      const float2 z2 = make_float2(L.v(vwd, j & 3), L.v(vwd, (j & 3) + 1));
#endif
      const float2 r2 = fma2(z2, dup(vsf), Z);              // quantize.py:157 (linear: v itself, :185)
      const float2 vp2 = LINEAR ? r2 : fma2(r2, r2, Z);
      m2 = add2(fma2(dup(h.b1), mp2, Z), fma2(dup(h.omb1), g2, Z));
      const float2 v2 = add2(fma2(dup(h.b2), vp2, Z), fma2(dup(h.omb2), fma2(g2, g2, Z), Z));
      constexpr bool WIDE_ROOT = FO_SQRT_WIDE && (BC & 2) && !SAFE;
      if (!SAFE && VG) {
        if (FO_PROBE != 4) mlo = __vimin3_u32(mlo, (__float_as_uint(m2.x) << 1) - 2u, (__float_as_uint(m2.y) << 1) - 2u);
        if (!WIDE_ROOT) vlo = __vimin3_u32(vlo, (__float_as_uint(v2.x) << 1) - 2u, (__float_as_uint(v2.y) << 1) - 2u);
      }
      const float2 mh = (BC & 1) ? m2 : quot_y<SAFE>(m2, h.bc1, h.rbc1);
      float2 rt2;  // RN(sqrt(v)), also quantize.py:145
      float2 den;
      if (BC & 2) {
        if (RSCALED) {
          // root * 2^30 (sqrt_rn2_wide without its final exact * 2^-30); the
          // 2^-30 is folded into den's FFMA2 and the variance epilogue
          rt2 = sqrt_rn2(mul2(v2, dup(0x1p60f)));
          den = fma2(rt2, dup(0x1p-30f), dup(h.eps));  // RN(root + eps): root'*2^-30 is exact
        } else {
          rt2 = WIDE_ROOT ? sqrt_rn2_wide(v2) : root2<SAFE>(v2);
          den = add2(rt2, dup(h.eps));
        }
      } else {
        if (!LINEAR) rt2 = root2<SAFE>(v2);
        den = add2(root2<SAFE>(quot_y<SAFE>(v2, h.bc2, h.rbc2)), dup(h.eps));
      }
      // the quantity the variance epilogue groups: the root (companded) or v (linear)
      root[j] = LINEAR ? v2.x : rt2.x;
      root[j + 1] = LINEAR ? v2.y : rt2.y;
#if FO_PROBE == 3  // energy probe (not exact): no division in the update
      const float2 u = add2(mul2(mh, den), fma2(dup(h.wd), th2, Z));
#else
      const float2 u = add2(quot<SAFE>(mh, den), fma2(dup(h.wd), th2, Z));
#endif
      tn2 = add2(th2, neg2(fma2(dup(h.lr), u, Z)));
    } else if (OPT == FO_OPT_SGD) {
      m2 = add2(fma2(dup(h.mu), mp2, Z), g2);
      const float2 u = add2(m2, fma2(dup(h.wd), th2, Z));
      tn2 = add2(th2, neg2(fma2(dup(h.lr), u, Z)));
    } else {
      const float2 c2 = add2(fma2(dup(h.b1), mp2, Z), fma2(dup(h.omb1), g2, Z));
      // np.sign with sign(+-0) = +0: copysign(1, c), or +0 for c == 0.  A
      // NaN c (non-finite input) makes m NaN too, which sends the tile to
      // the exact path, so NaN need not propagate here.
      const float2 s2 = make_float2(
          __uint_as_float(c2.x == 0.0f ? 0u : ((__float_as_uint(c2.x) & 0x80000000u) | 0x3F800000u)),
          __uint_as_float(c2.y == 0.0f ? 0u : ((__float_as_uint(c2.y) & 0x80000000u) | 0x3F800000u)));
      m2 = add2(fma2(dup(h.b2), mp2, Z), fma2(dup(h.omb2), g2, Z));
      const float2 u = add2(s2, fma2(dup(h.wd), th2, Z));
      tn2 = add2(th2, neg2(fma2(dup(h.lr), u, Z)));
    }
    m[j] = m2.x;
    m[j + 1] = m2.y;
    // split (formats.py:232-245)
    uint32_t pr;  // the two correction codes in bytes 0, 1 (int16: halves 0, 1)
    if (SAFE) {
      uint32_t cl, ch;
      int ql, qh;
      split1<127>(tn2.x, cl, ql);
      split1<127>(tn2.y, ch, qh);
      cw[k] = cl | (ch << 16);
      pr = (uint32_t)(ql & 0xFF) | ((uint32_t)(qh & 0xFF) << 8);
    } else {
      __nv_bfloat162 c2 = __floats2bfloat162_rn(tn2.x, tn2.y);  // RNE, overflow -> inf
      cw[k] = *reinterpret_cast<uint32_t*>(&c2);
      const float2 lp2 = make_float2(__uint_as_float(cw[k] << 16), __uint_as_float(cw[k] & 0xFFFF0000u));
      const float2 e2 = add2(tn2, neg2(lp2));  // exact residual
      if (C16) {
        // e_n = e * 2^-ell exactly; rho = rint(RN(e_n * 32767)) (formats.py:
        // 223-225) -- the product is not exact, so RN first, then rint.
        // K16 = 32767 * 2^-ell * 2^-21 = (32767/16384) * 2^(128 - expf): one
        // LOP3; RN(e*K16) = RN(e_n*32767) * 2^-21 and 6.0 has ulp 2^-21
        const float2 k2 = make_float2(__uint_as_float(k16_bits(__float_as_uint(tn2.x))),
                                      __uint_as_float(k16_bits(__float_as_uint(tn2.y))));
        // (the product is an FFMA2 with -0 so ptxas cannot contract it into
        // the add: that would round the exact product once, not twice)
        const float2 t2 = add2(fma2(e2, k2, Z), dup(6.0f));
        pr = prmt(__float_as_uint(t2.x), __float_as_uint(t2.y), 0x5410u);
      } else {
#if FO_SPLIT_K13
      // K = 127 * 2^-ell with ell = expf(theta) - 135 (the binade-bottom rule
      // is implied by theta's own exponent).  K * 2^-13 = (127/64) *
      // 2^(128 - expf) has exponent field 255 - expf, i.e. the complement of
      // theta's: ONE LOP3 per element, normal for every expf in [1, 254].
      const float2 k2 = make_float2(__uint_as_float(k13_bits(__float_as_uint(tn2.x))),
                                    __uint_as_float(k13_bits(__float_as_uint(tn2.y))));
      // e*K*2^-13 is exact (<= 24 significant bits, |.| < 2^-6) and 1536 has
      // ulp 2^-13, so RN(e*K*2^-13 + 1536) = 1536 + rint(e*K) * 2^-13
      // (ties-to-even): the code sits in the low mantissa bits.
      const float2 q2 = fma2(e2, k2, dup(1536.0f));
#else
      // K = 127 * 2^-ell with ell = expf(theta) - 135: the binade-bottom rule
      // is implied by theta's own exponent; valid for expf(theta) in [14, 254].
      const float2 k2 = make_float2(__uint_as_float(0x867E0000u - (__float_as_uint(tn2.x) & 0x7F800000u)),
                                    __uint_as_float(0x867E0000u - (__float_as_uint(tn2.y) & 0x7F800000u)));
      // e*K is exact (<= 24 significant bits), so adding 1.5*2^23 in the same
      // FFMA2 leaves rint(e*K) (ties-to-even) in the low mantissa bits.
      const float2 q2 = fma2(e2, k2, dup(12582912.0f));
#endif
      pr = prmt(__float_as_uint(q2.x), __float_as_uint(q2.y), 0x0040u);
      }
    }
    if (C16) ro[k] = pr;
    else if (k & 1) ro[k >> 1] = prmt(ro[k >> 1], pr, 0x5410u);
    else ro[k >> 1] = pr;
    if (FO_PROBE != 4) {
      tmin = fminf(tmin, fminf(fabsf(tn2.x), fabsf(tn2.y)));
      tmax = maxnan3(tmax, fabsf(tn2.x), fabsf(tn2.y));
    }
  }
  // |theta_new| in [2^-113, bf16 max): the split's exponent rule holds, and
  // the reconstruct's zero cases (NaN, or a zero whose sign may differ from
  // the reference's) are excluded.  NaN fails both comparisons.
  if (SAFE) {
    // only the reference's error conditions remain: a non-finite weight
    // (split-nonfinite) or gradient (gradient-nonfinite)
    bad |= !(tmax <= 3.4028235e38f) || gnf != 0;
  } else {
    bad |= !(tmin >= 0x1p-113f) || !(tmax < 0x1.FFp127f);
    if (VG) {
      if (ADAM) bad |= mlo < 2u * 0x15800000u - 2u || vlo < 2u * 0x10800000u - 2u;  // 0 < |m| < 2^-84, 0 < v < 2^-94
      // (vlo stays at its initial maximum when the wide root needs no v guard)
    } else if (sizeof(GradT) == 2) {
      bad |= __vcmpltu2(gmin, 0x2DFF2DFFu) != 0;
    } else {
      bad |= gmin < (0x2E000000u * 2u - 1u);
    }
  }
  bad |= __vcmplts2(rmin, C16 ? 0x80018001u : 0x81008100u) != 0;

  // ---- epilogue: momentum (quantize.py:109-122), exact ----
  float amax = 0.0f;
#pragma unroll
  for (int j = 0; j < E; j += 2) amax = maxnan3(amax, fabsf(m[j]), fabsf(m[j + 1]));
#pragma unroll
  for (int o = 1; o < LPG; o <<= 1) amax = maxnan(amax, __shfl_xor_sync(0xffffffffu, amax, o));
  bad |= !(amax <= 65504.0f);  // non-finite m or scale overflow: exact path reports it
  const uint32_t new_msb = (uint32_t)__half_as_ushort(__float2half_ru(amax));
  uint32_t mo[NB];
  {
    const float s = half_bits_to_float(new_msb);
    const float den = (s == 0.0f) ? 1.0f : s;
    const float y = rcp_rn_normal(den);
#if FO_MQ_APPROX
    if (!SAFE) {
      // T = 254 m' / (1 + |m'|) without the two exact quotients: m' ~ m *
      // RN(254 / s), 1 + |m'| by one FFMA, one MUFU reciprocal.  |T - T_ref|
      // < 2^-12 against the reference's RN(RN(RN(m/s) / RN(1 + |m/s|)) * 254)
      // (error budget in DESIGN.md §3.2; selftest modes 8-9), so wherever T
      // is at least 2^-12 away from a half-integer rint(T) is the reference's
      // code.  A lane with any element closer than that recomputes its codes
      // exactly below (one element in ~2000).
      const float y254 = __fmul_rn(y, 254.0f);
      float emax = 0.0f;
#pragma unroll
      for (int j = 0; j < E; j += 2) {
        const float2 T = mq_T(make_float2(m[j], m[j + 1]), y254);
        const float2 t = add2(T, dup(12582912.0f));  // rint(T) in the low bits
        const float2 e = add2(T, neg2(add2(t, dup(-12582912.0f))));  // T - rint(T)
        emax = fmaxf(emax, fmaxf(fabsf(e.x), fabsf(e.y)));
        const uint32_t pr = prmt(__float_as_uint(t.x), __float_as_uint(t.y), 0x0040u);
        if (j & 2) mo[j >> 2] = prmt(mo[j >> 2], pr, 0x5410u);
        else mo[j >> 2] = pr;
      }
      if (!(emax <= 0.5f - 0x1p-12f)) {
#pragma unroll
        for (int j = 0; j < E; j += 2) {
          const float2 mn = quot_y<SAFE>(make_float2(m[j], m[j + 1]), den, y);
          const float2 d = make_float2(__fadd_rn(1.0f, fabsf(mn.x)), __fadd_rn(1.0f, fabsf(mn.y)));
          const float2 zh = quot<SAFE>(mn, d);
          const float2 t = add2(fma2(zh, dup(254.0f), Z), dup(12582912.0f));
          const uint32_t pr = prmt(__float_as_uint(t.x), __float_as_uint(t.y), 0x0040u);
          if (j & 2) mo[j >> 2] = prmt(mo[j >> 2], pr, 0x5410u);
          else mo[j >> 2] = pr;
        }
      }
    } else {
#else
    {
#endif
#pragma unroll
    for (int j = 0; j < E; j += 2) {
#if FO_PROBE == 1  // energy probe (not exact): momentum codes by one multiply
      const float2 zh = mul2(make_float2(m[j], m[j + 1]), dup(y));
#else
      const float2 mn = quot_y<SAFE>(make_float2(m[j], m[j + 1]), den, y);  // RN(m/s)
      const float2 d = make_float2(__fadd_rn(1.0f, fabsf(mn.x)), __fadd_rn(1.0f, fabsf(mn.y)));
      // RN(2m'/(1+|m'|)) = 2*RN(m'/(1+|m'|)) (power-of-two scaling), so
      // RN(z*127) = RN(RN(m'/d)*254)
      const float2 zh = quot<SAFE>(mn, d);
#endif
      const float2 t = add2(fma2(zh, dup(254.0f), Z), dup(12582912.0f));  // rint(RN(z*127))
      const uint32_t pr = prmt(__float_as_uint(t.x), __float_as_uint(t.y), 0x0040u);
      if (j & 2) mo[j >> 2] = prmt(mo[j >> 2], pr, 0x5410u);
      else mo[j >> 2] = pr;
    }
    }
  }

  // ---- epilogue: variance (quantize.py:134-149), exact ----
  uint32_t new_vsb = 0, vo[NB];
  if (ADAM) {
    float rmax = 0.0f;
#pragma unroll
    for (int j = 0; j < E; j += 2) rmax = maxnan3(rmax, root[j], root[j + 1]);
#pragma unroll
    for (int o = 1; o < LPG; o <<= 1) rmax = maxnan(rmax, __shfl_xor_sync(0xffffffffu, rmax, o));
    bad |= !(rmax <= 65504.0f * RS);
    new_vsb = (uint32_t)__half_as_ushort(__float2half_ru(QSCALED ? __fmul_rn(rmax, 1.0f / RS) : rmax));
    const float s = half_bits_to_float(new_vsb);
    // RSCALED: RN(root'/(s*2^30)) with y = RN(1/s)*2^-30 is the same
    // Markstein quotient as RN(root/s) with every intermediate scaled exactly
    const float den = QSCALED ? __fmul_rn((s == 0.0f) ? 1.0f : s, RS) : ((s == 0.0f) ? 1.0f : s);
    const float y = QSCALED ? __fmul_rn(rcp_rn_normal((s == 0.0f) ? 1.0f : s), 1.0f / RS) : rcp_rn_normal(den);
#pragma unroll
    for (int j = 0; j < E; j += 2) {
#if FO_PROBE == 2  // energy probe (not exact): variance codes by one multiply
      const float2 vn = mul2(make_float2(root[j], root[j + 1]), dup(y));
#else
      const float2 vn = quot_y<SAFE>(make_float2(root[j], root[j + 1]), den, y);  // RN(r/s)
#endif
      const float2 t = add2(fma2(vn, dup(255.0f), Z), dup(12582912.0f));           // rint(RN(vn*255))
      const uint32_t pr = prmt(__float_as_uint(t.x), __float_as_uint(t.y), 0x0040u);
      if (j & 2) vo[j >> 2] = prmt(vo[j >> 2], pr, 0x5410u);
      else vo[j >> 2] = pr;
    }
  }

  // ---- any guard tripped anywhere in the warp: recompute the tile exactly ----
  if (__any_sync(0xffffffffu, bad)) {
    if (SAFE) process_tile_exact<OPT, GradT, FEPL, 127, false, PEER>(T, h, base, lane, fix, &peers);  // `fix` = error word here
    else if (lane == 0) atomicOr(fix + (fix_idx >> 5), 1u << (fix_idx & 31));
    return;
  }

  // ---- stores ----
  if (full) {
#pragma unroll
    for (int c = 0; c < NW / 4; ++c) {
      const uint4 wv = make_uint4(cw[4 * c], cw[4 * c + 1], cw[4 * c + 2], cw[4 * c + 3]);
      stcs4(T.lp + e0 + 8 * c, wv);
      if (PEER)
        for (int r = 0; r < peers.n; ++r) stcs4(peers.at(T.lp + e0 + 8 * c, r), wv);
    }
    if (C16) {
      int16_t* r16 = reinterpret_cast<int16_t*>(T.rho) + e0;
      stcs4(r16, make_uint4(ro[0], ro[1], ro[2], ro[3]));
      stcs4(r16 + 8, make_uint4(ro[4], ro[5], ro[6], ro[7]));
    } else {
      store_bytes<NB>(T.rho + e0, ro);
    }
    store_bytes<NB>(T.mq + e0, mo);
    if (ADAM) store_bytes<NB>(T.vq + e0, vo);
  } else {
#pragma unroll
    for (int j = 0; j < E; ++j) {
      const int64_t i = e0 + j;
      if (i < n) {
        T.lp[i] = (uint16_t)(cw[j >> 1] >> (16 * (j & 1)));
        if (PEER)
          for (int r = 0; r < peers.n; ++r) *peers.at(T.lp + i, r) = (uint16_t)(cw[j >> 1] >> (16 * (j & 1)));
        if (C16) reinterpret_cast<int16_t*>(T.rho)[i] = (int16_t)(ro[j >> 1] >> (16 * (j & 1)));
        else T.rho[i] = (int8_t)(ro[j >> 2] >> (8 * (j & 3)));
        T.mq[i] = (int8_t)(mo[j >> 2] >> (8 * (j & 3)));
        if (ADAM) T.vq[i] = (uint8_t)(vo[j >> 2] >> (8 * (j & 3)));
      }
    }
  }
  if ((lane & (LPG - 1)) == 0 && e0 < n) {
    T.ms[e0 >> 5] = (uint16_t)new_msb;
    if (ADAM) T.vs[e0 >> 5] = (uint16_t)new_vsb;
  }
  (void)err;
}

// A full tile straight from global memory with 128-bit loads.
template <int OPT, typename GradT, int NCORR = 127>
__device__ __forceinline__ void load6_global_full(const TArg& T, int64_t base, int lane, TileIn6<GradT, NCORR>& in) {
  constexpr bool ADAM = (OPT == FO_OPT_ADAMW);
  constexpr int E = FEPL, NG = TileIn6<GradT, NCORR>::NG;
  const int64_t e0 = base + (int64_t)lane * E;
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    const uint4 a = ldcs4(T.lp + e0 + 8 * c);
    in.lw[4 * c] = a.x; in.lw[4 * c + 1] = a.y; in.lw[4 * c + 2] = a.z; in.lw[4 * c + 3] = a.w;
  }
#pragma unroll
  for (int c = 0; c < NG / 4; ++c) {
    const uint4 a = ldcs4(reinterpret_cast<const GradT*>(T.g) + e0 + (16 / sizeof(GradT)) * c);
    in.gw[4 * c] = a.x; in.gw[4 * c + 1] = a.y; in.gw[4 * c + 2] = a.z; in.gw[4 * c + 3] = a.w;
  }
  if (NCORR == 127) {
    load_bytes<4>(T.rho + e0, in.rw);
  } else {
    load_bytes<4>(reinterpret_cast<const int16_t*>(T.rho) + e0, in.rw);
    load_bytes<4>(reinterpret_cast<const int16_t*>(T.rho) + e0 + 8, in.rw + 4);
  }
  load_bytes<4>(T.mq + e0, in.mw);
  if (ADAM) load_bytes<4>(T.vq + e0, in.vw);
  in.msb = T.ms[e0 >> 5];
  in.vsb = ADAM ? (uint32_t)T.vs[e0 >> 5] : 0u;
}

// One flagged slice in the fix-up launch: the SAFE tile (exact everywhere the
// fast one needed guards), or the straight restatement for error cases.
template <int OPT, typename GradT, int BC, int NCORR = 127, bool LINEAR = false, bool PEER = false>
__device__ __forceinline__ void safe_tile(const TArg& T, const fo_hparams& h, int64_t base, int lane, float negzero,
                                          uint32_t* err_out, const PeerSet& peers = PeerSet{nullptr, 0}) {
  if constexpr (NCORR != 127 || LINEAR) {
    // the optional layouts' flagged slices: the straight restatement
    (void)negzero;
    process_tile_exact<OPT, GradT, FEPL, NCORR, LINEAR>(T, h, base, lane, err_out);
    return;
  } else {
    const bool full = (T.n - base) >= FTILE;
    TileIn6<GradT> in;
    if (full) load6_global_full<OPT, GradT>(T, base, lane, in);
    else load6_global<OPT, GradT>(T, base, lane, in);
    const RegSrc<GradT> src{in, in.msb, in.vsb};
    uint32_t err = 0;
    const NoLut L;
    compute_tile6<OPT, GradT, BC, RegSrc<GradT>, NoLut, true, 127, false, PEER>(T, h, base, lane, err, L, negzero,
                                                                               err_out, 0, full, src, peers);
  }
}
