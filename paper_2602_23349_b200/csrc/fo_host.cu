// fo_host.cu -- fo_step_host(): the reference's calling convention (state and
// gradient in host memory; optim.py:187-258 operate on NumPy arrays) on the
// B200.  The parameter list is cut into group-aligned pieces that are packed
// into device "slots"; each slot goes through
//     H2D copy (stream h2d) -> fused step (stream comp) -> D2H copy (stream d2h)
// and three slots rotate so the copy engines and the SMs overlap.  The call is
// synchronous, like the reference function it replaces.  Pinned host memory
// gives full PCIe bandwidth; pageable memory works but the driver stages it.
//
// Reentrancy: the slots, streams and error word of one call form a context.
// Contexts live in a pool; a call takes an idle context of its device (or
// makes one) and returns it when done, so concurrent calls from several host
// threads never share device buffers and hold no lock while they run.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <vector>

#include "fo_internal.h"

namespace fo {
namespace {

constexpr int kSlots = 3;
constexpr int64_t kAlign = 512;  // element offset of every piece inside a slot (tile-aligned)
constexpr int64_t kScaleAlign = 8;  // fp16 scale offset of every piece (16 bytes: bulk-copy alignment)

struct Slot {
  uint8_t* base = nullptr;  // one allocation per slot
  uint16_t* lp;
  uint8_t* rho;
  int8_t* mq;
  uint16_t* ms;
  uint8_t* vq;
  uint16_t* vs;
  uint8_t* g;
  cudaEvent_t h2d_done, comp_done, d2h_done;
};

struct Piece {
  int32_t tensor;
  int64_t off, len;    // element range inside the tensor (off % G == 0)
  int64_t slot_off;    // element offset inside the slot (multiple of kAlign)
  int64_t scale_off;   // fp16 scale offset inside the slot (multiple of kScaleAlign)
};

// Scale entries a slot needs for pieces of group size G packed into `cap`
// elements: every piece holds <= ceil(len/G) <= len/G + 1 scales plus up to
// kScaleAlign - 1 of padding, and a slot holds at most cap/kAlign pieces.
int64_t scale_cap(int64_t cap, int32_t G) { return cap / G + (cap / kAlign + 1) * kScaleAlign; }

struct HostCtx {
  int device = -1;
  int64_t cap = 0, scap = 0;  // elements / fp16 scales per slot
  int rho_bytes = 0, grad_bytes = 0;
  Slot slots[kSlots];
  cudaStream_t h2d = nullptr, comp = nullptr, d2h = nullptr;
  uint32_t* d_err = nullptr;

  void free_slots() {
    for (Slot& s : slots) {
      if (s.base) {
        cudaFree(s.base);
        cudaEventDestroy(s.h2d_done);
        cudaEventDestroy(s.comp_done);
        cudaEventDestroy(s.d2h_done);
        s.base = nullptr;
      }
    }
    cap = scap = 0;
  }

  void destroy() {
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    free_slots();
    if (h2d) {
      cudaStreamDestroy(h2d);
      cudaStreamDestroy(comp);
      cudaStreamDestroy(d2h);
      cudaFree(d_err);
    }
    cudaSetDevice(prev);
  }

  int ensure(int64_t elems, int64_t scales, int rho_b, int grad_b) {
    cudaError_t e;
    if (!h2d) {
      if ((e = cudaStreamCreateWithFlags(&h2d, cudaStreamNonBlocking)) != cudaSuccess) return (int)e;
      if ((e = cudaStreamCreateWithFlags(&comp, cudaStreamNonBlocking)) != cudaSuccess) return (int)e;
      if ((e = cudaStreamCreateWithFlags(&d2h, cudaStreamNonBlocking)) != cudaSuccess) return (int)e;
      if ((e = cudaMalloc(&d_err, sizeof(uint32_t))) != cudaSuccess) return (int)e;
    }
    if (elems <= cap && scales <= scap && rho_b == rho_bytes && grad_b == grad_bytes) return 0;
    free_slots();
    const size_t bytes = (size_t)elems * (2 + rho_b + 1 + 1 + grad_b) + (size_t)scales * 4 + 8 * 256;
    for (Slot& s : slots) {
      if ((e = cudaMalloc(&s.base, bytes)) != cudaSuccess) {
        s.base = nullptr;
        free_slots();
        return (int)e;
      }
      uint8_t* p = s.base;
      auto take = [&](size_t n) {
        uint8_t* q = p;
        p += (n + 255) & ~size_t(255);
        return q;
      };
      s.lp = (uint16_t*)take((size_t)elems * 2);
      s.rho = take((size_t)elems * rho_b);
      s.mq = (int8_t*)take((size_t)elems);
      s.vq = take((size_t)elems);
      s.g = take((size_t)elems * grad_b);
      s.ms = (uint16_t*)take((size_t)scales * 2);
      s.vs = (uint16_t*)take((size_t)scales * 2);
      cudaEventCreateWithFlags(&s.h2d_done, cudaEventDisableTiming);
      cudaEventCreateWithFlags(&s.comp_done, cudaEventDisableTiming);
      cudaEventCreateWithFlags(&s.d2h_done, cudaEventDisableTiming);
      cudaEventRecord(s.d2h_done, d2h);
    }
    cap = elems;
    scap = scales;
    rho_bytes = rho_b;
    grad_bytes = grad_b;
    return 0;
  }
};

// Idle contexts (all devices).  Only the pool itself is guarded; a call
// holds no lock while it streams.
std::mutex g_pool_mu;
std::vector<HostCtx*> g_idle;

HostCtx* acquire(int dev) {
  std::lock_guard<std::mutex> lock(g_pool_mu);
  for (size_t i = 0; i < g_idle.size(); ++i) {
    if (g_idle[i]->device == dev) {
      HostCtx* c = g_idle[i];
      g_idle.erase(g_idle.begin() + (ptrdiff_t)i);
      return c;
    }
  }
  HostCtx* c = new HostCtx;
  c->device = dev;
  return c;
}

void give_back(HostCtx* c) {
  std::lock_guard<std::mutex> lock(g_pool_mu);
  g_idle.push_back(c);
}

struct CtxLease {
  HostCtx* c;
  explicit CtxLease(int dev) : c(acquire(dev)) {}
  ~CtxLease() { give_back(c); }
};

// Checked enqueue: the first failing CUDA call ends the call with its code.
#define FO_TRY(expr)                         \
  do {                                       \
    cudaError_t e_ = (expr);                 \
    if (e_ != cudaSuccess) return (int)e_;   \
  } while (0)

int run(HostCtx& R, int opt, const fo_tensor* ts, int32_t nt, const fo_hparams* hps, int32_t nhp, int grad_dtype,
        int rho_bits, int32_t G, int var_scheme, int64_t chunk_elems, uint32_t* h_err) {
  const bool adam = opt == FO_OPT_ADAMW;
  const int rho_b = rho_bits / 8, grad_b = grad_dtype == FO_GRAD_BF16 ? 2 : 4;
  int64_t cap = chunk_elems > 0 ? chunk_elems : (int64_t(1) << 26);
  cap = std::max<int64_t>(cap, G);  // a piece holds at least one whole group
  cap = std::max<int64_t>(kAlign, (cap + kAlign - 1) / kAlign * kAlign);
  const int64_t scap = scale_cap(cap, G);
  int rc = R.ensure(cap, scap, rho_b, grad_b);
  if (rc) return rc;
  FO_TRY(cudaMemsetAsync(R.d_err, 0, sizeof(uint32_t), R.comp));

  // Cut every tensor into group-aligned pieces (a multiple of G elements,
  // except a tensor's tail) and pack them into batches of at most `cap`
  // elements and `scap` scales.
  std::vector<std::vector<Piece>> batches(1);
  int64_t used = 0, sused = 0;
  const int64_t step = cap / G * G;
  for (int32_t i = 0; i < nt; ++i) {
    for (int64_t off = 0; off < ts[i].n; off += step) {
      const int64_t len = std::min<int64_t>(step, ts[i].n - off);
      const int64_t need = (len + kAlign - 1) / kAlign * kAlign;
      const int64_t sneed = ((len + G - 1) / G + kScaleAlign - 1) / kScaleAlign * kScaleAlign;
      if (used + need > cap || sused + sneed > scap) {
        batches.emplace_back();
        used = sused = 0;
      }
      batches.back().push_back(Piece{i, off, len, used, sused});
      used += need;
      sused += sneed;
    }
  }

  std::vector<fo_tensor> dev;
  for (size_t b = 0; b < batches.size(); ++b) {
    const std::vector<Piece>& pcs = batches[b];
    if (pcs.empty()) continue;
    Slot& S = R.slots[b % kSlots];
    FO_TRY(cudaStreamWaitEvent(R.h2d, S.d2h_done, 0));  // slot free again
    dev.clear();
    for (const Piece& pc : pcs) {
      const fo_tensor& t = ts[pc.tensor];
      const int64_t g0 = pc.off / G, ng = (pc.len + G - 1) / G, so = pc.slot_off, sg = pc.scale_off;
      const cudaMemcpyKind k = cudaMemcpyHostToDevice;
      FO_TRY(cudaMemcpyAsync(S.lp + so, (const uint16_t*)t.lp + pc.off, pc.len * 2, k, R.h2d));
      FO_TRY(cudaMemcpyAsync(S.rho + so * rho_b, (const uint8_t*)t.rho + pc.off * rho_b, pc.len * rho_b, k, R.h2d));
      FO_TRY(cudaMemcpyAsync(S.mq + so, (const int8_t*)t.m_codes + pc.off, pc.len, k, R.h2d));
      FO_TRY(cudaMemcpyAsync(S.ms + sg, (const uint16_t*)t.m_scales + g0, ng * 2, k, R.h2d));
      if (adam) {
        FO_TRY(cudaMemcpyAsync(S.vq + so, (const uint8_t*)t.v_codes + pc.off, pc.len, k, R.h2d));
        FO_TRY(cudaMemcpyAsync(S.vs + sg, (const uint16_t*)t.v_scales + g0, ng * 2, k, R.h2d));
      }
      FO_TRY(cudaMemcpyAsync(S.g + so * grad_b, (const uint8_t*)t.grad + pc.off * grad_b, pc.len * grad_b, k, R.h2d));
      dev.push_back(fo_tensor{S.lp + so, S.rho + so * rho_b, S.mq + so, S.ms + sg, adam ? S.vq + so : nullptr,
                              adam ? S.vs + sg : nullptr, S.g + so * grad_b, pc.len, t.hp_index, 0});
    }
    FO_TRY(cudaEventRecord(S.h2d_done, R.h2d));
    FO_TRY(cudaStreamWaitEvent(R.comp, S.h2d_done, 0));
    rc = step_mt(opt, dev.data(), (int32_t)dev.size(), hps, nhp, grad_dtype, rho_bits, G, var_scheme, R.d_err,
                 R.comp);
    if (rc) return rc;
    FO_TRY(cudaEventRecord(S.comp_done, R.comp));
    FO_TRY(cudaStreamWaitEvent(R.d2h, S.comp_done, 0));
    for (const Piece& pc : pcs) {
      const fo_tensor& t = ts[pc.tensor];
      const int64_t g0 = pc.off / G, ng = (pc.len + G - 1) / G, so = pc.slot_off, sg = pc.scale_off;
      const cudaMemcpyKind k = cudaMemcpyDeviceToHost;
      FO_TRY(cudaMemcpyAsync((uint16_t*)t.lp + pc.off, S.lp + so, pc.len * 2, k, R.d2h));
      FO_TRY(cudaMemcpyAsync((uint8_t*)t.rho + pc.off * rho_b, S.rho + so * rho_b, pc.len * rho_b, k, R.d2h));
      FO_TRY(cudaMemcpyAsync((int8_t*)t.m_codes + pc.off, S.mq + so, pc.len, k, R.d2h));
      FO_TRY(cudaMemcpyAsync((uint16_t*)t.m_scales + g0, S.ms + sg, ng * 2, k, R.d2h));
      if (adam) {
        FO_TRY(cudaMemcpyAsync((uint8_t*)t.v_codes + pc.off, S.vq + so, pc.len, k, R.d2h));
        FO_TRY(cudaMemcpyAsync((uint16_t*)t.v_scales + g0, S.vs + sg, ng * 2, k, R.d2h));
      }
    }
    FO_TRY(cudaEventRecord(S.d2h_done, R.d2h));
  }
  FO_TRY(cudaStreamSynchronize(R.comp));
  FO_TRY(cudaStreamSynchronize(R.d2h));
  FO_TRY(cudaStreamSynchronize(R.h2d));
  uint32_t err = 0;
  FO_TRY(cudaMemcpy(&err, R.d_err, sizeof(uint32_t), cudaMemcpyDeviceToHost));
  if (h_err) *h_err = err;
  return 0;
}

}  // namespace

int step_host(int opt, const fo_tensor* ts, int32_t nt, const fo_hparams* hps, int32_t nhp, int grad_dtype,
              int rho_bits, int32_t G, int var_scheme, int64_t chunk_elems, uint32_t* h_err) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return (int)e;
  CtxLease lease(dev);
  const int rc = run(*lease.c, opt, ts, nt, hps, nhp, grad_dtype, rho_bits, G, var_scheme, chunk_elems, h_err);
  if (rc) {
    // leave no half-finished work on the context's streams for the next call
    cudaStreamSynchronize(lease.c->h2d);
    cudaStreamSynchronize(lease.c->comp);
    cudaStreamSynchronize(lease.c->d2h);
  }
  return rc;
}

void host_release() {
  std::vector<HostCtx*> idle;
  {
    std::lock_guard<std::mutex> lock(g_pool_mu);
    idle.swap(g_idle);
  }
  for (HostCtx* c : idle) {
    c->destroy();
    delete c;
  }
}

}  // namespace fo
