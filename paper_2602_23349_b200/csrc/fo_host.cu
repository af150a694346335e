// fo_host.cu -- fo_step_host(): the reference's calling convention (state and
// gradient in host memory, optim.py:385-459 operate on NumPy arrays) on the
// B200.  The parameter list is cut into group-aligned pieces that are packed
// into device "slots"; each slot goes through
//     H2D copy (stream h2d) -> fused step (stream comp) -> D2H copy (stream d2h)
// and three slots rotate so the copy engines and the SMs overlap.  The call is
// synchronous, like the reference function it replaces.  Pinned host memory
// gives full PCIe bandwidth; pageable memory works but the driver stages it.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <vector>

#include "fo_internal.h"

namespace fo {
namespace {

constexpr int kSlots = 3;
constexpr int64_t kAlign = 512;  // piece offsets inside a slot (tile-aligned)

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
  int64_t off, len;   // element range inside the tensor (off % 32 == 0)
  int64_t slot_off;   // element offset inside the slot
};

struct HostRuntime {
  int device = -1;
  int64_t cap = 0;  // elements per slot
  int rho_bytes = 1, grad_bytes = 2;
  Slot slots[kSlots];
  cudaStream_t h2d = nullptr, comp = nullptr, d2h = nullptr;
  uint32_t* d_err = nullptr;

  void release() {
    for (Slot& s : slots) {
      if (s.base) {
        cudaFree(s.base);
        cudaEventDestroy(s.h2d_done);
        cudaEventDestroy(s.comp_done);
        cudaEventDestroy(s.d2h_done);
        s.base = nullptr;
      }
    }
    cap = 0;
  }

  int ensure(int64_t elems, int rho_b, int grad_b) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return (int)e;
    if (dev == device && elems <= cap && rho_b == rho_bytes && grad_b == grad_bytes) return 0;
    if (device >= 0 && dev != device) {
      release();
      h2d = comp = d2h = nullptr;
      d_err = nullptr;
    }
    release();
    device = dev;
    cap = elems;
    rho_bytes = rho_b;
    grad_bytes = grad_b;
    if (!h2d) {
      cudaStreamCreateWithFlags(&h2d, cudaStreamNonBlocking);
      cudaStreamCreateWithFlags(&comp, cudaStreamNonBlocking);
      cudaStreamCreateWithFlags(&d2h, cudaStreamNonBlocking);
      if ((e = cudaMalloc(&d_err, sizeof(uint32_t))) != cudaSuccess) return (int)e;
    }
    const int64_t ng = cap / 32 + 1;
    const size_t bytes = (size_t)cap * (2 + rho_b + 1 + 1 + grad_b) + (size_t)ng * 4 + 1024;
    for (Slot& s : slots) {
      if ((e = cudaMalloc(&s.base, bytes)) != cudaSuccess) return (int)e;
      uint8_t* p = s.base;
      auto take = [&](size_t n) {
        uint8_t* q = p;
        p += (n + 255) & ~size_t(255);
        return q;
      };
      s.lp = (uint16_t*)take((size_t)cap * 2);
      s.rho = take((size_t)cap * rho_b);
      s.mq = (int8_t*)take((size_t)cap);
      s.vq = take((size_t)cap);
      s.g = take((size_t)cap * grad_b);
      s.ms = (uint16_t*)take((size_t)ng * 2);
      s.vs = (uint16_t*)take((size_t)ng * 2);
      cudaEventCreateWithFlags(&s.h2d_done, cudaEventDisableTiming);
      cudaEventCreateWithFlags(&s.comp_done, cudaEventDisableTiming);
      cudaEventCreateWithFlags(&s.d2h_done, cudaEventDisableTiming);
      cudaEventRecord(s.d2h_done, d2h);
    }
    return 0;
  }
};

HostRuntime g_rt;
std::mutex g_mu;

}  // namespace

int step_host(int opt, const fo_tensor* ts, int32_t nt, const fo_hparams* hps, int32_t nhp, int grad_dtype,
              int rho_bits, int32_t G, int var_scheme, int64_t chunk_elems, uint32_t* h_err) {
  std::lock_guard<std::mutex> lock(g_mu);
  const bool adam = opt == FO_OPT_ADAMW;
  const int rho_b = rho_bits / 8, grad_b = grad_dtype == FO_GRAD_BF16 ? 2 : 4;
  int64_t cap = chunk_elems > 0 ? chunk_elems : (int64_t(1) << 26);
  cap = std::max<int64_t>(kAlign, (cap + kAlign - 1) / kAlign * kAlign);
  if (G <= 0 || cap % G != 0) return FO_EINVAL;
  int rc = g_rt.ensure(cap, rho_b, grad_b);
  if (rc) return rc;
  HostRuntime& R = g_rt;
  cudaMemsetAsync(R.d_err, 0, sizeof(uint32_t), R.comp);

  // cut every tensor into group-aligned pieces and pack them into batches of
  // at most `cap` elements (each piece starts tile-aligned inside the slot)
  std::vector<std::vector<Piece>> batches(1);
  int64_t used = 0;
  const int64_t step = cap / G * G;
  for (int32_t i = 0; i < nt; ++i) {
    for (int64_t off = 0; off < ts[i].n; off += step) {
      const int64_t len = std::min<int64_t>(step, ts[i].n - off);
      const int64_t need = (len + kAlign - 1) / kAlign * kAlign;
      if (used + need > cap) {
        batches.emplace_back();
        used = 0;
      }
      batches.back().push_back(Piece{i, off, len, used});
      used += need;
    }
  }

  std::vector<fo_tensor> dev;
  for (size_t b = 0; b < batches.size(); ++b) {
    const std::vector<Piece>& pcs = batches[b];
    if (pcs.empty()) continue;
    Slot& S = R.slots[b % kSlots];
    cudaStreamWaitEvent(R.h2d, S.d2h_done, 0);  // slot free again
    dev.clear();
    for (const Piece& pc : pcs) {
      const fo_tensor& t = ts[pc.tensor];
      const int64_t g0 = pc.off / G, ng = (pc.len + G - 1) / G, so = pc.slot_off, sg = so / G;
      cudaMemcpyAsync(S.lp + so, (const uint16_t*)t.lp + pc.off, pc.len * 2, cudaMemcpyHostToDevice, R.h2d);
      cudaMemcpyAsync(S.rho + so * rho_b, (const uint8_t*)t.rho + pc.off * rho_b, pc.len * rho_b,
                      cudaMemcpyHostToDevice, R.h2d);
      cudaMemcpyAsync(S.mq + so, (const int8_t*)t.m_codes + pc.off, pc.len, cudaMemcpyHostToDevice, R.h2d);
      cudaMemcpyAsync(S.ms + sg, (const uint16_t*)t.m_scales + g0, ng * 2, cudaMemcpyHostToDevice, R.h2d);
      if (adam) {
        cudaMemcpyAsync(S.vq + so, (const uint8_t*)t.v_codes + pc.off, pc.len, cudaMemcpyHostToDevice, R.h2d);
        cudaMemcpyAsync(S.vs + sg, (const uint16_t*)t.v_scales + g0, ng * 2, cudaMemcpyHostToDevice, R.h2d);
      }
      cudaMemcpyAsync(S.g + so * grad_b, (const uint8_t*)t.grad + pc.off * grad_b, pc.len * grad_b,
                      cudaMemcpyHostToDevice, R.h2d);
      dev.push_back(fo_tensor{S.lp + so, S.rho + so * rho_b, S.mq + so, S.ms + sg, adam ? S.vq + so : nullptr,
                              adam ? S.vs + sg : nullptr, S.g + so * grad_b, pc.len, t.hp_index, 0});
    }
    cudaEventRecord(S.h2d_done, R.h2d);
    cudaStreamWaitEvent(R.comp, S.h2d_done, 0);
    rc = step_mt(opt, dev.data(), (int32_t)dev.size(), hps, nhp, grad_dtype, rho_bits, G, var_scheme, R.d_err,
                 R.comp);
    if (rc) return rc;
    cudaEventRecord(S.comp_done, R.comp);
    cudaStreamWaitEvent(R.d2h, S.comp_done, 0);
    for (const Piece& pc : pcs) {
      const fo_tensor& t = ts[pc.tensor];
      const int64_t g0 = pc.off / G, ng = (pc.len + G - 1) / G, so = pc.slot_off, sg = so / G;
      cudaMemcpyAsync((uint16_t*)t.lp + pc.off, S.lp + so, pc.len * 2, cudaMemcpyDeviceToHost, R.d2h);
      cudaMemcpyAsync((uint8_t*)t.rho + pc.off * rho_b, S.rho + so * rho_b, pc.len * rho_b, cudaMemcpyDeviceToHost,
                      R.d2h);
      cudaMemcpyAsync((int8_t*)t.m_codes + pc.off, S.mq + so, pc.len, cudaMemcpyDeviceToHost, R.d2h);
      cudaMemcpyAsync((uint16_t*)t.m_scales + g0, S.ms + sg, ng * 2, cudaMemcpyDeviceToHost, R.d2h);
      if (adam) {
        cudaMemcpyAsync((uint8_t*)t.v_codes + pc.off, S.vq + so, pc.len, cudaMemcpyDeviceToHost, R.d2h);
        cudaMemcpyAsync((uint16_t*)t.v_scales + g0, S.vs + sg, ng * 2, cudaMemcpyDeviceToHost, R.d2h);
      }
    }
    cudaEventRecord(S.d2h_done, R.d2h);
  }
  cudaError_t e = cudaStreamSynchronize(R.comp);
  if (e == cudaSuccess) e = cudaStreamSynchronize(R.d2h);
  if (e == cudaSuccess) e = cudaStreamSynchronize(R.h2d);
  uint32_t err = 0;
  if (e == cudaSuccess) e = cudaMemcpy(&err, R.d_err, sizeof(uint32_t), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return (int)e;
  if (h_err) *h_err = err;
  return 0;
}

void host_release() {
  std::lock_guard<std::mutex> lock(g_mu);
  g_rt.release();
}

}  // namespace fo
