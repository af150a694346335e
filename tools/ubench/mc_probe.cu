// Probe: a one-device NVLS multicast object in one process, multimem.st
// through its mapping, read back through the unicast mapping.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>
#include <vector>

#define CK(x) do { CUresult r_ = (x); if (r_ != CUDA_SUCCESS) { const char* s_; cuGetErrorString(r_, &s_); \
  printf("%s failed: %d %s\n", #x, (int)r_, s_); return 1; } } while (0)

__global__ void mc_store(uint4* mc, const uint4* src, size_t n16) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v = src[i];
    asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(mc + i), "r"(v.x), "r"(v.y),
                 "r"(v.z), "r"(v.w) : "memory");
  }
}

__global__ void mc_store_bf16(uint4* mc, const uint4* src, size_t n16) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v = src[i];
    asm volatile("multimem.st.global.v4.bf16x2 [%0], {%1, %2, %3, %4};" ::"l"(mc + i), "r"(v.x), "r"(v.y),
                 "r"(v.z), "r"(v.w) : "memory");
  }
}

int main() {
  CK(cuInit(0));
  CUdevice dev;
  CK(cuDeviceGet(&dev, 0));
  CUcontext ctx;
  CK(cuDevicePrimaryCtxRetain(&ctx, dev));
  CK(cuCtxSetCurrent(ctx));
  int mc_ok = 0;
  CK(cuDeviceGetAttribute(&mc_ok, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev));
  printf("multicast supported: %d\n", mc_ok);
  const size_t want = 64ull << 20;
  for (int ht = 0; ht < 3; ++ht) {
    CUmulticastObjectProp mp = {};
    mp.numDevices = 1;
    mp.handleTypes = ht == 0 ? CU_MEM_HANDLE_TYPE_NONE : (ht == 1 ? CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR : CU_MEM_HANDLE_TYPE_FABRIC);
    size_t gmin = 0, grec = 0;
    mp.size = want;
    CUresult r1 = cuMulticastGetGranularity(&gmin, &mp, CU_MULTICAST_GRANULARITY_MINIMUM);
    CUresult r2 = cuMulticastGetGranularity(&grec, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED);
    printf("handleTypes=%d granularity rc=%d/%d min=%zu rec=%zu\n", ht, (int)r1, (int)r2, gmin, grec);
    if (r1) continue;
    size_t size = (want + grec - 1) / grec * grec;
    mp.size = size;
    CUmemGenericAllocationHandle mc;
    CUresult rc = cuMulticastCreate(&mc, &mp);
    printf("  cuMulticastCreate rc=%d size=%zu\n", (int)rc, size);
    if (rc) continue;
    CK(cuMulticastAddDevice(mc, dev));
    CUmemAllocationProp ap = {};
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = 0;
    ap.requestedHandleTypes = (CUmemAllocationHandleType)mp.handleTypes;
    size_t ag = 0;
    CK(cuMemGetAllocationGranularity(&ag, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
    CUmemGenericAllocationHandle phys;
    CK(cuMemCreate(&phys, size, &ap, 0));
    CK(cuMulticastBindMem(mc, 0, phys, 0, size, 0));
    CUdeviceptr uc, mcp;
    CK(cuMemAddressReserve(&uc, size, grec, 0, 0));
    CK(cuMemMap(uc, size, 0, phys, 0));
    CUmemAccessDesc acc = {};
    acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc.location.id = 0;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    CK(cuMemSetAccess(uc, size, &acc, 1));
    CK(cuMemAddressReserve(&mcp, size, grec, 0, 0));
    CK(cuMemMap(mcp, size, 0, mc, 0));
    CK(cuMemSetAccess(mcp, size, &acc, 1));
    void* src;
    cudaMalloc(&src, size);
    std::vector<uint32_t> h(size / 4);
    for (size_t i = 0; i < h.size(); ++i) h[i] = (uint32_t)(i * 2654435761u) ^ 0x7FC01234u;  // includes NaN-like patterns
    cudaMemcpy(src, h.data(), size, cudaMemcpyHostToDevice);
    cudaMemset((void*)uc, 0, size);
    for (int kind = 0; kind < 2; ++kind) {
      cudaMemset((void*)uc, 0, size);
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      if (kind == 0) mc_store<<<148 * 8, 256>>>((uint4*)mcp, (const uint4*)src, size / 16);
      else mc_store_bf16<<<148 * 8, 256>>>((uint4*)mcp, (const uint4*)src, size / 16);
      cudaEventRecord(a);
      for (int it = 0; it < 10; ++it) {
        if (kind == 0) mc_store<<<148 * 8, 256>>>((uint4*)mcp, (const uint4*)src, size / 16);
        else mc_store_bf16<<<148 * 8, 256>>>((uint4*)mcp, (const uint4*)src, size / 16);
      }
      cudaEventRecord(b);
      cudaError_t e = cudaDeviceSynchronize();
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      std::vector<uint32_t> back(size / 4);
      cudaMemcpy(back.data(), (void*)uc, size, cudaMemcpyDeviceToHost);
      size_t bad = 0;
      for (size_t i = 0; i < h.size(); ++i) bad += back[i] != h[i];
      printf("  kind=%s err=%s mismatches=%zu  %.1f GB/s (read+mc write)\n", kind == 0 ? "v4.f32" : "v4.bf16x2",
             cudaGetErrorString(e), bad, 2.0 * size * 10 / (ms * 1e-3) / 1e9);
    }
    return 0;
  }
  return 0;
}
