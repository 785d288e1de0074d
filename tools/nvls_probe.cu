// NVLS (multicast object) capability probe for one box.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tools/nvls_probe.bin tools/nvls_probe.cu -lcuda
// Prints the multicast attributes of every visible device, then builds a
// multicast object over all of them (one device on a gpurun lease), binds a
// VMM allocation per device, and runs multimem.st / multimem.ld_reduce through
// the multicast address.  Exit code 0 = NVLS usable.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

#define CK(x) do { CUresult r_ = (x); if (r_ != CUDA_SUCCESS) { const char* s = nullptr; cuGetErrorString(r_, &s); \
  printf("FAIL %s -> %d (%s)\n", #x, (int)r_, s ? s : "?"); return 1; } } while (0)

__global__ void mc_store(float* mc, int n, float v) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) asm volatile("multimem.st.global.f32 [%0], %1;" :: "l"(mc + i), "f"(v + i) : "memory");
}
__global__ void mc_reduce(const float* mc, float* out, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    float r;
    asm volatile("multimem.ld_reduce.global.add.f32 %0, [%1];" : "=f"(r) : "l"(mc + i) : "memory");
    out[i] = r;
  }
}
__global__ void mc_reduce_bf16x2(const uint32_t* mc, uint32_t* out, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    uint32_t r;
    asm volatile("multimem.ld_reduce.global.add.acc::f32.bf16x2 %0, [%1];" : "=r"(r) : "l"(mc + i) : "memory");
    out[i] = r;
  }
}

int main() {
  CK(cuInit(0));
  int ndev = 0;
  CK(cuDeviceGetCount(&ndev));
  printf("devices %d\n", ndev);
  for (int d = 0; d < ndev; ++d) {
    CUdevice dev; CK(cuDeviceGet(&dev, d));
    int mc = 0, fab = 0, fd = 0, vmm = 0;
    cuDeviceGetAttribute(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev);
    cuDeviceGetAttribute(&fab, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED, dev);
    cuDeviceGetAttribute(&fd, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED, dev);
    cuDeviceGetAttribute(&vmm, CU_DEVICE_ATTRIBUTE_VIRTUAL_MEMORY_MANAGEMENT_SUPPORTED, dev);
    printf("dev %d multicast=%d fabric_handle=%d posix_fd=%d vmm=%d\n", d, mc, fab, fd, vmm);
  }
  CUdevice dev0; CK(cuDeviceGet(&dev0, 0));
  CUcontext ctx; CK(cuDevicePrimaryCtxRetain(&ctx, dev0)); CK(cuCtxSetCurrent(ctx));
  int mcs = 0; cuDeviceGetAttribute(&mcs, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev0);
  if (!mcs) { printf("NVLS unavailable: CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED=0\n"); return 2; }

  const int n = 1 << 20;
  size_t bytes = n * sizeof(float);
  CUmulticastObjectProp mp = {};
  mp.numDevices = 1;
  mp.size = bytes;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t gran = 0, rgran = 0;
  CK(cuMulticastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_MINIMUM));
  CK(cuMulticastGetGranularity(&rgran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  printf("mc granularity min %zu recommended %zu\n", gran, rgran);
  bytes = (bytes + rgran - 1) / rgran * rgran;
  mp.size = bytes;
  CUmemGenericAllocationHandle mch;
  {
    // try the handle types / sizes the driver may insist on
    const CUmemAllocationHandleType hts[] = {CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, CU_MEM_HANDLE_TYPE_NONE,
                                             CU_MEM_HANDLE_TYPE_FABRIC};
    const size_t sizes[] = {bytes, gran, 2 * gran, 32 * gran};
    int ok = 0;
    for (auto ht : hts) for (size_t sz : sizes) for (int nd = 1; nd <= 2 && !ok; ++nd) {
      CUmulticastObjectProp q = mp; q.handleTypes = ht; q.size = sz; q.numDevices = nd;
      CUresult r = cuMulticastCreate(&mch, &q);
      const char* es = nullptr; cuGetErrorString(r, &es);
      printf("cuMulticastCreate(ht=%d size=%zu ndev=%d) -> %d %s\n", (int)ht, sz, nd, (int)r, es ? es : "");
      if (r == CUDA_SUCCESS) {
        if (nd == 1) { ok = 1; mp = q; bytes = sz; } else cuMemRelease(mch);
      }
    }
    if (!ok) { printf("NVLS unavailable: no multicast object could be created\n"); return 3; }
  }
  CK(cuMulticastAddDevice(mch, dev0));

  CUmemAllocationProp ap = {};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = 0;
  ap.requestedHandleTypes = (CUmemAllocationHandleType)mp.handleTypes;
  size_t ag = 0; CK(cuMemGetAllocationGranularity(&ag, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
  printf("alloc granularity %zu\n", ag);
  CUmemGenericAllocationHandle uch;
  CK(cuMemCreate(&uch, bytes, &ap, 0));
  CK(cuMulticastBindMem(mch, 0, uch, 0, bytes, 0));

  CUdeviceptr uva, mva;
  CK(cuMemAddressReserve(&uva, bytes, rgran, 0, 0));
  CK(cuMemMap(uva, bytes, 0, uch, 0));
  CK(cuMemAddressReserve(&mva, bytes, rgran, 0, 0));
  CK(cuMemMap(mva, bytes, 0, mch, 0));
  CUmemAccessDesc acc = {};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE; acc.location.id = 0;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CK(cuMemSetAccess(uva, bytes, &acc, 1));
  CK(cuMemSetAccess(mva, bytes, &acc, 1));

  float* out; cudaMalloc(&out, n * sizeof(float));
  mc_store<<<n / 256, 256>>>((float*)mva, n, 1.5f);
  mc_reduce<<<n / 256, 256>>>((const float*)mva, out, n);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("FAIL kernel: %s\n", cudaGetErrorString(e)); return 1; }
  std::vector<float> h(n), u(n);
  cudaMemcpy(h.data(), out, n * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(u.data(), (void*)uva, n * 4, cudaMemcpyDeviceToHost);
  long bad = 0;
  for (int i = 0; i < n; ++i) if (h[i] != 1.5f + i || u[i] != 1.5f + i) ++bad;
  printf("multimem.st + ld_reduce.f32 over 1 device: %ld mismatches\n", bad);
  mc_reduce_bf16x2<<<n / 256, 256>>>((const uint32_t*)mva, (uint32_t*)out, n);
  e = cudaDeviceSynchronize();
  printf("ld_reduce.bf16x2: %s\n", e == cudaSuccess ? "ok" : cudaGetErrorString(e));
  // bandwidth of the multicast path on one device
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int it = 0; it < 20; ++it) mc_reduce<<<n / 256, 256>>>((const float*)mva, out, n);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms = 0; cudaEventElapsedTime(&ms, a, b);
  printf("ld_reduce f32 4 MiB x20: %.3f ms (%.1f GB/s read+write)\n", ms, 20.0 * 2 * n * 4 / (ms * 1e6));
  printf(bad == 0 ? "NVLS OK\n" : "NVLS MISMATCH\n");
  return bad == 0 ? 0 : 1;
}
