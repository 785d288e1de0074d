// NVLS (NVLink SHARP) multicast region of a team: the B200 form of the
// reference's node-team collectives multimem_ld_reduce / multimem_st
// (ovs/shmem.py:335-385; the paper's multimem_ld_reduce_v4 / multimem_st_v4,
// PAPER.md:1884-1942).
//
// One multicast object spans every PE's physical allocation of `nvls_bytes`
// (cuMulticastCreate / cuMulticastAddDevice / cuMemCreate / cuMulticastBindMem).
// Each PE keeps a unicast mapping of its own copy (kernels write partials there)
// and the process maps the multicast handle once: a multimem.ld_reduce through
// the multicast VA returns the element-wise sum of every PE's copy, reduced in
// the NVSwitch; a multimem.st writes all copies with one NVLink transfer.
//
// Local teams (all PEs in this process) build everything in tf_team_nvls_create.
// IPC teams (one PE per process): rank 0 creates the object and exports a POSIX
// file descriptor (passed to the peers over a Unix socket by the Python side,
// shmem.Team.enable_nvls), the others import it; every rank then adds its
// device, and after a barrier binds and maps its memory.
//
// Opt-in behind CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED and successful object
// creation; without it the P2P paths (tf_team_reduce / tf_team_broadcast, the
// two-shot allreduce) stay in use.  The summation order inside the switch is
// not the reference's ascending rank order: bf16 / f32 sums agree to rounding,
// integer sums exactly.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include "tf_internal.h"
#include "tf_ptx.cuh"
#include "tf_team.h"

namespace tf {
namespace {

struct DriverApi {
  decltype(&cuDeviceGet) DeviceGet = nullptr;
  decltype(&cuDeviceGetAttribute) DeviceGetAttribute = nullptr;
  decltype(&cuMulticastCreate) MulticastCreate = nullptr;
  decltype(&cuMulticastAddDevice) MulticastAddDevice = nullptr;
  decltype(&cuMulticastBindMem) MulticastBindMem = nullptr;
  decltype(&cuMulticastUnbind) MulticastUnbind = nullptr;
  decltype(&cuMulticastGetGranularity) MulticastGetGranularity = nullptr;
  decltype(&cuMemCreate) MemCreate = nullptr;
  decltype(&cuMemRelease) MemRelease = nullptr;
  decltype(&cuMemAddressReserve) MemAddressReserve = nullptr;
  decltype(&cuMemAddressFree) MemAddressFree = nullptr;
  decltype(&cuMemMap) MemMap = nullptr;
  decltype(&cuMemUnmap) MemUnmap = nullptr;
  decltype(&cuMemSetAccess) MemSetAccess = nullptr;
  decltype(&cuMemExportToShareableHandle) MemExportToShareableHandle = nullptr;
  decltype(&cuMemImportFromShareableHandle) MemImportFromShareableHandle = nullptr;
  decltype(&cuGetErrorString) GetErrorString = nullptr;
  bool ok = false;
};

const DriverApi& drv() {
  static DriverApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    bool ok = true;
    auto load = [&](const char* name, auto& fn) {
      void* p = nullptr;
      cudaDriverEntryPointQueryResult q;
      if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess ||
          q != cudaDriverEntryPointSuccess || !p) {
        ok = false;
        return;
      }
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(p);
    };
    load("cuDeviceGet", api.DeviceGet);
    load("cuDeviceGetAttribute", api.DeviceGetAttribute);
    load("cuMulticastCreate", api.MulticastCreate);
    load("cuMulticastAddDevice", api.MulticastAddDevice);
    load("cuMulticastBindMem", api.MulticastBindMem);
    load("cuMulticastUnbind", api.MulticastUnbind);
    load("cuMulticastGetGranularity", api.MulticastGetGranularity);
    load("cuMemCreate", api.MemCreate);
    load("cuMemRelease", api.MemRelease);
    load("cuMemAddressReserve", api.MemAddressReserve);
    load("cuMemAddressFree", api.MemAddressFree);
    load("cuMemMap", api.MemMap);
    load("cuMemUnmap", api.MemUnmap);
    load("cuMemSetAccess", api.MemSetAccess);
    load("cuMemExportToShareableHandle", api.MemExportToShareableHandle);
    load("cuMemImportFromShareableHandle", api.MemImportFromShareableHandle);
    load("cuGetErrorString", api.GetErrorString);
    api.ok = ok;
  });
  return api;
}

int cu_fail(const char* what, CUresult r) {
  const char* s = nullptr;
  if (drv().GetErrorString) drv().GetErrorString(r, &s);
  return fail(r == CUDA_ERROR_NOT_SUPPORTED || r == CUDA_ERROR_INVALID_VALUE ? TF_ERR_CONFIG : TF_ERR_CUDA,
              std::string(what) + " failed (" + std::to_string(static_cast<int>(r)) + " " + (s ? s : "?") + ")");
}
#define TF_CU_TRY(call, what)                  \
  do {                                         \
    CUresult r_ = (call);                      \
    if (r_ != CUDA_SUCCESS) return ::tf::cu_fail(what, r_); \
  } while (0)

size_t round_up(size_t x, size_t g) { return (x + g - 1) / g * g; }

int device_multicast_ok(int device) {
  const DriverApi& d = drv();
  if (!d.ok) return fail(TF_ERR_CONFIG, "driver lacks the multicast / VMM entry points");
  CUdevice dev;
  TF_CU_TRY(d.DeviceGet(&dev, device), "cuDeviceGet");
  int mc = 0;
  TF_CU_TRY(d.DeviceGetAttribute(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev), "cuDeviceGetAttribute");
  if (!mc) return fail(TF_ERR_CONFIG, "device " + std::to_string(device) + " does not support multicast (NVLS)");
  return TF_OK;
}

int create_object(tf_team* t, size_t bytes, bool exportable) {
  const DriverApi& d = drv();
  CUmulticastObjectProp prop;
  std::memset(&prop, 0, sizeof(prop));
  prop.numDevices = static_cast<unsigned int>(t->world);
  prop.handleTypes = exportable ? CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR : CU_MEM_HANDLE_TYPE_NONE;
  prop.size = bytes;
  size_t gran = 0;
  TF_CU_TRY(d.MulticastGetGranularity(&gran, &prop, CU_MULTICAST_GRANULARITY_RECOMMENDED),
            "cuMulticastGetGranularity");
  if (gran == 0) gran = 2u << 20;
  prop.size = round_up(bytes, gran);
  CUmemGenericAllocationHandle h;
  TF_CU_TRY(d.MulticastCreate(&h, &prop), "cuMulticastCreate");
  t->nvls_mc_handle = h;
  t->nvls_bytes = prop.size;
  t->nvls_gran = gran;
  t->nvls_state = 1;
  t->nvls_phys.assign(t->world, 0);
  t->nvls_uc.assign(t->world, nullptr);
  return TF_OK;
}

int add_device(tf_team* t, int device) {
  CUdevice dev;
  TF_CU_TRY(drv().DeviceGet(&dev, device), "cuDeviceGet");
  TF_CU_TRY(drv().MulticastAddDevice(t->nvls_mc_handle, dev), "cuMulticastAddDevice");
  return TF_OK;
}

// physical memory of PE pe on its device, bound into the object, mapped unicast
int bind_pe(tf_team* t, int pe, const int* access_devs, int n_access) {
  const DriverApi& d = drv();
  const int device = t->pes[pe].device;
  DeviceGuard g(device);
  CUmemAllocationProp ap;
  std::memset(&ap, 0, sizeof(ap));
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = device;
  ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  CUmemGenericAllocationHandle ph;
  TF_CU_TRY(d.MemCreate(&ph, t->nvls_bytes, &ap, 0), "cuMemCreate");
  t->nvls_phys[pe] = ph;
  TF_CU_TRY(d.MulticastBindMem(t->nvls_mc_handle, 0, ph, 0, t->nvls_bytes, 0), "cuMulticastBindMem");
  CUdeviceptr va;
  TF_CU_TRY(d.MemAddressReserve(&va, t->nvls_bytes, t->nvls_gran, 0, 0), "cuMemAddressReserve");
  TF_CU_TRY(d.MemMap(va, t->nvls_bytes, 0, ph, 0), "cuMemMap(unicast)");
  for (int i = 0; i < n_access; ++i) {
    CUmemAccessDesc acc;
    std::memset(&acc, 0, sizeof(acc));
    acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc.location.id = access_devs[i];
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    TF_CU_TRY(d.MemSetAccess(va, t->nvls_bytes, &acc, 1), "cuMemSetAccess(unicast)");
  }
  t->nvls_uc[pe] = reinterpret_cast<uint8_t*>(va);
  TF_CUDA_TRY(cudaMemset(t->nvls_uc[pe], 0, t->nvls_bytes));
  return TF_OK;
}

int map_multicast(tf_team* t, const int* devs, int n) {
  const DriverApi& d = drv();
  CUdeviceptr va;
  TF_CU_TRY(d.MemAddressReserve(&va, t->nvls_bytes, t->nvls_gran, 0, 0), "cuMemAddressReserve");
  TF_CU_TRY(d.MemMap(va, t->nvls_bytes, 0, t->nvls_mc_handle, 0), "cuMemMap(multicast)");
  for (int i = 0; i < n; ++i) {
    CUmemAccessDesc acc;
    std::memset(&acc, 0, sizeof(acc));
    acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc.location.id = devs[i];
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    TF_CU_TRY(d.MemSetAccess(va, t->nvls_bytes, &acc, 1), "cuMemSetAccess(multicast)");
  }
  t->nvls_mc = reinterpret_cast<uint8_t*>(va);
  return TF_OK;
}

// ------------------------------------------------------------------ kernels
// out[i] = sum over every PE of copy[i], reduced in the switch (16-byte vectors)
template <int DT>
__global__ void __launch_bounds__(256) nvls_reduce_kernel(const uint8_t* mc, void* out, long long count) {
  const long long tid = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  asm volatile("fence.proxy.alias;" ::: "memory");  // copies were written through unicast aliases
  if constexpr (DT == 0) {  // bf16, fp32 accumulation in the switch
    const long long nv = count / 8;
    for (long long v = tid; v < nv; v += stride) {
      uint32_t a, b, c, d;
      asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.bf16x2 {%0, %1, %2, %3}, [%4];"
                   : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "l"(mc + v * 16) : "memory");
      reinterpret_cast<uint4*>(out)[v] = make_uint4(a, b, c, d);
    }
    for (long long i = nv * 8 + tid; i < count; i += stride) {  // tail: bf16 pairs
      const long long pair = i & ~1ll;
      uint32_t r;
      asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.bf16x2 %0, [%1];"
                   : "=r"(r) : "l"(mc + pair * 2) : "memory");
      static_cast<uint16_t*>(out)[i] = static_cast<uint16_t>((i & 1) ? (r >> 16) : (r & 0xFFFF));
    }
  } else if constexpr (DT == 1) {  // fp32
    const long long nv = count / 4;
    for (long long v = tid; v < nv; v += stride) {
      float a, b, c, d;
      asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0, %1, %2, %3}, [%4];"
                   : "=f"(a), "=f"(b), "=f"(c), "=f"(d) : "l"(mc + v * 16) : "memory");
      reinterpret_cast<float4*>(out)[v] = make_float4(a, b, c, d);
    }
    for (long long i = nv * 4 + tid; i < count; i += stride) {
      float r;
      asm volatile("multimem.ld_reduce.relaxed.sys.global.add.f32 %0, [%1];" : "=f"(r) : "l"(mc + i * 4) : "memory");
      static_cast<float*>(out)[i] = r;
    }
  } else {  // int64 (two's complement add == u64 add)
    for (long long i = tid; i < count; i += stride) {
      unsigned long long r;
      asm volatile("multimem.ld_reduce.relaxed.sys.global.add.u64 %0, [%1];" : "=l"(r) : "l"(mc + i * 8) : "memory");
      static_cast<unsigned long long*>(out)[i] = r;
    }
  }
}

// every PE's copy[0:bytes) := src (one NVLink transfer per 16 bytes, replicated by the switch)
__global__ void __launch_bounds__(256) nvls_store_kernel(uint8_t* mc, const uint8_t* src, long long bytes) {
  const long long tid = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  const long long nv = bytes / 16;
  for (long long v = tid; v < nv; v += stride) {
    const uint4 q = reinterpret_cast<const uint4*>(src)[v];
    asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(mc + v * 16),
                 "f"(__uint_as_float(q.x)), "f"(__uint_as_float(q.y)), "f"(__uint_as_float(q.z)),
                 "f"(__uint_as_float(q.w))
                 : "memory");
  }
  for (long long i = nv * 16 / 4 + tid; i < bytes / 4; i += stride) {
    const uint32_t w = reinterpret_cast<const uint32_t*>(src)[i];
    asm volatile("multimem.st.relaxed.sys.global.b32 [%0], %1;" ::"l"(mc + i * 4), "r"(w) : "memory");
  }
}

int grid_for(long long work) {
  const int sms = num_sms_of_current_device();
  long long g = (work + 255) / 256;
  if (g > 4LL * sms) g = 4LL * sms;
  return static_cast<int>(g < 1 ? 1 : g);
}

}  // namespace

void nvls_release(tf_team* t) {
  if (!t || !t->nvls_state) return;
  const DriverApi& d = drv();
  if (!d.ok) return;
  if (t->nvls_mc) {
    d.MemUnmap(reinterpret_cast<CUdeviceptr>(t->nvls_mc), t->nvls_bytes);
    d.MemAddressFree(reinterpret_cast<CUdeviceptr>(t->nvls_mc), t->nvls_bytes);
  }
  for (int pe = 0; pe < static_cast<int>(t->nvls_uc.size()); ++pe) {
    if (t->nvls_uc[pe]) {
      DeviceGuard g(t->pes[pe].device);
      cudaDeviceSynchronize();
      d.MemUnmap(reinterpret_cast<CUdeviceptr>(t->nvls_uc[pe]), t->nvls_bytes);
      d.MemAddressFree(reinterpret_cast<CUdeviceptr>(t->nvls_uc[pe]), t->nvls_bytes);
      CUdevice dev;
      if (d.DeviceGet(&dev, t->pes[pe].device) == CUDA_SUCCESS)
        d.MulticastUnbind(t->nvls_mc_handle, dev, 0, t->nvls_bytes);
    }
    if (t->nvls_phys[pe]) d.MemRelease(t->nvls_phys[pe]);
  }
  d.MemRelease(t->nvls_mc_handle);
  t->nvls_state = 0;
  t->nvls_mc = nullptr;
}

bool nvls_workspace(tf_team* t, const std::string& key, size_t bytes, size_t* off) {
  if (!t || t->nvls_state != 3 || getenv("TF_NO_NVLS")) return false;
  auto it = t->nvls_ws.find(key);
  if (it != t->nvls_ws.end()) {
    *off = it->second;
    return true;
  }
  const size_t o = (t->nvls_top + 1023) / 1024 * 1024;
  if (o + bytes > t->nvls_bytes) return false;
  t->nvls_top = o + bytes;
  t->nvls_ws[key] = o;
  *off = o;
  return true;
}

// device copy of a region of the team's NVLS multicast space
int nvls_check_range(const tf_team* t, uint64_t off, size_t bytes) {
  if (t->nvls_state != 3) return fail(TF_ERR_CONFIG, "NVLS is not enabled on this team");
  if (off + bytes > t->nvls_bytes) return fail(TF_ERR_INVALID, "range outside the NVLS region");
  if (off % 16) return fail(TF_ERR_INVALID, "NVLS offsets must be 16-byte aligned");
  return TF_OK;
}

}  // namespace tf

using tf::fail;

extern "C" {

int tf_nvls_supported(int device, int* supported) {
  if (!supported) return fail(TF_ERR_INVALID, "NULL argument");
  *supported = tf::device_multicast_ok(device) == TF_OK ? 1 : 0;
  return TF_OK;
}

int tf_team_nvls_create(tf_team* t, size_t bytes, int* fd_out) {
  if (!t || bytes == 0) return fail(TF_ERR_INVALID, "bad team or size");
  if (t->nvls_state) return fail(TF_ERR_PROTOCOL, "NVLS region already created");
  if (!t->ipc) {
    if (!t->distinct_devices) return fail(TF_ERR_CONFIG, "NVLS needs one GPU per PE");
    int devs[TF_MAX_WORLD];
    for (int p = 0; p < t->world; ++p) {
      devs[p] = t->pes[p].device;
      int rc = tf::device_multicast_ok(devs[p]);
      if (rc) return rc;
    }
    tf::DeviceGuard g(devs[0]);
    int rc = tf::create_object(t, bytes, false);
    if (rc) return rc;
    for (int p = 0; p < t->world; ++p) {
      rc = tf::add_device(t, devs[p]);
      if (rc) { tf::nvls_release(t); return rc; }
    }
    for (int p = 0; p < t->world; ++p) {
      rc = tf::bind_pe(t, p, devs, t->world);
      if (rc) { tf::nvls_release(t); return rc; }
    }
    rc = tf::map_multicast(t, devs, t->world);
    if (rc) { tf::nvls_release(t); return rc; }
    t->nvls_state = 3;
    if (fd_out) *fd_out = -1;
    return TF_OK;
  }
  // IPC: the creating rank exports a POSIX fd for its peers
  if (!fd_out) return fail(TF_ERR_INVALID, "fd_out is NULL");
  const int dev = t->pes[t->my_rank].device;
  int rc = tf::device_multicast_ok(dev);
  if (rc) return rc;
  tf::DeviceGuard g(dev);
  rc = tf::create_object(t, bytes, true);
  if (rc) return rc;
  int fd = -1;
  CUresult r = tf::drv().MemExportToShareableHandle(&fd, t->nvls_mc_handle,
                                                    CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0);
  if (r != CUDA_SUCCESS) { tf::nvls_release(t); return tf::cu_fail("cuMemExportToShareableHandle", r); }
  *fd_out = fd;
  return TF_OK;
}

int tf_team_nvls_import(tf_team* t, size_t bytes, int fd) {
  if (!t || !t->ipc) return fail(TF_ERR_INVALID, "nvls_import needs an IPC team");
  if (t->nvls_state) return fail(TF_ERR_PROTOCOL, "NVLS region already created");
  const int dev = t->pes[t->my_rank].device;
  int rc = tf::device_multicast_ok(dev);
  if (rc) return rc;
  tf::DeviceGuard g(dev);
  CUmemGenericAllocationHandle h;
  TF_CU_TRY(tf::drv().MemImportFromShareableHandle(&h, reinterpret_cast<void*>(static_cast<uintptr_t>(fd)),
                                                   CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR),
            "cuMemImportFromShareableHandle");
  CUmulticastObjectProp prop;
  std::memset(&prop, 0, sizeof(prop));
  prop.numDevices = static_cast<unsigned int>(t->world);
  prop.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  prop.size = bytes;
  size_t gran = 0;
  TF_CU_TRY(tf::drv().MulticastGetGranularity(&gran, &prop, CU_MULTICAST_GRANULARITY_RECOMMENDED),
            "cuMulticastGetGranularity");
  if (gran == 0) gran = 2u << 20;
  t->nvls_mc_handle = h;
  t->nvls_gran = gran;
  t->nvls_bytes = tf::round_up(bytes, gran);
  t->nvls_state = 1;
  t->nvls_phys.assign(t->world, 0);
  t->nvls_uc.assign(t->world, nullptr);
  return TF_OK;
}

int tf_team_nvls_add_device(tf_team* t) {
  if (!t || !t->ipc || t->nvls_state != 1) return fail(TF_ERR_PROTOCOL, "create or import the NVLS object first");
  const int rc = tf::add_device(t, t->pes[t->my_rank].device);
  if (rc) return rc;
  t->nvls_state = 2;
  return TF_OK;
}

int tf_team_nvls_bind(tf_team* t) {
  if (!t || !t->ipc || t->nvls_state != 2)
    return fail(TF_ERR_PROTOCOL, "every rank must add its device (and barrier) before binding");
  const int dev = t->pes[t->my_rank].device;
  int rc = tf::bind_pe(t, t->my_rank, &dev, 1);
  if (rc) return rc;
  rc = tf::map_multicast(t, &dev, 1);
  if (rc) return rc;
  t->nvls_state = 3;
  return TF_OK;
}

int tf_nvls_enabled(tf_team* t, int* enabled, size_t* bytes) {
  if (!t || !enabled) return fail(TF_ERR_INVALID, "NULL argument");
  *enabled = t->nvls_state == 3 ? 1 : 0;
  if (bytes) *bytes = t->nvls_bytes;
  return TF_OK;
}

int tf_nvls_alloc(tf_team* t, size_t nbytes, size_t align, uint64_t* offset) {
  if (!t || !offset) return fail(TF_ERR_INVALID, "NULL argument");
  if (t->nvls_state != 3) return fail(TF_ERR_CONFIG, "NVLS is not enabled on this team");
  if (align < 16) align = 16;
  if (align & (align - 1)) return fail(TF_ERR_INVALID, "align must be a power of two");
  const size_t off = (t->nvls_top + align - 1) / align * align;
  if (off + nbytes > t->nvls_bytes)
    return fail(TF_ERR_ALLOC, "NVLS region exhausted: need " + std::to_string(off + nbytes) + " bytes, capacity " +
                                  std::to_string(t->nvls_bytes));
  t->nvls_top = off + nbytes;
  *offset = off;
  return TF_OK;
}

int tf_nvls_ptr(tf_team* t, int pe, uint64_t offset, void** uc, void** mc) {
  if (!t || pe < 0 || pe >= t->world) return fail(TF_ERR_INVALID, "pe out of range");
  if (t->nvls_state != 3) return fail(TF_ERR_CONFIG, "NVLS is not enabled on this team");
  if (offset > t->nvls_bytes) return fail(TF_ERR_INVALID, "offset outside the NVLS region");
  if (uc) {
    if (!t->nvls_uc[pe]) return fail(TF_ERR_INVALID, "PE's unicast NVLS copy is not mapped in this process");
    *uc = t->nvls_uc[pe] + offset;
  }
  if (mc) *mc = t->nvls_mc + offset;
  return TF_OK;
}

int tf_nvls_reduce(tf_team* t, int pe, uint64_t offset, int dtype, int64_t count, void* out, void* stream) {
  if (!t || pe < 0 || pe >= t->world || !out) return fail(TF_ERR_INVALID, "bad arguments");
  if (!t->is_local(pe)) return fail(TF_ERR_INVALID, "pe is not owned by this process");
  if (dtype < 0 || dtype > 2) return fail(TF_ERR_INVALID, "dtype code must be 0 (bf16), 1 (f32) or 2 (int64)");
  const size_t esz = dtype == 0 ? 2 : dtype == 1 ? 4 : 8;
  int rc = tf::nvls_check_range(t, offset, static_cast<size_t>(count) * esz);
  if (rc) return rc;
  if (reinterpret_cast<uintptr_t>(out) % 16) return fail(TF_ERR_INVALID, "out must be 16-byte aligned");
  if (count <= 0) return TF_OK;
  tf::DeviceGuard g(t->pes[pe].device);
  auto s = static_cast<cudaStream_t>(stream);
  const uint8_t* mc = t->nvls_mc + offset;
  const int grid = tf::grid_for(count / (dtype == 0 ? 8 : dtype == 1 ? 4 : 1) + 1);
  if (dtype == 0) tf::nvls_reduce_kernel<0><<<grid, 256, 0, s>>>(mc, out, count);
  else if (dtype == 1) tf::nvls_reduce_kernel<1><<<grid, 256, 0, s>>>(mc, out, count);
  else tf::nvls_reduce_kernel<2><<<grid, 256, 0, s>>>(mc, out, count);
  TF_CUDA_TRY(cudaGetLastError());
  return TF_OK;
}

int tf_nvls_broadcast(tf_team* t, int pe, uint64_t offset, const void* src, size_t bytes, void* stream) {
  if (!t || pe < 0 || pe >= t->world || (!src && bytes)) return fail(TF_ERR_INVALID, "bad arguments");
  if (!t->is_local(pe)) return fail(TF_ERR_INVALID, "pe is not owned by this process");
  int rc = tf::nvls_check_range(t, offset, bytes);
  if (rc) return rc;
  if (bytes % 4 || reinterpret_cast<uintptr_t>(src) % 16)
    return fail(TF_ERR_INVALID, "broadcast needs a 16-byte aligned source and a multiple of 4 bytes");
  if (!bytes) return TF_OK;
  tf::DeviceGuard g(t->pes[pe].device);
  auto s = static_cast<cudaStream_t>(stream);
  tf::nvls_store_kernel<<<tf::grid_for(static_cast<long long>(bytes / 16) + 1), 256, 0, s>>>(
      t->nvls_mc + offset, static_cast<const uint8_t*>(src), static_cast<long long>(bytes));
  TF_CUDA_TRY(cudaGetLastError());
  return TF_OK;
}

}  // extern "C"
