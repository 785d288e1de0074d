// Symmetric-memory runtime: teams, heaps, signals, barriers, one-sided copies.
//
// Replaces the simulated SymmetricHeap (ovs/shmem.py:87-473).  A team is
// `world` PEs.  Each PE owns one device allocation:
//     [ data region: heap_bytes ][ signal region: signal_slots x uint64 ]
// and every PE's allocation is addressable from every other PE's device:
//   * local team  (one process): plain pointers + cudaDeviceEnablePeerAccess;
//     several PEs may share one device (single-GPU emulation of a TP group);
//   * IPC team    (one process per GPU, torchrun): cudaIpcGetMemHandle /
//     cudaIpcOpenMemHandle, blobs exchanged by the Python side.
// symm_at(offset, pe) is base[pe] + offset -- identical offsets on every PE by
// construction of the bump allocator (shmem.py:109-121).
//
// Signal slots [0, world) of every PE are reserved for barrier_all; slot
// `world` holds the PE's device error word (spin timeouts).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "tf_internal.h"
#include "tf_ptx.cuh"
#include "tf_team.h"

namespace tf {

namespace {
thread_local std::string g_last_error;
}

void set_error(const std::string& msg) { g_last_error = msg; }
const char* last_error_cstr() { return g_last_error.c_str(); }
int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

namespace {
// ---------------------------------------------------------------- device helpers
__global__ void signal_op_kernel(uint64_t* p, uint64_t v, int add) {
  if (add) red_add_release_sys(p, v);
  else st_release_sys(p, v);
}

__global__ void signal_wait_kernel(const uint64_t* p, int n, uint64_t v, int eq, uint64_t timeout_ns,
                                   unsigned long long* err) {
  const int i = threadIdx.x;
  if (i >= n) return;
  if (eq) wait_eq_sys(p + i, v, timeout_ns, err, 0x2000000ull | static_cast<unsigned>(i));
  else wait_geq_sys(p + i, v, timeout_ns, err, 0x2000000ull | static_cast<unsigned>(i));
}

__global__ void signal_fetch_add_kernel(uint64_t* p, uint64_t v, unsigned long long* old) {
  *old = atom_add_release_sys(p, v);
}

struct PeerSigs {
  uint64_t* sig[kMaxWorld];
};

__global__ void barrier_arrive_kernel(PeerSigs peers, int world, int rank, uint64_t epoch) {
  const int p = threadIdx.x;
  __threadfence_system();  // drain this stream's prior writes before announcing arrival
  if (p < world) st_release_sys(peers.sig[p] + rank, epoch);
}

__global__ void barrier_wait_kernel(const uint64_t* own_sig, int world, uint64_t epoch,
                                    uint64_t timeout_ns, unsigned long long* err) {
  const int p = threadIdx.x;
  if (p < world) wait_geq_sys(own_sig + p, epoch, timeout_ns, err, 0x3000000ull | p);
  __syncthreads();
}

using StreamWriteFn = CUresult (*)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);
StreamWriteFn get_stream_write_fn() {
  static StreamWriteFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue64", &ptr, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<StreamWriteFn>(ptr);
  });
  return fn;
}

}  // namespace

// stream-ordered signal store (copy-engine friendly: no kernel when the driver
// exposes stream memory operations; the default flags fence prior writes).
int stream_signal_set(tf_team* t, int pe, uint64_t slot, uint64_t value, cudaStream_t s) {
  uint64_t* ptr = t->pes[pe].sig + slot;
  static int mode = -1;  // -1 unknown, 0 kernel, 1 stream write
  if (mode < 0) mode = get_stream_write_fn() ? 1 : 0;
  if (mode == 1) {
    CUresult r = get_stream_write_fn()(reinterpret_cast<CUstream>(s),
                                       reinterpret_cast<CUdeviceptr>(ptr), value, 0);
    if (r == CUDA_SUCCESS) return TF_OK;
    mode = 0;
  }
  signal_op_kernel<<<1, 1, 0, s>>>(ptr, value, 0);
  TF_CUDA_TRY(cudaGetLastError());
  return TF_OK;
}

int team_barrier_arrive(tf_team* t, int rank, cudaStream_t s) {
  const uint64_t e = ++t->bar_epoch[rank];
  PeerSigs ps{};
  for (int p = 0; p < t->world; ++p) ps.sig[p] = t->pes[p].sig;
  barrier_arrive_kernel<<<1, 32, 0, s>>>(ps, t->world, rank, e);
  TF_CUDA_TRY(cudaGetLastError());
  return TF_OK;
}

int team_barrier_wait(tf_team* t, int rank, cudaStream_t s) {
  const uint64_t e = t->bar_epoch[rank];
  barrier_wait_kernel<<<1, 32, 0, s>>>(t->pes[rank].sig, t->world, e, t->timeout_ns,
                                       t->err_word(rank));
  TF_CUDA_TRY(cudaGetLastError());
  return TF_OK;
}

}  // namespace tf

using tf::fail;

void* tf_team::scratch(int device, size_t bytes) {
  auto it = scratch_bufs.find(device);
  if (it != scratch_bufs.end() && it->second.second >= bytes) return it->second.first;
  tf::DeviceGuard g(device);
  if (it != scratch_bufs.end()) {
    cudaDeviceSynchronize();
    cudaFree(it->second.first);
  }
  void* p = nullptr;
  if (cudaMalloc(&p, bytes) != cudaSuccess) return nullptr;
  scratch_bufs[device] = {p, bytes};
  return p;
}

unsigned long long* tf_team::err_word(int pe) {
  return reinterpret_cast<unsigned long long*>(pes[pe].sig + world);
}

tf::Workspace* tf_team::workspace(const std::string& key, size_t data_bytes, size_t sig_slots,
                              int* rc) {
  auto it = workspaces.find(key);
  if (it != workspaces.end()) return &it->second;
  tf::Workspace w;
  const size_t align = 1024;
  size_t off = (data_top + align - 1) / align * align;
  if (off + data_bytes > heap_bytes) {
    *rc = tf::fail(TF_ERR_ALLOC, "heap exhausted creating workspace '" + key + "': need " +
                                 std::to_string(off + data_bytes) + " bytes, capacity " +
                                 std::to_string(heap_bytes));
    return nullptr;
  }
  if (sig_top + sig_slots > signal_slots) {
    *rc = tf::fail(TF_ERR_ALLOC, "signal space exhausted creating workspace '" + key + "'");
    return nullptr;
  }
  w.epoch.assign(world, 0);
  w.data_off = off;
  w.data_bytes = data_bytes;
  w.sig_base = sig_top;
  w.sig_slots = sig_slots;
  data_top = off + data_bytes;
  sig_top += sig_slots;
  *rc = TF_OK;
  return &(workspaces[key] = w);
}



namespace tf {
struct ReducePtrs {
  const uint8_t* p[kMaxWorld];
};
// out[i] = sum over PEs (ascending) of PE q's element i; bf16 accumulates in fp32
__global__ void signal_cas_kernel(uint64_t* slot, uint64_t cmp, uint64_t val, unsigned long long* old) {
  *old = atom_cas_sys(slot, cmp, val);
}
template <int DT>
__global__ void team_reduce_kernel(ReducePtrs src, int world, int64_t count, void* out) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (DT == 0) {
      float acc = 0.f;
      for (int q = 0; q < world; ++q)
        acc += __uint_as_float(static_cast<uint32_t>(reinterpret_cast<const uint16_t*>(src.p[q])[i]) << 16);
      // round to nearest even
      uint32_t b = __float_as_uint(acc);
      b += 0x7FFFu + ((b >> 16) & 1u);
      static_cast<uint16_t*>(out)[i] = static_cast<uint16_t>(b >> 16);
    } else if (DT == 1) {
      float acc = 0.f;
      for (int q = 0; q < world; ++q) acc += reinterpret_cast<const float*>(src.p[q])[i];
      static_cast<float*>(out)[i] = acc;
    } else {
      long long acc = 0;
      for (int q = 0; q < world; ++q) acc += reinterpret_cast<const long long*>(src.p[q])[i];
      static_cast<long long*>(out)[i] = acc;
    }
  }
}
}  // namespace tf

extern "C" {

const char* tf_last_error(void) { return tf::last_error_cstr(); }
const char* tf_version(void) { return "tilefuse 0.1 sm_100a"; }

int tf_team_create_local(int world, const int* devices, size_t heap_bytes, size_t signal_slots,
                         tf_team** out) {
  if (!out) return fail(TF_ERR_INVALID, "out is NULL");
  if (world < 1 || world > TF_MAX_WORLD)
    return fail(TF_ERR_CONFIG, "world must be in [1, " + std::to_string(TF_MAX_WORLD) + "]");
  int ndev = 0;
  TF_CUDA_TRY(cudaGetDeviceCount(&ndev));
  auto* t = new tf_team();
  t->world = world;
  t->my_rank = -1;
  t->ipc = false;
  t->heap_bytes = heap_bytes;
  t->signal_slots = signal_slots + world + 1;
  t->sig_top = world + 1;
  t->pes.resize(world);
  t->bar_epoch.assign(world, 0);
  t->op_epoch.assign(world, 0);
  t->distinct_devices = true;
  for (int p = 0; p < world; ++p) {
    const int d = devices ? devices[p] : 0;
    if (d < 0 || d >= ndev) {
      delete t;
      return fail(TF_ERR_CONFIG, "device " + std::to_string(d) + " out of range");
    }
    for (int q = 0; q < p; ++q)
      if (t->pes[q].device == d) t->distinct_devices = false;
    t->pes[p].device = d;
  }
  // peer access between distinct devices
  for (int p = 0; p < world; ++p)
    for (int q = 0; q < world; ++q) {
      const int a = t->pes[p].device, b = t->pes[q].device;
      if (a == b) continue;
      tf::DeviceGuard g(a);
      int can = 0;
      cudaDeviceCanAccessPeer(&can, a, b);
      if (!can) {
        delete t;
        return fail(TF_ERR_CONFIG, "no peer access between devices " + std::to_string(a) +
                                       " and " + std::to_string(b));
      }
      cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) {
        delete t;
        return fail(TF_ERR_CUDA, std::string("cudaDeviceEnablePeerAccess: ") + cudaGetErrorString(e));
      }
      cudaGetLastError();
    }
  for (int p = 0; p < world; ++p) {
    tf::DeviceGuard g(t->pes[p].device);
    const size_t sig_off = (heap_bytes + 255) / 256 * 256;
    const size_t total = sig_off + t->signal_slots * sizeof(uint64_t);
    void* base = nullptr;
    cudaError_t e = cudaMalloc(&base, total);
    if (e != cudaSuccess) {
      tf_team_destroy(t);
      return fail(TF_ERR_ALLOC, std::string("cudaMalloc of symmetric heap failed: ") +
                                    cudaGetErrorString(e));
    }
    cudaMemset(base, 0, total);
    t->pes[p].base = static_cast<uint8_t*>(base);
    t->pes[p].sig = reinterpret_cast<uint64_t*>(t->pes[p].base + sig_off);
    t->pes[p].owned = true;
  }
  for (int p = 0; p < world; ++p) {
    tf::DeviceGuard g(t->pes[p].device);
    cudaDeviceSynchronize();
  }
  *out = t;
  return TF_OK;
}

int tf_team_create_ipc(int world, int rank, int device, size_t heap_bytes, size_t signal_slots,
                       tf_team** out) {
  if (!out) return fail(TF_ERR_INVALID, "out is NULL");
  if (world < 1 || world > TF_MAX_WORLD)
    return fail(TF_ERR_CONFIG, "world must be in [1, " + std::to_string(TF_MAX_WORLD) + "]");
  if (rank < 0 || rank >= world) return fail(TF_ERR_INVALID, "rank out of range");
  auto* t = new tf_team();
  t->world = world;
  t->my_rank = rank;
  t->ipc = true;
  t->heap_bytes = heap_bytes;
  t->signal_slots = signal_slots + world + 1;
  t->sig_top = world + 1;
  t->pes.resize(world);
  t->bar_epoch.assign(world, 0);
  t->op_epoch.assign(world, 0);
  t->distinct_devices = true;
  for (int p = 0; p < world; ++p) t->pes[p].device = device;  // peers: remote devices (opaque)
  tf::DeviceGuard g(device);
  const size_t sig_off = (heap_bytes + 255) / 256 * 256;
  const size_t total = sig_off + t->signal_slots * sizeof(uint64_t);
  void* base = nullptr;
  cudaError_t e = cudaMalloc(&base, total);
  if (e != cudaSuccess) {
    delete t;
    return fail(TF_ERR_ALLOC, std::string("cudaMalloc of symmetric heap failed: ") +
                                  cudaGetErrorString(e));
  }
  cudaMemset(base, 0, total);
  cudaDeviceSynchronize();
  t->pes[rank].base = static_cast<uint8_t*>(base);
  t->pes[rank].sig = reinterpret_cast<uint64_t*>(t->pes[rank].base + sig_off);
  t->pes[rank].owned = true;
  t->sig_off = sig_off;
  *out = t;
  return TF_OK;
}

int tf_team_export_handle(tf_team* t, void* blob, size_t blob_len) {
  if (!t || !t->ipc) return fail(TF_ERR_INVALID, "export_handle needs an IPC team");
  if (blob_len < sizeof(cudaIpcMemHandle_t)) return fail(TF_ERR_INVALID, "blob too small");
  tf::DeviceGuard g(t->pes[t->my_rank].device);
  cudaIpcMemHandle_t h;
  TF_CUDA_TRY(cudaIpcGetMemHandle(&h, t->pes[t->my_rank].base));
  std::memset(blob, 0, blob_len);
  std::memcpy(blob, &h, sizeof(h));
  return TF_OK;
}

int tf_team_open_peers(tf_team* t, const void* blobs, size_t blob_len) {
  if (!t || !t->ipc) return fail(TF_ERR_INVALID, "open_peers needs an IPC team");
  if (blob_len < sizeof(cudaIpcMemHandle_t)) return fail(TF_ERR_INVALID, "blob too small");
  tf::DeviceGuard g(t->pes[t->my_rank].device);
  for (int p = 0; p < t->world; ++p) {
    if (p == t->my_rank) continue;
    cudaIpcMemHandle_t h;
    std::memcpy(&h, static_cast<const uint8_t*>(blobs) + p * blob_len, sizeof(h));
    void* ptr = nullptr;
    TF_CUDA_TRY(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
    t->pes[p].base = static_cast<uint8_t*>(ptr);
    t->pes[p].sig = reinterpret_cast<uint64_t*>(t->pes[p].base + t->sig_off);
    t->pes[p].owned = false;
  }
  return TF_OK;
}

int tf_team_destroy(tf_team* t) {
  if (!t) return TF_OK;
  tf::layer_release_team(t);
  tf::nvls_release(t);
  for (int p = 0; p < t->world; ++p) {
    if (!t->pes[p].base) continue;
    tf::DeviceGuard g(t->pes[p].device);
    if (t->pes[p].owned) cudaFree(t->pes[p].base);
    else cudaIpcCloseMemHandle(t->pes[p].base);
  }
  for (auto& kv : t->dev_tables) {
    tf::DeviceGuard g(kv.first);
    cudaFree(kv.second);
  }
  for (auto& kv : t->scratch_bufs) {
    tf::DeviceGuard g(kv.first);
    cudaFree(kv.second.first);
  }
  delete t;
  return TF_OK;
}

int tf_team_world(tf_team* t, int* world) {
  if (!t || !world) return fail(TF_ERR_INVALID, "NULL argument");
  *world = t->world;
  return TF_OK;
}

int tf_team_device(tf_team* t, int pe, int* device) {
  if (!t || !device || pe < 0 || pe >= t->world) return fail(TF_ERR_INVALID, "bad pe");
  *device = t->pes[pe].device;
  return TF_OK;
}

int tf_team_check(tf_team* t) {
  if (!t) return fail(TF_ERR_INVALID, "NULL team");
  // read and clear every owned PE's error word, then report the first one set
  int first = -1;
  unsigned long long first_w = 0;
  for (int p = 0; p < t->world; ++p) {
    if (t->ipc && p != t->my_rank) continue;
    tf::DeviceGuard g(t->pes[p].device);
    unsigned long long w = 0;
    TF_CUDA_TRY(cudaMemcpy(&w, t->err_word(p), sizeof(w), cudaMemcpyDeviceToHost));
    if (w) {
      unsigned long long z = 0;
      cudaMemcpy(t->err_word(p), &z, sizeof(z), cudaMemcpyHostToDevice);
      if (first < 0) { first = p; first_w = w; }
    }
  }
  if (first >= 0) {
    const int p = first;
    const unsigned long long w = first_w;
    {
      const unsigned kind = static_cast<unsigned>(w >> 24);
      if (kind == 9)
        return fail(TF_ERR_PROTOCOL, "double release of scoreboard slot " + std::to_string(w & 0xFFFFFF) +
                                         " on PE " + std::to_string(p));
      if (kind == 8)
        return fail(TF_ERR_TIMEOUT, "device spin timed out on PE " + std::to_string(p) +
                                        ": scoreboard task slot " + std::to_string(w & 0xFFFFFF) +
                                        " (task = slot / max_tiles_per_op)");
      if (kind == 5 && (w & 0xFFFFFF) == 0xFFFFFF)
        return fail(TF_ERR_INVALID, "MoE receive buffer overflow on PE " + std::to_string(p) +
                                        ": a destination row >= max_recv (raise max_recv / capacity_factor); "
                                        "rows past it were not delivered");
      if (kind == 5 && ((w >> 20) & 0xF) == 3)
        return fail(TF_ERR_INVALID, "MoE routing index out of range on PE " + std::to_string(p) +
                                        " at (token, slot) entry " + std::to_string(w & 0xFFFFF) +
                                        " of a CTA's slice (expert ids must be in [-1, n_experts))");
      const char* what = kind == 1 ? "AllGather chunk flag" : kind == 2 ? "signal wait"
                       : kind == 3 ? "barrier_all" : kind == 4 ? "reduce-scatter tile counter"
                       : kind == 5 ? "moe dispatch flag" : "device wait";
      return fail(TF_ERR_TIMEOUT, std::string("device spin timed out on PE ") + std::to_string(p) +
                                      ": " + what + " slot " + std::to_string(w & 0xFFFFFF));
    }
  }
  return TF_OK;
}

int tf_heap_alloc(tf_team* t, size_t nbytes, size_t align, uint64_t* offset) {
  if (!t || !offset) return fail(TF_ERR_INVALID, "NULL argument");
  if (align == 0 || (align & (align - 1))) return fail(TF_ERR_INVALID, "align must be a power of two");
  const size_t off = (t->data_top + align - 1) / align * align;
  if (off + nbytes > t->heap_bytes)
    return fail(TF_ERR_ALLOC, "heap exhausted: need " + std::to_string(off + nbytes) +
                                  " bytes, capacity " + std::to_string(t->heap_bytes));
  t->data_top = off + nbytes;
  *offset = off;
  return TF_OK;
}

int tf_signal_alloc(tf_team* t, size_t nslots, uint64_t* base) {
  if (!t || !base) return fail(TF_ERR_INVALID, "NULL argument");
  if (t->sig_top + nslots > t->signal_slots)
    return fail(TF_ERR_ALLOC, "signal space exhausted: need " + std::to_string(t->sig_top + nslots) +
                                  " slots");
  *base = t->sig_top;
  t->sig_top += nslots;
  return TF_OK;
}

int tf_heap_ptr(tf_team* t, int pe, uint64_t offset, void** ptr) {
  if (!t || !ptr || pe < 0 || pe >= t->world) return fail(TF_ERR_INVALID, "pe out of range");
  if (!t->pes[pe].base) return fail(TF_ERR_PROTOCOL, "peer region not opened");
  if (offset > t->heap_bytes) return fail(TF_ERR_INVALID, "offset outside the heap");
  *ptr = t->pes[pe].base + offset;
  return TF_OK;
}

int tf_signal_ptr(tf_team* t, int pe, uint64_t slot, uint64_t** ptr) {
  if (!t || !ptr || pe < 0 || pe >= t->world) return fail(TF_ERR_INVALID, "pe out of range");
  if (!t->pes[pe].sig) return fail(TF_ERR_PROTOCOL, "peer region not opened");
  if (slot >= t->signal_slots) return fail(TF_ERR_INVALID, "slot out of range");
  *ptr = t->pes[pe].sig + slot;
  return TF_OK;
}

int tf_signal_read(tf_team* t, int pe, uint64_t base, size_t n, uint64_t* host_out) {
  if (!t || pe < 0 || pe >= t->world) return fail(TF_ERR_INVALID, "pe out of range");
  if (base + n > t->signal_slots) return fail(TF_ERR_INVALID, "slots out of range");
  if (n == 0) return TF_OK;
  tf::DeviceGuard g(t->ipc ? t->pes[t->my_rank].device : t->pes[pe].device);
  TF_CUDA_TRY(cudaMemcpy(host_out, t->pes[pe].sig + base, n * sizeof(uint64_t), cudaMemcpyDefault));
  return TF_OK;
}

int tf_signal_reset(tf_team* t, int pe, uint64_t base, size_t n, void* stream) {
  if (!t || pe < 0 || pe >= t->world) return fail(TF_ERR_INVALID, "pe out of range");
  if (base + n > t->signal_slots) return fail(TF_ERR_INVALID, "slots out of range");
  if (n == 0) return TF_OK;
  TF_CUDA_TRY(cudaMemsetAsync(t->pes[pe].sig + base, 0, n * sizeof(uint64_t),
                              static_cast<cudaStream_t>(stream)));
  return TF_OK;
}

int tf_putmem(tf_team* t, int to_pe, uint64_t dst_off, const void* src, size_t nbytes,
              void* stream) {
  if (!t || to_pe < 0 || to_pe >= t->world) return fail(TF_ERR_INVALID, "pe out of range");
  if (dst_off + nbytes > t->heap_bytes) return fail(TF_ERR_INVALID, "range exceeds the heap");
  if (nbytes == 0) return TF_OK;
  TF_CUDA_TRY(cudaMemcpyAsync(t->pes[to_pe].base + dst_off, src, nbytes, cudaMemcpyDefault,
                              static_cast<cudaStream_t>(stream)));
  return TF_OK;
}

int tf_getmem(tf_team* t, int from_pe, uint64_t src_off, void* dst, size_t nbytes, void* stream) {
  if (!t || from_pe < 0 || from_pe >= t->world) return fail(TF_ERR_INVALID, "pe out of range");
  if (src_off + nbytes > t->heap_bytes) return fail(TF_ERR_INVALID, "range exceeds the heap");
  if (nbytes == 0) return TF_OK;
  TF_CUDA_TRY(cudaMemcpyAsync(dst, t->pes[from_pe].base + src_off, nbytes, cudaMemcpyDefault,
                              static_cast<cudaStream_t>(stream)));
  return TF_OK;
}

int tf_team_reduce(tf_team* t, int pe, uint64_t offset, int dtype, int64_t count, void* out,
                   void* stream) {
  if (!t || pe < 0 || pe >= t->world) return fail(TF_ERR_INVALID, "pe out of range");
  if (dtype < 0 || dtype > 2) return fail(TF_ERR_INVALID, "dtype must be 0 (bf16), 1 (fp32) or 2 (int64)");
  const int esz = dtype == 0 ? 2 : dtype == 1 ? 4 : 8;
  if (count < 0 || offset + static_cast<uint64_t>(count) * esz > t->heap_bytes)
    return fail(TF_ERR_INVALID, "range exceeds the heap");
  if (count == 0) return TF_OK;
  if (offset % esz) return fail(TF_ERR_INVALID, "offset must be aligned to the element size");
  tf::ReducePtrs src{};
  for (int q = 0; q < t->world; ++q) src.p[q] = t->pes[q].base + offset;
  const int threads = 256;
  const int64_t blocks64 = std::min<int64_t>((count + threads - 1) / threads, 148 * 16);
  const unsigned blocks = static_cast<unsigned>(std::max<int64_t>(blocks64, 1));
  auto s = static_cast<cudaStream_t>(stream);
  if (dtype == 0) tf::team_reduce_kernel<0><<<blocks, threads, 0, s>>>(src, t->world, count, out);
  else if (dtype == 1) tf::team_reduce_kernel<1><<<blocks, threads, 0, s>>>(src, t->world, count, out);
  else tf::team_reduce_kernel<2><<<blocks, threads, 0, s>>>(src, t->world, count, out);
  TF_CUDA_TRY(cudaGetLastError());
  return TF_OK;
}

int tf_signal_cas(tf_team* t, int pe, uint64_t slot, uint64_t cmp, uint64_t value, uint64_t* old_out,
                  void* stream) {
  if (!t || pe < 0 || pe >= t->world) return fail(TF_ERR_INVALID, "pe out of range");
  if (slot >= t->signal_slots) return fail(TF_ERR_INVALID, "slot out of range");
  if (!old_out) return fail(TF_ERR_INVALID, "old_out is NULL");
  const int me = t->ipc ? t->my_rank : pe;
  tf::DeviceGuard guard(t->pes[me].device);
  auto s = static_cast<cudaStream_t>(stream);
  unsigned long long* dold = nullptr;
  TF_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&dold), sizeof(unsigned long long), s));
  tf::signal_cas_kernel<<<1, 1, 0, s>>>(t->pes[pe].sig + slot, cmp, value, dold);
  TF_CUDA_TRY(cudaGetLastError());
  TF_CUDA_TRY(cudaMemcpyAsync(old_out, dold, sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
  TF_CUDA_TRY(cudaFreeAsync(dold, s));
  TF_CUDA_TRY(cudaStreamSynchronize(s));  // the old value is the caller's answer
  return TF_OK;
}

int tf_putmem_strided(tf_team* t, int to_pe, uint64_t dst_off, size_t dst_pitch, const void* src,
                      size_t src_pitch, size_t row_bytes, size_t rows, void* stream) {
  if (!t || to_pe < 0 || to_pe >= t->world) return fail(TF_ERR_INVALID, "pe out of range");
  if (rows == 0 || row_bytes == 0) return TF_OK;
  if (dst_pitch < row_bytes || src_pitch < row_bytes) return fail(TF_ERR_INVALID, "pitch < row bytes");
  if (dst_off + (rows - 1) * dst_pitch + row_bytes > t->heap_bytes)
    return fail(TF_ERR_INVALID, "range exceeds the heap");
  TF_CUDA_TRY(cudaMemcpy2DAsync(t->pes[to_pe].base + dst_off, dst_pitch, src, src_pitch, row_bytes, rows,
                                cudaMemcpyDefault, static_cast<cudaStream_t>(stream)));
  return TF_OK;
}

int tf_team_broadcast(tf_team* t, int from_pe, uint64_t offset, const void* src, size_t nbytes,
                      void* stream) {
  if (!t || from_pe < 0 || from_pe >= t->world) return fail(TF_ERR_INVALID, "pe out of range");
  if (offset + nbytes > t->heap_bytes) return fail(TF_ERR_INVALID, "range exceeds the heap");
  for (int q = 0; q < t->world; ++q) {
    const int pe = (from_pe + q) % t->world;  // own copy first, then the ring order
    int rc = tf_putmem(t, pe, offset, src, nbytes, stream);
    if (rc) return rc;
  }
  return TF_OK;
}

int tf_putmem_signal(tf_team* t, int to_pe, uint64_t dst_off, const void* src, size_t nbytes,
                     uint64_t sig_slot, uint64_t value, int op_add, void* stream) {
  int rc = tf_putmem(t, to_pe, dst_off, src, nbytes, stream);
  if (rc) return rc;
  return tf_signal_op(t, to_pe, sig_slot, value, op_add, stream);
}

int tf_signal_op(tf_team* t, int pe, uint64_t slot, uint64_t value, int op_add, void* stream) {
  if (!t || pe < 0 || pe >= t->world) return fail(TF_ERR_INVALID, "pe out of range");
  if (slot >= t->signal_slots) return fail(TF_ERR_INVALID, "slot out of range");
  auto s = static_cast<cudaStream_t>(stream);
  if (!op_add) return tf::stream_signal_set(t, pe, slot, value, s);
  tf::signal_op_kernel<<<1, 1, 0, s>>>(t->pes[pe].sig + slot, value, 1);
  TF_CUDA_TRY(cudaGetLastError());
  return TF_OK;
}

int tf_signal_wait_cmp(tf_team* t, int pe, uint64_t slot, size_t n, uint64_t value, int cmp,
                       void* stream) {
  if (!t || pe < 0 || pe >= t->world) return fail(TF_ERR_INVALID, "pe out of range");
  if (n < 1 || n > 1024) return fail(TF_ERR_INVALID, "wait needs 1 <= num_slots <= 1024");
  if (slot + n > t->signal_slots) return fail(TF_ERR_INVALID, "slots out of range");
  if (cmp != TF_CMP_GE && cmp != TF_CMP_EQ) return fail(TF_ERR_INVALID, "cmp must be TF_CMP_GE or TF_CMP_EQ");
  const int me = t->ipc ? t->my_rank : pe;
  tf::signal_wait_kernel<<<1, static_cast<unsigned>((n + 31) / 32 * 32), 0,
                           static_cast<cudaStream_t>(stream)>>>(t->pes[pe].sig + slot,
                                                                static_cast<int>(n), value,
                                                                cmp == TF_CMP_EQ, t->timeout_ns,
                                                                t->err_word(me));
  TF_CUDA_TRY(cudaGetLastError());
  return TF_OK;
}

int tf_signal_wait(tf_team* t, int pe, uint64_t slot, size_t n, uint64_t value, void* stream) {
  return tf_signal_wait_cmp(t, pe, slot, n, value, TF_CMP_GE, stream);
}

int tf_signal_fetch_add(tf_team* t, int pe, uint64_t slot, uint64_t value, uint64_t* old_out,
                        void* stream) {
  if (!t || pe < 0 || pe >= t->world) return fail(TF_ERR_INVALID, "pe out of range");
  if (slot >= t->signal_slots) return fail(TF_ERR_INVALID, "slot out of range");
  if (!old_out) return fail(TF_ERR_INVALID, "old_out is NULL");
  const int me = t->ipc ? t->my_rank : pe;
  tf::DeviceGuard guard(t->pes[me].device);
  auto s = static_cast<cudaStream_t>(stream);
  unsigned long long* dold = nullptr;
  TF_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&dold), sizeof(unsigned long long), s));
  tf::signal_fetch_add_kernel<<<1, 1, 0, s>>>(t->pes[pe].sig + slot, value, dold);
  TF_CUDA_TRY(cudaGetLastError());
  TF_CUDA_TRY(cudaMemcpyAsync(old_out, dold, sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
  TF_CUDA_TRY(cudaFreeAsync(dold, s));
  TF_CUDA_TRY(cudaStreamSynchronize(s));  // the old value is the caller's answer
  return TF_OK;
}

int tf_barrier_arrive(tf_team* t, int rank, void* stream) {
  if (!t || rank < 0 || rank >= t->world) return fail(TF_ERR_INVALID, "rank out of range");
  return tf::team_barrier_arrive(t, rank, static_cast<cudaStream_t>(stream));
}

int tf_barrier_wait(tf_team* t, int rank, void* stream) {
  if (!t || rank < 0 || rank >= t->world) return fail(TF_ERR_INVALID, "rank out of range");
  return tf::team_barrier_wait(t, rank, static_cast<cudaStream_t>(stream));
}

int tf_barrier_all(tf_team* t, int rank, void* stream) {
  int rc = tf_barrier_arrive(t, rank, stream);
  if (rc) return rc;
  return tf_barrier_wait(t, rank, stream);
}

}  // extern "C"
