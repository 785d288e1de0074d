// Team / symmetric-heap state shared by the runtime and the fused-op launchers.
#pragma once
#include <cstddef>
#include <cstdint>
#include <map>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "tf_internal.h"

namespace tf {

struct PE {
  int device = 0;
  uint8_t* base = nullptr;   // data region (heap_bytes)
  uint64_t* sig = nullptr;   // signal region (signal_slots)
  bool owned = false;
};

// A per-op workspace carved from the symmetric heap (same offsets on all PEs).
struct Workspace {
  size_t data_off = 0, data_bytes = 0;
  size_t sig_base = 0, sig_slots = 0;
  std::vector<uint64_t> epoch;  // per-rank call epoch of this workspace's protocol
};

const char* last_error_cstr();

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

}  // namespace tf

struct tf_team {
  int world = 1;
  int my_rank = -1;            // IPC team: this process's PE; local team: -1
  bool ipc = false;
  bool distinct_devices = true;
  size_t heap_bytes = 0, signal_slots = 0;
  size_t sig_off = 0;          // offset of the signal region inside each PE allocation
  size_t data_top = 0, sig_top = 0;
  uint64_t timeout_ns = 20ull * 1000 * 1000 * 1000;
  std::vector<tf::PE> pes;
  std::vector<uint64_t> bar_epoch;  // barrier epoch per rank
  std::vector<uint64_t> op_epoch;   // collective-call epoch per rank
  std::map<std::string, tf::Workspace> workspaces;
  std::map<int, void*> dev_tables;  // per-device scratch (freed at destroy)

  std::map<int, std::pair<void*, size_t>> scratch_bufs;  // per-device private scratch

  // NVLS multicast region (tf_nvls.cu): one multicast object over every PE's
  // physical allocation of nvls_bytes; per local PE a unicast mapping, and one
  // multicast VA through which multimem.ld_reduce / multimem.st reach all copies.
  size_t nvls_bytes = 0, nvls_top = 0;
  int nvls_state = 0;                       // 0 none, 1 object, 2 device added, 3 bound (usable)
  unsigned long long nvls_mc_handle = 0;    // CUmemGenericAllocationHandle
  std::vector<unsigned long long> nvls_phys;// per PE (local PEs only)
  std::vector<uint8_t*> nvls_uc;            // per PE unicast VA (local PEs only)
  uint8_t* nvls_mc = nullptr;               // multicast VA (this process)
  size_t nvls_gran = 0;
  std::map<std::string, size_t> nvls_ws;    // per-op workspaces carved from the NVLS region

  unsigned long long* err_word(int pe);
  void* scratch(int device, size_t bytes);
  tf::Workspace* workspace(const std::string& key, size_t data_bytes, size_t sig_slots, int* rc);
  bool is_local(int pe) const { return !ipc || pe == my_rank; }
};

namespace tf {
int stream_signal_set(tf_team* t, int pe, uint64_t slot, uint64_t value, cudaStream_t s);
int team_barrier_arrive(tf_team* t, int rank, cudaStream_t s);
int team_barrier_wait(tf_team* t, int rank, cudaStream_t s);
void nvls_release(tf_team* t);
// offset of an op workspace in the NVLS region (allocated on first use); false if
// NVLS is off or the region is too small (callers then keep their P2P path)
bool nvls_workspace(tf_team* t, const std::string& key, size_t bytes, size_t* off);
}  // namespace tf
