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

  unsigned long long* err_word(int pe);
  void* scratch(int device, size_t bytes);
  tf::Workspace* workspace(const std::string& key, size_t data_bytes, size_t sig_slots, int* rc);
  bool is_local(int pe) const { return !ipc || pe == my_rank; }
};

namespace tf {
int stream_signal_set(tf_team* t, int pe, uint64_t slot, uint64_t value, cudaStream_t s);
int team_barrier_arrive(tf_team* t, int rank, cudaStream_t s);
int team_barrier_wait(tf_team* t, int rank, cudaStream_t s);
}  // namespace tf
