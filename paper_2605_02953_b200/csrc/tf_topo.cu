// SM -> die map of a B200 (two dies, one L2 partition each).
//
// The two L2 partitions keep near copies of lines homed on the other die's memory
// (a second touch costs the same from either die), so operand tiles that both dies
// read occupy both partitions and cross the die-to-die fabric.  The persistent GEMM
// can rank its clusters die by die (tf_gemm.cu, TF_GEMM_DIE) so each die works on a
// compact block of every wave; for that it needs to know which die each SM is on.
// CUDA exposes no such attribute, so it is measured once per device: for every SM in
// turn (L2 flushed first) one thread times its first, dependent load of each of 64
// lines spread over 1 GiB -- a line homed on the other die pays the die-to-die hop
// (measured: ~675 clk near, ~1050 clk far) -- and the host splits the SMs in two by
// their latency patterns (2-means).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <map>
#include <mutex>
#include <vector>

#include "tf_internal.h"

namespace tf {
namespace {

constexpr int kNL = 64;
constexpr int kMaxSm = 256;

__global__ void topo_flush_kernel(uint4* p, size_t n) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    p[i] = make_uint4(static_cast<unsigned>(i), 0u, 0u, 0u);
}

__global__ void topo_probe_kernel(const uint64_t* buf, size_t stride_words, int target, int* claimed,
                                  unsigned* lat) {
  unsigned smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  if (smid != static_cast<unsigned>(target) || threadIdx.x != 0) return;
  if (atomicCAS(claimed + target, 0, 1) != 0) return;
  uint64_t dep = 0;
  for (int i = 0; i < kNL; ++i) {
    const uint64_t* q = buf + static_cast<size_t>(i) * stride_words + (dep & 1);
    const long long t0 = clock64();
    uint64_t v, w;
    asm volatile("ld.global.cg.u64 %0, [%1];" : "=l"(v) : "l"(q) : "memory");
    asm volatile("add.u64 %0, %1, 1;" : "=l"(w) : "l"(v));  // waits for the load
    const long long t1 = clock64();
    dep += w - 1;
    lat[target * kNL + i] = static_cast<unsigned>(t1 - t0);
  }
  if (dep == 42) lat[0] = 0;
}

struct DieMap {
  bool done = false;
  bool ok = false;
  int n_sms = 0;
  uint8_t host[kMaxSm] = {};
  uint8_t* dev = nullptr;
  unsigned long long* ctr = nullptr;  // ring of per-launch die counters
  unsigned seq = 0;
};
std::mutex g_mu;
std::map<int, DieMap> g_maps;

int probe(int dev, DieMap& m) {
  int nsm = 0;
  TF_CUDA_TRY(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  if (nsm < 2 || nsm > kMaxSm) return TF_OK;
  m.n_sms = nsm;
  const size_t bytes = size_t(1) << 30, fbytes = size_t(192) << 20;  // flush > 126 MB of L2
  uint64_t* buf = nullptr;
  uint4* fl = nullptr;
  int* claimed = nullptr;
  unsigned* lat = nullptr;
  cudaStream_t s;
  TF_CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  bool ok = cudaMalloc(&buf, bytes) == cudaSuccess && cudaMalloc(&fl, fbytes) == cudaSuccess &&
            cudaMalloc(&claimed, kMaxSm * sizeof(int)) == cudaSuccess &&
            cudaMalloc(&lat, kMaxSm * kNL * sizeof(unsigned)) == cudaSuccess;
  std::vector<int> cl(kMaxSm, 0);
  std::vector<unsigned> h(kMaxSm * kNL, 0);
  if (ok) {
    cudaMemsetAsync(buf, 0, bytes, s);
    cudaMemsetAsync(claimed, 0, kMaxSm * sizeof(int), s);
    cudaMemsetAsync(lat, 0, kMaxSm * kNL * sizeof(unsigned), s);
    const size_t stride_words = (bytes / kNL + 4096) / 8;
    for (int t = 0; t < nsm; ++t) {
      topo_flush_kernel<<<nsm * 4, 256, 0, s>>>(fl, fbytes / 16);
      topo_probe_kernel<<<nsm * 16, 32, 0, s>>>(buf, stride_words, t, claimed, lat);
    }
    ok = cudaStreamSynchronize(s) == cudaSuccess &&
         cudaMemcpy(cl.data(), claimed, kMaxSm * sizeof(int), cudaMemcpyDeviceToHost) == cudaSuccess &&
         cudaMemcpy(h.data(), lat, h.size() * sizeof(unsigned), cudaMemcpyDeviceToHost) == cudaSuccess;
  }
  cudaFree(buf);
  cudaFree(fl);
  cudaFree(claimed);
  cudaFree(lat);
  cudaStreamDestroy(s);
  cudaGetLastError();
  if (!ok) return TF_OK;
  std::vector<int> sms;
  for (int t = 0; t < nsm; ++t)
    if (cl[t]) sms.push_back(t);
  if (static_cast<int>(sms.size()) != nsm) return TF_OK;  // some SM never ran the probe
  // 2-means on the latency vectors, seeded by the correlation with SM sms[0]
  std::vector<double> med(kNL);
  for (int i = 0; i < kNL; ++i) {
    std::vector<unsigned> v;
    for (int t : sms) v.push_back(h[t * kNL + i]);
    std::nth_element(v.begin(), v.begin() + v.size() / 2, v.end());
    med[i] = v[v.size() / 2];
  }
  std::vector<int> grp(kMaxSm, 0);
  for (int t : sms) {
    double c = 0;
    for (int i = 0; i < kNL; ++i) c += (h[t * kNL + i] - med[i]) * (h[sms[0] * kNL + i] - med[i]);
    grp[t] = c >= 0 ? 0 : 1;
  }
  double gap = 0;
  for (int it = 0; it < 10; ++it) {
    std::vector<double> c0(kNL, 0), c1(kNL, 0);
    int n0 = 0, n1 = 0;
    for (int t : sms) {
      auto& c = grp[t] ? c1 : c0;
      (grp[t] ? n1 : n0)++;
      for (int i = 0; i < kNL; ++i) c[i] += h[t * kNL + i];
    }
    if (!n0 || !n1) return TF_OK;
    gap = 0;
    for (int i = 0; i < kNL; ++i) {
      c0[i] /= n0;
      c1[i] /= n1;
      gap += std::abs(c0[i] - c1[i]);
    }
    gap /= kNL;
    for (int t : sms) {
      double d0 = 0, d1 = 0;
      for (int i = 0; i < kNL; ++i) {
        d0 += (h[t * kNL + i] - c0[i]) * (h[t * kNL + i] - c0[i]);
        d1 += (h[t * kNL + i] - c1[i]) * (h[t * kNL + i] - c1[i]);
      }
      grp[t] = d1 < d0 ? 1 : 0;
    }
  }
  if (gap < 100.0) return TF_OK;  // no clear two-die signal: leave die ranking off
  for (int t = 0; t < nsm; ++t) m.host[t] = static_cast<uint8_t>(grp[t]);
  TF_CUDA_TRY(cudaMalloc(&m.dev, kMaxSm));
  TF_CUDA_TRY(cudaMemcpy(m.dev, m.host, kMaxSm, cudaMemcpyHostToDevice));
  TF_CUDA_TRY(cudaMalloc(&m.ctr, kDieCtrSlots * sizeof(unsigned long long)));
  TF_CUDA_TRY(cudaMemset(m.ctr, 0, kDieCtrSlots * sizeof(unsigned long long)));
  m.ok = true;
  return TF_OK;
}

DieMap* get_map(int dev, int* rc) {
  std::lock_guard<std::mutex> lk(g_mu);
  DieMap& m = g_maps[dev];
  *rc = TF_OK;
  if (!m.done) {
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(dev);
    *rc = probe(dev, m);
    cudaSetDevice(prev);
    m.done = true;
  }
  return &m;
}

}  // namespace

// Device table [256] of die ids (0/1) by %smid and a fresh per-launch counter slot,
// or nullptr when the device shows no two-die structure.
const uint8_t* sm_die_table(int dev, unsigned long long** ctr_slot) {
  int rc = TF_OK;
  DieMap* m = get_map(dev, &rc);
  if (rc || !m->ok) return nullptr;
  std::lock_guard<std::mutex> lk(g_mu);
  *ctr_slot = m->ctr + (m->seq++ % kDieCtrSlots);
  return m->dev;
}

}  // namespace tf

extern "C" int tf_sm_die_map(int device, uint8_t* out, int cap, int* n_sms) {
  if (!out || !n_sms || cap < 1) return tf::fail(TF_ERR_INVALID, "NULL argument");
  int rc = TF_OK;
  tf::DieMap* m = tf::get_map(device, &rc);
  if (rc) return rc;
  if (!m->ok) {
    *n_sms = 0;
    return TF_OK;
  }
  *n_sms = m->n_sms;
  memcpy(out, m->host, static_cast<size_t>(std::min(cap, m->n_sms)));
  return TF_OK;
}
