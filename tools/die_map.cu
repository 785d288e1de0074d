// Which die is each SM on?  For every SM in turn (L2 flushed before each probe) one
// thread times its first, dependent load of each of NL lines spread over a 1 GiB
// buffer: a line homed on the other die's memory costs an extra die-to-die hop.  The
// host splits the SMs into two groups by their latency vectors (2-means on the
// per-line latency pattern) and prints smid -> group, plus the near/far means.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/die_map.bin tools/die_map.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

constexpr int NL = 256;

__global__ void flush_kernel(uint4* p, size_t n) {
  for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    p[i] = make_uint4(i, i, i, i);
}

__global__ void probe_kernel(const uint64_t* buf, size_t stride_words, int target, int* claimed,
                             unsigned* lat) {
  unsigned smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  if (smid != static_cast<unsigned>(target) || threadIdx.x != 0) return;
  if (atomicCAS(claimed + target, 0, 1) != 0) return;
  uint64_t dep = 0;
  for (int i = 0; i < NL; ++i) {
    const uint64_t* p = buf + (static_cast<size_t>(i) * stride_words) + (dep & 1);
    const long long t0 = clock64();
    uint64_t v;
    asm volatile("ld.global.cg.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    uint64_t w;
    asm volatile("add.u64 %0, %1, 1;" : "=l"(w) : "l"(v));  // waits for the load
    const long long t1 = clock64();
    dep += w - 1;
    lat[target * NL + i] = static_cast<unsigned>(t1 - t0);
  }
  // second touch: now an L2 hit; far lines stay slower only if L2 keeps no near copy
  for (int i = 0; i < NL; ++i) {
    const uint64_t* p = buf + (static_cast<size_t>(i) * stride_words) + (dep & 1);
    const long long t0 = clock64();
    uint64_t v;
    asm volatile("ld.global.cg.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    uint64_t w;
    asm volatile("add.u64 %0, %1, 1;" : "=l"(w) : "l"(v));
    const long long t1 = clock64();
    dep += w - 1;
    lat[1024 * NL + target * NL + i] = static_cast<unsigned>(t1 - t0);
  }
  if (dep == 42) lat[0] = 0;  // keep the chain
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const size_t bytes = size_t(1) << 30;
  uint64_t* buf;
  uint4* fl;
  int* claimed;
  unsigned* lat;
  cudaMalloc(&buf, bytes);
  cudaMemset(buf, 0, bytes);
  const size_t fbytes = size_t(512) << 20;
  cudaMalloc(&fl, fbytes);
  cudaMalloc(&claimed, 1024 * sizeof(int));
  cudaMemset(claimed, 0, 1024 * sizeof(int));
  cudaMalloc(&lat, 2 * 1024 * NL * sizeof(unsigned));
  cudaMemset(lat, 0, 2 * 1024 * NL * sizeof(unsigned));
  const size_t stride_words = (bytes / NL + 4096) / 8;  // ~4 MiB + 32 KiB apart: varied channels
  int max_smid = 0;
  for (int target = 0; target < 2 * nsm && target < 1024; ++target) {
    flush_kernel<<<nsm * 4, 256>>>(fl, fbytes / 16);
    probe_kernel<<<nsm * 16, 32>>>(buf, stride_words, target, claimed, lat);
  }
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("error %s\n", cudaGetErrorString(e));
    return 1;
  }
  std::vector<int> cl(1024);
  std::vector<unsigned> h(2 * 1024 * NL);
  cudaMemcpy(cl.data(), claimed, 1024 * sizeof(int), cudaMemcpyDeviceToHost);
  cudaMemcpy(h.data(), lat, h.size() * sizeof(unsigned), cudaMemcpyDeviceToHost);
  std::vector<int> sms;
  for (int s = 0; s < 1024; ++s)
    if (cl[s]) sms.push_back(s), max_smid = s;
  printf("probed %zu SMs (max smid %d)\n", sms.size(), max_smid);
  // per-line median over SMs; sign pattern of (lat - median) per SM; 2-means on patterns
  std::vector<double> med(NL);
  for (int i = 0; i < NL; ++i) {
    std::vector<unsigned> v;
    for (int s : sms) v.push_back(h[s * NL + i]);
    std::nth_element(v.begin(), v.begin() + v.size() / 2, v.end());
    med[i] = v[v.size() / 2];
  }
  std::vector<int> grp(1024, 0);
  // seed: group 1 = SMs whose pattern anti-correlates with the first SM
  auto corr = [&](int a, int b) {
    double s = 0;
    for (int i = 0; i < NL; ++i) s += (h[a * NL + i] - med[i]) * (h[b * NL + i] - med[i]);
    return s;
  };
  for (int s : sms) grp[s] = corr(s, sms[0]) >= 0 ? 0 : 1;
  for (int it = 0; it < 10; ++it) {
    std::vector<double> c0(NL, 0), c1(NL, 0);
    int n0 = 0, n1 = 0;
    for (int s : sms) {
      auto& c = grp[s] ? c1 : c0;
      (grp[s] ? n1 : n0)++;
      for (int i = 0; i < NL; ++i) c[i] += h[s * NL + i];
    }
    for (int i = 0; i < NL; ++i) {
      c0[i] /= std::max(n0, 1);
      c1[i] /= std::max(n1, 1);
    }
    for (int s : sms) {
      double d0 = 0, d1 = 0;
      for (int i = 0; i < NL; ++i) {
        d0 += (h[s * NL + i] - c0[i]) * (h[s * NL + i] - c0[i]);
        d1 += (h[s * NL + i] - c1[i]) * (h[s * NL + i] - c1[i]);
      }
      grp[s] = d1 < d0 ? 1 : 0;
    }
    if (it == 9) {
      // near/far summary: per line, the lower group mean is "near"
      double near = 0, far = 0;
      int home0 = 0;
      for (int i = 0; i < NL; ++i) {
        near += std::min(c0[i], c1[i]);
        far += std::max(c0[i], c1[i]);
        home0 += c0[i] < c1[i];
      }
      printf("group sizes %d / %d; mean first-touch latency near %.0f clk, far %.0f clk; lines homed on group 0: %d of %d\n",
             n0, n1, near / NL, far / NL, home0, NL);
      // second touch, split by the first-touch home of each line
      double hn = 0, hf = 0;
      int nn = 0, nf = 0;
      for (int s : sms)
        for (int i = 0; i < NL; ++i) {
          const bool is_near = (grp[s] == 0) == (c0[i] < c1[i]);
          (is_near ? hn : hf) += h[1024 * NL + s * NL + i];
          (is_near ? nn : nf)++;
        }
      printf("second touch (L2 hit): near-homed %.0f clk, far-homed %.0f clk\n", hn / std::max(nn, 1),
             hf / std::max(nf, 1));
    }
  }
  printf("smid->group:");
  for (int s : sms) printf(" %d:%d", s, grp[s]);
  printf("\n");
  return 0;
}
