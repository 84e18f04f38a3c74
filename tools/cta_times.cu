// Per-CTA start / end times of the cell-map kernel (static round-robin tile
// schedule): how far apart do the persistent CTAs finish?
//   nvcc ... -DHW_CM_CTA_TIMES tools/cta_times.cu -o tools/cta_times; tools/cta_times [n]
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../paper_1802_05246_b200/csrc/cellmap.cuh"

using namespace hw;

template <int M, int SCH>
void run(int64_t n, bool dyn) {
  using C = CMCfg<M, SCH>;
  CellMapArgs a;
  memset(&a, 0, sizeof(a));
  double *f0, *f1, *o0, *o1, *w;
  int *oc, *ic;
  cudaMalloc(&f0, n * n * C::P0 * 8);
  cudaMalloc(&f1, n * n * (C::P1 ? C::P1 : 1) * 8);
  cudaMalloc(&o0, n * n * C::O0 * 8);
  cudaMalloc(&o1, n * n * (C::O1 ? C::O1 : 1) * 8);
  cudaMalloc(&w, C::NK * C::NT * 32 * 8);
  cudaMalloc(&oc, C::NT * 8 * 4);
  cudaMalloc(&ic, C::NK * 4 * 4);
  cudaMemset(f0, 0, n * n * C::P0 * 8);
  cudaMemset(f1, 0, n * n * (C::P1 ? C::P1 : 1) * 8);
  cudaMemset(w, 0, C::NK * C::NT * 32 * 8);
  std::vector<int> h(C::NT * 8);
  for (int i = 0; i < C::NT * 8; ++i) {
    const int o = i % C::DO;
    h[i] = o < C::O0 ? o : (1 << 16) | (o - C::O0);
  }
  cudaMemcpy(oc, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  cudaMemset(ic, 0, C::NK * 4 * 4);
  a.f0 = {f0, nullptr, nullptr, 0, n};
  a.f1 = {f1, nullptr, nullptr, 0, n};
  a.wfrag = w; a.ocode = oc; a.icode = ic; a.prev = o0; a.out0 = o0; a.out1 = o1;
  a.nx = a.ny = n; a.ntrows = n; a.nty = n; a.periodic = 1;
  int* sched = nullptr;
  cudaMalloc(&sched, 8);
  cudaMemset(sched, 0, 8);
  a.sched = dyn ? sched : nullptr;
  auto k = cellmap_kernel<M, SCH, 0>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int64_t ntiles = ((n + C::TJ - 1) / C::TJ) * ((n + C::TR - 1) / C::TR);
  for (int r = 0; r < 6; ++r) {
    std::vector<unsigned long long> z(2 * 1024, 0);
    cudaMemcpyToSymbol(hw_cm_cta_t, z.data(), z.size() * 8);
    k<<<nsm, C::NTHREADS, C::SMEM>>>(a);
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(z.data(), hw_cm_cta_t, z.size() * 8);
    unsigned long long s0 = ~0ull, s1 = 0, e0 = ~0ull, e1 = 0;
    std::vector<double> busy;
    for (int b = 0; b < nsm; ++b) {
      s0 = std::min(s0, z[2 * b]); s1 = std::max(s1, z[2 * b]);
      e0 = std::min(e0, z[2 * b + 1]); e1 = std::max(e1, z[2 * b + 1]);
      busy.push_back((z[2 * b + 1] - z[2 * b]) * 1e-3);
    }
    std::sort(busy.begin(), busy.end());
    printf("{\"dynamic\": %d, \"m\": %d, \"scheme\": %d, \"n\": %ld, \"tiles\": %ld, \"ctas\": %d, \"start_spread_us\": %.2f, "
           "\"first_end_us\": %.2f, \"last_end_us\": %.2f, \"busy_us_min\": %.2f, \"busy_us_p50\": %.2f, "
           "\"busy_us_p90\": %.2f, \"busy_us_max\": %.2f, \"err\": \"%s\"}\n",
           (int)dyn, M, SCH, (long)n, (long)ntiles, nsm, (s1 - s0) * 1e-3, (e0 - s0) * 1e-3, (e1 - s0) * 1e-3, busy[0],
           busy[busy.size() / 2], busy[busy.size() * 9 / 10], busy.back(), cudaGetErrorString(cudaGetLastError()));
  }
  cudaFree(sched); cudaFree(f0); cudaFree(f1); cudaFree(o0); cudaFree(o1); cudaFree(w); cudaFree(oc); cudaFree(ic);
}

int main(int argc, char** argv) {
  const int64_t n = argc > 1 ? atoll(argv[1]) : 1024;
  setvbuf(stdout, nullptr, _IOLBF, 0);
  for (int d = 0; d < 2; ++d) {
    run<4, kDiss>(n, d);
    run<6, kDiss>(n, d);
    run<2, kDiss>(n, d);
    run<5, kCons>(n, d);
  }
  return 0;
}
