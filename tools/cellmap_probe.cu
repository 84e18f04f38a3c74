// Where does the cell-map kernel's time go?  Times the product kernel against
// variants without staging (MODE 1) and without tensor-core work (MODE 2) on
// a periodic n x n grid of random data (values are irrelevant here).
//   tools/cellmap_probe [n]
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../paper_1802_05246_b200/csrc/cellmap.cuh"

using namespace hw;

template <int M, int SCH, int MODE>
float time_variant(const CellMapArgs& a) {
  using C = CMCfg<M, SCH>;
  auto k = cellmap_kernel<M, SCH, MODE>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
  int nsm = 0, per = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, C::NTHREADS, C::SMEM);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    k<<<nsm * per, C::NTHREADS, C::SMEM>>>(a);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (r > 0 && ms < best) best = ms;
  }
  return best * (per > 0 ? 1.0f : -1.0f);
}

__global__ void fill(double* p, int64_t n, double scale) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = scale * (double)((i * 2654435761ll) % 1000003 - 500001) / 500001.0;
}

template <int M, int SCH>
void probe(int64_t n, bool zeros) {
  using C = CMCfg<M, SCH>;
  CellMapArgs a;
  memset(&a, 0, sizeof(a));
  double *f0, *f1, *o0, *o1, *w, *wl;
  int *oc, *ic;
  cudaMalloc(&f0, n * n * C::P0 * 8);
  cudaMalloc(&f1, n * n * (C::P1 ? C::P1 : 1) * 8);
  cudaMalloc(&o0, n * n * C::O0 * 8);
  cudaMalloc(&o1, n * n * (C::O1 ? C::O1 : 1) * 8);
  cudaMalloc(&w, C::NK * C::NTB * 32 * 8);
  cudaMalloc(&wl, (C::WLN > 0 ? C::WLN : 1) * 8);  // hybrid-tile SIMT weights
  cudaMemset(wl, 0, (C::WLN > 0 ? C::WLN : 1) * 8);
  cudaMalloc(&oc, C::NT * 8 * 4);
  cudaMalloc(&ic, C::NK * 4 * 4);
  cudaMemset(f0, 0, n * n * C::P0 * 8);
  cudaMemset(f1, 0, n * n * (C::P1 ? C::P1 : 1) * 8);
  cudaMemset(w, 0, C::NK * C::NTB * 32 * 8);
  if (!zeros) {
    fill<<<1184, 256>>>(f0, n * n * C::P0, 1.0);
    if (C::P1) fill<<<1184, 256>>>(f1, n * n * C::P1, 1.0);
    fill<<<64, 256>>>(w, C::NK * C::NTB * 32, 0.1);
  }
  std::vector<int> h(C::NT * 8);
  for (int i = 0; i < C::NT * 8; ++i) {  // cover every output of both fields (the drain's inverse map)
    const int o = i % C::DO;
    h[i] = o < C::O0 ? o : (1 << 16) | (o - C::O0);
  }
  cudaMemcpy(oc, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  cudaMemset(ic, 0, C::NK * 4 * 4);
  a.f0 = {f0, nullptr, nullptr, 0, n};
  a.f1 = {f1, nullptr, nullptr, 0, n};
  a.wfrag = w;
  a.wleft = wl;
  a.ocode = oc;
  a.icode = ic;
  a.prev = o0;
  a.out0 = o0;
  a.out1 = o1;
  a.nx = a.ny = n;
  a.trow0 = 0;
  a.ntrows = n;
  a.nty = n;
  a.periodic = 1;
  fprintf(stderr, "probe m=%d sch=%d zeros=%d: %s\n", M, SCH, (int)zeros, cudaGetErrorString(cudaDeviceSynchronize()));
  const float t0 = time_variant<M, SCH, 0>(a);
  // 20 back-to-back launches alternating the parity offset (as a time loop does)
  float tloop = 0.f;
  {
    using C = CMCfg<M, SCH>;
    auto k = cellmap_kernel<M, SCH, 0>;
    int nsm = 0, per = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, C::NTHREADS, C::SMEM);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    CellMapArgs b = a;
    cudaEventRecord(e0);
    for (int r = 0; r < 20; ++r) {
      b.off = -(r & 1);
      k<<<nsm * per, C::NTHREADS, C::SMEM>>>(b);
    }
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&tloop, e0, e1);
    tloop /= 20.f;
  }
  fprintf(stderr, "  t0 %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  const float t1 = time_variant<M, SCH, 1>(a);
  const float t2 = time_variant<M, SCH, 2>(a);
  fprintf(stderr, "  t2 %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  const float t3 = time_variant<M, SCH, 3>(a);
  fprintf(stderr, "  t3 %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  printf("{\"zeros\": %d, \"m\": %d, \"scheme\": %d, \"n\": %ld, \"full_ms\": %.4f, \"loop20_alt_parity_ms\": %.4f, \"no_staging_ms\": %.4f, \"staging_only_ms\": %.4f, \"no_hbm_stores_ms\": %.4f, "
         "\"err\": \"%s\"}\n",
         (int)zeros, M, SCH, (long)n, t0, tloop, t1, t2, t3, cudaGetErrorString(cudaDeviceSynchronize()));
  cudaFree(f0); cudaFree(f1); cudaFree(o0); cudaFree(o1); cudaFree(w); cudaFree(wl); cudaFree(oc); cudaFree(ic);
}

int main(int argc, char** argv) {
  const int64_t n = argc > 1 ? atoll(argv[1]) : 1024;
  const char* only = argc > 2 ? argv[2] : nullptr;  // e.g. "d2" (dissipative m = 2) or "c5"
  auto want = [&](const char* k) { return only == nullptr || strcmp(only, k) == 0; };
  setvbuf(stdout, nullptr, _IOLBF, 0);
  for (int z = 1; z >= 1; --z) {
    if (want("d2")) probe<2, kDiss>(n, z);
    if (want("d3")) probe<3, kDiss>(n, z);
    if (want("d4")) probe<4, kDiss>(n, z);
    if (want("d5")) probe<5, kDiss>(n, z);
    if (want("d6")) probe<6, kDiss>(n, z);
    if (want("d7")) probe<7, kDiss>(n, z);
    if (want("d8")) probe<8, kDiss>(n, z);
    if (want("c3")) probe<3, kCons>(n, z);
    if (want("c4")) probe<4, kCons>(n, z);
    if (want("c5")) probe<5, kCons>(n, z);
    if (want("c8")) probe<8, kCons>(n, z);
  }
  return 0;
}
