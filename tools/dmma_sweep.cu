// DMMA (mma.sync m8n8k4 f64) throughput vs resident warps and independent
// accumulator chains per warp, to size the cell-map kernel's occupancy.
// Also: DMMA mixed with DADD (does the butterfly steal tensor throughput?).
// Prints one JSON object per line.
#include <cstdio>
#include <cuda_runtime.h>

template <int NACC, int NADD>
__global__ void dmma_kernel(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-3, b = 0.5;
  double c[NACC][2];
#pragma unroll
  for (int q = 0; q < NACC; ++q) c[q][0] = c[q][1] = 0.0;
  double x = threadIdx.x, y = 1.0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int q = 0; q < NACC; ++q) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[q][0]), "+d"(c[q][1])
                   : "d"(a), "d"(b));
    }
#pragma unroll
    for (int q = 0; q < NADD; ++q) {
      x = x + y;
      y = y - x;
    }
  }
  double s = x + y;
#pragma unroll
  for (int q = 0; q < NACC; ++q) s += c[q][0] + c[q][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int NACC, int NADD>
void run(int sms, int blocks_per_sm, int threads, double* out) {
  const int blocks = sms * blocks_per_sm;
  const int iters = 20000 / NACC;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  dmma_kernel<NACC, NADD><<<blocks, threads>>>(out, 10);
  float best = 1e30f;
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(e0);
    dmma_kernel<NACC, NADD><<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double warps = (double)blocks * threads / 32;
  const double tf = 512.0 * NACC * (double)iters * warps / (best * 1e-3) / 1e12;
  printf("{\"warps_per_sm\": %d, \"acc_per_warp\": %d, \"dadd_pairs_per_iter\": %d, \"dmma_tflops\": %.2f, \"ms\": %.3f}\n",
         blocks_per_sm * threads / 32, NACC, NADD, tf, best);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
}

int main() {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* out;
  cudaMalloc(&out, sizeof(double) * sms * 16 * 1024);
  const int bps[] = {1, 2, 4};
  for (int bp : bps) {
    run<1, 0>(sms, bp, 128, out);
    run<2, 0>(sms, bp, 128, out);
    run<4, 0>(sms, bp, 128, out);
    run<8, 0>(sms, bp, 128, out);
    run<16, 0>(sms, bp, 128, out);
  }
  for (int bp : bps) {
    run<4, 0>(sms, bp, 256, out);
    run<8, 0>(sms, bp, 256, out);
    run<16, 0>(sms, bp, 256, out);
  }
  // DADD interference: 8 accumulators + k DADD pairs per 8 DMMAs
  run<8, 1>(sms, 2, 256, out);
  run<8, 2>(sms, 2, 256, out);
  run<8, 4>(sms, 2, 256, out);
  run<8, 8>(sms, 2, 256, out);
  cudaError_t err = cudaDeviceSynchronize();
  printf("{\"status\": \"%s\"}\n", cudaGetErrorString(err));
  return err == cudaSuccess ? 0 : 1;
}
