// FP64 peak probes for the roofline denominator (the driver's
// MEASURED_PEAKS.json has HBM and bf16 only):
//  * DFMA: 8 independent FMA chains per thread, 148 x 8 CTAs x 256 threads.
//  * DMMA: warp-level mma.sync m8n8k4 f64 (the only FP64 tensor path on
//    sm_100a; tcgen05.mma has no f64 kind), 4 independent accumulators.
// Prints one JSON line.  Timed with CUDA events after a warm-up launch.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double* out, int iters, double b, double c) {
  double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6,
         a7 = a0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
      a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

__global__ void dmma_kernel(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-3, b = 0.5;
  double c[4][2] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[q][0]), "+d"(c[q][1])
                     : "d"(a), "d"(b));
      }
    }
  }
  double s = 0;
  for (int q = 0; q < 4; ++q) s += c[q][0] + c[q][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int blocks = sms * 8, threads = 256;
  double* out;
  cudaMalloc(&out, sizeof(double) * blocks * threads);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int it = 4000;
  float best = 1e30f;
  dfma_kernel<<<blocks, threads>>>(out, 100, 0.999999, 1e-7);
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    dfma_kernel<<<blocks, threads>>>(out, it, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double dfma_tf = 2.0 * 8 * 16 * (double)it * blocks * threads / (best * 1e-3) / 1e12;
  float bestm = 1e30f;
  const int itm = 1000;
  dmma_kernel<<<blocks, threads>>>(out, 10);
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    dmma_kernel<<<blocks, threads>>>(out, itm);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < bestm) bestm = ms;
  }
  const double warps = (double)blocks * threads / 32;
  const double dmma_tf = 512.0 * 16 * 4 * (double)itm * warps / (bestm * 1e-3) / 1e12;
  cudaError_t err = cudaGetLastError();
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("{\"dfma_tflops\": %.3f, \"dmma_tflops\": %.3f, \"sms\": %d, \"clock_khz\": %d, \"dfma_ms\": %.3f, "
         "\"dmma_ms\": %.3f, \"status\": \"%s\", \"how\": \"tools/fp64_peak.cu: best of 5, CUDA events\"}\n",
         dfma_tf, dmma_tf, sms, clk, best, bestm, cudaGetErrorString(err));
  return err == cudaSuccess ? 0 : 1;
}
