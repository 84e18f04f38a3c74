// Micro-benchmark of the cell-map k-step loop in isolation (operands resident
// in shared memory, no staging, no stores) to see what limits DMMA issue:
//   V0 full k-step: 4 corner LDS per M-tile + sign flips + butterfly, NT B LDS
//   V1 B fragments held in registers (no B LDS)
//   V2 no butterfly (A = one corner LDS per M-tile and class)
//   V3 A and B from registers (DMMA only)
// Prints DMMA TFLOP/s per variant and warps per SM.
#include <cstdio>
#include <cuda_runtime.h>

constexpr int KCP = 20, TJ = 32, NODES = 9 * 33, NTMAX = 20;

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}
__device__ __forceinline__ void dmma0(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%4};\n"
               : "=d"(d[0]), "=d"(d[1])
               : "d"(a), "d"(b), "d"(0.0));
}
__device__ __forceinline__ double flip(double x, unsigned long long m) {
  return __longlong_as_double(__double_as_longlong(x) ^ m);
}

template <int V, int MT, int BAR, int MINB, int NT>
__global__ void __launch_bounds__(256, MINB) loop_kernel(double* out, int iters) {
  extern __shared__ double sm[];
  double* cb = sm;
  double* wb = sm + NODES * KCP;
  for (int i = threadIdx.x; i < NODES * KCP + 4 * NTMAX * 32; i += blockDim.x) sm[i] = 1e-3 * (i % 17);
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double acc[MT][NT][2];
#pragma unroll
  for (int t = 0; t < MT; ++t)
#pragma unroll
    for (int n = 0; n < NT; ++n) acc[t][n][0] = acc[t][n][1] = 0.0;
  double breg[NT], areg[MT][4];
#pragma unroll
  for (int n = 0; n < NT; ++n) breg[n] = wb[n * 32 + lane];
#pragma unroll
  for (int t = 0; t < MT; ++t)
#pragma unroll
    for (int c = 0; c < 4; ++c) areg[t][c] = cb[t * 64 + c * 8 + lane];
  unsigned long long mx = (unsigned long long)(lane & 1) << 63, my = (unsigned long long)(lane & 2) << 62;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
      double A[MT][4];
#pragma unroll
      for (int t = 0; t < MT; ++t) {
        const int mt = warp * MT + t;
        const int trl = mt / 4, tc = (mt % 4) * 8;  // TR = 2 * MT rows
        const double* p = cb + (trl * (TJ + 1) + tc + (lane >> 2)) * KCP + ks * 4 + (lane & 3);
        if (V == 0 || V == 1) {
          const double c00 = p[0], c01 = flip(p[KCP], my), c10 = flip(p[(TJ + 1) * KCP], mx),
                       c11 = flip(p[(TJ + 2) * KCP], mx ^ my);
          const double ap = c00 + c10, am = c00 - c10, bp = c01 + c11, bm = c01 - c11;
          A[t][0] = ap + bp;
          A[t][1] = ap - bp;
          A[t][2] = am + bm;
          A[t][3] = am - bm;
        } else if (V == 2) {
          A[t][0] = p[0];
          A[t][1] = p[KCP];
          A[t][2] = p[(TJ + 1) * KCP];
          A[t][3] = p[(TJ + 2) * KCP];
        } else {
#pragma unroll
          for (int c = 0; c < 4; ++c) A[t][c] = areg[t][c];
        }
      }
      const double* wk = wb + ks * NT * 32 + lane;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const int c = (nt * 4) / NT;
        const double b = (V == 1 || V == 3) ? breg[nt] : wk[nt * 32];
        if (BAR >= 3 && ks == 0 && it % 3 == 0) {
#pragma unroll
          for (int t = 0; t < MT; ++t) dmma0(acc[t][nt], A[t][c], b);
        } else {
#pragma unroll
          for (int t = 0; t < MT; ++t) dmma(acc[t][nt], A[t][c], b);
        }
      }
    }
    if (BAR) __syncthreads();
    if (BAR == 3 && it % 3 == 2) {  // stores of a realistic pattern, no reset (next tile starts with C = 0)
      double* o = out + (size_t)(blockIdx.x * 8 + warp) * MT * 8 * 41;
#pragma unroll
      for (int t = 0; t < MT; ++t)
#pragma unroll
        for (int n = 0; n < NT; ++n)
#pragma unroll
          for (int i = 0; i < 2; ++i) o[(t * 8 + (lane >> 2)) * 41 + (n * 8 + (lane & 3) * 2 + i) % 41] = acc[t][n][i];
    }
    if (BAR == 4 && it % 3 == 2) {  // stores staged through shared memory, written coalesced
      double* o = out + (size_t)(blockIdx.x * 8 + warp) * MT * 8 * 41;
      double* st = sm + NODES * KCP + 4 * NTMAX * 32 + warp * 8 * 41;
#pragma unroll
      for (int t = 0; t < MT; ++t) {
#pragma unroll
        for (int n = 0; n < NT; ++n)
#pragma unroll
          for (int i = 0; i < 2; ++i) st[(lane >> 2) * 41 + (n * 8 + (lane & 3) * 2 + i) % 41] = acc[t][n][i];
        __syncwarp();
        for (int q = lane; q < 8 * 41; q += 32) o[t * 8 * 41 + q] = st[q];
        __syncwarp();
      }
    }
    if (BAR == 2 && it % 3 == 2) {  // epilogue-like stores + reset
#pragma unroll
      for (int t = 0; t < MT; ++t)
#pragma unroll
        for (int n = 0; n < NT; ++n) {
          out[(blockIdx.x * blockDim.x + threadIdx.x) * 64 + (n * 2 + t) % 64] = acc[t][n][0] + acc[t][n][1];
          acc[t][n][0] = acc[t][n][1] = 0.0;
        }
    }
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < MT; ++t)
#pragma unroll
    for (int n = 0; n < NT; ++n) s += acc[t][n][0] + acc[t][n][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int V, int MT, int BAR, int MINB, int NT = 7>
void run(int sms, int bps, double* out) {
  const int smem = (NODES * KCP + 4 * NTMAX * 32 + 8 * 8 * 41) * 8;
  cudaFuncSetAttribute(loop_kernel<V, MT, BAR, MINB, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 2000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  loop_kernel<V, MT, BAR, MINB, NT><<<sms * bps, 256, smem>>>(out, 10);
  float best = 1e30f;
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(e0);
    loop_kernel<V, MT, BAR, MINB, NT><<<sms * bps, 256, smem>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double dmmas = (double)sms * bps * 8 * iters * 4 * NT * MT;
  printf("{\"nt\": %d, \"variant\": %d, \"mt\": %d, \"bar\": %d, \"warps_per_sm\": %d, \"dmma_tflops\": %.2f, \"err\": \"%s\"}\n", NT, V, MT, BAR, bps * 8,
         dmmas * 512 / (best * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, (size_t)sms * 4 * 256 * 64 * 8);
  run<0, 2, 1, 2, 7>(sms, 2, out);
  run<0, 1, 1, 1, 20>(sms, 1, out);
  run<0, 1, 1, 2, 20>(sms, 2, out);
  run<1, 1, 1, 1, 20>(sms, 1, out);
  run<2, 1, 1, 1, 20>(sms, 1, out);
  run<3, 1, 1, 1, 20>(sms, 1, out);
  run<0, 2, 1, 1, 10>(sms, 1, out);
  run<0, 2, 1, 2, 10>(sms, 2, out);
  run<0, 1, 1, 2, 10>(sms, 2, out);
  run<0, 4, 1, 1, 5>(sms, 1, out);
  return 0;
}
