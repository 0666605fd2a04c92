// FP64 peak probe for B200 (sm_100a): DMMA (mma.sync m8n8k4 f64) vs DFMA throughput,
// all SMs, long independent chains. Prints TFLOP/s (2 flops per FMA).
#include <cstdio>
#include <cuda_runtime.h>

template <int CHAINS>
__global__ void dmma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[CHAINS][2];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) { c[i][0] = 0.0; c[i][1] = 0.0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[0] = s;
}

template <int CHAINS>
__global__ void dfma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[CHAINS];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) c[i] = fma(c[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += c[i];
  if (s == 12345.0) out[0] = s;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  double* out; cudaMalloc(&out, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  printf("{\"sms\": %d, \"clock_khz\": %d}\n", sms, clk);
  for (int warps : {4, 8, 16}) {
    for (int bps : {1, 2}) {
      int iters = 4000;
      dim3 grid(sms * bps), block(32 * warps);
      dmma_loop<8><<<grid, block>>>(out, 10);
      cudaEventRecord(e0);
      dmma_loop<8><<<grid, block>>>(out, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double fl = 2.0 * 256.0 * 8 * iters * (double)grid.x * warps;
      printf("{\"probe\": \"dmma_m8n8k4\", \"warps_per_cta\": %d, \"ctas_per_sm\": %d, \"ms\": %.3f, \"tflops\": %.2f}\n", warps, bps, ms, fl / ms / 1e9);
      dfma_loop<8><<<grid, block>>>(out, 10);
      cudaEventRecord(e0);
      dfma_loop<8><<<grid, block>>>(out, iters * 8);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      fl = 2.0 * 8 * iters * 8 * (double)grid.x * block.x;
      printf("{\"probe\": \"dfma\", \"warps_per_cta\": %d, \"ctas_per_sm\": %d, \"ms\": %.3f, \"tflops\": %.2f}\n", warps, bps, ms, fl / ms / 1e9);
    }
  }
  // sustained DMMA: ~3 s back to back
  {
    dim3 grid(sms * 2), block(256);
    int iters = 20000;
    cudaEventRecord(e0);
    int reps = 0; float ms = 0;
    while (ms < 3000.f) {
      dmma_loop<8><<<grid, block>>>(out, iters); ++reps;
      cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    }
    double fl = 2.0 * 256.0 * 8 * iters * (double)grid.x * 8 * reps;
    printf("{\"probe\": \"dmma_sustained\", \"ms\": %.1f, \"tflops\": %.2f}\n", ms, fl / ms / 1e9);
  }
  cudaError_t err = cudaGetLastError();
  printf("{\"status\": \"%s\"}\n", cudaGetErrorString(err));
  return err != cudaSuccess;
}
