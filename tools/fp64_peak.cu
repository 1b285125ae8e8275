// FP64 peak microbenchmarks for the roofline denominators (SURVEY.md §8(d):
// "FP64 peak is not in MEASURED_PEAKS.json ... measure before reporting fractions").
// dfma: independent DFMA chains per thread; dmma: mma.sync.m8n8k4.f64 chains per warp.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  double x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__global__ void dmma_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[4][2] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[s][0]), "+d"(c[s][1]) : "d"(a), "d"(b));
      }
    }
  }
  double s = 0;
  for (int k = 0; k < 4; ++k) s += c[k][0] + c[k][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int dev = 0; cudaDeviceProp prop; cudaGetDeviceProperties(&prop, dev);
  int sms = prop.multiProcessorCount;
  double* out; cudaMalloc(&out, sizeof(double) * sms * 8 * 1024);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 4096;
  // 3 timed launches after a ~2 s sustained burst (clocks sampled during it: tools record nvidia-smi alongside)
  for (int w = 0; w < 200; ++w) dfma_kernel<<<sms * 4, 512>>>(out, iters, 0.999999, 1e-7);
  cudaDeviceSynchronize();
  for (int rep = 0; rep < 3; ++rep) {
    int blocks = sms * 4, threads = 512;
    cudaEventRecord(e0);
    dfma_kernel<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * 16 * (double)iters * blocks * threads;
    printf("{\"kind\": \"dfma\", \"tflops\": %.3f, \"ms\": %.3f}\n", flops / ms / 1e9, ms);
  }
  for (int w = 0; w < 200; ++w) dmma_kernel<<<sms * 4, 512>>>(out, iters / 4);
  cudaDeviceSynchronize();
  for (int rep = 0; rep < 3; ++rep) {
    int blocks = sms * 4, threads = 512;
    cudaEventRecord(e0);
    dmma_kernel<<<blocks, threads>>>(out, iters / 4);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * 8 * 4 * 16 * 4 * (double)(iters / 4) * blocks * (threads / 32);
    printf("{\"kind\": \"dmma\", \"tflops\": %.3f, \"ms\": %.3f}\n", flops / ms / 1e9, ms);
  }
  cudaError_t err = cudaGetLastError();
  printf("{\"sms\": %d, \"err\": \"%s\", \"clock_khz\": %d}\n", sms, cudaGetErrorString(err), prop.clockRate);
  return 0;
}
