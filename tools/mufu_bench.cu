// Throughput of the SFU (XU pipe) instructions the pair kernels use, per SM per clock, on this GPU.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mufu_bench tools/mufu_bench.cu && tools/mufu_bench
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void k(double* out, int iters, double seed) {
  double a[8];
  for (int i = 0; i < 8; ++i) a[i] = seed + threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      double r;
      if (OP == 0) asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(a[i]));
      else if (OP == 1) asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(a[i]));
      else if (OP == 2) { float f; asm volatile("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(f) : "f"((float)a[i])); r = f; }
      else if (OP == 3) { float f = (float)a[i]; r = (double)f; }
      else { asm volatile("fma.rn.f64 %0, %1, %2, %3;" : "=d"(r) : "d"(a[i]), "d"(a[i]), "d"(1e-9)); }
      a[i] = (OP == 4) ? r : a[i] + r * 1e-30;   // keep a dependency-light chain
    }
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double* out;
  cudaMalloc(&out, sizeof(double) * sms * 8 * 1024);
  const char* names[] = {"rsqrt.approx.f64 (MUFU.RSQ64H)", "rcp.approx.f64 (MUFU.RCP64H)", "f64->f32 cvt + rsqrt.f32 + cvt",
                         "f64->f32->f64 cvt", "DFMA"};
  for (int op = 0; op < 5; ++op) {
    const int iters = 2000, thr = 1024, blocks = sms * 2;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      switch (op) {
        case 0: k<0><<<blocks, thr>>>(out, iters, 1.5); break;
        case 1: k<1><<<blocks, thr>>>(out, iters, 1.5); break;
        case 2: k<2><<<blocks, thr>>>(out, iters, 1.5); break;
        case 3: k<3><<<blocks, thr>>>(out, iters, 1.5); break;
        default: k<4><<<blocks, thr>>>(out, iters, 1.5); break;
      }
      cudaEventRecord(b);
      cudaEventSynchronize(b);
    }
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const double ops = (double)blocks * thr * iters * 8;
    printf("%-36s %.3e thread-ops/s = %.2f per SM per clock (at %d MHz nominal)\n", names[op], ops / (ms * 1e-3),
           ops / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
  }
  return 0;
}
