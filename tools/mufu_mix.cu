// Does the SFU's fp64 seed instruction (MUFU.RSQ64H) share the FP64 pipe?  Time DFMA streams alone, MUFU.RSQ64H
// streams alone and both interleaved in one warp (independent chains): additive time = shared resource.
#include <cstdio>
#include <cuda_runtime.h>

template <int NF, int NM, int KINDM>
__global__ void k(double* out, int iters) {
  double a[8], b[4];
  float f[4];
  for (int i = 0; i < 8; ++i) a[i] = 1.0 + threadIdx.x * 1e-6 + i;
  for (int i = 0; i < 4; ++i) { b[i] = 1.5 + i; f[i] = 1.5f + i; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NF; ++i) a[i & 7] = fma(a[i & 7], 0.999999, 1e-7);
#pragma unroll
    for (int i = 0; i < NM; ++i) {
      if (KINDM == 0) { double r; asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(b[i & 3])); b[i & 3] = r + 1.0; }
      else { float r; asm volatile("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(f[i & 3])); f[i & 3] = r + 1.0f; }
    }
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  for (int i = 0; i < 4; ++i) s += b[i] + f[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int NF, int NM, int KM>
void run(const char* name, double* out, int sms) {
  const int iters = 4000, thr = 512, blocks = sms * 4;
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  float ms = 0;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(a);
    k<NF, NM, KM><<<blocks, thr>>>(out, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
  }
  const double warp_iters = (double)blocks * thr / 32 * iters;
  printf("%-40s %.3f ms  = %.2f SMSP-cycles per warp-iteration (DFMA %d, MUFU %d)\n", name, ms,
         ms * 1e-3 * 1.965e9 * sms * 4 / warp_iters, NF, NM);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, sizeof(double) * sms * 4 * 512);
  run<8, 0, 0>("8 DFMA", out, sms);
  run<0, 2, 0>("2 MUFU.RSQ64H", out, sms);
  run<8, 2, 0>("8 DFMA + 2 MUFU.RSQ64H", out, sms);
  run<16, 2, 0>("16 DFMA + 2 MUFU.RSQ64H", out, sms);
  run<0, 2, 1>("2 MUFU.RSQ (fp32)", out, sms);
  run<8, 2, 1>("8 DFMA + 2 MUFU.RSQ (fp32)", out, sms);
  return 0;
}
