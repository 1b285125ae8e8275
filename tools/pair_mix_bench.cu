// Achievable cost of one far-field pair evaluation (green_far_r, the grid kernel's inner loop body) on this GPU:
// the same instruction mix -- dot-product distance, MUFU.RSQ64H + Newton, MUFU.RCP64H of the bin midpoint, 8-byte
// shared-memory table read, cubic log1p, accumulate -- with sources taken from registers (no staging, no barriers,
// no partial warps), many independent chains per thread.  Reports SMSP-cycles per warp-pair to compare with the
// grid kernel's measured ~44.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_1906_04209_b200/csrc -o tools/pair_mix_bench tools/pair_mix_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "green.cuh"

using namespace nc;

template <int KIND, int TPT, int NS, int S32>
__global__ void __launch_bounds__(256) k_mix(const double2* __restrict__ tsrc, int fn, int fbase, int iters,
                                             double* out) {
  extern __shared__ double2 ft[];
  for (int j = threadIdx.x; j < fn / 2; j += blockDim.x) ft[j] = tsrc[j];
  __syncthreads();
  const unsigned tb = (unsigned)__cvta_generic_to_shared(ft) - 8u * (unsigned)fbase;
  const int lim = KIND == 1 ? fbase + fn - 1 : fbase;
  double a2 = -0.50000313945533437, a3 = 0.33333636142100315;
  if (iters < 0) { a2 = out[0]; a3 = out[1]; }   // opaque constants
  double x[TPT], y[TPT], z[TPT], cq[TPT], acc[TPT];
  for (int u = 0; u < TPT; ++u) {
    const double th = 0.3 + 0.001 * (threadIdx.x + 256 * u);
    x[u] = -0.5 * sin(th); y[u] = 0.0; z[u] = -0.5 * cos(th);
    cq[u] = 0.5 * (x[u] * x[u] + y[u] * y[u] + z[u] * z[u] + 0.25);
    acc[u] = 0.0;
  }
  double4 s[NS];
  for (int k = 0; k < NS; ++k) {
    const double ph = 1.0 + 0.013 * k + 0.0001 * blockIdx.x;
    s[k] = make_double4(0.5 * sin(ph), 0.01 * k, 0.5 * cos(ph), 1e-3 * (k + 1));
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < TPT; ++u) cq[u] += 1e-17;   // not loop-invariant (1 DADD per 8 pairs)
#pragma unroll
    for (int k = 0; k < NS; ++k) {
#pragma unroll
      for (int u = 0; u < TPT; ++u) {
        const double qh = fma(x[u], s[k].x, fma(y[u], s[k].y, fma(z[u], s[k].z, cq[u])));
        acc[u] = fma(s[k].w, green_far_r<KIND, 7, 3, S32>(qh, tb, lim, a2, a3, 1 << 12), acc[u]);
      }
    }
  }
  double t = 0;
  for (int u = 0; u < TPT; ++u) t += acc[u];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  // a table large enough for the indices this geometry produces (interior form, exponents 1000..1024)
  const int fbase = 1000 * 128, fn = 25 * 128;
  double2* tab;
  cudaMalloc(&tab, (fn / 2 + 1) * sizeof(double2));
  cudaMemset(tab, 0, (fn / 2 + 1) * sizeof(double2));
  double* out;
  cudaMalloc(&out, sizeof(double) * sms * 8 * 256);
  const int iters = 200, NS = 8;
  for (int s32 = 0; s32 < 4; ++s32)
  for (int blocksPerSm : {3, 4}) {
    const int blocks = sms * blocksPerSm;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float ms = 0;
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(a);
      if (s32 == 0) k_mix<0, 2, NS, 0><<<blocks, 256, fn * 8>>>(tab, fn, fbase, iters, out);
      if (s32 == 1) k_mix<0, 2, NS, 1><<<blocks, 256, fn * 8>>>(tab, fn, fbase, iters, out);
      if (s32 == 2) k_mix<0, 2, NS, 2><<<blocks, 256, fn * 8>>>(tab, fn, fbase, iters, out);
      if (s32 == 3) k_mix<0, 2, NS, 3><<<blocks, 256, fn * 8>>>(tab, fn, fbase, iters, out);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
    }
    const double warp_pairs = (double)blocks * 256 / 32 * iters * NS * 2;
    printf("S32 %d (bit0 fp32 rsqrt seed, bit1 fp32 rcp), TPT 2, %d CTAs of 256 per SM: %.3f ms, %.2f SMSP-cycles per "
           "warp-pair (at 1.965 GHz)\n", s32, blocksPerSm, ms, ms * 1e-3 * 1.965e9 * sms * 4 / warp_pairs);
  }
  return 0;
}
