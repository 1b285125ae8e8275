// blas.cu -- GMRES vector kernels (a7 of SURVEY.md §8(a)) and the I_sigma column sum (a8).
//
// HBM-bound; all reductions are two-stage with a fixed order (bitwise reproducible run to run).
// multidot reads w once per group of 8 basis vectors (CGS projections h = V^T w), gemv_sub applies
// w -= V h in one pass, lincomb forms x = V y at the end of the solve.
#include "nc_common.cuh"

namespace nc {

constexpr int kRedBlocks = 592;   // 4 x 148 SMs
constexpr int kGroup = 8;

int64_t multidot_partials(int64_t n) { (void)n; return kRedBlocks; }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__global__ void __launch_bounds__(256) k_multidot(const double* __restrict__ V, int64_t ldv, int nv,
                                                  const double* __restrict__ w, int64_t n, double* __restrict__ part) {
  __shared__ double red[kGroup][8];
  const int g0 = blockIdx.y * kGroup;
  double acc[kGroup];
#pragma unroll
  for (int q = 0; q < kGroup; ++q) acc[q] = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double wi = w[i];
#pragma unroll
    for (int q = 0; q < kGroup; ++q)
      if (g0 + q < nv) acc[q] = fma(V[(int64_t)(g0 + q) * ldv + i], wi, acc[q]);
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < kGroup; ++q) {
    double v = warp_sum(acc[q]);
    if (lane == 0) red[q][warp] = v;
  }
  __syncthreads();
  if (threadIdx.x < kGroup && g0 + (int)threadIdx.x < nv) {
    double v = 0.0;
    for (int k = 0; k < 8; ++k) v += red[threadIdx.x][k];
    part[(int64_t)(g0 + threadIdx.x) * gridDim.x + blockIdx.x] = v;
  }
}

__global__ void k_reduce_rows(const double* __restrict__ part, int nb, int nv, double* __restrict__ out) {
  const int i = blockIdx.x;
  if (i >= nv) return;
  double v = 0.0;
  for (int b = threadIdx.x; b < nb; b += 32) v += part[(int64_t)i * nb + b];
  v = warp_sum(v);
  if (threadIdx.x == 0) out[i] = v;
}

void launch_multidot(const double* V, int64_t ldv, int nv, const double* w, int64_t n, double* part, double* out,
                     cudaStream_t s) {
  dim3 grid(kRedBlocks, (nv + kGroup - 1) / kGroup);
  k_multidot<<<grid, 256, 0, s>>>(V, ldv, nv, w, n, part);
  k_reduce_rows<<<nv, 32, 0, s>>>(part, kRedBlocks, nv, out);
}

__global__ void __launch_bounds__(256) k_gemv_sub(const double* __restrict__ V, int64_t ldv, int nv,
                                                  const double* __restrict__ h, double* __restrict__ w, int64_t n) {
  extern __shared__ double hs[];
  for (int i = threadIdx.x; i < nv; i += blockDim.x) hs[i] = h[i];
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double v = w[i];
    for (int q = 0; q < nv; ++q) v = fma(-hs[q], V[(int64_t)q * ldv + i], v);
    w[i] = v;
  }
}

void launch_gemv_sub(const double* V, int64_t ldv, int nv, const double* h, double* w, int64_t n, cudaStream_t s) {
  k_gemv_sub<<<kRedBlocks * 2, 256, nv * sizeof(double), s>>>(V, ldv, nv, h, w, n);
}

__global__ void __launch_bounds__(256) k_lincomb(const double* __restrict__ V, int64_t ldv, int nv,
                                                 const double* __restrict__ y, double* __restrict__ x, int64_t n) {
  extern __shared__ double ys[];
  for (int i = threadIdx.x; i < nv; i += blockDim.x) ys[i] = y[i];
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double v = 0.0;
    for (int q = 0; q < nv; ++q) v = fma(ys[q], V[(int64_t)q * ldv + i], v);
    x[i] = v;
  }
}

void launch_lincomb(const double* V, int64_t ldv, int nv, const double* y, double* x, int64_t n, cudaStream_t s) {
  k_lincomb<<<kRedBlocks * 2, 256, max(nv, 1) * sizeof(double), s>>>(V, ldv, nv, y, x, n);
}

__global__ void k_scale(double* __restrict__ dst, const double* __restrict__ src, const double* __restrict__ alpha,
                        int invert, int64_t n) {
  const double a = invert ? 1.0 / alpha[0] : alpha[0];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[i] * a;
}

void launch_scale(double* dst, const double* src, const double* alpha_dev, int invert, int64_t n, cudaStream_t s) {
  k_scale<<<kRedBlocks * 2, 256, 0, s>>>(dst, src, alpha_dev, invert, n);
}

__global__ void k_fill_rows(double* __restrict__ dst, const double* __restrict__ row, int K, int64_t rows) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows * K; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = row[i % K];
}

void launch_fill_rows(double* dst, const double* row_dev, int K, int64_t rows, cudaStream_t s) {
  k_fill_rows<<<kRedBlocks, 256, 0, s>>>(dst, row_dev, K, rows);
}

// column sums of a rows x K matrix: out[k] = sum_r X[r, k]
__global__ void k_colsum_part(const double* __restrict__ X, int64_t rows, int K, double* __restrict__ part) {
  const int64_t r0 = (rows * blockIdx.x) / gridDim.x, r1 = (rows * (blockIdx.x + 1)) / gridDim.x;
  for (int k = threadIdx.x; k < K; k += blockDim.x) {
    double v = 0.0;
    for (int64_t r = r0; r < r1; ++r) v += X[r * K + k];
    part[(int64_t)blockIdx.x * K + k] = v;
  }
}

__global__ void k_colsum_final(const double* __restrict__ part, int nb, int K, double* __restrict__ out) {
  for (int k = threadIdx.x; k < K; k += blockDim.x) {
    double v = 0.0;
    for (int b = 0; b < nb; ++b) v += part[(int64_t)b * K + k];
    out[k] = v;
  }
}

void launch_colsum(const double* X, int64_t rows, int K, double* part, double* out, cudaStream_t s) {
  k_colsum_part<<<kRedBlocks, 256, 0, s>>>(X, rows, K, part);
  k_colsum_final<<<1, 256, 0, s>>>(part, kRedBlocks, K, out);
}

}  // namespace nc
