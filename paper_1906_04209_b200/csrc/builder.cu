// builder.cu -- NEXT-1, the GPU part of the Step-1 table build: the Gaussian sketch of the
// interpolative decomposition that compresses a patch's outgoing field (§7.1; Step 1(b),
// PAPER.md:1295-1299; the randomised ID of the paper's reference [liberty07]):
//
//   Y = Omega A,   A_{tf} = G(x^t_t, x^f_f)   (training points on the far-field region x fine-grid points)
//
// The CPU builder (nc_tables/skeleton.py interp_decomp) forms A in 512-row chunks with numpy and multiplies; here A
// is generated once in HBM by k_green_matrix (one thread per (f, t) entry, G in the exact single-log form with
// libdevice log / sqrt, the kernel symmetric in its arguments) and the sketch is one fp64 tensor-core GEMM
// (k_gemm_dmma).  The column-pivoted QR of the small l x n_f sketch stays on the host (nc_tables).
#include <math.h>

#include <string>

#include "nc_common.cuh"

namespace nc {

// Gt[f, t] = G(fine_f, train_t): row-major n_fine x n_train (the GEMM's Bt operand)
__global__ void k_green_matrix(int kind, const double* __restrict__ train, int64_t n_train,
                               const double* __restrict__ fine, int64_t n_fine, double* __restrict__ Gt) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t f = blockIdx.y;
  if (t >= n_train) return;
  const double dx = fine[3 * f] - train[3 * t], dy = fine[3 * f + 1] - train[3 * t + 1],
               dz = fine[3 * f + 2] - train[3 * t + 2];
  const double d = sqrt(fma(dz, dz, fma(dy, dy, dx * dx)));
  const double w = 2.0 / d;
  // G_E = w - log(1 + w);  G_I = w - log((d^2 / 4)(1 + w))   (eq:Gextonsurface / eq:Gintonsurface, single log)
  Gt[f * n_train + t] = kind == NC_EXTERIOR ? w - log1p(w) : w - log(0.25 * d * d * (1.0 + w));
}

}  // namespace nc

extern "C" int nc_id_sketch(int kind, int device, int64_t n_train, const double* train, int64_t n_fine,
                            const double* fine, int l, const double* omega, double* Y) {
  using namespace nc;
  if ((kind != NC_INTERIOR && kind != NC_EXTERIOR) || n_train < 1 || n_fine < 1 || l < 1 || !train || !fine ||
      !omega || !Y || n_fine > 65535 * 1024LL)
    return fail(NC_EINVAL, "nc_id_sketch: bad argument");
  NC_CUDA_TRY(cudaSetDevice(device));
  cudaStream_t s = nullptr;
  double *d_tr = nullptr, *d_fi = nullptr, *d_om = nullptr, *d_G = nullptr, *d_Y = nullptr;
  cudaError_t e = cudaMalloc(&d_tr, (size_t)n_train * 3 * sizeof(double));
  if (e == cudaSuccess) e = cudaMalloc(&d_fi, (size_t)n_fine * 3 * sizeof(double));
  if (e == cudaSuccess) e = cudaMalloc(&d_om, (size_t)l * n_train * sizeof(double));
  if (e == cudaSuccess) e = cudaMalloc(&d_G, (size_t)n_fine * n_train * sizeof(double));
  if (e == cudaSuccess) e = cudaMalloc(&d_Y, (size_t)l * n_fine * sizeof(double));
  int rc = NC_OK;
  if (e != cudaSuccess) {
    (void)cudaGetLastError();
    rc = fail(NC_ENOMEM, "nc_id_sketch: device allocation failed");
  } else {
    e = cudaMemcpy(d_tr, train, (size_t)n_train * 3 * sizeof(double), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(d_fi, fine, (size_t)n_fine * 3 * sizeof(double), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(d_om, omega, (size_t)l * n_train * sizeof(double), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) {
      for (int64_t f0 = 0; f0 < n_fine; f0 += 65535) {   // grid.y limit
        const int64_t nf = std::min<int64_t>(65535, n_fine - f0);
        dim3 grid((unsigned)((n_train + 255) / 256), (unsigned)nf);
        k_green_matrix<<<grid, 256, 0, s>>>(kind, d_tr, n_train, d_fi + 3 * f0, nf, d_G + f0 * n_train);
      }
      // Y (l x n_fine) = Omega (l x n_train) . Gt^T
      launch_gemm_dmma(d_om, n_train, 1, 0, d_G, l, (int)n_fine, (int)n_train, d_Y, n_fine, 1, nullptr, 0, s);
      e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpy(Y, d_Y, (size_t)l * n_fine * sizeof(double), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) rc = cuda_fail(e, "nc_id_sketch");
  }
  for (double* b : {d_tr, d_fi, d_om, d_G, d_Y}) cudaFree(b);
  return rc;
}
