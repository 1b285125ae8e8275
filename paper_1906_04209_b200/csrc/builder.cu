// builder.cu -- NEXT-1, the GPU part of the Step-1 table build: (i) the modal kernels of the
// one-patch solver (nc_modal_kernels, below) and (ii) the Gaussian sketch of the
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
#include <vector>

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

// Gd[p, f] = G(d_pf) with d^2 = A_p + B_p s2_f (the modal-kernel integrand, nc_tables/kernel.py modal)
__global__ void k_modal_integrand(int kind, const double* __restrict__ A, const double* __restrict__ B, int64_t np_,
                                  const double* __restrict__ s2, int nphi, double* __restrict__ Gd) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t p = blockIdx.y;
  if (f >= nphi) return;
  const double d = sqrt(fma(B[p], s2[f], A[p]));
  const double w = 2.0 / d;
  // eq:Gextonsurface / eq:Gintonsurface in the single-log form (w = 2/d): G_E = w - log(1 + w), G_I = w - log(d^2/4 (1 + w))
  Gd[p * nphi + f] = kind == NC_EXTERIOR ? w - log1p(w) : w - log(0.25 * d * d * (1.0 + w));
}

}  // namespace nc

extern "C" int nc_modal_kernels(int kind, int device, int64_t npairs, const double* t, const double* tp, int M,
                                int nphi, const double* phi, const double* wphi, double* out) {
  using namespace nc;
  if ((kind != NC_INTERIOR && kind != NC_EXTERIOR) || npairs < 1 || M < 0 || nphi < 1 || !t || !tp || !phi || !wphi ||
      !out || npairs > 65535LL * 4096)
    return fail(NC_EINVAL, "nc_modal_kernels: bad argument");
  NC_CUDA_TRY(cudaSetDevice(device));
  // host: the pair terms (A, B), the phi factors s2 = sin^2(phi/2) and the cosine weights C[m, f] = w_f cos(m phi_f) / pi
  std::vector<double> A(npairs), B(npairs), s2(nphi), C((size_t)(M + 1) * nphi);
  for (int64_t p = 0; p < npairs; ++p) {
    const double h = sin(0.5 * (t[p] - tp[p]));
    A[p] = 4.0 * h * h;
    B[p] = 4.0 * sin(t[p]) * sin(tp[p]);
  }
  for (int f = 0; f < nphi; ++f) {
    const double sh = sin(0.5 * phi[f]);
    s2[f] = sh * sh;
    for (int m = 0; m <= M; ++m) C[(size_t)m * nphi + f] = wphi[f] * cos(m * phi[f]) / M_PI;
  }
  double *d_A = nullptr, *d_B = nullptr, *d_s2 = nullptr, *d_C = nullptr, *d_G = nullptr, *d_out = nullptr;
  cudaError_t e = cudaMalloc(&d_A, npairs * sizeof(double));
  if (e == cudaSuccess) e = cudaMalloc(&d_B, npairs * sizeof(double));
  if (e == cudaSuccess) e = cudaMalloc(&d_s2, nphi * sizeof(double));
  if (e == cudaSuccess) e = cudaMalloc(&d_C, C.size() * sizeof(double));
  if (e == cudaSuccess) e = cudaMalloc(&d_G, (size_t)npairs * nphi * sizeof(double));
  if (e == cudaSuccess) e = cudaMalloc(&d_out, (size_t)npairs * (M + 1) * sizeof(double));
  int rc = NC_OK;
  if (e != cudaSuccess) {
    (void)cudaGetLastError();
    rc = fail(NC_ENOMEM, "nc_modal_kernels: device allocation failed");
  } else {
    e = cudaMemcpy(d_A, A.data(), npairs * sizeof(double), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(d_B, B.data(), npairs * sizeof(double), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(d_s2, s2.data(), nphi * sizeof(double), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(d_C, C.data(), C.size() * sizeof(double), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) {
      for (int64_t p0 = 0; p0 < npairs; p0 += 65535) {   // grid.y limit
        const int64_t np_ = std::min<int64_t>(65535, npairs - p0);
        dim3 grid((unsigned)((nphi + 255) / 256), (unsigned)np_);
        k_modal_integrand<<<grid, 256>>>(kind, d_A + p0, d_B + p0, np_, d_s2, nphi, d_G + p0 * nphi);
      }
      // out (npairs x (M+1)) = Gd (npairs x nphi) . C^T, C row-major (M+1) x nphi
      launch_gemm_dmma(d_G, nphi, 1, 0, d_C, npairs, M + 1, nphi, d_out, M + 1, 1, nullptr, 0, nullptr);
      e = cudaGetLastError();
    }
    if (e == cudaSuccess)
      e = cudaMemcpy(out, d_out, (size_t)npairs * (M + 1) * sizeof(double), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) rc = cuda_fail(e, "nc_modal_kernels");
  }
  for (double* b : {d_A, d_B, d_s2, d_C, d_G, d_out}) cudaFree(b);
  return rc;
}

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
