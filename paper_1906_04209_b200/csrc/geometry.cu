// geometry.cu -- patch frames and global node sets (Step 2(b): "For each patch,
// construct the Zernike sampling grid").
//
// Frame rule (R8, part of the ABI; the paper only says "a coordinate system fixed about the
// centre"): e1 = normalize(xhat - (xhat.c) c), with yhat in place of xhat when
// |c.xhat| > 0.9; e2 = c x e1; R_i = [e1 e2 c_i].  Global nodes z_{ik} = R_i zhat_k, s_{jm} = R_j shat_m.
#include "nc_common.cuh"

namespace nc {

__global__ void k_frames(const double* __restrict__ c, int64_t N, double* __restrict__ R) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= N) return;
  double cx = c[3 * i], cy = c[3 * i + 1], cz = c[3 * i + 2];
  double ax = 1.0, ay = 0.0;
  if (fabs(cx) > 0.9) { ax = 0.0; ay = 1.0; }
  double dot = ax * cx + ay * cy;
  double ex = ax - dot * cx, ey = ay - dot * cy, ez = -dot * cz;
  double inv = 1.0 / sqrt(ex * ex + ey * ey + ez * ez);
  ex *= inv; ey *= inv; ez *= inv;
  // e2 = c x e1
  double fx = cy * ez - cz * ey, fy = cz * ex - cx * ez, fz = cx * ey - cy * ex;
  double* r = R + 9 * i;   // column-major: r[0..2] = e1, r[3..5] = e2, r[6..8] = c
  r[0] = ex; r[1] = ey; r[2] = ez;
  r[3] = fx; r[4] = fy; r[5] = fz;
  r[6] = cx; r[7] = cy; r[8] = cz;
}

__device__ __forceinline__ void apply_frame(const double* r, double a, double b, double c, double& x, double& y,
                                            double& z) {
  x = r[0] * a + r[3] * b + r[6] * c;
  y = r[1] * a + r[4] * b + r[7] * c;
  z = r[2] * a + r[5] * b + r[8] * c;
}

__global__ void k_targets(const double* __restrict__ R, int64_t row_begin, int64_t row_count,
                          const double* __restrict__ zhat, int Kstar, double scale, double* tx, double* ty,
                          double* tz) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= row_count * Kstar) return;
  int64_t i = row_begin + t / Kstar;
  int k = (int)(t % Kstar);
  double x, y, z;
  apply_frame(R + 9 * i, zhat[3 * k], zhat[3 * k + 1], zhat[3 * k + 2], x, y, z);
  tx[t] = scale * x; ty[t] = scale * y; tz[t] = scale * z;
}

__global__ void k_sources(const double* __restrict__ R, int64_t N, const double* __restrict__ shat, int p,
                          double scale, double* __restrict__ src4) {
  int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= N * p) return;
  int64_t j = s / p;
  int m = (int)(s % p);
  double x, y, z;
  apply_frame(R + 9 * j, shat[3 * m], shat[3 * m + 1], shat[3 * m + 2], x, y, z);
  src4[4 * s] = scale * x; src4[4 * s + 1] = scale * y; src4[4 * s + 2] = scale * z; src4[4 * s + 3] = 0.0;
}

void launch_frames(const double* centers, int64_t N, double* frames, cudaStream_t s) {
  k_frames<<<(unsigned)((N + 255) / 256), 256, 0, s>>>(centers, N, frames);
}

void launch_targets(const double* frames, int64_t row_begin, int64_t row_count, const double* zhat, int Kstar,
                    double scale, double* tx, double* ty, double* tz, cudaStream_t s) {
  int64_t n = row_count * Kstar;
  if (n == 0) return;
  k_targets<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(frames, row_begin, row_count, zhat, Kstar, scale, tx, ty,
                                                       tz);
}

void launch_sources(const double* frames, int64_t N, const double* shat, int p, double scale, double* src4,
                    cudaStream_t s) {
  int64_t n = N * p;
  k_sources<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(frames, N, shat, p, scale, src4);
}

}  // namespace nc
