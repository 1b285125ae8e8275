// field.cu -- NEXT-3 and NEXT-4.
//
// NEXT-3: the single-layer potential of the solved densities at off-surface points,
//
//   interior (narrow escape):   v(p) = sum_j sum_m G_I(p, s_jm) rho_jm      eq:intBVPansatz
//   exterior (narrow capture):  u(p) = sum_j sum_m G_E(p, s_jm) rho_jm      eq:urep
//
// every patch's density in its compressed outgoing representation (skeleton nodes s_jm, charges rho_j = T fhat_j,
// eq:outgoingcompressed PAPER.md:1078-1096), with the off-surface Neumann Green's functions
//   G_I(x, x') = 2/|x - x'| + log( 2 / (1 - x.x' + |x - x'|) )                   eq:Gintoffsurface
//   G_E(x, x') = 2/|x - x'| + log( (|x| - x.x') / (1 - x.x' + |x - x'|) )        eq:Gextoffsurface
// The exterior ratio is evaluated without cancellation: with a = |x|, c = x.x', d = |x - x'| and
// d^2 = a^2 - 2c + 1, (1 - c + d)(d - 1 + c) = a^2 - c^2, so the ratio equals (d + c - 1) / (a + c), used when
// c >= 0 (the literal form is 0/0 for x on the ray through x'); the literal form when c < 0.
// Targets must be off the surface on the problem's side and well separated from every patch (nc_field checks).
// One CTA of 256 threads per tile of targets x one segment of the source records; fixed-order segment reduction.
#include <math.h>

#include <algorithm>

#include "green.cuh"
#include "nc_common.cuh"

namespace nc {

constexpr int kFieldThreads = 256;
constexpr int kFieldStage = 512;   // source records per shared-memory stage

template <int KIND>
__device__ __forceinline__ double green_off(double px, double py, double pz, double a, double sx, double sy,
                                            double sz) {
  const double dx = px - sx, dy = py - sy, dz = pz - sz;
  const double d2 = fma(dz, dz, fma(dy, dy, dx * dx));
  const double rd = rsqrt(d2);
  const double d = d2 * rd;
  const double c = fma(pz, sz, fma(py, sy, px * sx));
  if (KIND == 0) return 2.0 * rd + (0.69314718055994530942 - log((1.0 - c) + d));
  if (c >= 0.0) return 2.0 * rd + log(((d + c) - 1.0) / (a + c));
  return 2.0 * rd + log((a - c) / ((1.0 - c) + d));
}

// The same G from the squared distance alone (the sum kernel's form, round 2): with a = |x|, |x'| = 1 and
// d^2 = |x - x'|^2 (coordinate differences, no cancellation), 1 - x.x' = (d^2 + 1 - a^2) / 2, so
//   G_I = 2/d + log 2 - log(d^2 / 2 + d + B),                B = (1 - a^2) / 2 per point
//   G_E = 2/d + log(d - d^2 / 2 - B) - log(a + (a^2 + 1 - d^2) / 2)      (the c >= 0 rewrite of R27; B = (1 - a^2)/2)
// with 1/d by the MUFU seed and a third-order Newton step (fast_rsqrt, full precision) and log by the exponent-reduced
// 1024-entry mantissa table (fast_log, ~1e-16 relative): ~25 FP64 instructions per pair instead of libdevice's ~50.
// The exterior form is used for c = (a^2 + 1 - d^2) / 2 >= 0, the literal ratio otherwise (as green_off).
template <int KIND>
__device__ __forceinline__ double green_off_fast(double px, double py, double pz, double a, double B, double sx,
                                                 double sy, double sz, const double2* __restrict__ tbl) {
  const double dx = px - sx, dy = py - sy, dz = pz - sz;
  const double d2 = fma(dz, dz, fma(dy, dy, dx * dx));
  const double rd = fast_rsqrt(d2);
  const double d = d2 * rd;
  if (KIND == 0) return fma(2.0, rd, 0.69314718055994530942) - fast_log(fma(0.5, d2, B) + d, tbl);
  const double c = fma(-0.5, d2, 0.5 * (a * a + 1.0));
  if (c >= 0.0) return 2.0 * rd + (fast_log(d - fma(0.5, d2, B), tbl) - fast_log(a + c, tbl));
  return 2.0 * rd + (fast_log(a - c, tbl) - fast_log((1.0 - c) + d, tbl));
}

template <int KIND>
__global__ void __launch_bounds__(kFieldThreads) k_field(const double* __restrict__ pts, int64_t n,
                                                         const double4* __restrict__ s4, int64_t nrec, int nseg,
                                                         double* __restrict__ part, double* __restrict__ dpart,
                                                         const double2* __restrict__ logsrc) {
  __shared__ double4 sm[kFieldStage];
  __shared__ double2 logtab[kLogTableSize];
  init_log_table(logtab, logsrc);
  const int64_t t = (int64_t)blockIdx.x * kFieldThreads + threadIdx.x;
  const int64_t tc = t < n ? t : n - 1;
  const double px = pts[3 * tc], py = pts[3 * tc + 1], pz = pts[3 * tc + 2];
  const double a = sqrt(fma(pz, pz, fma(py, py, px * px)));
  const double B = 0.5 * (1.0 - a * a);
  const int seg = blockIdx.y;
  const int64_t r0 = nrec * seg / nseg, r1 = nrec * (seg + 1) / nseg;
  double acc = 0.0, dm = INFINITY;
  for (int64_t c0 = r0; c0 < r1; c0 += kFieldStage) {
    const int nc = (int)min((int64_t)kFieldStage, r1 - c0);
    __syncthreads();
    for (int r = threadIdx.x; r < nc; r += kFieldThreads) sm[r] = s4[c0 + r];
    __syncthreads();
#pragma unroll 2
    for (int r = 0; r < nc; ++r) {
      const double4 s = sm[r];   // coordinates stored x 1/2
      const double sx = 2.0 * s.x, sy = 2.0 * s.y, sz = 2.0 * s.z;
      const double dx = px - sx, dy = py - sy, dz = pz - sz;
      dm = fmin(dm, fma(dz, dz, fma(dy, dy, dx * dx)));
      acc = fma(s.w, green_off_fast<KIND>(px, py, pz, a, B, sx, sy, sz, logtab), acc);
    }
  }
  if (t < n) {
    part[(int64_t)seg * n + t] = acc;
    dpart[(int64_t)seg * n + t] = dm;
  }
}

__global__ void k_field_reduce(const double* __restrict__ part, const double* __restrict__ dpart, int64_t n, int nseg,
                               double* __restrict__ out, double* __restrict__ dmin) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  double v = 0.0, m = INFINITY;
  for (int s = 0; s < nseg; ++s) {
    v += part[(int64_t)s * n + t];
    m = fmin(m, dpart[(int64_t)s * n + t]);
  }
  out[t] = v;
  dmin[t] = sqrt(m);
}

// segments so that the launch fills about two waves of CTAs
int field_segments(int64_t n, int64_t nrec) {
  int sms = 148, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t tiles = (n + kFieldThreads - 1) / kFieldThreads;
  int64_t nseg = (2 * 4 * (int64_t)sms + tiles - 1) / std::max<int64_t>(tiles, 1);
  nseg = std::max<int64_t>(1, std::min<int64_t>(nseg, std::max<int64_t>(1, nrec / kFieldStage)));
  return (int)std::min<int64_t>(nseg, 1024);
}

void launch_field(int kind, const double* pts, int64_t n, const double* src4, int64_t nrec, int nseg, double* part,
                  double* dpart, double* out, double* dmin, cudaStream_t s) {
  if (n <= 0) return;
  dim3 grid((unsigned)((n + kFieldThreads - 1) / kFieldThreads), (unsigned)nseg);
  const double4* s4 = reinterpret_cast<const double4*>(src4);
  if (kind == NC_EXTERIOR)
    k_field<1><<<grid, kFieldThreads, 0, s>>>(pts, n, s4, nrec, nseg, part, dpart, log_table_device());
  else
    k_field<0><<<grid, kFieldThreads, 0, s>>>(pts, n, s4, nrec, nseg, part, dpart, log_table_device());
  k_field_reduce<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(part, dpart, n, nseg, out, dmin);
}

// NEXT-4: the relative L2 residual of the multiple-scattering system on patch i (eq:l2res),
//   res_i = || S sigma_i + sum_{j != i} S_ij sigma_j - 1 ||_{L2(Gamma_i)} / |Gamma_i|
// on the tables' residual grid.  The field of the other patches comes from the direct pair kernel (api.cu launches
// k_pairs_direct per listed patch with the grid as its targets); this kernel adds the self term res_S fhat_i,
// subtracts the data 1, and forms the weighted norm.  One CTA per listed patch; fixed-order reductions.
__global__ void k_residual(int n_sel, int n_res, int K, int nseg, const int64_t* __restrict__ rows,
                           const double* __restrict__ x_all, const double* __restrict__ S,
                           const double* __restrict__ w, const double* __restrict__ upart,
                           double* __restrict__ pointwise, double* __restrict__ res) {
  __shared__ double red[256];
  const int q = blockIdx.x;
  const double* xi = x_all + rows[q] * K;
  const double* up = upart + (size_t)q * nseg * n_res;
  double acc = 0.0, area = 0.0;
  for (int k = threadIdx.x; k < n_res; k += blockDim.x) {
    double u = 0.0;
    for (int sg = 0; sg < nseg; ++sg) u += up[(size_t)sg * n_res + k];
    double self = 0.0;
    for (int a = 0; a < K; ++a) self = fma(S[(size_t)k * K + a], xi[a], self);
    const double r = (self + u) - 1.0;
    pointwise[(size_t)q * n_res + k] = r;
    acc = fma(w[k] * r, r, acc);
    area += w[k];
  }
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  const double tot = red[0];
  __syncthreads();
  red[threadIdx.x] = area;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) res[q] = sqrt(tot) / red[0];
}

// density recovery (NEXT-3, eq:recoversig PAPER.md:797-807): gather the listed patches' coefficient rows
__global__ void k_gather_rows(const double* __restrict__ x_all, const int64_t* __restrict__ rows, int n_sel, int K,
                              double* __restrict__ out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)n_sel * K) return;
  out[t] = x_all[rows[t / K] * K + t % K];
}

void launch_gather_rows(const double* x_all, const int64_t* rows, int n_sel, int K, double* out, cudaStream_t s) {
  if (n_sel <= 0) return;
  k_gather_rows<<<(unsigned)(((int64_t)n_sel * K + 255) / 256), 256, 0, s>>>(x_all, rows, n_sel, K, out);
}

void launch_residual(int n_sel, int n_res, int K, int nseg, const int64_t* rows, const double* x_all, const double* S,
                     const double* w, const double* upart, double* pointwise, double* res, cudaStream_t s) {
  if (n_sel <= 0) return;
  k_residual<<<(unsigned)n_sel, 256, 0, s>>>(n_sel, n_res, K, nseg, rows, x_all, S, w, upart, pointwise, res);
}

}  // namespace nc
