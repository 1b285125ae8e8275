// nearfield.cu -- NEXT-3 near the surface (the MFPT is plotted on the sphere of
// radius 1 - eps/5, inside the layer where the compressed skeleton of a patch is not valid).
//
// The potential of the solution at an off-surface point p is  v(p) = sum_j int_{Gamma_j} G_off(p, x') sigma_j dS
// (eq:intBVPansatz PAPER.md:556-558 interior, eq:urep PAPER.md:466-468 exterior).  nc_field evaluates every patch
// through its compressed skeleton, valid >= 3 eps from the skeleton nodes (R27).  Here the patches whose
// centre is closer than kNearRadius eps to p are evaluated through their density itself, sigma_j = B fhat_j
// (eq:recoversig PAPER.md:797-807), known at the one-patch solver's radial nodes:
//   sigma_j(t, theta) = sum_m A_m(t) cos(m theta) + B_m(t) sin(m theta),  A_m(t) = sum_{a: m_a = m, cos} fhat_a sigma_a(t)
// by the quadrature  int_0^eps sin t int_0^2pi G_off(p, x'(t, theta)) sigma(t, theta) dtheta dt  with
//   * radial: the solver's panels; a regular panel whose length exceeds half the distance from p to its ring band is
//     bisected until every piece is at most that, each piece with the panel's Gauss-Legendre rule and sigma from the
//     panel's degree-(k-1) interpolant (barycentric); the last panel (the 1/sqrt(eps - t) edge density, Gauss-Jacobi
//     weights folded into the table's w) is always native, which bounds how close p may come (kNearMinHeight);
//   * angular: the trapezoid rule on 2^k points, k chosen per radius so that the aliasing error of the analytic
//     periodic integrand, ~exp(-n alpha) with alpha = acosh(1 + d^2 / (2 rho_p sin t)) the imaginary distance of its
//     nearest singularity (d = distance from p to the ring), is below 1e-16.
// One CTA per (point, near patch) pair: the patch's profiles at all native radial nodes in shared memory; each warp
// takes radial nodes, its lanes the angles (sigma synthesised by the cos / sin recurrences, the 32 profile values held
// in every lane's registers by warp shuffles).  The pair's correction  (density quadrature - compressed skeleton sum)
// is added to nc_field's compressed total in fixed pair order (deterministic).
#include <math.h>

#include <algorithm>

#include "nc_common.cuh"

namespace nc {

constexpr int kNearThreads = 256;
constexpr int kNearMaxNodes = 2048;    // radial nodes per pair (native + refined)
constexpr int kNearMaxM1 = 16;         // angular orders 0..15 (2 M1 <= 32 profile components: one per lane)
constexpr int kTrigN = kNearTrigN;     // the angle table; the largest trapezoid rule

template <int KIND>
__device__ __forceinline__ double green_off_near(double px, double py, double pz, double a, double sx, double sy,
                                                 double sz) {
  // eq:Gintoffsurface / eq:Gextoffsurface; the exterior ratio without cancellation as in
  // field.cu (R27)
  const double dx = px - sx, dy = py - sy, dz = pz - sz;
  const double d2 = fma(dz, dz, fma(dy, dy, dx * dx));
  const double rd = rsqrt(d2);
  const double d = d2 * rd;
  const double c = fma(pz, sz, fma(py, sy, px * sx));
  if (KIND == 0) return 2.0 * rd + (0.69314718055994530942 - log((1.0 - c) + d));
  if (c >= 0.0) return 2.0 * rd + log(((d + c) - 1.0) / (a + c));
  return 2.0 * rd + log((a - c) / ((1.0 - c) + d));
}

// near pairs: patches whose centre is within r of the point (brute force over the centres, tiles in shared memory)
__global__ void k_near_count(const double* __restrict__ pts, int64_t n, const double* __restrict__ cen, int64_t N,
                             double r2, int64_t* __restrict__ cnt, int64_t* __restrict__ list, const int64_t* off) {
  __shared__ double sc[3 * 256];
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t tc = t < n ? t : n - 1;
  const double px = pts[3 * tc], py = pts[3 * tc + 1], pz = pts[3 * tc + 2];
  int64_t c = 0;
  const int64_t o = (list && t < n) ? off[t] : 0;
  for (int64_t j0 = 0; j0 < N; j0 += 256) {
    const int nj = (int)min((int64_t)256, N - j0);
    __syncthreads();
    for (int e = threadIdx.x; e < 3 * nj; e += blockDim.x) sc[e] = cen[3 * j0 + e];
    __syncthreads();
    for (int j = 0; j < nj; ++j) {
      const double dx = px - sc[3 * j], dy = py - sc[3 * j + 1], dz = pz - sc[3 * j + 2];
      if (fma(dz, dz, fma(dy, dy, dx * dx)) < r2) {
        if (list && t < n) list[o + c] = j0 + j;
        ++c;
      }
    }
  }
  if (t < n && !list) cnt[t] = c;
}


template <int KIND>
__global__ void __launch_bounds__(kNearThreads) k_near_quad(const int64_t* __restrict__ pair_pt,
                                                            const int64_t* __restrict__ pair_patch, int64_t npairs,
                                                            const double* __restrict__ pts,
                                                            const double* __restrict__ frames,
                                                            const double* __restrict__ x_all, NearDev nd,
                                                            const double* __restrict__ rec, int p0,
                                                            double* __restrict__ corr, int* __restrict__ status) {
  extern __shared__ double smn[];
  double* prof = smn;                                           // n_r x 2 M1 profile values (A_m, B_m) at native nodes
  double* nd_t = prof + (size_t)nd.n_r * 2 * nd.M1;
  double* nd_w = nd_t + kNearMaxNodes;
  int* nd_src = reinterpret_cast<int*>(nd_w + kNearMaxNodes);
  __shared__ double red[kNearThreads / 32];
  __shared__ double sp[6];                                      // p in the patch frame, |p|, rho_p
  __shared__ int nnodes, bad;
  const int64_t q = blockIdx.x;
  const int64_t pt = pair_pt[q], j = pair_patch[q];
  const int M1 = nd.M1, C = 2 * M1;
  if (threadIdx.x == 0) {
    const double* R = frames + 9 * j;                           // [e1 | e2 | c], column-major
    const double px = pts[3 * pt], py = pts[3 * pt + 1], pz = pts[3 * pt + 2];
    const double lx = R[0] * px + R[1] * py + R[2] * pz;
    const double ly = R[3] * px + R[4] * py + R[5] * pz;
    const double lz = R[6] * px + R[7] * py + R[8] * pz;
    sp[0] = lx; sp[1] = ly; sp[2] = lz;
    sp[3] = sqrt(lx * lx + ly * ly + lz * lz);
    sp[4] = sqrt(lx * lx + ly * ly);
    bad = 0;
    // radial nodes: native panels, or the panel bisected until each piece is <= half its distance to p
    const double a2 = sp[3] * sp[3], rho = sp[4], tp = atan2(rho, lz);
    auto dist = [&](double lo, double hi) {
      const double tt = fmin(fmax(tp, lo), hi);
      return sqrt(fmax(a2 + 1.0 - 2.0 * (rho * sin(tt) + lz * cos(tt)), 0.0));
    };
    int n = 0;
    for (int i = 0; i < nd.npan && !bad; ++i) {
      const double lo = nd.edges[i], hi = nd.edges[i + 1];
      if (i == nd.npan - 1 || hi - lo <= 0.5 * dist(lo, hi)) {
        if (n + nd.k > kNearMaxNodes) { bad = 1; break; }
        for (int e = 0; e < nd.k; ++e) {
          nd_t[n] = nd.t[i * nd.k + e];
          nd_w[n] = nd.w[i * nd.k + e];
          nd_src[n] = i * nd.k + e;
          ++n;
        }
        continue;
      }
      double stl[48], sth[48];
      int ns = 0;
      stl[ns] = lo; sth[ns] = hi; ++ns;
      while (ns > 0 && !bad) {
        --ns;
        const double l = stl[ns], hh = sth[ns];
        if (hh - l <= 0.5 * dist(l, hh)) {
          if (n + nd.k > kNearMaxNodes) { bad = 1; break; }
          for (int e = 0; e < nd.k; ++e) {
            const double tt = 0.5 * (l + hh) + 0.5 * (hh - l) * nd.gl_x[e];
            nd_t[n] = tt;
            nd_w[n] = 0.5 * (hh - l) * nd.gl_w[e] * sin(tt);
            nd_src[n] = -(i + 1);
            ++n;
          }
        } else if (ns + 2 > 48) {
          bad = 1;
        } else {
          const double m = 0.5 * (l + hh);
          stl[ns] = m; sth[ns] = hh; ++ns;
          stl[ns] = l; sth[ns] = m; ++ns;
        }
      }
    }
    nnodes = n;
  }
  // profiles at the native nodes: A_m(t_r) = sum over the basis columns of order m (cos) of fhat_a sigma_a(t_r)
  const double* xj = x_all + (size_t)j * nd.K;
  for (int e = threadIdx.x; e < nd.n_r * C; e += kNearThreads) {
    const int r = e / C, comp = e - r * C;
    double v = 0.0;
    for (int a = nd.mc_off[comp]; a < nd.mc_off[comp + 1]; ++a) {
      const int col = nd.mc_col[a];
      v = fma(xj[col], nd.sigma[(size_t)col * nd.n_r + r], v);
    }
    prof[e] = v;
  }
  __syncthreads();
  if (bad) {
    if (threadIdx.x == 0) atomicExch(status, 1);
    return;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double lx = sp[0], ly = sp[1], lz = sp[2], pa = sp[3], rho = sp[4];
  double acc = 0.0;
  for (int r = warp; r < nnodes; r += kNearThreads / 32) {
    const double t = nd_t[r], wt = nd_w[r];
    const int src = nd_src[r];
    double val = 0.0;
    if (lane < C) {
      if (src >= 0) {
        val = prof[(size_t)src * C + lane];
      } else {                                                  // barycentric interpolation on the parent panel
        const int i = -src - 1;
        const double* tn = nd.t + i * nd.k;
        double num = 0.0, den = 0.0;
        int hit = -1;
        for (int e = 0; e < nd.k; ++e) {
          const double dt = t - tn[e];
          if (dt == 0.0) hit = e;
          const double f = nd.bary[e] / dt;
          num = fma(f, prof[(size_t)(i * nd.k + e) * C + lane], num);
          den += f;
        }
        val = hit >= 0 ? prof[(size_t)(i * nd.k + hit) * C + lane] : num / den;
      }
    }
    double A[kNearMaxM1], B[kNearMaxM1];
#pragma unroll
    for (int m = 0; m < kNearMaxM1; ++m) {
      A[m] = __shfl_sync(0xffffffffu, val, 2 * m);
      B[m] = __shfl_sync(0xffffffffu, val, 2 * m + 1);
    }
    const double st = sin(t), ct = cos(t);
    const double d2 = fmax(pa * pa + 1.0 - 2.0 * (rho * st + lz * ct), 1e-300);
    const double rs = rho * st;
    const double alpha = rs > 0.0 ? acosh(1.0 + d2 / (2.0 * rs)) : 1e30;
    int nth = 64;
    while (nth < kTrigN && nth * alpha < 40.0) nth *= 2;
    if (nth * alpha < 36.0 && lane == 0) atomicExch(status, 2);   // too close: the rule would not converge
    const int stride = kTrigN / nth;
    double ring = 0.0;
    for (int k = lane; k < nth; k += 32) {
      const double ca = nd.trig[2 * (k * stride)], sa = nd.trig[2 * (k * stride) + 1];
      const double sx = st * ca, sy = st * sa;
      const double g = green_off_near<KIND>(lx, ly, lz, pa, sx, sy, ct);
      // sigma(theta) = sum_m A_m cos(m theta) + B_m sin(m theta), cos / sin (m theta) by the two-term recurrences
      double cm = 1.0, sm = 0.0, cp = ca, spv = -sa;
      const double tc = 2.0 * ca;
      double sig = 0.0;
#pragma unroll
      for (int m = 0; m < kNearMaxM1; ++m) {
        if (m < M1) sig = fma(A[m], cm, fma(B[m], sm, sig));
        const double cn = fma(tc, cm, -cp), sn = fma(tc, sm, -spv);
        cp = cm; spv = sm; cm = cn; sm = sn;
      }
      ring = fma(g, sig, ring);
    }
    acc = fma(ring, wt * (6.283185307179586476925286766559 / nth), acc);
  }
  // minus the patch's compressed skeleton contribution, which nc_field's total over all patches holds (the records
  // are in global coordinates x 1/2, rho in slot 3)
  {
    const double gx = pts[3 * pt], gy = pts[3 * pt + 1], gz = pts[3 * pt + 2];
    for (int m = threadIdx.x; m < p0; m += kNearThreads) {
      const double* s = rec + ((size_t)j * p0 + m) * 4;
      acc -= s[3] * green_off_near<KIND>(gx, gy, gz, pa, 2.0 * s[0], 2.0 * s[1], 2.0 * s[2]);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) red[warp] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < kNearThreads / 32; ++w) s += red[w];
    corr[q] = s;
  }
}

// out[t] += sum of the corrections of point t's pairs (CSR, fixed order)
__global__ void k_near_apply(const int64_t* __restrict__ off, const double* __restrict__ corr, int64_t n,
                             double* __restrict__ out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  double v = out[t];
  for (int64_t q = off[t]; q < off[t + 1]; ++q) v += corr[q];
  out[t] = v;
}

size_t near_quad_smem(int n_r, int M1) {
  return (size_t)n_r * 2 * M1 * sizeof(double) + (size_t)kNearMaxNodes * (2 * sizeof(double) + sizeof(int));
}

void launch_near_count(const double* pts, int64_t n, const double* cen, int64_t N, double r, int64_t* cnt,
                       int64_t* list, const int64_t* off, cudaStream_t s) {
  if (n <= 0) return;
  k_near_count<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(pts, n, cen, N, r * r, cnt, list, off);
}

int launch_near_quad(int kind, const int64_t* pair_pt, const int64_t* pair_patch, int64_t npairs, const double* pts,
                     const double* frames, const double* x_all, const NearDev& nd, const double* rec, int p0,
                     double* corr, int* status, cudaStream_t s) {
  if (npairs <= 0) return 0;
  const size_t shm = near_quad_smem(nd.n_r, nd.M1);
  if (kind == NC_EXTERIOR) {
    cudaFuncSetAttribute(k_near_quad<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm);
    k_near_quad<1><<<(unsigned)npairs, kNearThreads, shm, s>>>(pair_pt, pair_patch, npairs, pts, frames, x_all, nd, rec,
                                                              p0, corr, status);
  } else {
    cudaFuncSetAttribute(k_near_quad<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm);
    k_near_quad<0><<<(unsigned)npairs, kNearThreads, shm, s>>>(pair_pt, pair_patch, npairs, pts, frames, x_all, nd, rec,
                                                              p0, corr, status);
  }
  return 0;
}

void launch_near_apply(const int64_t* off, const double* corr, int64_t n, double* out, cudaStream_t s) {
  if (n <= 0) return;
  k_near_apply<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(off, corr, n, out);
}

}  // namespace nc
