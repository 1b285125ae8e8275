// direct.cu -- the tiled direct multiple-scattering sum (a2 of SURVEY.md §8(a)):
//
//   u_{ik} = sum_{j != i} sum_{m=1..p} G(z_{ik}, s_{jm}) rho_{jm}        (eq:mssums with eq:outgoingcompressed)
//
// Design (B200, fp64-pipe bound): one thread per target node z_{ik}; a CTA holds 256 targets and walks
// a segment of source patches, staging whole source patches (p records of (x, y, z, rho), 32 B each,
// coalesced 16 B loads) in shared memory; every thread reads each record as a broadcast and does one
// rsqrt + one log + ~10 DFMA per pair.  Self-exclusion (j != i) is a per-thread patch skip, so tiles may
// straddle patches for any Kstar.  The source range is split into `nseg` segments (grid.y) so the grid
// has many waves on 148 SMs; the segments' partial fields are summed deterministically inside the
// step-5 GEMM's operand load (gemm.cu).
#include "green.cuh"
#include "nc_common.cuh"

namespace nc {

template <int KIND>
__global__ void __launch_bounds__(kPairThreads) k_pairs_direct(const double* __restrict__ tx,
                                                                const double* __restrict__ ty,
                                                                const double* __restrict__ tz, int64_t n_tgt,
                                                                int Kstar, int64_t tgt_patch0,
                                                                const double* __restrict__ src4, int p, int64_t N,
                                                                int nseg, int chp, double* __restrict__ upart) {
  extern __shared__ double4 sm[];
  const int64_t t = (int64_t)blockIdx.x * kPairThreads + threadIdx.x;
  const bool valid = t < n_tgt;
  const int64_t tt = valid ? t : n_tgt - 1;
  const double x = tx[tt], y = ty[tt], z = tz[tt];
  const int64_t my_patch = tgt_patch0 + tt / Kstar;
  const int seg = blockIdx.y;
  const int64_t j0 = (N * seg) / nseg, j1 = (N * (seg + 1)) / nseg;
  const double4* __restrict__ s4 = reinterpret_cast<const double4*>(src4);
  double acc = 0.0;
  for (int64_t jc = j0; jc < j1; jc += chp) {
    const int nch = (int)min((int64_t)chp, j1 - jc);
    const int nrec = nch * p;
    __syncthreads();
    for (int r = threadIdx.x; r < nrec; r += kPairThreads) sm[r] = s4[jc * p + r];
    __syncthreads();
    for (int q = 0; q < nch; ++q) {
      if (jc + q == my_patch) continue;  // j != i
      const double4* __restrict__ sp = sm + q * p;
#pragma unroll 4
      for (int m = 0; m < p; ++m) {
        const double4 s = sp[m];
        const double dx = x - s.x, dy = y - s.y, dz = z - s.z;
        const double d2 = fma(dz, dz, fma(dy, dy, dx * dx));
        acc = fma(s.w, green_from_d2<KIND>(d2), acc);
      }
    }
  }
  if (valid) upart[(int64_t)seg * n_tgt + t] = acc;
}

void launch_pairs_direct(int kind, const double* tx, const double* ty, const double* tz, int64_t n_tgt, int Kstar,
                         int64_t tgt_patch0, const double* src4, int p, int64_t N, int nseg, double* upart,
                         cudaStream_t s) {
  if (n_tgt <= 0) return;
  int chp = max(1, 1024 / p);            // source patches per shared-memory stage (<= 32 KB)
  size_t smem = (size_t)chp * p * sizeof(double4);
  dim3 grid((unsigned)((n_tgt + kPairThreads - 1) / kPairThreads), (unsigned)nseg);
  if (kind == NC_EXTERIOR)
    k_pairs_direct<1><<<grid, kPairThreads, smem, s>>>(tx, ty, tz, n_tgt, Kstar, tgt_patch0, src4, p, N, nseg, chp,
                                                       upart);
  else
    k_pairs_direct<0><<<grid, kPairThreads, smem, s>>>(tx, ty, tz, n_tgt, Kstar, tgt_patch0, src4, p, N, nseg, chp,
                                                       upart);
}

}  // namespace nc
