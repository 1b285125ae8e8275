// direct.cu -- the tiled direct multiple-scattering sum (a2 of SURVEY.md §8(a)):
//
//   u_{ik} = sum_{j != i} sum_{m=1..p} G(z_{ik}, s_{jm}) rho_{jm}        (eq:mssums with eq:outgoingcompressed)
//
// Design (B200, fp64-pipe bound): TPT (1 or 2) target nodes z_{ik} per thread; a CTA holds 256*TPT targets and walks
// a segment of source patches, staging whole source patches (p records of (x, y, z, rho), 32 B each,
// coalesced 16 B loads) in shared memory; every thread reads each record as a broadcast and does one
// rsqrt + one log + ~10 DFMA per pair.  Self-exclusion (j != i) is a per-thread patch skip, so tiles may
// straddle patches for any Kstar.  The source range is split into `nseg` segments (grid.y) so the grid
// has many waves on 148 SMs; the segments' partial fields are summed deterministically inside the
// step-5 GEMM's operand load (gemm.cu).
#include "green.cuh"
#include "nc_common.cuh"

namespace nc {

template <int KIND, int TPT>
__global__ void __launch_bounds__(kPairThreads) k_pairs_direct(const double* __restrict__ tx,
                                                                const double* __restrict__ ty,
                                                                const double* __restrict__ tz, int64_t n_tgt,
                                                                int Kstar, int64_t tgt_patch0,
                                                                const double* __restrict__ src4, int p, int64_t N,
                                                                int nseg, int chp, double* __restrict__ upart) {
  extern __shared__ double4 sm[];
  __shared__ double2 logtab[kLogTableSize];
  init_log_table(logtab);
  // TPT targets per thread (t0 + u * kPairThreads): independent accumulation chains sharing each source load
  double x[TPT], y[TPT], z[TPT], acc[TPT];
  int64_t patch[TPT];
  const int64_t t0 = (int64_t)blockIdx.x * kPairThreads * TPT + threadIdx.x;
#pragma unroll
  for (int u = 0; u < TPT; ++u) {
    const int64_t t = min(t0 + u * kPairThreads, n_tgt - 1);
    x[u] = tx[t]; y[u] = ty[t]; z[u] = tz[t];
    patch[u] = tgt_patch0 + t / Kstar;
    acc[u] = 0.0;
  }
  const int seg = blockIdx.y;
  const int64_t j0 = (N * seg) / nseg, j1 = (N * (seg + 1)) / nseg;
  const double4* __restrict__ s4 = reinterpret_cast<const double4*>(src4);
  for (int64_t jc = j0; jc < j1; jc += chp) {
    const int nch = (int)min((int64_t)chp, j1 - jc);
    const int nrec = nch * p;
    __syncthreads();
    for (int r = threadIdx.x; r < nrec; r += kPairThreads) sm[r] = s4[jc * p + r];
    __syncthreads();
    for (int qq = 0; qq < nch; ++qq) {
      const int64_t j = jc + qq;
      const double4* __restrict__ sp = sm + qq * p;
      bool all = true, none = true;
#pragma unroll
      for (int u = 0; u < TPT; ++u) {
        all = all && (patch[u] != j);
        none = none && (patch[u] == j);
      }
      if (none) continue;                               // j != i for every target of this thread
      if (all) {
#pragma unroll 2
        for (int m = 0; m < p; ++m) {
          const double4 s = sp[m];
#pragma unroll
          for (int u = 0; u < TPT; ++u) {
            const double dx = x[u] - s.x, dy = y[u] - s.y, dz = z[u] - s.z;
            const double q = fma(dz, dz, fma(dy, dy, dx * dx));   // |z - s|^2 / 4 (scaled coordinates)
            acc[u] = fma(s.w, green_q<KIND>(q, logtab), acc[u]);
          }
        }
      } else {                                          // some (not all) targets are on patch j: skip those
#pragma unroll
        for (int u = 0; u < TPT; ++u) {
          if (patch[u] == j) continue;
          for (int m = 0; m < p; ++m) {
            const double4 s = sp[m];
            const double dx = x[u] - s.x, dy = y[u] - s.y, dz = z[u] - s.z;
            const double q = fma(dz, dz, fma(dy, dy, dx * dx));
            acc[u] = fma(s.w, green_q<KIND>(q, logtab), acc[u]);
          }
        }
      }
    }
  }
#pragma unroll
  for (int u = 0; u < TPT; ++u) {
    const int64_t t = t0 + u * kPairThreads;
    if (t < n_tgt) upart[(int64_t)seg * n_tgt + t] = acc[u];
  }
}

static int chp_for(int p) { return max(1, 512 / p); }   // source patches per smem stage (<= 16 KB unless p > 512)

int pairs_direct_blocks_per_sm(int p, int tpt) {
  int nb = 0;
  size_t smem = (size_t)chp_for(p) * p * sizeof(double4);
  if (tpt == 2)
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_pairs_direct<1, 2>, kPairThreads, smem);
  else
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_pairs_direct<1, 1>, kPairThreads, smem);
  return max(nb, 1);
}

void launch_pairs_direct(int kind, int tpt, const double* tx, const double* ty, const double* tz, int64_t n_tgt,
                         int Kstar, int64_t tgt_patch0, const double* src4, int p, int64_t N, int nseg, double* upart,
                         cudaStream_t s) {
  if (n_tgt <= 0) return;
  const int chp = chp_for(p);
  const size_t smem = (size_t)chp * p * sizeof(double4);
  const int64_t per_block = (int64_t)kPairThreads * tpt;
  dim3 grid((unsigned)((n_tgt + per_block - 1) / per_block), (unsigned)nseg);
#define NC_LAUNCH(KD, TP) \
  k_pairs_direct<KD, TP><<<grid, kPairThreads, smem, s>>>(tx, ty, tz, n_tgt, Kstar, tgt_patch0, src4, p, N, nseg, chp, upart)
  if (kind == NC_EXTERIOR) {
    if (tpt == 2) NC_LAUNCH(1, 2); else NC_LAUNCH(1, 1);
  } else {
    if (tpt == 2) NC_LAUNCH(0, 2); else NC_LAUNCH(0, 1);
  }
#undef NC_LAUNCH
}

}  // namespace nc
