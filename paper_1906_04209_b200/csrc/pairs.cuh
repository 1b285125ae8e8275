// pairs.cuh -- the shared inner loop of every Green's-function sum on the hot path:
//
//   acc_u += sum over source patches j in a list (j != excl_u) of sum_m G(target_u, s_jm) rho_jm
//
// used by the direct sum (a2), the hierarchical interaction-list / neighbour evaluations on incoming grids
// (a3, a4) and the near-list evaluations at Zernike nodes (a4, reading R12).  Whole source patches
// (p records of (x, y, z, rho), 32 B each, coordinates pre-scaled by 1/2) are staged in shared memory with
// coalesced 16 B loads; each thread owns TPT targets (independent FP64 chains sharing every broadcast load).
#pragma once

#include "green.cuh"
#include "nc_common.cuh"

namespace nc {

constexpr int kStagePatchesMax = 64;     // source patches per shared-memory stage (bounded by 512 records)

__host__ __device__ inline int stage_patches(int p) {
  int c = 512 / p;
  if (c < 1) c = 1;
  if (c > kStagePatchesMax) c = kStagePatchesMax;
  return c;
}

// patch_at(k) -> patch index of the k-th list entry.  All threads of the CTA must call (barriers inside).
// UNROLL: source records in flight per target (independent FP64 chains = TPT x UNROLL); Tab: double2 (c_j, -log c_j)
// or double (-log c_j, c_j recomputed: green.cuh log8_c).
template <int KIND, int TPT, int UNROLL = 2, class Tab = double2, class PatchAt>
__device__ __forceinline__ void accumulate_list(const double (&x)[TPT], const double (&y)[TPT], const double (&z)[TPT],
                                                const int64_t (&excl)[TPT], double (&acc)[TPT], int64_t nlist,
                                                PatchAt patch_at, const double4* __restrict__ s4, int p,
                                                double4* __restrict__ sm, int64_t* __restrict__ sm_pid, int chp,
                                                const Tab* __restrict__ logtab, bool active) {
  for (int64_t c0 = 0; c0 < nlist; c0 += chp) {
    const int nch = (int)min((int64_t)chp, nlist - c0);
    __syncthreads();
    if (threadIdx.x < nch) sm_pid[threadIdx.x] = patch_at(c0 + threadIdx.x);
    __syncthreads();
    for (int r = threadIdx.x; r < nch * p; r += blockDim.x) {
      const int q = r / p;
      sm[r] = s4[sm_pid[q] * p + (r - q * p)];
    }
    __syncthreads();
    if (!active) continue;
    for (int q = 0; q < nch; ++q) {
      const int64_t j = sm_pid[q];
      const double4* __restrict__ sp = sm + q * p;
      bool all = true, none = true;
#pragma unroll
      for (int u = 0; u < TPT; ++u) {
        all = all && (excl[u] != j);
        none = none && (excl[u] == j);
      }
      if (none) continue;
      if (all) {
#pragma unroll UNROLL
        for (int m = 0; m < p; ++m) {
          const double4 s = sp[m];
#pragma unroll
          for (int u = 0; u < TPT; ++u) {
            const double dx = x[u] - s.x, dy = y[u] - s.y, dz = z[u] - s.z;
            const double qd = fma(dz, dz, fma(dy, dy, dx * dx));   // |z - s|^2 / 4 (scaled coordinates)
            acc[u] = fma(s.w, green_q<KIND>(qd, logtab), acc[u]);
          }
        }
      } else {
#pragma unroll
        for (int u = 0; u < TPT; ++u) {
          if (excl[u] == j) continue;
          for (int m = 0; m < p; ++m) {
            const double4 s = sp[m];
            const double dx = x[u] - s.x, dy = y[u] - s.y, dz = z[u] - s.z;
            const double qd = fma(dz, dz, fma(dy, dy, dx * dx));
            acc[u] = fma(s.w, green_q<KIND>(qd, logtab), acc[u]);
          }
        }
      }
    }
  }
}

// Incoming-grid variant (no self exclusion: grid sources never include the target's own patch).  FAR = false: the
// exact kernel of accumulate_list.  FAR = true (far-field evaluation, hierarchical mode only): the squared distance
// from the dot product, q = |X|^2 + 1/4 - 2 X.S with the target pre-scaled T = -2X (3 DFMA instead of 6 FP64 ops;
// absolute error ~3e-16, i.e. relative ~1e-10 at the closest grid pairs q ~ eps^2/4, far below the hierarchical
// tolerance) and the one-Newton rsqrt.  x/y/z hold T when FAR, and cq[u] = |X_u|^2 + 1/4.
template <int KIND, int TPT, int UNROLL, bool FAR, class Tab, class PatchAt>
__device__ __forceinline__ void accumulate_grid(const double (&x)[TPT], const double (&y)[TPT], const double (&z)[TPT],
                                                const double (&cq)[TPT], double (&acc)[TPT], int64_t nlist,
                                                PatchAt patch_at, const double4* __restrict__ s4, int p,
                                                double4* __restrict__ sm, int64_t* __restrict__ sm_pid, int chp,
                                                const Tab* __restrict__ logtab, bool active) {
  for (int64_t c0 = 0; c0 < nlist; c0 += chp) {
    const int nch = (int)min((int64_t)chp, nlist - c0);
    __syncthreads();
    if (threadIdx.x < nch) sm_pid[threadIdx.x] = patch_at(c0 + threadIdx.x);
    __syncthreads();
    for (int r = threadIdx.x; r < nch * p; r += blockDim.x) {
      const int q = r / p;
      sm[r] = s4[sm_pid[q] * p + (r - q * p)];
    }
    __syncthreads();
    if (!active) continue;
    const int nrec = nch * p;
#pragma unroll UNROLL
    for (int m = 0; m < nrec; ++m) {
      const double4 s = sm[m];
#pragma unroll
      for (int u = 0; u < TPT; ++u) {
        if (FAR) {
          const double qd = fma(x[u], s.x, fma(y[u], s.y, fma(z[u], s.z, cq[u])));
          acc[u] = fma(s.w, green_q_far<KIND>(qd, logtab), acc[u]);
        } else {
          const double dx = x[u] - s.x, dy = y[u] - s.y, dz = z[u] - s.z;
          const double qd = fma(dz, dz, fma(dy, dy, dx * dx));
          acc[u] = fma(s.w, green_q<KIND>(qd, logtab), acc[u]);
        }
      }
    }
  }
}

// Variant without shared-memory staging: every warp reads the source records straight from global memory with
// warp-uniform addresses (one L1 broadcast per record), so warps never wait on CTA barriers.
template <int KIND, int TPT, class PatchAt>
__device__ __forceinline__ void accumulate_list_ldg(const double (&x)[TPT], const double (&y)[TPT],
                                                    const double (&z)[TPT], const int64_t (&excl)[TPT],
                                                    double (&acc)[TPT], int64_t nlist, PatchAt patch_at,
                                                    const double4* __restrict__ s4, int p,
                                                    const double2* __restrict__ logtab) {
  const double2* __restrict__ s2 = reinterpret_cast<const double2*>(s4);
  for (int64_t k = 0; k < nlist; ++k) {
    const int64_t j = patch_at(k);
    bool all = true, none = true;
#pragma unroll
    for (int u = 0; u < TPT; ++u) {
      all = all && (excl[u] != j);
      none = none && (excl[u] == j);
    }
    if (none) continue;
    const double2* __restrict__ sp = s2 + 2 * j * p;
    if (all) {
#pragma unroll 2
      for (int m = 0; m < p; ++m) {
        const double2 a = __ldg(sp + 2 * m), b = __ldg(sp + 2 * m + 1);
#pragma unroll
        for (int u = 0; u < TPT; ++u) {
          const double dx = x[u] - a.x, dy = y[u] - a.y, dz = z[u] - b.x;
          const double qd = fma(dz, dz, fma(dy, dy, dx * dx));
          acc[u] = fma(b.y, green_q<KIND>(qd, logtab), acc[u]);
        }
      }
    } else {
#pragma unroll
      for (int u = 0; u < TPT; ++u) {
        if (excl[u] == j) continue;
        for (int m = 0; m < p; ++m) {
          const double2 a = __ldg(sp + 2 * m), b = __ldg(sp + 2 * m + 1);
          const double dx = x[u] - a.x, dy = y[u] - a.y, dz = z[u] - b.x;
          const double qd = fma(dz, dz, fma(dy, dy, dx * dx));
          acc[u] = fma(b.y, green_q<KIND>(qd, logtab), acc[u]);
        }
      }
    }
  }
}

}  // namespace nc
