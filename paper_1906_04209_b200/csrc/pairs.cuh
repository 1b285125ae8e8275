// pairs.cuh -- the shared inner loop of every Green's-function sum on the hot path:
//
//   acc_u += sum over source patches j in a list (j != excl_u) of sum_m G(target_u, s_jm) rho_jm
//
// used by the direct sum (a2), the hierarchical interaction-list / neighbour evaluations on incoming grids
// (a3, a4) and the near-list evaluations at Zernike nodes (a4, reading R12).  Whole source patches
// (p records: the static coordinates (x, y, z, -) of 32 B, pre-scaled by 1/2, and rho = T fhat from the compact
// per-rung array K1 writes) are staged in shared memory as (x, y, z, rho); each thread owns TPT targets (independent
// FP64 chains sharing every broadcast load).
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
// (c_j, -log c_j).
// green(q) evaluates G from q = |z - s|^2 / 4 (green_q with the mantissa table, or green_exact_r)
// GreenFar: a functor (qh) -> G for well-separated pairs (green_exact_far), used for a whole staged patch when every
// target of the warp is at least sqrt(4 far_q) (unscaled) from its first record; far_q <= 0 disables it
template <int KIND, int TPT, int UNROLL = 2, class GreenQ, class PatchAt, class GreenFar = GreenQ>
__device__ __forceinline__ void accumulate_list(const double (&x)[TPT], const double (&y)[TPT], const double (&z)[TPT],
                                                const int64_t (&excl)[TPT], double (&acc)[TPT], int64_t nlist,
                                                PatchAt patch_at, const double4* __restrict__ s4,
                                                const double* __restrict__ rho, int p,
                                                double4* __restrict__ sm, int64_t* __restrict__ sm_pid, int chp,
                                                GreenQ green, bool active, GreenFar greenfar, double far_q) {
  double cq[TPT];   // (|X|^2 + 1/4) / 2: qh = cq - X.S for the far path
#pragma unroll
  for (int u = 0; u < TPT; ++u) cq[u] = 0.5 * fma(x[u], x[u], fma(y[u], y[u], fma(z[u], z[u], 0.25)));
  for (int64_t c0 = 0; c0 < nlist; c0 += chp) {
    const int nch = (int)min((int64_t)chp, nlist - c0);
    __syncthreads();
    if (threadIdx.x < nch) sm_pid[threadIdx.x] = patch_at(c0 + threadIdx.x);
    __syncthreads();
    for (int r = threadIdx.x; r < nch * p; r += blockDim.x) {
      const int q = r / p;
      const int64_t g = sm_pid[q] * p + (r - q * p);
      double4 v = s4[g];
      v.w = rho[g];
      sm[r] = v;
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
        bool far = false;
        if (far_q > 0.0) {   // warp-uniform among the lanes here: every target far from the patch's first node
          const double4 s0 = sp[0];
          double mq = 1e300;
#pragma unroll
          for (int u = 0; u < TPT; ++u) {
            const double dx = x[u] - s0.x, dy = y[u] - s0.y, dz = z[u] - s0.z;
            mq = fmin(mq, fma(dz, dz, fma(dy, dy, dx * dx)));
          }
          far = __all_sync(__activemask(), mq >= far_q);
        }
        if (far) {
#pragma unroll UNROLL
          for (int m = 0; m < p; ++m) {
            const double4 s = sp[m];
#pragma unroll
            for (int u = 0; u < TPT; ++u) {
              const double qh = fma(-x[u], s.x, fma(-y[u], s.y, fma(-z[u], s.z, cq[u])));
              acc[u] = fma(s.w, greenfar(qh), acc[u]);
            }
          }
          continue;
        }
#pragma unroll UNROLL
        for (int m = 0; m < p; ++m) {
          const double4 s = sp[m];
#pragma unroll
          for (int u = 0; u < TPT; ++u) {
            const double dx = x[u] - s.x, dy = y[u] - s.y, dz = z[u] - s.z;
            const double qd = fma(dz, dz, fma(dy, dy, dx * dx));   // |z - s|^2 / 4 (scaled coordinates)
            acc[u] = fma(s.w, green(qd), acc[u]);
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
            acc[u] = fma(s.w, green(qd), acc[u]);
          }
        }
      }
    }
  }
}

// Incoming-grid variant (no self exclusion: grid sources never include the target's own patch).  FAR = false: the
// exact kernel of accumulate_list.  FAR = true (far-field evaluation, hierarchical mode only): half the squared
// distance from the dot product, qh = (|X|^2 + 1/4)/2 - X.S with the target pre-negated (3 DFMA instead of 6 FP64
// ops; absolute error ~2e-16, i.e. relative ~1e-10 at the closest grid pairs qh ~ eps^2/8, far below the
// hierarchical tolerance) and a far form below.  x/y/z hold -X when FAR, and cq[u] = (|X_u|^2 + 1/4)/2.
// FAR (the grid kernel's far forms): 5 = green_far_r (R25: FB = 7 cubic, clamped index), 7 = green_far_n FB = 7
// cubic (R32: unclamped, scaled-index table load), 8 = green_far_n FB = 9 quadratic (R32), 9 / 10 = green_far_hl
// (R35: the forms of 8 / 7 with high-word SFU seeds and a one-instruction table address)
__host__ __device__ constexpr int far_table_bits(int far) { return far == 8 || far == 9 ? 9 : 7; }
// 0: 16-byte (c, L) entries; 1: 8-byte L for c = rcp.approx(midpoint); 2: 8-byte L for c = rcp_seed_hl(midpoint word)
__host__ __device__ constexpr int far_table_rcp(int far) { return far >= 9 ? 2 : far >= 5 ? 1 : 0; }
inline void far_poly(int far, double* a2, double* a3) {   // the polynomial constants the table carries (host)
  if (far == 8 || far == 9) {   // quadratic r (c1 + c2 r): c2 in the a2 slot, c1 in the a3 slot
    *a2 = FarQuad<9>::c2;
    *a3 = FarQuad<9>::c1;
    return;
  }
  *a2 = FarPoly<7, 3>::a2;
  *a3 = 0.0;
}
template <int KIND, int FAR>
__device__ __forceinline__ double green_far_any(double qh, const double2* __restrict__ logtab, unsigned tbase,
                                                int lim, double a2, double a3, int kmid,
                                                const double* __restrict__ ftd = nullptr) {
  static_assert(FAR == 5 || FAR == 7 || FAR == 8 || FAR == 9 || FAR == 10, "far form");
  if constexpr (FAR == 5) return green_far_r<KIND, 7, 3>(qh, tbase, lim, a2, a3, kmid);
  if constexpr (FAR == 7) return green_far_n<KIND, 7, 3>(qh, ftd, a2, a3, kmid);
  if constexpr (FAR == 8) return green_far_n<KIND, 9, 2>(qh, ftd, a2, a3, kmid);
  // tbase: byte address of table index 0; the midpoint word carries + 4 (green_far_hl)
  if constexpr (FAR == 9) return green_far_hl<KIND, 9, 2>(qh, tbase - 4u, a2, a3, kmid);
  if constexpr (FAR == 10) return green_far_hl<KIND, 7, 3>(qh, tbase - 4u, a2, a3, kmid);
}

// the records [0, nrec) of a staged chunk against the thread's targets (incoming-grid sums, no self exclusion)
template <int KIND, int TPT, int UNROLL, int FAR, class Tab>
__device__ __forceinline__ void accumulate_span(const double (&x)[TPT], const double (&y)[TPT], const double (&z)[TPT],
                                                const double (&cq)[TPT], double (&acc)[TPT],
                                                const double4* __restrict__ sm, int nrec, bool single,
                                                const Tab* __restrict__ logtab, unsigned ftb, int flim, double fa2,
                                                double fa3, int fmid = 0, const double* __restrict__ ftd = nullptr) {
  if (single) {   // warp-uniform: a tail warp with <= 32 points evaluates one target per lane
#pragma unroll UNROLL
    for (int m = 0; m < nrec; ++m) {
      const double4 s = sm[m];
      if constexpr (FAR != 0) {
        const double qh = fma(x[0], s.x, fma(y[0], s.y, fma(z[0], s.z, cq[0])));
        acc[0] = fma(s.w, green_far_any<KIND, FAR>(qh, logtab, ftb, flim, fa2, fa3, fmid, ftd), acc[0]);
      } else {
        const double dx = x[0] - s.x, dy = y[0] - s.y, dz = z[0] - s.z;
        const double qd = fma(dz, dz, fma(dy, dy, dx * dx));
        acc[0] = fma(s.w, green_q<KIND>(qd, logtab), acc[0]);
      }
    }
    return;
  }
#pragma unroll UNROLL
  for (int m = 0; m < nrec; ++m) {
    const double4 s = sm[m];
#pragma unroll
    for (int u = 0; u < TPT; ++u) {
      if constexpr (FAR != 0) {
        const double qh = fma(x[u], s.x, fma(y[u], s.y, fma(z[u], s.z, cq[u])));
        acc[u] = fma(s.w, green_far_any<KIND, FAR>(qh, logtab, ftb, flim, fa2, fa3, fmid, ftd), acc[u]);
      } else {
        const double dx = x[u] - s.x, dy = y[u] - s.y, dz = z[u] - s.z;
        const double qd = fma(dz, dz, fma(dy, dy, dx * dx));
        acc[u] = fma(s.w, green_q<KIND>(qd, logtab), acc[u]);
      }
    }
  }
}

// the half-warp split of k_pairs_grid_w (TPT = 4, R35): records sm[0], sm[2], ... (sm already offset by the
// half-warp's parity), npair of them, against the lane's 4 targets
template <int KIND, int TPT, int UNROLL, int FAR>
__device__ __forceinline__ void accumulate_span_split(const double (&x)[TPT], const double (&y)[TPT],
                                                      const double (&z)[TPT], const double (&cq)[TPT],
                                                      double (&acc)[TPT], const double4* __restrict__ sm, int npair,
                                                      unsigned ftb, double fa2, double fa3, int fmid,
                                                      const double* __restrict__ ftd) {
#pragma unroll UNROLL
  for (int m = 0; m < npair; ++m) {
    const double4 s = sm[2 * m];
#pragma unroll
    for (int u = 0; u < TPT; ++u) {
      const double qh = fma(x[u], s.x, fma(y[u], s.y, fma(z[u], s.z, cq[u])));
      acc[u] = fma(s.w, green_far_any<KIND, FAR>(qh, nullptr, ftb, 0, fa2, fa3, fmid, ftd), acc[u]);
    }
  }
}

template <int KIND, int TPT, int UNROLL, int FAR, class Tab, class PatchAt>
__device__ __forceinline__ void accumulate_grid(const double (&x)[TPT], const double (&y)[TPT], const double (&z)[TPT],
                                                const double (&cq)[TPT], double (&acc)[TPT], int64_t nlist,
                                                PatchAt patch_at, const double4* __restrict__ s4,
                                                const double* __restrict__ rho, int p,
                                                double4* __restrict__ sm, int64_t* __restrict__ sm_pid, int chp,
                                                const Tab* __restrict__ logtab, bool active,
                                                bool single = false, unsigned ftb = 0, int flim = 0,
                                                double fa2 = 0.0, double fa3 = 0.0, int fmid = 0) {
  for (int64_t c0 = 0; c0 < nlist; c0 += chp) {
    const int nch = (int)min((int64_t)chp, nlist - c0);
    __syncthreads();
    if (threadIdx.x < nch) sm_pid[threadIdx.x] = patch_at(c0 + threadIdx.x);
    __syncthreads();
    for (int r = threadIdx.x; r < nch * p; r += blockDim.x) {
      const int q = r / p;
      const int64_t g = sm_pid[q] * p + (r - q * p);
      double4 v = s4[g];
      v.w = rho[g];
      sm[r] = v;
    }
    __syncthreads();
    if (!active) continue;
    accumulate_span<KIND, TPT, UNROLL, FAR>(x, y, z, cq, acc, sm, nch * p, single, logtab, ftb, flim, fa2, fa3, fmid);
  }
}

// cp.async (global -> shared, 16-byte pieces, no registers in flight): the warp-level grid kernel's double buffer
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

// Variant without shared-memory staging: every warp reads the source records straight from global memory with
// warp-uniform addresses (one L1 broadcast per record), so warps never wait on CTA barriers.
template <int KIND, int TPT, class PatchAt>
__device__ __forceinline__ void accumulate_list_ldg(const double (&x)[TPT], const double (&y)[TPT],
                                                    const double (&z)[TPT], const int64_t (&excl)[TPT],
                                                    double (&acc)[TPT], int64_t nlist, PatchAt patch_at,
                                                    const double4* __restrict__ s4, const double* __restrict__ rho,
                                                    int p, const double2* __restrict__ logtab) {
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
    const double* __restrict__ rp = rho + j * p;
    if (all) {
#pragma unroll 2
      for (int m = 0; m < p; ++m) {
        const double2 a = __ldg(sp + 2 * m), b = __ldg(sp + 2 * m + 1);
        const double w = __ldg(rp + m);
#pragma unroll
        for (int u = 0; u < TPT; ++u) {
          const double dx = x[u] - a.x, dy = y[u] - a.y, dz = z[u] - b.x;
          const double qd = fma(dz, dz, fma(dy, dy, dx * dx));
          acc[u] = fma(w, green_q<KIND>(qd, logtab), acc[u]);
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
          acc[u] = fma(__ldg(rp + m), green_q<KIND>(qd, logtab), acc[u]);
        }
      }
    }
  }
}

}  // namespace nc
