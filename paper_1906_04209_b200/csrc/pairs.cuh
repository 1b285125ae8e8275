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
// (c_j, -log c_j).
// green(q) evaluates G from q = |z - s|^2 / 4 (green_q with the mantissa table, or green_exact_r)
// GreenFar: a functor (qh) -> G for well-separated pairs (green_exact_far), used for a whole staged patch when every
// target of the warp is at least sqrt(4 far_q) (unscaled) from its first record; far_q <= 0 disables it
template <int KIND, int TPT, int UNROLL = 2, class GreenQ, class PatchAt, class GreenFar = GreenQ>
__device__ __forceinline__ void accumulate_list(const double (&x)[TPT], const double (&y)[TPT], const double (&z)[TPT],
                                                const int64_t (&excl)[TPT], double (&acc)[TPT], int64_t nlist,
                                                PatchAt patch_at, const double4* __restrict__ s4, int p,
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
// hierarchical tolerance) and green_far_h.  x/y/z hold -X when FAR, and cq[u] = (|X_u|^2 + 1/4)/2.
// FAR >= 2: the exponent-indexed far table.  green_far_t (16-byte (c, L) entries): 2 = 7 bits cubic, 3 = 7 bits
// quartic, 4 = 8 bits cubic; green_far_r (8-byte L entries, c from the SFU): 5 = 7 bits cubic, 6 = 6 bits quartic
__host__ __device__ constexpr int far_table_bits(int far) { return far == 4 ? 8 : far == 6 ? 6 : 7; }
__host__ __device__ constexpr bool far_table_rcp(int far) { return far >= 5; }
inline void far_poly(int far, double* a2, double* a3) {   // the polynomial constants the table carries (host)
  *a2 = far == 3 ? FarPoly<7, 4>::a2 : far == 4 ? FarPoly<8, 3>::a2 : far == 6 ? FarPoly<6, 4>::a2 : FarPoly<7, 3>::a2;
  *a3 = far == 3 ? FarPoly<7, 4>::a3 : far == 6 ? FarPoly<6, 4>::a3 : 0.0;
}
template <int KIND, int FAR>
__device__ __forceinline__ double green_far_any(double qh, const double2* __restrict__ logtab, unsigned tbase,
                                                int lim, double a2, double a3, int kmid) {
  if (FAR == 1) return green_far_h<KIND>(qh, logtab);
  if (FAR == 2) return green_far_t<KIND, 7, 3>(qh, tbase, lim, a2, a3);
  if (FAR == 3) return green_far_t<KIND, 7, 4>(qh, tbase, lim, a2, a3);
  if (FAR == 4) return green_far_t<KIND, 8, 3>(qh, tbase, lim, a2, a3);
  if (FAR == 5) return green_far_r<KIND, 7, 3>(qh, tbase, lim, a2, a3, kmid);
  return green_far_r<KIND, 6, 4>(qh, tbase, lim, a2, a3, kmid);
}

// the records [0, nrec) of a staged chunk against the thread's targets (incoming-grid sums, no self exclusion)
template <int KIND, int TPT, int UNROLL, int FAR, class Tab>
__device__ __forceinline__ void accumulate_span(const double (&x)[TPT], const double (&y)[TPT], const double (&z)[TPT],
                                                const double (&cq)[TPT], double (&acc)[TPT],
                                                const double4* __restrict__ sm, int nrec, bool single,
                                                const Tab* __restrict__ logtab, unsigned ftb, int flim, double fa2,
                                                double fa3, int fmid = 0) {
  if (single) {   // warp-uniform: a tail warp with <= 32 points evaluates one target per lane
#pragma unroll UNROLL
    for (int m = 0; m < nrec; ++m) {
      const double4 s = sm[m];
      if (FAR) {
        const double qh = fma(x[0], s.x, fma(y[0], s.y, fma(z[0], s.z, cq[0])));
        acc[0] = fma(s.w, green_far_any<KIND, FAR>(qh, logtab, ftb, flim, fa2, fa3, fmid), acc[0]);
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
      if (FAR) {
        const double qh = fma(x[u], s.x, fma(y[u], s.y, fma(z[u], s.z, cq[u])));
        acc[u] = fma(s.w, green_far_any<KIND, FAR>(qh, logtab, ftb, flim, fa2, fa3, fmid), acc[u]);
      } else {
        const double dx = x[u] - s.x, dy = y[u] - s.y, dz = z[u] - s.z;
        const double qd = fma(dz, dz, fma(dy, dy, dx * dx));
        acc[u] = fma(s.w, green_q<KIND>(qd, logtab), acc[u]);
      }
    }
  }
}

template <int KIND, int TPT, int UNROLL, int FAR, class Tab, class PatchAt>
__device__ __forceinline__ void accumulate_grid(const double (&x)[TPT], const double (&y)[TPT], const double (&z)[TPT],
                                                const double (&cq)[TPT], double (&acc)[TPT], int64_t nlist,
                                                PatchAt patch_at, const double4* __restrict__ s4, int p,
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
      sm[r] = s4[sm_pid[q] * p + (r - q * p)];
    }
    __syncthreads();
    if (!active) continue;
    accumulate_span<KIND, TPT, UNROLL, FAR>(x, y, z, cq, acc, sm, nch * p, single, logtab, ftb, flim, fa2, fa3, fmid);
  }
}

// Asynchronous double-buffered variant: the unit's source list (<= 32 patches) is staged once; chunk c + 1 is copied
// global -> shared with cp.async (16-byte pieces, no registers in flight) while chunk c is evaluated, so the warps
// wait at the chunk barrier only for the slowest warp, not for the copy.  bufs: 2 x brec records.
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <int KIND, int TPT, int UNROLL, int FAR, class Tab>
__device__ __forceinline__ void accumulate_grid_async(const double (&x)[TPT], const double (&y)[TPT],
                                                      const double (&z)[TPT], const double (&cq)[TPT],
                                                      double (&acc)[TPT], int nsrc, const int32_t* __restrict__ lst,
                                                      const double4* __restrict__ s4, int p,
                                                      double4* __restrict__ bufs, int brec, int32_t* __restrict__ slst,
                                                      const Tab* __restrict__ logtab, bool active, bool single,
                                                      unsigned ftb, int flim, double fa2, double fa3, int fmid) {
  __syncthreads();   // the previous unit is done with slst and the buffers
  if ((int)threadIdx.x < nsrc) slst[threadIdx.x] = lst[threadIdx.x];
  __syncthreads();
  const int chp = max(1, brec / p);
  const int nch = (nsrc + chp - 1) / chp;
  auto issue = [&](int c) {
    const int k0 = c * chp, k1 = min(nsrc, k0 + chp);
    double2* dst = reinterpret_cast<double2*>(bufs + (size_t)(c & 1) * brec);
    const int n16 = (k1 - k0) * p * 2;
    for (int t = threadIdx.x; t < n16; t += blockDim.x) {
      const int rr = t >> 1, q = rr / p, m = rr - q * p;
      cp_async16(dst + t, reinterpret_cast<const double2*>(s4 + (size_t)slst[k0 + q] * p + m) + (t & 1));
    }
    cp_async_commit();
  };
  issue(0);
  for (int c = 0; c < nch; ++c) {
    if (c + 1 < nch) {
      issue(c + 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();   // chunk c is in shared memory for every thread
    if (active)
      accumulate_span<KIND, TPT, UNROLL, FAR>(x, y, z, cq, acc, bufs + (size_t)(c & 1) * brec,
                                              (min(nsrc, (c + 1) * chp) - c * chp) * p, single, logtab, ftb, flim,
                                              fa2, fa3, fmid);
    __syncthreads();   // every thread is done with buffer c & 1 before chunk c + 2 overwrites it
  }
}

// ------------------------------------------------------------------------------------------------
// Bulk-copy (TMA) pipeline for the incoming-grid sums: one elected thread streams whole source patches (p contiguous
// 32-byte records each) into two shared-memory buffers with cp.async.bulk, completion tracked by a `full` mbarrier per
// buffer (transaction bytes); each consumer warp releases a buffer by arriving on its `empty` mbarrier.  No CTA-wide
// barrier in the loop: the copy of chunk c+1 overlaps the evaluation of chunk c, and warps drift freely.
// ------------------------------------------------------------------------------------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n NC_WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra NC_WAIT_%=;\n}" ::"r"(
          smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// bufs: 2 x brec records; bars: full[2], empty[2] (initialised here; the caller __syncthreads() before the first
// wait is done inside).  Threads of warps with no active target must not call (they return before).  nwarps_act:
// warps that call.  lst: the unit's source-patch list (nsrc entries), s4: the rung's records.
template <int KIND, int TPT, int UNROLL, int FAR, class Tab>
__device__ __forceinline__ void accumulate_grid_tma(const double (&x)[TPT], const double (&y)[TPT],
                                                    const double (&z)[TPT], const double (&cq)[TPT],
                                                    double (&acc)[TPT], int nsrc, const int32_t* __restrict__ lst,
                                                    const double4* __restrict__ s4, int p, double4* __restrict__ bufs,
                                                    int brec, uint64_t* __restrict__ bars,
                                                    const Tab* __restrict__ logtab) {
  uint64_t* full = bars;
  uint64_t* empty = bars + 2;
  const int chp = brec / p;                              // patches per chunk (>= 1: brec >= p)
  const int nch = (nsrc + chp - 1) / chp;
  const bool producer = threadIdx.x == 0;
  auto issue = [&](int c) {
    const int b = c & 1, k0 = c * chp, k1 = min(nsrc, k0 + chp);
    mbar_expect_tx(&full[b], (unsigned)((k1 - k0) * p * sizeof(double4)));
    for (int k = k0; k < k1; ++k)
      bulk_g2s(bufs + (size_t)b * brec + (size_t)(k - k0) * p, s4 + (size_t)lst[k] * p, (unsigned)(p * sizeof(double4)),
               &full[b]);
  };
  if (producer) issue(0);
  for (int c = 0; c < nch; ++c) {
    const int b = c & 1;
    if (producer && c + 1 < nch) {
      if (c >= 1) mbar_wait(&empty[(c + 1) & 1], (unsigned)(((c - 1) >> 1) & 1));   // chunk c-1 released its buffer
      issue(c + 1);
    }
    mbar_wait(&full[b], (unsigned)((c >> 1) & 1));
    const double4* __restrict__ sp = bufs + (size_t)b * brec;
    const int nrec = (min(nsrc, (c + 1) * chp) - c * chp) * p;
#pragma unroll UNROLL
    for (int m = 0; m < nrec; ++m) {
      const double4 s = sp[m];
#pragma unroll
      for (int u = 0; u < TPT; ++u) {
        if (FAR) {
          const double qh = fma(x[u], s.x, fma(y[u], s.y, fma(z[u], s.z, cq[u])));
          acc[u] = fma(s.w, green_far_h<KIND>(qh, logtab), acc[u]);
        } else {
          const double dx = x[u] - s.x, dy = y[u] - s.y, dz = z[u] - s.z;
          const double qd = fma(dz, dz, fma(dy, dy, dx * dx));
          acc[u] = fma(s.w, green_q<KIND>(qd, logtab), acc[u]);
        }
      }
    }
    __syncwarp();
    if ((threadIdx.x & 31) == 0) mbar_arrive(&empty[b]);
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
