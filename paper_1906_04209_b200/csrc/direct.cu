// direct.cu -- pair-sum kernels built on pairs.cuh:
//
//  k_pairs_direct  (a2, direct mode)   u_{ik} = sum_{j != i} sum_m G(z_ik, s_jm) rho_jm over a segment of patches
//  k_pairs_grid    (a3/a4, hier mode)  grid_g(x) += sum_{j in slice} sum_m G(x, s_jm) rho_jm  (one work unit:
//                                      <= 256 points of one incoming grid x one slice of its source-patch list)
//  k_pairs_near    (a4, hier mode)     u_{ik} += sum_{j in near(i)} sum_m G(z_ik, s_jm) rho_jm
//
// Direct mode: one CTA per (target tile of 256*TPT nodes, source segment); the source range is split into `nseg`
// segments (grid.y) chosen so the CTA count fills the last wave (api.cu); segment partials are summed in the
// step-5 GEMM's operand load (gemm.cu), deterministic.
#include <stdlib.h>

#include <stdio.h>

#include <algorithm>
#include <type_traits>

#include "pairs.cuh"

namespace nc {

template <int KIND, int TPT>
__global__ void __launch_bounds__(kPairThreads, 2) k_pairs_direct(const double* __restrict__ tx,
                                                                const double* __restrict__ ty,
                                                                const double* __restrict__ tz, int64_t n_tgt,
                                                                int Kstar, int64_t tgt_patch0,
                                                                const double* __restrict__ src4, int p, int64_t N,
                                                                int nseg, int chp, double* __restrict__ upart,
                                                                const double2* __restrict__ logsrc) {
  extern __shared__ double4 sm[];
  __shared__ double2 logtab[kLogTableSize];
  __shared__ int64_t pid[kStagePatchesMax];
  init_log_table(logtab, logsrc);
  double x[TPT], y[TPT], z[TPT], acc[TPT];
  int64_t excl[TPT];
  const int64_t t0 = (int64_t)blockIdx.x * kPairThreads * TPT + threadIdx.x;
#pragma unroll
  for (int u = 0; u < TPT; ++u) {
    const int64_t t = min(t0 + u * kPairThreads, n_tgt - 1);
    x[u] = tx[t]; y[u] = ty[t]; z[u] = tz[t];
    excl[u] = tgt_patch0 + t / Kstar;         // j != i
    acc[u] = 0.0;
  }
  const int seg = blockIdx.y;
  const int64_t j0 = (N * seg) / nseg, j1 = (N * (seg + 1)) / nseg;
  if (chp == 0) {
    __syncthreads();
    accumulate_list_ldg<KIND, TPT>(x, y, z, excl, acc, j1 - j0, [=] __device__(int64_t k) { return j0 + k; },
                                   reinterpret_cast<const double4*>(src4), p, logtab);
  } else {
    accumulate_list<KIND, TPT>(x, y, z, excl, acc, j1 - j0, [=] __device__(int64_t k) { return j0 + k; },
                               reinterpret_cast<const double4*>(src4), p, sm, pid, chp, logtab, true);
  }
#pragma unroll
  for (int u = 0; u < TPT; ++u) {
    const int64_t t = t0 + u * kPairThreads;
    if (t < n_tgt) upart[(int64_t)seg * n_tgt + t] = acc[u];
  }
}

static bool stage_ldg();

int pairs_direct_blocks_per_sm(int p, int tpt) {
  int nb = 0;
  size_t smem = stage_ldg() ? 0 : (size_t)stage_patches(p) * p * sizeof(double4);
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
  const int chp = stage_ldg() ? 0 : stage_patches(p);
  const size_t smem = (size_t)chp * p * sizeof(double4);
  const int64_t per_block = (int64_t)kPairThreads * tpt;
  dim3 grid((unsigned)((n_tgt + per_block - 1) / per_block), (unsigned)nseg);
#define NC_LAUNCH(KD, TP) \
  k_pairs_direct<KD, TP><<<grid, kPairThreads, smem, s>>>(tx, ty, tz, n_tgt, Kstar, tgt_patch0, src4, p, N, nseg, chp, upart, \
                                                          log_table_device())
  if (kind == NC_EXTERIOR) {
    if (tpt == 2) NC_LAUNCH(1, 2); else NC_LAUNCH(1, 1);
  } else {
    if (tpt == 2) NC_LAUNCH(0, 2); else NC_LAUNCH(0, 1);
  }
#undef NC_LAUNCH
}

// ------------------------------------------------------------------------------------------------
// hierarchical mode: interaction-list / leaf-neighbour sources on incoming grids
// ------------------------------------------------------------------------------------------------
// One CTA of kGridThreads threads per work unit: <= kGridThreads * TPT adjacent points of one incoming grid x one
// slice (<= kSliceMax patches, one outgoing-operator rung) of its source list.  Sources are staged in shared memory
// `chp` patches at a time; the log table is double2 (LOG8 = false) or the 8-byte table of green.cuh (LOG8 = true).
template <int KIND, int TPT, int UNROLL, bool LOG8, bool FAR>
__global__ void __launch_bounds__(kGridThreads) k_pairs_grid(const GridUnit* __restrict__ units,
                                                              const double* __restrict__ gx,
                                                              const double* __restrict__ gy,
                                                              const double* __restrict__ gz,
                                                              const int32_t* __restrict__ srclist,
                                                              const double* __restrict__ src4, int stage_records,
                                                              double* __restrict__ part,
                                                              const void* __restrict__ logsrc) {
  using Tab = typename std::conditional<LOG8, double, double2>::type;
  extern __shared__ double4 sm[];
  __shared__ Tab logtab[kLogTableSize];
  __shared__ int64_t pid[kStagePatchesMax];
  init_table(logtab, reinterpret_cast<const Tab*>(logsrc));
  const GridUnit U = units[blockIdx.x];
  double x[TPT], y[TPT], z[TPT], cq[TPT], acc[TPT];
  // adjacent points per thread (l = TPT t + u): a partial chunk leaves at most one partially idle warp
  const bool any = (int)(TPT * threadIdx.x) < U.npt;
#pragma unroll
  for (int u = 0; u < TPT; ++u) {
    const int l = TPT * threadIdx.x + u;
    const int64_t g = U.pt0 + min(l, U.npt - 1);
    x[u] = gx[g]; y[u] = gy[g]; z[u] = gz[g];
    cq[u] = fma(x[u], x[u], fma(y[u], y[u], fma(z[u], z[u], 0.25)));
    if (FAR) { x[u] *= -2.0; y[u] *= -2.0; z[u] *= -2.0; }
    acc[u] = 0.0;
  }
  const int32_t* __restrict__ lst = srclist + U.src0;
  const double4* __restrict__ s4 = reinterpret_cast<const double4*>(src4 + U.soff);   // the unit's rung
  int chp = stage_records / U.p;
  chp = chp < 1 ? 1 : (chp > kStagePatchesMax ? kStagePatchesMax : chp);
  accumulate_grid<KIND, TPT, UNROLL, FAR, Tab>(x, y, z, cq, acc, U.nsrc,
                                               [=] __device__(int64_t k) { return (int64_t)lst[k]; }, s4, U.p, sm, pid,
                                               chp, logtab, any);
  const int upts = kGridThreads * TPT;
#pragma unroll
  for (int u = 0; u < TPT; ++u) {
    const int l = TPT * threadIdx.x + u;
    if (l < U.npt) part[(int64_t)blockIdx.x * upts + l] = acc[u];
  }
}

static bool stage_ldg() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("NC_PAIR_STAGE");
    v = (e && e[0] == 's') ? 0 : (e && e[0] == 'l') ? 1 : kDefaultStageLdg;
  }
  return v == 1;
}

// grid-kernel variant: NC_GRID_VARIANT="TPT,UNROLL,LOG8,STAGE" (default kGridVariantDefault)
static GridVariant grid_variant() {
  static GridVariant v = {0, 0, 0, 0, 0};
  if (v.tpt == 0) {
    v = kGridVariantDefault;
    if (const char* e = getenv("NC_GRID_VARIANT")) {
      GridVariant w = v;
      const int n = sscanf(e, "%d,%d,%d,%d,%d", &w.tpt, &w.unroll, &w.log8, &w.stage, &w.far);
      if (n >= 4 && (w.tpt == 2 || w.tpt == 4) && (w.unroll == 1 || w.unroll == 2 || w.unroll == 4) &&
          (w.log8 == 0 || w.log8 == 1) && w.stage >= 32 && (w.far == 0 || w.far == 1))
        v = w;
    }
  }
  return v;
}

int grid_far_variant() { return grid_variant().far; }

int grid_unit_points() { return kGridThreads * grid_variant().tpt; }

template <int KIND, int TPT, int UNROLL, bool LOG8, bool FAR>
static void launch_grid_t(const GridUnit* units, int64_t nunits, const double* gx, const double* gy, const double* gz,
                          const int32_t* srclist, const double* src4, int stage, size_t smem, double* part,
                          cudaStream_t s) {
  const void* tab = LOG8 ? (const void*)log8_table_device() : (const void*)log_table_device();
  auto kern = k_pairs_grid<KIND, TPT, UNROLL, LOG8, FAR>;
  if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  kern<<<(unsigned)nunits, kGridThreads, smem, s>>>(units, gx, gy, gz, srclist, src4, stage, part, tab);
}

void launch_pairs_grid(int kind, const GridUnit* units, int64_t nunits, const double* gx, const double* gy,
                       const double* gz, const int32_t* srclist, const double* src4, int pmax, double* part,
                       cudaStream_t s) {
  if (nunits <= 0) return;
  const GridVariant v = grid_variant();
  const size_t smem = (size_t)std::max(v.stage, pmax) * sizeof(double4);   // >= chp * p and >= one whole patch
#define NC_G(KD, TP, UR, L8, FR) \
  if (kind == KD && v.tpt == TP && v.unroll == UR && v.log8 == L8 && v.far == FR) \
    return launch_grid_t<KD, TP, UR, L8, FR>(units, nunits, gx, gy, gz, srclist, src4, std::max(v.stage, pmax), smem, part, s);
#define NC_GK(KD) \
  NC_G(KD, 2, 2, 0, 0) NC_G(KD, 2, 4, 0, 0) NC_G(KD, 2, 2, 0, 1) NC_G(KD, 2, 4, 0, 1) NC_G(KD, 2, 1, 0, 1) \
  NC_G(KD, 4, 2, 0, 0) NC_G(KD, 4, 2, 0, 1) NC_G(KD, 2, 4, 1, 0)
  NC_GK(0)
  NC_GK(1)
#undef NC_GK
#undef NC_G
}

// ------------------------------------------------------------------------------------------------
// hierarchical mode: near-list sources evaluated directly at the target patch's Zernike nodes
// ------------------------------------------------------------------------------------------------
template <int KIND, int TPT>
__global__ void __launch_bounds__(kPairThreads) k_pairs_near(const double* __restrict__ tx,
                                                              const double* __restrict__ ty,
                                                              const double* __restrict__ tz, int Kstar,
                                                              const int32_t* __restrict__ work,  // local patch ids
                                                              const int64_t* __restrict__ near_off,
                                                              const int32_t* __restrict__ near,
                                                              const double* __restrict__ src4, int p, int chp,
                                                              double* __restrict__ udir,
                                                              const double2* __restrict__ logsrc) {
  extern __shared__ double4 sm[];
  __shared__ double2 logtab[kLogTableSize];
  __shared__ int64_t pid[kStagePatchesMax];
  init_log_table(logtab, logsrc);
  const int tiles = (Kstar + kPairThreads * TPT - 1) / (kPairThreads * TPT);
  const int64_t i = work[blockIdx.x / tiles];           // local target patch
  const int tile = blockIdx.x % tiles;
  double x[TPT], y[TPT], z[TPT], acc[TPT];
  int64_t excl[TPT];
#pragma unroll
  for (int u = 0; u < TPT; ++u) {
    const int k = min(tile * kPairThreads * TPT + (int)threadIdx.x + u * kPairThreads, Kstar - 1);
    const int64_t t = i * Kstar + k;
    x[u] = tx[t]; y[u] = ty[t]; z[u] = tz[t];
    excl[u] = -1;
    acc[u] = 0.0;
  }
  const int64_t o0 = near_off[i], o1 = near_off[i + 1];
  const int32_t* __restrict__ lst = near + o0;
  if (chp == 0) {
    __syncthreads();
    accumulate_list_ldg<KIND, TPT>(x, y, z, excl, acc, o1 - o0, [=] __device__(int64_t k) { return (int64_t)lst[k]; },
                                   reinterpret_cast<const double4*>(src4), p, logtab);
  } else {
    accumulate_list<KIND, TPT>(x, y, z, excl, acc, o1 - o0, [=] __device__(int64_t k) { return (int64_t)lst[k]; },
                               reinterpret_cast<const double4*>(src4), p, sm, pid, chp, logtab, true);
  }
#pragma unroll
  for (int u = 0; u < TPT; ++u) {
    const int k = tile * kPairThreads * TPT + (int)threadIdx.x + u * kPairThreads;
    if (k < Kstar) udir[i * Kstar + k] = acc[u];
  }
}

void launch_pairs_near(int kind, const double* tx, const double* ty, const double* tz, int Kstar, const int32_t* work,
                       int64_t nwork, const int64_t* near_off, const int32_t* near, const double* src4, int p,
                       double* udir, cudaStream_t s) {
  if (nwork <= 0) return;
  const int chp = stage_ldg() ? 0 : stage_patches(p);
  const size_t smem = (size_t)chp * p * sizeof(double4);
  const int tiles = (Kstar + kPairThreads * 2 - 1) / (kPairThreads * 2);
  const unsigned nb = (unsigned)(nwork * tiles);
  if (kind == NC_EXTERIOR)
    k_pairs_near<1, 2><<<nb, kPairThreads, smem, s>>>(tx, ty, tz, Kstar, work, near_off, near, src4, p, chp, udir,
                                                      log_table_device());
  else
    k_pairs_near<0, 2><<<nb, kPairThreads, smem, s>>>(tx, ty, tz, Kstar, work, near_off, near, src4, p, chp, udir,
                                                      log_table_device());
}

}  // namespace nc
