// gemm.cu -- the two per-patch operator applications of the matvec as fp64 tensor-core GEMMs.
//
//   step 1: rho_i = T fhat_i for all i      -> C = X T^T        (N x p)
//   step 5: y_i = fhat_i + P u_i for all i  -> Y = X + U P^T    (N x K)
//
// B200 has no fp64 kind in tcgen05; the fp64 tensor path is the legacy warp-level
// mma.sync.aligned.m8n8k4.f64 (SASS DMMA.8x8x4), measured at 37.1 TF/s on this pool
// (profiles/r01_fp64_peak.txt).  CTA tile 64 x 64 x 16, 8 warps (4 x 2), each warp 16 x 32 = 2 x 4 DMMA tiles;
// operands staged in padded shared memory (row stride BK+4 doubles: conflict-free fragment loads).
// For step 5 the A operand is the sum of the direct kernel's per-segment partial fields (fused
// deterministic reduction), and the epilogue adds the identity term.  For step 1 with several outgoing-operator rungs
// one GEMM applies the concatenated T_k of all rungs in use, its epilogue scattering column (k, m) into rung k's
// source records through a per-column (base, row stride) map.
#include <stdint.h>
#include <stdlib.h>

#include "nc_common.cuh"

namespace nc {

namespace {
constexpr int BM = 64, BN = 64, BK = 16, LDS = BK + 4;

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}
}  // namespace

__global__ void __launch_bounds__(256) k_gemm_dmma(const double* __restrict__ A, int64_t lda, int nparts,
                                                   int64_t part_stride, const double* __restrict__ Bt, int64_t rows,
                                                   int ncols, int kd, double* __restrict__ C, int64_t ldc,
                                                   int cstride, const double* __restrict__ X, int64_t ldx,
                                                   const int64_t* __restrict__ colbase,
                                                   const int64_t* __restrict__ colrstride, int64_t crow0) {
  __shared__ double As[BM][LDS];
  __shared__ double Bs[BN][LDS];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 1, wn = warp & 1;
  const int64_t row0 = (int64_t)blockIdx.x * BM;
  const int col0 = blockIdx.y * BN;

  double acc[2][4][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

  for (int k0 = 0; k0 < kd; k0 += BK) {
    // stage A (sum of parts) and Bt tiles; consecutive threads read consecutive k (coalesced)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      int r = (tid >> 4) + 16 * q, c = tid & 15;
      int64_t gr = row0 + r;
      int gk = k0 + c;
      double v = 0.0;
      if (gr < rows && gk < kd) {
        const double* pa = A + gr * lda + gk;
        v = pa[0];
        for (int s = 1; s < nparts; ++s) v += pa[s * part_stride];
      }
      As[r][c] = v;
      int n = col0 + r;
      Bs[r][c] = (n < ncols && gk < kd) ? Bt[(int64_t)n * kd + gk] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[2], bf[4];
#pragma unroll
      for (int mi = 0; mi < 2; ++mi) af[mi] = As[wm * 16 + mi * 8 + (lane >> 2)][kk + (lane & 3)];
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) bf[ni] = Bs[wn * 32 + ni * 8 + (lane >> 2)][kk + (lane & 3)];
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) dmma(acc[mi][ni], af[mi], bf[ni]);
    }
    __syncthreads();
  }
  // epilogue: C(i, n) = [X(i, n) +] acc
#pragma unroll
  for (int mi = 0; mi < 2; ++mi) {
    int64_t gr = row0 + wm * 16 + mi * 8 + (lane >> 2);
    if (gr >= rows) continue;
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        int n = col0 + wn * 32 + ni * 8 + (lane & 3) * 2 + e;
        if (n >= ncols) continue;
        double v = acc[mi][ni][e];
        if (X) v += X[gr * ldx + n];
        if (colbase)   // column map: element (i, n) -> C[colbase[n] + (crow0 + i) colrstride[n]]
          C[colbase[n] + (crow0 + gr) * colrstride[n]] = v;
        else
          C[gr * ldc + (int64_t)n * cstride] = v;
      }
    }
  }
}

// ------------------------------------------------------------------------------------------------
// Pipelined variant (single A operand): CTA tile 128 x 64 x 16, 8 warps (4 x 2) of 32 x 32 = 4 x 4 DMMA tiles (8
// fragment loads per 16 DMMA), both operands copied global -> shared by cp.async into a double buffer (zero-filled
// beyond the matrix edges), so the next k-slab streams in while the current one is multiplied (the
// single-buffered kernel above reached 0.38 / 0.46 of the DMMA peak on K1 / P-apply).
// ------------------------------------------------------------------------------------------------
namespace {
constexpr int PM = 128, PK = 16, PLD = PK + 4;

__device__ __forceinline__ void cp16_zfill(void* dst, const void* src, bool valid) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  const int n = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(n) : "memory");
}
}  // namespace

// NF: n8 fragments per warp (4: 64-column CTA tiles; 3: 48 -- K3's 136 columns then pad to 144 instead of 192)
template <int NF>
__global__ void __launch_bounds__(256) k_gemm_dmma_pipe(const double* __restrict__ A, int64_t lda,
                                                        const double* __restrict__ Bt, int64_t rows, int ncols, int kd,
                                                        double* __restrict__ C, int64_t ldc, int cstride,
                                                        const double* __restrict__ X, int64_t ldx,
                                                        const int64_t* __restrict__ colbase,
                                                        const int64_t* __restrict__ colrstride, int64_t crow0) {
  constexpr int PNt = 16 * NF;                   // CTA tile columns (2 warps x NF x 8)
  extern __shared__ __align__(16) double gsm[];
  double* As = gsm;                              // [2][PM][PLD]
  double* Bs = gsm + 2 * PM * PLD;               // [2][PNt][PLD]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 1, wn = warp & 1;       // warp tile rows wm*32.., cols wn*8NF..
  // column tiles vary fastest (blockIdx.x): the CTAs resident together share their A row tile through L2, so A is read
  // from DRAM once rather than once per column tile (the K1 epilogue's record writes otherwise evict it)
  const int64_t row0 = (int64_t)blockIdx.y * PM;
  const int col0 = blockIdx.x * PNt;
  auto issue = [&](int k0, int b) {
    // A: 128 rows x 16 k = 1024 16-byte pieces (2 doubles), 4 per thread; B: 64 x 16 = 512, 2 per thread
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int e = tid + 256 * q, r = e >> 3, c = (e & 7) * 2;
      const int64_t gr = row0 + r;
      const int gk = k0 + c;
      const bool ok = gr < rows && gk < kd;   // kd even: a piece is all in or all out
      cp16_zfill(As + ((size_t)b * PM + r) * PLD + c, ok ? (const void*)(A + gr * lda + gk) : (const void*)A, ok);
    }
#pragma unroll
    for (int q = 0; q < (PNt * 8 + 255) / 256; ++q) {   // B: PNt rows x 16 k = PNt x 8 pieces
      const int e = tid + 256 * q, r = e >> 3, c = (e & 7) * 2;
      if (r >= PNt) break;
      const int n = col0 + r;
      const int gk = k0 + c;
      const bool ok = n < ncols && gk < kd;
      cp16_zfill(Bs + ((size_t)b * PNt + r) * PLD + c, ok ? (const void*)(Bt + (int64_t)n * kd + gk) : (const void*)Bt,
                 ok);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  double acc[4][NF][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < NF; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  const int nk = (kd + PK - 1) / PK;
  issue(0, 0);
  for (int s = 0; s < nk; ++s) {
    if (s + 1 < nk) {
      issue((s + 1) * PK, (s + 1) & 1);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    const double* as = As + (size_t)(s & 1) * PM * PLD;
    const double* bs = Bs + (size_t)(s & 1) * PNt * PLD;
#pragma unroll
    for (int kk = 0; kk < PK; kk += 4) {
      double af[4], bf[NF];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) af[mi] = as[(wm * 32 + mi * 8 + (lane >> 2)) * PLD + kk + (lane & 3)];
#pragma unroll
      for (int ni = 0; ni < NF; ++ni) bf[ni] = bs[(wn * 8 * NF + ni * 8 + (lane >> 2)) * PLD + kk + (lane & 3)];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < NF; ++ni) dmma(acc[mi][ni], af[mi], bf[ni]);
    }
    __syncthreads();   // every warp is done with buffer s & 1 before slab s + 2 is copied into it
  }
#pragma unroll
  for (int mi = 0; mi < 4; ++mi) {
    const int64_t gr = row0 + wm * 32 + mi * 8 + (lane >> 2);
    if (gr >= rows) continue;
#pragma unroll
    for (int ni = 0; ni < NF; ++ni) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int n = col0 + wn * 8 * NF + ni * 8 + (lane & 3) * 2 + e;
        if (n >= ncols) continue;
        double v = acc[mi][ni][e];
        if (X) v += X[gr * ldx + n];
        if (colbase)
          C[colbase[n] + (crow0 + gr) * colrstride[n]] = v;
        else
          C[gr * ldc + (int64_t)n * cstride] = v;
      }
    }
  }
}

static bool gemm_pipe_ok(const double* A, int64_t lda, const double* Bt, int kd) {
  // cp.async needs 16-byte aligned rows: even leading dimensions and 16-byte aligned bases
  return (lda % 2 == 0) && (kd % 2 == 0) && ((uintptr_t)A % 16 == 0) && ((uintptr_t)Bt % 16 == 0) &&
         !tuning_env("NC_GEMM_SIMPLE");
}

template <int NF>
static void launch_pipe_nf(const double* A, int64_t lda, const double* Bt, int64_t rows, int ncols, int kd, double* C,
                           int64_t ldc, int cstride, const double* X, int64_t ldx, const int64_t* colbase,
                           const int64_t* colrstride, int64_t crow0, cudaStream_t s) {
  constexpr int PNt = 16 * NF;
  const size_t smem = (size_t)2 * (PM + PNt) * PLD * sizeof(double);
  cudaFuncSetAttribute(k_gemm_dmma_pipe<NF>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  dim3 grid((unsigned)((ncols + PNt - 1) / PNt), (unsigned)((rows + PM - 1) / PM));
  k_gemm_dmma_pipe<NF><<<grid, 256, smem, s>>>(A, lda, Bt, rows, ncols, kd, C, ldc, cstride, X, ldx, colbase,
                                               colrstride, crow0);
}
// the column tile that pads the output columns least (64 on ties)
static void launch_pipe(const double* A, int64_t lda, const double* Bt, int64_t rows, int ncols, int kd, double* C,
                        int64_t ldc, int cstride, const double* X, int64_t ldx, const int64_t* colbase,
                        const int64_t* colrstride, int64_t crow0, cudaStream_t s) {
  const int pad64 = (ncols + 63) / 64 * 64, pad48 = (ncols + 47) / 48 * 48;
  if (pad48 < pad64)
    return launch_pipe_nf<3>(A, lda, Bt, rows, ncols, kd, C, ldc, cstride, X, ldx, colbase, colrstride, crow0, s);
  launch_pipe_nf<4>(A, lda, Bt, rows, ncols, kd, C, ldc, cstride, X, ldx, colbase, colrstride, crow0, s);
}

void launch_gemm_dmma(const double* A, int64_t lda, int nparts, int64_t part_stride, const double* Bt, int64_t rows,
                      int ncols, int kd, double* C, int64_t ldc, int cstride, const double* X, int64_t ldx,
                      cudaStream_t s) {
  if (rows <= 0) return;
  if (nparts == 1 && gemm_pipe_ok(A, lda, Bt, kd))
    return launch_pipe(A, lda, Bt, rows, ncols, kd, C, ldc, cstride, X, ldx, nullptr, nullptr, 0, s);
  dim3 grid((unsigned)((rows + BM - 1) / BM), (unsigned)((ncols + BN - 1) / BN));
  k_gemm_dmma<<<grid, 256, 0, s>>>(A, lda, nparts, part_stride, Bt, rows, ncols, kd, C, ldc, cstride, X, ldx, nullptr,
                                   nullptr, 0);
}

void launch_gemm_dmma_colmap(const double* A, int64_t lda, const double* Bt, int64_t rows, int ncols, int kd, double* C,
                             const int64_t* colbase, const int64_t* colrstride, int64_t row0, cudaStream_t s) {
  if (rows <= 0 || ncols <= 0) return;
  if (gemm_pipe_ok(A, lda, Bt, kd))
    return launch_pipe(A, lda, Bt, rows, ncols, kd, C, 0, 0, nullptr, 0, colbase, colrstride, row0, s);
  dim3 grid((unsigned)((rows + BM - 1) / BM), (unsigned)((ncols + BN - 1) / BN));
  k_gemm_dmma<<<grid, 256, 0, s>>>(A, lda, 1, 0, Bt, rows, ncols, kd, C, 0, 0, nullptr, 0, colbase, colrstride, row0);
}

}  // namespace nc
