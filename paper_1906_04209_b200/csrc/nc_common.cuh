// nc_common.cuh -- internal declarations shared by the libnc translation units (not part of the ABI).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/nc.h"

#if NC_WITH_NCCL
#include <nccl.h>
#endif

namespace nc {

// ------------------------------------------------------------------------------------------------
// error plumbing
// ------------------------------------------------------------------------------------------------
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);

#define NC_CUDA_TRY(expr)                                   \
  do {                                                      \
    cudaError_t _e = (expr);                                \
    if (_e != cudaSuccess) return ::nc::cuda_fail(_e, #expr); \
  } while (0)

#define NC_TRY(expr)             \
  do {                           \
    int _rc = (expr);            \
    if (_rc != NC_OK) return _rc; \
  } while (0)

constexpr int kMaxP = 1024;
constexpr int kPairThreads = 256;   // threads per CTA in the direct pair-sum kernel
constexpr int kDefaultPairTpt = 2;  // targets per thread (NC_PAIR_TPT=1|2 overrides)
constexpr int kDefaultStageLdg = 0; // 1: pair kernels read sources via L1 broadcasts (NC_PAIR_STAGE=ldg|smem)

// The tuning knobs (NC_GRID_VARIANT, NC_INTERP_*, NC_COST_*, NC_RING_*, NC_*_MARGIN, NC_GRID_TOL_FACTOR, ...) change
// the kernels or the plan and hence the numerics; they are read only when NC_TUNING=1 is also set (sweeps and the
// variant tests set it), so a default run cannot be altered by a stray environment variable.
inline const char* tuning_env(const char* name) {
  static const bool on = [] {
    const char* e = getenv("NC_TUNING");
    return e && e[0] == '1';
  }();
  return on ? getenv(name) : nullptr;
}

// setup phase timer (NC_SETUP_TIMING=1 prints wall-clock ms per phase to stderr)
void setup_tick(const char* phase);

// ------------------------------------------------------------------------------------------------
// hierarchical-mode state (hier.cu) and its step-2/3 work unit (direct.cu)
// ------------------------------------------------------------------------------------------------
struct HierState;

// k_pairs_grid variant {threads per CTA, targets per thread, source unroll, staged source records (per buffer when
// tma), far-field arithmetic, bulk-copy mbarrier pipeline}; NC_GRID_VARIANT overrides (tools/sweep_grid.py)
struct GridVariant {
  int nt, tpt, unroll, stage, far, tma, minb;   // minb: __launch_bounds__ min blocks per SM (register cap)
  int persist;                                  // 1: persistent CTAs taking units from an atomic counter
};
#define kGridVariantDefault (GridVariant{8, 2, 4, 64, 9, 3, 2, 1})   // warp-level units (tma = 3), R35 quadratic
#define kGridVariantPrecise (GridVariant{8, 2, 4, 64, 10, 3, 3, 1})  // R35 cubic: requested precision < 1e-10
constexpr double kGridQuadMinPrecision = 1e-10;   // the quadratic far form's log error is 7.7e-11 absolute
GridVariant grid_variant_for(double precision);   // the variant a handle uses (NC_GRID_VARIANT overrides)
int grid_far_table_bits(const GridVariant& v);    // bits of the far table the variant needs (0: none)
void grid_far_poly(const GridVariant& v, double* a2, double* a3);   // its log1p constants (carried after the table)
int grid_far_table_rcp(const GridVariant& v);     // 1: c from rcp.approx, L alone in the table (8-byte entries);
                                                  // 2: the same with c = rcp_seed_hl (R35)
struct FarTable {                      // exponent-indexed far log table (green.cuh green_far_t) on device
  const double2* d = nullptr;
  int n = 0, base = 0;
};
// host: build and upload the far table for (kind, eps, bits) (green_table.cu); *base = first index (biased
// exponent << bits), *n entries, followed by one extra entry (a2, a3); the caller owns *d (cudaFree).  0 on success.
// rcp != 0: the entries are L alone (8 bytes, two per double2; n even) for c = rcp.approx(bin midpoint).
// exact != 0: the table of the exact form (green_exact_r: interior x = q (1 + w), L without ln 2).
int far_table_build(int kind, double eps, int bits, int rcp, double a2, double a3, double2** d, int* n, int* base,
                    int exact = 0);
int grid_unit_points(const GridVariant& v);   // grid points per work unit = (threads per CTA or warp) x targets per thread

struct GridUnit {      // <= grid_unit_points() points of one incoming grid x one slice of its source-patch list
  int64_t pt0;         // first grid point (global grid-point index)
  int64_t src0;        // first entry in the source-patch list
  int64_t soff;        // offset (doubles) of the outgoing-operator rung's source records in d_src4
  int32_t npt;         // points in this unit (<= grid_unit_points())
  int32_t nsrc;        // source patches in this unit
  int32_t p;           // skeleton size of the rung
  int32_t pad_;
};

// ------------------------------------------------------------------------------------------------
// the handle
// ------------------------------------------------------------------------------------------------
}  // namespace nc

struct nc_handle {
  int kind = 0, mode = 0, device = 0, world = 1, rank = 0;
  bool emulated = false;          // world > 1 without a communicator (nc_matvec_emulated; partition tests)
  int64_t N = 0, row_begin = 0, row_count = 0;
  std::vector<int64_t> rank_begin, rank_count;   // partition of the internal rows over all ranks
  int M = 0, K = 0, Kstar = 0, p = 0;
  double eps = 0.0, precision = 1e-9;
  cudaStream_t stream = nullptr;  // library's own stream (used when caller passes NULL to setup ops)

  // tables on device
  double* d_T = nullptr;   // p x K
  double* d_P = nullptr;   // K x Kstar
  double* d_I = nullptr;   // K
  double* d_zhat = nullptr;  // Kstar x 3
  double* d_shat = nullptr;  // p x 3
  std::vector<double> h_P1;  // P . 1 (K), the physical right-hand side of every patch
  std::vector<double> h_I;

  // layout (internal order)
  std::vector<int64_t> perm;      // perm[internal] = caller index
  double* d_centers = nullptr;    // N x 3 (internal order)
  double* d_frames = nullptr;     // N x 9, R_i column-major: [e1 | e2 | c]

  // direct-mode geometry and work buffers
  double* d_tx = nullptr;         // row_count*Kstar targets (SoA)
  double* d_ty = nullptr;
  double* d_tz = nullptr;
  double* d_src4 = nullptr;       // per rung k: N * p_k records (x, y, z, -), coordinates scaled by 1/2 (static)
  double* d_rho = nullptr;        // per rung k: N * p_k values rho = T_k fhat (K1 output), at d_src4's offset / 4
  nc::FarTable xtab;              // exact-form log table of the direct / near-list kernels (green_exact_r)
  double2* d_xtab = nullptr;
  // outgoing-operator rungs: 0 = base (T, shat, p); 1.. = per-level ladder
  int nrung = 1;
  std::vector<double> rung_r;     // inner radius (arc length) of validity
  std::vector<int> rung_p;
  std::vector<int64_t> rung_trow; // first row of the rung in d_T (rows of K)
  std::vector<int64_t> rung_soff; // offset (doubles) of the rung's records in d_src4
  std::vector<char> rung_used;    // rungs whose rho K1 must produce
  double* d_shat_all = nullptr;   // sum p_k x 3
  double* d_Tcat = nullptr;       // concatenated T_k of the rungs in use (ncat x K), fused K1
  int64_t* d_colbase = nullptr;   // per concatenated column: record offset of (rung, m) and row stride 4 p_k
  int64_t* d_colrstride = nullptr;
  int ncat = 0;
  double* d_xall = nullptr;       // world > 1: all ranks' coefficient rows (N x K), gathered every matvec
  double* d_xpad = nullptr;       // world > 1: the padded all-gather buffer (world x max rows x K)
  int64_t max_rows = 0;           // world > 1: the largest rank row count (the all-gather's per-rank count)
  double* d_upart = nullptr;      // nseg x (row_count*Kstar) partial fields
  int nseg = 1;
  int pair_tpt = 1;               // targets per thread in the direct kernel (1 or 2)

  // GMRES workspace
  double* d_V = nullptr;
  int V_cap = 0;
  double* d_red = nullptr;        // reduction scratch
  int64_t red_cap = 0;
  double* h_red = nullptr;        // pinned host mirror
  double* d_b = nullptr;          // scratch rhs
  double* d_hx = nullptr;         // host-API staging (x and y)
  double* d_hy = nullptr;

  // stream ordering: a matvec shares the handle's work buffers (records, grids, partials) with every other matvec,
  // so a matvec issued on a stream other than the previous one's waits for that one first
  cudaStream_t last_stream = nullptr;
  bool have_last_stream = false;
  cudaEvent_t ev_order = nullptr;
  // nc_matvec_host (world 1): x copied in row blocks on a second stream, each block's K1 as soon as it has landed
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t copy_ev[5] = {};

  // per-stage timing
  bool time_stages = false;
  bool stages_pending = false;    // events of the last matvec recorded, not yet read (nc_stats reads them)
  cudaEvent_t ev[9] = {};           // [8]: after the hier grid reduction (k_reduce_chunks)
  double ms_last[8] = {};
  int launches_last = 0;          // kernels launched by the last nc_matvec
  double gmres_ortho_ms = 0.0;    // GMRES CGS2 orthogonalisation device time / algorithmic bytes (time_stages on)
  double gmres_ortho_bytes = 0.0;
  int64_t gmres_ortho_iters = 0;
  int64_t matvecs = 0;
  double pairs_per_matvec = 0.0;
  double device_bytes = 0.0;

  nc::HierState* hier = nullptr;

#if NC_WITH_NCCL
  ncclComm_t comm = nullptr;
#endif
};

namespace nc {

// ------------------------------------------------------------------------------------------------
// kernels / launchers (geometry.cu, gemm.cu, direct.cu, blas.cu)
// ------------------------------------------------------------------------------------------------
// frames R_i (ABI rule) and global node sets
void launch_frames(const double* centers, int64_t N, double* frames, cudaStream_t s);
// (coordinates written pre-multiplied by `scale`; the pair kernels use scale = 1/2, see green.cuh)
// step-4 proxy rule (proxy.cu, R36): returns n (0: none); pts n x 3, Int Ks x n, kappa (min D / h), h
int proxy_rule_build(const double* zhat, int Ks, int deg, int nring, double cphi, double tol, std::vector<double>& pts,
                     std::vector<double>& Int, double* kappa, double* h_out);
void launch_targets(const double* frames, int64_t row_begin, int64_t row_count, const double* zhat, int Kstar,
                    double scale, double* tx, double* ty, double* tz, cudaStream_t s);
void launch_sources(const double* frames, int64_t N, const double* shat, int p, double scale, double* src4,
                    cudaStream_t s);

// C[i, n] (+)= sum_k A[i, k] * Bt[n, k]   (fp64 DMMA m8n8k4)
//   A: rows x kd, leading dim lda; if nparts > 1, A is the sum of nparts matrices spaced part_stride apart
//   Bt: ncols x kd row-major
//   C element (i, n) is stored at C[i * ldc + n * cstride]; if X != nullptr, C = X + A Bt^T with X (ldx)
void launch_gemm_dmma(const double* A, int64_t lda, int nparts, int64_t part_stride, const double* Bt, int64_t rows,
                      int ncols, int kd, double* C, int64_t ldc, int cstride, const double* X, int64_t ldx,
                      cudaStream_t s);
// C[colbase[n] + (row0 + i) colrstride[n]] = sum_k A[i, k] Bt[n, k]   (scattered epilogue, one launch)
void launch_gemm_dmma_colmap(const double* A, int64_t lda, const double* Bt, int64_t rows, int ncols, int kd, double* C,
                             const int64_t* colbase, const int64_t* colrstride, int64_t row0, cudaStream_t s);

// direct pair sums: upart[seg][t] = sum over source patches j in segment seg, j != patch(t), of
// sum_m G(target t, s_jm) rho_jm
void launch_pairs_direct(int kind, int tpt, const double* tx, const double* ty, const double* tz, int64_t n_tgt,
                         int Kstar, int64_t tgt_patch0, const double* src4, const double* rho, int p, int64_t N,
                         int nseg, double* upart, const FarTable& xt, double eps, cudaStream_t s);

int pairs_direct_blocks_per_sm(int p, int tpt, const FarTable& xt);
void split_rows(const double* w, int64_t N, int world, int64_t* begin, int64_t* count);
void launch_pairs_grid(const GridVariant& v, int kind, const GridUnit* units, int64_t nunits, const double* gx,
                       const double* gy, const double* gz, const int32_t* srclist, const double* src4,
                       const double* rho, int pmax, double* part, int* counter /* device int, persistent variant */,
                       const FarTable& ft, cudaStream_t s);
void launch_pairs_near(int kind, const double* tx, const double* ty, const double* tz, int Kstar, const int32_t* work,
                       int64_t nwork, const int64_t* near_off, const int32_t* near, const double* src4,
                       const double* rho, int p, double* udir, const FarTable& xt, cudaStream_t s);

// off-surface field (field.cu, NEXT-3): out[t] = sum over all source records of G_off(pts_t, s) rho_s, dmin[t] =
// min |pts_t - s|; part / dpart: nseg x n scratch
int field_segments(int64_t n, int64_t nrec);
void launch_field(int kind, const double* pts, int64_t n, const double* src4, int64_t nrec, int nseg, double* part,
                  double* dpart, double* out, double* dmin, cudaStream_t s);

// L2 residual diagnostic (field.cu, NEXT-4): per listed patch q (internal row rows[q]), pointwise[q][k] =
// (S x_q)_k + sum_seg upart[q][seg][k] - 1 and res[q] = sqrt(sum_k w_k pointwise^2) / sum_k w_k
void launch_residual(int n_sel, int n_res, int K, int nseg, const int64_t* rows, const double* x_all, const double* S,
                     const double* w, const double* upart, double* pointwise, double* res, cudaStream_t s);

void launch_gather_rows(const double* x_all, const int64_t* rows, int n_sel, int K, double* out, cudaStream_t s);

// NEXT-3 near the surface (nearfield.cu): the density quadrature of the patches near each point
struct NearDev {
  int npan, k, n_r, M1, K;
  const double* edges;   // npan + 1
  const double* t;       // n_r
  const double* w;       // n_r
  const double* sigma;   // K x n_r
  const int* mc_off;     // 2 M1 + 1: CSR over (m, cos|sin) of the basis columns
  const int* mc_col;     // K
  const double* gl_x;    // k reference Gauss-Legendre nodes on [-1, 1] (of the regular panels)
  const double* gl_w;    // k weights
  const double* bary;    // k barycentric weights of those nodes
  const double* trig;    // 4096 x (cos, sin) of 2 pi k / 4096
};
constexpr double kNearRadius = 4.0;          // a patch is near a point closer than this x eps to its centre
constexpr double kNearMinHeight = 0.01;      // points near a patch must be >= this x eps off the sphere
constexpr int kNearTrigN = 4096;
// list == nullptr: cnt[t] = the number of centres within r of point t; else list[off[t] ..] = their indices
void launch_near_count(const double* pts, int64_t n, const double* cen, int64_t N, double r, int64_t* cnt,
                       int64_t* list, const int64_t* off, cudaStream_t s);
size_t near_quad_smem(int n_r, int M1);
int launch_near_quad(int kind, const int64_t* pair_pt, const int64_t* pair_patch, int64_t npairs, const double* pts,
                     const double* frames, const double* x_all, const NearDev& nd, const double* rec, int p0,
                     double* corr, int* status, cudaStream_t s);
void launch_near_apply(const int64_t* off, const double* corr, int64_t n, double* out, cudaStream_t s);

// BLAS-1 style helpers for GMRES (deterministic two-stage reductions)
int64_t multidot_partials(int64_t n);
void launch_multidot(const double* V, int64_t ldv, int nv, const double* w, int64_t n, double* part, double* out,
                     cudaStream_t s);  // out[i] = V_i . w, i < nv
void launch_gemv_sub(const double* V, int64_t ldv, int nv, const double* h, double* w, int64_t n,
                     cudaStream_t s);  // w -= sum_i h_i V_i, h on device
void launch_lincomb(const double* V, int64_t ldv, int nv, const double* y, double* x, int64_t n,
                    cudaStream_t s);  // x = sum_i y_i V_i
void launch_scale(double* dst, const double* src, const double* alpha_dev, int invert, int64_t n,
                  cudaStream_t s);  // dst = src * (*alpha or 1/ *alpha)
void launch_fill_rows(double* dst, const double* row_dev, int K, int64_t rows, cudaStream_t s);
void launch_colsum(const double* X, int64_t rows, int K, double* part, double* out, cudaStream_t s);

}  // namespace nc
