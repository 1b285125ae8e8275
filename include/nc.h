/*
 * nc.h -- C ABI of libnc: the preconditioned multiple-scattering matvec of Kaye & Greengard,
 * "A fast solver for the narrow capture and narrow escape problems in the sphere"
 * (arXiv:1906.04209; PAPER.md = the paper's LaTeX source), its GMRES solve and its scalar read-out,
 * on NVIDIA B200 (sm_100a), fp64.
 *
 * The operator (eq:opinteqnsdisc; step 3 of §8):
 *
 *     y_i = fhat_i + P sum_{j != i} S_ij B fhat_j,    i = 1..N,
 *
 * with the source patches in their skeletonised outgoing representation (eq:outgoingcompressed,
 * PAPER.md:1078-1096; eq:Tmap):
 *
 *     (S_ij B fhat_j)(z_{ik}) = sum_m G(z_{ik}, s_{jm}) rho_{jm},   rho_j = T fhat_j,
 *
 * G = G_I (interior / narrow escape, eq:Gintonsurface) or G_E (exterior / narrow
 * capture, eq:Gextonsurface), z_{ik} = R_i zhat_k the Zernike sampling nodes and
 * s_{jm} = R_j shat_m the skeleton nodes of patch j in its frame R_j.
 *
 * Conventions for every entry point:
 *   - return 0 (NC_OK) on success, a negative NC_E* code on failure; nc_last_error() returns a
 *     thread-local human-readable message for the last failure of the calling thread.
 *   - "host" pointers are ordinary CPU memory, "device" pointers are CUDA global memory on the
 *     handle's device.  All arrays are fp64, C order (row-major), densely packed.
 *   - Coefficient vectors use the library's INTERNAL patch order (see nc_partition) and are sharded
 *     by rank: rank r owns rows [row_begin, row_begin + row_count), each row = K contiguous doubles.
 *   - One handle per host thread.  Multi-rank calls (world > 1) are collective: every rank must
 *     make the same sequence of calls.
 *   - There is no CPU fallback: every arithmetic step runs in this library's CUDA kernels.
 */
#ifndef NC_H_
#define NC_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NC_OK 0
#define NC_EINVAL (-1)   /* invalid argument (sizes, null pointers, non-unit centres, K mismatch) */
#define NC_ESEP (-2)     /* two patch centres closer than 3 eps in arc length */
#define NC_ENOMEM (-3)   /* device allocation failed */
#define NC_ECUDA (-4)    /* CUDA runtime error (message has the CUDA error string) */
#define NC_ENCCL (-5)    /* NCCL error (world > 1) */
#define NC_ESTATE (-6)   /* call not valid in the handle's state (e.g. I_sigma <= 0 for the interior) */
#define NC_ENOCONV (-7)  /* GMRES reached max_iter above rtol; x holds the last iterate */
#define NC_EUNSUP (-8)   /* option not supported by this build */

#define NC_INTERIOR 0    /* narrow escape, G_I, read-out mu (eq:mufromsigma2) */
#define NC_EXTERIOR 1    /* narrow capture, G_E, read-out J = -4 pi I_sigma (reading R2) */

#define NC_DIRECT 0      /* tiled direct sum over all source patches j != i (eq:mssums) */
#define NC_HIER 1        /* hierarchical O(N log N) scheme of §8 steps 1-5 */

/* Patch-operator tables: Step-1 outputs for one patch radius, host memory,
 * copied by nc_setup (the caller may free them afterwards).  Canonical frame: patch centre at +z,
 * azimuth theta = 0 along +x. */
typedef struct nc_tables {
  int32_t M;           /* Zernike truncation; K must equal (M+1)(M+2)/2      */
  int32_t K;           /* compressed dofs per patch                                             */
  int32_t Kstar;       /* Zernike sampling nodes per patch, >= K             */
  int32_t p;           /* skeleton size (rank of the ID), 1 <= p <= 1024    */
  const double* zhat;  /* Kstar x 3  Zernike sampling nodes (unit vectors)                      */
  const double* P;     /* K x Kstar  discrete Zernike transform               */
  const double* shat;  /* p x 3      skeleton nodes x^f_{pi(m)} (unit vectors, inside the patch) */
  const double* T;     /* p x K      outgoing map rho = T fhat (eq:Tmap)                         */
  const double* I;     /* K          integration row, I_sigma = I . sum_i fhat_i (eq:getI)       */
  /* Optional per-level outgoing operators ("one matrix T per level"), used by NC_HIER on
   * incoming grids whose nearest point is at arc distance >= ladder_r[k] from the source centre.  The base
   * (shat, T, p) above is valid beyond 2 eps.  n_ladder = 0 (and NULL pointers) disables. */
  int32_t n_ladder;           /* number of rungs                                                   */
  const double* ladder_r;     /* n_ladder inner radii (arc length), increasing, > 2 eps            */
  const int32_t* ladder_p;    /* n_ladder skeleton sizes, 1..1024                                  */
  const double* ladder_shat;  /* sum(ladder_p) x 3 skeleton nodes, rung-major                      */
  const double* ladder_T;     /* sum(ladder_p) x K outgoing maps, rung-major                       */
  double ladder_tol;          /* ID tolerance of the rungs (0: unknown).  NC_HIER uses the ladder   */
                              /* only when the requested precision is >= this; the matvec error     */
                              /* at that boundary is measured <= the precision (R22,      */
                              /* tests/test_parity_golden_gpu.py test_ladder_gate_boundary)          */
} nc_tables;

typedef struct nc_opts {
  int32_t mode;          /* NC_DIRECT or NC_HIER                                                 */
  double precision;      /* NC_HIER: requested matvec precision (default 1e-9 when <= 0)         */
  int32_t device;        /* CUDA device ordinal (-1: current device)                             */
  int32_t world;         /* number of ranks (1 = single GPU)                                     */
  int32_t rank;          /* this rank, 0 <= rank < world                                         */
  const void* nccl_id;   /* world > 1: pointer to the 128-byte ncclUniqueId made by rank 0;      */
                         /* NULL with world > 1 = rank EMULATION: no communicator, this handle  */
                         /* serves nc_matvec_emulated only (single-GPU tests of the partition)  */
  int32_t check_separation; /* 1: verify the 3 eps separation (NC_ESEP on failure); 0: trust input */
} nc_opts;

typedef struct nc_stats_t {
  int64_t N, row_begin, row_count;
  int32_t K, Kstar, p, mode, world, rank;
  int64_t matvecs;              /* matvecs applied since setup                                     */
  double pairs_per_matvec;      /* kernel evaluations G(x,y) rho per matvec on this rank           */
  double gemm_flops_per_matvec; /* 2 p K n + 2 K Kstar n on this rank (n = row_count)              */
  double ms_last[8];            /* per-stage device ms of the last matvec run with nc_time_stages:  */
                                /*   [0] T-apply  [1] all-gather  [2] direct pair sums  [3] P-apply */
                                /*   [4] hier k_pairs_grid alone (steps 2-3 on incoming grids)      */
                                /*   [5] hier grid reduce + transform + near list + step 4          */
                                /*   [6] total  [7] hier grid reduction alone (k_reduce_chunks)     */
  int32_t tree_levels;          /* NC_HIER: depth L of the sphere quadtree                         */
  int64_t tree_groups;          /* NC_HIER: number of non-empty boxes over all levels              */
  double hier_grid_pairs;       /* NC_HIER: pair evaluations on incoming grids per matvec (steps 2-3) */
  double hier_near_pairs;       /* NC_HIER: pair evaluations at Zernike nodes (near lists)          */
  double hier_interp_terms;     /* NC_HIER: node x coefficient terms of the step-4 interpolation    */
  int64_t hier_grid_points;     /* NC_HIER: incoming-grid points held by this rank                  */
  int64_t hier_grid_units;      /* NC_HIER: step-2/3 work units (CTAs) per matvec                   */
  double device_bytes;          /* device memory held by the handle                                */
  int32_t launches_per_matvec;  /* kernels this library launched in the last nc_matvec              */
  double gmres_ortho_ms;        /* GMRES CGS2 orthogonalisation device ms summed over the iterations */
  double gmres_ortho_bytes;     /*   run with nc_time_stages on, and its algorithmic HBM bytes       */
  int64_t gmres_ortho_iters;    /*   (iterations counted)                                          */
  double pair_fp64_flops_direct; /* FP64 flops executed per pair (2 per DFMA, 1 per DMUL/DADD; SASS  */
  double pair_fp64_inst_direct;  /*   count, verified with ncu) and FP64-pipe instructions per pair,  */
  double pair_fp64_flops_grid;   /*   for the direct / near-list kernels and for k_pairs_grid's       */
  double pair_fp64_inst_grid;    /*   variant in use (kind-dependent)                                */
  double hier_grid_fill;         /* NC_HIER: grid pairs / (work-unit thread slots x sources x p)     */
  double hier_grid_warp_fill;    /* NC_HIER: grid pairs / (active-warp thread slots x sources x p)   */
  int32_t grid_variant[8];       /* NC_HIER: k_pairs_grid variant in use {warps or threads per CTA,  */
                                 /*   targets per thread, unroll, stage, far form, tma, minb, persist} */
  double hier_unit_points;       /* NC_HIER: sum over work units of their grid points: the partial   */
                                 /*   values k_pairs_grid writes and k_reduce_chunks reads per matvec  */
  int32_t proxy_n;               /* NC_HIER: step-4 proxies per patch (0: every level at the nodes; R36) */
  double proxy_kappa;            /*   far-level threshold D / h of the rule (nc_proxy_rule)           */
  double proxy_far_frac;         /*   (patch, multi-member level with grids) pairs evaluated at the    */
                                 /*   proxies / all such pairs                                         */
} nc_stats_t;

typedef struct nc_handle nc_handle;

/* Build the per-layout state (Step 2): frames R_i, global Zernike and skeleton
 * nodes, and (NC_HIER) the sphere quadtree, interaction lists and incoming grids.
 *   kind    NC_INTERIOR | NC_EXTERIOR
 *   N       number of patches (>= 1)
 *   centers host, N x 3, unit vectors, caller order
 *   eps     patch radius (arc length, > 0)
 * Frames follow the ABI rule (R8): e1 = normalize(xhat - (xhat.c)c) (yhat instead of xhat
 * when |c.xhat| > 0.9), e2 = c x e1, R_i = [e1 e2 c_i].
 * Errors: NC_EINVAL, NC_ESEP, NC_ENOMEM, NC_ECUDA, NC_ENCCL.  On error *h is set to NULL. */
int nc_setup(nc_handle** h, int kind, int64_t N, const double* centers, double eps, const nc_tables* tab,
             const nc_opts* opt);

/* This rank's shard and the internal order.  perm (host, N entries, nullable): perm[internal] =
 * caller index.  Errors: NC_EINVAL (null handle). */
int nc_partition(const nc_handle* h, int64_t* row_begin, int64_t* row_count, int64_t* perm);

/* y = (I + A_off) x on this rank's rows (eq:sysmatapply).  x, y: device, row_count x K, must not
 * alias.  stream: cudaStream_t (NULL = legacy default stream).  Asynchronous with respect to the
 * host for world == 1; collective (one all-gather) for world > 1.  Errors: NC_EINVAL, NC_ECUDA,
 * NC_ENCCL. */
int nc_matvec(nc_handle* h, const double* x, double* y, void* stream);

/* Rank emulation (handle set up with world > 1 and nccl_id == NULL): the same map for this rank's rows, with
 * the all-gather replaced by computing every rank's outgoing records from the FULL input.
 *   x_all  device, N x K (all rows, internal order);  y  device, row_count x K (this rank's rows)
 * Exercises the rank's partition (row range, work-weighted cut, redundant straddling groups, near lists) on one
 * GPU.  Errors: NC_EINVAL, NC_ECUDA. */
int nc_matvec_emulated(nc_handle* h, const double* x_all, double* y, void* stream);

/* Same map with HOST buffers (row_count x K each): copies x in, applies, copies y out, synchronizes.
 * This is the end-to-end entry point timed as "e2e" by bench.py. */
int nc_matvec_host(nc_handle* h, const double* x_host, double* y_host);

/* Unrestarted GMRES for (I + A_off) x = b, x0 = 0, classical Gram-Schmidt with
 * one full re-orthogonalisation (CGS2), stop when the implicit residual ||b - A x|| / ||b|| <= rtol.
 *   b     device, row_count x K, or NULL for the physical right-hand side b_i = P 1 (eq:opinteqnsdisc)
 *   x     device, row_count x K (output)
 *   iters host (output), number of iterations (= matvecs) performed
 *   hist  host, max_iter + 1 doubles or NULL: relative residual after 0..iters iterations
 * Synchronizes the stream.  Errors: NC_ENOCONV (x = last iterate), NC_EINVAL, NC_ECUDA, NC_ENCCL. */
int nc_gmres(nc_handle* h, const double* b, double rtol, int max_iter, double* x, int* iters, double* hist,
             void* stream);

/* Read-out (eq:getI): I_sigma = I . sum_i x_i over all ranks (collective), then
 * value = mu = 1/(3 I_sigma) - 3/5 (interior, eq:mufromsigma2) or J = -4 pi I_sigma (exterior,
 * DESIGN.md R2).  x: device, row_count x K.  I_sigma, value: host.  Synchronizes.
 * Errors: NC_ESTATE when the interior I_sigma <= 0 (the Lemma of PAPER.md:579-590 needs I_sigma != 0). */
int nc_flux_or_mfpt(nc_handle* h, const double* x, double* I_sigma, double* value);

/* Off-surface field of the solution (NEXT-3): the single-layer potential
 *   interior  v(p) = int G_I(p, x') sigma dS   (eq:intBVPansatz; the MFPT is
 *             vbar = (v - 1) / (3 D) + (1 - |p|^2) / 6 with D = -I_sigma, eq:vtilde PAPER.md:533-536)
 *   exterior  u(p) = int G_E(p, x') sigma dS   (eq:urep)
 * with the off-surface Green's functions eq:Gintoffsurface / eq:Gextoffsurface and each
 * patch's density in its compressed outgoing representation (skeleton nodes, rho_j = T fhat_j, eq:outgoingcompressed).
 *   x_all  device, N x K: the coefficients of ALL patches, internal order (world 1: the nc_gmres solution)
 *   pts    host, n_pts x 3 (row-major); interior: every |p| < 1, exterior: every |p| > 1
 *   out    host, n_pts: the potential at each point
 *   dmin   host, n_pts or NULL: the distance from each point to the nearest skeleton node
 * The compressed representation is valid only away from the patches: every point must be at least 3 eps from every
 * skeleton node (the skeleton is certified >= 2 eps from a patch centre; R27).  Uses the handle's stream
 * and synchronizes.  Errors: NC_EINVAL (null argument, a point on the wrong side of the sphere or closer than
 * 3 eps to a skeleton node: out and dmin are still written), NC_ENOMEM, NC_ECUDA. */
int nc_field(nc_handle* h, const double* x_all, int64_t n_pts, const double* pts, double* out, double* dmin);

/* Near-field table of a patch radius (NEXT-3; nc_tables/nearfield.py): the one-patch solver's radial panels and
 * basis densities sigma_a(t), canonical frame.  n_r = npan k. */
typedef struct nc_near_tables {
  int32_t npan, k;           /* panels; Gauss nodes per panel (k <= 32)                                   */
  const double* edges;       /* npan + 1 panel breakpoints in t (arc length from the centre), 0 .. eps     */
  const double* t;           /* n_r radial nodes, panel-major (Gauss-Legendre; Gauss-Jacobi on the last)    */
  const double* w;           /* n_r weights: int_0^eps F(t) sigma(t) sin t dt = sum_j w_j F(t_j) sigma(t_j) */
  const double* sigma;       /* K x n_r: sigma_a(t_j) of basis column a (row-major)                       */
  const int32_t* m;          /* K: angular order of column a (0 .. 15)                                     */
  const int32_t* c;          /* K: +1 cos(m theta), -1 sin(m theta)                                        */
} nc_near_tables;

/* NEXT-3 at any off-surface point, including the layer near the patches where the compressed skeleton is not valid
 * (PAPER.md:2069-2097 plot the MFPT on the sphere of radius 1 - eps/5): v (interior) or u (exterior) as in nc_field,
 * with the patches whose centre is closer than 4 eps to a point evaluated from their density sigma = B fhat
 * (eq:recoversig) by panel-refined radial x converged trapezoid angular quadrature
 * (csrc/nearfield.cu), the others from their compressed skeleton.
 *   x_all  device, N x K (all patches, internal order; world 1: the nc_gmres solution)
 *   pts    host, n_pts x 3: interior |p| < 1, exterior |p| > 1; a point within 4 eps of a patch centre must be at
 *          least eps / 100 off the sphere (the angular rule's resolution limit)
 *   nt     the near-field table of this eps (nc_tables/nearfield.py)
 *   out    host, n_pts (output): the potential
 *   mfpt   host, n_pts or NULL (output, interior only): the mean first passage time
 *          vbar = (v - 1) / (3 D) + (1 - |p|^2) / 6, D = -I_sigma (eq:vtilde PAPER.md:533-536, Lemma PAPER.md:556-566),
 *          I_sigma = I . sum_i fhat_i from x_all (eq:getI)
 *   n_near host or NULL (output): the number of (point, near patch) pairs evaluated by quadrature
 * Synchronous.  Errors: NC_EINVAL (bad argument, a point on the wrong side or too close to the sphere near a patch,
 * or mfpt requested for the exterior problem), NC_ENOMEM, NC_ECUDA. */
int nc_field_near(nc_handle* h, const double* x_all, int64_t n_pts, const double* pts, const nc_near_tables* nt,
                  double* out, double* mfpt, int64_t* n_near);

/* L2 residual diagnostic (NEXT-4): the paper's accuracy metric eq:l2res,
 *   res_i = || S sigma_i + sum_{j != i} S_ij sigma_j - 1 ||_{L2(Gamma_i)} / |Gamma_i|
 * for n_sel listed patches, by quadrature on a residual grid that is independent of the solve's grids
 * (PAPER.md:1720-1724): S sigma_i = res_S fhat_i (the self-patch potential of the basis solutions, a per-eps table
 * built by nc_tables/residual.py), the other patches through their compressed outgoing representation.
 *   x_all     device, N x K: the coefficients of ALL patches, internal order (world 1: the nc_gmres solution)
 *   patches   host, n_sel caller patch indices (0 <= index < N)
 *   res_rhat  host, n_res x 3: the residual grid in the canonical frame (patch centre +z, theta = 0 along +x)
 *   res_w     host, n_res: quadrature weights of int_Gamma f dS (their sum is |Gamma|)
 *   res_S     host, n_res x K row-major
 *   res       host, n_sel (output);  pointwise  host, n_sel x n_res or NULL (output: the residual at each point)
 * Uses the handle's stream and synchronizes.  Errors: NC_EINVAL (bad argument or index), NC_ENOMEM, NC_ECUDA. */
int nc_residual(nc_handle* h, const double* x_all, int n_sel, const int64_t* patches, int n_res,
                const double* res_rhat, const double* res_w, const double* res_S, double* res, double* pointwise);

/* Density recovery (NEXT-3; eq:recoversig PAPER.md:797-807): sigma_i = B fhat_i, the density of
 * each listed patch at the one-patch solver's fine grid (B: n_f x K, the per-eps basis solutions sampled there,
 * nc_tables onepatch.fine_grid; with the fine weights w, w . sigma_i = I . fhat_i = int sigma_i dS).
 *   x_all   device, N x K (all patches, internal order);  patches  host, n_sel caller indices
 *   B       host, n_f x K row-major;  sigma  host, n_sel x n_f (output)
 * One fp64 tensor-core GEMM.  Synchronizes.  Errors: NC_EINVAL, NC_ENOMEM, NC_ECUDA. */
int nc_density(nc_handle* h, const double* x_all, int n_sel, const int64_t* patches, int n_f, const double* B,
               double* sigma);

/* Step-1 table build, GPU part (NEXT-1): the Gaussian sketch of the interpolative decomposition
 * that compresses a patch's outgoing field (Step 1(b) PAPER.md:1295-1299; nc_tables/skeleton.py)
 *   Y = Omega A,   A_{tf} = G(x^t_t, x^f_f)   (on-surface G of `kind`, eq:Gintonsurface / eq:Gextonsurface)
 *   train  host, n_train x 3 training points (far-field region);  fine  host, n_fine x 3 fine-grid points
 *   omega  host, l x n_train (row-major) Gaussian test matrix;    Y     host, l x n_fine (output)
 * Needs no handle: allocates on `device`, generates A in HBM (n_fine x n_train doubles), one fp64 tensor-core GEMM,
 * synchronous.  Errors: NC_EINVAL, NC_ENOMEM, NC_ECUDA. */
int nc_id_sketch(int kind, int device, int64_t n_train, const double* train, int64_t n_fine, const double* fine,
                 int l, const double* omega, double* Y);

/* Step-1 table build, GPU part (NEXT-1): the modal kernels of the one-patch solver (§8.2;
 * nc_tables/kernel.py modal), G_m(t, t') = (1/pi) int_0^pi G(d) cos(m phi) dphi for m = 0..M at npairs (t, t')
 * pairs, d^2 = 4 sin^2((t - t')/2) + 4 sin t sin t' sin^2(phi/2), by the caller's phi rule:
 *   t, tp  host, npairs radii (geodesic, in [0, pi]);  phi, wphi  host, nphi nodes and weights on [0, pi]
 *   out    host, npairs x (M+1) row-major (output)
 * The integrand matrix is generated in HBM (npairs x nphi) and contracted with the cosine weights by one fp64
 * tensor-core GEMM.  Synchronous.  Errors: NC_EINVAL, NC_ENOMEM, NC_ECUDA. */
int nc_modal_kernels(int kind, int device, int64_t npairs, const double* t, const double* tp, int M, int nphi,
                     const double* phi, const double* wphi, double* out);

/* Counters and the last matvec's per-stage device times.  nc_time_stages(h, 1) makes the next
 * matvecs record per-stage CUDA events on the matvec's stream (no host synchronisation inside nc_matvec);
 * nc_stats waits for the last recorded matvec's events and converts them to ms_last. */
int nc_stats(const nc_handle* h, nc_stats_t* out);
int nc_time_stages(nc_handle* h, int enable);

/* Debug/introspection (NC_HIER): number of (level, target group, source group) interaction-list
 * entries and leaf-neighbour entries, copied to host arrays of 3 int64 per entry when non-NULL.
 * Used by the exactly-once pair-coverage audit (tests/test_hier.py). */
int nc_tree_lists(const nc_handle* h, int64_t* n_ilist, int64_t* ilist, int64_t* n_nbr, int64_t* nbr,
                  int64_t* box_of_patch /* L+1 x N, nullable */);

/* Introspection (NC_HIER): the number of near-list source patches (R12: sources evaluated directly at the
 * patch's Zernike nodes) of each of this rank's rows, internal order.  counts: host, row_count int64.  Used by the
 * parity tests to pick rows whose near lists are not empty.  Errors: NC_EINVAL, NC_ESTATE (not NC_HIER). */
int nc_near_counts(const nc_handle* h, int64_t* counts);

/* Diagnostic: the grid kernel's pair evaluation (far form `far` = 5, 7 or 8 of k_pairs_grid_w,
 * kind NC_INTERIOR / NC_EXTERIOR) run in isolation -- sources in registers, no staging, no barriers, 16 independent
 * chains per thread, ctas_per_sm CTAs of 256 threads per SM -- on the current device.  Returns the best device
 * time of three launches (ms, host) and the warp-pair evaluations each launch performs (host), so that the caller
 * can express the loop body's cost in SM-sub-partition cycles per warp-pair at the measured clock.  Synchronous.
 * Errors: NC_EINVAL (bad arguments, unsupported far form, launch failure). */
int nc_pair_mix(int kind, int far, int ctas_per_sm, double* ms, double* warp_pairs);

/* Host-only helper (no GPU needed): the contiguous row partition used by nc_setup.  Rank r of `world` gets
 * rows [begin[r], begin[r] + count[r]) of the internal order, cut so that the prefix sums of (weights[i] + 1)
 * are split evenly (weights NULL = equal split, as in NC_DIRECT; NC_HIER passes its per-patch work).
 * begin, count: host arrays of `world` entries.  Errors: NC_EINVAL. */
int nc_split_rows(const double* weights, int64_t N, int world, int64_t* begin, int64_t* count);

/* Host-only helper (no GPU needed): the step-4 proxy rule of NC_HIER handles (R36; PAPER.md:1381-1397,
 * "evaluate the interpolant ... at the Zernike sampling nodes", carried out for far levels through proxy points).
 * zhat: host, Kstar x 3 canonical node unit vectors (the tables' zhat).  The proxies are a polar point set on the
 * node disk of radius h = 1.01 max |(zhat_x, zhat_y)|: the centre plus nring rings at r_k = h cos((k + 1/2) pi /
 * (2 nring)), max(6, round(cphi r_k / h)) angles each (odd rings offset by half a step), lifted to the unit sphere.
 * Int maps values at the proxies to the nodes by least squares in the Chebyshev-product basis of total degree <= deg
 * (it reproduces every such polynomial exactly).  kappa: the smallest D / h (multiples of 1/8 in [1.5, 64]) from
 * which point sources at distance D h give an interpolation error below tol (relative to max 2/d over the nodes);
 * HUGE_VAL if none.  Outputs (host): pts (n x 3, nullable), Int (Kstar x n row-major, nullable), kappa, h.
 * Returns n (> 0) or a negative error code: NC_EINVAL (bad arguments, rank-deficient basis, n > nmax). */
int nc_proxy_rule(const double* zhat, int Kstar, int deg, int nring, double cphi, double tol, int nmax,
                  double* pts, double* Int, double* kappa, double* h);

/* world > 1 bootstrap: rank 0 creates the 128-byte NCCL unique id (host buffer), the caller broadcasts it
 * (e.g. torch.distributed) and passes it as nc_opts.nccl_id on every rank.  NC_EUNSUP without NCCL. */
int nc_nccl_unique_id(void* id_out);

void nc_destroy(nc_handle* h);
const char* nc_last_error(void);
const char* nc_version(void);

#ifdef __cplusplus
}
#endif
#endif /* NC_H_ */
