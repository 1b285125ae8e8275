// hier.cu -- the hierarchical O(N log N) matvec (SURVEY.md §8(a) a0, a3-a5; §7.2-§8, :1176-1415).
//
// Setup (Step 2), on device:
//   * keys: project each centre by the ray from the origin onto the cube [-1,1]^3; face by the
//     largest |coordinate| (ties x > y > z), Morton-interleaved cell indices at kLmax levels -> 51-bit key;
//   * sort (CUB radix sort) -> internal patch order; depth L = the first level at which all non-empty boxes hold one
//     patch (adjacent-key separation levels, max-reduced) -- DESIGN.md reading R11 (uniform depth, pruned);
//   * boxes per level by run-length of key prefixes (flags + CUB scan): every box is a contiguous patch range;
//   * neighbours: the 8 cells around a box, folded across cube edges (7 at cube corners),
//     looked up by binary search; interaction lists: children of the parent's neighbours (parent included) that are
//     not neighbours; level 0 = the six faces under a virtual root (opposite faces interact);
//   * bounding circles: Badoiu-Clarkson iterations for the smallest cap around member centres,
//     radius padded by eps (reading R14).
// Host bookkeeping: for every (group, source patch) pair of the interaction list (and leaf neighbours, step 3,
// PAPER.md:1364-1375) decide incoming grid vs direct near-list evaluation (skeleton validity > 2 eps, PAPER.md:1057;
// DESIGN.md reading R12, with a cost model; up to three grids per group, R24), size each grid from its nearest grid
// source with ring-adaptive angular counts filled to whole warps (R26b), and build the warp-level
// work units (64 grid points x a slice of sources, each with the outgoing rung valid at its own gap, R22).
//
// Matvec (Step 3): K1 (api.cu) -> k_pairs_grid_w (steps 2-3, direct.cu) -> k_reduce_chunks ->
// k_transform (samples -> parity-restricted Chebyshev-Fourier coefficients) -> k_pairs_near ->
// k_interp + k_interp_sep (step 4: every group's expansion at its members' Zernike nodes, summed over levels; R26,
// R26c) -> K3 (api.cu).
#include <cub/cub.cuh>
#include <omp.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <cmath>
#include <numeric>
#include <string>
#include <vector>

#include "hier.cuh"
#include "pairs.cuh"

namespace nc {

constexpr int kLmax = 24;
constexpr int kSliceMax = 32;          // source patches per grid work unit
constexpr int kMaxGrids = 4;           // incoming grids per group (source bands by distance; R24)
constexpr int kDefaultGrids = 3;       // NC_MAX_GRIDS overrides (1..kMaxGrids)
constexpr int kGridCutQuantiles = 48;  // candidate cut points of the multi-grid search
constexpr double kBetaMin = 1.45;      // smallest source distance / circle radius served by a grid
constexpr double kCostNear = 1.0, kCostInterp = 0.15, kCostTransform = 0.1;   // grid-vs-near cost model (grid-pair units)
constexpr double kGridTolFactor = 1000.0;  // per-grid tolerance / requested precision (calibrated: DESIGN.md R21; 1500 withdrawn: the physical solve's L2 residual follows this factor)

struct ChunkRec {
  int64_t pt0;
  int64_t u0;
  int32_t npt;
  int32_t nu;
};

struct HierState {
  int L = 0;
  int64_t ngroups = 0;
  std::vector<int64_t> lvl_off;     // L+2
  std::vector<int64_t> gkey;
  std::vector<int32_t> gfirst, glast, glevel;
  std::vector<int32_t> nbr;         // 8 per group
  std::vector<int64_t> il_off;
  std::vector<int32_t> il;
  std::vector<double> gc, gR;       // circle centre (3/group), radius
  std::vector<int32_t> pgroup;      // (L+1) x N
  std::vector<int64_t> keys;        // sorted keys (internal order)
  // incoming grids (up to kMaxGrids per group; arrays indexed by grid id)
  int64_t ngrids = 0;
  std::vector<int64_t> ggrid0;      // G+1: grids of group g are [ggrid0[g], ggrid0[g+1])
  std::vector<int32_t> gnr, gna, grid_group;
  std::vector<int64_t> goff, coff;  // ngrids+1 point / coefficient offsets (0-sized for other ranks' groups)
  std::vector<int64_t> rbase;       // ngrids+1: grid k's ring offsets are roff[rbase[k] .. rbase[k] + n_r]
  std::vector<int32_t> roff;        // per local grid: n_r + 1 point offsets of its rings (ring-adaptive, R26b)
  int64_t* d_rbase = nullptr;
  int32_t* d_roff = nullptr;
  int64_t Q = 0, C = 0;
  int qmax = 0, cmax = 0, pmax = 0, namax = 0, nrmax = 0, cgroupmax = 0;
  std::vector<int32_t> grid_ids;    // grids with points on this rank
  // device
  int64_t* d_keys = nullptr;
  double* d_gframe = nullptr;
  double* d_gR = nullptr;
  double* d_gRinv = nullptr;        // 1 / R per group (step 4: x = arc / R)
  double2* d_twtab = nullptr;       // step 4a twiddles: (cos, sin)(2 pi l / n) at n (n - 1) / 2 + l, n <= namax
  int asin_terms = 0;               // step 4 node geometry: terms of the asin series (0: atan2 per node)
  int32_t *d_gnr = nullptr, *d_gna = nullptr;
  int64_t *d_goff = nullptr, *d_coff = nullptr;
  int32_t* d_grid_ids = nullptr;
  int* d_counter = nullptr;         // work counter of the persistent grid kernel
  double2* d_ftab = nullptr;        // far log table of the grid kernel (FAR >= 2)
  // separable step 4 for single-member groups (k_interp_sep): node rings of the canonical Zernike nodes
  bool sep_nodes = false;           // the nodes lie on rings (detected from the tables; NC_INTERP_SEP=0 disables)
  int nring = 0;
  std::vector<double> ring_t;       // geodesic radius of each ring
  std::vector<int32_t> node_ring;   // ring of each node
  std::vector<double> node_cs;      // (cos, sin) of each node's angle in the canonical frame
  uint8_t* d_gsep = nullptr;        // group evaluated by k_interp_sep
  int32_t* d_work_sep = nullptr;    // local patches with at least one such level
  int64_t nwork_sep = 0;
  double* d_ring_t = nullptr;
  int32_t* d_node_ring = nullptr;
  double* d_node_cs = nullptr;
  double sep_terms = 0.0;           // node x coefficient terms those groups represent (part of interp_terms)
  double interp_lt = 0.0;           // ln(1 / grid tol) for the per-node order truncation of step 4 (R26c; 0: off)
  // step 4 through patch-local proxies for far levels (R36, proxy.cu)
  // up to kMaxProxyRules rules, by point count ascending (threshold descending); rule r serves the (patch, level)
  // pairs whose nearest grid source is >= kh[r] away and < kh[r - 1]; nearer ones stay at the nodes
  int nprule = 0;
  int proxy_n = 0;                  // points of the smallest rule (0: every level evaluated at the Zernike nodes)
  double proxy_kappa = 0.0;         // the smallest threshold D / h in use (calibrated, proxy_rule_build)
  struct PRule {
    int n = 0;
    double kh = 0.0;                // threshold (arc)
    double *ptx = nullptr, *pty = nullptr, *ptz = nullptr;   // rc x n proxies (scaled by 1/2)
    double* V = nullptr;            // rc x n: the rule's levels summed at its proxies
    double* Int = nullptr;          // Ks x n: proxies -> nodes
  } prule[3];
  uint64_t* d_pcode = nullptr;      // per local patch, 2 bits per level: 0 nodes, r + 1 rule r
  int32_t* d_pwork1 = nullptr;      // local patches with a level evaluated at the nodes (the first pass's CTAs)
  int64_t npwork1 = 0;
  double proxy_pairs = 0.0, proxy_far = 0.0;   // (patch, level) pairs with grids; of which far (host count)
  FarTable ftab;
  int32_t* d_grid_group = nullptr;
  int64_t* d_ggrid0 = nullptr;
  double *d_gx = nullptr, *d_gy = nullptr, *d_gz = nullptr, *d_gval = nullptr, *d_gcoef = nullptr;
  GridUnit* d_units = nullptr;
  int64_t nunits = 0;
  GridVariant gv = kGridVariantDefault;   // the grid kernel's variant (grid_variant_for(precision), R32)
  int upts = 256;                   // grid points per work unit (grid_unit_points(gv))
  int32_t* d_srclist = nullptr;
  double* d_part = nullptr;
  ChunkRec* d_chunks = nullptr;
  int64_t nchunks = 0;
  int64_t* d_gch0 = nullptr;        // per grid: first chunk (NG + 1)
  bool fuse_reduce = false;         // k_transform_w sums the partials itself (no k_reduce_chunks, no grid values)
  bool transform_w = true;          // NC_TRANSFORM=0: k_reduce_chunks + the CTA-per-grid transform (read at setup)
  int32_t* d_work_near = nullptr;
  int64_t nwork_near = 0;
  int64_t* d_near_off = nullptr;
  int32_t* d_near = nullptr;
  int32_t* d_pgl = nullptr;         // (L+1) x row_count group ids of local patches
  double *d_tx = nullptr, *d_ty = nullptr, *d_tz = nullptr;
  double *d_udir = nullptr, *d_u = nullptr;
  double pairs_grid = 0, pairs_near = 0, interp_terms = 0, slot_pairs = 0, warp_slot_pairs = 0;
  double unit_points = 0;           // sum of npt over the work units (partial values written / read back per matvec)
  double bytes = 0;
  std::vector<int32_t> near_count;      // host copy for nc_near_counts: near-list sources per local patch
  std::vector<int64_t> ilist_entries;   // host copies for nc_tree_lists: (level, target group, source group)
  std::vector<int64_t> nbr_entries;
};

// ------------------------------------------------------------------------------------------------
// device helpers: cube faces, Morton codes
// ------------------------------------------------------------------------------------------------
__host__ __device__ inline void face_uv(double x, double y, double z, int& f, double& u, double& v) {
  double ax = fabs(x), ay = fabs(y), az = fabs(z);
  int a = (ax >= ay && ax >= az) ? 0 : (ay >= az ? 1 : 2);   // ties: x > y > z (R15)
  double c[3] = {x, y, z};
  double m = fabs(c[a]);
  f = 2 * a + (c[a] < 0.0 ? 1 : 0);
  u = c[(a + 1) % 3] / m;
  v = c[(a + 2) % 3] / m;
}

__host__ __device__ inline uint64_t part1by1(uint64_t x) {
  x &= 0xFFFFFFull;
  x = (x | (x << 16)) & 0x0000FFFF0000FFFFull;
  x = (x | (x << 8)) & 0x00FF00FF00FF00FFull;
  x = (x | (x << 4)) & 0x0F0F0F0F0F0F0F0Full;
  x = (x | (x << 2)) & 0x3333333333333333ull;
  x = (x | (x << 1)) & 0x5555555555555555ull;
  return x;
}
__host__ __device__ inline uint32_t compact1by1(uint64_t x) {
  x &= 0x5555555555555555ull;
  x = (x | (x >> 1)) & 0x3333333333333333ull;
  x = (x | (x >> 2)) & 0x0F0F0F0F0F0F0F0Full;
  x = (x | (x >> 4)) & 0x00FF00FF00FF00FFull;
  x = (x | (x >> 8)) & 0x0000FFFF0000FFFFull;
  x = (x | (x >> 16)) & 0x00000000FFFFFFFFull;
  return (uint32_t)x;
}
__host__ __device__ inline int64_t cell_prefix(int f, uint32_t iu, uint32_t iv, int lvl) {
  return ((int64_t)f << (2 * lvl)) | (int64_t)((part1by1(iu) << 1) | part1by1(iv));
}
__host__ __device__ inline uint32_t clamp_cell(double u, int lvl) {
  double n = (double)(1u << lvl);
  double c = floor((u + 1.0) * 0.5 * n);
  if (c < 0) c = 0;
  if (c > n - 1) c = n - 1;
  return (uint32_t)c;
}

__global__ void k_keys(const double* __restrict__ c, int64_t N, int64_t* __restrict__ key, int64_t* __restrict__ idx) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= N) return;
  int f;
  double u, v;
  face_uv(c[3 * i], c[3 * i + 1], c[3 * i + 2], f, u, v);
  key[i] = cell_prefix(f, clamp_cell(u, kLmax), clamp_cell(v, kLmax), kLmax);
  idx[i] = i;
}

// separation level of adjacent sorted keys: first level at which they fall in different boxes
__global__ void k_sep(const int64_t* __restrict__ key, int64_t N, int* __restrict__ sep, int* __restrict__ dup) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i + 1 >= N) return;
  uint64_t a = (uint64_t)key[i], b = (uint64_t)key[i + 1];
  int s;
  if (a == b) {
    s = kLmax;
    *dup = 1;
  } else if ((a >> (2 * kLmax)) != (b >> (2 * kLmax))) {
    s = 0;
  } else {
    uint64_t d = a ^ b;
    int hb = 63 - __clzll((long long)d);        // highest differing bit (< 2*kLmax)
    s = (2 * kLmax - 1 - hb) / 2 + 1;
  }
  sep[i] = s;
}

__global__ void k_box_flags(const int64_t* __restrict__ key, int64_t N, int lvl, int* __restrict__ flag) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= N) return;
  int sh = 2 * (kLmax - lvl);
  flag[i] = (i == 0 || (key[i] >> sh) != (key[i - 1] >> sh)) ? 1 : 0;
}

// neighbours of every group (same level, folded across cube edges)
__global__ void k_neighbors(const int64_t* __restrict__ gkey, const int64_t* __restrict__ lvl_off, int L,
                            int64_t ngroups, int32_t* __restrict__ nbr) {
  int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= ngroups) return;
  int lvl = 0;
  while (lvl < L && g >= lvl_off[lvl + 1]) ++lvl;
  const int64_t key = gkey[g];
  const int f = (int)(key >> (2 * lvl));
  const uint64_t mort = (uint64_t)key & ((lvl == 0) ? 0ull : ((1ull << (2 * lvl)) - 1));
  const int iu = (int)compact1by1(mort >> 1), iv = (int)compact1by1(mort);
  const int n = 1 << lvl;
  const int a = f / 2;
  const double sgn = (f & 1) ? -1.0 : 1.0;
  const int64_t lo = lvl_off[lvl], hi = lvl_off[lvl + 1];
  int cnt = 0;
  for (int du = -1; du <= 1; ++du)
    for (int dv = -1; dv <= 1; ++dv) {
      if (du == 0 && dv == 0) continue;
      double u = (2.0 * (iu + du) + 1.0) / n - 1.0, v = (2.0 * (iv + dv) + 1.0) / n - 1.0;
      bool ou = fabs(u) > 1.0, ov = fabs(v) > 1.0;
      if (ou && ov) continue;                                    // across a cube corner: no cell
      double P[3];
      P[a] = sgn;
      P[(a + 1) % 3] = u;
      P[(a + 2) % 3] = v;
      if (ou) {
        double e = fabs(u) - 1.0;
        P[(a + 1) % 3] = (u > 0) ? 1.0 : -1.0;
        P[a] = sgn * (1.0 - e);
      }
      if (ov) {
        double e = fabs(v) - 1.0;
        P[(a + 2) % 3] = (v > 0) ? 1.0 : -1.0;
        P[a] = sgn * (1.0 - e);
      }
      int f2;
      double u2, v2;
      face_uv(P[0], P[1], P[2], f2, u2, v2);
      int64_t want = cell_prefix(f2, clamp_cell(u2, lvl), clamp_cell(v2, lvl), lvl);
      // binary search in [lo, hi)
      int64_t l = lo, r = hi;
      while (l < r) {
        int64_t m = (l + r) >> 1;
        if (gkey[m] < want) l = m + 1; else r = m;
      }
      if (l < hi && gkey[l] == want && l != g) {
        bool dupn = false;
        for (int k = 0; k < cnt; ++k) dupn = dupn || (nbr[8 * g + k] == (int32_t)l);
        if (!dupn && cnt < 8) nbr[8 * g + cnt++] = (int32_t)l;
      }
    }
  for (int k = cnt; k < 8; ++k) nbr[8 * g + k] = -1;
}

__device__ inline int64_t lower_bound_key(const int64_t* gkey, int64_t lo, int64_t hi, int64_t want) {
  while (lo < hi) {
    int64_t m = (lo + hi) >> 1;
    if (gkey[m] < want) lo = m + 1; else hi = m;
  }
  return lo;
}

// interaction lists: pass 0 counts, pass 1 fills (offsets from an exclusive scan of the counts)
__global__ void k_ilist(const int64_t* __restrict__ gkey, const int64_t* __restrict__ lvl_off, int L,
                        int64_t ngroups, const int32_t* __restrict__ nbr, const int32_t* __restrict__ gfirst,
                        const int32_t* __restrict__ pgroup, int64_t N, const int64_t* __restrict__ off,
                        int64_t* __restrict__ cnt, int32_t* __restrict__ out) {
  int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= ngroups) return;
  int lvl = 0;
  while (lvl < L && g >= lvl_off[lvl + 1]) ++lvl;
  const int32_t* mynb = nbr + 8 * g;
  int64_t c = 0, w = off ? off[g] : 0;
  auto emit = [&](int64_t child) {
    if (child == g) return;
    for (int k = 0; k < 8; ++k)
      if (mynb[k] == (int32_t)child) return;
    if (off) out[w + c] = (int32_t)child;
    ++c;
  };
  if (lvl == 0) {
    for (int64_t ch = lvl_off[0]; ch < lvl_off[1]; ++ch) emit(ch);
  } else {
    const int64_t parent = pgroup[(int64_t)(lvl - 1) * N + gfirst[g]];
    int32_t pn[9];
    pn[0] = (int32_t)parent;
    for (int k = 0; k < 8; ++k) pn[k + 1] = nbr[8 * parent + k];
    for (int k = 0; k < 9; ++k) {
      if (pn[k] < 0) continue;
      const int64_t pk = gkey[pn[k]];
      const int64_t lo = lower_bound_key(gkey, lvl_off[lvl], lvl_off[lvl + 1], pk << 2);
      const int64_t hi = lower_bound_key(gkey, lvl_off[lvl], lvl_off[lvl + 1], (pk << 2) + 4);
      for (int64_t ch = lo; ch < hi; ++ch) emit(ch);
    }
  }
  if (!off) cnt[g] = c;
}

__device__ inline double arc_between(double ax, double ay, double az, double bx, double by, double bz) {
  double cx = ay * bz - az * by, cy = az * bx - ax * bz, cz = ax * by - ay * bx;
  return atan2(sqrt(cx * cx + cy * cy + cz * cz), ax * bx + ay * by + az * bz);
}

// smallest enclosing cap of member centres (Badoiu-Clarkson), one warp per group
__global__ void k_circles(const double* __restrict__ cen, const int32_t* __restrict__ gfirst,
                          const int32_t* __restrict__ glast, int64_t ngroups, double eps, double* __restrict__ gc,
                          double* __restrict__ gR) {
  const int64_t g = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (g >= ngroups) return;
  const int64_t a = gfirst[g], b = glast[g];
  double sx = 0, sy = 0, sz = 0;
  for (int64_t i = a + lane; i < b; i += 32) {
    sx += cen[3 * i]; sy += cen[3 * i + 1]; sz += cen[3 * i + 2];
  }
  for (int o = 16; o; o >>= 1) {
    sx += __shfl_xor_sync(0xffffffffu, sx, o);
    sy += __shfl_xor_sync(0xffffffffu, sy, o);
    sz += __shfl_xor_sync(0xffffffffu, sz, o);
  }
  double nrm = sqrt(sx * sx + sy * sy + sz * sz);
  double cx = sx / nrm, cy = sy / nrm, cz = sz / nrm;
  double bx = cx, by = cy, bz = cz, best = 1e300;
  const int iters = (b - a > 1) ? 48 : 1;
  for (int it = 0; it < iters; ++it) {
    double far = -1.0;
    int64_t fi = a;
    for (int64_t i = a + lane; i < b; i += 32) {
      double d = arc_between(cx, cy, cz, cen[3 * i], cen[3 * i + 1], cen[3 * i + 2]);
      if (d > far) { far = d; fi = i; }
    }
    for (int o = 16; o; o >>= 1) {
      double of = __shfl_xor_sync(0xffffffffu, far, o);
      int64_t oi = __shfl_xor_sync(0xffffffffu, fi, o);
      if (of > far || (of == far && oi < fi)) { far = of; fi = oi; }
    }
    if (far < best) { best = far; bx = cx; by = cy; bz = cz; }
    const double t = 1.0 / (it + 2.0);
    cx += t * (cen[3 * fi] - cx);
    cy += t * (cen[3 * fi + 1] - cy);
    cz += t * (cen[3 * fi + 2] - cz);
    nrm = sqrt(cx * cx + cy * cy + cz * cz);
    cx /= nrm; cy /= nrm; cz /= nrm;
  }
  if (lane == 0) {
    gc[3 * g] = bx; gc[3 * g + 1] = by; gc[3 * g + 2] = bz;
    gR[g] = best + eps;
  }
}

// group frames (ABI rule of geometry.cu applied to circle centres): [e1 | e2 | c]
__global__ void k_group_frames(const double* __restrict__ gc, int64_t ngroups, double* __restrict__ F) {
  int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= ngroups) return;
  double cx = gc[3 * g], cy = gc[3 * g + 1], cz = gc[3 * g + 2];
  double ax = 1.0, ay = 0.0;
  if (fabs(cx) > 0.9) { ax = 0.0; ay = 1.0; }
  double dot = ax * cx + ay * cy;
  double ex = ax - dot * cx, ey = ay - dot * cy, ez = -dot * cz;
  double inv = 1.0 / sqrt(ex * ex + ey * ey + ez * ez);
  ex *= inv; ey *= inv; ez *= inv;
  double fx = cy * ez - cz * ey, fy = cz * ex - cx * ez, fz = cx * ey - cy * ex;
  double* r = F + 9 * g;
  r[0] = ex; r[1] = ey; r[2] = ez; r[3] = fx; r[4] = fy; r[5] = fz; r[6] = cx; r[7] = cy; r[8] = cz;
}

// A group with one member takes that patch's own centre and frame (the ABI frame rule gives the same frame up to
// rounding): the member's Zernike nodes then sit exactly on their canonical rings in the group frame, which the
// separable step-4 evaluation (k_interp_sep) relies on.
__global__ void k_single_frames(const int32_t* __restrict__ gfirst, const int32_t* __restrict__ glast, int64_t ngroups,
                                const double* __restrict__ frames, double* __restrict__ gc, double* __restrict__ F) {
  int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= ngroups || glast[g] - gfirst[g] != 1) return;
  const double* R = frames + 9 * (int64_t)gfirst[g];   // [e1 | e2 | c], the same order as the group rows
  for (int t = 0; t < 9; ++t) F[9 * g + t] = R[t];
  for (int t = 0; t < 3; ++t) gc[3 * g + t] = R[6 + t];
}

// incoming-grid points: r_k = R cos(pi (k + 1/2) / (2 n_r)) (positive half of a 2 n_r Chebyshev grid),
// theta_l = 2 pi l / n_a;  x = cos(r) c + sin(r) (cos(theta) e1 + sin(theta) e2), stored x 1/2
__global__ void k_grid_points(const int32_t* __restrict__ grids, int64_t ngr, const int32_t* __restrict__ grid_group,
                              const double* __restrict__ F, const double* __restrict__ gR,
                              const int32_t* __restrict__ gnr, const int32_t* __restrict__ gna,
                              const int64_t* __restrict__ goff, const int64_t* __restrict__ rbase,
                              const int32_t* __restrict__ roff, double* gx, double* gy, double* gz) {
  const int64_t gi = blockIdx.x;
  if (gi >= ngr) return;
  const int k = grids[gi];
  const int g = grid_group[k];
  const int nr = gnr[k];
  const int32_t* ro = roff + rbase[k];   // ring kr holds points [ro[kr], ro[kr + 1]) (R26b: ring-adaptive)
  const double* r9 = F + 9 * (int64_t)g;
  for (int t = threadIdx.x; t < ro[nr]; t += blockDim.x) {
    int kr = 0;
    while (t >= ro[kr + 1]) ++kr;
    const int na = ro[kr + 1] - ro[kr], l = t - ro[kr];
    const double r = gR[g] * cospi((kr + 0.5) / (2.0 * nr));
    double st, ct, sr, cr;
    sincospi(2.0 * l / na, &st, &ct);
    sincos(r, &sr, &cr);
    const double a = sr * ct, b = sr * st;
    const int64_t o = goff[k] + t;
    gx[o] = 0.5 * (r9[0] * a + r9[3] * b + r9[6] * cr);
    gy[o] = 0.5 * (r9[1] * a + r9[4] * b + r9[7] * cr);
    gz[o] = 0.5 * (r9[2] * a + r9[5] * b + r9[8] * cr);
  }
}

// One thread per grid point of a chunk (256-thread CTAs over 256 / upts chunks); each thread issues the loads of up
// to 8 units' partial values before summing them in unit order (the same fixed order as one load at a time, so the
// result is unchanged bit for bit, with up to 8 loads in flight: the partials mostly come from DRAM)
__global__ void __launch_bounds__(256) k_reduce_chunks(const ChunkRec* __restrict__ ch, int64_t nch,
                                                       const double* __restrict__ part, int upts,
                                                       double* __restrict__ gval) {
  const int per = 256 / upts;                                   // chunks per CTA (upts divides 256)
  const int64_t c = (int64_t)blockIdx.x * per + threadIdx.x / upts;
  const int t = threadIdx.x % upts;
  if (c >= nch) return;
  const ChunkRec R = ch[c];
  if (t >= R.npt) return;
  double v = 0.0;
  for (int s0 = 0; s0 < R.nu; s0 += 8) {
    double a[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) a[e] = (s0 + e < R.nu) ? part[(R.u0 + s0 + e) * upts + t] : 0.0;
#pragma unroll
    for (int e = 0; e < 8; ++e)
      if (s0 + e < R.nu) v += a[e];
  }
  gval[R.pt0 + t] = v;
}

// step 4a: samples f(r_k, theta_l) (ring k: n_a(k) equispaced angles, radius-major) ->
// parity-restricted Chebyshev-Fourier coefficients c[m][j][cs], layout ((m * n_r + j) * 2 + cs), n = (m & 1) + 2 j:
//   Fourier:   AB[k][m][cs] = (2 - delta) / n_a(k) sum_l f(r_k, theta_l) {cos, sin}(2 pi m l / n_a(k)),  2m <= n_a(k);
//              0 for the orders ring k does not resolve (their amplitude there is below the grid tolerance, R26b)
//   Chebyshev: c[m][j][cs]  = (2 - delta_n0) / n_r sum_k AB[k][m][cs] cos(n pi (2k + 1) / (4 n_r))
// Twiddles are tabulated per ring in shared memory (exact index reduction, no per-term sincos).
__global__ void k_transform(const int32_t* __restrict__ grids, int64_t ngr, const int32_t* __restrict__ gnr,
                            const int32_t* __restrict__ gna, const int64_t* __restrict__ goff,
                            const int64_t* __restrict__ coff, const int64_t* __restrict__ rbase,
                            const int32_t* __restrict__ roff, const double* __restrict__ gval,
                            double* __restrict__ coef, const double2* __restrict__ twtab) {
  extern __shared__ double sh[];
  const int g = grids[blockIdx.x];   // grid id
  const int nr = gnr[g], M = gna[g] / 2;
  const int32_t* ro = roff + rbase[g];
  const int q = ro[nr];
  double* f = sh;                      // q samples
  double* AB = f + ((q + 1) & ~1);     // nr * (M+1) * 2 (16-byte aligned: tw is read as double2)
  double* tw = AB + nr * (M + 1) * 2;  // 2 q: ring k's (cos, sin)(2 pi r / n_a(k)) at 2 (ro[k] + r)
  double* ch = tw + 2 * q;             // 8 * nr: cos(pi r / (4 nr))
  for (int t = threadIdx.x; t < q; t += blockDim.x) {
    f[t] = gval[goff[g] + t];
    int kr = 0;
    while (t >= ro[kr + 1]) ++kr;
    // (cos, sin)(2 pi l / n) of ring kr (n = n_a(kr) angles) from the handle's table: entry n (n - 1) / 2 + l
    const int n = ro[kr + 1] - ro[kr], l = t - ro[kr];
    reinterpret_cast<double2*>(tw)[t] = twtab[(int64_t)n * (n - 1) / 2 + l];
  }
  for (int t = threadIdx.x; t < 8 * nr; t += blockDim.x) ch[t] = cospi((double)t / (4.0 * nr));
  __syncthreads();
  // one thread per (ring k, order m): both components from one 16-byte (cos, sin) twiddle read per sample (the
  // twiddle gathers at l m mod n_a are the kernel's shared-memory wavefront cost), same summation order as one
  // component per thread
  const double2* __restrict__ tw2 = reinterpret_cast<const double2*>(tw);
  for (int t = threadIdx.x; t < nr * (M + 1); t += blockDim.x) {
    const int k = t / (M + 1), m = t % (M + 1);
    const int na = ro[k + 1] - ro[k];
    double sc = 0.0, ss = 0.0;
    if (2 * m <= na) {
      const double* fk = f + ro[k];
      const double2* twk = tw2 + ro[k];
      int r = 0;
      for (int l = 0; l < na; ++l) {
        const double2 w = twk[r];
        sc = fma(fk[l], w.x, sc);
        ss = fma(fk[l], w.y, ss);
        r += m;
        if (r >= na) r -= na;
      }
      const bool edge = m == 0 || 2 * m == na;
      sc *= edge ? 1.0 / na : 2.0 / na;
      ss = edge ? 0.0 : ss * (2.0 / na);
    }
    AB[2 * t] = sc;
    AB[2 * t + 1] = ss;
  }
  __syncthreads();
  for (int t = threadIdx.x; t < (M + 1) * 2 * nr; t += blockDim.x) {
    const int m = t / (2 * nr), rem = t % (2 * nr), j = rem >> 1, cs = rem & 1;
    const int n = (m & 1) + 2 * j;
    const int P = 8 * nr, step = (2 * n) % P;
    int idx = n % P;                                   // n (2k + 1) mod 8 n_r, exactly reduced
    double s = 0.0;
    for (int k = 0; k < nr; ++k) {
      s = fma(AB[(k * (M + 1) + m) * 2 + cs], ch[idx], s);
      idx += step;
      if (idx >= P) idx -= P;
    }
    s *= 2.0 / nr;
    if (n == 0) s *= 0.5;
    coef[coff[g] + t] = s;
  }
}

// Warp-per-grid variant of step 4a (default, round 2): the same coefficients, with the Fourier sums of each ring by
// Clenshaw's recurrence instead of tabulated twiddles (R37):
//   b_l = f_l + 2 cos(w) b_{l+1} - b_{l+2}  (l = n_a - 1 .. 0, b_{n_a} = b_{n_a + 1} = 0),  w = 2 pi m / n_a(k),
//   sum_l f_l cos(l w) = b_0 - cos(w) b_1,   sum_l f_l sin(l w) = sin(w) b_1,
// 2 FP64 per (sample, order) and one broadcast shared-memory read, no per-sample index arithmetic; (cos w, sin w) from
// the long-double twiddle table.  Each warp transforms one grid with no CTA barrier (the CTA-per-grid kernel above
// spent its time on barriers and per-sample gathers: FP64 pipe 13%, profiles/r02o_ncu_full_transform.json).  Items
// (ring k, orders m and m + H) are spread over the lanes; the Chebyshev step is the kernel above's, per warp.
template <int WPC>
__global__ void __launch_bounds__(32 * WPC) k_transform_w(const int32_t* __restrict__ grids, int64_t ngr,
                                                          const int32_t* __restrict__ gnr, const int32_t* __restrict__ gna,
                                                          const int64_t* __restrict__ goff,
                                                          const int64_t* __restrict__ coff,
                                                          const int64_t* __restrict__ rbase,
                                                          const int32_t* __restrict__ roff,
                                                          const double* __restrict__ gval, double* __restrict__ coef,
                                                          const double2* __restrict__ twtab, int wsh,
                                                          const ChunkRec* __restrict__ chunks,
                                                          const int64_t* __restrict__ gch0,
                                                          const double* __restrict__ part, int upts) {
  extern __shared__ double sh[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // persistent warps (grid-stride over the grids) with the next grid's metadata loaded one grid ahead: the dependent
  // chain grids -> (n_r, M, offsets) no longer stalls every grid
  struct Meta {
    int g, nr, na;
    int64_t rb, go, co, c0, c1;
  };
  auto meta = [&](int g) {   // the loads of grid g's metadata (g < 0: none)
    Meta m{};
    m.g = g;
    if (g >= 0) {
      m.nr = gnr[g];
      m.na = gna[g];
      m.rb = rbase[g];
      m.go = goff[g];
      m.co = coff[g];
      if (part) {
        m.c0 = gch0[g];
        m.c1 = gch0[g + 1];
      }
    }
    return m;
  };
  const int64_t nw = (int64_t)gridDim.x * WPC;
  int64_t gi = (int64_t)blockIdx.x * WPC + warp;
  Meta mn = meta(gi < ngr ? grids[gi] : -1);
  int gn2 = gi + nw < ngr ? grids[gi + nw] : -1;   // two grids ahead: the id; one ahead: the metadata
  for (; gi < ngr; gi += nw) {
  const Meta mc = mn;
  mn = meta(gn2);
  gn2 = gi + 2 * nw < ngr ? grids[gi + 2 * nw] : -1;
  const int nr = mc.nr, M = mc.na / 2;
  const int32_t* ro = roff + mc.rb;
  const int q = ro[nr];
  double* f = sh + (size_t)warp * wsh;                   // q samples
  double2* AB = reinterpret_cast<double2*>(f + ((q + 1) & ~1));   // nr x (M + 1) (cos, sin) sums
  double* ch = reinterpret_cast<double*>(AB + nr * (M + 1));      // 8 nr: cos(pi r / (4 nr))
  if (part) {
    // fused grid reduction (k_reduce_chunks' sum, same unit order): the grid's chunks of upts points, each point the
    // sum of its units' partial values, straight into shared memory (no grid-value array in HBM)
    // (a lane owns points t and t + 32 of every chunk: 16 loads in flight per batch of 8 units)
    const int64_t pbase = mc.go;
    for (int64_t c = mc.c0; c < mc.c1; ++c) {
      const ChunkRec R = chunks[c];
      const bool in0 = lane < R.npt, in1 = lane + 32 < R.npt && upts > 32;
      double v0 = 0.0, v1 = 0.0;
      for (int s0 = 0; s0 < R.nu; s0 += 8) {
        double a0[8], a1[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const double* pp = part + (R.u0 + s0 + e) * upts + lane;
          a0[e] = (in0 && s0 + e < R.nu) ? pp[0] : 0.0;
          a1[e] = (in1 && s0 + e < R.nu) ? pp[32] : 0.0;
        }
#pragma unroll
        for (int e = 0; e < 8; ++e)
          if (s0 + e < R.nu) {
            v0 += a0[e];
            v1 += a1[e];
          }
      }
      if (in0) f[R.pt0 - pbase + lane] = v0;
      if (in1) f[R.pt0 - pbase + lane + 32] = v1;
    }
  }
  const double* __restrict__ gv = gval + mc.go;
  for (int t0 = 0; !part && t0 < q; t0 += 32 * 8) {   // eight loads in flight per lane
    double v[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int t = t0 + lane + 32 * e;
      v[e] = t < q ? gv[t] : 0.0;
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int t = t0 + lane + 32 * e;
      if (t < q) f[t] = v[e];
    }
  }
  for (int t = lane; t < 8 * nr; t += 32) ch[t] = cospi((double)t / (4.0 * nr));
  __syncwarp();
  // a lane takes two orders m and m + H (H = ceil((M + 1) / 2)) of one ring: two independent recurrences sharing
  // every sample read
  const int H = (M + 2) / 2, items = nr * H;
  for (int t = lane; t < items; t += 32) {
    const int k = t / H, m1 = t - k * H, m2 = m1 + H;
    const int r0 = ro[k], na = ro[k + 1] - r0;
    const bool ok1 = 2 * m1 <= na, ok2 = m2 <= M && 2 * m2 <= na;
    const double2* __restrict__ twn = twtab + (int64_t)na * (na - 1) / 2;
    const double2 w1 = ok1 ? twn[m1] : make_double2(0.0, 0.0);   // (cos, sin)(2 pi m / na)
    const double2 w2 = ok2 ? twn[m2] : make_double2(0.0, 0.0);
    const double c21 = 2.0 * w1.x, c22 = 2.0 * w2.x;
    const double* __restrict__ fk = f + r0;
    double b11 = 0.0, b12 = 0.0, b21 = 0.0, b22 = 0.0;
    if (ok1) {
#pragma unroll 4
      for (int l = na - 1; l >= 0; --l) {
        const double fl = fk[l];
        const double n1 = fma(c21, b11, fl - b12);
        const double n2 = fma(c22, b21, fl - b22);
        b12 = b11;
        b11 = n1;
        b22 = b21;
        b21 = n2;
      }
    }
    double A1 = fma(-w1.x, b12, b11), B1 = w1.y * b12;   // b_0 - cos(w) b_1, sin(w) b_1
    double A2 = fma(-w2.x, b22, b21), B2 = w2.y * b22;
    const bool e1 = m1 == 0 || 2 * m1 == na, e2 = 2 * m2 == na;
    A1 = ok1 ? A1 * (e1 ? 1.0 / na : 2.0 / na) : 0.0;
    B1 = (ok1 && !e1) ? B1 * (2.0 / na) : 0.0;
    A2 = ok2 ? A2 * (e2 ? 1.0 / na : 2.0 / na) : 0.0;
    B2 = (ok2 && !e2) ? B2 * (2.0 / na) : 0.0;
    AB[k * (M + 1) + m1] = make_double2(A1, B1);
    if (m2 <= M) AB[k * (M + 1) + m2] = make_double2(A2, B2);
  }
  __syncwarp();
  for (int t = lane; t < (M + 1) * 2 * nr; t += 32) {
    const int m = t / (2 * nr), rem = t % (2 * nr), j = rem >> 1, cs = rem & 1;
    const int n = (m & 1) + 2 * j;
    const int P = 8 * nr, step = (2 * n) % P;
    int idx = n % P;   // n (2k + 1) mod 8 n_r, exactly reduced
    double sacc = 0.0;
    for (int k = 0; k < nr; ++k) {
      const double2 ab = AB[k * (M + 1) + m];
      sacc = fma(cs ? ab.y : ab.x, ch[idx], sacc);
      idx += step;
      if (idx >= P) idx -= P;
    }
    sacc *= 2.0 / nr;
    if (n == 0) sacc *= 0.5;
    coef[mc.co + t] = sacc;
  }
  __syncwarp();   // every lane is done with this grid's shared memory before the next grid fills it
  }
}

// One grid's expansion at NPT nodes, angular sums first (MB = 0 variant of k_interp): per parity of m,
//   E_j = sum_{m of that parity} c[m][j] . (cos m theta, sin m theta)        (2 FMA per (m, j, node))
//   u  += sum_j E_j T_{par + 2 j}(x)                                          (once per grid and parity)
// The n_r accumulators per node live in registers (NR = n_r exactly, one instantiation per n_r: no idle FMAs).
// PF (k_interp MB = 3, n_r <= kPfNrMax): the coefficient pairs of order m + 2 are loaded from shared memory while
// order m is accumulated (two register buffers in ping-pong, the m loop unrolled by two): without it the compiler,
// short of registers, reuses one buffer and every LDS.128 is followed by its two consumers (short-scoreboard stalls,
// profiles/r01w_ncu_full_interp.json).  The prefetch index is clamped to M (same parity) so it never leaves the grid.
constexpr int kPfNrMax = 8;   // MB = 3; MB = 4 prefetches at every n_r <= kAngNrMax
template <int NR, int NPT, bool PF>
__device__ __forceinline__ void ang_orders_pf(const double2* __restrict__ cg, int par, int M, double (&E)[NPT][NR],
                                              double (&cm)[NPT], double (&sm)[NPT], double (&cp)[NPT],
                                              double (&sp)[NPT], const double (&t2)[NPT]) {
  auto step = [&](const double2 (&c)[NR]) {
#pragma unroll
    for (int j = 0; j < NR; ++j) {
#pragma unroll
      for (int q = 0; q < NPT; ++q) E[q][j] = fma(c[j].x, cm[q], fma(c[j].y, sm[q], E[q][j]));
    }
#pragma unroll
    for (int q = 0; q < NPT; ++q) {
      const double cn = fma(t2[q], cm[q], -cp[q]), sn = fma(t2[q], sm[q], -sp[q]);
      cp[q] = cm[q]; sp[q] = sm[q]; cm[q] = cn; sm[q] = sn;
    }
  };
  double2 ca[NR], cb[NR];
#pragma unroll
  for (int j = 0; j < NR; ++j) ca[j] = cg[par * NR + j];
  for (int m = par;;) {
    int mn = m + 2 <= M ? m + 2 : m;
#pragma unroll
    for (int j = 0; j < NR; ++j) cb[j] = cg[mn * NR + j];
    step(ca);
    m += 2;
    if (m > M) break;
    mn = m + 2 <= M ? m + 2 : m;
#pragma unroll
    for (int j = 0; j < NR; ++j) ca[j] = cg[mn * NR + j];
    step(cb);
    m += 2;
    if (m > M) break;
  }
}

template <int NR, int NPT, int PF = 0>
__device__ __forceinline__ void grid_eval_ang(const double2* __restrict__ cg, int M, const double (&x)[NPT],
                                              const double (&w2)[NPT], const double (&c1)[NPT],
                                              const double (&s1)[NPT], double (&acc)[NPT]) {
#pragma unroll
  for (int par = 0; par < 2; ++par) {
    if (par > M) break;
    double E[NPT][NR];
    double cm[NPT], sm[NPT], cp[NPT], sp[NPT], t2[NPT];   // cos/sin(m theta), ((m - 2) theta); 2 cos 2 theta
#pragma unroll
    for (int q = 0; q < NPT; ++q) {
#pragma unroll
      for (int j = 0; j < NR; ++j) E[q][j] = 0.0;
      const double c2 = fma(2.0 * c1[q], c1[q], -1.0), s2 = 2.0 * s1[q] * c1[q];
      t2[q] = 2.0 * c2;
      if (par == 0) { cm[q] = 1.0; sm[q] = 0.0; cp[q] = c2; sp[q] = -s2; }
      else { cm[q] = c1[q]; sm[q] = s1[q]; cp[q] = c1[q]; sp[q] = -s1[q]; }
    }
    if ((PF == 1 && NR <= kPfNrMax) || PF == 2) {
      ang_orders_pf<NR, NPT, true>(cg, par, M, E, cm, sm, cp, sp, t2);
    } else {
      for (int m = par; m <= M; m += 2) {
        const double2* __restrict__ cmj = cg + m * NR;
#pragma unroll
        for (int j = 0; j < NR; ++j) {
          const double2 c = cmj[j];
#pragma unroll
          for (int q = 0; q < NPT; ++q) E[q][j] = fma(c.x, cm[q], fma(c.y, sm[q], E[q][j]));
        }
#pragma unroll
        for (int q = 0; q < NPT; ++q) {   // (m, m - 2) -> (m + 2, m)
          const double cn = fma(t2[q], cm[q], -cp[q]), sn = fma(t2[q], sm[q], -sp[q]);
          cp[q] = cm[q]; sp[q] = sm[q]; cm[q] = cn; sm[q] = sn;
        }
      }
    }
#pragma unroll
    for (int q = 0; q < NPT; ++q) {   // sum_j E_j T_{par + 2 j}(x), T_{n+2} = w2 T_n - T_{n-2}
      double ta = par ? x[q] : 1.0;                                               // T_par
      double tb = par ? x[q] * fma(4.0 * x[q], x[q], -3.0) : fma(2.0 * x[q], x[q], -1.0);   // T_{par+2}
      double v = E[q][0] * ta;
#pragma unroll
      for (int j = 1; j < NR; ++j) {
        v = fma(E[q][j], tb, v);
        const double tn = fma(w2[q], tb, -ta);
        ta = tb;
        tb = tn;
      }
      acc[q] += v;
    }
  }
}

constexpr int kAngNrMax = 12;   // grid_eval_ang instantiations (n_r = 1..12)

// asin(s) = s sum_k c_k s^(2k), c_k = (2k)! / (4^k (k!)^2 (2k + 1))  (k_interp node geometry)
__constant__ double kAsinC[10] = {1.0, 1.0 / 6.0, 3.0 / 40.0, 5.0 / 112.0, 35.0 / 1152.0, 63.0 / 2816.0,
                                  231.0 / 13312.0, 143.0 / 10240.0, 6435.0 / 557056.0, 12155.0 / 1245184.0};

template <int NPT, int PF = 0>
__device__ __forceinline__ bool grid_eval_ang_any(int nr, const double2* __restrict__ cg, int M, const double (&x)[NPT],
                                                  const double (&w2)[NPT], const double (&c1)[NPT],
                                                  const double (&s1)[NPT], double (&acc)[NPT]) {
  switch (nr) {
#define NC_GE(R) \
  case R: grid_eval_ang<R, NPT, PF>(cg, M, x, w2, c1, s1, acc); return true;
    NC_GE(1) NC_GE(2) NC_GE(3) NC_GE(4) NC_GE(5) NC_GE(6) NC_GE(7) NC_GE(8) NC_GE(9) NC_GE(10) NC_GE(11) NC_GE(12)
#undef NC_GE
    default: return false;
  }
}

// step 4b: u_i(node) = udir + sum over levels of the level's group expansions at the node,
//   u(x, theta) = sum_m sum_j c[m][j] . (cos m theta, sin m theta) T_{(m & 1) + 2 j}(rho / R)
// (rho = geodesic distance from the cap centre).  One CTA of NT threads per target patch, NPT nodes per thread.
// Per level, the coefficients of all the group's grids (<= kMaxGrids) are staged in shared memory in one pass and
// the node geometry (rho / R, theta) is computed once; then, per grid and order m, the j loop advances the
// parity's Chebyshev recurrence T_{n+2} = w2 T_n - T_{n-2} and accumulates both trig components from one broadcast
// shared-memory load of the coefficient pair (3 FMA per (m, j, node)).  MB > 1: MB orders per j loop (both parity
// recurrences advanced once, 2 + 2/MB FMA per pair; measured slower at C5, kept selectable).
template <int NT, int NPT, int MB, int MINB>
__global__ void __launch_bounds__(NT, MINB) k_interp(int L, int64_t rc, int Kstar, const int32_t* __restrict__ pgl,
                                               const int64_t* __restrict__ ggrid0,
                                               const double* __restrict__ F, const double* __restrict__ gRinv,
                                               const int32_t* __restrict__ gnr, const int32_t* __restrict__ gna,
                                               const int64_t* __restrict__ coff, const double* __restrict__ coef,
                                               const double* __restrict__ tx, const double* __restrict__ ty,
                                               const double* __restrict__ tz, const double* __restrict__ udir,
                                               double* __restrict__ u, const uint8_t* __restrict__ gsep,
                                               int nr_big, double lt, const double* __restrict__ cen,
                                               int asin_terms, int cap, int sel, const uint64_t* __restrict__ pcode,
                                               const int32_t* __restrict__ work) {
  // MB = 0 evaluates the grids with n_r <= kAngNrMax only (grid_eval_ang); a second pass (MB = 1, nr_big = 1) adds
  // the rest to u when any exists (tight precisions): the register-held accumulators of the first pass then need
  // no fallback code in the same kernel
  extern __shared__ double2 c2[];
  // per level (one thread each, once per CTA): the group's grids (count, n_r, M, coefficient offset), frame, 1 / R,
  // and the patch centre's (arc, sin arc, cos arc) about the group centre -- the level loop then reads no global
  // metadata (its dependent load chains were the kernel's long-scoreboard stalls, profiles/r02d_ncu_full_interp)
  __shared__ double lv_a0[kLmax + 1], lv_r0[kLmax + 1], lv_c0[kLmax + 1], lv_invR[kLmax + 1], lv_r9[kLmax + 1][9];
  __shared__ int64_t lv_coff[kLmax + 1][kMaxGrids];
  __shared__ int lv_ng[kLmax + 1], lv_nr[kLmax + 1][kMaxGrids], lv_M[kLmax + 1][kMaxGrids];
  const int64_t i = work ? work[blockIdx.x] : blockIdx.x;
  if ((int)threadIdx.x <= L) {
    const int lvl = threadIdx.x;
    const int g = pgl[(int64_t)lvl * rc + i];
    const int64_t kg0 = ggrid0[g], kg1 = ggrid0[g + 1];
    // R36: sel 1 keeps the levels evaluated at the nodes, sel 2 + r those of proxy rule r (the level's 2-bit code in
    // pcode[i], decided once on the host: the passes partition the levels)
    const bool keep = sel == 0 || (int)((pcode[i] >> (2 * lvl)) & 3u) == sel - 1;
    const bool ok = keep && kg0 != kg1 && gnr[kg0] != 0 && !(gsep && gsep[g]);
    lv_ng[lvl] = ok ? (int)(kg1 - kg0) : 0;
    if (ok) {
      for (int64_t kg = kg0; kg < kg1; ++kg) {
        lv_nr[lvl][kg - kg0] = gnr[kg];
        lv_M[lvl][kg - kg0] = gna[kg] / 2;
        lv_coff[lvl][kg - kg0] = coff[kg];
      }
      const double* r9 = F + 9 * (int64_t)g;
      for (int e = 0; e < 9; ++e) lv_r9[lvl][e] = r9[e];
      lv_invR[lvl] = gRinv[g];
      if (asin_terms > 0) {
        const double cx = cen[3 * i], cy = cen[3 * i + 1], czc = cen[3 * i + 2];
        const double sx = r9[0] * cx + r9[1] * cy + r9[2] * czc;
        const double sy = r9[3] * cx + r9[4] * cy + r9[5] * czc;
        const double cz = r9[6] * cx + r9[7] * cy + r9[8] * czc;
        const double r0 = sqrt(sx * sx + sy * sy);
        lv_a0[lvl] = atan2(r0, cz);
        lv_r0[lvl] = r0;
        lv_c0[lvl] = cz;
      }
    }
  }
  __syncthreads();
  for (int kb = 0; kb < Kstar; kb += NPT * NT) {
    double acc[NPT], px[NPT], py[NPT], pz[NPT];
#pragma unroll
    for (int q = 0; q < NPT; ++q) {
      const int k = min(kb + (int)threadIdx.x + q * NT, Kstar - 1);
      const int64_t t = i * Kstar + k;
      px[q] = 2.0 * tx[t]; py[q] = 2.0 * ty[t]; pz[q] = 2.0 * tz[t];
      acc[q] = nr_big ? u[t] : (udir ? udir[t] : 0.0);   // second pass: add to the first's result
    }
    // the levels whose group has grids here (block-uniform: a group's grids are all local or none; single-member
    // groups are k_interp_sep's); the coefficients of every grid of the next such level are copied global ->
    // shared with cp.async into the other half of c2 while this level is evaluated (double buffer, cap pairs each)
    auto next_level = [&](int lv) {
      while (lv <= L && lv_ng[lv] == 0) ++lv;
      return lv;
    };
    auto stage = [&](int lv, double2* dst) {
      int base = 0;
      for (int q = 0; q < lv_ng[lv]; ++q) {
        const int ncp = (lv_M[lv][q] + 1) * lv_nr[lv][q];
        const double2* __restrict__ src = reinterpret_cast<const double2*>(coef + lv_coff[lv][q]);
        for (int t = threadIdx.x; t < ncp; t += NT) cp_async16(dst + base + t, src + t);
        base += ncp;
      }
      cp_async_commit();
    };
    // cap >= 0: double buffer (the next level's copy overlaps this level); cap < 0: one buffer of -cap pairs, each
    // level copied and then evaluated (half the shared memory: more resident CTAs for the 32-point proxy pass)
    const bool db = cap >= 0;
    int buf = 0;
    int lvl = next_level(0);
    if (db && lvl <= L) stage(lvl, c2);
    while (lvl <= L) {
      const int nxt = next_level(lvl + 1);
      if (!db) {
        stage(lvl, c2);
        cp_async_wait<0>();
      } else if (nxt <= L) {
        stage(nxt, c2 + (size_t)(buf ^ 1) * cap);
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      __syncthreads();                              // this level's coefficients are in shared memory
      const double2* __restrict__ cl = c2 + (size_t)buf * cap;
      const double* r9 = lv_r9[lvl];
      const double invR = lv_invR[lvl];
      double x[NPT], w2[NPT], c1[NPT], s1[NPT];
#pragma unroll
      for (int q = 0; q < NPT; ++q) {
        const double sx = r9[0] * px[q] + r9[1] * py[q] + r9[2] * pz[q];
        const double sy = r9[3] * px[q] + r9[4] * py[q] + r9[5] * pz[q];
        const double cz = r9[6] * px[q] + r9[7] * py[q] + r9[8] * pz[q];
        const double rho2 = fma(sx, sx, sy * sy);
        double rho = 0.0;
        if (rho2 > 0.0) {
          const double irho = fast_rsqrt(rho2);
          rho = rho2 * irho;
          c1[q] = sx * irho;
          s1[q] = sy * irho;
        } else {
          c1[q] = 1.0;
          s1[q] = 0.0;
        }
        double arc;
        if (asin_terms > 0) {
          // arc = arc(centre) + asin(sin(arc - arc(centre))), |arc - arc(centre)| <= eps: the series in s^2 (Horner,
          // asin_terms terms, block-uniform) instead of an fp64 atan2 per node and level
          const double sd = fma(rho, lv_c0[lvl], -cz * lv_r0[lvl]);
          const double z = sd * sd;
          double pa = kAsinC[asin_terms - 1];
          for (int k = asin_terms - 2; k >= 0; --k) pa = fma(pa, z, kAsinC[k]);
          arc = fma(sd, pa, lv_a0[lvl]);
        } else {
          arc = atan2(rho, cz);
        }
        x[q] = arc * invR;
        w2[q] = 4.0 * x[q] * x[q] - 2.0;
      }
      int base = 0;
      for (int qg = 0; qg < lv_ng[lvl]; ++qg) {
        const int nr = lv_nr[lvl][qg], M = lv_M[lvl][qg];
        const double2* __restrict__ cg = cl + base;
        base += (M + 1) * nr;
        if (MB == 0 || MB == 3 || MB == 4) {
          // orders this thread's nodes need (R26c): order m has amplitude ~(rho / beta)^m at radius rho R, and the
          // grid's M = n_a / 2 fixes ln beta >= 0.975 ln(1/tol) / (M - 2) (grid_size), so nodes at rho need
          // m <= 0.975 ln(1/tol) / (ln beta - ln rho) + 3; lt = 0 disables the truncation
          int Mq = M;
          if (lt > 0.0 && M > 4) {
            double xm = x[0];
#pragma unroll
            for (int q = 1; q < NPT; ++q) xm = fmax(xm, x[q]);
            const float lnb = (float)(0.975 * lt) / (float)(M - 2);
            const float den = lnb - __logf(fmaxf((float)xm, 1e-30f));
            if (den > 0.0f) Mq = min(M, (int)ceilf((float)(0.975 * lt) / den) + 3);
          }
          grid_eval_ang_any<NPT, MB == 3 ? 1 : MB == 4 ? 2 : 0>(nr, cg, Mq, x, w2, c1, s1, acc);   // n_r <= kAngNrMax (else: second pass)
          continue;
        }
        if (nr_big && nr <= kAngNrMax) continue;                    // second pass: done by the first
        double cm[NPT], sm[NPT], cmm[NPT], smm[NPT];   // cos/sin(m theta), ((m - 1) theta)
#pragma unroll
        for (int q = 0; q < NPT; ++q) { cm[q] = 1.0; sm[q] = 0.0; cmm[q] = c1[q]; smm[q] = -s1[q]; }
        if (MB <= 1) {
          // orders in pairs (m even, m + 1 odd); cos/sin(m theta) advanced in place two orders at a time and the
          // Chebyshev pair (T_n, T_{n+2}) advanced in place two degrees at a time: no register rotation moves
          double ce[NPT], se[NPT], co[NPT], so[NPT];
#pragma unroll
          for (int q = 0; q < NPT; ++q) { ce[q] = 1.0; se[q] = 0.0; co[q] = c1[q]; so[q] = s1[q]; }
          for (int m = 0; m <= M; m += 2) {
#pragma unroll
            for (int par = 0; par < 2; ++par) {
              if (m + par > M) break;
              const double2* __restrict__ cmj = cg + (m + par) * nr;
              double A[NPT], B[NPT], ta[NPT], tb[NPT];
              const double2 c0 = cmj[0];
#pragma unroll
              for (int q = 0; q < NPT; ++q) {
                ta[q] = par ? x[q] : 1.0;                                              // T_par
                tb[q] = par ? x[q] * (4.0 * x[q] * x[q] - 3.0) : 2.0 * x[q] * x[q] - 1.0;   // T_{par + 2}
                A[q] = c0.x * ta[q];
                B[q] = c0.y * ta[q];
              }
              int j = 1;
              for (; j + 1 < nr; j += 2) {
                const double2 ca = cmj[j], cb = cmj[j + 1];
#pragma unroll
                for (int q = 0; q < NPT; ++q) {
                  A[q] = fma(ca.x, tb[q], A[q]);
                  B[q] = fma(ca.y, tb[q], B[q]);
                  ta[q] = fma(w2[q], tb[q], -ta[q]);   // T_{par + 2 (j + 1)}
                  A[q] = fma(cb.x, ta[q], A[q]);
                  B[q] = fma(cb.y, ta[q], B[q]);
                  tb[q] = fma(w2[q], ta[q], -tb[q]);   // T_{par + 2 (j + 2)}
                }
              }
              if (j < nr) {
                const double2 ca = cmj[j];
#pragma unroll
                for (int q = 0; q < NPT; ++q) {
                  A[q] = fma(ca.x, tb[q], A[q]);
                  B[q] = fma(ca.y, tb[q], B[q]);
                }
              }
#pragma unroll
              for (int q = 0; q < NPT; ++q)
                acc[q] = par ? fma(A[q], co[q], fma(B[q], so[q], acc[q])) : fma(A[q], ce[q], fma(B[q], se[q], acc[q]));
            }
#pragma unroll
            for (int q = 0; q < NPT; ++q) {   // (m, m + 1) -> (m + 2, m + 3)
              const double t = 2.0 * c1[q];
              ce[q] = fma(t, co[q], -ce[q]);
              se[q] = fma(t, so[q], -se[q]);
              co[q] = fma(t, ce[q], -co[q]);
              so[q] = fma(t, se[q], -so[q]);
            }
          }
        } else {
          for (int m0 = 0; m0 <= M; m0 += MB) {
            double A[MB > 1 ? MB : 1][NPT], B[MB > 1 ? MB : 1][NPT], te[NPT], tep[NPT], to[NPT], top[NPT];
            // T_0 = 1, T_1 = x; the step-2 recurrence starts from T_{-2} = T_2 and T_{-1} = T_1 (T_{-n} = T_n)
#pragma unroll
            for (int q = 0; q < NPT; ++q) {
              te[q] = 1.0; tep[q] = 2.0 * x[q] * x[q] - 1.0;
              to[q] = x[q]; top[q] = x[q];
            }
#pragma unroll
            for (int b = 0; b < MB; ++b) {   // m0 is even (MB even): the parity of m = m0 + b is b's, known here
              const int m = m0 + b;
              const double2 c = (m <= M) ? cg[m * nr] : make_double2(0.0, 0.0);
#pragma unroll
              for (int q = 0; q < NPT; ++q) {
                const double tv = (b & 1) ? to[q] : te[q];
                A[b][q] = c.x * tv;
                B[b][q] = c.y * tv;
              }
            }
            for (int j = 1; j < nr; ++j) {
#pragma unroll
              for (int q = 0; q < NPT; ++q) {   // advance: te = T_{2j}, to = T_{2j+1}
                const double ne = fma(w2[q], te[q], -tep[q]);
                const double no = fma(w2[q], to[q], -top[q]);
                tep[q] = te[q]; te[q] = ne;
                top[q] = to[q]; to[q] = no;
              }
#pragma unroll
              for (int b = 0; b < MB; ++b) {
                const int m = m0 + b;
                const double2 c = (m <= M) ? cg[m * nr + j] : make_double2(0.0, 0.0);
#pragma unroll
                for (int q = 0; q < NPT; ++q) {
                  const double tv = (b & 1) ? to[q] : te[q];
                  A[b][q] = fma(c.x, tv, A[b][q]);
                  B[b][q] = fma(c.y, tv, B[b][q]);
                }
              }
            }
#pragma unroll
            for (int b = 0; b < MB; ++b) {
#pragma unroll
              for (int q = 0; q < NPT; ++q) {
                acc[q] = fma(A[b][q], cm[q], fma(B[b][q], sm[q], acc[q]));
                const double cn = 2.0 * c1[q] * cm[q] - cmm[q], sn = 2.0 * c1[q] * sm[q] - smm[q];
                cmm[q] = cm[q]; smm[q] = sm[q]; cm[q] = cn; sm[q] = sn;
              }
            }
          }
        }
      }
      __syncthreads();                              // every reader of buffer `buf` is done before it is refilled
      lvl = nxt;
      if (db) buf ^= 1;
    }
#pragma unroll
    for (int q = 0; q < NPT; ++q) {
      const int k = kb + (int)threadIdx.x + q * NT;
      if (k < Kstar) u[i * Kstar + k] = acc[q];
    }
  }
}

// step 4b for single-member groups (evaluated separably): the group frame is the member's own
// (k_single_frames), so node k lies at geodesic radius t_a (its ring a) and angle theta_k, and
//   u_k += sum_m A_a[m] . (cos m theta_k, sin m theta_k),   A_a[m] = sum_j c[m][j] T_{(m & 1) + 2 j}(t_a / R)
// costs nA (M+1) n_r + K* (M+1) terms per grid instead of K* (M+1) n_r.  One CTA per patch of `work`, all its
// single-member levels; runs after k_interp (which skipped those levels) and adds to u.
template <int NT, int NPT>
__global__ void __launch_bounds__(NT) k_interp_sep(int L, int64_t rc, int Ks, const int32_t* __restrict__ work,
                                                   const int32_t* __restrict__ pgl, const uint8_t* __restrict__ gsep,
                                                   const int64_t* __restrict__ ggrid0, const double* __restrict__ gR,
                                                   const int32_t* __restrict__ gnr, const int32_t* __restrict__ gna,
                                                   const int64_t* __restrict__ coff, const double* __restrict__ coef,
                                                   int nA, const double* __restrict__ ring_t,
                                                   const int32_t* __restrict__ node_ring,
                                                   const double* __restrict__ node_cs, int cpairs, int Mmax,
                                                   int nrmax, double* __restrict__ u) {
  extern __shared__ double2 sx2[];
  double2* cb = sx2;                                  // the grid's coefficient pairs c[m][j]
  double2* A = sx2 + cpairs;                          // nA x (Mmax + 1)
  double* T = reinterpret_cast<double*>(A + (size_t)nA * (Mmax + 1));   // nA x (2 nrmax + 1)
  const int TS = 2 * nrmax + 1;
  const int64_t i = work[blockIdx.x];
  double acc[NPT], c1[NPT], s1[NPT];
  int ring[NPT];
#pragma unroll
  for (int q = 0; q < NPT; ++q) {
    const int k = min((int)threadIdx.x + q * NT, Ks - 1);
    acc[q] = 0.0;
    ring[q] = node_ring[k];
    c1[q] = node_cs[2 * k];
    s1[q] = node_cs[2 * k + 1];
  }
  // the patch's separable levels (group, first and last grid), gathered by one thread per level up front: the level
  // loop then waits on no dependent global loads (pgl -> gsep -> ggrid0 per level was the kernel's long-scoreboard
  // stall)
  __shared__ int sl_g[kLmax + 1];
  __shared__ int64_t sl_k0[kLmax + 1], sl_k1[kLmax + 1];
  if ((int)threadIdx.x <= L) {
    const int g = pgl[(int64_t)threadIdx.x * rc + i];
    sl_g[threadIdx.x] = gsep[g] ? g : -1;
    sl_k0[threadIdx.x] = ggrid0[g];
    sl_k1[threadIdx.x] = ggrid0[g + 1];
  }
  __syncthreads();
  for (int lvl = 0; lvl <= L; ++lvl) {
    const int g = sl_g[lvl];
    if (g < 0) continue;                                        // block-uniform
    const double invR = 1.0 / gR[g];
    for (int64_t kg = sl_k0[lvl]; kg < sl_k1[lvl]; ++kg) {
      const int nr = gnr[kg], M = gna[kg] / 2;
      __syncthreads();                                          // previous grid's readers are done
      {
        const int ncp = (M + 1) * nr;
        const double2* __restrict__ src = reinterpret_cast<const double2*>(coef + coff[kg]);
        for (int t = threadIdx.x; t < ncp; t += NT) cb[t] = src[t];
      }
      for (int a = threadIdx.x; a < nA; a += NT) {              // T_n(t_a / R), n <= 2 nr - 1
        const double x = ring_t[a] * invR;
        double* Ta = T + a * TS;
        double tm = 1.0, tn = x;
        Ta[0] = 1.0;
        Ta[1] = x;
        for (int n = 2; n < 2 * nr; ++n) {
          const double t2 = fma(2.0 * x, tn, -tm);
          Ta[n] = t2;
          tm = tn;
          tn = t2;
        }
      }
      __syncthreads();
      for (int t = threadIdx.x; t < nA * (M + 1); t += NT) {   // A_a[m]
        const int a = t / (M + 1), m = t - a * (M + 1);
        const double2* __restrict__ cm = cb + m * nr;
        const double* __restrict__ Ta = T + a * TS + (m & 1);
        double ax = 0.0, ay = 0.0;
        for (int j = 0; j < nr; ++j) {
          const double tv = Ta[2 * j];
          ax = fma(cm[j].x, tv, ax);
          ay = fma(cm[j].y, tv, ay);
        }
        A[a * (Mmax + 1) + m] = make_double2(ax, ay);
      }
      __syncthreads();
#pragma unroll
      for (int q = 0; q < NPT; ++q) {
        const double2* __restrict__ Aa = A + ring[q] * (Mmax + 1);
        double cm = 1.0, sm = 0.0, cp = c1[q], sp = -s1[q];   // cos/sin(m theta), ((m - 1) theta)
        const double tc = 2.0 * c1[q];
        double v = 0.0;
        for (int m = 0; m <= M; ++m) {
          const double2 am = Aa[m];
          v = fma(am.x, cm, fma(am.y, sm, v));
          const double cn = fma(tc, cm, -cp), sn = fma(tc, sm, -sp);
          cp = cm; sp = sm; cm = cn; sm = sn;
        }
        acc[q] += v;
      }
    }
  }
#pragma unroll
  for (int q = 0; q < NPT; ++q) {
    const int k = (int)threadIdx.x + q * NT;
    if (k < Ks) u[i * Ks + k] += acc[q];
  }
}

// interpolation variant: NC_INTERP_VARIANT="NT,NPT,MB,MINB" (k_interp<NT,NPT,MB,MINB>, NC_INTERP_LIST below;
// MB = 0: grid_eval_ang for n_r <= 12, MB = 1: Chebyshev sums first, MB = 2: two orders per radial loop, MB = 3:
// grid_eval_ang with the coefficient prefetch for n_r <= kPfNrMax)
struct InterpVariant {
  int nt, npt, mb, minb;
};
static InterpVariant interp_variant() {
  static InterpVariant v = {-1, 0, 0, 0};
  if (v.nt < 0) {
    v = {256, 2, 0, 2};   // angular sums first (grid_eval_ang), measured fastest at C5 (profiles/r01l_interp_*)
    if (const char* e = tuning_env("NC_INTERP_VARIANT")) {
      InterpVariant w = v;
      w.minb = 1;
      if (sscanf(e, "%d,%d,%d,%d", &w.nt, &w.npt, &w.mb, &w.minb) >= 3) v = w;
    }
  }
  return v;
}

template <int NT, int NPT, int MB, int MINB>
static int launch_interp_t(size_t shm, int L, int64_t rc, int Ks, const int32_t* pgl, const int64_t* ggrid0,
                           const double* F, const double* gRinv, const int32_t* gnr, const int32_t* gna,
                           const int64_t* coff, const double* coef, const double* tx, const double* ty,
                           const double* tz, const double* udir, double* u, const uint8_t* gsep, cudaStream_t s,
                           int nr_big, double lt, const double* cen, int asin_terms, int sel, const uint64_t* pfar,
                           const int32_t* work, int64_t nblocks) {
  auto kern = k_interp<NT, NPT, MB, MINB>;
  // shm: the two coefficient buffers (cap = shm / 32 pairs each, 16-byte aligned halves); the one-warp CTAs of the
  // 32-point proxy pass take one buffer of half the size (cap < 0: 20 resident CTAs per SM instead of 10)
  const bool single = NT <= 32;
  const size_t sh = single ? shm / 2 : shm;
  const int cap = single ? -(int)(sh / sizeof(double2)) : (int)(shm / (2 * sizeof(double2)));
  if (sh > 48 * 1024) NC_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh));
  if (nblocks <= 0) return NC_OK;
  kern<<<(unsigned)nblocks, NT, sh, s>>>(L, rc, Ks, pgl, ggrid0, F, gRinv, gnr, gna, coff, coef, tx, ty, tz, udir, u,
                                         gsep, nr_big, lt, cen, asin_terms, cap, sel, pfar, work);
  return NC_OK;
}

// the instantiated first-pass variants (the default of each K* range, and the alternatives the step-4 tests compare)
#define NC_INTERP_LIST(X) X(128, 2, 3, 4) X(256, 2, 0, 2) X(128, 2, 0, 4) X(128, 4, 1, 4) X(128, 4, 2, 4) \
  X(96, 1, 3, 6) X(128, 1, 3, 5) X(64, 1, 3, 8) X(32, 1, 3, 16)
static bool interp_listed(const InterpVariant& v) {
#define NC_I(NT, NPT, MB, MINB) if (v.nt == NT && v.npt == NPT && v.mb == MB && v.minb == MINB) return true;
  NC_INTERP_LIST(NC_I)
#undef NC_I
  return false;
}

static int launch_interp(size_t shm, int L, int64_t rc, int Ks, int nrmax, int namax, const int32_t* pgl,
                         const int64_t* ggrid0, const double* F, const double* gRinv, const int32_t* gnr,
                         const int32_t* gna, const int64_t* coff, const double* coef, const double* tx,
                         const double* ty, const double* tz, const double* udir, double* u, const uint8_t* gsep,
                         double lt, const double* cen, int asin_terms, cudaStream_t s, int sel = 0,
                         const uint64_t* pfar = nullptr, const int32_t* work = nullptr, int64_t nwork = -1) {
  const int64_t nb = work ? nwork : rc;   // CTAs: one per patch of the work list (all local patches without one)
  (void)namax;
  // defaults: the 248-node rule takes one 128-thread CTA per patch with the coefficient prefetch (MB = 3: rest of
  // the C5 step 20.07 -> 18.32 ms, bitwise-identical output, profiles/r01w_interp_prefetch_c5.jsonl); larger K*
  // the 256-thread angular-sums-first kernel.  NC_INTERP_VARIANT must name a listed variant (else: the default,
  // with a warning -- never a silently skipped first pass)
  InterpVariant dflt = Ks <= 256 ? InterpVariant{128, 2, 3, 4} : InterpVariant{256, 2, 0, 2};
  // the proxy passes (sel >= 2, R36): one point per thread, the CTA the size of the proxy set in whole warps
  if (sel >= 2) dflt = Ks <= 32 ? InterpVariant{32, 1, 3, 16} : Ks <= 64 ? InterpVariant{64, 1, 3, 8}
                     : Ks <= 96 ? InterpVariant{96, 1, 3, 6} : InterpVariant{128, 1, 3, 5};
  InterpVariant v = (tuning_env("NC_INTERP_VARIANT") && sel < 2) ? interp_variant() : dflt;
  if (!interp_listed(v)) {
    fprintf(stderr, "[nc] NC_INTERP_VARIANT=%s is not an instantiated variant; using the default\n",
            tuning_env("NC_INTERP_VARIANT"));
    v = dflt;
  }
  // the angular-sums-first kernels (MB 0, 3) evaluate grids with n_r <= kAngNrMax; a second pass (MB = 1, nr_big)
  // adds the larger ones
  const bool two_pass = (v.mb == 0 || v.mb == 3) && nrmax > kAngNrMax;
#define NC_I(NT, NPT, MB, MINB)                                                                                  \
  if (v.nt == NT && v.npt == NPT && v.mb == MB && v.minb == MINB)                                                \
    NC_TRY((launch_interp_t<NT, NPT, MB, MINB>(shm, L, rc, Ks, pgl, ggrid0, F, gRinv, gnr, gna, coff, coef, tx,   \
                                               ty, tz, udir, u, gsep, s, 0, lt, cen, asin_terms, sel, pfar, work, nb)));
  NC_INTERP_LIST(NC_I)
#undef NC_I
  if (two_pass)
    return launch_interp_t<128, 4, 1, 4>(shm, L, rc, Ks, pgl, ggrid0, F, gRinv, gnr, gna, coff, coef, tx, ty, tz, udir,
                                         u, gsep, s, 1, 0.0, cen, asin_terms, sel, pfar, work, nb);
  return NC_OK;
}

// ------------------------------------------------------------------------------------------------
// host helpers
// ------------------------------------------------------------------------------------------------
template <class T>
static int halloc(nc_handle* h, T** p, size_t count) {
  if (count == 0) count = 1;
  cudaError_t e = cudaMalloc((void**)p, count * sizeof(T));
  if (e != cudaSuccess) {
    (void)cudaGetLastError();
    return fail(NC_ENOMEM, "cudaMalloc (hier) of " + std::to_string(count * sizeof(T)) + " bytes failed");
  }
  h->device_bytes += (double)count * sizeof(T);
  return NC_OK;
}

template <class T>
static int upload(nc_handle* h, T** dst, const std::vector<T>& src, cudaStream_t s) {
  NC_TRY(halloc(h, dst, src.size()));
  if (!src.empty()) NC_CUDA_TRY(cudaMemcpyAsync(*dst, src.data(), src.size() * sizeof(T), cudaMemcpyHostToDevice, s));
  return NC_OK;
}

template <class T>
static int download(std::vector<T>& dst, const T* src, size_t n, cudaStream_t s) {
  dst.resize(n);
  if (n) NC_CUDA_TRY(cudaMemcpyAsync(dst.data(), src, n * sizeof(T), cudaMemcpyDeviceToHost, s));
  NC_CUDA_TRY(cudaStreamSynchronize(s));
  return NC_OK;
}

// incoming-grid size for a nearest grid source at beta = (distance - eps) / R and tolerance tol
// (parity-restricted Chebyshev-Fourier; fitted to point-source interpolation tests, DESIGN.md "Incoming grids";
// verified by tests/test_hier_gpu.py against the direct sum)
static int nr_margin() {   // rings added beyond the radial fit (NC_NR_MARGIN, default 1; R21)
  static int v = -1;
  if (v < 0) {
    const char* e = tuning_env("NC_NR_MARGIN");
    v = e ? std::max(0, atoi(e)) : 1;
  }
  return v;
}

static int na_margin() {   // angles added beyond the azimuthal fit on the outer ring (NC_NA_MARGIN, default 4)
  static int v = -1;
  if (v < 0) {
    const char* e = tuning_env("NC_NA_MARGIN");
    v = e ? std::max(0, atoi(e)) : 4;
  }
  return v;
}

static void grid_size(double beta, double tol, int& nr, int& na) {
  const double lt = log(1.0 / tol);
  nr = (int)ceil(0.56 * lt / acosh(std::max(beta, 1.0 + 1e-9))) + nr_margin();
  na = (int)ceil(1.95 * lt / log(std::max(beta, 1.0 + 1e-9))) + na_margin();
  na += na & 1;
  nr = std::max(nr, 3);
  na = std::max(na, 8);
}

// Ring-adaptive angular resolution (R26b): the field of a source at beta R has azimuthal orders of
// amplitude ~(rho / beta)^m on the ring at radius rho R, so ring k (rho_k = cos((k + 1/2) pi / (2 n_r))) needs the
// outer ring's count with beta replaced by beta / rho_k: n_a(k) = min(n_a, 1.95 ln(1/tol) / ln(beta / rho_k) + 8),
// then trimmed towards a whole number of 32-point warps (ring_fill) but never below the margin-6 sizes.
// NC_RING_ADAPT=0 keeps n_a on every ring (the tensor grid).
static bool ring_adapt() {
  static int v = -1;
  if (v < 0) {
    const char* e = tuning_env("NC_RING_ADAPT");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}
static int ring_margin() {   // points added to every adapted ring beyond the fit (NC_RING_MARGIN, default 8)
  static int v = -1;
  if (v < 0) {
    const char* e = tuning_env("NC_RING_MARGIN");
    v = e ? std::max(0, atoi(e)) : 8;
  }
  return v;
}
// ring radii rho_k = cos((k + 1/2) pi / (2 n_r)) per n_r, computed once (the same expression as inline)
constexpr int kRingMax = 64;
static const double* ring_rho(int nr) {
  static const std::vector<double> tab = [] {
    std::vector<double> t((size_t)(kRingMax + 1) * kRingMax, 0.0);
    for (int n = 1; n <= kRingMax; ++n)
      for (int k = 0; k < n; ++k) t[(size_t)n * kRingMax + k] = cos((k + 0.5) * M_PI / (2.0 * n));
    return t;
  }();
  return tab.data() + (size_t)nr * kRingMax;
}
// per ring k: 1.95 ln(1/tol) / ln(beta / rho_k), the ring-adaptive count before the margin (allocation-free: the
// routing calls this for every candidate band of every group)
static void ring_fit(double beta, double tol, int nr, double* fit) {
  const double lt = log(1.0 / tol);
  const double* rho = ring_rho(nr);
  for (int k = 0; k < nr; ++k) fit[k] = 1.95 * lt / log(std::max(beta, 1.0 + 1e-9) / rho[k]);
}
static int ring_points_margin_fit(const double* fit, int nr, int na, int margin, int* out) {
  int q = 0;
  for (int k = 0; k < nr; ++k) {
    int nk = na;
    if (ring_adapt()) {
      nk = (int)ceil(fit[k]) + margin;
      nk += nk & 1;
      nk = std::min(na, std::max(nk, 8));
    }
    if (out) out[k] = nk;
    q += nk;
  }
  return q;
}

// Warp-slot cost of a grid of q points in 64-point work units whose last unit runs one point per lane when it has
// <= 32 points (k_pairs_grid_w): full units x 64 + (0 | 32 | 64)
static int warp_slots(int q) {
  const int rem = q % 64;
  return q - rem + (rem == 0 ? 0 : rem <= 32 ? 32 : 64);
}

// NC_RING_FILL (default on): when a multiple of 32 points lies between the grid at the floor margin (6) and at the
// default margin (8), trim the default grid down to it (two points at a time, outermost adapted rings first, never
// below the floor's ring sizes): the last work unit then has no idle lanes.
static bool ring_fill() {
  static int v = -1;
  if (v < 0) {
    const char* e = tuning_env("NC_RING_FILL");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

static int ring_floor() {   // the smallest margin ring filling may trim to (NC_RING_FLOOR, default 6)
  static int v = -1;
  if (v < 0) {
    const char* e = tuning_env("NC_RING_FLOOR");
    v = e ? std::max(0, atoi(e)) : 6;
  }
  return v;
}

static int ring_points(double beta, double tol, int nr, int na, int* out /* nr, or nullptr */) {
  if (nr > kRingMax) nr = kRingMax;   // (grid_size gives n_r ~ 10 at the tightest precisions)
  double fit[kRingMax];
  int hi[kRingMax], lo[kRingMax];
  ring_fit(beta, tol, nr, fit);
  const int qh = ring_points_margin_fit(fit, nr, na, ring_margin(), hi);
  if (!ring_adapt() || !ring_fill() || ring_margin() <= ring_floor()) {
    if (out) std::copy(hi, hi + nr, out);
    return qh;
  }
  const int ql = ring_points_margin_fit(fit, nr, na, ring_floor(), lo);
  int target = qh - (qh % 32);   // the largest multiple of 32 <= qh
  if (target < ql || warp_slots(target) >= warp_slots(qh)) target = qh;
  int q = qh;
  for (bool progress = true; q > target && progress;) {
    progress = false;
    for (int k = 0; k < nr && q > target; ++k)
      if (hi[k] - 2 >= lo[k]) {
        hi[k] -= 2;
        q -= 2;
        progress = true;
      }
  }
  if (out) std::copy(hi, hi + nr, out);
  return q;
}
static inline double harc(const double* a, const double* b) {
  double cx = a[1] * b[2] - a[2] * b[1], cy = a[2] * b[0] - a[0] * b[2], cz = a[0] * b[1] - a[1] * b[0];
  return atan2(sqrt(cx * cx + cy * cy + cz * cz), a[0] * b[0] + a[1] * b[1] + a[2] * b[2]);
}

// ------------------------------------------------------------------------------------------------
// entry points used by api.cu
// ------------------------------------------------------------------------------------------------
int hier_order(nc_handle* h, std::vector<double>& centers) {
  const int64_t N = h->N;
  HierState* H = new HierState();
  H->gv = grid_variant_for(h->precision);
  h->hier = H;
  cudaStream_t s = h->stream;
  double* d_c = nullptr;
  int64_t *d_k0 = nullptr, *d_i0 = nullptr, *d_i1 = nullptr;
  int* d_sep = nullptr;
  int* d_dup = nullptr;
  NC_TRY(halloc(h, &d_c, 3 * N));
  NC_TRY(halloc(h, &d_k0, N));
  NC_TRY(halloc(h, &H->d_keys, N));
  NC_TRY(halloc(h, &d_i0, N));
  NC_TRY(halloc(h, &d_i1, N));
  NC_TRY(halloc(h, &d_sep, std::max<int64_t>(N, 1)));
  NC_TRY(halloc(h, &d_dup, 1));
  NC_CUDA_TRY(cudaMemcpyAsync(d_c, centers.data(), 3 * N * sizeof(double), cudaMemcpyHostToDevice, s));
  NC_CUDA_TRY(cudaMemsetAsync(d_dup, 0, sizeof(int), s));
  k_keys<<<(unsigned)((N + 255) / 256), 256, 0, s>>>(d_c, N, d_k0, d_i0);
  size_t tmp = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp, d_k0, H->d_keys, d_i0, d_i1, (int)N, 0, 3 + 2 * kLmax, s);
  void* d_tmp = nullptr;
  NC_CUDA_TRY(cudaMalloc(&d_tmp, std::max<size_t>(tmp, 16)));
  cub::DeviceRadixSort::SortPairs(d_tmp, tmp, d_k0, H->d_keys, d_i0, d_i1, (int)N, 0, 3 + 2 * kLmax, s);
  int L = 0;
  if (N > 1) {
    k_sep<<<(unsigned)((N + 255) / 256), 256, 0, s>>>(H->d_keys, N, d_sep, d_dup);
    int* d_L = d_dup + 0;   // reuse after reading dup
    int dup = 0;
    NC_CUDA_TRY(cudaMemcpyAsync(&dup, d_dup, sizeof(int), cudaMemcpyDeviceToHost, s));
    NC_CUDA_TRY(cudaStreamSynchronize(s));
    if (dup) {
      cudaFree(d_tmp);
      return fail(NC_ESEP, "nc_setup (hier): two centres fall in the same finest cube cell (coincident patches)");
    }
    size_t tmp2 = 0;
    cub::DeviceReduce::Max(nullptr, tmp2, d_sep, d_L, (int)(N - 1), s);
    if (tmp2 > tmp) {
      cudaFree(d_tmp);
      NC_CUDA_TRY(cudaMalloc(&d_tmp, tmp2));
      tmp = tmp2;
    }
    cub::DeviceReduce::Max(d_tmp, tmp, d_sep, d_L, (int)(N - 1), s);
    NC_CUDA_TRY(cudaMemcpyAsync(&L, d_L, sizeof(int), cudaMemcpyDeviceToHost, s));
  }
  std::vector<int64_t> perm;
  NC_TRY(download(perm, d_i1, N, s));
  NC_TRY(download(H->keys, H->d_keys, N, s));
  cudaFree(d_tmp);
  cudaFree(d_c); cudaFree(d_k0); cudaFree(d_i0); cudaFree(d_i1); cudaFree(d_sep); cudaFree(d_dup);
  h->device_bytes -= (double)(3 * N + 3 * N) * 8 + 4.0 * std::max<int64_t>(N, 1) + 4;
  H->L = L;
  h->perm = perm;
  std::vector<double> sorted(3 * N);
  for (int64_t i = 0; i < N; ++i)
    for (int d = 0; d < 3; ++d) sorted[3 * i + d] = centers[3 * perm[i] + d];
  centers.swap(sorted);
  return NC_OK;
}

// Step 4 through proxies (R36, proxy.cu): the rules for the tables' nodes, their thresholds, the per-grid
// nearest-source arcs, the proxies of every local patch and the buffers of the proxy passes.  Off (nprule = 0) with
// NC_PROXY=0 (tuning).  A rule is dropped when it cannot be built, never meets its tolerance, would not save evaluations
// (n > K* / 2), or does not lower the threshold of the smaller rules.  The rules' tolerance is kProxyTolFactor x the
// grids' own (NC_PROXY_TOL overrides); NC_PROXY_RULES="deg,nring,cphi;..." overrides the rule list.
constexpr double kProxyTolFactor = 0.1;
constexpr int kMaxProxyRules = 3;
template <class Plan>
static int proxy_setup(nc_handle* h, HierState* H, const std::vector<Plan>& plans, const std::vector<int32_t>& pgl,
                       const std::vector<double>& cen, double tol, cudaStream_t s) {
  const int Ks = h->Kstar;
  const int64_t rc = h->row_count, rb = h->row_begin;
  H->nprule = 0;
  H->proxy_n = 0;
  if (const char* e = tuning_env("NC_PROXY"))
    if (e[0] == '0') return NC_OK;
  if (rc <= 0 || H->L > 31) return NC_OK;
  // default rules: 32 points (degree 6) and 64 (degree 8), thresholds D / h = 9 and 5.4 at the default tolerance
  // (profiles/r03l_proxy_rules_sweep.jsonl: C5 step 4 + rest 9.20 ms with these two, 9.42 with the 64-point rule
  // alone, 9.30 / 9.53 with a 124-point degree-13 rule (threshold 3.1) added for the levels now at the nodes)
  struct Spec {
    int deg, nring;
    double cphi;
  };
  std::vector<Spec> specs = {{6, 3, 15.0}, {8, 4, 24.0}};
  if (const char* e = tuning_env("NC_PROXY_RULES")) {
    specs.clear();
    const char* p = e;
    Spec sp;
    int used = 0;
    while (sscanf(p, "%d,%d,%lf%n", &sp.deg, &sp.nring, &sp.cphi, &used) == 3) {
      specs.push_back(sp);
      p += used;
      if (*p != ';') break;
      ++p;
    }
  }
  double tf = kProxyTolFactor;
  if (const char* e = tuning_env("NC_PROXY_TOL")) tf = atof(e);
  std::vector<double> z;
  NC_TRY(download(z, h->d_zhat, (size_t)3 * Ks, s));
  struct Built {
    int n = 0;
    double kappa = HUGE_VAL, h = 0.0;
    std::vector<double> pts, Int;
  };
  std::vector<Built> built;
  for (const Spec& sp : specs) {
    Built b;
    b.n = proxy_rule_build(z.data(), Ks, sp.deg, sp.nring, sp.cphi, tf * tol, b.pts, b.Int, &b.kappa, &b.h);
    if (b.n > 0 && b.kappa < HUGE_VAL && 2 * b.n <= Ks && !(b.n & 1)) built.push_back(std::move(b));
  }
  std::sort(built.begin(), built.end(), [](const Built& a, const Built& b) { return a.n < b.n; });
  std::vector<Built> rules;
  for (Built& b : built)
    if ((int)rules.size() < kMaxProxyRules && (rules.empty() || b.kappa < rules.back().kappa))
      rules.push_back(std::move(b));
  if (rules.empty()) return NC_OK;
  const double hh = rules[0].h;
  H->nprule = (int)rules.size();
  H->proxy_n = rules[0].n;
  H->proxy_kappa = rules.back().kappa;
  for (int r = 0; r < H->nprule; ++r) {
    HierState::PRule& R = H->prule[r];
    R.n = rules[r].n;
    R.kh = rules[r].kappa * hh;
    NC_TRY(upload(h, &R.Int, rules[r].Int, s));
    double* d_ph = nullptr;
    NC_TRY(upload(h, &d_ph, rules[r].pts, s));
    NC_TRY(halloc(h, &R.ptx, rc * R.n));
    NC_TRY(halloc(h, &R.pty, rc * R.n));
    NC_TRY(halloc(h, &R.ptz, rc * R.n));
    NC_TRY(halloc(h, &R.V, rc * R.n));
    launch_targets(h->d_frames, rb, rc, d_ph, R.n, 0.5, R.ptx, R.pty, R.ptz, s);
    NC_CUDA_TRY(cudaStreamSynchronize(s));
    cudaFree(d_ph);
  }
  // per grid: arc from its cap centre to the nearest source node, beta R = d - eps (R12/R21: the skeleton lies within
  // eps of its patch centre), so a patch centre at arc a0 from the cap centre is >= beta R - a0 from every source
  std::vector<double> gd(std::max<size_t>(plans.size(), 1), 0.0);
  for (size_t k = 0; k < plans.size(); ++k) gd[k] = plans[k].beta * H->gR[plans[k].group];
  // the split, once, on the host: the 2-bit code of patch i's level lvl is r + 1 for the smallest rule r whose
  // threshold its grids' nearest source clears, 0 (nodes) if none (single-member groups stay with k_interp_sep)
  const int L = H->L;
  std::vector<uint64_t> pcode(rc, 0ull);
  std::vector<int32_t> work1;
  double npair = 0.0, nfar = 0.0;
  std::vector<int64_t> per_rule(H->nprule + 1, 0);
  const double dbin[] = {2.0, 3.0, 3.125, 4.0, 5.375, 7.0, 9.0, 12.0, 20.0, HUGE_VAL};
  int64_t dhist[10] = {0};   // NC_HIER_DIAG: D / h of the (patch, multi-member level) pairs
  for (int64_t i = 0; i < rc; ++i) {
    bool near_level = false;
    for (int lvl = 0; lvl <= L; ++lvl) {
      const int32_t g = pgl[(size_t)lvl * rc + i];
      const int64_t kg0 = H->ggrid0[g], kg1 = H->ggrid0[g + 1];
      if (kg0 == kg1 || H->gnr[kg0] == 0) continue;
      if (H->sep_nodes && H->glast[g] - H->gfirst[g] == 1) continue;   // k_interp_sep's
      double dmin = HUGE_VAL;
      for (int64_t kg = kg0; kg < kg1; ++kg) dmin = std::min(dmin, gd[kg]);
      npair += 1.0;
      const double dist = dmin - harc(&H->gc[3 * (int64_t)g], &cen[3 * (rb + i)]);
      {
        int b = 0;
        while (dist / hh >= dbin[b]) ++b;
        ++dhist[b];
      }
      int code = 0;
      for (int r = 0; r < H->nprule && !code; ++r)
        if (dist >= H->prule[r].kh) code = r + 1;
      ++per_rule[code];
      if (code) {
        pcode[i] |= (uint64_t)code << (2 * lvl);
        nfar += 1.0;
      } else {
        near_level = true;
      }
    }
    if (near_level) work1.push_back((int32_t)i);
  }
  H->proxy_pairs = npair;
  H->proxy_far = nfar;
  H->npwork1 = (int64_t)work1.size();
  NC_TRY(upload(h, &H->d_pcode, pcode, s));
  if (work1.empty()) work1.push_back(0);
  NC_TRY(upload(h, &H->d_pwork1, work1, s));
  if (getenv("NC_HIER_DIAG")) {
    fprintf(stderr, "[nc hier diag] step-4 proxies (h %.3g): nodes %lld", hh, (long long)per_rule[0]);
    for (int r = 0; r < H->nprule; ++r)
      fprintf(stderr, ", rule %d (n %d, kappa %.3f) %lld", r, H->prule[r].n, H->prule[r].kh / hh,
              (long long)per_rule[r + 1]);
    fprintf(stderr, " (patch, level) pairs\n[nc hier diag] D/h histogram (upper edges 2 3 3.125 4 5.375 7 9 12 20 inf):");
    for (int b = 0; b < 10; ++b) fprintf(stderr, " %lld", (long long)dhist[b]);
    fprintf(stderr, "\n");
  }
  return NC_OK;
}

int hier_setup(nc_handle* h, const std::vector<double>& cen, cudaStream_t s) {
  HierState* H = h->hier;
  const int64_t N = h->N;
  // the host parts of the setup run on OpenMP threads; the ranks of one node share its cores (one process per GPU),
  // so each takes its share (NC_SETUP_THREADS overrides)
  if (const char* e = getenv("NC_SETUP_THREADS")) {
    omp_set_num_threads(std::max(1, atoi(e)));
  } else if (h->world > 1) {
    omp_set_num_threads(std::max(1, omp_get_num_procs() / h->world));
  }
  const int L = H->L;
  const double eps = h->eps;
  const int Ks = h->Kstar, p = h->p;
  // ---- node rings of the canonical Zernike nodes (separable step 4 for single-member groups) ----
  {
    const char* e = tuning_env("NC_INTERP_SEP");
    std::vector<double> z;
    NC_TRY(download(z, h->d_zhat, (size_t)3 * Ks, s));
    H->node_ring.assign(Ks, -1);
    H->node_cs.assign(2 * (size_t)Ks, 0.0);
    H->ring_t.clear();
    bool ok = !(e && e[0] == '0');
    for (int k = 0; k < Ks && ok; ++k) {
      const double rho = std::hypot(z[3 * k], z[3 * k + 1]);
      const double t = std::atan2(rho, z[3 * k + 2]);   // geodesic radius (unit sphere)
      if (!(rho > 0.0)) { ok = false; break; }         // a node at the centre has no angle
      H->node_cs[2 * k] = z[3 * k] / rho;
      H->node_cs[2 * k + 1] = z[3 * k + 1] / rho;
      int a = 0;
      for (; a < (int)H->ring_t.size(); ++a)
        if (std::fabs(H->ring_t[a] - t) <= 1e-13 * std::max(1.0, t)) break;
      if (a == (int)H->ring_t.size()) H->ring_t.push_back(t);
      H->node_ring[k] = a;
    }
    // worth it only when the rings are few (a tensor-product node set: nA rings x angles)
    H->nring = (int)H->ring_t.size();
    H->sep_nodes = ok && H->nring > 0 && 4 * H->nring <= Ks;
  }
  // ---- boxes per level (device flags + scan) ----
  int *d_flag = nullptr, *d_scan = nullptr;
  NC_TRY(halloc(h, &d_flag, N));
  NC_TRY(halloc(h, &d_scan, N));
  size_t tmp = 0;
  cub::DeviceScan::InclusiveSum(nullptr, tmp, d_flag, d_scan, (int)N, s);
  void* d_tmp = nullptr;
  NC_CUDA_TRY(cudaMalloc(&d_tmp, std::max<size_t>(tmp, 16)));
  H->lvl_off.assign(L + 2, 0);
  H->pgroup.assign((size_t)(L + 1) * N, 0);
  std::vector<int> flag(N), scan(N);
  for (int lvl = 0; lvl <= L; ++lvl) {
    k_box_flags<<<(unsigned)((N + 255) / 256), 256, 0, s>>>(H->d_keys, N, lvl, d_flag);
    cub::DeviceScan::InclusiveSum(d_tmp, tmp, d_flag, d_scan, (int)N, s);
    NC_TRY(download(flag, d_flag, N, s));
    NC_TRY(download(scan, d_scan, N, s));
    const int64_t nb = scan[N - 1];
    const int64_t base = H->lvl_off[lvl];
    H->lvl_off[lvl + 1] = base + nb;
    for (int64_t i = 0; i < N; ++i) {
      const int64_t g = base + scan[i] - 1;
      H->pgroup[(size_t)lvl * N + i] = (int32_t)g;
      if (flag[i]) {
        H->gfirst.push_back((int32_t)i);
        H->gkey.push_back(H->keys[i] >> (2 * (kLmax - lvl)));
        H->glevel.push_back(lvl);
      }
    }
  }
  cudaFree(d_flag); cudaFree(d_scan); cudaFree(d_tmp);
  h->device_bytes -= 8.0 * N;
  const int64_t G = H->lvl_off[L + 1];
  H->ngroups = G;
  H->glast.resize(G);
  for (int lvl = 0; lvl <= L; ++lvl)
    for (int64_t g = H->lvl_off[lvl]; g < H->lvl_off[lvl + 1]; ++g)
      H->glast[g] = (g + 1 < H->lvl_off[lvl + 1]) ? H->gfirst[g + 1] : (int32_t)N;

  setup_tick("boxes per level");
  // ---- neighbours, interaction lists, circles (device) ----
  int64_t *d_gkey = nullptr, *d_lvl = nullptr, *d_cnt = nullptr, *d_off = nullptr;
  int32_t *d_nbr = nullptr, *d_gfirst = nullptr, *d_glast = nullptr, *d_pg = nullptr, *d_il = nullptr;
  double *d_cen = nullptr, *d_gc = nullptr;
  NC_TRY(upload(h, &d_gkey, H->gkey, s));
  NC_TRY(upload(h, &d_lvl, H->lvl_off, s));
  NC_TRY(upload(h, &d_gfirst, H->gfirst, s));
  NC_TRY(upload(h, &d_glast, H->glast, s));
  NC_TRY(upload(h, &d_pg, H->pgroup, s));
  NC_TRY(upload(h, &d_cen, cen, s));
  NC_TRY(halloc(h, &d_nbr, 8 * G));
  NC_TRY(halloc(h, &d_cnt, G));
  NC_TRY(halloc(h, &d_off, G + 1));
  NC_TRY(halloc(h, &d_gc, 3 * G));
  NC_TRY(halloc(h, &H->d_gR, G));
  NC_TRY(halloc(h, &H->d_gframe, 9 * G));
  const unsigned gb = (unsigned)((G + 127) / 128);
  k_neighbors<<<gb, 128, 0, s>>>(d_gkey, d_lvl, L, G, d_nbr);
  k_ilist<<<gb, 128, 0, s>>>(d_gkey, d_lvl, L, G, d_nbr, d_gfirst, d_pg, N, nullptr, d_cnt, nullptr);
  tmp = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp, d_cnt, d_off, (int)G, s);
  NC_CUDA_TRY(cudaMalloc(&d_tmp, std::max<size_t>(tmp, 16)));
  cub::DeviceScan::ExclusiveSum(d_tmp, tmp, d_cnt, d_off, (int)G, s);
  std::vector<int64_t> cnt;
  NC_TRY(download(cnt, d_cnt, G, s));
  NC_TRY(download(H->il_off, d_off, G, s));
  H->il_off.push_back(G ? H->il_off[G - 1] + cnt[G - 1] : 0);
  const int64_t nil = H->il_off[G];
  NC_TRY(halloc(h, &d_il, std::max<int64_t>(nil, 1)));
  k_ilist<<<gb, 128, 0, s>>>(d_gkey, d_lvl, L, G, d_nbr, d_gfirst, d_pg, N, d_off, d_cnt, d_il);
  k_circles<<<(unsigned)((32 * G + 127) / 128), 128, 0, s>>>(d_cen, d_gfirst, d_glast, G, eps, d_gc, H->d_gR);
  k_group_frames<<<gb, 128, 0, s>>>(d_gc, G, H->d_gframe);
  if (H->sep_nodes) k_single_frames<<<gb, 128, 0, s>>>(d_gfirst, d_glast, G, h->d_frames, d_gc, H->d_gframe);
  NC_TRY(download(H->nbr, d_nbr, 8 * G, s));
  NC_TRY(download(H->il, d_il, nil, s));
  NC_TRY(download(H->gc, d_gc, 3 * G, s));
  NC_TRY(download(H->gR, H->d_gR, G, s));
  {
    std::vector<double> rinv(G);
    for (int64_t g = 0; g < G; ++g) rinv[g] = 1.0 / H->gR[g];
    NC_TRY(upload(h, &H->d_gRinv, rinv, s));
  }
  // step-4 node geometry (k_interp): a node's arc from the group centre is arc(patch centre) + asin(sin(difference));
  // |difference| <= eps, and the series s (1 + s^2/6 + 3 s^4/40 + ...) needs n terms for |s|^(2n+1)/(2n+1) < 1e-17
  {
    const double smax = std::sin(1.02 * eps);
    H->asin_terms = 0;
    if (smax < 0.2)
      for (int n = 1; n <= 10; ++n)
        if (std::pow(smax, 2 * n + 1) / (2 * n + 1) < 1e-17) {
          H->asin_terms = n;
          break;
        }
  }
  cudaFree(d_tmp);
  for (void* q : {(void*)d_gkey, (void*)d_lvl, (void*)d_cnt, (void*)d_off, (void*)d_nbr, (void*)d_gfirst,
                  (void*)d_glast, (void*)d_pg, (void*)d_il, (void*)d_cen, (void*)d_gc})
    cudaFree(q);
  NC_CUDA_TRY(cudaGetLastError());

  setup_tick("neighbours, lists, caps (dev)");
  // ---- grid vs near routing, grid sizes (host) ----
  // per-grid interpolation tolerance = kGridTolFactor x requested precision (calibrated, R21;
  // NC_GRID_TOL_FACTOR overrides for calibration runs)
  double tol_factor = kGridTolFactor;
  if (const char* e = tuning_env("NC_GRID_TOL_FACTOR")) tol_factor = atof(e);
  const double tol = tol_factor * h->precision;
  {
    const char* et = tuning_env("NC_INTERP_TRUNC");
    H->interp_lt = (et && et[0] == '0') ? 0.0 : log(1.0 / tol);
  }
  // relative costs in grid-pair units (measured at C5): a near-list pair (exact form), one
  // interpolation term (node x coefficient), one transform term; NC_COST_NEAR / _INTERP / _TRANSFORM override
  double c_near = kCostNear, c_interp = kCostInterp, c_trans = kCostTransform;
  if (const char* e = tuning_env("NC_COST_NEAR")) c_near = atof(e);
  if (const char* e = tuning_env("NC_COST_INTERP")) c_interp = atof(e);
  if (const char* e = tuning_env("NC_COST_TRANSFORM")) c_trans = atof(e);
  // Incoming grids per group (§8.1 :1424-1434): the group's interaction-list / leaf-neighbour
  // sources, sorted by beta = (distance - eps) / R descending, are cut into up to kMaxGrids consecutive bands, each
  // on its own grid sized by the band's nearest source, and a near tail evaluated directly at the members' Zernike
  // nodes (R12, R24).  The cut minimises the cost model (grid-pair units).
  int max_grids = kDefaultGrids;
  if (const char* e = tuning_env("NC_MAX_GRIDS")) max_grids = std::max(1, std::min(kMaxGrids, atoi(e)));
  int ncuts = kGridCutQuantiles;
  if (const char* e = tuning_env("NC_GRID_CUTS")) ncuts = std::max(4, std::min(512, atoi(e)));
  // every group's candidate sources, sorted, in flat arrays: group g's live at [cand_off[g], cand_off[g + 1]); its
  // grids take consecutive bands of them, its near tail the rest (sorted by patch).  No per-group heap objects: the
  // routing runs over ~2e5 groups at C5 and per-group vectors made it allocator-bound.
  std::vector<int64_t> cand_off(G + 1, 0);
#pragma omp parallel for schedule(dynamic, 256)
  for (int64_t g = 0; g < G; ++g) {
    int64_t c = 0;
    for (int64_t k = H->il_off[g]; k < H->il_off[g + 1]; ++k) c += H->glast[H->il[k]] - H->gfirst[H->il[k]];
    if (H->glevel[g] == L)
      for (int k = 0; k < 8; ++k)
        if (H->nbr[8 * g + k] >= 0) c += H->glast[H->nbr[8 * g + k]] - H->gfirst[H->nbr[8 * g + k]];
    cand_off[g + 1] = c;
  }
  for (int64_t g = 0; g < G; ++g) cand_off[g + 1] += cand_off[g];
  std::vector<int32_t> F_src((size_t)cand_off[G]);
  std::vector<int32_t> F_rung((size_t)cand_off[G]);
  std::vector<double> F_dist((size_t)cand_off[G]);   // arc distance from the group's cap centre to each source centre
  struct GridPlan {
    int32_t group = 0, nr = 0, na = 0;
    int32_t cnt = 0;            // its sources: F_src / F_rung / F_dist [off, off + cnt)
    int64_t off = 0;
    double beta = 0.0;          // the grid's nearest source (its size)
  };
  std::vector<GridPlan> gp_slot((size_t)G * kMaxGrids);
  std::vector<int8_t> gp_cnt(G, 0);
  std::vector<int64_t> near_beg(G, 0), near_end(G, 0);   // the near tail of group g: F_src [near_beg, near_end)
  std::vector<double> gwork(G, 0.0);
  const bool diag = getenv("NC_HIER_DIAG") != nullptr;
  double diag_cost = 0.0;
  int64_t diag_groups2 = 0;
  // groups are independent: host threads (OpenMP) with per-thread scratch, results in per-group slots
  const bool sub_timing = getenv("NC_SETUP_TIMING") != nullptr;
  std::vector<double> rt_acc((size_t)std::max(1, omp_get_max_threads()) * 6, 0.0);   // per-thread sub-phase seconds
#pragma omp parallel reduction(+ : diag_cost, diag_groups2)
  {
  double* rt = rt_acc.data() + (size_t)omp_get_thread_num() * 6;
  double tmark = 0.0;
  auto lap = [&](int k) {
    if (!sub_timing) return;
    const double t = omp_get_wtime();
    if (k >= 0) rt[k] += t - tmark;
    tmark = t;
  };
  std::vector<std::pair<double, int32_t>> cand;
  std::vector<int> rung_of;
  std::vector<double> psum, qi, ovh, dp;
  std::vector<size_t> qs, cuts;
  std::vector<int> from;
  // dynamic 1: the few coarse-level groups (thousands of candidates each) come first and must spread over threads
#pragma omp for schedule(dynamic, 1)
  for (int64_t g = 0; g < G; ++g) {
    const int lvl = H->glevel[g];
    const double* cg = &H->gc[3 * g];
    const double R = H->gR[g];
    const int64_t mem = H->glast[g] - H->gfirst[g];
    cand.clear();
    lap(-1);
    auto add_box = [&](int64_t b) {
      for (int32_t j = H->gfirst[b]; j < H->glast[b]; ++j) {
        const double d = harc(cg, &cen[3 * (int64_t)j]);
        const bool valid = d >= R + 2.0 * eps * (1.0 + 1e-12);
        const double beta = valid ? (d - eps) / R : 0.0;
        cand.push_back({beta, j});
      }
    };
    for (int64_t k = H->il_off[g]; k < H->il_off[g + 1]; ++k) add_box(H->il[k]);
    if (lvl == L)
      for (int k = 0; k < 8; ++k)
        if (H->nbr[8 * g + k] >= 0) add_box(H->nbr[8 * g + k]);
    if (cand.empty()) continue;
    lap(0);
    std::sort(cand.begin(), cand.end(), [](const std::pair<double, int32_t>& a, const std::pair<double, int32_t>& b) {
      return a.first > b.first || (a.first == b.first && a.second < b.second);
    });
    lap(1);
    // grid sources use the outgoing-operator rung valid at their distance to the nearest grid point,
    // gap = d - R = R (beta - 1) + eps (per-level recompression)
    const size_t nc = cand.size();
    const int p0 = h->rung_p[0];
    rung_of.assign(nc, 0);
    psum.assign(nc + 1, 0.0);   // sum of the rung sizes of the n farthest candidates
    for (size_t n = 0; n < nc; ++n) {
      const double gap = R * (cand[n].first - 1.0) + eps;
      int rung = 0;   // the smallest skeleton among the rungs valid on the whole grid (r_k <= gap)
      for (int k = 1; k < h->nrung; ++k)
        if (h->rung_r[k] <= gap * (1.0 - 1e-12) && h->rung_p[k] <= h->rung_p[rung]) rung = k;
      rung_of[n] = rung;
      psum[n + 1] = psum[n] + h->rung_p[rung];
    }
    // a band [a, b) of the sorted candidates on one grid sized by cand[b - 1]: pair evaluations on its q points
    // (each source with its own rung) + interpolation to the members' nodes + transform
    auto band = [&](size_t a, size_t b, int& nr, int& na) {
      grid_size(cand[b - 1].first, tol, nr, na);
      const double q = (double)ring_points(cand[b - 1].first, tol, nr, na, nullptr);
      return q * (psum[b] - psum[a]) + c_interp * (double)mem * Ks * q + c_trans * q * (nr + na);
    };
    auto near_cost = [&](size_t b) { return c_near * (double)mem * Ks * (double)(nc - b) * p0; };
    lap(2);
    size_t n_ok = 0;   // candidates a grid may serve (beta >= kBetaMin)
    while (n_ok < nc && cand[n_ok].first >= kBetaMin) ++n_ok;
    double best_cost = near_cost(0);   // all direct
    size_t cut2 = 0;                   // best single grid: [0, cut2)
    for (size_t n = 1; n <= n_ok; ++n) {   // one grid: exhaustive over distinct betas
      if (n < nc && cand[n].first == cand[n - 1].first) continue;
      int nr, na;
      const double c = band(0, n, nr, na) + near_cost(n);
      if (c < best_cost) { best_cost = c; cut2 = n; }
    }
    // K >= 2 bands: dynamic programme over cut points on kGridCutQuantiles quantiles of the servable candidates;
    // a band ending at cut i lives on a grid sized by cand[cut_i - 1] (its q and overhead precomputed per cut)
    lap(3);
    cuts.clear();   // band boundaries chosen (ascending, last = end of the grid-served prefix)
    if (max_grids >= 2 && n_ok >= 2) {
      qs.clear();
      for (int k = 1; k <= ncuts; ++k) qs.push_back(std::max<size_t>(1, (n_ok * k) / ncuts));
      qs.erase(std::unique(qs.begin(), qs.end()), qs.end());
      const int Q = (int)qs.size();
      qi.assign(Q, 0.0);
      ovh.assign(Q, 0.0);
      for (int i = 0; i < Q; ++i) {
        int nr, na;
        grid_size(cand[qs[i] - 1].first, tol, nr, na);
        qi[i] = (double)ring_points(cand[qs[i] - 1].first, tol, nr, na, nullptr);
        ovh[i] = c_interp * (double)mem * Ks * qi[i] + c_trans * qi[i] * (nr + na);
      }
      // dp[k Q + i]: cheapest cover of [0, qs[i]) by k bands; from[k Q + i]: previous cut index (-1: starts at 0)
      dp.assign((size_t)(max_grids + 1) * Q, 1e300);
      from.assign((size_t)(max_grids + 1) * Q, -1);
      for (int i = 0; i < Q; ++i) dp[1 * Q + i] = qi[i] * psum[qs[i]] + ovh[i];
      for (int k = 2; k <= max_grids; ++k)
        for (int i = 1; i < Q; ++i)
          for (int j = 0; j < i; ++j) {
            const double c = dp[(k - 1) * Q + j] + qi[i] * (psum[qs[i]] - psum[qs[j]]) + ovh[i];
            if (c < dp[k * Q + i]) { dp[k * Q + i] = c; from[k * Q + i] = j; }
          }
      int bk = 0, bi = -1;
      for (int k = 2; k <= max_grids; ++k)
        for (int i = 0; i < Q; ++i) {
          const double c = dp[k * Q + i] + near_cost(qs[i]);
          if (c < best_cost) { best_cost = c; bk = k; bi = i; }
        }
      for (int k = bk, i = bi; k >= 1 && i >= 0; i = from[k * Q + i], --k) cuts.push_back(qs[i]);
      std::reverse(cuts.begin(), cuts.end());
    }
    lap(4);
    if (cuts.empty() && cut2 > 0) cuts.push_back(cut2);   // the best single grid
    const int64_t o0 = cand_off[g];
    auto emit = [&](size_t a, size_t b) {
      GridPlan gp;
      gp.group = (int32_t)g;
      grid_size(cand[b - 1].first, tol, gp.nr, gp.na);
      gp.beta = cand[b - 1].first;
      gp.off = o0 + (int64_t)a;
      gp.cnt = (int32_t)(b - a);
      for (size_t n = a; n < b; ++n) {
        F_src[o0 + n] = cand[n].second;
        F_rung[o0 + n] = rung_of[n];
        F_dist[o0 + n] = R * cand[n].first + eps;   // beta = (d - eps) / R
      }
      gp_slot[(size_t)g * kMaxGrids + gp_cnt[g]++] = gp;
    };
    size_t prev = 0;
    for (size_t c : cuts) {
      emit(prev, c);
      prev = c;
    }
    for (size_t n = prev; n < nc; ++n) F_src[o0 + n] = cand[n].second;
    std::sort(F_src.begin() + o0 + prev, F_src.begin() + o0 + nc);
    near_beg[g] = o0 + (int64_t)prev;
    near_end[g] = o0 + (int64_t)nc;
    gwork[g] = best_cost;
    diag_cost += best_cost;
    diag_groups2 += cuts.size() > 1;
    lap(5);
  }
  }
  if (sub_timing) {
    double tot[6] = {0, 0, 0, 0, 0, 0};
    for (size_t t = 0; t < rt_acc.size(); ++t) tot[t % 6] += rt_acc[t];
    fprintf(stderr, "[nc setup]   routing thread-seconds: gather %.3f sort %.3f rungs %.3f single-grid %.3f dp %.3f "
                    "emit %.3f\n", tot[0], tot[1], tot[2], tot[3], tot[4], tot[5]);
  }
  setup_tick("routing: per-group plans (host, parallel)");
  std::vector<GridPlan> plans;
  H->ggrid0.assign(G + 1, 0);
  for (int64_t g = 0; g < G; ++g) {
    H->ggrid0[g] = (int64_t)plans.size();
    for (int q = 0; q < gp_cnt[g]; ++q) plans.push_back(gp_slot[(size_t)g * kMaxGrids + q]);
  }
  H->ggrid0[G] = (int64_t)plans.size();
  if (diag)
    fprintf(stderr, "[nc hier diag] cost %.4g, grids %zu, groups with several grids %lld, max grids %d\n", diag_cost,
            plans.size(), (long long)diag_groups2, max_grids);

  setup_tick("routing + grid bands (host)");
  // rungs in use: a global decision (identical on every rank, so the per-rung all-gathers match)
  {
    std::vector<char> used((size_t)std::max(1, omp_get_max_threads()) * h->nrung, 0);
#pragma omp parallel for schedule(dynamic, 1024)
    for (int64_t k = 0; k < (int64_t)plans.size(); ++k) {
      char* u = used.data() + (size_t)omp_get_thread_num() * h->nrung;
      for (int32_t n = 0; n < plans[k].cnt; ++n) u[F_rung[plans[k].off + n]] = 1;
    }
    for (size_t e = 0; e < used.size(); ++e)
      if (used[e]) h->rung_used[e % h->nrung] = 1;
  }

  // ---- partition: contiguous internal rows, weighted by work (world > 1) ----
  {
    std::vector<double> w(N, 0.0);
    for (int64_t g = 0; g < G; ++g) {
      const int64_t mem = H->glast[g] - H->gfirst[g];
      for (int32_t i = H->gfirst[g]; i < H->glast[g]; ++i) w[i] += gwork[g] / (double)mem;
    }
    h->rank_begin.assign(h->world, 0);
    h->rank_count.assign(h->world, 0);
    split_rows(w.data(), N, h->world, h->rank_begin.data(), h->rank_count.data());
    h->row_begin = h->rank_begin[h->rank];
    h->row_count = h->rank_count[h->rank];
  }
  const int64_t rb = h->row_begin, rc = h->row_count, re = rb + rc;

  // ---- groups relevant to this rank: those containing a local patch ----
  std::vector<char> rel(G, 0);
  for (int lvl = 0; lvl <= L && rc > 0; ++lvl) {
    const int64_t g0 = H->pgroup[(size_t)lvl * N + rb], g1 = H->pgroup[(size_t)lvl * N + re - 1];
    for (int64_t g = g0; g <= g1; ++g) rel[g] = 1;
  }
  // per-grid sizes and point / coefficient offsets (grids of irrelevant groups get no points)
  const int64_t NG = (int64_t)plans.size();
  H->ngrids = NG;
  H->gnr.assign(NG, 0);
  H->gna.assign(NG, 0);
  H->grid_group.assign(NG, 0);
  H->goff.assign(NG + 1, 0);
  H->coff.assign(NG + 1, 0);
  H->rbase.assign(NG + 1, 0);
  H->roff.clear();
  H->grid_ids.clear();
  // ring sizes of every relevant grid in parallel (ring_points per grid), then the offsets in grid order
  std::vector<int64_t> qk(NG, 0), rb0(NG + 1, 0);
  for (int64_t k = 0; k < NG; ++k) rb0[k + 1] = rb0[k] + (rel[plans[k].group] ? plans[k].nr + 1 : 0);
  H->roff.assign((size_t)rb0[NG], 0);
#pragma omp parallel for schedule(dynamic, 256)
  for (int64_t k = 0; k < NG; ++k) {
    const GridPlan& gp = plans[k];
    if (!rel[gp.group]) continue;
    int rs[kRingMax];
    qk[k] = ring_points(gp.beta, tol, gp.nr, gp.na, rs);
    int32_t* ro = H->roff.data() + rb0[k];
    ro[0] = 0;
    for (int kr = 0; kr < gp.nr; ++kr) ro[kr + 1] = ro[kr] + rs[kr];
  }
  for (int64_t k = 0; k < NG; ++k) {
    const GridPlan& gp = plans[k];
    H->grid_group[k] = gp.group;
    int64_t q = 0, c = 0;
    H->rbase[k] = rb0[k];
    if (rel[gp.group]) {
      H->gnr[k] = gp.nr;
      H->gna[k] = gp.na;
      q = qk[k];
      c = (int64_t)(gp.na / 2 + 1) * 2 * gp.nr;
      H->grid_ids.push_back((int32_t)k);
      H->qmax = std::max<int>(H->qmax, (int)q);
      H->cmax = std::max<int>(H->cmax, (int)c);
      H->namax = std::max<int>(H->namax, gp.na);
      H->nrmax = std::max<int>(H->nrmax, gp.nr);
    }
    H->goff[k + 1] = H->goff[k] + q;
    H->coff[k + 1] = H->coff[k] + c;
  }
  H->rbase[NG] = (int64_t)H->roff.size();
  H->Q = H->goff[NG];
  H->C = H->coff[NG];
  for (int64_t g = 0; g < G; ++g)
    H->cgroupmax = std::max<int>(H->cgroupmax, (int)(H->coff[H->ggrid0[g + 1]] - H->coff[H->ggrid0[g]]));

  // work units (steps 2-3) and reduction chunks
  H->upts = grid_unit_points(H->gv);
  std::vector<double> rung_pairs(h->nrung, 0.0);
  std::vector<GridUnit> units;
  std::vector<ChunkRec> chunks;
  std::vector<int32_t> srclist;
  // per-chunk rungs (default; NC_CHUNK_RUNGS=0: one rung per (grid, source)): a work unit's points lie on the rings
  // r_kr = R cos((kr + 1/2) pi / (2 n_r)) from its first ring kr0 inward, so the gap from a source to the unit's
  // points is >= d - r_kr0 >= d - R, and the unit may use the smallest skeleton valid at that gap (PAPER.md:1436-1457:
  // the per-level recompression, here keyed by the distance to the unit's points instead of the whole grid's)
  const char* ecr = tuning_env("NC_CHUNK_RUNGS");
  const bool chunk_rungs = !(ecr && ecr[0] == '0');
  bool ladder_monotone = true;   // r_k ascending and p_k non-increasing over k >= 1: binary search
  for (int kk = 2; kk < h->nrung; ++kk)
    ladder_monotone = ladder_monotone && h->rung_r[kk] > h->rung_r[kk - 1] && h->rung_p[kk] <= h->rung_p[kk - 1];
  ladder_monotone = ladder_monotone && (h->nrung < 2 || h->rung_p[1] <= h->rung_p[0]);
  auto best_rung = [&](double gap) {
    const double g = gap * (1.0 - 1e-12);
    if (ladder_monotone) {   // the largest k >= 1 with r_k <= g (0 if none)
      int lo = 1, hi = h->nrung - 1, best = 0;
      while (lo <= hi) {
        const int mid = (lo + hi) / 2;
        if (h->rung_r[mid] <= g) { best = mid; lo = mid + 1; } else hi = mid - 1;
      }
      return best;
    }
    int rung = 0;
    for (int kk = 1; kk < h->nrung; ++kk)
      if (h->rung_r[kk] <= g && h->rung_p[kk] <= h->rung_p[rung]) rung = kk;
    return rung;
  };
  struct Slice { int64_t src0; int32_t nsrc; int rung; };
  // grids are independent: blocks of kBlk grids go to host threads, each appending to its own buffers (no per-grid
  // heap objects); the blocks are then copied into place in grid order with their offsets shifted (in parallel)
  constexpr int64_t kBlk = 8;   // small: the coarse-level grids (thousands of sources each) come first in grid order
  const int64_t NGL = (int64_t)H->grid_ids.size();
  const int64_t nblk = (NGL + kBlk - 1) / kBlk;
  struct BlockOut {
    int thr = 0;
    int64_t u0 = 0, nu = 0, c0 = 0, nc = 0, s0 = 0, ns = 0;   // ranges in the thread's buffers
    double pairs = 0, slot = 0, wslot = 0;
  };
  std::vector<BlockOut> blk(nblk);
  const int nthr = std::max(1, omp_get_max_threads());
  std::vector<std::vector<GridUnit>> T_units(nthr);
  std::vector<std::vector<ChunkRec>> T_chunks(nthr);
  std::vector<std::vector<int32_t>> T_src(nthr);
  std::vector<std::vector<double>> T_rp(nthr, std::vector<double>(h->nrung, 0.0));
  const int tpt_fill = H->gv.tpt, wpts_fill = H->gv.tma == 3 ? H->upts : 32 * tpt_fill;   // points per warp
  std::vector<double> ut_acc((size_t)nthr * 3, 0.0);   // per-thread sub-phase seconds (NC_SETUP_TIMING)
#pragma omp parallel
  {
    const int th = omp_get_thread_num();
    double* ut = ut_acc.data() + (size_t)th * 3;
    double umark = 0.0;
    auto ulap = [&](int k) {
      if (!sub_timing) return;
      const double t = omp_get_wtime();
      if (k >= 0) ut[k] += t - umark;
      umark = t;
    };
    ulap(-1);
    std::vector<GridUnit>& TU = T_units[th];
    std::vector<ChunkRec>& TC = T_chunks[th];
    std::vector<int32_t>& TS = T_src[th];
    std::vector<double>& TR = T_rp[th];
    std::vector<std::pair<int, int32_t>> rs;
    std::vector<Slice> slices;
    std::vector<int> ring_rung;   // per (source, ring)
#pragma omp for schedule(dynamic, 1)
    for (int64_t bi = 0; bi < nblk; ++bi) {
      BlockOut& bo = blk[bi];
      bo.thr = th;
      bo.u0 = (int64_t)TU.size();
      bo.c0 = (int64_t)TC.size();
      bo.s0 = (int64_t)TS.size();
      for (int64_t gi = bi * kBlk; gi < std::min(NGL, (bi + 1) * kBlk); ++gi) {
        const int32_t k = H->grid_ids[gi];
        const GridPlan& gp = plans[k];
        const int64_t q = H->goff[k + 1] - H->goff[k];
        const double Rg = H->gR[gp.group];
        const size_t ns_all = (size_t)gp.cnt;
        const int32_t* g_src = F_src.data() + gp.off;
        const int32_t* g_rung = F_rung.data() + gp.off;
        const double* g_dist = F_dist.data() + gp.off;
        ulap(2);
        if (chunk_rungs) {
          ring_rung.assign(ns_all * gp.nr, 0);
          for (int kr = 0; kr < gp.nr; ++kr) {
            const double rr = Rg * std::cos((kr + 0.5) * M_PI / (2.0 * gp.nr));
            for (size_t n = 0; n < ns_all; ++n) ring_rung[n * gp.nr + kr] = best_rung(g_dist[n] - rr);   // >= d - R
          }
        }
        // the unit's sources bucketed by rung (sorted by patch within a bucket); slices never mix rungs; slice
        // offsets are block-relative (shifted when the block is copied into place)
        ulap(0);
        auto make_slices = [&](int kr0) {
          ulap(2);
          rs.clear();
          slices.clear();
          for (size_t n = 0; n < ns_all; ++n)
            rs.push_back({chunk_rungs ? ring_rung[n * gp.nr + kr0] : g_rung[n], g_src[n]});
          std::sort(rs.begin(), rs.end());
          size_t a = 0;
          while (a < rs.size()) {
            size_t b = a;
            while (b < rs.size() && rs[b].first == rs[a].first) ++b;
            const int64_t s0 = (int64_t)TS.size() - bo.s0;
            for (size_t k2 = a; k2 < b; ++k2) TS.push_back(rs[k2].second);
            const int64_t ns = (int64_t)(b - a);
            const int64_t nsl = (ns + kSliceMax - 1) / kSliceMax;
            for (int64_t sl = 0; sl < nsl; ++sl) {
              const int64_t x0 = s0 + (ns * sl) / nsl, x1 = s0 + (ns * (sl + 1)) / nsl;
              slices.push_back({x0, (int32_t)(x1 - x0), rs[a].first});
            }
            a = b;
          }
          ulap(1);
        };
        if (!chunk_rungs) make_slices(0);   // one list per grid, shared by its units
        int kr_cached = -1;                 // chunks with the same first ring share their lists
        for (int64_t c0 = 0; c0 < q; c0 += H->upts) {
          ChunkRec cr;
          cr.pt0 = H->goff[k] + c0;
          cr.npt = (int32_t)std::min<int64_t>(H->upts, q - c0);
          if (chunk_rungs) {
            const int32_t* ro = H->roff.data() + H->rbase[k];
            int kr0 = 0;
            while (c0 >= ro[kr0 + 1]) ++kr0;
            if (kr0 != kr_cached) {
              make_slices(kr0);
              kr_cached = kr0;
            }
          }
          cr.u0 = (int64_t)TU.size() - bo.u0;
          cr.nu = (int32_t)slices.size();
          TC.push_back(cr);
          for (const Slice& sl : slices) {
            GridUnit u;
            u.pt0 = cr.pt0;
            u.npt = cr.npt;
            u.src0 = sl.src0;
            u.nsrc = sl.nsrc;
            u.soff = h->rung_soff[sl.rung];
            u.p = h->rung_p[sl.rung];
            u.pad_ = 0;
            TU.push_back(u);
            const double pr = (double)cr.npt * sl.nsrc * h->rung_p[sl.rung];   // integers: sums are exact
            bo.pairs += pr;
            TR[sl.rung] += pr;
            bo.slot += (double)H->upts * u.nsrc * u.p;
            // active-warp lane slots; a tail warp with <= 32 points runs one point per lane (direct.cu)
            const int full = u.npt / wpts_fill, rem = u.npt - full * wpts_fill;
            const int tail = rem == 0 ? 0 : (tpt_fill > 1 && rem <= 32 ? 32 : wpts_fill);
            bo.wslot += (double)(full * wpts_fill + tail) * u.nsrc * u.p;
          }
        }
      }
      bo.nu = (int64_t)TU.size() - bo.u0;
      bo.nc = (int64_t)TC.size() - bo.c0;
      bo.ns = (int64_t)TS.size() - bo.s0;
      ulap(2);
    }
  }
  if (sub_timing) {
    double tot[3] = {0, 0, 0};
    for (size_t t = 0; t < ut_acc.size(); ++t) tot[t % 3] += ut_acc[t];
    fprintf(stderr, "[nc setup]   units thread-seconds: ring rungs %.3f slices %.3f units %.3f (threads %d)\n", tot[0],
            tot[1], tot[2], nthr);
  }
  setup_tick("units: per-grid (host, parallel)");
  {   // place the blocks in grid order (offsets shifted), statistics summed in block order (exact: integer-valued)
    std::vector<int64_t> ub(nblk + 1, 0), cb(nblk + 1, 0), sb(nblk + 1, 0);
    for (int64_t bi = 0; bi < nblk; ++bi) {
      ub[bi + 1] = ub[bi] + blk[bi].nu;
      cb[bi + 1] = cb[bi] + blk[bi].nc;
      sb[bi + 1] = sb[bi] + blk[bi].ns;
      H->pairs_grid += blk[bi].pairs;
      H->slot_pairs += blk[bi].slot;
      H->warp_slot_pairs += blk[bi].wslot;
    }
    units.resize(ub[nblk]);
    chunks.resize(cb[nblk]);
    srclist.resize(sb[nblk]);
    std::vector<std::vector<char>> used(nthr, std::vector<char>(h->nrung, 0));
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t bi = 0; bi < nblk; ++bi) {
      const BlockOut& bo = blk[bi];
      std::vector<char>& us = used[omp_get_thread_num()];
      const GridUnit* su = T_units[bo.thr].data() + bo.u0;
      for (int64_t e = 0; e < bo.nu; ++e) {
        GridUnit u = su[e];
        u.src0 += sb[bi];
        units[ub[bi] + e] = u;
        for (int kk = 0; kk < h->nrung; ++kk)
          if (u.soff == h->rung_soff[kk]) us[kk] = 1;
      }
      const ChunkRec* sc = T_chunks[bo.thr].data() + bo.c0;
      for (int64_t e = 0; e < bo.nc; ++e) {
        ChunkRec c = sc[e];
        c.u0 += ub[bi];
        chunks[cb[bi] + e] = c;
      }
      std::copy(T_src[bo.thr].begin() + bo.s0, T_src[bo.thr].begin() + bo.s0 + bo.ns, srclist.begin() + sb[bi]);
    }
    for (int t = 0; t < nthr; ++t)
      for (int kk = 0; kk < h->nrung; ++kk) {
        if (used[t][kk]) h->rung_used[kk] = 1;
        rung_pairs[kk] += T_rp[t][kk];
      }
  }
  if (diag) {
    fprintf(stderr, "[nc hier diag] grid pairs by rung (r/eps: pairs):");
    for (int k = 0; k < h->nrung; ++k) fprintf(stderr, " %.3g:%.3g", h->rung_r[k] / eps, rung_pairs[k]);
    fprintf(stderr, "\n");
  }
  setup_tick("partition, offsets, units");
  // near lists for local patches (concatenated over levels)
  std::vector<int64_t> near_off(rc + 1, 0);
  std::vector<int32_t> near_all;
  std::vector<int32_t> work_near;
  {   // per local row: the near tails of its groups at every level (exactly-once coverage: no duplicates), sorted
    std::vector<int64_t> cnt(rc, 0);
#pragma omp parallel for schedule(static, 1024)
    for (int64_t i = 0; i < rc; ++i) {
      int64_t c = 0;
      for (int lvl = 0; lvl <= L; ++lvl) {
        const int64_t g = H->pgroup[(size_t)lvl * N + rb + i];
        c += near_end[g] - near_beg[g];
      }
      cnt[i] = c;
    }
    for (int64_t i = 0; i < rc; ++i) near_off[i + 1] = near_off[i] + cnt[i];
    near_all.resize((size_t)near_off[rc]);
#pragma omp parallel for schedule(dynamic, 256)
    for (int64_t i = 0; i < rc; ++i) {
      int64_t o = near_off[i];
      for (int lvl = 0; lvl <= L; ++lvl) {
        const int64_t g = H->pgroup[(size_t)lvl * N + rb + i];
        for (int64_t e = near_beg[g]; e < near_end[g]; ++e) near_all[o++] = F_src[e];
      }
      std::sort(near_all.begin() + near_off[i], near_all.begin() + near_off[i + 1]);
    }
    for (int64_t i = 0; i < rc; ++i) {
      if (cnt[i]) work_near.push_back((int32_t)i);
      H->near_count.push_back((int32_t)cnt[i]);
      H->pairs_near += (double)cnt[i] * Ks * p;
    }
  }
  std::vector<double> lvl_terms(L + 1, 0.0), lvl_single(L + 1, 0.0);
  for (int64_t i = rb; i < re; ++i)
    for (int lvl = 0; lvl <= L; ++lvl) {
      const int32_t g = H->pgroup[(size_t)lvl * N + i];
      for (int64_t kg = H->ggrid0[g]; kg < H->ggrid0[g + 1]; ++kg) {
        const double t = (double)Ks * H->gnr[kg] * H->gna[kg];
        H->interp_terms += t;
        lvl_terms[lvl] += t;
        if (H->glast[g] - H->gfirst[g] == 1) lvl_single[lvl] += t;
      }
    }
  if (diag) {
    fprintf(stderr, "[nc hier diag] interpolation terms by level (all / single-member groups):");
    for (int lvl = 0; lvl <= L; ++lvl) fprintf(stderr, " %d:%.3g/%.3g", lvl, lvl_terms[lvl], lvl_single[lvl]);
    fprintf(stderr, "\n");
  }
  setup_tick("near lists");
  if (getenv("NC_SETUP_DIGEST")) {   // FNV-1a digests of the host plan (refactors of the setup must reproduce it)
    auto fnv = [](const void* p, size_t n) {
      uint64_t hsh = 1469598103934665603ull;
      const unsigned char* b = (const unsigned char*)p;
      for (size_t i = 0; i < n; ++i) hsh = (hsh ^ b[i]) * 1099511628211ull;
      return (unsigned long long)hsh;
    };
    fprintf(stderr, "[nc setup digest] units %llx chunks %llx srclist %llx gnr %llx gna %llx goff %llx roff %llx "
                    "ggrid0 %llx near_off %llx near %llx work_near %llx pairs %.17g\n",
            fnv(units.data(), units.size() * sizeof(GridUnit)), fnv(chunks.data(), chunks.size() * sizeof(ChunkRec)),
            fnv(srclist.data(), srclist.size() * 4), fnv(H->gnr.data(), H->gnr.size() * 4),
            fnv(H->gna.data(), H->gna.size() * 4), fnv(H->goff.data(), H->goff.size() * 8),
            fnv(H->roff.data(), H->roff.size() * 4), fnv(H->ggrid0.data(), H->ggrid0.size() * 8),
            fnv(near_off.data(), near_off.size() * 8), fnv(near_all.data(), near_all.size() * 4),
            fnv(work_near.data(), work_near.size() * 4), H->pairs_grid);
  }
  for (int k = 0; k < h->nrung; ++k) H->pmax = std::max(H->pmax, h->rung_p[k]);
  // ---- uploads and device grids ----
  H->nunits = (int64_t)units.size();
  for (const GridUnit& u : units) H->unit_points += u.npt;
  H->nchunks = (int64_t)chunks.size();
  H->nwork_near = (int64_t)work_near.size();
  NC_TRY(upload(h, &H->d_gnr, H->gnr, s));
  NC_TRY(upload(h, &H->d_gna, H->gna, s));
  NC_TRY(upload(h, &H->d_goff, H->goff, s));
  NC_TRY(upload(h, &H->d_coff, H->coff, s));
  NC_TRY(upload(h, &H->d_rbase, H->rbase, s));
  NC_TRY(upload(h, &H->d_roff, H->roff, s));
  NC_TRY(upload(h, &H->d_grid_ids, H->grid_ids, s));
  {   // the ring twiddles of every angle count up to namax, in long double (k_transform reads them, no sincospi)
    const int nmax = std::max(H->namax, 1);
    std::vector<double2> tw((size_t)nmax * (nmax + 1) / 2);
    for (int n = 1; n <= nmax; ++n)
      for (int l = 0; l < n; ++l) {
        const long double a = 2.0L * 3.14159265358979323846264338327950288L * l / n;
        tw[(size_t)n * (n - 1) / 2 + l] = make_double2((double)cosl(a), (double)sinl(a));
      }
    NC_TRY(upload(h, &H->d_twtab, tw, s));
  }
  NC_TRY(halloc(h, &H->d_counter, 1));
  if (const int fb = grid_far_table_bits(H->gv)) {   // far log table of the grid kernel (green.cuh)
    double a2 = 0.0, a3 = 0.0;
    grid_far_poly(H->gv, &a2, &a3);
    if (far_table_build(h->kind, h->eps, fb, grid_far_table_rcp(H->gv), a2, a3, &H->d_ftab, &H->ftab.n,
                        &H->ftab.base))
      return fail(NC_ECUDA, "nc_setup: far log table upload failed");
    H->ftab.d = H->d_ftab;
    h->device_bytes += (double)H->ftab.n * sizeof(double2);
  }
  NC_TRY(upload(h, &H->d_grid_group, H->grid_group, s));
  NC_TRY(upload(h, &H->d_ggrid0, H->ggrid0, s));
  NC_TRY(upload(h, &H->d_units, units, s));
  NC_TRY(upload(h, &H->d_chunks, chunks, s));
  {   // per grid: its chunks [gch0[k], gch0[k + 1]) (chunks are in grid order; the fused reduction + transform)
    std::vector<int64_t> gch0(NG + 1, 0);
    int64_t c = 0;
    bool ordered = true;
    for (int64_t k = 0; k < NG; ++k) {
      gch0[k] = c;
      while (c < (int64_t)chunks.size() && chunks[c].pt0 < H->goff[k + 1]) {
        ordered = ordered && chunks[c].pt0 >= H->goff[k];
        ++c;
      }
    }
    gch0[NG] = c;
    H->fuse_reduce = ordered && c == (int64_t)chunks.size() && H->upts <= 64;   // a lane sums <= 2 points per chunk
    NC_TRY(upload(h, &H->d_gch0, gch0, s));
    const char* etw = tuning_env("NC_TRANSFORM");
    H->transform_w = !(etw && etw[0] == '0');
  }
  NC_TRY(upload(h, &H->d_srclist, srclist, s));
  NC_TRY(upload(h, &H->d_near_off, near_off, s));
  NC_TRY(upload(h, &H->d_near, near_all, s));
  NC_TRY(upload(h, &H->d_work_near, work_near, s));
  std::vector<int32_t> pgl((size_t)(L + 1) * std::max<int64_t>(rc, 1), 0);
  for (int lvl = 0; lvl <= L; ++lvl)
    for (int64_t i = 0; i < rc; ++i) pgl[(size_t)lvl * rc + i] = H->pgroup[(size_t)lvl * N + rb + i];
  NC_TRY(upload(h, &H->d_pgl, pgl, s));
  if (H->sep_nodes) {   // single-member groups with local grids go to k_interp_sep
    std::vector<uint8_t> gsep(G, 0);
    for (int64_t g = 0; g < G; ++g)
      gsep[g] = H->glast[g] - H->gfirst[g] == 1 && H->ggrid0[g] < H->ggrid0[g + 1] && H->gnr[H->ggrid0[g]] > 0;
    std::vector<int32_t> work_sep;
    for (int64_t i = 0; i < rc; ++i) {
      bool any = false;
      for (int lvl = 0; lvl <= L; ++lvl) {
        const int32_t g = pgl[(size_t)lvl * rc + i];
        if (gsep[g]) {
          any = true;
          for (int64_t kg = H->ggrid0[g]; kg < H->ggrid0[g + 1]; ++kg) H->sep_terms += (double)Ks * H->gnr[kg] * H->gna[kg];
        }
      }
      if (any) work_sep.push_back((int32_t)i);
    }
    H->nwork_sep = (int64_t)work_sep.size();
    NC_TRY(upload(h, &H->d_gsep, gsep, s));
    NC_TRY(upload(h, &H->d_work_sep, work_sep, s));
    NC_TRY(upload(h, &H->d_ring_t, H->ring_t, s));
    NC_TRY(upload(h, &H->d_node_ring, H->node_ring, s));
    NC_TRY(upload(h, &H->d_node_cs, H->node_cs, s));
    if (diag) fprintf(stderr, "[nc hier diag] separable step 4: %lld patches, %.3g of %.3g interpolation terms\n",
                      (long long)H->nwork_sep, H->sep_terms, H->interp_terms);
  }
  NC_TRY(halloc(h, &H->d_gx, H->Q));
  NC_TRY(halloc(h, &H->d_gy, H->Q));
  NC_TRY(halloc(h, &H->d_gz, H->Q));
  NC_TRY(halloc(h, &H->d_gval, H->Q));
  NC_TRY(halloc(h, &H->d_gcoef, H->C));
  NC_TRY(halloc(h, &H->d_part, (size_t)H->nunits * H->upts));
  NC_TRY(halloc(h, &H->d_tx, rc * Ks));
  NC_TRY(halloc(h, &H->d_ty, rc * Ks));
  NC_TRY(halloc(h, &H->d_tz, rc * Ks));
  NC_TRY(halloc(h, &H->d_udir, rc * Ks));
  NC_TRY(halloc(h, &H->d_u, rc * Ks));
  if (!H->grid_ids.empty())
    k_grid_points<<<(unsigned)H->grid_ids.size(), 128, 0, s>>>(H->d_grid_ids, (int64_t)H->grid_ids.size(),
                                                               H->d_grid_group, H->d_gframe, H->d_gR, H->d_gnr,
                                                               H->d_gna, H->d_goff, H->d_rbase, H->d_roff, H->d_gx,
                                                               H->d_gy, H->d_gz);
  launch_targets(h->d_frames, rb, rc, h->d_zhat, Ks, 0.5, H->d_tx, H->d_ty, H->d_tz, s);
  NC_TRY(proxy_setup(h, H, plans, pgl, cen, tol, s));
  NC_CUDA_TRY(cudaGetLastError());
  h->pairs_per_matvec = H->pairs_grid + H->pairs_near;
  return NC_OK;
}

int hier_matvec(nc_handle* h, const double* x, double* y, cudaStream_t s) {
  HierState* H = h->hier;
  const int64_t rc = h->row_count;
  const int Ks = h->Kstar, K = h->K;
  // steps 2-3: interaction-list and leaf-neighbour sources on the incoming grids
  launch_pairs_grid(H->gv, h->kind, H->d_units, H->nunits, H->d_gx, H->d_gy, H->d_gz, H->d_srclist, h->d_src4, h->d_rho,
                    H->pmax,
                    H->d_part, H->d_counter, H->ftab, s);
  h->launches_last += H->nunits > 0;
  if (h->time_stages) cudaEventRecord(h->ev[3], s);
  const bool tw = H->transform_w;   // NC_TRANSFORM=0: k_reduce_chunks + the CTA-per-grid transform (tested alternative)
  const bool fused = tw && H->fuse_reduce;
  if (H->nchunks && !fused) {
    const int per = 256 / H->upts;   // upts = 64 (warp-level units) or 256 (CTA units)
    k_reduce_chunks<<<(unsigned)((H->nchunks + per - 1) / per), 256, 0, s>>>(H->d_chunks, H->nchunks, H->d_part,
                                                                            H->upts, H->d_gval);
    h->launches_last++;
  }
  if (h->time_stages) cudaEventRecord(h->ev[8], s);
  // step 4a: grid samples -> coefficients
  if (!H->grid_ids.empty()) {
    const int64_t ng = (int64_t)H->grid_ids.size();
    if (tw) {
      constexpr int WPC = 4;
      const int wsh = ((H->qmax + 1) & ~1) + H->cmax + 8 * H->nrmax;   // doubles per warp
      const size_t shm = (size_t)WPC * wsh * sizeof(double);
      if (shm > 48 * 1024)
        NC_CUDA_TRY(cudaFuncSetAttribute(k_transform_w<WPC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm));
      int per = 1, dev = 0, sms = 148;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_transform_w<WPC>, 32 * WPC, shm);
      const int64_t nb = std::min<int64_t>((ng + WPC - 1) / WPC, (int64_t)std::max(per, 1) * sms);
      k_transform_w<WPC><<<(unsigned)nb, 32 * WPC, shm, s>>>(
          H->d_grid_ids, ng, H->d_gnr, H->d_gna, H->d_goff, H->d_coff, H->d_rbase, H->d_roff, H->d_gval, H->d_gcoef,
          H->d_twtab, wsh, H->d_chunks, H->d_gch0, fused ? H->d_part : nullptr, H->upts);
    } else {
      const size_t shm = (size_t)(3 * H->qmax + 1 + H->cmax + 8 * H->nrmax) * sizeof(double);
      if (shm > 48 * 1024) NC_CUDA_TRY(cudaFuncSetAttribute(k_transform, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm));
      k_transform<<<(unsigned)ng, 128, shm, s>>>(H->d_grid_ids, ng, H->d_gnr, H->d_gna, H->d_goff, H->d_coff,
                                                 H->d_rbase, H->d_roff, H->d_gval, H->d_gcoef, H->d_twtab);
    }
    h->launches_last++;
  }
  // near lists at the Zernike nodes
  NC_CUDA_TRY(cudaMemsetAsync(H->d_udir, 0, (size_t)rc * Ks * sizeof(double), s));
  launch_pairs_near(h->kind, H->d_tx, H->d_ty, H->d_tz, Ks, H->d_work_near, H->nwork_near, H->d_near_off, H->d_near,
                    h->d_src4, h->d_rho, h->p, H->d_udir, h->xtab, s);
  h->launches_last += H->nwork_near > 0;
  // step 4b: interpolation to the Zernike nodes, summed over levels
  if (rc > 0) {
    // two buffers for all grids of one group (cgroupmax doubles, even: pairs)
    const size_t shm = 2 * (size_t)std::max(H->cgroupmax, 2) * sizeof(double);
    const int np = H->nprule;
    const double* cen = h->d_centers + 3 * h->row_begin;
    if (!np) {   // every level at the Zernike nodes, on top of the near-list sums
      NC_TRY(launch_interp(shm, H->L, rc, Ks, H->nrmax, H->namax, H->d_pgl, H->d_ggrid0, H->d_gframe, H->d_gRinv,
                           H->d_gnr, H->d_gna, H->d_coff, H->d_gcoef, H->d_tx, H->d_ty, H->d_tz, H->d_udir, H->d_u,
                           H->d_gsep, H->interp_lt, cen, H->asin_terms, s));
      h->launches_last++;
    } else {     // R36: each rule's levels at its proxies, u = udir + sum_r V_r Int_r^T; the rest at the nodes, in place
      for (int r = 0; r < np; ++r) {
        const HierState::PRule& R = H->prule[r];
        NC_TRY(launch_interp(shm, H->L, rc, R.n, H->nrmax, H->namax, H->d_pgl, H->d_ggrid0, H->d_gframe, H->d_gRinv,
                             H->d_gnr, H->d_gna, H->d_coff, H->d_gcoef, R.ptx, R.pty, R.ptz, nullptr, R.V, H->d_gsep,
                             H->interp_lt, cen, H->asin_terms, s, 2 + r, H->d_pcode));
        launch_gemm_dmma(R.V, R.n, 1, 0, R.Int, rc, Ks, R.n, H->d_u, Ks, 1, r == 0 ? H->d_udir : H->d_u, Ks, s);
      }
      NC_TRY(launch_interp(shm, H->L, rc, Ks, H->nrmax, H->namax, H->d_pgl, H->d_ggrid0, H->d_gframe, H->d_gRinv,
                           H->d_gnr, H->d_gna, H->d_coff, H->d_gcoef, H->d_tx, H->d_ty, H->d_tz, H->d_u, H->d_u,
                           H->d_gsep, H->interp_lt, cen, H->asin_terms, s, 1, H->d_pcode, H->d_pwork1, H->npwork1));
      h->launches_last += 2 * np + (H->npwork1 > 0);
    }
  }
  if (H->nwork_sep) {   // single-member groups, separably (adds to u)
    const int Mmax = H->namax / 2, cpairs = std::max(H->cmax / 2, 1);
    const size_t shm = (size_t)cpairs * sizeof(double2) + (size_t)H->nring * (Mmax + 1) * sizeof(double2) +
                       (size_t)H->nring * (2 * H->nrmax + 1) * sizeof(double);
    auto kern = Ks <= 256 ? k_interp_sep<128, 2> : k_interp_sep<128, 4>;   // node slots >= K*
    if (shm > 48 * 1024) NC_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm));
    kern<<<(unsigned)H->nwork_sep, 128, shm, s>>>(H->L, rc, Ks, H->d_work_sep, H->d_pgl, H->d_gsep, H->d_ggrid0,
                                                   H->d_gR, H->d_gnr, H->d_gna, H->d_coff, H->d_gcoef, H->nring,
                                                   H->d_ring_t, H->d_node_ring, H->d_node_cs, cpairs, Mmax, H->nrmax,
                                                   H->d_u);
    h->launches_last++;
  }
  // step 5: y = x + U P^T
  if (h->time_stages) cudaEventRecord(h->ev[7], s);
  launch_gemm_dmma(H->d_u, Ks, 1, 0, h->d_P, rc, K, Ks, y, K, 1, x, K, s);
  h->launches_last++;
  if (h->time_stages) cudaEventRecord(h->ev[4], s);
  return NC_OK;
}

void hier_fill_stats(const nc_handle* h, nc_stats_t* o) {
  const HierState* H = h->hier;
  if (!H) return;
  o->tree_levels = H->L;
  o->tree_groups = H->ngroups;
  o->hier_grid_pairs = H->pairs_grid;
  o->hier_near_pairs = H->pairs_near;
  o->hier_interp_terms = H->interp_terms;
  o->hier_grid_points = H->Q;
  o->hier_grid_units = H->nunits;
  o->hier_grid_fill = H->slot_pairs > 0 ? H->pairs_grid / H->slot_pairs : 0.0;
  o->hier_grid_warp_fill = H->warp_slot_pairs > 0 ? H->pairs_grid / H->warp_slot_pairs : 0.0;
  hier_grid_variant(h, o->grid_variant);
  o->hier_unit_points = H->unit_points;
  o->proxy_n = H->proxy_n;
  o->proxy_kappa = H->proxy_kappa;
  o->proxy_far_frac = H->proxy_pairs > 0 ? H->proxy_far / H->proxy_pairs : 0.0;
}

int hier_grid_far(const nc_handle* h) { return h->hier ? h->hier->gv.far : -1; }
void hier_grid_variant(const nc_handle* h, int* v8) {
  const GridVariant g = h->hier ? h->hier->gv : GridVariant{0, 0, 0, 0, 0, 0, 0, 0};
  const int a[8] = {g.nt, g.tpt, g.unroll, g.stage, g.far, g.tma, g.minb, g.persist};
  for (int k = 0; k < 8; ++k) v8[k] = a[k];
}

void hier_destroy(nc_handle* h) {
  HierState* H = h->hier;
  if (!H) return;
  void* bufs[] = {H->d_keys, H->d_gframe, H->d_gR, H->d_gRinv, H->d_twtab, H->d_gnr, H->d_gna, H->d_goff, H->d_coff, H->d_grid_ids,
                  H->d_grid_group, H->d_ggrid0, H->d_counter, H->d_ftab, H->d_rbase, H->d_roff, H->d_gsep, H->d_work_sep, H->d_ring_t,
                  H->d_node_ring, H->d_node_cs,
                  H->d_gx, H->d_gy, H->d_gz, H->d_gval, H->d_gcoef, H->d_units, H->d_srclist, H->d_part,
                  H->d_chunks, H->d_gch0, H->d_work_near, H->d_near_off, H->d_near, H->d_pgl, H->d_tx, H->d_ty, H->d_tz,
                  H->d_udir, H->d_u, H->d_pcode, H->d_pwork1};
  for (void* b : bufs)
    if (b) cudaFree(b);
  for (HierState::PRule& R : H->prule)
    for (void* b : {(void*)R.ptx, (void*)R.pty, (void*)R.ptz, (void*)R.V, (void*)R.Int})
      if (b) cudaFree(b);
  delete H;
  h->hier = nullptr;
}

}  // namespace nc

extern "C" int nc_near_counts(const nc_handle* h, int64_t* counts) {
  if (!h || !counts) return nc::fail(NC_EINVAL, "nc_near_counts: null argument");
  const nc::HierState* H = h->hier;
  if (!H) return nc::fail(NC_ESTATE, "nc_near_counts: handle is not NC_HIER");
  for (size_t k = 0; k < H->near_count.size(); ++k) counts[k] = H->near_count[k];
  return NC_OK;
}

extern "C" int nc_tree_lists(const nc_handle* h, int64_t* n_ilist, int64_t* ilist, int64_t* n_nbr, int64_t* nbr,
                             int64_t* box_of_patch) {
  if (!h) return nc::fail(NC_EINVAL, "nc_tree_lists: null handle");
  const nc::HierState* H = h->hier;
  if (!H) return nc::fail(NC_ESTATE, "nc_tree_lists: handle is not NC_HIER");
  // the audit lists (level, target group, source group), built on first request (the setup does not need them)
  nc::HierState* Hm = const_cast<nc::HierState*>(H);
  if (Hm->ilist_entries.empty() && Hm->nbr_entries.empty()) {
    const int64_t G = (int64_t)H->il_off.size() - 1;
    for (int64_t g = 0; g < G; ++g) {
      for (int64_t k = H->il_off[g]; k < H->il_off[g + 1]; ++k) {
        Hm->ilist_entries.push_back(H->glevel[g]);
        Hm->ilist_entries.push_back(g);
        Hm->ilist_entries.push_back(H->il[k]);
      }
      if (H->glevel[g] == H->L)
        for (int k = 0; k < 8; ++k)
          if (H->nbr[8 * g + k] >= 0) {
            Hm->nbr_entries.push_back(H->L);
            Hm->nbr_entries.push_back(g);
            Hm->nbr_entries.push_back(H->nbr[8 * g + k]);
          }
    }
  }
  if (n_ilist) *n_ilist = (int64_t)H->ilist_entries.size() / 3;
  if (n_nbr) *n_nbr = (int64_t)H->nbr_entries.size() / 3;
  if (ilist) std::copy(H->ilist_entries.begin(), H->ilist_entries.end(), ilist);
  if (nbr) std::copy(H->nbr_entries.begin(), H->nbr_entries.end(), nbr);
  if (box_of_patch)
    for (size_t k = 0; k < H->pgroup.size(); ++k) box_of_patch[k] = H->pgroup[k];
  return NC_OK;
}
