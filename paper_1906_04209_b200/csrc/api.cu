// api.cu -- the C ABI of libnc (include/nc.h): setup, matvec, GMRES, read-out.
//
// Matvec pipeline per call (direct mode), all in this library's kernels:
//   K1  rho = X T^T          fp64 DMMA GEMM, epilogue writes rho into the packed source records
//   AG  ncclAllGather of the source records (world > 1 only)
//   K2  pair sums            u_{ik} = sum_{j != i} sum_m G(z_ik, s_jm) rho_jm  (direct.cu)
//   K3  Y = X + U P^T        fp64 DMMA GEMM with the segment reduction fused into its operand load
#include <math.h>
#include <stdlib.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <string>
#include <unordered_map>
#include <thread>
#include <vector>

#include "green.cuh"
#include "hier.cuh"
#include "nc_common.cuh"

namespace nc {

static thread_local std::string g_err;

void setup_tick(const char* phase) {
  static const bool on = getenv("NC_SETUP_TIMING") != nullptr;
  static thread_local std::chrono::steady_clock::time_point last;
  if (!on) return;
  const auto now = std::chrono::steady_clock::now();
  if (phase) fprintf(stderr, "[nc setup] %-28s %9.1f ms\n", phase, std::chrono::duration<double, std::milli>(now - last).count());
  last = now;
}

void set_error(const std::string& msg) { g_err = msg; }
int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}
int cuda_fail(cudaError_t e, const char* what) {
  g_err = std::string("CUDA error ") + cudaGetErrorString(e) + " in " + what;
  return NC_ECUDA;
}

template <class T>
static int dalloc(nc_handle* h, T** p, size_t count) {
  if (count == 0) count = 1;
  cudaError_t e = cudaMalloc((void**)p, count * sizeof(T));
  if (e != cudaSuccess) {
    (void)cudaGetLastError();
    return fail(NC_ENOMEM, "cudaMalloc of " + std::to_string(count * sizeof(T)) + " bytes failed: " +
                               cudaGetErrorString(e));
  }
  h->device_bytes += (double)count * sizeof(T);
  return NC_OK;
}

// -------------------------------------------------------------------------------------------------
// host-side validation helpers
// -------------------------------------------------------------------------------------------------
// Minimum arc separation >= 3 eps (§3) via a uniform 3-D cell grid on chords: the points sorted by
// cell key, each point's 27 neighbour cells found by binary search; the check runs on the host threads and reports the
// first offending pair in index order (deterministic).
static int check_separation(const double* c, int64_t N, double eps) {
  const double min_arc = 3.0 * eps * (1.0 - 1e-12);
  const double chord = 2.0 * sin(0.5 * std::min(min_arc, M_PI));
  const double cell = std::max(chord, 1e-6);
  const int64_t nc = (int64_t)ceil(2.0 / cell) + 2;
  auto key = [&](int64_t a, int64_t b, int64_t d) { return (a * nc + b) * nc + d; };
  auto cidx = [&](double v) { return (int64_t)floor((v + 1.0) / cell); };
  std::vector<std::pair<int64_t, int64_t>> kc((size_t)N);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < N; ++i) kc[i] = {key(cidx(c[3 * i]), cidx(c[3 * i + 1]), cidx(c[3 * i + 2])), i};
  std::sort(kc.begin(), kc.end());
  int64_t bad_i = N, bad_j = N;
  double bad_arc = 0.0;
#pragma omp parallel for schedule(dynamic, 1024)
  for (int64_t i = 0; i < N; ++i) {
    const int64_t a = cidx(c[3 * i]), b = cidx(c[3 * i + 1]), d = cidx(c[3 * i + 2]);
    for (int da = -1; da <= 1; ++da)
      for (int db = -1; db <= 1; ++db)
        for (int dd = -1; dd <= 1; ++dd) {
          const int64_t kk = key(a + da, b + db, d + dd);
          auto it = std::lower_bound(kc.begin(), kc.end(), std::make_pair(kk, (int64_t)-1));
          for (; it != kc.end() && it->first == kk; ++it) {
            const int64_t j = it->second;
            if (j <= i) continue;
            const double dx = c[3 * i] - c[3 * j], dy = c[3 * i + 1] - c[3 * j + 1], dz = c[3 * i + 2] - c[3 * j + 2];
            const double ch = sqrt(dx * dx + dy * dy + dz * dz);
            const double arc = 2.0 * asin(std::min(1.0, 0.5 * ch));
            if (arc < min_arc) {
#pragma omp critical(nc_sep)
              if (i < bad_i || (i == bad_i && j < bad_j)) {
                bad_i = i;
                bad_j = j;
                bad_arc = arc;
              }
            }
          }
        }
  }
  if (bad_i < N) {
    char buf[256];
    snprintf(buf, sizeof buf, "patches %lld and %lld are %.6g apart in arc length (< 3 eps = %.6g)",
             (long long)bad_i, (long long)bad_j, bad_arc, 3.0 * eps);
    return fail(NC_ESEP, buf);
  }
  return NC_OK;
}

// Source segments of the direct kernel (grid.y): pick the count whose total CTA count wastes the least
// of the last wave (all CTAs carry equal work, so waves stay in lock-step), with >= 4 waves when possible.
// contiguous partition of N rows over `world` ranks with (approximately) equal total weight: rank r gets
// [begin[r], begin[r] + count[r]); cut where the prefix sum of (w_i + 1) crosses r/world of the total
// (the +1 keeps every rank non-empty when N >= world).  Host-only; exported as nc_split_rows.
void split_rows(const double* w, int64_t N, int world, int64_t* begin, int64_t* count) {
  std::vector<double> pre(N + 1, 0.0);
  for (int64_t i = 0; i < N; ++i) pre[i + 1] = pre[i] + (w ? w[i] : 0.0) + 1.0;
  int64_t prev = 0;
  for (int r = 0; r < world; ++r) {
    int64_t end = N;
    if (r + 1 < world) {
      const double target = pre[N] * (double)(r + 1) / world;
      end = std::lower_bound(pre.begin(), pre.end(), target) - pre.begin();
      end = std::max(prev, std::min<int64_t>(end, N));
    }
    begin[r] = prev;
    count[r] = end - prev;
    prev = end;
  }
}

static void compute_nseg(nc_handle* h) {
  const char* ev = tuning_env("NC_PAIR_TPT");
  h->pair_tpt = (ev && atoi(ev) == 1) ? 1 : (ev && atoi(ev) == 2) ? 2 : kDefaultPairTpt;
  const int64_t per_block = (int64_t)kPairThreads * h->pair_tpt;
  int64_t tiles = (h->row_count * h->Kstar + per_block - 1) / per_block;
  if (tiles < 1) tiles = 1;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h->device);
  const int64_t W = (int64_t)sms * pairs_direct_blocks_per_sm(h->p, h->pair_tpt, h->xtab);
  const int64_t cap = std::min<int64_t>(h->N, 64);
  int best = 1;
  double best_cost = 1e30;
  for (int64_t s = 1; s <= cap; ++s) {
    int64_t B = tiles * s;
    int64_t waves = (B + W - 1) / W;
    double eff = (double)B / (double)(waves * W);          // useful fraction of the launched waves
    double cost = (1.0 / eff) * (1.0 + 0.002 * s);           // small penalty per extra partial buffer
    if (B < 4 * W && s < cap) cost *= 1.0 + 0.05 * (double)(4 * W - B) / (4.0 * W);
    if (cost < best_cost - 1e-12) {
      best_cost = cost;
      best = (int)s;
    }
  }
  h->nseg = best;
}

static int ensure_red(nc_handle* h, int64_t count) {
  if (count <= h->red_cap) return NC_OK;
  if (h->d_red) cudaFree(h->d_red);
  if (h->h_red) cudaFreeHost(h->h_red);
  h->d_red = nullptr;
  h->h_red = nullptr;
  NC_TRY(dalloc(h, &h->d_red, (size_t)count));
  NC_CUDA_TRY(cudaMallocHost((void**)&h->h_red, count * sizeof(double)));
  h->red_cap = count;
  return NC_OK;
}

static int allreduce_sum(nc_handle* h, double* dev, int64_t count, cudaStream_t s) {
  if (h->world <= 1) return NC_OK;
#if NC_WITH_NCCL
  ncclResult_t r = ncclAllReduce(dev, dev, (size_t)count, ncclDouble, ncclSum, h->comm, s);
  if (r != ncclSuccess) return fail(NC_ENCCL, std::string("ncclAllReduce: ") + ncclGetErrorString(r));
  return NC_OK;
#else
  (void)dev; (void)count; (void)s;
  return fail(NC_EUNSUP, "built without NCCL");
#endif
}

}  // namespace nc

using namespace nc;

extern "C" {

const char* nc_last_error(void) { return g_err.c_str(); }
const char* nc_version(void) { return "libnc 0.1 (sm_100a, fp64)"; }

int nc_setup(nc_handle** out, int kind, int64_t N, const double* centers, double eps, const nc_tables* tab,
             const nc_opts* opt) {
  if (!out) return fail(NC_EINVAL, "nc_setup: null output handle pointer");
  *out = nullptr;
  if (!centers || !tab || !opt) return fail(NC_EINVAL, "nc_setup: null centers/tables/opts");
  if (kind != NC_INTERIOR && kind != NC_EXTERIOR) return fail(NC_EINVAL, "nc_setup: kind must be 0 or 1");
  if (N < 1) return fail(NC_EINVAL, "nc_setup: N must be >= 1");
  if (!(eps > 0.0) || !(eps < 1.0)) return fail(NC_EINVAL, "nc_setup: eps must be in (0, 1)");
  if (tab->M < 0 || tab->K != (tab->M + 1) * (tab->M + 2) / 2)
    return fail(NC_EINVAL, "nc_setup: K != (M+1)(M+2)/2");
  if (tab->K > 1024) return fail(NC_EINVAL, "nc_setup: K > 1024 not supported");
  if (tab->Kstar < 1 || tab->p < 1 || tab->p > kMaxP) return fail(NC_EINVAL, "nc_setup: bad Kstar or p");
  if (!tab->zhat || !tab->P || !tab->shat || !tab->T || !tab->I) return fail(NC_EINVAL, "nc_setup: null table");
  if (tab->n_ladder < 0 || (tab->n_ladder > 0 && (!tab->ladder_r || !tab->ladder_p || !tab->ladder_shat ||
                                                   !tab->ladder_T)))
    return fail(NC_EINVAL, "nc_setup: inconsistent ladder tables");
  for (int k = 0; k < tab->n_ladder; ++k) {
    if (tab->ladder_p[k] < 1 || tab->ladder_p[k] > kMaxP) return fail(NC_EINVAL, "nc_setup: bad ladder_p");
    if (!(tab->ladder_r[k] > 2.0 * eps) || (k > 0 && !(tab->ladder_r[k] > tab->ladder_r[k - 1])))
      return fail(NC_EINVAL, "nc_setup: ladder_r must increase and exceed 2 eps");
  }
  if (opt->mode != NC_DIRECT && opt->mode != NC_HIER) return fail(NC_EINVAL, "nc_setup: bad mode");
  if (opt->world < 1 || opt->rank < 0 || opt->rank >= opt->world) return fail(NC_EINVAL, "nc_setup: bad rank/world");
  for (int64_t i = 0; i < N; ++i) {
    double r = sqrt(centers[3 * i] * centers[3 * i] + centers[3 * i + 1] * centers[3 * i + 1] +
                    centers[3 * i + 2] * centers[3 * i + 2]);
    if (!(fabs(r - 1.0) < 1e-10)) return fail(NC_EINVAL, "nc_setup: centre " + std::to_string(i) + " is not unit");
  }
  setup_tick(nullptr);
  if (opt->check_separation) NC_TRY(check_separation(centers, N, eps));
  setup_tick("separation check");
#if !NC_WITH_NCCL
  if (opt->world > 1 && opt->nccl_id) return fail(NC_EUNSUP, "nc_setup: world > 1 needs a build with NCCL");
#endif

  nc_handle* h = new nc_handle();
  auto bail = [&](int rc) {
    std::string keep = g_err;
    nc_destroy(h);
    g_err = keep;
    return rc;
  };
  h->kind = kind;
  h->mode = opt->mode;
  h->world = opt->world;
  h->rank = opt->rank;
  h->N = N;
  h->M = tab->M;
  h->K = tab->K;
  h->Kstar = tab->Kstar;
  h->p = tab->p;
  h->eps = eps;
  h->precision = opt->precision > 0 ? opt->precision : 1e-9;
  if (opt->device >= 0) {
    cudaError_t e = cudaSetDevice(opt->device);
    if (e != cudaSuccess) return bail(cuda_fail(e, "cudaSetDevice"));
  }
  {
    cudaError_t e = cudaGetDevice(&h->device);
    if (e != cudaSuccess) return bail(cuda_fail(e, "cudaGetDevice"));
    e = cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) return bail(cuda_fail(e, "cudaStreamCreate"));
    for (auto& ev : h->ev) {
      e = cudaEventCreate(&ev);
      if (e != cudaSuccess) return bail(cuda_fail(e, "cudaEventCreate"));
    }
  }
  cudaStream_t s = h->stream;
  const int K = h->K, Ks = h->Kstar, p = h->p;
  if (!log_table_device()) return bail(fail(NC_ECUDA, "nc_setup: log table upload failed"));
  {   // exact-form log table of the direct / near-list pair kernels (green_exact_r; NC_EXACT_TABLE=0: mantissa table)
    const char* e = tuning_env("NC_EXACT_TABLE");
    if (!(e && e[0] == '0')) {
      if (far_table_build(h->kind, h->eps, 7, 1, FarPoly<7, 4>::a2, FarPoly<7, 4>::a3, &h->d_xtab, &h->xtab.n,
                          &h->xtab.base, 1))
        return bail(fail(NC_ECUDA, "nc_setup: exact-form log table upload failed"));
      h->xtab.d = h->d_xtab;
    }
  }

  // tables; outgoing-operator rungs (0 = base, 1.. = ladder, NC_HIER only)
  int rc;
  // the ladder serves NC_HIER only, and only when the requested precision is not tighter than the rungs' measured
  // field error (their compression error would otherwise set the floor)
  const bool use_ladder = opt->mode == NC_HIER && tab->n_ladder > 0 &&
                          !(tab->ladder_tol > 0.0 && opt->precision > 0.0 && opt->precision < tab->ladder_tol);
  h->nrung = 1 + (use_ladder ? tab->n_ladder : 0);
  h->rung_r.assign(1, 2.0 * eps);
  h->rung_p.assign(1, p);
  for (int k = 1; k < h->nrung; ++k) {
    h->rung_r.push_back(tab->ladder_r[k - 1]);
    h->rung_p.push_back(tab->ladder_p[k - 1]);
  }
  h->rung_trow.assign(h->nrung, 0);
  h->rung_soff.assign(h->nrung, 0);
  h->rung_used.assign(h->nrung, 0);
  h->rung_used[0] = 1;
  int64_t ptot = 0;
  for (int k = 0; k < h->nrung; ++k) {
    h->rung_trow[k] = ptot;
    h->rung_soff[k] = 4 * N * ptot;
    ptot += h->rung_p[k];
  }
  if ((rc = dalloc(h, &h->d_T, (size_t)ptot * K)) || (rc = dalloc(h, &h->d_P, (size_t)K * Ks)) ||
      (rc = dalloc(h, &h->d_I, (size_t)K)) || (rc = dalloc(h, &h->d_zhat, (size_t)Ks * 3)) ||
      (rc = dalloc(h, &h->d_shat, (size_t)ptot * 3)))
    return bail(rc);
  h->h_I.assign(tab->I, tab->I + K);
  h->h_P1.assign(K, 0.0);
  for (int a = 0; a < K; ++a) {
    double v = 0.0;
    for (int k = 0; k < Ks; ++k) v += tab->P[(size_t)a * Ks + k];
    h->h_P1[a] = v;
  }
#define UP(dst, src, cnt)                                                                   \
  do {                                                                                      \
    cudaError_t _e = cudaMemcpyAsync(dst, src, (cnt) * sizeof(double), cudaMemcpyHostToDevice, s); \
    if (_e != cudaSuccess) return bail(cuda_fail(_e, "upload " #src));                      \
  } while (0)
  UP(h->d_T, tab->T, (size_t)p * K);
  UP(h->d_P, tab->P, (size_t)K * Ks);
  UP(h->d_I, tab->I, (size_t)K);
  UP(h->d_zhat, tab->zhat, (size_t)Ks * 3);
  UP(h->d_shat, tab->shat, (size_t)p * 3);
  if (h->nrung > 1) {
    UP(h->d_T + (size_t)p * K, tab->ladder_T, (size_t)(ptot - p) * K);
    UP(h->d_shat + (size_t)p * 3, tab->ladder_shat, (size_t)(ptot - p) * 3);
  }

  // internal order: identity (direct); the tree order (hierarchical) is applied by hier_setup
  h->perm.resize(N);
  for (int64_t i = 0; i < N; ++i) h->perm[i] = i;
  std::vector<double> cs(centers, centers + 3 * N);
  if (h->mode == NC_HIER) {
    setup_tick("tables, stream");
    rc = hier_order(h, cs);          // Morton order of the cube-face quadtree; fills h->perm, permutes cs
    if (rc) return bail(rc);
    setup_tick("keys, sort (device)");
  }

  if ((rc = dalloc(h, &h->d_centers, (size_t)N * 3)) || (rc = dalloc(h, &h->d_frames, (size_t)N * 9))) return bail(rc);
  UP(h->d_centers, cs.data(), (size_t)N * 3);
  launch_frames(h->d_centers, N, h->d_frames, s);

  // source records (x, y, z, rho) for all N patches and every rung, coordinates scaled by 1/2 (green.cuh)
  if ((rc = dalloc(h, &h->d_src4, (size_t)N * ptot * 4)) || (rc = dalloc(h, &h->d_rho, (size_t)N * ptot)))
    return bail(rc);
  for (int k = 0; k < h->nrung; ++k)
    launch_sources(h->d_frames, N, h->d_shat + 3 * h->rung_trow[k], h->rung_p[k], 0.5, h->d_src4 + h->rung_soff[k],
                   s);

  if (h->mode == NC_DIRECT) {
    // partition: contiguous row ranges of equal size (every row carries the same work in direct mode)
    h->rank_begin.assign(h->world, 0);
    h->rank_count.assign(h->world, 0);
    split_rows(nullptr, N, h->world, h->rank_begin.data(), h->rank_count.data());
    h->row_begin = h->rank_begin[h->rank];
    h->row_count = h->rank_count[h->rank];
    const int64_t nt = h->row_count * Ks;
    if ((rc = dalloc(h, &h->d_tx, (size_t)nt)) || (rc = dalloc(h, &h->d_ty, (size_t)nt)) ||
        (rc = dalloc(h, &h->d_tz, (size_t)nt)))
      return bail(rc);
    launch_targets(h->d_frames, h->row_begin, h->row_count, h->d_zhat, Ks, 0.5, h->d_tx, h->d_ty, h->d_tz, s);
    compute_nseg(h);
    if ((rc = dalloc(h, &h->d_upart, (size_t)h->nseg * nt))) return bail(rc);
    h->pairs_per_matvec = (double)h->row_count * Ks * (double)(N - 1) * p;
  } else {
    rc = hier_setup(h, cs, s);       // tree, lists, grids, work-weighted partition
    if (rc) return bail(rc);
    setup_tick("hier setup (rest)");
  }
  if ((rc = ensure_red(h, 4096))) return bail(rc);

  // fused K1 over the rungs in use (several rungs: one GEMM with a column map instead of one GEMM per rung)
  {
    int nused = 0, ncat = 0;
    for (int k = 0; k < h->nrung; ++k)
      if (h->rung_used[k]) { ++nused; ncat += h->rung_p[k]; }
    if (nused > 1) {
      std::vector<int64_t> cb, cr;
      std::vector<double> Tc;
      std::vector<double> Th((size_t)(h->rung_trow[h->nrung - 1] + h->rung_p[h->nrung - 1]) * K);
      NC_CUDA_TRY(cudaMemcpyAsync(Th.data(), h->d_T, Th.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
      NC_CUDA_TRY(cudaStreamSynchronize(s));
      for (int k = 0; k < h->nrung; ++k) {
        if (!h->rung_used[k]) continue;
        const int pk = h->rung_p[k];
        for (int m = 0; m < pk; ++m) {
          cb.push_back(h->rung_soff[k] / 4 + m);   // rung k's compact rho: rho_k[i p_k + m]
          cr.push_back((int64_t)pk);
        }
        Tc.insert(Tc.end(), Th.begin() + (size_t)h->rung_trow[k] * K, Th.begin() + (size_t)(h->rung_trow[k] + pk) * K);
      }
      if ((rc = dalloc(h, &h->d_Tcat, Tc.size())) || (rc = dalloc(h, &h->d_colbase, cb.size())) ||
          (rc = dalloc(h, &h->d_colrstride, cr.size())))
        return bail(rc);
      UP(h->d_Tcat, Tc.data(), Tc.size());
      NC_CUDA_TRY(cudaMemcpyAsync(h->d_colbase, cb.data(), cb.size() * sizeof(int64_t), cudaMemcpyHostToDevice, s));
      NC_CUDA_TRY(cudaMemcpyAsync(h->d_colrstride, cr.data(), cr.size() * sizeof(int64_t), cudaMemcpyHostToDevice, s));
      h->ncat = ncat;
    }
  }
  setup_tick("fused K1 tables");

  h->emulated = h->world > 1 && !opt->nccl_id;   // rank emulation: no communicator, nc_matvec_emulated only
  if (h->world > 1 && !h->emulated) {
    h->max_rows = *std::max_element(h->rank_count.begin(), h->rank_count.end());
    if ((rc = dalloc(h, &h->d_xall, (size_t)N * K)) || (rc = dalloc(h, &h->d_xpad, (size_t)h->world * h->max_rows * K)))
      return bail(rc);
  }
#if NC_WITH_NCCL
  if (h->world > 1 && !h->emulated) {
    ncclUniqueId id;
    memcpy(&id, opt->nccl_id, sizeof(id));
    ncclResult_t r = ncclCommInitRank(&h->comm, h->world, id, h->rank);
    if (r != ncclSuccess) return bail(fail(NC_ENCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(r)));
  }
#endif
  {
    cudaError_t e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return bail(cuda_fail(e, "nc_setup sync"));
    e = cudaGetLastError();
    if (e != cudaSuccess) return bail(cuda_fail(e, "nc_setup kernels"));
  }
#undef UP
  *out = h;
  return NC_OK;
}

int nc_partition(const nc_handle* h, int64_t* row_begin, int64_t* row_count, int64_t* perm) {
  if (!h) return fail(NC_EINVAL, "nc_partition: null handle");
  if (row_begin) *row_begin = h->row_begin;
  if (row_count) *row_count = h->row_count;
  if (perm) memcpy(perm, h->perm.data(), h->N * sizeof(int64_t));
  return NC_OK;
}

int nc_time_stages(nc_handle* h, int enable) {
  if (!h) return fail(NC_EINVAL, "nc_time_stages: null handle");
  h->time_stages = enable != 0;
  return NC_OK;
}

static inline void mark(nc_handle* h, int i, cudaStream_t s) {
  if (h->time_stages) cudaEventRecord(h->ev[i], s);
}

// K1 for rows [r0, r0 + nr) of the internal order (x points at row r0): rho_i = T_k fhat_i for every rung in use,
// written into the rung's compact rho array (contiguous rows of p_k: full-sector writes)
static void outgoing(nc_handle* h, const double* x, int64_t r0, int64_t nr, cudaStream_t s) {
  const int K = h->K;
  if (h->ncat > 0) {   // all rungs in use in one GEMM (scattered epilogue)
    launch_gemm_dmma_colmap(x, K, h->d_Tcat, nr, h->ncat, K, h->d_rho, h->d_colbase, h->d_colrstride, r0, s);
    h->launches_last++;
    return;
  }
  for (int k = 0; k < h->nrung; ++k) {
    if (!h->rung_used[k]) continue;
    const int pk = h->rung_p[k];
    launch_gemm_dmma(x, K, 1, 0, h->d_T + (size_t)h->rung_trow[k] * K, nr, pk, K,
                     h->d_rho + h->rung_soff[k] / 4 + (size_t)r0 * pk, (int64_t)pk, 1, nullptr, 0, s);
    h->launches_last++;
  }
}

// everything after the source records are complete: pair sums (direct) or steps 2-4 (hier), then step 5
static int matvec_tail(nc_handle* h, const double* x, double* y, cudaStream_t s) {
  const int K = h->K, p = h->p, Ks = h->Kstar;
  mark(h, 2, s);
  if (h->mode == NC_DIRECT) {
    launch_pairs_direct(h->kind, h->pair_tpt, h->d_tx, h->d_ty, h->d_tz, h->row_count * Ks, Ks, h->row_begin, h->d_src4,
                        h->d_rho, p, h->N,
                        h->nseg, h->d_upart, h->xtab, h->eps, s);
    mark(h, 3, s);
    // K3: Y = X + (sum_seg U_seg) P^T
    launch_gemm_dmma(h->d_upart, Ks, h->nseg, h->row_count * Ks, h->d_P, h->row_count, K, Ks, y, K, 1, x, K, s);
    h->launches_last += 2;
    mark(h, 4, s);
  } else {
    NC_TRY(hier_matvec(h, x, y, s));   // records ev[3] right after its pair kernel, ev[7] before step 5, ev[4] at the end
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "nc_matvec launch");
  h->stages_pending = h->time_stages;
  h->matvecs++;
  return NC_OK;
}

// order a matvec on stream s after the previous matvec of this handle when that ran on another stream
static int serialize_stream(nc_handle* h, cudaStream_t s) {
  if (h->have_last_stream && h->last_stream != s) {
    if (!h->ev_order) NC_CUDA_TRY(cudaEventCreateWithFlags(&h->ev_order, cudaEventDisableTiming));
    NC_CUDA_TRY(cudaEventRecord(h->ev_order, h->last_stream));
    NC_CUDA_TRY(cudaStreamWaitEvent(s, h->ev_order, 0));
  }
  h->last_stream = s;
  h->have_last_stream = true;
  return NC_OK;
}

// Host wait at the collective sync points (GMRES, read-out).  world == 1: cudaStreamSynchronize.  world > 1: a failed
// peer or a communicator error surfaces as an asynchronous NCCL error while this rank's collective kernel would spin
// forever, so the wait polls the stream and ncclCommGetAsyncError, aborting the communicator on an error.
static int wait_stream(nc_handle* h, cudaStream_t s, const char* where) {
#if NC_WITH_NCCL
  if (h->world > 1 && h->comm) {
    for (;;) {
      const cudaError_t e = cudaStreamQuery(s);
      if (e == cudaSuccess) return NC_OK;
      if (e != cudaErrorNotReady) return cuda_fail(e, where);
      ncclResult_t ae = ncclSuccess;
      const ncclResult_t r = ncclCommGetAsyncError(h->comm, &ae);
      if (r != ncclSuccess || (ae != ncclSuccess && ae != ncclInProgress)) {
        ncclCommAbort(h->comm);
        h->comm = nullptr;
        return fail(NC_ENCCL, std::string(where) + ": asynchronous NCCL error (communicator aborted): " +
                                  ncclGetErrorString(r != ncclSuccess ? r : ae));
      }
      std::this_thread::yield();
    }
  }
#endif
  const cudaError_t e = cudaStreamSynchronize(s);
  return e == cudaSuccess ? NC_OK : cuda_fail(e, where);
}

int nc_matvec(nc_handle* h, const double* x, double* y, void* stream) {
  if (!h || !x || !y) return fail(NC_EINVAL, "nc_matvec: null argument");
  if (x == y) return fail(NC_EINVAL, "nc_matvec: x and y must not alias");
  if (h->world > 1 && h->emulated)
    return fail(NC_ESTATE, "nc_matvec: emulated rank (no communicator): use nc_matvec_emulated");
  NC_CUDA_TRY(cudaSetDevice(h->device));
  cudaStream_t s = (cudaStream_t)stream;
  NC_TRY(serialize_stream(h, s));
  h->launches_last = 0;
  mark(h, 0, s);
  if (h->world == 1) {
    outgoing(h, x, h->row_begin, h->row_count, s);
    mark(h, 1, s);
    return matvec_tail(h, x, y, s);
  }
#if NC_WITH_NCCL
  // world > 1: all-gather the coefficient vectors (N K doubles: 109 MB at N = 1e5, a quarter of the rho values of
  // all rungs and an eighth of their records), then every rank forms the outgoing records of ALL patches itself (K1
  // over N rows, ~2 ms): the exchange does not grow with the number of outgoing-operator rungs.  The work-weighted
  // row ranges differ in length, so the exchange is one ncclAllGather of max_rows rows per rank into a padded
  // buffer (NVLS-eligible, unlike a group of broadcasts), compacted into N x K by one copy per rank.  Everything
  // after is exactly nc_matvec_emulated's path.
  {
    const size_t per = (size_t)h->max_rows * h->K;
    NC_CUDA_TRY(cudaMemcpyAsync(h->d_xpad + (size_t)h->rank * per, x, (size_t)h->row_count * h->K * sizeof(double),
                                cudaMemcpyDeviceToDevice, s));
    ncclResult_t r = ncclAllGather(h->d_xpad + (size_t)h->rank * per, h->d_xpad, per, ncclDouble, h->comm, s);
    if (r != ncclSuccess) return fail(NC_ENCCL, std::string("all-gather of x: ") + ncclGetErrorString(r));
    for (int q = 0; q < h->world; ++q)
      if (h->rank_count[q] > 0)
        NC_CUDA_TRY(cudaMemcpyAsync(h->d_xall + (size_t)h->rank_begin[q] * h->K, h->d_xpad + (size_t)q * per,
                                    (size_t)h->rank_count[q] * h->K * sizeof(double), cudaMemcpyDeviceToDevice, s));
  }
  mark(h, 1, s);
  outgoing(h, h->d_xall, 0, h->N, s);
  return matvec_tail(h, x, y, s);
#else
  return fail(NC_EUNSUP, "nc_matvec: world > 1 needs a build with NCCL");
#endif
}

int nc_matvec_emulated(nc_handle* h, const double* x_all, double* y, void* stream) {
  if (!h || !x_all || !y) return fail(NC_EINVAL, "nc_matvec_emulated: null argument");
  NC_CUDA_TRY(cudaSetDevice(h->device));
  cudaStream_t s = (cudaStream_t)stream;
  h->launches_last = 0;
  mark(h, 0, s);
  outgoing(h, x_all, 0, h->N, s);   // every rank's rows: stands in for the all-gather of the records
  mark(h, 1, s);
  const double* xl = x_all + (size_t)h->row_begin * h->K;
  if (xl == y) return fail(NC_EINVAL, "nc_matvec_emulated: y aliases x");
  return matvec_tail(h, xl, y, s);
}

// per-stage device times of the last timed matvec (waits for its events)
static int read_stages(nc_handle* h) {
  if (!h->stages_pending) return NC_OK;
  h->stages_pending = false;
  NC_CUDA_TRY(cudaEventSynchronize(h->ev[4]));
  float ms;
  for (double& v : h->ms_last) v = 0.0;
  cudaEventElapsedTime(&ms, h->ev[0], h->ev[1]); h->ms_last[0] = ms;
  cudaEventElapsedTime(&ms, h->ev[1], h->ev[2]); h->ms_last[1] = ms;
  if (h->mode == NC_DIRECT) {
    cudaEventElapsedTime(&ms, h->ev[2], h->ev[3]); h->ms_last[2] = ms;
    cudaEventElapsedTime(&ms, h->ev[3], h->ev[4]); h->ms_last[3] = ms;
  } else {
    cudaEventElapsedTime(&ms, h->ev[2], h->ev[3]); h->ms_last[4] = ms;   // k_pairs_grid (steps 2-3)
    cudaEventElapsedTime(&ms, h->ev[3], h->ev[7]); h->ms_last[5] = ms;   // reduce, transform, near list, step 4
    cudaEventElapsedTime(&ms, h->ev[7], h->ev[4]); h->ms_last[3] = ms;   // step 5 (P-apply GEMM)
    cudaEventElapsedTime(&ms, h->ev[3], h->ev[8]); h->ms_last[7] = ms;   // grid reduction (k_reduce_chunks)
  }
  cudaEventElapsedTime(&ms, h->ev[0], h->ev[4]); h->ms_last[6] = ms;
  return NC_OK;
}

int nc_matvec_host(nc_handle* h, const double* x_host, double* y_host) {
  if (!h || !x_host || !y_host) return fail(NC_EINVAL, "nc_matvec_host: null argument");
  NC_CUDA_TRY(cudaSetDevice(h->device));
  const size_t n = (size_t)h->row_count * h->K;
  if (!h->d_hx) {
    NC_TRY(dalloc(h, &h->d_hx, n));
    NC_TRY(dalloc(h, &h->d_hy, n));
  }
  cudaStream_t s = h->stream;
  if (h->world > 1) {   // collective: the whole x first (the all-gather needs it)
    NC_CUDA_TRY(cudaMemcpyAsync(h->d_hx, x_host, n * sizeof(double), cudaMemcpyHostToDevice, s));
    NC_TRY(nc_matvec(h, h->d_hx, h->d_hy, s));
  } else {
    // x in kHostBlocks row blocks on the copy stream; K1 of each block on the compute stream as soon as it has
    // landed (the host-to-device copy overlaps the outgoing GEMM), then the rest of the matvec
    constexpr int kHostBlocks = 4;
    if (!h->copy_stream) {
      NC_CUDA_TRY(cudaStreamCreateWithFlags(&h->copy_stream, cudaStreamNonBlocking));
      for (auto& ev : h->copy_ev) NC_CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    }
    NC_TRY(serialize_stream(h, s));
    NC_CUDA_TRY(cudaEventRecord(h->copy_ev[kHostBlocks], s));   // the previous use of d_hx is done
    NC_CUDA_TRY(cudaStreamWaitEvent(h->copy_stream, h->copy_ev[kHostBlocks], 0));
    const int64_t rc = h->row_count, K = h->K;
    for (int b = 0; b < kHostBlocks; ++b) {
      const int64_t r0 = rc * b / kHostBlocks, r1 = rc * (b + 1) / kHostBlocks;
      NC_CUDA_TRY(cudaMemcpyAsync(h->d_hx + r0 * K, x_host + r0 * K, (size_t)(r1 - r0) * K * sizeof(double),
                                  cudaMemcpyHostToDevice, h->copy_stream));
      NC_CUDA_TRY(cudaEventRecord(h->copy_ev[b], h->copy_stream));
    }
    h->launches_last = 0;
    mark(h, 0, s);
    for (int b = 0; b < kHostBlocks; ++b) {
      const int64_t r0 = rc * b / kHostBlocks, r1 = rc * (b + 1) / kHostBlocks;
      NC_CUDA_TRY(cudaStreamWaitEvent(s, h->copy_ev[b], 0));
      if (r1 > r0) outgoing(h, h->d_hx + r0 * K, h->row_begin + r0, r1 - r0, s);
    }
    mark(h, 1, s);
    NC_TRY(matvec_tail(h, h->d_hx, h->d_hy, s));
  }
  NC_CUDA_TRY(cudaMemcpyAsync(y_host, h->d_hy, n * sizeof(double), cudaMemcpyDeviceToHost, s));
  NC_CUDA_TRY(cudaStreamSynchronize(s));
  return NC_OK;
}

// helper: device dot products of V[0..nv) with w into d_out (nv doubles), all-reduced across ranks
static int dots(nc_handle* h, const double* V, int64_t ldv, int nv, const double* w, int64_t n, double* d_out,
                cudaStream_t s) {
  double* part = h->d_red + 2048;   // partial buffer region (needs nv * 592 doubles)
  launch_multidot(V, ldv, nv, w, n, part, d_out, s);
  return allreduce_sum(h, d_out, nv, s);
}

int nc_gmres(nc_handle* h, const double* b, double rtol, int max_iter, double* x, int* iters, double* hist,
             void* stream) {
  if (!h || !x || max_iter < 1 || !(rtol > 0)) return fail(NC_EINVAL, "nc_gmres: bad arguments");
  if (h->world > 1 && h->emulated) return fail(NC_ESTATE, "nc_gmres: emulated rank has no communicator");
  NC_CUDA_TRY(cudaSetDevice(h->device));
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t n = h->row_count * h->K;
  const int64_t ldv = std::max<int64_t>(n, 1);
  // Krylov basis: allocated for min(max_iter + 1, 64) vectors and doubled on demand inside the iteration (a C5
  // vector is 109 MB: allocating max_iter + 1 = 301 of them up front would put a 33 GB cudaMalloc in every solve)
  auto grow_V = [&](int need, int nkeep) -> int {
    if (h->V_cap >= need) return NC_OK;
    const int cap = std::min(max_iter + 1, std::max(need, std::max(64, 2 * h->V_cap)));
    double* nv = nullptr;
    NC_TRY(dalloc(h, &nv, (size_t)cap * ldv));
    if (h->d_V && nkeep > 0)
      NC_CUDA_TRY(cudaMemcpyAsync(nv, h->d_V, (size_t)nkeep * ldv * sizeof(double), cudaMemcpyDeviceToDevice, s));
    if (h->d_V) {
      NC_CUDA_TRY(cudaStreamSynchronize(s));
      cudaFree(h->d_V);
      h->device_bytes -= (double)h->V_cap * ldv * sizeof(double);
    }
    h->d_V = nv;
    h->V_cap = cap;
    return NC_OK;
  };
  NC_TRY(grow_V(std::min(max_iter + 1, 64), 0));
  // reduction scratch: [0, 2048) small vectors, [2048, ...) multidot partials
  NC_TRY(ensure_red(h, 2048 + (int64_t)(max_iter + 2) * multidot_partials(n) + 16));
  double* V = h->d_V;                 // (re-read after every growth of the basis)
  double* d_h1 = h->d_red;            // first-pass projections  (<= max_iter+1)
  double* d_h2 = h->d_red + 640;      // second-pass projections
  double* d_nrm = h->d_red + 1280;    // ||w||^2
  if (max_iter + 1 > 640) return fail(NC_EINVAL, "nc_gmres: max_iter must be <= 639");

  // v0 = b / ||b||
  if (b) {
    NC_CUDA_TRY(cudaMemcpyAsync(V, b, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
  } else {
    if (!h->d_b) NC_TRY(dalloc(h, &h->d_b, (size_t)h->K));
    NC_CUDA_TRY(cudaMemcpyAsync(h->d_b, h->h_P1.data(), h->K * sizeof(double), cudaMemcpyHostToDevice, s));
    launch_fill_rows(V, h->d_b, h->K, h->row_count, s);
  }
  NC_TRY(dots(h, V, ldv, 1, V, n, d_nrm, s));
  NC_CUDA_TRY(cudaMemcpyAsync(h->h_red, d_nrm, sizeof(double), cudaMemcpyDeviceToHost, s));
  NC_TRY(wait_stream(h, s, "nc_gmres"));
  const double beta = sqrt(h->h_red[0]);
  if (hist) hist[0] = 1.0;
  if (beta == 0.0) {
    NC_CUDA_TRY(cudaMemsetAsync(x, 0, n * sizeof(double), s));
    if (iters) *iters = 0;
    NC_CUDA_TRY(cudaStreamSynchronize(s));
    return NC_OK;
  }
  {
    double inv = beta;
    NC_CUDA_TRY(cudaMemcpyAsync(d_nrm, &inv, sizeof(double), cudaMemcpyHostToDevice, s));
    launch_scale(V, V, d_nrm, 1, n, s);
  }
  const int m = max_iter;
  std::vector<double> H((size_t)(m + 1) * m, 0.0), cs(m), sn(m), g(m + 1, 0.0);
  auto Hc = [&](int i, int j) -> double& { return H[(size_t)i * m + j]; };
  g[0] = beta;
  int k = 0;
  bool converged = false;
  for (int j = 0; j < m; ++j) {
    if (j + 2 > h->V_cap) {   // room for v_{j+1}
      NC_TRY(grow_V(j + 2, j + 1));
      V = h->d_V;
    }
    double* w = V + (size_t)(j + 1) * ldv;
    NC_TRY(nc_matvec(h, V + (size_t)j * ldv, w, s));
    // CGS2: two classical Gram-Schmidt passes
    if (h->time_stages) NC_CUDA_TRY(cudaEventRecord(h->ev[5], s));
    NC_TRY(dots(h, V, ldv, j + 1, w, n, d_h1, s));
    launch_gemv_sub(V, ldv, j + 1, d_h1, w, n, s);
    NC_TRY(dots(h, V, ldv, j + 1, w, n, d_h2, s));
    launch_gemv_sub(V, ldv, j + 1, d_h2, w, n, s);
    NC_TRY(dots(h, w, ldv, 1, w, n, d_nrm, s));
    if (h->time_stages) NC_CUDA_TRY(cudaEventRecord(h->ev[6], s));
    NC_CUDA_TRY(cudaMemcpyAsync(h->h_red, h->d_red, 1281 * sizeof(double), cudaMemcpyDeviceToHost, s));
    NC_TRY(wait_stream(h, s, "nc_gmres"));
    if (h->time_stages) {
      // HBM-bound orthogonalisation (K9): algorithmic bytes = two (multidot + gemv_sub) passes + the norm, with
      // multidot re-reading w once per group of 8 basis vectors
      float ms = 0.f;
      cudaEventElapsedTime(&ms, h->ev[5], h->ev[6]);
      const double nv = j + 1;
      h->gmres_ortho_ms += ms;
      h->gmres_ortho_bytes += 8.0 * (double)n * (2.0 * (nv + std::ceil(nv / 8.0)) + 2.0 * (nv + 2.0) + 1.0);
      h->gmres_ortho_iters++;
    }
    for (int i = 0; i <= j; ++i) Hc(i, j) = h->h_red[i] + h->h_red[640 + i];
    double hn = sqrt(std::max(0.0, h->h_red[1280]));
    Hc(j + 1, j) = hn;
    if (hn > 0) {
      NC_CUDA_TRY(cudaMemcpyAsync(d_nrm, &Hc(j + 1, j), sizeof(double), cudaMemcpyHostToDevice, s));
      launch_scale(w, w, d_nrm, 1, n, s);
    }
    for (int i = 0; i < j; ++i) {
      double t = cs[i] * Hc(i, j) + sn[i] * Hc(i + 1, j);
      Hc(i + 1, j) = -sn[i] * Hc(i, j) + cs[i] * Hc(i + 1, j);
      Hc(i, j) = t;
    }
    double r = hypot(Hc(j, j), Hc(j + 1, j));
    cs[j] = Hc(j, j) / r;
    sn[j] = Hc(j + 1, j) / r;
    Hc(j, j) = r;
    Hc(j + 1, j) = 0.0;
    g[j + 1] = -sn[j] * g[j];
    g[j] = cs[j] * g[j];
    k = j + 1;
    double rel = fabs(g[j + 1]) / beta;
    if (hist) hist[k] = rel;
    if (rel <= rtol) {
      converged = true;
      break;
    }
    if (hn == 0.0) break;   // lucky breakdown
  }
  std::vector<double> yv(k, 0.0);
  for (int i = k - 1; i >= 0; --i) {
    double v = g[i];
    for (int l = i + 1; l < k; ++l) v -= Hc(i, l) * yv[l];
    yv[i] = v / Hc(i, i);
  }
  NC_CUDA_TRY(cudaMemcpyAsync(h->d_red, yv.data(), k * sizeof(double), cudaMemcpyHostToDevice, s));
  launch_lincomb(V, ldv, k, h->d_red, x, n, s);
  NC_CUDA_TRY(cudaStreamSynchronize(s));
  NC_CUDA_TRY(cudaGetLastError());
  if (iters) *iters = k;
  if (!converged && fabs(g[k]) / beta > rtol)
    return fail(NC_ENOCONV, "nc_gmres: no convergence in " + std::to_string(k) + " iterations");
  return NC_OK;
}

// The synchronous diagnostics below (read-out, field, residual, density) run on the handle's private stream.  They
// take x from the caller, written by work on any stream (a matvec / GMRES on the caller's stream, torch ops on the
// legacy stream): wait for all device work issued so far before reading it.
static int order_after_caller(nc_handle* h) {
  NC_CUDA_TRY(cudaSetDevice(h->device));
  NC_CUDA_TRY(cudaDeviceSynchronize());
  return NC_OK;
}

// The base rung's source records (coordinates of every patch's skeleton nodes, scaled by 1/2, and rho = T fhat) in a
// buffer of the call's own: the field and residual entry points never write the matvec's records or rho.
// Layout: N p0 records (x, y, z, rho) for the field kernels, then the same rho compactly (N p0) for the pair kernels.
static int base_records(nc_handle* h, const double* x_all, cudaStream_t s, double** out) {
  const int K = h->K, p0 = h->rung_p[0];
  const size_t n = (size_t)h->N * p0 * 4;
  double* d = nullptr;
  if (cudaMalloc(&d, (n + n / 4) * sizeof(double)) != cudaSuccess) {
    (void)cudaGetLastError();
    return fail(NC_ENOMEM, "base records: device allocation failed");
  }
  cudaError_t e = cudaMemcpyAsync(d, h->d_src4 + h->rung_soff[0], n * sizeof(double), cudaMemcpyDeviceToDevice, s);
  if (e == cudaSuccess) {   // rho of the base rung for all N patches (K1 restricted to rung 0) into slot 3
    launch_gemm_dmma(x_all, K, 1, 0, h->d_T + (size_t)h->rung_trow[0] * K, h->N, p0, K, d + 3, (int64_t)p0 * 4, 4,
                     nullptr, 0, s);
    launch_gemm_dmma(x_all, K, 1, 0, h->d_T + (size_t)h->rung_trow[0] * K, h->N, p0, K, d + n, (int64_t)p0, 1,
                     nullptr, 0, s);
    e = cudaGetLastError();
  }
  if (e != cudaSuccess) {
    cudaFree(d);
    return cuda_fail(e, "base records");
  }
  *out = d;
  return NC_OK;
}

int nc_flux_or_mfpt(nc_handle* h, const double* x, double* I_sigma, double* value) {
  if (!h || !x) return fail(NC_EINVAL, "nc_flux_or_mfpt: null argument");
  if (h->world > 1 && h->emulated) return fail(NC_ESTATE, "nc_flux_or_mfpt: emulated rank has no communicator");
  NC_TRY(order_after_caller(h));
  cudaStream_t s = h->stream;
  NC_TRY(ensure_red(h, std::max<int64_t>(4096, 1024 + (int64_t)592 * h->K + 16)));
  double* d_sum = h->d_red;             // K <= 1024 (checked in nc_setup)
  double* part = h->d_red + 1024;
  launch_colsum(x, h->row_count, h->K, part, d_sum, s);
  NC_TRY(allreduce_sum(h, d_sum, h->K, s));
  std::vector<double> col(h->K);
  NC_CUDA_TRY(cudaMemcpyAsync(col.data(), d_sum, h->K * sizeof(double), cudaMemcpyDeviceToHost, s));
  NC_TRY(wait_stream(h, s, "nc_flux_or_mfpt"));
  double Is = 0.0;
  for (int a = 0; a < h->K; ++a) Is += h->h_I[a] * col[a];
  if (I_sigma) *I_sigma = Is;
  double v;
  if (h->kind == NC_INTERIOR) {
    if (!(Is > 0.0)) return fail(NC_ESTATE, "nc_flux_or_mfpt: interior I_sigma <= 0");
    v = 1.0 / (3.0 * Is) - 3.0 / 5.0;   // eq:mufromsigma2
  } else {
    v = -4.0 * M_PI * Is;                // J = -4 pi I_sigma (R2)
  }
  if (value) *value = v;
  return NC_OK;
}

int nc_field(nc_handle* h, const double* x_all, int64_t n_pts, const double* pts, double* out, double* dmin) {
  if (!h || !x_all || n_pts < 0 || (n_pts > 0 && (!pts || !out))) return fail(NC_EINVAL, "nc_field: bad argument");
  if (n_pts == 0) return NC_OK;
  for (int64_t t = 0; t < n_pts; ++t) {   // the problem's side of the sphere (interior: inside, exterior: outside)
    const double r = std::sqrt(pts[3 * t] * pts[3 * t] + pts[3 * t + 1] * pts[3 * t + 1] + pts[3 * t + 2] * pts[3 * t + 2]);
    if (!(h->kind == NC_EXTERIOR ? r > 1.0 : r < 1.0))
      return fail(NC_EINVAL, "nc_field: point " + std::to_string(t) + " is not on the " +
                                 (h->kind == NC_EXTERIOR ? "exterior" : "interior") + " side of the unit sphere");
  }
  NC_TRY(order_after_caller(h));
  cudaStream_t s = h->stream;
  const int p0 = h->rung_p[0];
  double* d_rec = nullptr;
  NC_TRY(base_records(h, x_all, s, &d_rec));
  const int64_t nrec = h->N * p0;
  const int nseg = field_segments(n_pts, nrec);
  double *d_pts = nullptr, *d_part = nullptr, *d_out = nullptr;
  cudaError_t e = cudaMalloc(&d_pts, (size_t)n_pts * 3 * sizeof(double));
  if (e == cudaSuccess) e = cudaMalloc(&d_part, (size_t)2 * nseg * n_pts * sizeof(double));
  if (e == cudaSuccess) e = cudaMalloc(&d_out, (size_t)2 * n_pts * sizeof(double));
  int rc = NC_OK;
  if (e != cudaSuccess) {
    (void)cudaGetLastError();
    rc = fail(NC_ENOMEM, "nc_field: device allocation failed");
  } else {
    e = cudaMemcpyAsync(d_pts, pts, (size_t)n_pts * 3 * sizeof(double), cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) {
      launch_field(h->kind, d_pts, n_pts, d_rec, nrec, nseg, d_part, d_part + (size_t)nseg * n_pts, d_out,
                   d_out + n_pts, s);
      e = cudaGetLastError();
    }
    std::vector<double> dm(n_pts);
    if (e == cudaSuccess) e = cudaMemcpyAsync(out, d_out, (size_t)n_pts * sizeof(double), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(dm.data(), d_out + n_pts, (size_t)n_pts * sizeof(double), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) {
      rc = cuda_fail(e, "nc_field");
    } else {
      if (dmin) std::copy(dm.begin(), dm.end(), dmin);
      for (int64_t t = 0; t < n_pts && rc == NC_OK; ++t)
        if (!(dm[t] >= 3.0 * h->eps))
          rc = fail(NC_EINVAL, "nc_field: point " + std::to_string(t) + " is " + std::to_string(dm[t] / h->eps) +
                                   " eps from a skeleton node (< 3 eps: the compressed representation is not valid)");
    }
  }
  cudaFree(d_pts);
  cudaFree(d_part);
  cudaFree(d_out);
  cudaFree(d_rec);
  return rc;
}

int nc_field_near(nc_handle* h, const double* x_all, int64_t n_pts, const double* pts, const nc_near_tables* nt,
                  double* out, double* mfpt, int64_t* n_near) {
  if (!h || !x_all || n_pts < 0 || (n_pts > 0 && (!pts || !out)) || !nt || !nt->edges || !nt->t || !nt->w ||
      !nt->sigma || !nt->m || !nt->c || nt->npan < 1 || nt->k < 2 || nt->k > 32)
    return fail(NC_EINVAL, "nc_field_near: bad argument");
  if (mfpt && h->kind != NC_INTERIOR) return fail(NC_EINVAL, "nc_field_near: the MFPT is an interior quantity");
  const int K = h->K, n_r = nt->npan * nt->k;
  int M1 = 0;
  for (int a = 0; a < K; ++a) {
    if (nt->m[a] < 0 || nt->m[a] > 15 || (nt->c[a] != 1 && nt->c[a] != -1))
      return fail(NC_EINVAL, "nc_field_near: basis orders must be 0..15 with c = +-1");
    M1 = std::max(M1, nt->m[a] + 1);
  }
  if (n_near) *n_near = 0;
  if (n_pts == 0) return NC_OK;
  for (int64_t t = 0; t < n_pts; ++t) {
    const double r = std::sqrt(pts[3 * t] * pts[3 * t] + pts[3 * t + 1] * pts[3 * t + 1] + pts[3 * t + 2] * pts[3 * t + 2]);
    if (!(h->kind == NC_EXTERIOR ? r > 1.0 : r < 1.0))
      return fail(NC_EINVAL, "nc_field_near: point " + std::to_string(t) + " is not on the " +
                                 (h->kind == NC_EXTERIOR ? "exterior" : "interior") + " side of the unit sphere");
  }
  NC_TRY(order_after_caller(h));
  cudaStream_t s = h->stream;
  const int p0 = h->rung_p[0];
  double* d_rec = nullptr;
  NC_TRY(base_records(h, x_all, s, &d_rec));
  const int64_t nrec = h->N * p0;
  const int nseg = field_segments(n_pts, nrec);
  // host-built near table: reference Gauss nodes / weights of the regular panels (from the first panel), their
  // barycentric weights, the (m, cos | sin) CSR of the basis columns, the angle table
  std::vector<double> glx(nt->k), glw(nt->k), bary(nt->k), trig(2 * kNearTrigN);
  {
    const double a = nt->edges[0], b = nt->edges[1], hh = 0.5 * (b - a);
    for (int e = 0; e < nt->k; ++e) {
      glx[e] = (nt->t[e] - a) / hh - 1.0;
      glw[e] = nt->w[e] / (hh * std::sin(nt->t[e]));
    }
    for (int e = 0; e < nt->k; ++e) {
      long double pr = 1.0L;
      for (int f = 0; f < nt->k; ++f)
        if (f != e) pr *= (long double)(glx[e] - glx[f]);
      bary[e] = (double)(1.0L / pr);
    }
    for (int k = 0; k < kNearTrigN; ++k) {
      const long double th = 2.0L * 3.14159265358979323846264338327950288L * k / kNearTrigN;
      trig[2 * k] = (double)cosl(th);
      trig[2 * k + 1] = (double)sinl(th);
    }
  }
  std::vector<int> mc_off(2 * M1 + 1, 0), mc_col;
  for (int comp = 0; comp < 2 * M1; ++comp) {
    for (int a = 0; a < K; ++a)
      if (2 * nt->m[a] + (nt->c[a] > 0 ? 0 : 1) == comp) mc_col.push_back(a);
    mc_off[comp + 1] = (int)mc_col.size();
  }
  std::vector<void*> bufs;
  auto dup = [&](const void* src, size_t bytes, void** dst) -> cudaError_t {
    cudaError_t e = cudaMalloc(dst, std::max<size_t>(bytes, 16));
    if (e != cudaSuccess) return e;
    bufs.push_back(*dst);
    return cudaMemcpyAsync(*dst, src, bytes, cudaMemcpyHostToDevice, s);
  };
  NearDev nd{};
  nd.npan = nt->npan; nd.k = nt->k; nd.n_r = n_r; nd.M1 = M1; nd.K = K;
  double *d_pts = nullptr, *d_part = nullptr, *d_out = nullptr, *d_corr = nullptr;
  int64_t *d_cnt = nullptr, *d_off = nullptr, *d_list = nullptr, *d_ppt = nullptr;
  int* d_status = nullptr;
  int rc = NC_OK;
  cudaError_t e = cudaSuccess;
  void* v = nullptr;
#define NC_DUP(ptr, bytes, field) \
  if (e == cudaSuccess) { e = dup(ptr, bytes, &v); field = (decltype(field))v; }
  NC_DUP(nt->edges, (size_t)(nt->npan + 1) * 8, nd.edges)
  NC_DUP(nt->t, (size_t)n_r * 8, nd.t)
  NC_DUP(nt->w, (size_t)n_r * 8, nd.w)
  NC_DUP(nt->sigma, (size_t)K * n_r * 8, nd.sigma)
  NC_DUP(mc_off.data(), mc_off.size() * sizeof(int), nd.mc_off)
  NC_DUP(mc_col.data(), mc_col.size() * sizeof(int), nd.mc_col)
  NC_DUP(glx.data(), glx.size() * 8, nd.gl_x)
  NC_DUP(glw.data(), glw.size() * 8, nd.gl_w)
  NC_DUP(bary.data(), bary.size() * 8, nd.bary)
  NC_DUP(trig.data(), trig.size() * 8, nd.trig)
  NC_DUP(pts, (size_t)n_pts * 3 * 8, d_pts)
#undef NC_DUP
  auto dal = [&](size_t bytes, void** dst) -> cudaError_t {
    cudaError_t e2 = cudaMalloc(dst, std::max<size_t>(bytes, 16));
    if (e2 == cudaSuccess) bufs.push_back(*dst);
    return e2;
  };
  if (e == cudaSuccess) e = dal((size_t)2 * nseg * n_pts * 8, &v), d_part = (double*)v;
  if (e == cudaSuccess) e = dal((size_t)2 * n_pts * 8, &v), d_out = (double*)v;
  if (e == cudaSuccess) e = dal((size_t)(n_pts + 1) * 8, &v), d_cnt = (int64_t*)v;
  if (e == cudaSuccess) e = dal((size_t)(n_pts + 1) * 8, &v), d_off = (int64_t*)v;
  if (e == cudaSuccess) e = dal(sizeof(int), &v), d_status = (int*)v;
  int64_t npairs = 0;
  std::vector<int64_t> off(n_pts + 1, 0);
  if (e == cudaSuccess) {
    // the compressed field of every patch, then the near pairs
    launch_field(h->kind, d_pts, n_pts, d_rec, nrec, nseg, d_part, d_part + (size_t)nseg * n_pts, d_out,
                 d_out + n_pts, s);
    launch_near_count(d_pts, n_pts, h->d_centers, h->N, kNearRadius * h->eps, d_cnt, nullptr, nullptr, s);
    std::vector<int64_t> cnt(n_pts);
    e = cudaMemcpyAsync(cnt.data(), d_cnt, (size_t)n_pts * 8, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    for (int64_t t = 0; t < n_pts && e == cudaSuccess; ++t) {
      off[t + 1] = off[t] + cnt[t];
      const double r = std::sqrt(pts[3 * t] * pts[3 * t] + pts[3 * t + 1] * pts[3 * t + 1] + pts[3 * t + 2] * pts[3 * t + 2]);
      if (cnt[t] > 0 && std::fabs(1.0 - r) < kNearMinHeight * h->eps && rc == NC_OK)
        rc = fail(NC_EINVAL, "nc_field_near: point " + std::to_string(t) + " is closer than eps/100 to the sphere "
                             "near a patch");
    }
    npairs = off[n_pts];
  }
  if (e == cudaSuccess && rc == NC_OK && npairs > 0) {
    std::vector<int64_t> ppt(npairs);
    for (int64_t t = 0; t < n_pts; ++t)
      for (int64_t q = off[t]; q < off[t + 1]; ++q) ppt[q] = t;
    e = cudaMemcpyAsync(d_off, off.data(), (size_t)(n_pts + 1) * 8, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = dal((size_t)npairs * 8, &v), d_list = (int64_t*)v;
    if (e == cudaSuccess) e = dal((size_t)npairs * 8, &v), d_corr = (double*)v;
    if (e == cudaSuccess) e = dup(ppt.data(), (size_t)npairs * 8, &v), d_ppt = (int64_t*)v;
    if (e == cudaSuccess) e = cudaMemsetAsync(d_status, 0, sizeof(int), s);
    if (e == cudaSuccess) {
      launch_near_count(d_pts, n_pts, h->d_centers, h->N, kNearRadius * h->eps, nullptr, d_list, d_off, s);
      launch_near_quad(h->kind, d_ppt, d_list, npairs, d_pts, h->d_frames, x_all, nd, d_rec, p0, d_corr, d_status, s);
      launch_near_apply(d_off, d_corr, n_pts, d_out, s);
      e = cudaGetLastError();
    }
    int status = 0;
    if (e == cudaSuccess) e = cudaMemcpyAsync(&status, d_status, sizeof(int), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e == cudaSuccess && status)
      rc = fail(NC_EINVAL, status == 1 ? "nc_field_near: a point needs more than the radial node budget"
                                       : "nc_field_near: a point is too close to a patch for the angular rule");
  }
  if (e == cudaSuccess && rc == NC_OK) e = cudaMemcpyAsync(out, d_out, (size_t)n_pts * 8, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess && rc == NC_OK) rc = cuda_fail(e, "nc_field_near");
  if (rc == NC_OK && mfpt) {   // vbar (eq:vtilde) with D = -I_sigma; I_sigma = I . sum_i fhat_i (eq:getI)
    rc = ensure_red(h, std::max<int64_t>(4096, 1024 + (int64_t)592 * h->K + 16));
    if (rc == NC_OK) {
      double* d_sum = h->d_red;
      launch_colsum(x_all, h->N, h->K, h->d_red + 1024, d_sum, s);
      std::vector<double> col(h->K);
      e = cudaMemcpyAsync(col.data(), d_sum, h->K * sizeof(double), cudaMemcpyDeviceToHost, s);
      if (e == cudaSuccess) e = cudaStreamSynchronize(s);
      if (e != cudaSuccess) rc = cuda_fail(e, "nc_field_near (I_sigma)");
      double Is = 0.0;
      for (int a = 0; a < h->K; ++a) Is += h->h_I[a] * col[a];
      const double D = -Is;
      for (int64_t t = 0; t < n_pts && rc == NC_OK; ++t) {
        const double r2 = pts[3 * t] * pts[3 * t] + pts[3 * t + 1] * pts[3 * t + 1] + pts[3 * t + 2] * pts[3 * t + 2];
        mfpt[t] = (out[t] - 1.0) / (3.0 * D) + (1.0 - r2) / 6.0;
      }
    }
  }
  if (n_near) *n_near = npairs;
  for (void* b : bufs) cudaFree(b);
  cudaFree(d_rec);
  return rc;
}

int nc_residual(nc_handle* h, const double* x_all, int n_sel, const int64_t* patches, int n_res,
                const double* res_rhat, const double* res_w, const double* res_S, double* res, double* pointwise) {
  if (!h || !x_all || n_sel < 0 || n_res < 1 || (n_sel > 0 && (!patches || !res_rhat || !res_w || !res_S || !res)))
    return fail(NC_EINVAL, "nc_residual: bad argument");
  if (n_sel == 0) return NC_OK;
  std::vector<int64_t> inv(h->N);
  for (int64_t r = 0; r < h->N; ++r) inv[h->perm[r]] = r;
  std::vector<int64_t> rows(n_sel);
  for (int q = 0; q < n_sel; ++q) {
    if (patches[q] < 0 || patches[q] >= h->N)
      return fail(NC_EINVAL, "nc_residual: patch index " + std::to_string(patches[q]) + " out of range");
    rows[q] = inv[patches[q]];
  }
  NC_TRY(order_after_caller(h));
  cudaStream_t s = h->stream;
  const int K = h->K, p0 = h->rung_p[0];
  double* d_rec = nullptr;
  NC_TRY(base_records(h, x_all, s, &d_rec));
  const double* src0 = d_rec;
  const int nseg = (int)std::min<int64_t>(h->N, 128);
  const size_t nr = (size_t)n_res;
  double *d_rhat = nullptr, *d_w = nullptr, *d_S = nullptr, *d_t = nullptr, *d_up = nullptr, *d_out = nullptr;
  int64_t* d_rows = nullptr;
  cudaError_t e = cudaMalloc(&d_rhat, nr * 3 * sizeof(double));
  if (e == cudaSuccess) e = cudaMalloc(&d_w, nr * sizeof(double));
  if (e == cudaSuccess) e = cudaMalloc(&d_S, nr * K * sizeof(double));
  if (e == cudaSuccess) e = cudaMalloc(&d_t, (size_t)n_sel * nr * 3 * sizeof(double));
  if (e == cudaSuccess) e = cudaMalloc(&d_up, (size_t)n_sel * nseg * nr * sizeof(double));
  if (e == cudaSuccess) e = cudaMalloc(&d_out, ((size_t)n_sel * nr + n_sel) * sizeof(double));
  if (e == cudaSuccess) e = cudaMalloc(&d_rows, (size_t)n_sel * sizeof(int64_t));
  int rc = NC_OK;
  if (e != cudaSuccess) {
    (void)cudaGetLastError();
    rc = fail(NC_ENOMEM, "nc_residual: device allocation failed");
  } else {
    e = cudaMemcpyAsync(d_rhat, res_rhat, nr * 3 * sizeof(double), cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(d_w, res_w, nr * sizeof(double), cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(d_S, res_S, nr * K * sizeof(double), cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(d_rows, rows.data(), (size_t)n_sel * sizeof(int64_t), cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) {
      for (int q = 0; q < n_sel; ++q) {   // the residual grid on patch rows[q] (scaled by 1/2), then the other patches' field
        double* tx = d_t + (size_t)q * nr * 3;
        launch_targets(h->d_frames, rows[q], 1, d_rhat, n_res, 0.5, tx, tx + nr, tx + 2 * nr, s);
        launch_pairs_direct(h->kind, h->pair_tpt, tx, tx + nr, tx + 2 * nr, n_res, n_res, rows[q], src0,
                            src0 + (size_t)h->N * p0 * 4, p0, h->N, nseg,
                            d_up + (size_t)q * nseg * nr, h->xtab, h->eps, s);
      }
      launch_residual(n_sel, n_res, K, nseg, d_rows, x_all, d_S, d_w, d_up, d_out, d_out + (size_t)n_sel * nr, s);
      e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpyAsync(res, d_out + (size_t)n_sel * nr, (size_t)n_sel * sizeof(double), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess && pointwise)
      e = cudaMemcpyAsync(pointwise, d_out, (size_t)n_sel * nr * sizeof(double), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) rc = cuda_fail(e, "nc_residual");
  }
  for (void* b : {(void*)d_rhat, (void*)d_w, (void*)d_S, (void*)d_t, (void*)d_up, (void*)d_out, (void*)d_rows,
                  (void*)d_rec})
    cudaFree(b);
  return rc;
}

int nc_density(nc_handle* h, const double* x_all, int n_sel, const int64_t* patches, int n_f, const double* B,
               double* sigma) {
  if (!h || !x_all || n_sel < 0 || n_f < 1 || (n_sel > 0 && (!patches || !B || !sigma)))
    return fail(NC_EINVAL, "nc_density: bad argument");
  if (n_sel == 0) return NC_OK;
  std::vector<int64_t> inv(h->N), rows(n_sel);
  for (int64_t r = 0; r < h->N; ++r) inv[h->perm[r]] = r;
  for (int q = 0; q < n_sel; ++q) {
    if (patches[q] < 0 || patches[q] >= h->N)
      return fail(NC_EINVAL, "nc_density: patch index " + std::to_string(patches[q]) + " out of range");
    rows[q] = inv[patches[q]];
  }
  NC_TRY(order_after_caller(h));
  cudaStream_t s = h->stream;
  const int K = h->K;
  double *d_B = nullptr, *d_x = nullptr, *d_s = nullptr;
  int64_t* d_rows = nullptr;
  cudaError_t e = cudaMalloc(&d_B, (size_t)n_f * K * sizeof(double));
  if (e == cudaSuccess) e = cudaMalloc(&d_x, (size_t)n_sel * K * sizeof(double));
  if (e == cudaSuccess) e = cudaMalloc(&d_s, (size_t)n_sel * n_f * sizeof(double));
  if (e == cudaSuccess) e = cudaMalloc(&d_rows, (size_t)n_sel * sizeof(int64_t));
  int rc = NC_OK;
  if (e != cudaSuccess) {
    (void)cudaGetLastError();
    rc = fail(NC_ENOMEM, "nc_density: device allocation failed");
  } else {
    e = cudaMemcpyAsync(d_B, B, (size_t)n_f * K * sizeof(double), cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(d_rows, rows.data(), (size_t)n_sel * sizeof(int64_t), cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) {
      launch_gather_rows(x_all, d_rows, n_sel, K, d_x, s);
      // sigma (n_sel x n_f) = X_sel (n_sel x K) . B^T
      launch_gemm_dmma(d_x, K, 1, 0, d_B, n_sel, n_f, K, d_s, n_f, 1, nullptr, 0, s);
      e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpyAsync(sigma, d_s, (size_t)n_sel * n_f * sizeof(double), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) rc = cuda_fail(e, "nc_density");
  }
  for (void* b : {(void*)d_B, (void*)d_x, (void*)d_s, (void*)d_rows}) cudaFree(b);
  return rc;
}

int nc_stats(const nc_handle* h, nc_stats_t* o) {
  if (!h || !o) return fail(NC_EINVAL, "nc_stats: null argument");
  NC_TRY(read_stages(const_cast<nc_handle*>(h)));
  memset(o, 0, sizeof(*o));
  o->N = h->N;
  o->row_begin = h->row_begin;
  o->row_count = h->row_count;
  o->K = h->K;
  o->Kstar = h->Kstar;
  o->p = h->p;
  o->mode = h->mode;
  o->world = h->world;
  o->rank = h->rank;
  o->matvecs = h->matvecs;
  o->pairs_per_matvec = h->pairs_per_matvec;
  double psum = 0.0;
  for (int k = 0; k < h->nrung; ++k)
    if (h->rung_used[k]) psum += h->rung_p[k];
  o->gemm_flops_per_matvec = 2.0 * h->row_count * (psum * h->K + (double)h->K * h->Kstar);
  for (int i = 0; i < 8; ++i) o->ms_last[i] = h->ms_last[i];
  o->device_bytes = h->device_bytes;
  o->launches_per_matvec = h->launches_last;
  o->gmres_ortho_ms = h->gmres_ortho_ms;
  o->gmres_ortho_bytes = h->gmres_ortho_bytes;
  o->gmres_ortho_iters = h->gmres_ortho_iters;
  // per-pair FP64 work of the pair kernels (green.cuh / pairs.cuh; SASS counts, checked against ncu's
  // sass_thread_inst_executed_op_{dfma,dmul,dadd}): exact form 11 DFMA + 4 DMUL + 7 DADD exterior, 12 DFMA + 4 DMUL +
  // 6 DADD interior;
  // far-field form (R23, green_far_h) 10 DFMA + 2 DMUL + 4 DADD exterior, 11 DFMA + 2 DMUL + 3 DADD interior
  const int interior = h->kind == NC_INTERIOR;
  // exact form with the exact-form table (green_exact_r, default): 11 DFMA + 3 DMUL + 5 DADD exterior (30 flops),
  // 12 + 3 + 4 interior (31)
  o->pair_fp64_inst_direct = h->xtab.d ? 19 : 22;
  o->pair_fp64_flops_direct = h->xtab.d ? 30 + interior : 33 + interior;
  // far table (R25, green_far_t) cubic: 10 DFMA + 1 DMUL + 2 DADD exterior (23 flops), 11 + 1 + 1 interior (24);
  // quartic: one DFMA more
  const int far = hier_grid_far(h);
  if (far == 8 || far == 9) {   // FB = 9 quadratic (R32, R35): 9 DFMA + 1 DMUL + 2 DADD exterior (21 flops), 10 + 1 + 1 interior (22)
    o->pair_fp64_inst_grid = 12;
    o->pair_fp64_flops_grid = 21 + interior;
  } else if (far >= 2) {
    const int quartic = far == 3 || far == 6;
    o->pair_fp64_inst_grid = 13 + quartic;
    o->pair_fp64_flops_grid = 23 + interior + 2 * quartic;
  } else {
    o->pair_fp64_inst_grid = far ? 16 : 22;
    o->pair_fp64_flops_grid = far ? 26 + interior : 33 + interior;
  }
  hier_fill_stats(h, o);
  return NC_OK;
}

int nc_split_rows(const double* weights, int64_t N, int world, int64_t* begin, int64_t* count) {
  if (N < 0 || world < 1 || !begin || !count) return fail(NC_EINVAL, "nc_split_rows: bad arguments");
  split_rows(weights, N, world, begin, count);
  return NC_OK;
}

int nc_nccl_unique_id(void* id_out) {
  if (!id_out) return fail(NC_EINVAL, "nc_nccl_unique_id: null buffer");
#if NC_WITH_NCCL
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) return fail(NC_ENCCL, std::string("ncclGetUniqueId: ") + ncclGetErrorString(r));
  memcpy(id_out, &id, sizeof(id));
  return NC_OK;
#else
  return fail(NC_EUNSUP, "built without NCCL");
#endif
}

void nc_destroy(nc_handle* h) {
  if (!h) return;
  cudaSetDevice(h->device);
  if (h->stream) cudaStreamSynchronize(h->stream);
  hier_destroy(h);
  double* bufs[] = {h->d_T, h->d_P, h->d_I, h->d_zhat, h->d_shat, h->d_centers, h->d_frames, h->d_tx, h->d_ty,
                    h->d_tz, h->d_src4, h->d_rho, h->d_upart, h->d_V, h->d_red, h->d_b, h->d_hx, h->d_hy, h->d_Tcat, h->d_xall,
                    h->d_xpad};
  if (h->d_xtab) cudaFree(h->d_xtab);
  for (double* b : bufs)
    if (b) cudaFree(b);
  if (h->d_colbase) cudaFree(h->d_colbase);
  if (h->d_colrstride) cudaFree(h->d_colrstride);
  if (h->h_red) cudaFreeHost(h->h_red);
  for (auto& ev : h->ev)
    if (ev) cudaEventDestroy(ev);
  if (h->ev_order) cudaEventDestroy(h->ev_order);
  for (auto& ev : h->copy_ev)
    if (ev) cudaEventDestroy(ev);
  if (h->copy_stream) cudaStreamDestroy(h->copy_stream);
  if (h->stream) cudaStreamDestroy(h->stream);
#if NC_WITH_NCCL
  if (h->comm) ncclCommDestroy(h->comm);
#endif
  delete h;
}

}  // extern "C"
