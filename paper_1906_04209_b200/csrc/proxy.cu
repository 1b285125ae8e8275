// proxy.cu -- patch-local proxy points for step 4 (R36; host-side setup arithmetic only).
//
// Step 4 evaluates, for every patch and every level, the group's incoming expansion at the
// patch's K* Zernike nodes.  At a level whose grid sources are all far from the patch (distance D >= kappa h from
// the patch centre, h = the node disk's radius), the expansion restricted to the patch is a smooth function of the
// patch's tangent-plane coordinates (u, v): polynomials of total degree <= d reproduce it to ~(h / 2D)^d.  Such
// levels are evaluated at n < K* proxy points instead, summed over levels, and carried to the nodes by one fixed
// K* x n matrix (a DMMA GEMM over all patches):
//
//   u(nodes) = sum_{near levels} E_l(nodes) + Int . sum_{far levels} E_l(proxies),   Int = V_nodes pinv(V_prox),
//
// V the Chebyshev-product basis T_a(u / h) T_b(v / h), a + b <= d (well conditioned on the disk |(u, v)| <= h).
// The proxies are a polar set in the canonical patch frame (centre + n_ring rings at r_k = h cos((k + 1/2) pi /
// (2 n_ring)), round(c_phi r_k / h) >= 6 angles, odd rings rotated by half a step), mapped to the unit sphere as
// (u, v, sqrt(1 - u^2 - v^2)) -- the nodes' own embedding (zhat).  kappa is calibrated here, for the actual nodes,
// against point sources on the sphere (the two terms of the Green's function, 2/|x - s| and log|x - s|, eq:Gintonsurface
// PAPER.md:396-399): the smallest D / h from which the interpolation error of either term, relative to the Green's
// function's scale max 2/|x - s| over the nodes, stays below tol.
#include <math.h>
#include <stdint.h>

#include <algorithm>
#include <vector>

#include "nc_common.cuh"

namespace nc {

namespace {
typedef long double LD;

// Chebyshev-product basis of total degree <= deg at (u, v) (scaled by 1 / h): B = (deg + 1)(deg + 2) / 2 values
void cheb_basis(LD u, LD v, int deg, LD* out) {
  LD Tu[32], Tv[32];
  Tu[0] = Tv[0] = 1.0L;
  Tu[1] = u;
  Tv[1] = v;
  for (int k = 2; k <= deg; ++k) {
    Tu[k] = 2.0L * u * Tu[k - 1] - Tu[k - 2];
    Tv[k] = 2.0L * v * Tv[k - 1] - Tv[k - 2];
  }
  int c = 0;
  for (int a = 0; a <= deg; ++a)
    for (int b = 0; a + b <= deg; ++b) out[c++] = Tu[a] * Tv[b];
}
}  // namespace

// Builds the proxy rule for the Ks nodes zhat (canonical frame, unit vectors about (0, 0, 1)).  Returns the number
// of proxies n (0 on failure: degree too high for the point count, or a rank-deficient basis); pts: n x 3 unit vectors;
// Int: Ks x n (row-major); *kappa: calibrated min D / h for tol (HUGE_VAL if never met up to D / h = 64); *h_out: h.
int proxy_rule_build(const double* zhat, int Ks, int deg, int nring, double cphi, double tol, std::vector<double>& pts,
                     std::vector<double>& Int, double* kappa, double* h_out) {
  if (Ks <= 0 || deg < 1 || deg > 30 || nring < 1 || nring > 64) return 0;
  double h = 0.0;
  for (int k = 0; k < Ks; ++k) h = std::max(h, std::hypot(zhat[3 * k], zhat[3 * k + 1]));
  h *= 1.01;   // the outer ring reaches 0.96 h (n_ring = 6): every node inside the proxies' disk
  if (!(h > 0.0) || h >= 0.5) return 0;
  const LD PI = 3.14159265358979323846264338327950288L;
  std::vector<LD> pu, pv;
  pu.push_back(0.0L);
  pv.push_back(0.0L);
  for (int k = 0; k < nring; ++k) {
    const LD r = cosl(PI * (k + 0.5L) / (2.0L * nring));
    const int na = std::max(6, (int)lrintl((LD)cphi * r));
    const LD off = (k & 1) ? 0.5L : 0.0L;
    for (int l = 0; l < na; ++l) {
      const LD ph = 2.0L * PI * (l + off) / na;
      pu.push_back((LD)h * r * cosl(ph));
      pv.push_back((LD)h * r * sinl(ph));
    }
  }
  const int n = (int)pu.size(), B = (deg + 1) * (deg + 2) / 2;
  if (n < B) return 0;
  // Householder QR of V (n x B), column-major in long double; W = R^-1 Q^T (B x n); Int = V_nodes W
  std::vector<LD> V((size_t)n * B), row(B);
  for (int i = 0; i < n; ++i) {
    cheb_basis(pu[i] / h, pv[i] / h, deg, row.data());
    for (int c = 0; c < B; ++c) V[(size_t)c * n + i] = row[c];
  }
  std::vector<LD> Qt((size_t)n * n, 0.0L);   // accumulates Q^T (n x n), row-major
  for (int i = 0; i < n; ++i) Qt[(size_t)i * n + i] = 1.0L;
  std::vector<LD> vh(n);
  for (int c = 0; c < B; ++c) {
    LD* col = &V[(size_t)c * n];
    LD nrm = 0.0L;
    for (int i = c; i < n; ++i) nrm += col[i] * col[i];
    nrm = sqrtl(nrm);
    if (!(nrm > 0.0L)) return 0;
    const LD alpha = col[c] > 0 ? -nrm : nrm;
    for (int i = 0; i < n; ++i) vh[i] = i < c ? 0.0L : col[i];
    vh[c] -= alpha;
    LD vn = 0.0L;
    for (int i = c; i < n; ++i) vn += vh[i] * vh[i];
    if (!(vn > 0.0L)) return 0;
    for (int cc = c; cc < B; ++cc) {   // H = I - 2 v v^T / (v^T v) applied to the remaining columns
      LD* cl = &V[(size_t)cc * n];
      LD d = 0.0L;
      for (int i = c; i < n; ++i) d += vh[i] * cl[i];
      d = 2.0L * d / vn;
      for (int i = c; i < n; ++i) cl[i] -= d * vh[i];
    }
    for (int j = 0; j < n; ++j) {      // Q^T <- H Q^T (columns of Q^T)
      LD d = 0.0L;
      for (int i = c; i < n; ++i) d += vh[i] * Qt[(size_t)i * n + j];
      d = 2.0L * d / vn;
      for (int i = c; i < n; ++i) Qt[(size_t)i * n + j] -= d * vh[i];
    }
  }
  // rank check: |R_cc| against |R_00|
  for (int c = 0; c < B; ++c)
    if (!(fabsl(V[(size_t)c * n + c]) > 1e-12L * fabsl(V[0]))) return 0;
  std::vector<LD> W((size_t)B * n);          // W = R^-1 (Q^T)[0:B, :]
  for (int j = 0; j < n; ++j)
    for (int c = B - 1; c >= 0; --c) {
      LD sacc = Qt[(size_t)c * n + j];
      for (int cc = c + 1; cc < B; ++cc) sacc -= V[(size_t)cc * n + c] * W[(size_t)cc * n + j];
      W[(size_t)c * n + j] = sacc / V[(size_t)c * n + c];
    }
  Int.assign((size_t)Ks * n, 0.0);
  for (int k = 0; k < Ks; ++k) {
    cheb_basis((LD)zhat[3 * k] / h, (LD)zhat[3 * k + 1] / h, deg, row.data());
    for (int j = 0; j < n; ++j) {
      LD sacc = 0.0L;
      for (int c = 0; c < B; ++c) sacc += row[c] * W[(size_t)c * n + j];
      Int[(size_t)k * n + j] = (double)sacc;
    }
  }
  pts.assign((size_t)3 * n, 0.0);
  for (int i = 0; i < n; ++i) {
    pts[3 * i] = (double)pu[i];
    pts[3 * i + 1] = (double)pv[i];
    pts[3 * i + 2] = (double)sqrtl(1.0L - pu[i] * pu[i] - pv[i] * pv[i]);
  }
  // calibration: point sources on the unit sphere at geodesic distance D h from the patch centre, 16 directions;
  // error = max over nodes |Int f(proxies) - f(nodes)| / max |f(nodes)| for f = 2/|x - s| and log|x - s|
  std::vector<LD> xn((size_t)3 * Ks), xp((size_t)3 * n);
  for (int k = 0; k < Ks; ++k) {
    xn[3 * k] = zhat[3 * k];
    xn[3 * k + 1] = zhat[3 * k + 1];
    xn[3 * k + 2] = sqrtl(1.0L - xn[3 * k] * xn[3 * k] - xn[3 * k + 1] * xn[3 * k + 1]);
  }
  for (int i = 0; i < 3 * n; ++i) xp[i] = pts[i];
  std::vector<LD> fp(n), fn(Ks);
  auto err_at = [&](double D) {
    LD worst = 0.0L;
    const LD th = (LD)D * h;
    if (th >= PI) return (LD)0.0L;
    for (int a = 0; a < 16; ++a) {
      const LD ph = 2.0L * PI * a / 16.0L;
      const LD s[3] = {sinl(th) * cosl(ph), sinl(th) * sinl(ph), cosl(th)};
      for (int f = 0; f < 2; ++f) {
        auto F = [&](const LD* x) {
          const LD dx = x[0] - s[0], dy = x[1] - s[1], dz = x[2] - s[2];
          const LD d = sqrtl(dx * dx + dy * dy + dz * dz);
          return f == 0 ? 2.0L / d : logl(d);
        };
        for (int i = 0; i < n; ++i) fp[i] = F(&xp[3 * i]);
        LD fmax = 0.0L, emax = 0.0L;   // both terms' errors against the Green's function's scale, max 2/d
        for (int k = 0; k < Ks; ++k) {
          fn[k] = F(&xn[3 * k]);
          LD v = 0.0L;
          for (int j = 0; j < n; ++j) v += (LD)Int[(size_t)k * n + j] * fp[j];
          const LD dx = xn[3 * k] - s[0], dy = xn[3 * k + 1] - s[1], dz = xn[3 * k + 2] - s[2];
          fmax = std::max(fmax, 2.0L / sqrtl(dx * dx + dy * dy + dz * dz));
          emax = std::max(emax, fabsl(v - fn[k]));
        }
        worst = std::max(worst, emax / fmax);
      }
    }
    return worst;
  };
  *kappa = HUGE_VAL;
  *h_out = h;
  // the error falls monotonically with D: bisection on a 1/8 grid of D / h in [1.5, 64]
  if (err_at(64.0) > (LD)tol) return n;   // never met: *kappa stays HUGE_VAL
  int lo = 12, hi = 512;                  // D = k / 8: err(hi / 8) <= tol
  if (err_at(lo / 8.0) <= (LD)tol) hi = lo;
  while (hi - lo > 1) {
    const int mid = (lo + hi) / 2;
    if (err_at(mid / 8.0) <= (LD)tol) hi = mid; else lo = mid;
  }
  *kappa = hi / 8.0;
  return n;
}

}  // namespace nc

// C ABI (include/nc.h): the proxy rule alone, for tests and diagnostics (host arithmetic, no device needed)
extern "C" int nc_proxy_rule(const double* zhat, int Kstar, int deg, int nring, double cphi, double tol, int nmax,
                             double* pts, double* Int, double* kappa, double* h) {
  if (!zhat || Kstar <= 0 || !kappa || !h) return nc::fail(NC_EINVAL, "nc_proxy_rule: bad arguments");
  std::vector<double> P, I;
  const int n = nc::proxy_rule_build(zhat, Kstar, deg, nring, cphi, tol, P, I, kappa, h);
  if (n <= 0) return nc::fail(NC_EINVAL, "nc_proxy_rule: no rule for these parameters");
  if (n > nmax) return nc::fail(NC_EINVAL, "nc_proxy_rule: nmax too small");
  if (pts) std::copy(P.begin(), P.end(), pts);
  if (Int) std::copy(I.begin(), I.end(), Int);
  return n;
}
