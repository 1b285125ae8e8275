/*
 * oracle_field.c -- TEST INFRASTRUCTURE ONLY (the CPU oracle of SURVEY.md §8(c)).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
 * load this library.  It shares no code, header or table with the CUDA path
 * (paper_1906_04209_b200/csrc): it is a plain, slow, obviously-correct restatement of the paper.
 *
 * What it computes (the multiple-scattering field at target nodes):
 *
 *     u_t = sum over sources s with patch(s) != patch(t) of  G(x_t, y_s) * rho_s
 *
 * i.e. the sums  sum_{j != i} S_ij B fhat_j  of eq:mssums (§6) with each source
 * patch replaced by its skeletonised outgoing representation eq:outgoingcompressed
 * (§7): sum_l G(x, x^f_{j,l}) (sigma_j)_l w_l  ~=  sum_m G(x, x^f_{j,pi(m)}) rho_{j,m}.
 *
 * G is the on-surface Neumann Green's function in the paper's literal three-term form:
 *   interior (narrow escape, kind 0), eq:Gintonsurface:
 *       G_I = 2/|x-x'| + log(2/|x-x'|) - log(1 + |x-x'|/2)
 *   exterior (narrow capture, kind 1), eq:Gextonsurface:
 *       G_E = 2/|x-x'| - log(2/|x-x'|) - log(1 + |x-x'|/2)
 * with |x-x'| computed from coordinate differences.  Sums are Neumaier-compensated (R16).
 *
 * Parity pins: tests/test_oracle.py (sphere means of G_I = 2; G_E mean = 1;
 * G(d=2) = 1 - log 2; N=1 identity; dense-LU GMRES cross-check).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

double oracle_green(int kind, const double* x, const double* y) {
  double dx = x[0] - y[0], dy = x[1] - y[1], dz = x[2] - y[2];
  double d = sqrt(dx * dx + dy * dy + dz * dz);
  double first = 2.0 / d;
  double second = log(2.0 / d);
  double third = log(1.0 + 0.5 * d);
  if (kind == 0) return first + second - third; /* G_I, eq:Gintonsurface */
  return first - second - third;                /* G_E, eq:Gextonsurface */
}

/* Neumaier (improved Kahan) summation step */
static inline void neumaier_add(double* sum, double* comp, double v) {
  double t = *sum + v;
  if (fabs(*sum) >= fabs(v)) *comp += (*sum - t) + v;
  else *comp += (v - t) + *sum;
  *sum = t;
}

/*
 * targets: nt points (nt x 3, row-major) with owning patch ids tpatch[nt]
 * sources: ns points (ns x 3) with owning patch ids spatch[ns] and strengths rho[ns]
 * out:     u[nt]
 */
void oracle_field(int kind, int64_t nt, const double* tx, const int64_t* tpatch, int64_t ns,
                  const double* sx, const int64_t* spatch, const double* rho, double* u) {
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t t = 0; t < nt; ++t) {
    double sum = 0.0, comp = 0.0;
    for (int64_t s = 0; s < ns; ++s) {
      if (spatch[s] == tpatch[t]) continue; /* j != i in eq:mssums */
      neumaier_add(&sum, &comp, oracle_green(kind, tx + 3 * t, sx + 3 * s) * rho[s]);
    }
    u[t] = sum + comp;
  }
}

/*
 * Off-surface Neumann Green's functions (x anywhere, x' on the unit sphere), the paper's literal forms:
 *   interior, eq:Gintoffsurface:  G_I = 2/|x-x'| + log( 2 / (1 - x.x' + |x-x'|) )
 *   exterior, eq:Gextoffsurface:  G_E = 2/|x-x'| + log( (|x| - x.x') / (1 - x.x' + |x-x'|) )
 */
/* Evaluated literally, in long double (x87 80-bit): for an exterior point nearly on the ray through x', both
 * |x| - x.x' and 1 - x.x' + |x-x'| cancel catastrophically (each ~ |x| theta^2 / 2 for the angle theta between x
 * and x'); the 11 extra mantissa bits keep the literal form accurate to ~1e-15 relative at the angles a test
 * layout produces (theta >~ 1e-3), so the oracle needs no algebraic rewriting. */
double oracle_green_off(int kind, const double* x, const double* yin) {
  /* the formulas hold for x' on the sphere: the node (a unit vector only to ~4e-16 in fp64) is projected onto it
   * in long double first; without that, |x'| - 1 = delta enters the literal ratio as ~delta / theta^2 */
  long double yn = sqrtl((long double)yin[0] * yin[0] + (long double)yin[1] * yin[1] + (long double)yin[2] * yin[2]);
  long double y[3] = {yin[0] / yn, yin[1] / yn, yin[2] / yn};
  long double dx = (long double)x[0] - y[0], dy = (long double)x[1] - y[1], dz = (long double)x[2] - y[2];
  long double d = sqrtl(dx * dx + dy * dy + dz * dz);
  long double xy = (long double)x[0] * y[0] + (long double)x[1] * y[1] + (long double)x[2] * y[2];
  if (kind == 0) return (double)(2.0L / d + logl(2.0L / (1.0L - xy + d)));
  long double nx = sqrtl((long double)x[0] * x[0] + (long double)x[1] * x[1] + (long double)x[2] * x[2]);
  return (double)(2.0L / d + logl((nx - xy) / (1.0L - xy + d)));
}

/*
 * The single-layer potential of the compressed densities at off-surface points (NEXT-3, SURVEY.md §8(f);
 * eq:intBVPansatz PAPER.md:556-558 for the interior v, eq:urep PAPER.md:466-468 for the exterior u):
 *     out_t = sum_s G_off(p_t, y_s) rho_s ,      dmin_t = min_s |p_t - y_s|
 * over ALL sources (a target belongs to no patch).  Neumaier-compensated.
 */
void oracle_offsurface(int kind, int64_t nt, const double* px, int64_t ns, const double* sx, const double* rho,
                       double* out, double* dmin, double* absum) {
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t t = 0; t < nt; ++t) {
    double sum = 0.0, comp = 0.0, dm = INFINITY, as = 0.0;
    for (int64_t s = 0; s < ns; ++s) {
      const double* y = sx + 3 * s;
      double dx = px[3 * t] - y[0], dy = px[3 * t + 1] - y[1], dz = px[3 * t + 2] - y[2];
      double d = sqrt(dx * dx + dy * dy + dz * dz);
      if (d < dm) dm = d;
      double term = oracle_green_off(kind, px + 3 * t, y) * rho[s];
      neumaier_add(&sum, &comp, term);
      as += fabs(term);
    }
    out[t] = sum + comp;
    dmin[t] = dm;
    absum[t] = as; /* sum of |terms|: the scale of the sum's conditioning (parity bound for mixed-sign charges) */
  }
}

void oracle_green_off_batch(int kind, int64_t n, const double* x, const double* y, double* g) {
  for (int64_t i = 0; i < n; ++i) g[i] = oracle_green_off(kind, x + 3 * i, y + 3 * i);
}

/* Batched Green's function values (for the kernel pins in tests/test_oracle.py). */
void oracle_green_batch(int kind, int64_t n, const double* x, const double* y, double* g) {
  for (int64_t i = 0; i < n; ++i) g[i] = oracle_green(kind, x + 3 * i, y + 3 * i);
}

int oracle_num_threads(void) {
#ifdef _OPENMP
  extern int omp_get_max_threads(void);
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/*
 * Ring integrals of the near-surface potential (NEXT-3; eq:recoversig PAPER.md:797-807 for the
 * density, eq:Gintoffsurface / eq:Gextoffsurface for G): for each radius t[i] of a patch in its canonical frame
 * (centre +z, theta from +x),
 *     out[i] = (2 pi / ntheta) sum_k G_off(p, x'(t_i, theta_k)) sigma(t_i, theta_k),   theta_k = 2 pi k / ntheta,
 *     x'(t, theta) = (sin t cos theta, sin t sin theta, cos t),
 *     sigma(t_i, theta) = sum_{m < M1} AB[i][2m] cos(m theta) + AB[i][2m + 1] sin(m theta)
 * (the trapezoid rule: exact for the trigonometric polynomial sigma times the analytic periodic G up to the
 * aliasing error, which the caller drives down by doubling ntheta).  Neumaier-compensated.
 */
void oracle_rings(int kind, const double* p, int64_t nt, const double* t, int ntheta, int M1, const double* AB,
                  double* out, double* absum) {
  const double twopi = 6.283185307179586476925286766559;
  double* cs = (double*)malloc(sizeof(double) * 2 * (size_t)M1 * ntheta);
  for (int k = 0; k < ntheta; ++k)
    for (int m = 0; m < M1; ++m) {
      const double a = twopi * (double)(((int64_t)m * k) % ntheta) / ntheta;
      cs[(size_t)k * 2 * M1 + 2 * m] = cos(a);
      cs[(size_t)k * 2 * M1 + 2 * m + 1] = sin(a);
    }
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t i = 0; i < nt; ++i) {
    const double st = sin(t[i]), ct = cos(t[i]);
    double sum = 0.0, comp = 0.0, as = 0.0;
    for (int k = 0; k < ntheta; ++k) {
      const double* c = cs + (size_t)k * 2 * M1;
      double sig = 0.0;
      for (int m = 0; m < M1; ++m) sig += AB[i * 2 * M1 + 2 * m] * c[2 * m] + AB[i * 2 * M1 + 2 * m + 1] * c[2 * m + 1];
      const double y[3] = {st * c[2], st * c[3], ct};   /* c[2], c[3] = cos theta, sin theta (m = 1) */
      const double term = oracle_green_off(kind, p, y) * sig;
      neumaier_add(&sum, &comp, term);
      as += fabs(term);
    }
    out[i] = (sum + comp) * (twopi / ntheta);
    absum[i] = as * (twopi / ntheta);   /* the conditioning scale of the ring sum */
  }
  free(cs);
}
