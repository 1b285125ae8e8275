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
