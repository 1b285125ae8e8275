// green.cuh -- device evaluation of the on-surface Neumann Green's functions (the pair kernel of every
// hot loop: direct sums, interaction-list and neighbour evaluations).
//
// Paper forms (three terms, d = |x - x'|):
//   G_E = 2/d - log(2/d) - log(1 + d/2)      eq:Gextonsurface
//   G_I = 2/d + log(2/d) - log(1 + d/2)      eq:Gintonsurface
// Exact single-log rewrites used on the GPU: with w = 2/d and q = d^2/4,
//   G_E = w - log(1 + w)                     since w (1 + d/2) = w + 1
//   G_I = w - log(q (1 + w))                 since (2/d)/(1 + d/2) = 4/(d^2 + 2d) = 1/(q (1 + w)); q (1 + w) = fma(q, w, q)
// Coordinates are stored pre-scaled by 1/2 (exact), so the squared distance of the scaled points IS q and
// rsqrt(q) IS w: one reciprocal square root and one logarithm per pair, no division.
//
// fp64 rsqrt: MUFU.RSQ64H seed (rsqrt.approx.f64) + one third-order Newton correction
//   e = 1 - q y^2,  y <- y + y e (1/2 + 3/8 e)                           (relative error ~ 2^-53)
// fp64 log: x = 2^k m, m in [1,2); j = top 10 mantissa bits; c_j = 1/(1 + (j + 1/2)/1024) (table, smem);
//   r = m c_j - 1 = x (c_j 2^-k) - 1 (one FMA, |r| <= 2^-11);  log x = k ln2 - log c_j + log1p(r),
//   log1p(r) = r + r^2 (-1/2 + r/3 - r^2/4)   (truncation |r|^5/5 < 6e-18)
// 22 FP64-pipe instructions per pair (both kinds) instead of ~45 with libdevice log + rsqrt.
#pragma once

#include <stdint.h>

namespace nc {

constexpr int kLogTableBits = 10;
constexpr int kLogTableSize = 1 << kLogTableBits;
constexpr double kLn2 = 0.69314718055994530941723212145817657;

// (c_j, -log c_j) table: computed once on the host in long double (green_table.cu) and kept in global memory;
// every CTA copies it to shared memory.  Call with all threads of the CTA, then __syncthreads().
const double2* log_table_device();   // host: uploaded once per device; nullptr on failure

__device__ __forceinline__ void init_log_table(double2* tbl, const double2* __restrict__ src) {
  for (int j = threadIdx.x; j < kLogTableSize; j += blockDim.x) tbl[j] = src[j];
}

__device__ __forceinline__ double rsqrt_approx(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  return y;
}

// fp64 reciprocal square root, x in the normal range
__device__ __forceinline__ double fast_rsqrt(double x) {
  double y = rsqrt_approx(x);
  double t = x * y;
  double e = fma(-t, y, 1.0);
  double c = fma(0.375, e, 0.5);
  double ye = y * e;
  return fma(ye, c, y);
}

// fp64 natural log for positive normal x (absolute error ~1e-16 |log x| + 1e-17).  The table's c_j is rescaled by
// 2^-k with an integer subtract on its exponent field (x c_j 2^-k = m c_j exactly), so the mantissa m is never
// formed: r = fma(x, c_j 2^-k, -1) equals fma(m, c_j, -1) bit for bit.
__device__ __forceinline__ double fast_log(double x, const double2* __restrict__ tbl) {
  const int hi = __double2hiint(x);
  const int j = (hi >> (20 - kLogTableBits)) & (kLogTableSize - 1);
  // exponent k as a double without a conversion instruction: 2^52 + 2^31 + k  minus the magic
  const double kd = __hiloint2double(0x43300000, (int)(((unsigned)hi >> 20) - 1023u + 0x80000000u)) -
                    4503601774854144.0;   // 2^52 + 2^31
  const double2 t = tbl[j];
  const double c = __hiloint2double(__double2hiint(t.x) - (hi & 0x7FF00000) + 0x3FF00000, __double2loint(t.x));
  const double r = fma(x, c, -1.0);
  double p = fma(r, -0.25, 0.33333333333333333333);
  p = fma(p, r, -0.5);
  const double r2 = r * r;
  const double l1 = fma(r2, p, r);
  const double h = fma(kd, kLn2, t.y);
  return h + l1;
}

template <class Tab>
__device__ __forceinline__ void init_table(Tab* tbl, const Tab* __restrict__ src) {
  for (int j = threadIdx.x; j < kLogTableSize; j += blockDim.x) tbl[j] = src[j];
}

// G for scaled coordinates: q = |x - x'|^2 / 4  (KIND 1 = exterior G_E, KIND 0 = interior G_I)
template <int KIND, class Tab>
__device__ __forceinline__ double green_q(double q, const Tab* __restrict__ tbl) {
  const double w = fast_rsqrt(q);   // 2/d
  if (KIND == 1) return w - fast_log(1.0 + w, tbl);
  return w - fast_log(fma(q, w, q), tbl);   // q (1 + w), one rounding
}

// Far-field G (k_pairs_grid FAR variant, hierarchical mode only; R23), from qh = |x - x'|^2 / 8 (half the
// scaled squared distance, formed by the caller as a dot product).  Trimmed for the issue rate (an FP64 instruction
// holds the warp scheduler two cycles, any other one cycle):
//   w  = 2/d = rsqrt(2 qh): MUFU.RSQ64H seed of 2 qh (exponent + 1 on the integer pipe), one Newton step
//        w = y + y (1/2 - qh y^2)                                      [3 FP64; relative error ~(3/2) e0^2]
//   log: r = x c_j 2^-k - 1 with the table's c_j rescaled by an integer exponent subtract (no mantissa extraction),
//        log1p(r) = r + r^2 (-1/2 + r/3)  (|r| <= 2^-11: truncation r^4/4 < 1.5e-14 absolute)
//   interior: log(q (1 + w)) = log(qh (1 + w)) + ln 2, the ln 2 folded into the exponent's magic constant.
// 16 FP64 instructions (both kinds: the interior argument qh (1 + w) is one FMA), ~13 others.
template <int KIND>
__device__ __forceinline__ double green_far_h(double qh, const double2* __restrict__ tbl) {
  const double y = rsqrt_approx(__hiloint2double(__double2hiint(qh) + 0x00100000, __double2loint(qh)));
  const double t = qh * y;
  const double e = fma(-t, y, 0.5);
  const double w = fma(y, e, y);
  const double x = (KIND == 1) ? 1.0 + w : fma(qh, w, qh);   // 1 + w  |  qh (1 + w)
  const int hi = __double2hiint(x);
  const int j = (hi >> (20 - kLogTableBits)) & (kLogTableSize - 1);
  const double2 tj = tbl[j];
  // c_j 2^-k: subtract the unbiased exponent of x from c_j's exponent field (exact; no range issue for 2^-30..2^30)
  const double c = __hiloint2double(__double2hiint(tj.x) - (hi & 0x7FF00000) + 0x3FF00000, __double2loint(tj.x));
  const double r = fma(x, c, -1.0);
  const double p = fma(r, 0.33333333333333333333, -0.5);
  const double r2 = r * r;
  const double l1 = fma(r2, p, r);
  // k (+1 interior) as a double: 2^52 + 2^31 + e - 1023 minus the magic (minus one more for the interior ln 2)
  const double kd = __hiloint2double(0x43300000, (int)(((unsigned)hi >> 20) - 1023u + 0x80000000u)) -
                    (KIND == 1 ? 4503601774854144.0 : 4503601774854143.0);
  const double h = fma(kd, kLn2, tj.y);
  return w - (h + l1);
}

// Far-field G with an exponent-indexed log table (k_pairs_grid FAR >= 2, hierarchical mode only; R25).
// The table is indexed by the top 11 + FB bits of x (biased exponent and FB mantissa bits: one shift), and its
// entry (c, L) already carries the exponent: c = 1 / (2^e (1 + (j + 1/2) / 2^FB)), L = -log c (+ ln 2 interior, so
// that L + log1p(r) = log(2 x) = log(q (1 + w))).  Then log x = L + log1p(r) with r = x c - 1, |r| <= 2^-(FB+1),
// and log1p(r) = r (1 + r (a2 + r a3 [+ r^2 a4])) with minimax coefficients for |r| <= 1 / (2^(FB+1) + 1)
// (absolute error 9.9e-12 for FB = 7 cubic, 6.3e-14 FB = 7 quartic, 6.2e-13 FB = 8 cubic; fitted by
// tools/fit_log1p.py).  G = (w - L) - r p(r): no exponent extraction, no k ln 2 term.
// 13 FP64 instructions per pair with the caller's dot product and accumulate (cubic), 14 quartic.
// The table covers the x range of grid pairs (d >= eps / 4, far_table_build); the index is clamped on the open side.
template <int FB, int DEG>
struct FarPoly;
template <>
struct FarPoly<7, 3> {
  static constexpr double a2 = -0.50000313945533437, a3 = 0.33333636142100315, a4 = 0.0;
};
template <>
struct FarPoly<7, 4> {
  static constexpr double a2 = -0.49999999200264428, a3 = 0.33333636142100315, a4 = -0.25053074075115417;
};
template <>
struct FarPoly<6, 4> {
  static constexpr double a2 = -0.49999999926820904, a3 = 0.33334535235773449, a4 = -0.25002219360866496;
};
template <>
struct FarPoly<8, 3> {
  static constexpr double a2 = -0.50000078809143556, a3 = 0.33333409330333852, a4 = 0.0;
};

// tbase: shared-memory byte address of the table minus base * 16 (so that tbase + (hi(x) >> (20 - FB)) * 16 is the
// entry; one IMAD); lim: the index clamp (largest valid index exterior, smallest interior).  a2r (and a3r, quartic)
// are the polynomial constants held in registers by the caller (an FP64 FMA takes at most one immediate / uniform
// operand, and the compiler would otherwise rematerialise the second constant in the loop with two moves per pair).
template <int KIND, int FB, int DEG>
__device__ __forceinline__ double green_far_t(double qh, unsigned tbase, int lim, double a2r, double a3r) {
  const double y = rsqrt_approx(__hiloint2double(__double2hiint(qh) + 0x00100000, __double2loint(qh)));
  const double t = qh * y;
  const double e = fma(-t, y, 0.5);
  const double w = fma(y, e, y);
  const double x = (KIND == 1) ? 1.0 + w : fma(qh, w, qh);   // 1 + w  |  qh (1 + w) = q (1 + w) / 2
  int ix = __double2hiint(x) >> (20 - FB);
  ix = (KIND == 1) ? min(ix, lim) : max(ix, lim);
  double cj, lj;
  asm("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(cj), "=d"(lj) : "r"(tbase + ((unsigned)ix << 4)));
  const double r = fma(x, cj, -1.0);
  double p;
  if (DEG == 4) {
    p = fma(r, FarPoly<FB, DEG>::a4, a3r);
    p = fma(r, p, a2r);
  } else {
    p = fma(r, FarPoly<FB, DEG>::a3, a2r);
  }
  p = fma(r, p, 1.0);
  return fma(-r, p, w - lj);
}

// Far-field G, reciprocal-seeded variant (k_pairs_grid FAR 5, 6; R25).  Same reduction as green_far_t,
// but c = rcp.approx(x_mid) comes from the SFU (x_mid: x's high word with the mantissa below the top FB bits set to
// the bin midpoint) and only L = -log c (+ ln 2 interior) is read from shared memory: an 8-byte load instead of a
// 16-byte one.  The pair kernels are bound by shared-memory wavefronts (a warp's 32 random table reads conflict in
// the banks), so halving the entry halves the dominant traffic.  c is a deterministic function of x_mid's high word:
// far_table_build_rcp evaluates the same instruction on the device for every bin and tabulates L = -log c exactly.
__device__ __forceinline__ double rcp_approx(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  return y;
}
// fp32 SFU seeds (R31, measured and NOT used by the kernels: tools/pair_mix_bench.cu only).  The idea: an
// fp64 MUFU (RSQ64H, RCP64H) costs ~2.3 cycles of a saturated FP64 pipe (profiles/r01m_sfu_fp64_overlap.txt) while
// the fp32 MUFU overlaps the DFMA stream, so take the seeds from the fp32 unit with the format conversions on the
// integer pipe (a double in the fp32 normal range -> the fp32 of its top 23 mantissa bits: one funnel shift and one
// add, exponent rebias 1023 -> 127 modulo 2^9; fp32 -> the equal double: a shift-add and a shift).  Accurate
// (C3/C4 hierarchical error unchanged to 1e-16, profiles/r01w_s32.txt) but slower: the grid kernel is issue-bound
// and the ~3 extra integer instructions per pair cost more than the fp64 MUFU contention saved (66.3 -> 72.7 ms).
__device__ __forceinline__ double f32bits_to_double(unsigned u) {
  return __hiloint2double((int)((u >> 3) + 0x38000000u), (int)(u << 29));
}
__device__ __forceinline__ double rsqrt_seed32(double qh) {   // ~ rsqrt(2 qh), relative error < 2^-22
  const unsigned f = __funnelshift_l((unsigned)__double2loint(qh), (unsigned)__double2hiint(qh), 3) + 0x40800000u;
  float y;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(__uint_as_float(f)));
  return f32bits_to_double(__float_as_uint(y));
}
__device__ __forceinline__ double rcp_mid32(int h) {   // rcp.approx.f32 of the double (h, 0) (a bin midpoint)
  float c;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(c) : "f"(__uint_as_float(((unsigned)h << 3) + 0x40000000u)));
  return f32bits_to_double(__float_as_uint(c));
}

// kmid = 1 << (19 - FB), passed in at run time: the midpoint is then one LOP3 (x & ~mask) | kmid with kmid in a
// register, not two with two immediates.  S32 (R31, microbenchmark only): bit 0 the fp32 rsqrt seed, bit 1 the fp32
// midpoint reciprocal.
template <int KIND, int FB, int DEG, int S32 = 0>
__device__ __forceinline__ double green_far_r(double qh, unsigned tbase, int lim, double a2r, double a3r, int kmid) {
  const double y = (S32 & 1) ? rsqrt_seed32(qh)
                             : rsqrt_approx(__hiloint2double(__double2hiint(qh) + 0x00100000, __double2loint(qh)));
  const double t = qh * y;
  const double e = fma(-t, y, 0.5);
  const double w = fma(y, e, y);
  const double x = (KIND == 1) ? 1.0 + w : fma(qh, w, qh);
  const int hx = __double2hiint(x);
  const int hmid = (hx & ~((1 << (20 - FB)) - 1)) | kmid;
  const double c = (S32 & 2) ? rcp_mid32(hmid) : rcp_approx(__hiloint2double(hmid, 0));
  int ix = hx >> (20 - FB);
  ix = (KIND == 1) ? min(ix, lim) : max(ix, lim);
  double lj;
  asm("ld.shared.f64 %0, [%1];" : "=d"(lj) : "r"(tbase + ((unsigned)ix << 3)));
  const double r = fma(x, c, -1.0);
  double p;
  if (DEG == 4) {
    p = fma(r, FarPoly<FB, DEG>::a4, a3r);
    p = fma(r, p, a2r);
  } else {
    p = fma(r, FarPoly<FB, DEG>::a3, a2r);
  }
  p = fma(r, p, 1.0);
  return fma(-r, p, w - lj);
}

// Exact-form G with the reciprocal-seeded table (direct sums, near lists; R25): q = |z - s|^2 / 4 from
// coordinate differences (caller), w = 2/d by fast_rsqrt (third-order Newton), x = 1 + w (exterior) or q (1 + w)
// (interior, no ln 2: the table's L = -log c for this form), log x = L + log1p(r) with c = rcp.approx(bin midpoint),
// r = x c - 1 and the quartic minimax log1p of FB = 7 (absolute error 6.3e-14): 20 FP64 instructions per pair with
// the caller's distance and accumulate, and an 8-byte table read instead of the 16-byte (c_j, -log c_j) one.
template <int KIND>
__device__ __forceinline__ double green_exact_r(double q, unsigned tbase, int lim, double a2r, double a3r, int kmid) {
  const double w = fast_rsqrt(q);
  const double x = (KIND == 1) ? 1.0 + w : fma(q, w, q);
  const int hx = __double2hiint(x);
  const double c = rcp_approx(__hiloint2double((hx & ~((1 << 13) - 1)) | kmid, 0));   // kmid = 1 << 12 (run time)
  int ix = hx >> 13;
  ix = (KIND == 1) ? min(ix, lim) : max(ix, lim);
  double lj;
  asm("ld.shared.f64 %0, [%1];" : "=d"(lj) : "r"(tbase + ((unsigned)ix << 3)));
  const double r = fma(x, c, -1.0);
  double p = fma(r, FarPoly<7, 4>::a4, a3r);
  p = fma(r, p, a2r);
  p = fma(r, p, 1.0);
  return fma(-r, p, w - lj);
}

// Direct-sum pairs between well-separated patches (k_pairs_direct with FARD, R30): q from the dot product
// (qh = q/2 = (|X|^2 + 1/4)/2 - X.S for scaled coordinates, 3 DFMA) and w = 2/d by one Newton step from the SFU seed,
// then the exact-form table log (quartic).  Used only when the source patch is >= 0.12 + 2 eps away from every
// target of the warp, where the dot product's absolute rounding (~3e-16) is <= 2e-13 relative to q: 15 FP64
// instructions (interior; 14 exterior) instead of 19.
template <int KIND>
__device__ __forceinline__ double green_exact_far(double qh, unsigned tbase, int lim, double a2r, double a3r, int kmid) {
  const double y = rsqrt_approx(__hiloint2double(__double2hiint(qh) + 0x00100000, __double2loint(qh)));
  const double t = qh * y;
  const double e = fma(-t, y, 0.5);
  const double w = fma(y, e, y);
  double x;
  if (KIND == 1) {
    x = 1.0 + w;
  } else {
    const double xh = fma(qh, w, qh);   // q (1 + w) / 2
    x = xh + xh;                        // exact doubling
  }
  const int hx = __double2hiint(x);
  const double c = rcp_approx(__hiloint2double((hx & ~((1 << 13) - 1)) | kmid, 0));
  int ix = hx >> 13;
  ix = (KIND == 1) ? min(ix, lim) : max(ix, lim);
  double lj;
  asm("ld.shared.f64 %0, [%1];" : "=d"(lj) : "r"(tbase + ((unsigned)ix << 3)));
  const double r = fma(x, c, -1.0);
  double p = fma(r, FarPoly<7, 4>::a4, a3r);
  p = fma(r, p, a2r);
  p = fma(r, p, 1.0);
  return fma(-r, p, w - lj);
}

// the exact-form table as the kernels hold it: shared-memory base address (minus base * 8), clamp, constants
struct ExactTab {
  unsigned tb;
  int lim;
  double a2, a3;
  int kmid;   // the bin-midpoint bit 1 << 12, a run-time value (one LOP3 per pair, see green_far_r)
};
// Call with all threads of the CTA (then __syncthreads()): copies the n L entries (n / 2 double2) into smem and
// returns the kernel-side handle.  src[n / 2] holds (a2, a3).
__device__ __forceinline__ ExactTab init_exact_table(int kind, double2* smem, const double2* __restrict__ src, int n,
                                                     int base, int kmid) {
  for (int j = threadIdx.x; j < n / 2; j += blockDim.x) smem[j] = src[j];
  const double2 cst = __ldg(src + n / 2);
  ExactTab t;
  t.tb = (unsigned)__cvta_generic_to_shared(smem) - 8u * (unsigned)base;
  t.lim = kind == 1 ? base + n - 1 : base;
  t.a2 = cst.x;
  t.a3 = cst.y;
  t.kmid = kmid;
  return t;
}

// reference-accuracy variant (libdevice), used by the self-check path
template <int KIND>
__device__ __forceinline__ double green_q_libdevice(double q) {
  const double w = rsqrt(q);
  const double a = 1.0 + w;
  if (KIND == 1) return w - log(a);
  return w - log(q * a);
}

}  // namespace nc
