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

// Far-field G with an exponent-indexed log table (k_pairs_grid, hierarchical mode only; R25, R32).
// The table is indexed by the top 11 + FB bits of x (biased exponent and FB mantissa bits: one shift); for a bin
// of midpoint x_mid it holds L = -log c with c = rcp.approx(x_mid) (+ ln 2 interior, so that L + log1p(r) =
// log(2 x) = log(q (1 + w))).  Then log x = L + log1p(r) with r = x c - 1, |r| <= 2^-(FB+1) (1 + 2^-20), and
// log1p(r) = r (1 + r (a2 + r a3)) with minimax coefficients (absolute error 9.9e-12 for FB = 7; FarPoly<7, 4>, the
// quartic, 6.3e-14, serves the exact form of the direct sums).  G = (w - L) - r p(r): no exponent extraction.
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

// Far-field G, reciprocal-seeded (k_pairs_grid FAR 5; R25): c = rcp.approx(x_mid) comes from the SFU
// (x_mid: x's high word with the mantissa below the top FB bits set to the bin midpoint) and only the 8-byte L is
// read from shared memory (a 16-byte (c, L) entry made the kernel shared-memory-wavefront bound: a warp's 32
// table reads conflict in the banks).  c is a deterministic function of x_mid's high word: far_table_build
// evaluates the same instruction on the device for every bin and tabulates L = -log c exactly.  The index is
// clamped on the open side of the table (FAR 7 / 8, green_far_n below, drop the clamp).
__device__ __forceinline__ double rcp_approx(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  return y;
}
// kmid = 1 << (19 - FB), passed in at run time: the midpoint is then one LOP3 (x & ~mask) | kmid with kmid in a
// register, not two with two immediates.  (R31 measured fp32 SFU seeds with integer format conversions instead:
// accurate, but slower in this issue-bound loop, 66.3 -> 72.7 ms at C5; not kept.)
template <int KIND, int FB, int DEG>
__device__ __forceinline__ double green_far_r(double qh, unsigned tbase, int lim, double a2r, double a3r, int kmid) {
  const double y = rsqrt_approx(__hiloint2double(__double2hiint(qh) + 0x00100000, __double2loint(qh)));
  const double t = qh * y;
  const double e = fma(-t, y, 0.5);
  const double w = fma(y, e, y);
  const double x = (KIND == 1) ? 1.0 + w : fma(qh, w, qh);
  const int hx = __double2hiint(x);
  const int hmid = (hx & ~((1 << (20 - FB)) - 1)) | kmid;
  const double c = rcp_approx(__hiloint2double(hmid, 0));
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

// Unclamped far form (k_pairs_grid_w FAR 7 / 8; R32).  As green_far_r, with two changes to the
// non-FP64 instructions of the pair: (1) no index clamp -- the far table covers every x a grid pair can produce
// (far_table_build: chord d >= eps/2, while a grid pair is at arc >= eps because a rung is valid only >= 2 eps from
// its source centre and the skeleton lies within eps of it, R22); (2) the entry is read as tab[ix] with tab a
// shared-memory pointer already offset by -base, so the compiler forms the address with a scaled-index load
// instead of a shift-multiply-add.  FB = 7, DEG = 3: the cubic of green_far_r (13 FP64).  FB = 9, DEG = 2: a
// quadratic r (c1 + c2 r) on the 4x finer bins |r| <= 2^-10 (minimax, absolute error 7.7e-11): 12 FP64.
template <int FB>
struct FarQuad;
template <>
struct FarQuad<9> {
  static constexpr double c1 = 1.0000002379505932, c2 = -0.5000002185734317;
};
template <int KIND, int FB, int DEG>
__device__ __forceinline__ double green_far_n(double qh, const double* __restrict__ tab, double a2r, double a3r,
                                              int kmid) {
  const double y = rsqrt_approx(__hiloint2double(__double2hiint(qh) + 0x00100000, __double2loint(qh)));
  const double t = qh * y;
  const double e = fma(-t, y, 0.5);
  const double w = fma(y, e, y);
  const double x = (KIND == 1) ? 1.0 + w : fma(qh, w, qh);
  const int hx = __double2hiint(x);
  const int hmid = (hx & ~((1 << (20 - FB)) - 1)) | kmid;
  const double c = rcp_approx(__hiloint2double(hmid, 0));
  const double lj = tab[hx >> (20 - FB)];
  const double r = fma(x, c, -1.0);
  double p;
  if constexpr (DEG == 2) {
    p = fma(r, a2r, a3r);   // a2r = c2, a3r = c1 (FarQuad)
  } else {
    p = fma(r, FarPoly<FB, 3>::a3, a2r);
    p = fma(r, p, 1.0);
  }
  return fma(-r, p, w - lj);
}

// SFU seeds whose low word is NOT zeroed (far forms 9 / 10, R35).  MUFU.RSQ64H / MUFU.RCP64H read and
// write only the high word of a double; rsqrt.approx / rcp.approx then zero the low word, one IMAD.MOV per seed
// (two of the 22.6 instructions of a grid pair).  Here the seed's low word is the input's high word h itself, which
// already sits in the even register of the pair: the double is (hi = MUFU(h), lo = h), a relative perturbation of
// the seed below 2^-20 * h / 2^32 <= 2^-22 (h < 2^30 for any x < 2^1024 with the sign clear, which every x here is).
// The rsqrt seed goes through one Newton step (error 1.5 delta^2: 2^-22.9 seed error + 2^-22 -> 3e-13 relative);
// the rcp seed c is tabulated exactly as computed (far_table_build evaluates the same two instructions), so
// L = -log c stays exact and only |r| grows by <= 2^-22 over the bin half-width.
__device__ __forceinline__ double rsqrt_seed_hl(int h) {
  double y;
  asm("{\n\t.reg .f64 s, t;\n\t.reg .b32 tl, th;\n\tmov.b64 s, {%1, %1};\n\trsqrt.approx.ftz.f64 t, s;\n\t"
      "mov.b64 {tl, th}, t;\n\tmov.b64 %0, {%1, th};\n\t}"
      : "=d"(y)
      : "r"(h));
  return y;
}
__device__ __forceinline__ double rcp_seed_hl(int h) {
  double y;
  asm("{\n\t.reg .f64 s, t;\n\t.reg .b32 tl, th;\n\tmov.b64 s, {%1, %1};\n\trcp.approx.ftz.f64 t, s;\n\t"
      "mov.b64 {tl, th}, t;\n\tmov.b64 %0, {%1, th};\n\t}"
      : "=d"(y)
      : "r"(h));
  return y;
}

// Far form with high-word seeds (k_pairs_grid_w FAR 9 / 10, R35): green_far_n's arithmetic (FB = 9
// quadratic or FB = 7 cubic) with (1) the two seeds of rsqrt_seed_hl / rcp_seed_hl and (2) the table entry's address
// taken from the midpoint word in one shift-add: hmid >> (17 - FB) = (hx >> (20 - FB)) * 8 + 4 (kmid = 1 << (19 - FB)
// contributes the 4), so tadr = (table byte address of index 0) - 4.  12 (quadratic) / 13 (cubic) FP64, 2 MUFU,
// 4 integer (exponent bump, midpoint LOP3, address LEA.HI, table LDS) per pair.
template <int KIND, int FB, int DEG>
__device__ __forceinline__ double green_far_hl(double qh, unsigned tadr, double a2r, double a3r, int kmid) {
  const double y = rsqrt_seed_hl(__double2hiint(qh) + 0x00100000);
  const double t = qh * y;
  const double e = fma(-t, y, 0.5);
  const double w = fma(y, e, y);
  const double x = (KIND == 1) ? 1.0 + w : fma(qh, w, qh);
  const int hmid = (__double2hiint(x) & ~((1 << (20 - FB)) - 1)) | kmid;
  const double c = rcp_seed_hl(hmid);
  double lj;
  asm("ld.shared.f64 %0, [%1];" : "=d"(lj) : "r"(tadr + ((unsigned)hmid >> (17 - FB))));
  const double r = fma(x, c, -1.0);
  double p;
  if constexpr (DEG == 2) {
    p = fma(r, a2r, a3r);   // a2r = c2, a3r = c1 (FarQuad)
  } else {
    p = fma(r, FarPoly<FB, 3>::a3, a2r);
    p = fma(r, p, 1.0);
  }
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

}  // namespace nc
