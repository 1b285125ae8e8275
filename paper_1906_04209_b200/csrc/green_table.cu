// green_table.cu -- the fp64 log table of green.cuh (c_j = 1/(1 + (j + 1/2)/1024), -log c_j), built on the host
// in long double so every entry is correctly rounded, uploaded once per device.
#include <math.h>

#include <map>
#include <mutex>
#include <vector>

#include "green.cuh"
#include "nc_common.cuh"

namespace nc {

const double2* log_table_device() {
  static std::mutex mu;
  static std::map<int, double2*> tabs;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  std::lock_guard<std::mutex> lock(mu);
  auto it = tabs.find(dev);
  if (it != tabs.end()) return it->second;
  double2 host[kLogTableSize];
  for (int j = 0; j < kLogTableSize; ++j) {
    const double c = 1.0 / (1.0 + (j + 0.5) / (double)kLogTableSize);
    host[j] = make_double2(c, (double)(-logl((long double)c)));
  }
  double2* d = nullptr;
  if (cudaMalloc(&d, sizeof(host)) != cudaSuccess) return nullptr;
  if (cudaMemcpy(d, host, sizeof(host), cudaMemcpyHostToDevice) != cudaSuccess) return nullptr;
  tabs[dev] = d;
  return d;
}

// c of the reciprocal-seeded far form (green.cuh green_far_r), evaluated by the same instruction the pair kernel uses
// (hl = 1: c = rcp_seed_hl of the midpoint word, whose low word is that word -- green_far_hl, R35)
__global__ void k_far_rcp(int Elo, int bits, int cnt, int hl, double* c) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= cnt) return;
  const int per = 1 << bits;
  const int hx = ((Elo + t / per) << 20) | ((t % per) << (20 - bits));
  const int hmid = (hx & ~((1 << (20 - bits)) - 1)) | (1 << (19 - bits));
  c[t] = hl ? rcp_seed_hl(hmid) : rcp_approx(__hiloint2double(hmid, 0));
}

// far table (green.cuh green_far_t / green_far_r): entries for every biased exponent E that x takes on grid pairs.
// A grid pair is at chord distance d >= eps (the source's rung is valid from 2 eps of its centre, its skeleton lies
// within eps of it: DESIGN.md R22); the table covers d in [eps / 2, 2]: exterior x = 1 + 2/d in [2, 1 + 4/eps]
// (plus the exponent below 2, reachable by rounding of w ~ 1), interior x = d^2/8 + d/4 in [eps^2/32 + eps/8, 1];
// j = the top `bits` mantissa bits.  The kernel clamps the index on the open side (exterior above, interior below).
int far_table_build(int kind, double eps, int bits, int rcp, double a2, double a3, double2** d, int* n, int* base,
                    int exact) {
  // exact form (green_exact_r): interior x = q (1 + w) = d^2/4 + d/2 in [eps^2/16 + eps/4, 2], L without ln 2
  const double dlo = 0.5 * eps, sc = exact ? 2.0 : 1.0;
  const double xlo = kind == 1 ? 2.0 : sc * (dlo * dlo / 8.0 + dlo / 4.0);
  const double xhi = kind == 1 ? 1.0 + 2.0 / dlo : sc;
  int elo = 0, ehi = 0;
  frexp(xlo, &elo);   // x = f 2^e, f in [0.5, 1): biased exponent of x is e - 1 + 1023
  frexp(xhi, &ehi);
  const int Elo = elo - 1 + 1023 - (kind == 1 ? 1 : 0), Ehi = ehi - 1 + 1023;
  const int per = 1 << bits;
  const int cnt = (Ehi - Elo + 1) * per;
  std::vector<double> c((size_t)cnt);
  if (rcp) {   // c = rcp.approx(midpoint) as the device computes it
    double* dc = nullptr;
    if (cudaMalloc(&dc, c.size() * sizeof(double)) != cudaSuccess) return 1;
    k_far_rcp<<<(cnt + 255) / 256, 256>>>(Elo, bits, cnt, rcp == 2, dc);
    const bool ok = cudaMemcpy(c.data(), dc, c.size() * sizeof(double), cudaMemcpyDeviceToHost) == cudaSuccess;
    cudaFree(dc);
    if (!ok) return 1;
  } else {
    for (int t = 0; t < cnt; ++t)
      c[t] = (double)(1.0L / ldexpl(1.0L + ((t % per) + 0.5L) / per, Elo + t / per - 1023));
  }
  const int nvec = rcp ? cnt / 2 : cnt;
  std::vector<double2> host((size_t)nvec + 1);
  for (int t = 0; t < cnt; ++t) {
    long double L = -logl((long double)c[t]);
    if (kind == 0 && !exact) L += logl(2.0L);
    if (rcp)
      reinterpret_cast<double*>(host.data())[t] = (double)L;
    else
      host[t] = make_double2(c[t], (double)L);
  }
  host[(size_t)nvec] = make_double2(a2, a3);
  double2* p = nullptr;
  if (cudaMalloc(&p, host.size() * sizeof(double2)) != cudaSuccess) return 1;
  if (cudaMemcpy(p, host.data(), host.size() * sizeof(double2), cudaMemcpyHostToDevice) != cudaSuccess) {
    cudaFree(p);
    return 1;
  }
  *d = p;
  *n = cnt;
  *base = Elo * per;
  return 0;
}

}  // namespace nc
