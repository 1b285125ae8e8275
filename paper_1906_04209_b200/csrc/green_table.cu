// green_table.cu -- the fp64 log table of green.cuh (c_j = 1/(1 + (j + 1/2)/1024), -log c_j), built on the host
// in long double so every entry is correctly rounded, uploaded once per device.
#include <math.h>

#include <map>
#include <mutex>

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

}  // namespace nc
