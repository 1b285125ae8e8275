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

__global__ void k_log8_c(double* c) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < kLogTableSize) c[j] = log8_c(j);
}

// -log c_j for the 8-byte table: c_j from the device's own instruction sequence (log8_c), the log on the host in
// long double (correctly rounded), uploaded once per device
const double* log8_table_device() {
  static std::mutex mu;
  static std::map<int, double*> tabs;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  std::lock_guard<std::mutex> lock(mu);
  auto it = tabs.find(dev);
  if (it != tabs.end()) return it->second;
  double host[kLogTableSize];
  double* d = nullptr;
  if (cudaMalloc(&d, sizeof(host)) != cudaSuccess) return nullptr;
  k_log8_c<<<(kLogTableSize + 255) / 256, 256>>>(d);
  if (cudaMemcpy(host, d, sizeof(host), cudaMemcpyDeviceToHost) != cudaSuccess) return nullptr;
  for (int j = 0; j < kLogTableSize; ++j) host[j] = (double)(-logl((long double)host[j]));
  if (cudaMemcpy(d, host, sizeof(host), cudaMemcpyHostToDevice) != cudaSuccess) return nullptr;
  tabs[dev] = d;
  return d;
}

}  // namespace nc
