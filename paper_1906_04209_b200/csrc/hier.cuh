// hier.cuh -- hierarchical (NC_HIER) mode entry points used by api.cu (implemented in hier.cu).
#pragma once
#include <vector>

#include "nc_common.cuh"

namespace nc {
int hier_order(nc_handle* h, std::vector<double>& centers);   // tree order; fills h->perm, permutes centers
int hier_setup(nc_handle* h, const std::vector<double>& centers_internal, cudaStream_t s);  // tree, lists, grids; sets the partition
int hier_matvec(nc_handle* h, const double* x, double* y, cudaStream_t s);
void hier_fill_stats(const nc_handle* h, nc_stats_t* o);
int hier_grid_far(const nc_handle* h);                     // the grid kernel's far form (-1: not NC_HIER)
void hier_grid_variant(const nc_handle* h, int* v8);       // its variant {nt, tpt, unroll, stage, far, tma, minb, persist}
void hier_destroy(nc_handle* h);
}  // namespace nc
