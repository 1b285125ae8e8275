// hier.cu -- hierarchical mode (placeholder until the device tree lands).
#include "hier.cuh"

namespace nc {
int hier_order(nc_handle* h, std::vector<double>& centers) {
  (void)h; (void)centers;
  return fail(NC_EUNSUP, "NC_HIER not built yet");
}
int hier_partition(nc_handle* h) { (void)h; return fail(NC_EUNSUP, "NC_HIER not built yet"); }
int hier_setup(nc_handle* h, cudaStream_t s) { (void)h; (void)s; return fail(NC_EUNSUP, "NC_HIER not built yet"); }
int hier_matvec(nc_handle* h, const double* x, double* y, cudaStream_t s) {
  (void)h; (void)x; (void)y; (void)s;
  return fail(NC_EUNSUP, "NC_HIER not built yet");
}
void hier_fill_stats(const nc_handle* h, nc_stats_t* o) { (void)h; (void)o; }
void hier_destroy(nc_handle* h) { (void)h; }
}  // namespace nc

extern "C" int nc_tree_lists(const nc_handle* h, int64_t* n_ilist, int64_t* ilist, int64_t* n_nbr, int64_t* nbr,
                             int64_t* box_of_patch) {
  (void)h; (void)n_ilist; (void)ilist; (void)n_nbr; (void)nbr; (void)box_of_patch;
  return nc::fail(NC_EUNSUP, "NC_HIER not built yet");
}
