// Entry points declared in tpde_b200.h whose kernels land in later commits.
#include "tp_common.cuh"

extern "C" {

size_t tp_implicit_ws_bytes(int, int, int, int) { return 0; }
int tp_implicit_step_f64(int, int, int, int, const double*, const double*, const double*, const double*,
                         double*, int, double, double, int, double*, int*, void*, size_t, void*) {
  return TP_EUNSUPPORTED;
}

}  // extern "C"
