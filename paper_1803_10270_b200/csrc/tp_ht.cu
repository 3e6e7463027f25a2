// Batched hSVD truncation of hierarchical Tucker tensors (ht.truncate) -- kernels follow.
#include "tp_common.cuh"

extern "C" {

size_t tp_ht_truncate_ws_bytes(int, int, int, int) { return 0; }
int tp_ht_truncate_f64(int, int, int, int, const double*, const double*, int, double, double*, double*,
                       int*, double*, double*, void*, size_t, void*) {
  return TP_EUNSUPPORTED;
}

}  // extern "C"
