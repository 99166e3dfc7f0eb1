// Multi-GPU halo layer (placeholder: single-GPU build; multi-rank transports follow).
#include "comm.h"

namespace fastilu {

struct Comm {};

fastilu_status comm_setup(Comm *&out, const fastilu_options &, int64_t, int64_t, int64_t,
                          int64_t, cudaStream_t) {
  out = nullptr;
  return FASTILU_ERR_UNSUPPORTED;
}
fastilu_status comm_vector_halo(Comm *, double *, cudaStream_t, bool, bool) {
  return FASTILU_ERR_UNSUPPORTED;
}
fastilu_status comm_factor_halo(Comm *, double *, const int64_t *, double *, cudaStream_t) {
  return FASTILU_ERR_UNSUPPORTED;
}
fastilu_status comm_allreduce_host(Comm *, double *, int, ErrFlags &) {
  return FASTILU_ERR_UNSUPPORTED;
}
void comm_destroy(Comm *) {}

}  // namespace fastilu

extern "C" fastilu_status fastilu_group_create(fastilu_group *out, int) {
  if (out) *out = nullptr;
  return FASTILU_ERR_UNSUPPORTED;
}
extern "C" fastilu_status fastilu_group_destroy(fastilu_group) { return FASTILU_OK; }
extern "C" fastilu_status fastilu_nccl_unique_id(void *) { return FASTILU_ERR_UNSUPPORTED; }
