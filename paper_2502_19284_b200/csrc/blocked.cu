// blocked.cu -- CSB / MergeB / BCOH conversions and multiplies (placeholder until implemented).
#include "common.cuh"
#include "kernels.cuh"

namespace spmvcu {
extern thread_local std::string g_last_error;

int build_csb(Format&, const spmvlab_cuda_coo&, unsigned, bool, uint64_t, Arena&) {
  g_last_error = "csb not implemented yet";
  return kInvalidArgument;
}
int build_mergeb(Format&, const spmvlab_cuda_coo&, unsigned, bool, Arena&) {
  g_last_error = "mergeb not implemented yet";
  return kInvalidArgument;
}
int build_bcoh(Format&, const spmvlab_cuda_coo&, unsigned, unsigned, Arena&) {
  g_last_error = "bcoh not implemented yet";
  return kInvalidArgument;
}
int spmv_blocked(const Format&, const double*, double*, cudaStream_t) {
  g_last_error = "blocked not implemented yet";
  return kInvalidArgument;
}

}  // namespace spmvcu
