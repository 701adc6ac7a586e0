// tcgen05 (5th-gen tensor core) implicit-GEMM convolution, fp32 via BF16x3.
// (placeholder: filled in by the tensor-core milestone)
#include "common.cuh"

namespace dnnp {

bool tc_eligible(const ConvProblem&, int) { return false; }

cudaError_t tc_forward(const ConvProblem&, const float*, const float*, float*, double, double,
                       cudaStream_t) {
  return cudaErrorNotSupported;
}
cudaError_t tc_backward_data(const ConvProblem&, const float*, const float*, float*, bool,
                             cudaStream_t) {
  return cudaErrorNotSupported;
}
cudaError_t tc_backward_filter(const ConvProblem&, const float*, const float*, float*, bool,
                               cudaStream_t) {
  return cudaErrorNotSupported;
}

}  // namespace dnnp
