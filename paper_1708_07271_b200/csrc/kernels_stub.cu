// Entry points not yet implemented on the device: scatter form, multi-vector
// product and PageRank.  They fail loudly (no CPU fallback).
#include "internal.hpp"

namespace cmvg {
template <typename T>
void launch_scatter(cmvg_graph*, const T*, T*, cudaStream_t) {
  throw AbiError(CMVG_ERR_UNSUPPORTED, "scatter form not implemented yet");
}
template void launch_scatter<double>(cmvg_graph*, const double*, double*, cudaStream_t);
template void launch_scatter<float>(cmvg_graph*, const float*, float*, cudaStream_t);
void launch_matmat(cmvg_graph*, const float*, float*, uint32_t, cudaStream_t) {
  throw AbiError(CMVG_ERR_UNSUPPORTED, "multi-vector product not implemented yet");
}
}  // namespace cmvg
