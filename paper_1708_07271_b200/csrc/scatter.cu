// Scatter-form launch (y = x A on A's own compression).
#include "cuda/bvd_scatter.cuh"
#include "internal.hpp"

namespace cmvg {

template <typename T>
void launch_scatter(cmvg_graph* g, const T* x, T* y, cudaStream_t st) {
  const size_t n = g->n;
  g->scratch.alloc(2 * n * sizeof(double) + 64);
  double* hi = g->scratch.as<double>();
  double* lo = hi + n;
  CUDA_TRY(cudaMemsetAsync(hi, 0, 2 * n * sizeof(double), st));
  const ScatterSmem L = scatter_smem_layout(g->dims, g->stream_cap_words);
  auto kern = bvd_scatter_kernel<T>;
  CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.total));
  kern<<<g->nblocks, g->threads, L.total, st>>>(g->dev(), x, hi, lo);
  CUDA_TRY(cudaGetLastError());
  dd_round_kernel<T><<<(unsigned)((n + 255) / 256), 256, 0, st>>>(hi, lo, y, (uint32_t)n);
  CUDA_TRY(cudaGetLastError());
}

template void launch_scatter<double>(cmvg_graph*, const double*, double*, cudaStream_t);
template void launch_scatter<float>(cmvg_graph*, const float*, float*, cudaStream_t);

}  // namespace cmvg
