// Multi-vector product launch (cmvg_matmat_f32): BV-S slices, columns in
// chunks of kMmCols (cuda/bvs_matmat.cuh).
#include "cuda/bvs_matmat.cuh"
#include "internal.hpp"

namespace cmvg {

void launch_matmat(cmvg_graph* g, const float* X, float* Y, uint32_t k, cudaStream_t st) {
  ensure_layouts(g, true, false);
  const BvsMmSmem L = bvs_mm_smem_layout(g->dims);
  CUDA_TRY(cudaFuncSetAttribute(bvs_matmat_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.total));
  for (uint32_t c0 = 0; c0 < k; c0 += kMmCols) {
    const uint32_t kk = std::min(kMmCols, k - c0);
    bvs_matmat_kernel<<<g->nblocks, 512, L.total, st>>>(g->sdev(), X + c0, Y + c0, k, kk);
    CUDA_TRY(cudaGetLastError());
  }
}

}  // namespace cmvg
