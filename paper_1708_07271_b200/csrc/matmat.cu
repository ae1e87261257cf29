// Multi-vector product launch (cmvg_matmat_f32).
#include "cuda/bvd_matmat.cuh"
#include "internal.hpp"

namespace cmvg {

// Columns are processed in chunks of at most 16 (the k-wide deltas of a
// block live in shared memory); each chunk decodes the block once.
void launch_matmat(cmvg_graph* g, const float* X, float* Y, uint32_t k, cudaStream_t st) {
  int maxsm = 0;
  CUDA_TRY(cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerBlockOptin, g->device));
  uint32_t kc = std::min<uint32_t>(k, 16);
  while (kc > 1 && (int)matmat_smem_layout(g->dims, g->stream_cap_words, kc).total > maxsm) kc /= 2;
  const MatmatSmem L = matmat_smem_layout(g->dims, g->stream_cap_words, kc);
  if ((int)L.total > maxsm) throw AbiError(CMVG_ERR_UNSUPPORTED, "matmat: block deltas do not fit in shared memory");
  CUDA_TRY(cudaFuncSetAttribute(bvd_matmat_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.total));
  for (uint32_t c0 = 0; c0 < k; c0 += kc) {
    const uint32_t kk = std::min(kc, k - c0);
    bvd_matmat_kernel<<<g->nblocks, 512, L.total, st>>>(g->dev(), X + c0, Y + c0, kk, k);
    CUDA_TRY(cudaGetLastError());
  }
}

}  // namespace cmvg
