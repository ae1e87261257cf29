// Multi-vector product launch (cmvg_matmat_f32): on the BV-F layout, 4
// columns per pass (cuda/bvf_matmat.cuh), for the default block shape; the
// BV-S slices (cuda/bvs_matmat.cuh) otherwise.
#include "cuda/bvf_matmat.cuh"
#include "cuda/bvs_matmat.cuh"
#include "internal.hpp"

#include <cstdlib>

namespace cmvg {

namespace {
void launch_matmat_bvf(cmvg_graph* g, const float* X, float* Y, uint32_t k, cudaStream_t st) {
  constexpr BmmSmem L = bmm_smem_layout();
  if (!(g->fgather_attr & (1u << 12))) {
    CUDA_TRY(cudaFuncSetAttribute(bvf_matmat_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.total));
    CUDA_TRY(cudaFuncSetAttribute(bvf_matmat_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    g->fgather_attr |= 1u << 12;
  }
  BvfDev d{};
  d.words = g->fwords.as<uint32_t>();
  d.blocks = g->fblocks.as<BvfBlockInfo>();
  d.n = g->n;
  d.B = g->dims.block_rows;
  d.W = g->dims.window;
  d.max_depth = g->dims.max_depth;
  d.block_begin = g->block_begin;
  d.row_begin = g->row_begin;
  d.nlaunch = g->nblocks;
  {
    int sms = 148;
    (void)cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, g->device);
    d.ahead = std::getenv("CMVG_MM_AHEAD") ? (uint32_t)std::atoi(std::getenv("CMVG_MM_AHEAD")) : std::max(1u, 4u * (uint32_t)sms / ((k + kBmmCols - 1) / kBmmCols));
  }
  d.esc_base = g->fesc_base.as<uint32_t>();
  const uint64_t ne = g->fesc_base_h.empty() ? 0 : g->fesc_base_h[g->nblocks] - g->fesc_base_h[0];
  const uint32_t nch = (k + kBmmCols - 1) / kBmmCols;
  const bool vec = (k % 4u) == 0 && ((reinterpret_cast<uintptr_t>(X) | reinterpret_cast<uintptr_t>(Y)) & 15u) == 0;
  StreamScratch xe(g->device, ne * nch * 16 + 16, st);
  if (ne) {
    int sms = 148;
    (void)cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, g->device);
    const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((ne + 255) / 256, (uint64_t)sms * 8));
    bmm_esc_gather<<<dim3(grid, nch), 256, 0, st>>>(g->fesc.as<uint32_t>(), ne, X, k, vec, xe.as<float4>());
    CUDA_TRY(cudaGetLastError());
  }
  bvf_matmat_kernel<<<g->nblocks * nch, kBmmT, L.total, st>>>(d, X, k, vec, nch, xe.as<float4>(), ne, Y);
  CUDA_TRY(cudaGetLastError());
}
}  // namespace

void launch_matmat(cmvg_graph* g, const float* X, float* Y, uint32_t k, cudaStream_t st) {
  static const bool bvs = std::getenv("CMVG_MATMAT_BVS") != nullptr;  // the BV-S kernel (A/B)
  if (!bvs && g->dims.window == kBmmW && g->dims.block_rows == kBmmB) {
    launch_matmat_bvf(g, X, Y, k, st);
    return;
  }
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
