// Launches of the BV-F gather kernel (cuda/bvf_gather.cuh): y = A x^T in fp64
// and fp32, and the fused PageRank step.
#include "cuda/bvf_gather.cuh"
#include "internal.hpp"

#include <cstdlib>

namespace cmvg {

template <typename XT, typename YT, bool PR>
void launch_bvf(cmvg_graph* g, const XT* x, const XT* xfar, YT* y, const PrArgs& pr, cudaStream_t st, uint32_t b0,
                uint32_t b1) {
  b1 = std::min(b1, g->nblocks);
  if (b0 >= b1) return;
  const BvfSmem L = bvf_smem_layout(g->dims.window, g->dims.block_rows, sizeof(XT) == 8);
  const bool dflt = g->dims.window == 1536 && g->dims.block_rows == 1024;  // the default shape, specialised
  auto kern = dflt ? bvf_gather_kernel<XT, YT, PR, 1536, 1024> : bvf_gather_kernel<XT, YT, PR>;
  const unsigned bit = ((sizeof(XT) == 8 ? 1u : 2u) << (PR ? 2 : 0)) << (dflt ? 4 : 0);  // once per handle and variant
  if (!(g->fgather_attr & bit)) {
    CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.total));
    // the whole unified L1 as shared memory: 4 CTAs of ~56 KB per SM
    CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    g->fgather_attr |= bit;
  }
  BvfDev d{};
  d.words = g->fwords.as<uint32_t>();
  d.blocks = g->fblocks.as<BvfBlockInfo>() + b0;
  d.n = g->n;
  d.B = g->dims.block_rows;
  d.W = g->dims.window;
  d.max_depth = g->dims.max_depth;
  d.block_begin = g->block_begin + b0;
  d.row_begin = g->row_begin;
  d.nlaunch = b1 - b0;
  {
    int occ = 0, sms = 0;
    if (!g->fgather_res) {  // resident CTAs: the L2 prefetch distance (CMVG_PREFETCH_AHEAD overrides; 0 = off)
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kBvfThreads, L.total) != cudaSuccess) occ = 1;
      if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, g->device) != cudaSuccess) sms = 1;
      uint32_t a = (uint32_t)std::max(occ, 1) * (uint32_t)std::max(sms, 1);
      if (const char* e = std::getenv("CMVG_PREFETCH_AHEAD")) a = (uint32_t)std::strtoul(e, nullptr, 10);
      g->fgather_res = a | 0x80000000u;
    }
    d.ahead = g->fgather_res & 0x7fffffffu;
  }
  if (!xfar) xfar = x;
  // escape terms: their x values gathered first (stream-ordered scratch, so
  // concurrent products on distinct streams and graph captures stay independent)
  const uint64_t e0 = g->fesc_base_h.empty() ? 0 : g->fesc_base_h[b0];
  const uint64_t ne = g->fesc_base_h.empty() ? 0 : g->fesc_base_h[b1] - e0;
  StreamScratch xe(g->device, ne * sizeof(XT), st);
  if (ne) {
    int sms = 148;
    (void)cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, g->device);
    const uint64_t want = (ne + 1023) / 1024;
    const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(want, (uint64_t)sms * 8));
    bvf_esc_gather<XT><<<grid, 256, 0, st>>>(g->fesc.as<uint32_t>() + e0, ne, xfar, xe.as<XT>());
    CUDA_TRY(cudaGetLastError());
  }
  d.esc_base = g->fesc_base.as<uint32_t>() + b0;
  // the kernel indexes xe by the shard-global escape number
  const XT* xe_base = ne ? xe.as<XT>() - e0 : x;
  kern<<<b1 - b0, kBvfThreads, L.total, st>>>(d, x, xfar, xe_base, y, pr);
  CUDA_TRY(cudaGetLastError());
}

template void launch_bvf<double, double, false>(cmvg_graph*, const double*, const double*, double*, const PrArgs&,
                                                cudaStream_t, uint32_t, uint32_t);
template void launch_bvf<float, float, false>(cmvg_graph*, const float*, const float*, float*, const PrArgs&,
                                              cudaStream_t, uint32_t, uint32_t);
template void launch_bvf<double, double, true>(cmvg_graph*, const double*, const double*, double*, const PrArgs&,
                                               cudaStream_t, uint32_t, uint32_t);

}  // namespace cmvg
