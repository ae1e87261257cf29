// Scatter-form launch (y = x A on A's own compression): BV-T segmented sums
// per block, then the deterministic combine (cuda/bvt_scatter.cuh).
#include "cuda/bvt_scatter.cuh"
#include "internal.hpp"

namespace cmvg {

template <typename T>
void launch_scatter(cmvg_graph* g, const T* x, T* y, cudaStream_t st) {
  ensure_layouts(g, false, true);
  const size_t W = g->dims.window;
  const size_t nst = (size_t)g->nblocks * W;
  const size_t nfar = (size_t)g->tfar_end - g->tfar_begin;
  // staging: partial windows (hi f64 + lo f32) and the shard's far slots
  const size_t bytes = nst * 12 + nfar * 12 + 256;
  StreamScratch scratch(g->device, bytes, st);  // per launch: concurrent scatters never share it
  unsigned char* p = scratch.as<unsigned char>();
  BvtOut o;
  o.st_hi = reinterpret_cast<double*>(p);
  o.far_hi = o.st_hi + nst;
  o.st_lo = reinterpret_cast<float*>(o.far_hi + nfar);
  o.far_lo = o.st_lo + nst;
  o.far_hi -= g->tfar_begin;  // indexed by global far slot
  o.far_lo -= g->tfar_begin;
  const BvtSmem L = bvt_smem_layout(g->dims);
  const bool dflt = g->dims.window == kGatherDefault.W && g->dims.block_rows == kGatherDefault.B &&
                    g->threads == kGatherDefault.T;
  auto k1 = dflt ? bvt_scatter_kernel<T, kGatherDefault.W, kGatherDefault.B, kGatherDefault.T> : bvt_scatter_kernel<T>;
  const unsigned bit = sizeof(T) == 8 ? 4u : 8u;  // the attribute call is not free: once per handle and type
  if (!(g->gather_attr & bit)) {
    CUDA_TRY(cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.total));
    g->gather_attr |= bit;
  }
  k1<<<g->nblocks, g->threads, L.total, st>>>(g->tdev(), x, o);
  CUDA_TRY(cudaGetLastError());
  const uint32_t ntiles = g->dims.nblocks;
  bvt_combine_kernel<T><<<ntiles, 256, 0, st>>>(g->tdev(), g->tile_ptr.as<uint32_t>(), g->tile_blk.as<uint32_t>(),
                                                g->farp_ptr.as<uint32_t>(), g->farp.as<uint32_t>(), o, g->nblocks,
                                                g->tfar_begin, g->tfar_end, y);
  CUDA_TRY(cudaGetLastError());
}

template void launch_scatter<double>(cmvg_graph*, const double*, double*, cudaStream_t);
template void launch_scatter<float>(cmvg_graph*, const float*, float*, cudaStream_t);

}  // namespace cmvg
