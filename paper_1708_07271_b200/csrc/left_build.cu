// y = x A the reference's way: matvec_ref_left computes (A^T) x on
// compress(transpose(g)) (include/cmv/ref_matvec.hpp:37-41).  Here the
// transpose, its reference choice and its BV-F layout are all built on the
// GPU, from the handle's BV stream, the first time a product asks for it:
//   1. decode A (cuda/bv_decode.cuh) into a device CSR;
//   2. transpose: a stable radix sort of the (column, row) pairs by column
//      (rows stay ascending within each column) and the column offsets;
//   3. references for the rows of A^T, the rule of cmv::compress
//      (ref_matrix.hpp:58-69): among the previous W rows of the same
//      1024-row block (chains never leave a block, depth <= R when R is
//      bounded) the one with the smallest symmetric difference, ties to the
//      nearest, used only when strictly smaller than the row itself;
//   4. the BV-F block builder (host/bvf_block.hpp) on those rows and
//      references, then the gather kernel runs x A as (A^T) x.
#include <cub/device/device_radix_sort.cuh>

#include <memory>
#include <stdexcept>
#include <string>

#include "host/bvf_block.hpp"
#include "internal.hpp"

namespace cmvg {
namespace {

__global__ void lt_expand_rows(const uint64_t* __restrict__ ro, uint32_t n, uint32_t* __restrict__ rowid) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (uint64_t e = ro[i]; e < ro[i + 1]; ++e) rowid[e] = i;
}

// row offsets of A^T from its sorted column keys: rot[j] = first edge with key >= j
__global__ void lt_col_offsets(const uint32_t* __restrict__ keys, uint64_t m, uint32_t n, uint64_t* __restrict__ rot) {
  const uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= m) return;
  const int64_t prev = e ? (int64_t)keys[e - 1] : -1;
  for (int64_t j = prev + 1; j <= (int64_t)keys[e]; ++j) rot[j] = e;
  if (e == m - 1)
    for (uint64_t j = (uint64_t)keys[e] + 1; j <= n; ++j) rot[j] = m;
}

// |L delta R| of two sorted rows, stopping once it reaches `limit`
__device__ __forceinline__ uint32_t lt_symdiff(const uint32_t* L, uint32_t dl, const uint32_t* R, uint32_t dr,
                                               uint32_t limit) {
  uint32_t a = 0, b = 0, c = 0;
  while (a < dl && b < dr) {
    const uint32_t x = L[a], y = R[b];
    if (x == y) {
      ++a;
      ++b;
    } else {
      ++c;
      if (x < y) ++a;
      else ++b;
      if (c >= limit) return c;
    }
  }
  return c + (dl - a) + (dr - b);
}

// one thread per block of B rows of A^T, rows in order (a reference's depth
// is known before its children choose)
__global__ void lt_choose_refs(const uint64_t* __restrict__ ro, const uint32_t* __restrict__ co, uint32_t n,
                               uint32_t B, uint32_t window, uint32_t max_ref, uint8_t* __restrict__ ref,
                               uint8_t* __restrict__ depth) {
  const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t nb = (n + B - 1) / B;
  if (b >= nb) return;
  const uint32_t r0 = b * B, nr = min(B, n - r0);
  uint8_t* dep = depth + r0;
  for (uint32_t k = 0; k < nr; ++k) {
    const uint32_t i = r0 + k;
    const uint32_t di = (uint32_t)(ro[i + 1] - ro[i]);
    uint32_t best = 0, bestc = di;  // a reference only when strictly shorter than the row
    for (uint32_t r = 1; r <= window && r <= k && bestc; ++r) {
      if (max_ref && dep[k - r] >= max_ref) continue;
      const uint32_t j = i - r;
      const uint32_t c = lt_symdiff(co + ro[i], di, co + ro[j], (uint32_t)(ro[j + 1] - ro[j]), bestc);
      if (c < bestc) {  // ties keep the nearer reference
        bestc = c;
        best = r;
      }
    }
    ref[i] = (uint8_t)best;
    dep[k] = best ? (uint8_t)min(255u, dep[k - best] + 1u) : (uint8_t)0;
  }
}

}  // namespace

// The A^T handle of a whole-graph handle g (device memory only; products
// through launch_bvf on it).
std::unique_ptr<cmvg_graph> build_left_handle(cmvg_graph* g, cudaStream_t st) {
  if (!decode_tiles_ok(g)) throw std::runtime_error("x A (left): the stream's segments do not tile the decoder");
  const uint32_t n = g->n;
  const uint64_t m = g->m;
  auto t = std::make_unique<cmvg_graph>();
  t->device = g->device;
  t->n = n;
  t->m = m;
  t->params = g->params;
  t->row_begin = 0;
  t->row_end = n;
  t->block_begin = 0;
  t->dims = BvdDims{n, g->dims.block_rows, g->dims.window, g->params.min_interval,
                    (uint32_t)(((uint64_t)n + g->dims.block_rows - 1) / g->dims.block_rows), 0, 0, 0};
  t->nblocks = t->dims.nblocks;
  t->threads = g->threads;
  t->interval_mode = g->interval_mode;
  DevBuf rot, cot, ref;
  {
    DevBuf ro, co, rowid, keys;
    ro.alloc(((size_t)n + 1) * 8);
    co.alloc(m * 4 + 16);
    decode_device(g, ro.as<uint64_t>(), co.as<uint32_t>(), nullptr, st);
    rowid.alloc(m * 4 + 16);
    lt_expand_rows<<<(n + 255) / 256, 256, 0, st>>>(ro.as<uint64_t>(), n, rowid.as<uint32_t>());
    CUDA_TRY(cudaGetLastError());
    keys.alloc(m * 4 + 16);
    cot.alloc(m * 4 + 16);
    int end_bit = 1;
    while (end_bit < 32 && (1ull << end_bit) < (uint64_t)n) ++end_bit;
    size_t tmp_bytes = 0;
    CUDA_TRY(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, co.as<uint32_t>(), keys.as<uint32_t>(),
                                             rowid.as<uint32_t>(), cot.as<uint32_t>(), (int64_t)m, 0, end_bit, st));
    DevBuf tmp;
    tmp.alloc(tmp_bytes + 16);
    CUDA_TRY(cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, co.as<uint32_t>(), keys.as<uint32_t>(),
                                             rowid.as<uint32_t>(), cot.as<uint32_t>(), (int64_t)m, 0, end_bit, st));
    rot.alloc(((size_t)n + 1) * 8);
    if (m == 0) {
      CUDA_TRY(cudaMemsetAsync(rot.p, 0, ((size_t)n + 1) * 8, st));
    } else {
      lt_col_offsets<<<(unsigned)((m + 255) / 256), 256, 0, st>>>(keys.as<uint32_t>(), m, n, rot.as<uint64_t>());
      CUDA_TRY(cudaGetLastError());
    }
    CUDA_TRY(cudaStreamSynchronize(st));
  }
  ref.alloc((size_t)n + 16);
  {
    DevBuf depth;
    depth.alloc((size_t)n + 16);
    const uint32_t nb = t->nblocks;
    lt_choose_refs<<<(nb + 63) / 64, 64, 0, st>>>(rot.as<uint64_t>(), cot.as<uint32_t>(), n, t->dims.block_rows,
                                                  g->params.window, g->params.max_ref, ref.as<uint8_t>(),
                                                  depth.as<uint8_t>());
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaStreamSynchronize(st));
  }
  const BvfRowsView view{rot.as<uint64_t>(), cot.as<uint32_t>(), ref.as<uint8_t>(), n};
  DeviceBuildStats ds;
  build_bvf_from_rows(t.get(), view, st, ds);
  t->device_built = true;
  t->adds = ds.adds;
  t->stats.window_coverage = ds.window_coverage;
  return t;
}

}  // namespace cmvg
