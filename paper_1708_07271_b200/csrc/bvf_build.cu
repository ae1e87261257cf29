// Device build of the BV-F layout (cmvg_create): the GPU decodes the BV
// stream's instantaneous codes (cuda/bv_decode.cuh: gamma / unary / copy
// blocks / intervals / zeta_3 residuals) into a device CSR plus each row's
// reference distance, then transcodes every 1024-row block into its BV-F
// stream with the same block builder the host uses (host/bvf_block.hpp: one
// block per warp, lane 0, working memory in a device arena), and packs the
// blocks.  Reference: the product's A' rows (include/cmv/ref_matrix.hpp:13-76)
// taken from the BV stream, never through the host.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "host/bvf_block.hpp"
#include "internal.hpp"

namespace cmvg {
namespace {

// per block: its edges and its rows' reference edges (arena sizing)
__global__ void bvf_block_sizes(const uint64_t* __restrict__ ro, const uint8_t* __restrict__ ref, uint32_t n,
                                uint32_t B, uint32_t b0, uint32_t nb, uint64_t* __restrict__ E,
                                uint64_t* __restrict__ Er) {
  const uint32_t q = blockIdx.x;
  if (q >= nb) return;
  const uint32_t r0 = (b0 + q) * B, r1 = min(n, r0 + B);
  uint64_t e = 0, er = 0;
  for (uint32_t i = r0 + threadIdx.x; i < r1; i += blockDim.x) {
    e += ro[i + 1] - ro[i];
    const uint32_t r = ref[i];
    if (r && i - r >= r0) er += ro[i - r + 1] - ro[i - r];
  }
  for (int o = 16; o > 0; o >>= 1) {
    e += __shfl_down_sync(0xffffffffu, e, o);
    er += __shfl_down_sync(0xffffffffu, er, o);
  }
  __shared__ uint64_t se[8], ser[8];
  if ((threadIdx.x & 31) == 0) {
    se[threadIdx.x >> 5] = e;
    ser[threadIdx.x >> 5] = er;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (uint32_t w = 1; w < blockDim.x / 32; ++w) {
      e += se[w];
      er += ser[w];
    }
    E[q] = e;
    Er[q] = er;
  }
}

// one block per warp: lane 0 runs the shared builder (one block per thread
// measured 2-4x slower: divergence and cache contention)
__global__ void __launch_bounds__(32) bvf_build_blocks(BvfRowsView g, uint32_t B, uint32_t W, uint32_t lmin, uint32_t b0,
                                                       const uint32_t* __restrict__ ids, uint32_t nb,
                                                       uint32_t* __restrict__ arena, const uint64_t* __restrict__ aoff,
                                                       uint32_t* __restrict__ out, const uint64_t* __restrict__ ooff,
                                                       BvfBlockResult* __restrict__ res) {
  const uint32_t j = blockIdx.x;
  if (j >= nb || threadIdx.x != 0) return;
  BvfArena ar{arena + aoff[j], aoff[j + 1] - aoff[j], 0};
  res[j] = bvf_build_block(g, b0 + ids[j], B, W, lmin, ar, out + ooff[j], ooff[j + 1] - ooff[j]);
}

// packs block q's words to its final offset
__global__ void bvf_pack_blocks(const uint32_t* __restrict__ src_base, const uint64_t* __restrict__ src_off,
                                const uint64_t* __restrict__ dst_off, const uint32_t* __restrict__ nwords,
                                uint32_t* __restrict__ dst_base) {
  const uint32_t j = blockIdx.x;
  const uint32_t* src = src_base + src_off[j];
  uint32_t* dst = dst_base + dst_off[j];
  for (uint32_t i = threadIdx.x; i < nwords[j]; i += blockDim.x) dst[i] = src[i];
}

// the escape columns of block q (its stream's escape table) to the flat list
__global__ void bvf_pack_escapes(const uint32_t* __restrict__ fwords, const BvfBlockInfo* __restrict__ blocks,
                                 const uint64_t* __restrict__ ebase, uint32_t* __restrict__ esc) {
  const uint32_t q = blockIdx.x;
  const BvfBlockInfo b = blocks[q];
  if (!(b.flags & kBvfFlagEsc)) return;
  const uint32_t* es = fwords + b.word_offset + b.esc_off;
  const uint32_t ne = es[b.nact];
  const uint32_t* cols = es + bvf_align4(b.nact + 1u);
  for (uint32_t i = threadIdx.x; i < ne; i += blockDim.x) esc[ebase[q] + i] = cols[i];
}

}  // namespace

// Builds the handle's BV-F layout on the device (blocks [block_begin,
// block_begin + nblocks)).  Fills g->fwords / fblocks / fesc / fesc_base /
// fesc_base_h, the BV-F stats, win_need / far_need and the product stats.
// Returns false (nothing changed) when the tile decoder cannot serve the
// stream's segments; throws on a corrupt stream.
bool device_build_bvf(cmvg_graph* g, cudaStream_t st, DeviceBuildStats& ds) {
  if (!decode_tiles_ok(g)) return false;
  // decode (whole graph: references stay inside 1024-row segments)
  DevBuf dro, dco, dref;
  dro.alloc(((size_t)g->n + 1) * 8);
  dco.alloc(g->m * 4 + 16);
  dref.alloc((size_t)g->n + 16);
  decode_device(g, dro.as<uint64_t>(), dco.as<uint32_t>(), dref.as<uint8_t>(), st);
  const BvfRowsView view{dro.as<uint64_t>(), dco.as<uint32_t>(), dref.as<uint8_t>(), g->n};
  return build_bvf_from_rows(g, view, st, ds);
}

// The BV-F layout of g's blocks from device rows with reference distances
// (the decoded BV stream, or a transposed graph's chosen references).
bool build_bvf_from_rows(cmvg_graph* g, const BvfRowsView& view, cudaStream_t st, DeviceBuildStats& ds) {
  static const bool timing = getenv("CMVG_BUILD_TIMING") != nullptr;
  auto t0 = std::chrono::steady_clock::now();
  auto lap = [&](const char* what) {
    if (!timing) return;
    CUDA_TRY(cudaStreamSynchronize(st));
    const auto t1 = std::chrono::steady_clock::now();
    fprintf(stderr, "[device build] %-10s %8.2f ms\n", what, std::chrono::duration<double, std::milli>(t1 - t0).count());
    t0 = t1;
  };
  const uint32_t B = g->dims.block_rows, W = g->dims.window, lmin = g->params.min_interval;
  lap("rows");
  const uint32_t nb = g->nblocks, bb = g->block_begin;
  // per-block sizes
  std::vector<uint64_t> E(nb), Er(nb);
  {
    DevBuf dE, dEr;
    dE.alloc((size_t)nb * 8);
    dEr.alloc((size_t)nb * 8);
    bvf_block_sizes<<<nb, 256, 0, st>>>(view.ro, view.ref, g->n, B, bb, nb, dE.as<uint64_t>(), dEr.as<uint64_t>());
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaMemcpyAsync(E.data(), dE.p, (size_t)nb * 8, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(Er.data(), dEr.p, (size_t)nb * 8, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
  }
  lap("sizes");
  // batches of blocks whose arenas fit the budget
  // words of arena + output per batch: 12 GB, or a quarter of the free device
  // memory when less is free (CMVG_BUILD_BUDGET_WORDS overrides)
  uint64_t budget = 3ull << 30;
  {
    size_t fr = 0, tot = 0;
    if (cudaMemGetInfo(&fr, &tot) == cudaSuccess) budget = std::min<uint64_t>(budget, fr / 16);
    (void)cudaGetLastError();
    budget = std::max<uint64_t>(budget, 1ull << 24);
  }
  if (const char* e = getenv("CMVG_BUILD_BUDGET_WORDS")) budget = strtoull(e, nullptr, 10);
  std::vector<BvfBlockResult> res(nb);
  // Blocks are built in order of decreasing size (hub blocks of power-law
  // graphs together, so they overlap instead of stretching every batch), in
  // batches whose arenas fit the budget, into bounded per-block regions; each
  // batch is then packed into a compact buffer (block-local offsets).
  std::vector<uint64_t> need(nb);
  for (uint32_t q = 0; q < nb; ++q) {
    const uint32_t r0 = (bb + q) * B, nr = std::min<uint32_t>(B, g->n - r0);
    need[q] = bvf_block_scratch_words(E[q], Er[q], nr, lmin);
  }
  std::vector<uint32_t> order(nb);
  for (uint32_t q = 0; q < nb; ++q) order[q] = q;
  std::stable_sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) { return need[a] > need[b]; });
  struct Plan {
    std::vector<uint32_t> ids;
    std::vector<uint64_t> aoff, ooff;
  };
  std::vector<Plan> plans;
  uint64_t amax = 0, omax = 0;
  for (uint32_t k = 0; k < nb;) {
    Plan p{{}, {0}, {0}};
    uint64_t aw = 0, ow = 0;
    while (k < nb) {
      const uint32_t q = order[k], r0 = (bb + q) * B, nr = std::min<uint32_t>(B, g->n - r0);
      const uint64_t a = need[q] + 64;
      const uint64_t o = (bvf_block_out_words(E[q], Er[q], nr, lmin) + 3) & ~3ull;
      if (!p.ids.empty() && aw + ow + a + o > budget) break;
      aw += a;
      ow += o;
      p.ids.push_back(q);
      p.aoff.push_back(aw);
      p.ooff.push_back(ow);
      ++k;
    }
    amax = std::max(amax, aw);
    omax = std::max(omax, ow);
    plans.push_back(std::move(p));
  }
  struct Batch {
    std::vector<uint32_t> ids;
    std::vector<uint64_t> poff;  // block-local offsets in `packed`
    std::unique_ptr<DevBuf> packed;
  };
  std::vector<Batch> batches;
  {
    DevBuf arena, out;
    arena.alloc(amax * 4);
    out.alloc(omax * 4 + 16);
    lap("alloc");
    for (Plan& pl : plans) {
      const uint32_t n1 = (uint32_t)pl.ids.size();
      DevBuf dids, daoff, dooff, dres;
      dids.upload(pl.ids.data(), n1);
      daoff.upload(pl.aoff.data(), pl.aoff.size());
      dooff.upload(pl.ooff.data(), pl.ooff.size());
      dres.alloc((size_t)n1 * sizeof(BvfBlockResult));
      bvf_build_blocks<<<n1, 32, 0, st>>>(view, B, W, lmin, bb, dids.as<uint32_t>(), n1, arena.as<uint32_t>(),
                                          daoff.as<uint64_t>(), out.as<uint32_t>(), dooff.as<uint64_t>(),
                                          dres.as<BvfBlockResult>());
      CUDA_TRY(cudaGetLastError());
      std::vector<BvfBlockResult> br(n1);
      CUDA_TRY(cudaMemcpyAsync(br.data(), dres.p, (size_t)n1 * sizeof(BvfBlockResult), cudaMemcpyDeviceToHost, st));
      CUDA_TRY(cudaStreamSynchronize(st));
      lap("build");
      Batch bt{pl.ids, std::vector<uint64_t>(n1 + 1, 0), std::unique_ptr<DevBuf>(new DevBuf)};
      std::vector<uint32_t> nw(n1);
      for (uint32_t j = 0; j < n1; ++j) {
        const uint32_t q = pl.ids[j];
        if (br[j].err)
          throw std::runtime_error("BV-F device build: block " + std::to_string(bb + q) + " failed (code " +
                                   std::to_string(br[j].err) + ")");
        res[q] = br[j];
        nw[j] = br[j].nwords;
        bt.poff[j + 1] = bt.poff[j] + br[j].nwords;
      }
      bt.packed->alloc(bt.poff[n1] * 4 + 16);
      DevBuf dpoff, dnw;
      dpoff.upload(bt.poff.data(), n1);
      dnw.upload(nw.data(), n1);
      bvf_pack_blocks<<<n1, 256, 0, st>>>(out.as<uint32_t>(), dooff.as<uint64_t>(), dpoff.as<uint64_t>(),
                                          dnw.as<uint32_t>(), bt.packed->as<uint32_t>());
      CUDA_TRY(cudaGetLastError());
      CUDA_TRY(cudaStreamSynchronize(st));
      batches.push_back(std::move(bt));
      lap("pack");
    }
  }
  lap("free");
  // final offsets, block table, packing
  std::vector<BvfBlockInfo> fbl(nb);
  std::vector<uint64_t> foff(nb + 1, 0), ebase(nb + 1, 0);
  BvfStats fs;
  uint64_t adds = 0, gath = 0, inw = 0;
  uint32_t depth = 0;
  for (uint32_t q = 0; q < nb; ++q) {
    const BvfBlockResult& r = res[q];
    fbl[q] = r.info;
    fbl[q].word_offset = foff[q];
    foff[q + 1] = foff[q] + r.nwords;
    ebase[q + 1] = ebase[q] + ((r.info.flags & kBvfFlagEsc) ? r.esc_terms : 0);
    fs.terms += r.terms;
    fs.pad_terms += r.pad_terms;
    fs.slot_terms += r.slot_terms;
    fs.esc_terms += r.esc_terms;
    fs.esc_blocks += (r.info.flags & kBvfFlagEsc) ? 1 : 0;
    fs.max_K = std::max<uint32_t>(fs.max_K, r.info.K);
    fs.min_cbits = std::min<uint32_t>(fs.min_cbits, r.info.cbits);
    adds += r.adds;
    gath += r.gathered;
    inw += r.in_window;
    depth = std::max(depth, r.depth);
  }
  if (ebase[nb] > 0xffffffffull) throw std::runtime_error("BV-F: more than 2^32 escape terms in one shard");
  g->fwords.alloc((foff[nb] + 64) * 4);
  CUDA_TRY(cudaMemsetAsync(g->fwords.p, 0, (foff[nb] + 64) * 4, st));
  for (Batch& bt : batches) {  // each batch's blocks to their final offsets
    const uint32_t n1 = (uint32_t)bt.ids.size();
    std::vector<uint64_t> dst(n1);
    std::vector<uint32_t> nw(n1);
    for (uint32_t j = 0; j < n1; ++j) {
      dst[j] = foff[bt.ids[j]];
      nw[j] = res[bt.ids[j]].nwords;
    }
    DevBuf dsrc, ddst, dnw;
    dsrc.upload(bt.poff.data(), n1);
    ddst.upload(dst.data(), n1);
    dnw.upload(nw.data(), n1);
    bvf_pack_blocks<<<n1, 256, 0, st>>>(bt.packed->as<uint32_t>(), dsrc.as<uint64_t>(), ddst.as<uint64_t>(),
                                        dnw.as<uint32_t>(), g->fwords.as<uint32_t>());
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaStreamSynchronize(st));
    bt.packed.reset();
  }
  batches.clear();
  lap("concat");
  g->fblocks.upload(fbl.data(), fbl.size());
  {  // flat escape columns (the pre-gather's index list)
    std::vector<uint32_t> eb(nb + 1);
    for (uint32_t q = 0; q <= nb; ++q) eb[q] = (uint32_t)ebase[q];
    g->fesc.alloc((ebase[nb] + 4) * 4);
    CUDA_TRY(cudaMemsetAsync(g->fesc.p, 0, (ebase[nb] + 4) * 4, st));
    DevBuf deb;
    deb.upload(ebase.data(), ebase.size());
    bvf_pack_escapes<<<nb, 256, 0, st>>>(g->fwords.as<uint32_t>(), g->fblocks.as<BvfBlockInfo>(), deb.as<uint64_t>(),
                                         g->fesc.as<uint32_t>());
    CUDA_TRY(cudaGetLastError());
    g->fesc_base.upload(eb.data(), eb.size());
    g->fesc_base_h.assign(ebase.begin(), ebase.end());
    CUDA_TRY(cudaStreamSynchronize(st));
  }
  lap("escapes");
  g->f_stream_bytes = foff[nb] * 4;
  fs.stream_bytes = foff[nb] * 4;
  g->fstats = fs;
  // host pipelined gather: the x prefix each block's window and far columns need
  g->win_need.resize(nb);
  g->far_need.resize(nb);
  uint64_t pm = 0, fm = 0;
  for (uint32_t q = 0; q < nb; ++q) {
    pm = std::max<uint64_t>(pm, (uint64_t)fbl[q].wlo + W);
    fm = std::max<uint64_t>(fm, res[q].max_far);
    g->win_need[q] = (uint32_t)std::min<uint64_t>(pm, g->n);
    g->far_need[q] = (uint32_t)std::min<uint64_t>(fm, g->n);
  }
  g->dims.max_depth = std::max(g->dims.max_depth, depth);
  if (timing) {
    double cyc[6] = {0};
    uint64_t mx = 0;
    for (uint32_t q = 0; q < nb; ++q) {
      uint64_t t = 0;
      for (int k = 0; k < 6; ++k) {
        cyc[k] += (double)res[q].cyc[k];
        t += res[q].cyc[k];
      }
      mx = std::max(mx, t);
    }
    fprintf(stderr, "[device build] per-block Mcycles (mean): splits %.2f window %.2f far %.2f terms %.2f schedule %.2f "
                    "stream %.2f; slowest block %.1f\n",
            cyc[0] / nb / 1e6, cyc[1] / nb / 1e6, cyc[2] / nb / 1e6, cyc[3] / nb / 1e6, cyc[4] / nb / 1e6,
            cyc[5] / nb / 1e6, (double)mx / 1e6);
  }
  lap("finish");
  ds.adds = adds;
  ds.depth = depth;
  ds.window_coverage = gath ? (double)inw / (double)gath : 1.0;
  return true;
}

}  // namespace cmvg
