// bvd_gather: y = A * x^T on the BV-D layout -- the hot path, replacing the
// reference's sequential `matvec_ref_into` (include/cmv/ref_matvec.hpp:20-31,
// SPEC.md:197-205).
//
// One CTA per block of B rows (reference chains never leave a block):
//   1. thread 0 issues a TMA bulk copy of the block's coded stream into
//      shared memory (mbarrier completion) while all threads stage the
//      x-window x[wlo, wlo+W) and build its tile-local double-double prefix;
//   2. row setup: row bit offsets (scan of body lengths from the headers) and
//      warp rounds (rows counting-sorted by point-code count, so the 32 rows
//      a warp decodes together have near-equal work);
//   3. each warp decodes its rounds, one row per lane: a loop over point
//      codes (minus -> -x[c], residual -> +x[c]) then a loop over intervals
//      (O(1) from the prefix); delta_i is accumulated with Neumaier
//      compensation, so it carries no cancellation error into the chain;
//   4. level phases over chain depth: y_i = delta_i + y_{i-r} in
//      double-double (the reference's order, ref_matvec.hpp:23-25);
//   5. coalesced store of y.
#pragma once
#include <cstdint>

#include "bvd_common.cuh"

namespace cmvg {

struct GatherSmem {
  uint32_t off_x, off_yhi, off_ylo;
  RowSmem rows;
  uint32_t total;
};

__host__ __device__ inline GatherSmem gather_smem_layout(const BvdDims& d, uint32_t stream_cap_words, uint32_t xsize,
                                                         bool prefix) {
  GatherSmem s;
  uint32_t o = align16((stream_cap_words + 8) * 4);
  s.off_x = o;
  o = align16(o + xw_bytes(d.window, xsize, prefix));
  s.off_yhi = o;
  o = align16(o + d.block_rows * 8);
  s.off_ylo = o;
  o = align16(o + d.block_rows * 4);
  s.rows = row_smem_layout(o, d.block_rows);
  s.total = s.rows.total;
  return s;
}

// Phase A (point rounds): each warp takes 32 rows of similar point-code count
// (one per lane) and accumulates -x[c] for minus codes, +x[c] for residual
// codes; writes delta (hi, lo).  Phase B (interval rounds, after a barrier):
// the rows that have intervals, grouped by interval count, add their O(1)
// interval sums to delta.  Every row is owned by one lane in each phase.
template <class XWinT>
__device__ __forceinline__ void decode_points(const RowCtx& c, const uint32_t* __restrict__ base, const XWinT& xw,
                                              int32_t r0, double* s_yhi, float* s_ylo) {
  const uint32_t lane = threadIdx.x & 31u;
  const int nesc = c.misc[0];
  for (;;) {
    uint32_t rb = 0;  // next round of 32 rows, claimed dynamically (balances the warps)
    if (lane == 0) rb = 32u * (uint32_t)atomicAdd(&c.misc[3], 1);
    rb = __shfl_sync(0xffffffffu, rb, 0);
    if (rb >= c.nr) break;
    const uint32_t slot = rb + lane;
    const bool act = slot < c.nr;
    const uint32_t k = act ? c.perm[slot] : 0u;
    const uint32_t h = act ? base[k] : 0u;
    RowCounts rc{0, 0, 0};
    if (act) rc = row_counts(base, c.B, h, k, nesc);
    const uint32_t wp = hdr_wp(h);
    const int32_t i = r0 + (int32_t)k;
    const uint32_t np = rc.nm + rc.ns;
    uint32_t off = act ? c.rowoff[k] : 0u;
    double acc = 0.0, comp = 0.0;
    const uint32_t tp = __reduce_max_sync(0xffffffffu, np);
    for (uint32_t t = 0; t < tp; ++t) {
      double term = 0.0;
      if (t < np) {
        const int32_t col = i + unfold32(extract_bits(base, off, wp));
        const double xv = xw.at(col);
        term = t < rc.nm ? -xv : xv;
        off += wp;
      }
      nadd(acc, comp, term);
    }
    if (act) {
      const double hi = acc + comp;
      s_yhi[k] = hi;
      s_ylo[k] = (float)(comp - (hi - acc));
    }
  }
}

template <class XWinT>
__device__ __forceinline__ void decode_intervals(const RowCtx& c, const uint32_t* __restrict__ base, const XWinT& xw,
                                                 int32_t r0, uint32_t lmin, double* s_yhi, float* s_ylo) {
  const uint32_t lane = threadIdx.x & 31u;
  const int nesc = c.misc[0];
  const uint32_t nri = (uint32_t)c.misc[2];
  for (;;) {
    uint32_t rb = 0;
    if (lane == 0) rb = 32u * (uint32_t)atomicAdd(&c.misc[4], 1);
    rb = __shfl_sync(0xffffffffu, rb, 0);
    if (rb >= nri) break;
    const uint32_t slot = rb + lane;
    const bool act = slot < nri;
    const uint32_t k = act ? c.permi[slot] : 0u;
    const uint32_t h = act ? base[k] : 0u;
    RowCounts rc{0, 0, 0};
    if (act) rc = row_counts(base, c.B, h, k, nesc);
    const uint32_t wp = hdr_wp(h), wl = hdr_wl(h);
    const int32_t i = r0 + (int32_t)k;
    uint32_t off = act ? c.rowoff[k] + (rc.nm + rc.ns) * wp : 0u;
    double acc = 0.0, comp = 0.0;
    const uint32_t ti = __reduce_max_sync(0xffffffffu, rc.ni);
    for (uint32_t t = 0; t < ti; ++t) {
      double hi = 0.0, lo = 0.0;
      if (t < rc.ni) {
        const int32_t left = i + unfold32(extract_bits(base, off, wp));
        const uint32_t len = extract_bits(base, off + wp, wl) + lmin;
        hi = xw.isum(left, len, lo);
        off += wp + wl;
      }
      nadd(acc, comp, hi);
      comp += lo;
    }
    if (act) {
      double hi = s_yhi[k], lo = (double)s_ylo[k];
      dd_add(hi, lo, acc, comp);
      s_yhi[k] = hi;
      s_ylo[k] = (float)lo;
    }
  }
}

template <typename XT, typename YT, bool PREFIX>
__device__ __forceinline__ void gather_block(RowCtx& rc, const uint32_t* __restrict__ base, const XWin<XT, PREFIX>& xw,
                                             const BvdDims& D, uint32_t r0, double* s_yhi, float* s_ylo, YT* yb) {
  rc.base = base;
  row_setup(rc);
  decode_points(rc, base, xw, (int32_t)r0, s_yhi, s_ylo);
  __syncthreads();
  decode_intervals(rc, base, xw, (int32_t)r0, D.min_interval, s_yhi, s_ylo);
  __syncthreads();
  chain_and_store(s_yhi, s_ylo, rc, yb);
}

template <typename XT, typename YT, bool PREFIX>
__global__ void __launch_bounds__(256) bvd_gather_kernel(BvdDev g, const XT* __restrict__ x, YT* __restrict__ y) {
  extern __shared__ __align__(16) unsigned char smem[];
  const BvdDims& D = g.d;
  const GatherSmem L = gather_smem_layout(D, g.stream_cap_words, sizeof(XT), PREFIX);
  const uint32_t bl = blockIdx.x;  // index into this shard's tables
  const uint32_t b = g.block_begin + bl;
  const BvdBlockInfo bi = g.blocks[bl];
  const uint32_t r0 = b * D.block_rows;
  const uint32_t nr = min(D.block_rows, D.n - r0);

  RowCtx rc = carve_rows(smem, L.rows, D.block_rows, nr);
  uint32_t* s_stream = reinterpret_cast<uint32_t*>(smem);
  stage_stream_begin(g, bi, s_stream, rc.bar);
  XWin<XT, PREFIX> xw;
  xw.carve(smem + L.off_x, D.window);
  xw.x = x;
  xw.wlo = bi.wlo;
  xw.stage(D.n);  // ends with __syncthreads (also publishes the mbarrier init)
  mbar_wait(rc.bar, 0);

  double* s_yhi = reinterpret_cast<double*>(smem + L.off_yhi);
  float* s_ylo = reinterpret_cast<float*>(smem + L.off_ylo);
  YT* yb = y + (r0 - g.row_begin);
  if (bi.nwords <= g.stream_cap_words)  // CTA-uniform: shared-memory decode path
    gather_block<XT, YT, PREFIX>(rc, s_stream, xw, D, r0, s_yhi, s_ylo, yb);
  else
    gather_block<XT, YT, PREFIX>(rc, g.words + bi.word_offset, xw, D, r0, s_yhi, s_ylo, yb);
}

}  // namespace cmvg
