// bvd_gather: y = A * x^T on the BV-D layout -- the hot path, replacing the
// reference's sequential `matvec_ref_into` (include/cmv/ref_matvec.hpp:20-31,
// SPEC.md:197-205).
//
// One CTA per block of B rows (reference chains never leave a block):
//   1. thread 0 issues a TMA bulk copy of the block's coded stream into
//      shared memory (mbarrier completion) while all threads stage the
//      x-window x[wlo, wlo+W) and build its tile-local double-double prefix;
//   2. row setup: row bit offsets (scan of body lengths from the headers) and
//      warp rounds (near rows counting-sorted by point-code count, so the 32
//      rows a warp decodes together have near-equal work);
//   3. warps claim rounds dynamically; one row per lane: point codes
//      (minus -> -x[c], residual -> +x[c]) with no bounds checks; then the
//      rounds of rows with intervals (O(1) from the prefix); then the rare
//      `far` rows on a bounds-checked path.  delta_i is accumulated with
//      TwoSum compensation (no cancellation error enters the chain);
//   4. level scheduler over chain depth: y_i = delta_i + y_{i-r} in
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

struct RowDesc {
  uint32_t k, h, off;
  RowCounts rc;
  bool act;
};

template <class S>
__device__ __forceinline__ RowDesc round_row(const RowCtx& c, const S& src, const uint16_t* perm, uint32_t slot,
                                             uint32_t end, int nesc) {
  RowDesc r;
  r.act = slot < end;
  r.k = r.act ? perm[slot] : 0u;
  r.h = r.act ? src.w(r.k) : 0u;
  r.rc = RowCounts{0, 0, 0};
  if (r.act) r.rc = row_counts(src, c.B, r.h, r.k, nesc);
  r.off = r.act ? c.rowoff[r.k] : 0u;
  return r;
}

// Phase 1 (point rounds): one row per lane, rows of similar point-code count
// per warp.  minus -> -x[c], residual -> +x[c]; `far` rows (some column
// outside the block's x-window) take the bounds-checked accessor.
template <class S, class XW>
__device__ __forceinline__ void gather_points(const RowCtx& c, const S& src, const XW& xw, int32_t r0,
                                              double* s_yhi, float* s_ylo) {
  const int nesc = c.misc[kNesc];
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t npts = (uint32_t)c.misc[kNPts];
  uint32_t rb = claim_take(claim_issue(&c.misc[kRoundP]));
  while (rb < npts) {
    const uint32_t ticket = claim_issue(&c.misc[kRoundP]);
    const RowDesc r = round_row(c, src, c.perm, rb + lane, npts, nesc);
    const uint32_t wp = hdr_wp(r.h);
    const bool far = hdr_far(r.h);
    const bool any_far = __any_sync(0xffffffffu, far);
    // window-relative column of code value v: ib + v
    const uint32_t ib = (uint32_t)(r0 + (int32_t)r.k - (int32_t)code_bias(wp) - (int32_t)xw.wlo);
    const uint32_t np = r.rc.nm + r.rc.ns, nm = r.rc.nm;
    uint32_t off = r.off;
    double acc = 0.0, comp = 0.0;
    const uint32_t tp = __reduce_max_sync(0xffffffffu, np);
    if (!any_far) {
      // two independent compensated chains (even / odd codes) halve the
      // dependent FP64 latency per code
      double acc2 = 0.0, comp2 = 0.0;
      uint32_t t = 0;
#pragma unroll 2
      for (; t + 1 < tp; t += 2) {
        const bool on0 = t < np, on1 = t + 1 < np;
        const uint32_t v0 = extract_bits(src, off, wp);
        const uint32_t off1 = off + (on0 ? wp : 0u);
        const uint32_t v1 = extract_bits(src, off1, wp);
        const double x0 = xw.at_near(on0 ? ib + v0 : 0u);
        const double x1 = xw.at_near(on1 ? ib + v1 : 0u);
        tsum(acc, comp, on0 ? (t < nm ? -x0 : x0) : 0.0);
        tsum(acc2, comp2, on1 ? (t + 1 < nm ? -x1 : x1) : 0.0);
        off = off1 + (on1 ? wp : 0u);
      }
      if (t < tp) {
        const bool on = t < np;
        const uint32_t v = extract_bits(src, off, wp);
        const double xv = xw.at_near(on ? ib + v : 0u);
        tsum(acc, comp, on ? (t < nm ? -xv : xv) : 0.0);
      }
      tsum(acc, comp, acc2);
      comp += comp2;
    } else {
      for (uint32_t t = 0; t < tp; ++t) {
        const bool on = t < np;
        const uint32_t v = extract_bits(src, off, wp);
        double xv = 0.0;
        if (on) xv = far ? xw.at((int32_t)(ib + v) + (int32_t)xw.wlo) : xw.at_near(ib + v);
        const double term = on ? (t < nm ? -xv : xv) : 0.0;
        tsum(acc, comp, term);
        off += on ? wp : 0u;
      }
    }
    if (r.act) {
      const double hi = acc + comp;
      s_yhi[r.k] = hi;
      s_ylo[r.k] = (float)(comp - (hi - acc));
    }
    rb = claim_take(ticket);
  }
}

// Phase 2 (after a barrier): rows with intervals, grouped by interval count,
// add their O(1) interval sums to delta.
template <class S, class XW>
__device__ __forceinline__ void gather_intervals(const RowCtx& c, const S& src, const XW& xw, int32_t r0, uint32_t lmin,
                                                 double* s_yhi, float* s_ylo) {
  const int nesc = c.misc[kNesc];
  const uint32_t nri = (uint32_t)c.misc[kNInt];
  const uint32_t lane = threadIdx.x & 31u;
  uint32_t rb = claim_take(claim_issue(&c.misc[kRoundI]));
  while (rb < nri) {
    const uint32_t ticket = claim_issue(&c.misc[kRoundI]);
    const RowDesc r = round_row(c, src, c.permi, rb + lane, nri, nesc);
    const uint32_t wp = hdr_wp(r.h), wl = hdr_wl(r.h);
    const bool far = hdr_far(r.h);
    const uint32_t ib = (uint32_t)(r0 + (int32_t)r.k - (int32_t)code_bias(wp) - (int32_t)xw.wlo);
    uint32_t off = r.off + (r.rc.nm + r.rc.ns) * wp;
    double acc = 0.0, comp = 0.0;
    const uint32_t ti = __reduce_max_sync(0xffffffffu, r.rc.ni);
    for (uint32_t t = 0; t < ti; ++t) {
      const bool on = t < r.rc.ni;
      const uint32_t a = ib + extract_bits(src, off, wp);
      const uint32_t len = extract_bits(src, off + wp, wl) + lmin;
      double hi = 0.0, lo = 0.0;
      if (on) {
        if (!far) hi = xw.isum_near(a, len, lo);
        else hi = xw.isum((int32_t)a + (int32_t)xw.wlo, len, lo);
      }
      tsum(acc, comp, hi);
      comp += lo;
      off += on ? wp + wl : 0u;
    }
    if (r.act) {
      double hi = s_yhi[r.k], lo = (double)s_ylo[r.k];
      dd_add(hi, lo, acc, comp);
      s_yhi[r.k] = hi;
      s_ylo[r.k] = (float)lo;
    }
    rb = claim_take(ticket);
  }
}

// Heavy rows: one warp per row, lanes stride over the row's codes (fixed
// width, independently addressable), compensated partial sums combined with a
// double-double warp reduction.  Writes the full delta (points + intervals).
template <class S, class XW>
__device__ __forceinline__ void gather_heavy(const RowCtx& c, const S& src, const XW& xw, int32_t r0, uint32_t lmin,
                                             double* s_yhi, float* s_ylo) {
  const int nesc = c.misc[kNesc];
  const uint32_t nh = (uint32_t)c.misc[kNHeavy];
  const uint32_t lane = threadIdx.x & 31u;
  for (;;) {
    uint32_t q = 0;
    if (lane == 0) q = (uint32_t)atomicAdd(&c.misc[kRoundH], 1);
    q = __shfl_sync(0xffffffffu, q, 0);
    if (q >= nh) break;
    const uint32_t k = c.permh[q];
    const uint32_t h = src.w(k);
    const RowCounts rc = row_counts(src, c.B, h, k, nesc);
    const uint32_t wp = hdr_wp(h), wl = hdr_wl(h);
    const int32_t ib = r0 + (int32_t)k - (int32_t)code_bias(wp);
    const uint32_t off0 = c.rowoff[k], np = rc.nm + rc.ns;
    double acc = 0.0, comp = 0.0;
    for (uint32_t t = lane; t < np; t += 32) {
      const double xv = xw.at(ib + (int32_t)extract_bits(src, off0 + t * wp, wp));
      tsum(acc, comp, t < rc.nm ? -xv : xv);
    }
    const uint32_t ioff = off0 + np * wp;
    for (uint32_t t = lane; t < rc.ni; t += 32) {
      const uint32_t o = ioff + t * (wp + wl);
      const int32_t left = ib + (int32_t)extract_bits(src, o, wp);
      const uint32_t len = extract_bits(src, o + wp, wl) + lmin;
      double lo;
      const double hi = xw.isum(left, len, lo);
      tsum(acc, comp, hi);
      comp += lo;
    }
    double hi = acc + comp, lo = comp - (hi - acc);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double uh = __shfl_down_sync(0xffffffffu, hi, o), ul = __shfl_down_sync(0xffffffffu, lo, o);
      dd_add(hi, lo, uh, ul);
    }
    if (lane == 0) {
      s_yhi[k] = hi;
      s_ylo[k] = (float)lo;
    }
  }
}

template <typename XT, typename YT, bool PREFIX, class S, class EPI>
__device__ __forceinline__ void gather_block(RowCtx& rc, const S& src, XWin<XT, PREFIX>& xw, const BvdDims& D,
                                             uint32_t r0, int nesc, double* s_yhi, float* s_ylo, YT* yb, EPI& epi,
                                             const XT (&xpre)[XWin<XT, PREFIX>::kPre]) {
  row_setup(rc, src, nesc, /*split_heavy=*/true);
  xw.stage(D.n, xpre);  // ends with __syncthreads
  gather_heavy(rc, src, xw, (int32_t)r0, D.min_interval, s_yhi, s_ylo);
  gather_points(rc, src, xw, (int32_t)r0, s_yhi, s_ylo);
  __syncthreads();
  gather_intervals(rc, src, xw, (int32_t)r0, D.min_interval, s_yhi, s_ylo);
  __syncthreads();
  chain_and_store(s_yhi, s_ylo, rc, yb, epi, D.max_depth);
}

// PageRank step arguments (shard-relative pointers; see PageRankEpi).
struct PrArgs {
  const uint32_t* deg;
  const double* p_prev;
  double* q_next;
  double* partial;
  const double* dmass;  // device scalar: dangling mass D of the previous iterate (nullptr -> dmass_host)
  double dmass_host;
  double alpha;
  uint32_t n;
  int uniform;
};

template <typename XT, typename YT, bool PR = false>
__global__ void __launch_bounds__(256, 3) bvd_gather_kernel(BvdDev g, const XT* __restrict__ x, YT* __restrict__ y,
                                                          PrArgs pr) {
  extern __shared__ __align__(16) unsigned char smem[];
  const BvdDims& D = g.d;
  const GatherSmem L = gather_smem_layout(D, g.stream_cap_words, sizeof(XT), true);
  const uint32_t bl = blockIdx.x;  // index into this shard's tables
  const uint32_t b = g.block_begin + bl;
  const BvdBlockInfo bi = g.blocks[bl];
  const uint32_t r0 = b * D.block_rows;
  const uint32_t nr = min(D.block_rows, D.n - r0);

  RowCtx rc = carve_rows(smem, L.rows, D.block_rows, nr);
  uint32_t* s_stream = reinterpret_cast<uint32_t*>(smem);
  const bool staged = stage_stream_begin(g, bi, s_stream, rc.bar);
  XWin<XT, true> xw;
  xw.carve(smem + L.off_x, D.window);
  xw.x = x;
  xw.wlo = bi.wlo;
  XT xpre[XWin<XT, true>::kPre];
  xw.prefetch(D.n, xpre);  // in flight across the stream wait and row setup
  __syncthreads();         // publishes the mbarrier init
  mbar_wait(rc.bar, 0);

  double* s_yhi = reinterpret_cast<double*>(smem + L.off_yhi);
  float* s_ylo = reinterpret_cast<float*>(smem + L.off_ylo);
  YT* yb = y + (r0 - g.row_begin);
  if constexpr (PR) {
    const uint32_t sh = r0 - g.row_begin;
    PageRankEpi epi;
    epi.deg = pr.deg + sh;
    epi.p_prev = pr.p_prev ? pr.p_prev + sh : nullptr;
    epi.q_next = pr.q_next + sh;
    epi.partial = pr.partial;
    epi.base = pr.alpha / (double)pr.n;
    epi.scale = 1.0 - pr.alpha;
    const double dm = pr.dmass ? *pr.dmass : pr.dmass_host;
    epi.dn = pr.uniform ? dm / (double)pr.n : 0.0;
    epi.bl = bl;
    epi.dang = 0.0;
    epi.l1 = 0.0;
    if (staged) {
      const Src<true> src{smem_u32(s_stream)};
      gather_block<XT, YT, true>(rc, src, xw, D, r0, (int)bi.nesc, s_yhi, s_ylo, yb, epi, xpre);
    } else {
      const Src<false> src{g.words + bi.word_offset};
      gather_block<XT, YT, true>(rc, src, xw, D, r0, (int)bi.nesc, s_yhi, s_ylo, yb, epi, xpre);
    }
  } else {
    PlainEpi epi;
    if (staged) {  // CTA-uniform
      const Src<true> src{smem_u32(s_stream)};
      gather_block<XT, YT, true>(rc, src, xw, D, r0, (int)bi.nesc, s_yhi, s_ylo, yb, epi, xpre);
    } else {
      const Src<false> src{g.words + bi.word_offset};
      gather_block<XT, YT, true>(rc, src, xw, D, r0, (int)bi.nesc, s_yhi, s_ylo, yb, epi, xpre);
    }
  }
}

}  // namespace cmvg
