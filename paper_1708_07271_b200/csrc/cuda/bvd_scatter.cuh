// bvd_scatter: y = x A (the left product, reference matvec_ref_left,
// ref_matvec.hpp:37-41) computed on A's OWN BV-D layout, without a transpose:
//     x A = sum_i x_i row_i,  row_i = row_{i-r} + plus_i - minus_i
//         = sum_i c_i (plus_i - minus_i),  c_i = x_i + sum_{k: k - r_k = i} c_k
// (the paper's Proposition 1 applied to the transposed product).
//
// Per block (chain-closed):
//   1. coefficients c_i in double-double by the level scheduler run in
//      reverse: rows at depth d pull c from their children (rows i+1..i+7
//      whose reference is i), deepest level first, fixed child order;
//   2. one row per lane (rounds by point count): point codes add -/+ c_i to a
//      shared-memory window accumulator, intervals add +c_i at left and -c_i
//      at left+len to a difference array (O(1) per interval); far columns go
//      straight to the global accumulators;
//   3. the difference array is prefix-summed into the window and the window
//      is flushed to the global accumulators.
// Accumulators are double-double: every atomic add of hi captures its exact
// rounding error (TwoSum against the returned old value) into lo, so the
// result is accurate to ~1 ulp whatever the order of the adds.  A final pass
// rounds hi + lo to y.
#pragma once
#include <cstdint>

#include "bvd_common.cuh"

namespace cmvg {

struct ScatterSmem {
  uint32_t off_x, off_ch, off_cl, off_yh, off_yl, off_dh, off_dl;
  RowSmem rows;
  uint32_t total;
};

__host__ __device__ inline ScatterSmem scatter_smem_layout(const BvdDims& d, uint32_t stream_cap_words) {
  ScatterSmem s;
  const uint32_t B = d.block_rows, W1 = d.window + 1;
  uint32_t o = align16((stream_cap_words + 8) * 4);
  s.off_x = o;
  o = align16(o + B * 8);
  s.off_ch = o;
  o = align16(o + B * 8);
  s.off_cl = o;
  o = align16(o + B * 8);
  s.off_yh = o;
  o = align16(o + W1 * 8);
  s.off_yl = o;
  o = align16(o + W1 * 8);
  s.off_dh = o;
  o = align16(o + W1 * 8);
  s.off_dl = o;
  o = align16(o + W1 * 8);
  s.rows = row_smem_layout(o, B);
  s.total = s.rows.total;
  return s;
}

// double-double accumulate v = (vh, vl) into (*h, *l) with atomics
__device__ __forceinline__ void dd_atomic_add(double* h, double* l, double vh, double vl) {
  const double old = atomicAdd(h, vh);
  double s, e;
  two_sum(old, vh, s, e);
  atomicAdd(l, e + vl);
}

template <typename XT, class S>
__device__ __forceinline__ void scatter_block(RowCtx& c, const S& src, const BvdDims& D, const BvdBlockInfo& bi,
                                              uint32_t r0, const XT* __restrict__ x, double* s_x, double* ch,
                                              double* cl, double* yh, double* yl, double* dh, double* dl,
                                              double* __restrict__ gy_hi, double* __restrict__ gy_lo) {
  const uint32_t T = blockDim.x, tid = threadIdx.x, lane = tid & 31u;
  const uint32_t nr = c.nr, W = D.window, wlo = bi.wlo;
  row_setup(c, src, (int)bi.nesc);
  // ---- 1. coefficients: depth per row, then levels from the deepest up ----
  int dmax = 0;
  for (uint32_t k = tid; k < nr; k += T) {
    uint32_t d = 0, j = k;
    while (c.ref[j]) {
      j -= c.ref[j];
      ++d;
    }
    c.key[k] = (uint16_t)min(d, 65535u);
    dmax = max(dmax, (int)d);
    ch[k] = s_x[k];
    cl[k] = 0.0;
  }
  dmax = __reduce_max_sync(0xffffffffu, dmax);
  if (lane == 0 && dmax) atomicMax(&c.misc[1], dmax);
  __syncthreads();
  dmax = c.misc[1];
  for (int d = dmax - 1; d >= 0; --d) {
    for (uint32_t k = tid; k < nr; k += T) {
      if (c.key[k] != d) continue;
      double h = ch[k], l = cl[k];
      for (uint32_t r = 1; r <= 7 && k + r < nr; ++r)
        if (c.ref[k + r] == r) dd_add(h, l, ch[k + r], cl[k + r]);
      ch[k] = h;
      cl[k] = l;
    }
    __syncthreads();
  }
  // ---- 2. scatter -----------------------------------------------------------
  for (uint32_t j = tid; j <= W; j += T) {
    yh[j] = 0.0;
    yl[j] = 0.0;
    dh[j] = 0.0;
    dl[j] = 0.0;
  }
  __syncthreads();
  const int nesc = c.misc[kNesc];
  for (;;) {
    const uint32_t rb = next_round(&c.misc[kRoundP]);
    if (rb >= (uint32_t)c.misc[kNPts]) break;
    const uint32_t slot = rb + lane;
    const bool act = slot < (uint32_t)c.misc[kNPts];
    const uint32_t k = act ? c.perm[slot] : 0u;
    const uint32_t h = act ? src.w(k) : 0u;
    RowCounts rc{0, 0, 0};
    if (act) rc = row_counts(src, c.B, h, k, nesc);
    const uint32_t wp = hdr_wp(h), wl = hdr_wl(h);
    const int32_t ib = (int32_t)(r0 + k) - (int32_t)code_bias(wp);
    const double vh = act ? ch[k] : 0.0, vl = act ? cl[k] : 0.0;
    uint32_t off = act ? c.rowoff[k] : 0u;
    const uint32_t np = rc.nm + rc.ns;
    const uint32_t tp = __reduce_max_sync(0xffffffffu, np);
    for (uint32_t t = 0; t < tp; ++t) {
      if (t < np) {
        const int32_t col = ib + (int32_t)extract_bits(src, off, wp);
        const double sh = t < rc.nm ? -vh : vh, sl = t < rc.nm ? -vl : vl;
        const uint32_t j = (uint32_t)(col - (int32_t)wlo);
        if (j < W) dd_atomic_add(yh + j, yl + j, sh, sl);
        else dd_atomic_add(gy_hi + col, gy_lo + col, sh, sl);
        off += wp;
      }
    }
    const uint32_t ti = __reduce_max_sync(0xffffffffu, rc.ni);
    for (uint32_t t = 0; t < ti; ++t) {
      if (t < rc.ni) {
        const int32_t left = ib + (int32_t)extract_bits(src, off, wp);
        const uint32_t len = extract_bits(src, off + wp, wl) + D.min_interval;
        const uint32_t a = (uint32_t)(left - (int32_t)wlo);
        if (a < W && a + len <= W) {
          dd_atomic_add(dh + a, dl + a, vh, vl);
          dd_atomic_add(dh + a + len, dl + a + len, -vh, -vl);
        } else {
          for (uint32_t q = 0; q < len; ++q) dd_atomic_add(gy_hi + left + q, gy_lo + left + q, vh, vl);
        }
        off += wp + wl;
      }
    }
  }
  __syncthreads();
  // ---- 3. prefix of the difference array into the window, then flush -------
  if (tid < 32) {
    const uint32_t per = (W + 31u) / 32u;
    double rh = 0.0, rl = 0.0;
    for (uint32_t q = 0; q < per; ++q) {
      const uint32_t j = lane * per + q;
      if (j < W) dd_add(rh, rl, dh[j], dl[j]);
    }
    double ih = rh, il = rl;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double uh = __shfl_up_sync(0xffffffffu, ih, o), ul = __shfl_up_sync(0xffffffffu, il, o);
      if ((int)lane >= o) dd_add(ih, il, uh, ul);
    }
    double eh = __shfl_up_sync(0xffffffffu, ih, 1), el = __shfl_up_sync(0xffffffffu, il, 1);
    if (lane == 0) eh = el = 0.0;
    for (uint32_t q = 0; q < per; ++q) {
      const uint32_t j = lane * per + q;
      if (j < W) {
        dd_add(eh, el, dh[j], dl[j]);  // inclusive prefix at j
        double a = yh[j], b = yl[j];
        dd_add(a, b, eh, el);
        yh[j] = a;
        yl[j] = b;
      }
    }
  }
  __syncthreads();
  for (uint32_t j = tid; j < W; j += T) {
    const double a = yh[j], b = yl[j];
    if ((a != 0.0 || b != 0.0) && wlo + j < D.n) dd_atomic_add(gy_hi + wlo + j, gy_lo + wlo + j, a, b);
  }
}

template <typename XT>
__global__ void __launch_bounds__(256, 1) bvd_scatter_kernel(BvdDev g, const XT* __restrict__ x,
                                                          double* __restrict__ gy_hi, double* __restrict__ gy_lo) {
  extern __shared__ __align__(16) unsigned char smem[];
  const BvdDims& D = g.d;
  const ScatterSmem L = scatter_smem_layout(D, g.stream_cap_words);
  const uint32_t bl = blockIdx.x;
  const uint32_t b = g.block_begin + bl;
  const BvdBlockInfo bi = g.blocks[bl];
  const uint32_t r0 = b * D.block_rows;
  const uint32_t nr = min(D.block_rows, D.n - r0);
  RowCtx rc = carve_rows(smem, L.rows, D.block_rows, nr);
  uint32_t* s_stream = reinterpret_cast<uint32_t*>(smem);
  const bool staged = stage_stream_begin(g, bi, s_stream, rc.bar);
  double* s_x = reinterpret_cast<double*>(smem + L.off_x);
  for (uint32_t k = threadIdx.x; k < nr; k += blockDim.x) s_x[k] = (double)__ldg(x + r0 + k);
  __syncthreads();
  mbar_wait(rc.bar, 0);
  double* ch = reinterpret_cast<double*>(smem + L.off_ch);
  double* cl = reinterpret_cast<double*>(smem + L.off_cl);
  double* yh = reinterpret_cast<double*>(smem + L.off_yh);
  double* yl = reinterpret_cast<double*>(smem + L.off_yl);
  double* dh = reinterpret_cast<double*>(smem + L.off_dh);
  double* dl = reinterpret_cast<double*>(smem + L.off_dl);
  if (staged) {
    const Src<true> src{smem_u32(s_stream)};
    scatter_block<XT>(rc, src, D, bi, r0, x, s_x, ch, cl, yh, yl, dh, dl, gy_hi, gy_lo);
  } else {
    const Src<false> src{g.words + bi.word_offset};
    scatter_block<XT>(rc, src, D, bi, r0, x, s_x, ch, cl, yh, yl, dh, dl, gy_hi, gy_lo);
  }
}

template <typename YT>
__global__ void dd_round_kernel(const double* __restrict__ hi, const double* __restrict__ lo, YT* __restrict__ y,
                                uint32_t n) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) y[i] = (YT)(hi[i] + lo[i]);
}

}  // namespace cmvg
