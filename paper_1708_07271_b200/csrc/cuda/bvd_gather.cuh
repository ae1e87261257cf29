// bvd_gather: y = A * x^T on the BV-D layout -- the hot path, replacing the
// reference's sequential `matvec_ref_into` (include/cmv/ref_matvec.hpp:20-31,
// SPEC.md:197-205).
//
// One CTA per block of B rows (reference chains never leave a block):
//   1. one thread issues TMA bulk copies of the block's coded stream and of
//      the x-window x[wlo, wlo+W) into shared memory (mbarrier completion);
//   2. [PREFIX] warps build a tile-local (16-entry) exclusive prefix of the
//      window, tile totals and their prefix, so an interval costs O(1);
//   3. every thread decodes its lane: a contiguous, cost-balanced range of
//      rows, computing delta_i = -sum_minus x + sum_intervals x + sum_res x
//      in fp64 (no reference dependency: deltas are independent);
//   4. level phases: rows of chain depth d add y of their reference row,
//      d = 1..max depth (y_i = delta_i + y_{i-r}, the reference's order);
//   5. coalesced store of y.
#pragma once
#include <cstdint>

#include "../host/layout.hpp"
#include "bitreader.cuh"
#include "ptx.cuh"

namespace cmvg {

struct BvdDev {
  const uint32_t* words;
  const BvdBlockInfo* blocks;
  const uint32_t* lanes;
  BvdDims d;
  uint32_t block_begin;  // first block of this shard
  uint32_t row_begin;    // first row of this shard
  uint32_t stream_cap_words;  // blocks with more words decode from global memory
  uint32_t pad;
};

__host__ __device__ inline uint32_t align16(uint32_t v) { return (v + 15u) & ~15u; }

struct GatherSmem {
  uint32_t off_x, off_p, off_tt, off_q, off_y, off_ref, off_dep, off_bar, total;
};

__host__ __device__ inline GatherSmem gather_smem_layout(const BvdDims& d, uint32_t stream_cap_words, uint32_t xsize,
                                                         bool prefix) {
  GatherSmem s;
  uint32_t o = align16((stream_cap_words + 8) * 4);
  s.off_x = o;
  o = align16(o + d.window * xsize + 16);
  s.off_p = o;
  if (prefix) o = align16(o + (d.window + 16) * 8);
  s.off_tt = o;
  if (prefix) o = align16(o + (d.window / 16 + 1) * 8);
  s.off_q = o;
  if (prefix) o = align16(o + (d.window / 16 + 2) * 8);
  s.off_y = o;
  o = align16(o + d.block_rows * 8);
  s.off_ref = o;
  o = align16(o + d.block_rows);
  s.off_dep = o;
  o = align16(o + d.block_rows * 2);
  s.off_bar = o;
  o = align16(o + 16);
  s.total = o;
  return s;
}

template <typename XT, typename YT, bool PREFIX>
__global__ void __launch_bounds__(256) bvd_gather_kernel(BvdDev g, const XT* __restrict__ x, YT* __restrict__ y) {
  extern __shared__ __align__(16) unsigned char smem[];
  const BvdDims& D = g.d;
  const GatherSmem L = gather_smem_layout(D, g.stream_cap_words, sizeof(XT), PREFIX);
  uint32_t* s_stream = reinterpret_cast<uint32_t*>(smem);
  XT* s_x = reinterpret_cast<XT*>(smem + L.off_x);
  double* s_p = reinterpret_cast<double*>(smem + L.off_p);
  double* s_tt = reinterpret_cast<double*>(smem + L.off_tt);
  double* s_q = reinterpret_cast<double*>(smem + L.off_q);
  double* s_y = reinterpret_cast<double*>(smem + L.off_y);
  uint8_t* s_ref = reinterpret_cast<uint8_t*>(smem + L.off_ref);
  uint16_t* s_dep = reinterpret_cast<uint16_t*>(smem + L.off_dep);
  uint64_t* s_bar = reinterpret_cast<uint64_t*>(smem + L.off_bar);
  int* s_dmax = reinterpret_cast<int*>(smem + L.off_bar + 8);

  const uint32_t T = blockDim.x;
  const uint32_t tid = threadIdx.x;
  const uint32_t bl = blockIdx.x;  // index into this shard's tables
  const uint32_t b = g.block_begin + bl;
  const BvdBlockInfo bi = g.blocks[bl];
  const uint32_t r0 = b * D.block_rows;
  const uint32_t nr = min(D.block_rows, D.n - r0);
  const uint32_t W = D.window;
  const uint32_t wlo = bi.wlo;
  const bool staged = bi.nwords <= g.stream_cap_words;
  const uint32_t xvalid = wlo < D.n ? min(W, D.n - wlo) : 0u;
  const uint32_t xtma_bytes = (xvalid * (uint32_t)sizeof(XT)) & ~15u;
  const uint32_t xtma = xtma_bytes / (uint32_t)sizeof(XT);

  if (tid == 0) {
    mbar_init(s_bar, 1);
    *s_dmax = 0;
    uint32_t sbytes = staged ? bi.nwords * 4u : 0u;
    mbar_arrive_expect_tx(s_bar, sbytes + xtma_bytes);
    if (sbytes) bulk_g2s(s_stream, g.words + bi.word_offset, sbytes, s_bar);
    if (xtma_bytes) bulk_g2s(s_x, x + wlo, xtma_bytes, s_bar);
  }
  // window tail (not a 16-byte multiple, or past n) and stream guard words
  for (uint32_t j = xtma + tid; j < W; j += T) s_x[j] = (wlo + j < D.n) ? x[wlo + j] : XT(0);
  if (tid < 8) s_stream[(staged ? bi.nwords : 0u) + tid] = 0u;
  __syncthreads();
  mbar_wait(s_bar, 0);

  if constexpr (PREFIX) {
    // tile-local exclusive prefix (16-entry tiles) with half-warp scans
    const uint32_t lane = tid & 31u, warp = tid >> 5, nwarps = T >> 5;
    for (uint32_t base = warp * 32u; base < W; base += nwarps * 32u) {
      double v = (double)s_x[base + lane];
      double inc = v;
#pragma unroll
      for (int o = 1; o < 16; o <<= 1) {
        double u = __shfl_up_sync(0xffffffffu, inc, o, 16);
        if ((int)(lane & 15u) >= o) inc += u;
      }
      double ex = __shfl_up_sync(0xffffffffu, inc, 1, 16);
      if ((lane & 15u) == 0) ex = 0.0;
      s_p[base + lane] = ex;
      if ((lane & 15u) == 15u) s_tt[(base + lane) >> 4] = inc;
    }
    __syncthreads();
    if (warp == 0) {
      const uint32_t ntiles = W >> 4;
      const uint32_t per = (ntiles + 31u) / 32u;
      double loc = 0.0;
      for (uint32_t t = 0; t < per; ++t) {
        uint32_t k = lane * per + t;
        if (k < ntiles) loc += s_tt[k];
      }
      double inc = loc;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        double u = __shfl_up_sync(0xffffffffu, inc, o);
        if ((int)lane >= o) inc += u;
      }
      double run = __shfl_up_sync(0xffffffffu, inc, 1);
      if (lane == 0) run = 0.0;
      for (uint32_t t = 0; t < per; ++t) {
        uint32_t k = lane * per + t;
        if (k < ntiles) {
          s_q[k] = run;
          run += s_tt[k];
        }
      }
      if (lane == 31) s_q[ntiles] = inc;
    }
    __syncthreads();
  }

  auto X = [&](int32_t c) -> double {
    uint32_t j = (uint32_t)(c - (int32_t)wlo);
    return j < W ? (double)s_x[j] : (double)__ldg(x + c);
  };
  auto ISUM = [&](int32_t left, uint32_t len) -> double {
    uint32_t a = (uint32_t)(left - (int32_t)wlo);
    uint32_t e = a + len;
    double s = 0.0;
    if (a < W && e <= W) {
      if constexpr (PREFIX) {
        uint32_t ta = a >> 4, tb = e >> 4;
        if (ta == tb) return s_p[e] - s_p[a];
        s = s_tt[ta] - s_p[a];
        if (tb > ta + 1) s += s_q[tb] - s_q[ta + 1];
        if (e & 15u) s += s_p[e];
        return s;
      } else {
        for (uint32_t t = a; t < e; ++t) s += (double)s_x[t];
        return s;
      }
    }
    for (uint32_t t = 0; t < len; ++t) s += (double)__ldg(x + left + t);
    return s;
  };

  // ---- decode this thread's lane --------------------------------------------
  const uint32_t rowmask = (1u << D.row_bits) - 1u;
  const uint32_t* ltab = g.lanes + (size_t)bl * T;
  const uint32_t lt = ltab[tid];
  const uint32_t rs = lt & rowmask;
  const uint32_t re = (tid + 1 < T) ? (ltab[tid + 1] & rowmask) : nr;
  if (rs < re) {
    DevBits br;
    br.init(staged ? s_stream : g.words + bi.word_offset, lt >> D.row_bits);
    const int ref_bits = (int)D.ref_bits;
    const uint32_t lmin = D.min_interval;
    for (uint32_t k = rs; k < re; ++k) {
      const int32_t i = (int32_t)(r0 + k);
      const uint32_t r = br.bits(ref_bits);
      double acc = 0.0;
      if (r) {
        uint32_t nm = br.gamma();
        if (nm) {
          int32_t c = i + unfold_i32(br.zeta<3>());
          acc -= X(c);
          for (uint32_t t = 1; t < nm; ++t) {
            c += (int32_t)br.zeta<3>() + 1;
            acc -= X(c);
          }
        }
      }
      uint32_t ni = br.gamma();
      if (ni) {
        int32_t left = i + unfold_i32(br.gamma());
        uint32_t len = br.gamma() + lmin;
        acc += ISUM(left, len);
        int32_t end = left + (int32_t)len;
        for (uint32_t t = 1; t < ni; ++t) {
          left = end + (int32_t)br.gamma() + 1;
          len = br.gamma() + lmin;
          acc += ISUM(left, len);
          end = left + (int32_t)len;
        }
      }
      uint32_t nres = br.gamma();
      if (nres) {
        int32_t c = i + unfold_i32(br.zeta<3>());
        acc += X(c);
        for (uint32_t t = 1; t < nres; ++t) {
          c += (int32_t)br.zeta<3>() + 1;
          acc += X(c);
        }
      }
      s_y[k] = acc;
      s_ref[k] = (uint8_t)r;
    }
  }
  __syncthreads();

  // ---- reference-chain level phases ------------------------------------------
  int dmax = 0;
  for (uint32_t k = tid; k < nr; k += T) {
    uint32_t d = 0, j = k;
    while (s_ref[j]) {
      j -= s_ref[j];
      ++d;
    }
    s_dep[k] = (uint16_t)d;
    dmax = max(dmax, (int)d);
  }
  if (dmax) atomicMax(s_dmax, dmax);
  __syncthreads();
  dmax = *s_dmax;
  for (int d = 1; d <= dmax; ++d) {
    for (uint32_t k = tid; k < nr; k += T)
      if (s_dep[k] == d) s_y[k] += s_y[k - s_ref[k]];
    __syncthreads();
  }
  YT* yb = y + (r0 - g.row_begin);
  for (uint32_t k = tid; k < nr; k += T) yb[k] = (YT)s_y[k];
}

}  // namespace cmvg
