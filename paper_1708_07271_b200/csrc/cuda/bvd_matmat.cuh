// bvd_matmat: Y = A X for X of shape n x k (row-major fp32), BASELINE.json
// config 5 (k = 16).  The multi-vector extension of the reference's
// single-vector product (ref_matvec.hpp:20-31); decoding is amortised over
// the k columns: a group of G = pow2(k) lanes owns one row, every lane
// decodes the same codes (shared-memory broadcast) and accumulates its own
// column, so each X-row access is one contiguous k*4-byte read.
//
// Per block (chain-closed): TMA-staged stream, row setup (rounds sorted by
// point count), point codes (-/+ X[c, :]), intervals (sum of X rows over
// [left, left+len)), then the level scheduler over chain depth on the k-wide
// deltas kept in shared memory (fp64): Y_i = D_i + Y_{i-r}.
#pragma once
#include <cstdint>

#include "bvd_common.cuh"

namespace cmvg {

struct MatmatSmem {
  uint32_t off_d;
  RowSmem rows;
  uint32_t total;
};

__host__ __device__ inline MatmatSmem matmat_smem_layout(const BvdDims& d, uint32_t stream_cap_words, uint32_t k) {
  MatmatSmem s;
  uint32_t o = align16((stream_cap_words + 8) * 4);
  s.off_d = o;
  o = align16(o + d.block_rows * k * 8);
  s.rows = row_smem_layout(o, d.block_rows);
  s.total = s.rows.total;
  return s;
}

template <class S>
__device__ __forceinline__ void matmat_rows(const RowCtx& c, const S& src, const float* __restrict__ X, uint32_t k,
                                            uint32_t ld, uint32_t G, int32_t r0, uint32_t lmin, double* s_d) {
  const int nesc = c.misc[kNesc];
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t rpw = 32u / G;             // rows per warp per step
  const uint32_t sub = lane / G, col = lane % G;
  const bool colok = col < k;
  for (;;) {
    uint32_t rb = 0;
    if (lane == 0) rb = rpw * (uint32_t)atomicAdd(&c.misc[kRoundP], 1);
    rb = __shfl_sync(0xffffffffu, rb, 0);
    if (rb >= (uint32_t)c.misc[kNPts]) break;
    const uint32_t slot = rb + sub;
    const bool act = slot < (uint32_t)c.misc[kNPts];
    const uint32_t kk = act ? c.perm[slot] : 0u;
    const uint32_t h = act ? src.w(kk) : 0u;
    RowCounts rc{0, 0, 0};
    if (act) rc = row_counts(src, c.B, h, kk, nesc);
    const uint32_t wp = hdr_wp(h), wl = hdr_wl(h);
    const int32_t ib = r0 + (int32_t)kk - (int32_t)code_bias(wp);
    const uint32_t np = rc.nm + rc.ns;
    uint32_t off = act ? c.rowoff[kk] : 0u;
    double acc = 0.0;
    const uint32_t tp = __reduce_max_sync(0xffffffffu, np);
    for (uint32_t t = 0; t < tp; ++t) {
      const bool on = t < np;
      const int32_t cidx = ib + (int32_t)extract_bits(src, off, wp);
      float xv = 0.0f;
      if (on && colok) xv = __ldg(X + (size_t)cidx * ld + col);
      acc += on ? (t < rc.nm ? -(double)xv : (double)xv) : 0.0;
      off += on ? wp : 0u;
    }
    const uint32_t ti = __reduce_max_sync(0xffffffffu, rc.ni);
    for (uint32_t t = 0; t < ti; ++t) {
      if (t < rc.ni) {
        const int32_t left = ib + (int32_t)extract_bits(src, off, wp);
        const uint32_t len = extract_bits(src, off + wp, wl) + lmin;
        if (colok) {
          double s = 0.0;
          const float* px = X + (size_t)left * ld + col;
          for (uint32_t q = 0; q < len; ++q) s += (double)__ldg(px + (size_t)q * ld);
          acc += s;
        }
        off += wp + wl;
      }
    }
    if (act && colok) s_d[kk * k + col] = acc;
  }
}

// Level scheduler on k-wide rows: rows counting-sorted by chain depth,
// one barrier per level, (row, column) pairs spread over all threads.
__device__ __forceinline__ void matmat_chain(double* s_d, RowCtx& c, uint32_t k) {
  const uint32_t T = blockDim.x, tid = threadIdx.x, lane = tid & 31u;
  int* hd = c.hist;
  for (uint32_t q = tid; q < 64; q += T) hd[q] = 0;
  __syncthreads();
  int dmax = 0;
  for (uint32_t q = tid; q < c.nr; q += T) {
    uint32_t d = 0, j = q;
    while (c.ref[j]) {
      j -= c.ref[j];
      ++d;
    }
    c.key[q] = (uint16_t)d;
    dmax = max(dmax, (int)d);
    if (d) atomicAdd(&hd[min(d, 63u)], 1);
  }
  dmax = __reduce_max_sync(0xffffffffu, dmax);
  if (lane == 0 && dmax) atomicMax(&c.misc[1], dmax);
  __syncthreads();
  dmax = c.misc[1];
  if (dmax == 0) return;
  if (tid < 32) {
    const int v0 = hd[2 * lane], v1 = hd[2 * lane + 1];
    int tot;
    const int e2 = warp_excl_scan(v0 + v1, tot);
    hd[2 * lane] = e2;
    hd[2 * lane + 1] = e2 + v0;
    c.wscratch[2 * lane] = e2;
    c.wscratch[2 * lane + 1] = e2 + v0;
  }
  __syncthreads();
  for (uint32_t q = tid; q < c.nr; q += T) {
    const uint32_t d = c.key[q];
    if (d) c.perm[atomicAdd(&hd[min(d, 63u)], 1)] = (uint16_t)q;
  }
  __syncthreads();
  for (int d = 1; d <= min(dmax, 62); ++d) {
    const uint32_t a = (uint32_t)c.wscratch[d], e = (uint32_t)c.wscratch[d + 1];
    for (uint32_t idx = a * k + tid; idx < e * k; idx += T) {
      const uint32_t q = c.perm[idx / k], col = idx % k;
      s_d[q * k + col] += s_d[(q - c.ref[q]) * k + col];
    }
    __syncthreads();
  }
  if (dmax >= 63) {  // very deep chains: in row order, columns in parallel
    for (uint32_t q = 0; q < c.nr; ++q) {
      if (c.key[q] >= 63 && tid < k) s_d[q * k + tid] += s_d[(q - c.ref[q]) * k + tid];
      __syncthreads();
    }
  }
}

// X: n rows of stride ld (columns [0, k) used); Y: rows of stride ld.
__global__ void __launch_bounds__(512) bvd_matmat_kernel(BvdDev g, const float* __restrict__ X, float* __restrict__ Y,
                                                         uint32_t k, uint32_t ld) {
  extern __shared__ __align__(16) unsigned char smem[];
  const BvdDims& D = g.d;
  const MatmatSmem L = matmat_smem_layout(D, g.stream_cap_words, k);
  const uint32_t bl = blockIdx.x;
  const uint32_t b = g.block_begin + bl;
  const BvdBlockInfo bi = g.blocks[bl];
  const uint32_t r0 = b * D.block_rows;
  const uint32_t nr = min(D.block_rows, D.n - r0);
  RowCtx rc = carve_rows(smem, L.rows, D.block_rows, nr);
  uint32_t* s_stream = reinterpret_cast<uint32_t*>(smem);
  const bool staged = stage_stream_begin(g, bi, s_stream, rc.bar);
  __syncthreads();
  mbar_wait(rc.bar, 0);
  double* s_d = reinterpret_cast<double*>(smem + L.off_d);
  uint32_t G = 1;
  while (G < k) G <<= 1;
  if (staged) {
    const Src<true> src{smem_u32(s_stream)};
    row_setup(rc, src, (int)bi.nesc);
    matmat_rows(rc, src, X, k, ld, G, (int32_t)r0, D.min_interval, s_d);
  } else {
    const Src<false> src{g.words + bi.word_offset};
    row_setup(rc, src, (int)bi.nesc);
    matmat_rows(rc, src, X, k, ld, G, (int32_t)r0, D.min_interval, s_d);
  }
  __syncthreads();
  matmat_chain(s_d, rc, k);
  float* yb = Y + (size_t)(r0 - g.row_begin) * ld;
  for (uint32_t idx = threadIdx.x; idx < nr * k; idx += blockDim.x) yb[(size_t)(idx / k) * ld + idx % k] = (float)s_d[idx];
}

}  // namespace cmvg
