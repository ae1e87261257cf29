// bvs_matmat: Y = A X for X of shape n x k (row-major fp32, leading dimension
// ld), BASELINE.json config 5 (k = 16): the multi-vector extension of the
// reference's single-vector product (ref_matvec.hpp:20-31) on the BV-S slices
// of the gather (host/layout.hpp), so decoding is amortised over the columns.
//
// One CTA (256 threads, two per SM: 113 KB of shared memory) per chain-closed
// block, columns in chunks of KC = 8 (one launch per chunk; the block's stream
// is re-read per chunk):
//   1. the X rows of the block's x-window (this column chunk) are staged in
//      shared memory with coalesced 16-byte loads;
//   2. warps claim heavy rows, then slices; a lane owns one unit and
//      accumulates its KC columns in fp64 registers.  A near point code reads
//      its X row chunk from shared memory (2 x 16-byte loads, 8 DFMA), far codes from
//      global memory; an interval sums its X rows; minus codes subtract.
//      Multi slices combine a row's lanes with a segmented shuffle reduction;
//   3. the deltas D_i (KC fp64 per row) sit in shared memory; after one
//      barrier every (row, column) walks the row's ancestors,
//      Y_i = D_i + D_p1 + D_p2 + D_p3 (R = 3; the whole chain when unbounded),
//      and stores Y.
// fp64 accumulation keeps the fp32 outputs within 1e-5 of the fp64 oracle
// whatever the cancellation in the differential rows.
#pragma once
#include <cstdint>
#include <type_traits>

#include "bvd_common.cuh"
#include "bvs_gather.cuh"

namespace cmvg {

// Columns per pass and the staging type: KC = 8 columns staged as fp32 (the
// fp32 -> fp64 conversions then run per use, on the XU pipe), or KC = 4
// columns staged as fp64 (converted once per staged row; twice the passes,
// no conversions in the decode).  Both stage 32 bytes per window row.  KC = 8
// is the default: at the C5 shape (n = 2^24, k = 16) it measured 3.03 ms
// against 4.60 ms for KC = 4 -- the per-pass decode costs more than the
// conversions it would save.
#ifndef CMVG_MM_COLS
#define CMVG_MM_COLS 8
#endif
constexpr uint32_t kMmCols = CMVG_MM_COLS;
using MmStage = typename std::conditional<kMmCols == 4, double, float>::type;
static_assert(kMmCols * sizeof(MmStage) == 32, "32-byte staged rows");

struct BvsMmSmem {
  uint32_t off_x, off_d, off_ref, off_misc, total;
};

__host__ __device__ inline BvsMmSmem bvs_mm_smem_layout(const BvdDims& d) {
  BvsMmSmem s;
  uint32_t o = 0;
  s.off_x = o;  // [W][KC] MmStage: the X rows of the block's window, this column chunk
  o = align16(o + d.window * 32u);
  s.off_d = o;  // [B][KC] fp64 deltas
  o = align16(o + d.block_rows * kMmCols * 8);
  s.off_ref = o;  // 4-bit reference distances
  o = align16(o + d.block_rows / 2);
  s.off_misc = o;
  o = align16(o + 64);
  s.total = o;
  return s;
}

struct MmCtx {
  const float* __restrict__ X;  // column chunk base (X + c0)
  uint32_t ld, kk;              // leading dimension, columns in this chunk (<= KC)
  bool vec;                     // kk == KC and 16-byte aligned rows: vector loads
  const float4* xs;             // staged window rows (32 bytes each), zero-padded columns
  uint32_t wlo, W;
};

// acc[0..KC) += sgn * X[wlo + j, :] from the staged window.  The fp32 -> fp64
// conversions run on the XU pipe, which bounds this kernel (ncu: XU ~150% of
// its sustained rate); fp64 staging would need 96 KB and one CTA per SM,
// measured slower.
__device__ __forceinline__ void mm_add_near(const MmCtx& m, uint32_t j, bool neg, double (&acc)[kMmCols]) {
  const double sg = neg ? -1.0 : 1.0;
  if constexpr (kMmCols == 4) {
    const double2* r = reinterpret_cast<const double2*>(m.xs + 2 * j);
    const double2 a = r[0], b = r[1];
    const double v[4] = {a.x, a.y, b.x, b.y};
#pragma unroll
    for (uint32_t c = 0; c < 4; ++c) acc[c] = fma(sg, v[c], acc[c]);
  } else {
    const float4 a = m.xs[2 * j], b = m.xs[2 * j + 1];
    const float v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
    for (uint32_t c = 0; c < kMmCols; ++c) acc[c] = fma(sg, (double)v[c], acc[c]);
  }
}

// acc[0..KC) += sgn * X[row, 0..kk) from global memory (far columns)
__device__ __forceinline__ void mm_add_row(const MmCtx& m, uint32_t row, bool neg, double (&acc)[kMmCols]) {
  const float* p = m.X + (size_t)row * m.ld;
  const double sg = neg ? -1.0 : 1.0;
  if (m.vec) {
    float v[8];
    const float4 a = __ldg(reinterpret_cast<const float4*>(p));
    v[0] = a.x, v[1] = a.y, v[2] = a.z, v[3] = a.w;
    if constexpr (kMmCols == 8) {
      const float4 b = __ldg(reinterpret_cast<const float4*>(p) + 1);
      v[4] = b.x, v[5] = b.y, v[6] = b.z, v[7] = b.w;
    }
#pragma unroll
    for (uint32_t c = 0; c < kMmCols; ++c) acc[c] = fma(sg, (double)v[c], acc[c]);
  } else {
#pragma unroll
    for (uint32_t c = 0; c < kMmCols; ++c)
      if (c < m.kk) acc[c] = fma(sg, (double)__ldg(p + c), acc[c]);
  }
}

__device__ __forceinline__ void mm_add_run(const MmCtx& m, uint32_t left, uint32_t len, double (&acc)[kMmCols]) {
  const uint32_t a = left - m.wlo;
  if (a < m.W && a + len <= m.W) {
    for (uint32_t t = 0; t < len; ++t) mm_add_near(m, a + t, false, acc);
  } else {
    for (uint32_t t = 0; t < len; ++t) mm_add_row(m, left + t, false, acc);
  }
}

// reference distances, 4 bits per row (shared memory is at a premium: two CTAs per SM)
__device__ __forceinline__ void mm_set_ref(uint32_t* s_ref, uint32_t k, uint32_t r) {
  if (r) atomicOr(&s_ref[k >> 3], r << (4u * (k & 7u)));
}
__device__ __forceinline__ uint32_t mm_ref(const uint32_t* s_ref, uint32_t k) {
  return (s_ref[k >> 3] >> (4u * (k & 7u))) & 15u;
}

__device__ __forceinline__ void mm_store_delta(double* s_d, uint32_t k, const double (&acc)[kMmCols]) {
  double2* d = reinterpret_cast<double2*>(s_d + (size_t)k * kMmCols);
#pragma unroll
  for (uint32_t c = 0; c < kMmCols; c += 2) d[c / 2] = make_double2(acc[c], acc[c + 1]);
}

template <class S>
__device__ __forceinline__ void mm_heavy(const S& src, const MmCtx& m, int32_t r0, uint32_t lmin, int* misc,
                                         double* s_d, uint32_t* s_ref) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t nh = src.w(0) >> 16, htab = src.w(1), hbase = src.w(2) * 32u;
  for (;;) {
    const uint32_t q = ticket_take(ticket_issue(&misc[kBvsHeavyCtr]));
    if (q >= nh) break;
    const uint32_t e = htab + q * kBvsHeavyEntry;
    const uint32_t sa = src.w(e), nm = src.w(e + 1), ns = src.w(e + 2), ni = src.w(e + 3);
    const uint32_t off0 = hbase + src.w(e + 4);
    const uint32_t k = sa_k(sa), wp = sa_wp(sa), wl = sa_wl(sa);
    const int32_t ib = r0 + (int32_t)k - (int32_t)code_bias(wp);
    const uint32_t np = nm + ns;
    double acc[kMmCols] = {};
    for (uint32_t t = lane; t < np; t += 32)
      mm_add_row(m, (uint32_t)(ib + (int32_t)extract_bits(src, off0 + t * wp, wp)), t < nm, acc);
    const uint32_t ioff = off0 + np * wp;
    for (uint32_t t = 0; t < ni; ++t) {  // intervals: the warp strides over each run
      const uint32_t o = ioff + t * (wp + wl);
      const uint32_t left = (uint32_t)(ib + (int32_t)extract_bits(src, o, wp));
      const uint32_t len = extract_bits(src, o + wp, wl) + lmin;
      for (uint32_t u = lane; u < len; u += 32) mm_add_row(m, left + u, false, acc);
    }
#pragma unroll
    for (uint32_t c = 0; c < kMmCols; ++c) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc[c] += __shfl_down_sync(0xffffffffu, acc[c], o);
    }
    if (lane == 0) {
      mm_store_delta(s_d, k, acc);
      mm_set_ref(s_ref, k, sa_r(sa));
    }
  }
}

__device__ __forceinline__ void mm_slices(const uint32_t* __restrict__ bs, const MmCtx& m, uint32_t wlo, uint32_t W,
                                          uint32_t lmin, int* misc, double* s_d, uint32_t* s_ref) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t nsl = __ldg(bs) & 0xffffu;
  const uint32_t zc = bvs_pad_index(W);  // padding code of near slices
  uint32_t s = ticket_take(ticket_issue(&misc[kBvsSliceCtr]));
  while (s < nsl) {
    const uint32_t next = ticket_issue(&misc[kBvsSliceCtr]);
    const uint32_t* rec = bs + __ldg(bs + kBvsHead + 2 * s);
    const uint32_t meta = __ldg(bs + kBvsHead + 2 * s + 1);
    const uint32_t h = __ldg(rec + 1u + lane);
    const uint32_t* body = rec + 33u + lane;
    const uint32_t mnp = smeta_np(meta), mni = smeta_ni(meta);
    double acc[kMmCols] = {};
    if (!smeta_c32(meta) && !smeta_far(meta)) {
      const uint32_t mnpw = (mnp + 1u) >> 1;
      for (uint32_t q = 0; q < mnpw; ++q) {
        const uint32_t v = __ldg(body + q * 32u);
#pragma unroll
        for (uint32_t half = 0; half < 2; ++half) {
          const uint32_t c = half ? (v & 0xffffu) : (v >> 16);
          if (c != zc) {
            const uint32_t p = c & 0x7fffu;
            mm_add_near(m, p - p / 9u, (c >> 15) != 0, acc);
          }
        }
      }
      for (uint32_t u = 0; u < mni; ++u) {
        const uint32_t v = __ldg(body + (mnpw + u) * 32u);
        for (uint32_t t = 0, a = v >> 16, len = v & 0xffffu; t < len; ++t) mm_add_near(m, a + t, false, acc);
      }
    } else if (!smeta_c32(meta)) {
      const uint32_t nm = uh_nm(h), np = uh_np(h), ni = uh_ni(h);
      const uint32_t base = wlo - kBvsBias16, npw = (np + 1u) >> 1;
      for (uint32_t t = 0; t < mnp; ++t) {
        if (t < np) {
          const uint32_t v = __ldg(body + (t >> 1) * 32u);
          mm_add_row(m, base + ((t & 1u) ? (v & 0xffffu) : (v >> 16)), t < nm, acc);
        }
      }
      for (uint32_t u = 0; u < mni; ++u) {
        if (u < ni) {
          const uint32_t v = __ldg(body + (npw + u) * 32u);
          mm_add_run(m, base + (v >> 16), (v & 0xffffu) + lmin, acc);
        }
      }
    } else {
      const uint32_t nm = uh_nm(h), np = uh_np(h), ni = uh_ni(h);
      for (uint32_t t = 0; t < mnp; ++t)
        if (t < np) mm_add_row(m, __ldg(body + t * 32u), t < nm, acc);
      for (uint32_t u = 0; u < mni; ++u)
        if (u < ni) mm_add_run(m, __ldg(body + (np + 2u * u) * 32u), __ldg(body + (np + 2u * u + 1u) * 32u) + lmin, acc);
    }
    if (smeta_multi(meta)) {
      const uint32_t heads = __ballot_sync(0xffffffffu, uh_primary(h));
      const uint32_t above = heads & ~((2u << lane) - 1u);
      const uint32_t end = above ? (uint32_t)__ffs(above) - 2u : 31u;
      const uint32_t rounds = smeta_rounds(meta);
#pragma unroll
      for (uint32_t i = 0; i < 5; ++i) {
        if (i >= rounds) break;  // warp-uniform
        const uint32_t o = 1u << i;
#pragma unroll
        for (uint32_t c = 0; c < kMmCols; ++c) {
          const double u = __shfl_down_sync(0xffffffffu, acc[c], o);
          if (lane + o <= end) acc[c] += u;
        }
      }
    }
    if (uh_primary(h)) {
      const uint32_t k = uh_k(h);
      mm_store_delta(s_d, k, acc);
      mm_set_ref(s_ref, k, uh_r(h));
    }
    s = ticket_take(next);
  }
}

__global__ void __launch_bounds__(512, 2) bvs_matmat_kernel(BvdDev g, const float* __restrict__ X,
                                                             float* __restrict__ Y, uint32_t ld, uint32_t kk) {
  extern __shared__ __align__(16) unsigned char smem[];
  const BvdDims& D = g.d;
  const BvsMmSmem L = bvs_mm_smem_layout(D);
  const uint32_t T = blockDim.x, tid = threadIdx.x;
  const uint32_t bl = blockIdx.x;
  const uint32_t b = g.block_begin + bl;
  const BvdBlockInfo bi = g.blocks[bl];
  const uint32_t r0 = b * D.block_rows;
  const uint32_t nr = min(D.block_rows, D.n - r0);
  const uint32_t* bs = g.words + bi.word_offset;
  double* s_d = reinterpret_cast<double*>(smem + L.off_d);
  uint32_t* s_ref = reinterpret_cast<uint32_t*>(smem + L.off_ref);  // 4-bit entries, 8 rows per word
  int* misc = reinterpret_cast<int*>(smem + L.off_misc);
  if (tid == 0) {
    misc[kBvsHeavyCtr] = 0;
    misc[kBvsSliceCtr] = 0;
  }
  for (uint32_t w = tid; w < D.block_rows / 8u; w += T) s_ref[w] = 0u;
  if (tid == 32) bulk_prefetch_l2(bs, bi.nwords * 4u);
  __syncthreads();
  MmCtx m;
  m.X = X;
  m.ld = ld;
  m.kk = kk;
  m.vec = kk == kMmCols && (ld % 4u) == 0 && ((reinterpret_cast<uintptr_t>(X) & 15u) == 0);
  m.wlo = bi.wlo;
  m.W = D.window;
  {  // stage the window's X rows (this column chunk), coalesced; columns >= kk and rows >= n are 0
    float4* xs = reinterpret_cast<float4*>(smem + L.off_x);
    m.xs = xs;
    if constexpr (kMmCols == 4) {  // one 16-byte fp32 load per row, stored as 4 fp64 (32 bytes)
      for (uint32_t e = tid; e < D.window; e += T) {
        const uint32_t row = bi.wlo + e;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (row < D.n) {
          const float* p = X + (size_t)row * ld;
          if (m.vec) {
            v = __ldg(reinterpret_cast<const float4*>(p));
          } else {
            if (0 < kk) v.x = __ldg(p + 0);
            if (1 < kk) v.y = __ldg(p + 1);
            if (2 < kk) v.z = __ldg(p + 2);
            if (3 < kk) v.w = __ldg(p + 3);
          }
        }
        double2* d = reinterpret_cast<double2*>(xs + 2 * e);
        d[0] = make_double2(v.x, v.y);
        d[1] = make_double2(v.z, v.w);
      }
    } else {
      for (uint32_t e = tid; e < 2u * D.window; e += T) {
        const uint32_t row = bi.wlo + (e >> 1), c0 = (e & 1u) * 4u;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (row < D.n) {
          const float* p = X + (size_t)row * ld + c0;
          if (m.vec) {
            v = __ldg(reinterpret_cast<const float4*>(p));
          } else {
            if (c0 + 0 < kk) v.x = __ldg(p + 0);
            if (c0 + 1 < kk) v.y = __ldg(p + 1);
            if (c0 + 2 < kk) v.z = __ldg(p + 2);
            if (c0 + 3 < kk) v.w = __ldg(p + 3);
          }
        }
        xs[e] = v;
      }
    }
    __syncthreads();
  }
  const Src<false> src{bs};
  mm_heavy(src, m, (int32_t)r0, D.min_interval, misc, s_d, s_ref);
  mm_slices(bs, m, bi.wlo, D.window, D.min_interval, misc, s_d, s_ref);
  __syncthreads();
  // chains: one (row, column) per thread, walking the row's ancestors
  // (<= 3 for bounded chains; the full chain otherwise)
  float* yb = Y + (size_t)(r0 - g.row_begin) * ld;  // Y holds the shard's rows
  for (uint32_t e = tid; e < nr * kMmCols; e += T) {
    const uint32_t k = e / kMmCols, c = e % kMmCols;
    double y = s_d[e];
    uint32_t p = k, r = mm_ref(s_ref, k);
    while (r) {
      p -= r;
      y += s_d[p * kMmCols + c];
      r = mm_ref(s_ref, p);
    }
    if (c < kk) yb[(size_t)k * ld + c] = (float)y;
  }
}

}  // namespace cmvg
