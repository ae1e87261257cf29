// bvt_scatter: y = x A (the left product, reference matvec_ref_left,
// ref_matvec.hpp:37-41) on A's OWN differential rows, with atomic-free
// segmented accumulation (layout: BV-T, host/layout.hpp):
//     x A = sum_k x_k row_k,  row_k = row_{k-r} + plus_k - minus_k
//         = sum_k c_k (plus_k - minus_k),  c_k = x_k + sum_{j: j - r_j = k} c_j
// (the paper's Proposition 1 applied to the transposed product).
//
// Kernel 1 (one CTA per chain-closed block of B rows, 4 CTAs/SM):
//   1. coefficients c_k in double-double by the reference-chain level
//      scheduler run in reverse: the transcoder lists, per chain depth
//      (deepest first), the rows with children and their children masks;
//      each level is one barrier-separated data-parallel step in which a row
//      pulls its children (rows k+1..k+7 referencing it) in a fixed order;
//   2. the block's contributions, grouped by target column by the
//      transcoder, are summed per target with the gather's slice machinery
//      (one target unit per lane, codes k | minus << 15 read c_k from shared
//      memory, TwoSum accumulation, segmented shuffle reduction for targets
//      split over adjacent lanes, whole warps for heavy targets).  Point
//      targets and interval difference entries land in shared memory, far
//      targets in the block's far staging slots;
//   3. the difference entries are prefix-summed (double-double block scan)
//      and added to the point sums: the block's partial y over its window,
//      written densely to a staging buffer.
// Kernel 2 (one CTA per column tile): y_j = the staged partials of the
// blocks whose window covers j, in block order, plus j's far slots in
// (column, slot) order -- a fixed order, so results are deterministic.
// No atomics anywhere (B200's shared-memory fp64 and 64-bit atomics are CAS
// loops).
#pragma once
#include <cstdint>

#include "bvd_common.cuh"

namespace cmvg {

constexpr uint32_t kBvtSliceTab = 128;  // slice-table entries staged in shared memory

struct BvtSmem {
  uint32_t off_ch, off_cl, off_oh, off_ol, off_misc, total;
};

__host__ __device__ inline BvtSmem bvt_smem_layout(uint32_t B, uint32_t W) {
  BvtSmem s;
  uint32_t o = 0;
  s.off_ch = o;
  o = align16(o + (B + 1) * 8);
  s.off_cl = o;
  o = align16(o + (B + 1) * 4);
  s.off_oh = o;
  o = align16(o + 2 * W * 8);
  s.off_ol = o;
  o = align16(o + 2 * W * 4);
  s.off_misc = o;  // 16 ints + warp totals (32 ints) + slice table (kBvtSliceTab x 2 words)
  o = align16(o + 48 * 4 + kBvtSliceTab * 8);
  s.total = o;
  return s;
}
__host__ __device__ inline BvtSmem bvt_smem_layout(const BvdDims& d) { return bvt_smem_layout(d.block_rows, d.window); }

struct BvtOut {
  double* st_hi;  // staging: [block][W] partial y over the block's window
  float* st_lo;
  double* far_hi;  // far staging slots (global slot numbering)
  float* far_lo;
};

__device__ __forceinline__ void bvt_put(uint32_t t, double hi, double lo, uint32_t W2, double* s_oh, float* s_ol,
                                        const BvtOut& o, uint32_t fbase) {
  if (t < W2) {
    s_oh[t] = hi;
    s_ol[t] = (float)lo;
  } else {
    o.far_hi[fbase + t - W2] = hi;
    o.far_lo[fbase + t - W2] = (float)lo;
  }
}

// +(c_hi, c_lo) or -(c_hi, c_lo) of a code k | minus << 15; EXACT = false
// (fp32 x): plain fp64 sums of c_hi (error ~1e-16 x cancellation, far inside
// the fp32 tolerance)
template <bool EXACT = true>
__device__ __forceinline__ void bvt_term(uint32_t code, const double* ch, const float* cl, double& acc, double& comp) {
  const uint32_t k = code & 0x7fffu;
  const int sg = (int)((code << 16) & 0x80000000u);
  const double h = ch[k];
  if constexpr (EXACT) {
    const double l = (double)cl[k];
    tsum(acc, comp, __hiloint2double(__double2hiint(h) ^ sg, __double2loint(h)));
    comp += __hiloint2double(__double2hiint(l) ^ sg, __double2loint(l));
  } else {
    acc += __hiloint2double(__double2hiint(h) ^ sg, __double2loint(h));
  }
}

// A slice's epilogue: segmented reduction of a multi slice (its round count
// from the meta word), then the primary lane stores the target's sum.
__device__ __forceinline__ void bvt_slice_epilogue(uint32_t lane, uint32_t meta, uint32_t h, double hi, double lo,
                                                   uint32_t W2, double* s_oh, float* s_ol, const BvtOut& out,
                                                   uint32_t fbase) {
  if (tmeta_multi(meta)) {
    const uint32_t heads = __ballot_sync(0xffffffffu, (h >> 30) & 1u);
    const uint32_t above = heads & ~((2u << lane) - 1u);
    const uint32_t end = above ? (uint32_t)__ffs(above) - 2u : 31u;
    const uint32_t rounds = tmeta_rounds(meta);
#pragma unroll
    for (uint32_t i = 0; i < 5; ++i) {
      if (i >= rounds) break;  // warp-uniform
      const uint32_t o = 1u << i;
      const double uh = __shfl_down_sync(0xffffffffu, hi, o), ul = __shfl_down_sync(0xffffffffu, lo, o);
      if (lane + o <= end) dd_add(hi, lo, uh, ul);
    }
  }
  if ((h >> 30) == 3u) bvt_put(th_target(h), hi, lo, W2, s_oh, s_ol, out, fbase);
}

// CW, CB, CT: compile-time window, block rows and threads of the specialised
// kernel (0 = read at run time; see GatherShape)
template <typename XT, uint32_t CW = 0, uint32_t CB = 0, uint32_t CT = 0>
__global__ void __launch_bounds__(256, 4) bvt_scatter_kernel(BvdDev g, const XT* __restrict__ x, BvtOut out) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr bool kExact = sizeof(XT) == 8;
  const BvdDims& D = g.d;
  const uint32_t B = CB ? CB : D.block_rows, W = CW ? CW : D.window, W2 = 2u * W;
  const BvtSmem L = bvt_smem_layout(B, W);
  const uint32_t T = CT ? CT : blockDim.x, tid = threadIdx.x, lane = tid & 31u;
  const uint32_t bl = blockIdx.x;
  const uint32_t b = g.block_begin + bl;
  const BvdBlockInfo bi = g.blocks[bl];
  const uint32_t r0 = b * B;
  const uint32_t nr = min(B, D.n - r0);
  const uint32_t* __restrict__ bs = g.words + bi.word_offset;
  double* ch = reinterpret_cast<double*>(smem + L.off_ch);
  float* cl = reinterpret_cast<float*>(smem + L.off_cl);
  double* s_oh = reinterpret_cast<double*>(smem + L.off_oh);
  float* s_ol = reinterpret_cast<float*>(smem + L.off_ol);
  int* misc = reinterpret_cast<int*>(smem + L.off_misc);
  if (tid == 32) bulk_prefetch_l2(bs, bi.nwords * 4u);

  // ---- 1. coefficients ------------------------------------------------------
  constexpr uint32_t kPer = 4;  // rows per thread (block_rows <= 4 x threads): loads first, stores later
  XT xv[kPer];
#pragma unroll
  for (uint32_t q = 0; q < kPer; ++q) {
    const uint32_t k = tid + q * T;
    xv[q] = k < nr ? __ldg(x + r0 + k) : XT(0);
  }
  const uint32_t h0 = __ldg(bs);
  const uint32_t nsl = h0 & 0xffffu, nh = h0 >> 16;
  uint32_t* s_tab = reinterpret_cast<uint32_t*>(misc + 48);  // slice table (offset, meta), when it fits
  // staged without waiting for the slice count (bounded by the block's stream
  // length); used only when nsl <= kBvtSliceTab
  for (uint32_t i = tid; i < 2 * kBvtSliceTab; i += T)
    if (kBvtHead + i < bi.nwords) s_tab[i] = __ldg(bs + kBvtHead + i);
  for (uint32_t j = tid; j < W2; j += T) {
    s_oh[j] = 0.0;
    s_ol[j] = 0.0f;
  }
#pragma unroll
  for (uint32_t q = 0; q < kPer; ++q) {
    const uint32_t k = tid + q * T;
    if (k < nr) {
      ch[k] = (double)xv[q];
      cl[k] = 0.0f;
    }
  }
  for (uint32_t k = kPer * T + tid; k < nr; k += T) {  // block_rows > 4 x threads
    ch[k] = (double)__ldg(x + r0 + k);
    cl[k] = 0.0f;
  }
  for (uint32_t k = nr + tid; k <= B; k += T) {  // the zero coefficient (padding code B) and rows past n
    ch[k] = 0.0;
    cl[k] = 0.0f;
  }
  __syncthreads();
  {  // the transcoder's schedule: per level (deepest first) the rows with
     // children; each pulls its children's c in increasing distance.  Common
     // case (<= 4 levels, <= 2 entries per thread and level): the level
     // bounds and every entry this thread will use are loaded up front in two
     // rounds of independent loads, so the level barriers wait on shared
     // memory only, not on a chain of 2 x levels global-load round trips.
    const uint32_t* cs = bs + __ldg(bs + 4);
    constexpr uint32_t kLv = 4, kPer = 2;
    uint32_t lvs[kLv + 2];
#pragma unroll
    for (uint32_t l = 0; l < kLv + 2; ++l) lvs[l] = __ldg(cs + l);  // nlev, then level starts (stream words)
    const uint32_t nlev = lvs[0];
    const uint32_t* ent = cs + nlev + 2;
    auto pull = [&](uint32_t e) {
      const uint32_t k = e & 1023u;
      uint32_t m = e >> 10;
      double h = ch[k], l = (double)cl[k];
      while (m) {
        const uint32_t r = (uint32_t)__ffs(m);
        m &= m - 1u;
        dd_add(h, l, ch[k + r], (double)cl[k + r]);
      }
      ch[k] = h;
      cl[k] = (float)l;
    };
    bool fast = nlev <= kLv;
#pragma unroll
    for (uint32_t l = 0; l < kLv; ++l)
      if (l < nlev && lvs[l + 2] - lvs[l + 1] > kPer * T) fast = false;
    if (fast) {
      uint32_t pre[kLv][kPer];
#pragma unroll
      for (uint32_t l = 0; l < kLv; ++l)
#pragma unroll
        for (uint32_t j = 0; j < kPer; ++j) {
          const uint32_t i = lvs[l + 1] + tid + j * T;
          pre[l][j] = (l < nlev && i < lvs[l + 2]) ? __ldg(ent + i) : 0xffffffffu;
        }
#pragma unroll
      for (uint32_t l = 0; l < kLv; ++l) {
        if (l >= nlev) break;  // block-uniform
#pragma unroll
        for (uint32_t j = 0; j < kPer; ++j)
          if (pre[l][j] != 0xffffffffu) pull(pre[l][j]);
        __syncthreads();
      }
    } else {
      for (uint32_t lv = 0; lv < nlev; ++lv) {
        const uint32_t e0 = __ldg(cs + 1 + lv), e1 = __ldg(cs + 2 + lv);
        for (uint32_t i = e0 + tid; i < e1; i += T) pull(__ldg(ent + i));
        __syncthreads();
      }
    }
  }

  // ---- 2. per-target segmented sums ---------------------------------------
  const uint32_t fbase = bi.pad[0];
  {  // heavy targets: one warp each, fixed lane order
    const uint32_t htab = __ldg(bs + 1), hcode = __ldg(bs + 2);
    for (uint32_t q = tid >> 5; q < nh; q += T >> 5) {
      const uint32_t e = htab + q * kBvtHeavyEntry;
      const uint32_t t = __ldg(bs + e), ne = __ldg(bs + e + 1), co = hcode + __ldg(bs + e + 2);
      double acc = 0.0, comp = 0.0;
      for (uint32_t i = lane; i < ne; i += 32) {
        const uint32_t w = __ldg(bs + co + (i >> 1));
        bvt_term((i & 1u) ? (w & 0xffffu) : (w >> 16), ch, cl, acc, comp);
      }
      double hi = acc + comp, lo = comp - (hi - acc);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double uh = __shfl_down_sync(0xffffffffu, hi, o), ul = __shfl_down_sync(0xffffffffu, lo, o);
        dd_add(hi, lo, uh, ul);
      }
      if (lane == 0) bvt_put(t, hi, lo, W2, s_oh, s_ol, out, fbase);
    }
  }
  // slices, round-robin (sorted by cost), software-pipelined: a slice's words
  // are loaded into registers, and the previous slice's reduction and store
  // run while those loads are in flight
  bool have_prev = false;
  uint32_t prev_meta = 0, prev_h = 0;
  double prev_hi = 0.0, prev_lo = 0.0;
  for (uint32_t s = tid >> 5; s < nsl; s += T >> 5) {
    uint32_t roff, meta;
    if (nsl <= kBvtSliceTab) {
      roff = s_tab[2 * s];
      meta = s_tab[2 * s + 1];
    } else {
      roff = __ldg(bs + kBvtHead + 2 * s);
      meta = __ldg(bs + kBvtHead + 2 * s + 1);
    }
    const uint32_t* rec = bs + roff;
    const uint32_t h = __ldg(rec + 1u + lane);
    const uint32_t* body = rec + 33u + lane;
    const uint32_t mnw = (tmeta_ne(meta) + 1u) >> 1;
    uint32_t w[kBvtUnitCodes / 2];
#pragma unroll
    for (uint32_t q = 0; q < kBvtUnitCodes / 2; ++q) w[q] = q < mnw ? __ldg(body + q * 32u) : 0u;
    if (have_prev) bvt_slice_epilogue(lane, prev_meta, prev_h, prev_hi, prev_lo, W2, s_oh, s_ol, out, fbase);
    double acc = 0.0, comp = 0.0, acc2 = 0.0, comp2 = 0.0;
#pragma unroll
    for (uint32_t q = 0; q < kBvtUnitCodes / 2; ++q) {
      if (q >= mnw) break;  // warp-uniform
      bvt_term<kExact>(w[q] >> 16, ch, cl, acc, comp);
      bvt_term<kExact>(w[q] & 0xffffu, ch, cl, acc2, comp2);
    }
    tsum(acc, comp, acc2);
    comp += comp2;
    prev_hi = acc + comp;
    prev_lo = comp - (prev_hi - acc);
    prev_h = h;
    prev_meta = meta;
    have_prev = true;
  }
  if (have_prev) bvt_slice_epilogue(lane, prev_meta, prev_h, prev_hi, prev_lo, W2, s_oh, s_ol, out, fbase);
  __syncthreads();

  // ---- 3. window partial = point sums + inclusive prefix of the differences
  // block scan in double-double: per-thread chunk, warp shuffles, warp totals
  const uint32_t per = (W + T - 1) / T, j0 = min(W, tid * per), j1 = min(W, j0 + per);
  double th = 0.0, tl = 0.0;
  for (uint32_t j = j0; j < j1; ++j) dd_add(th, tl, s_oh[W + j], (double)s_ol[W + j]);
  double ih = th, il = tl;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double uh = __shfl_up_sync(0xffffffffu, ih, o), ul = __shfl_up_sync(0xffffffffu, il, o);
    if ((int)lane >= o) dd_add(ih, il, uh, ul);
  }
  double* wtot = reinterpret_cast<double*>(misc + 16);  // 8 warps x (hi, lo)
  const uint32_t warp = tid >> 5, nw = T >> 5;
  if (lane == 31) {
    wtot[2 * warp] = ih;
    wtot[2 * warp + 1] = il;
  }
  __syncthreads();
  double eh = __shfl_up_sync(0xffffffffu, ih, 1), el = __shfl_up_sync(0xffffffffu, il, 1);
  if (lane == 0) eh = el = 0.0;
  for (uint32_t w = 0; w < warp && w < nw; ++w) dd_add(eh, el, wtot[2 * w], wtot[2 * w + 1]);
  double* st_hi = out.st_hi + (size_t)bl * W;
  float* st_lo = out.st_lo + (size_t)bl * W;
  for (uint32_t j = j0; j < j1; ++j) {
    dd_add(eh, el, s_oh[W + j], (double)s_ol[W + j]);  // inclusive prefix of the differences at j
    double a = s_oh[j], c = (double)s_ol[j];
    dd_add(a, c, eh, el);
    st_hi[j] = a;
    st_lo[j] = (float)c;
  }
}

// Kernel 2: combine staged partials per column tile, fixed order.  The
// tile's covering blocks (their window offsets) and its far (column, slot)
// pairs are staged in shared memory first, so a column's sum issues its
// staging loads back to back instead of walking global tables.
constexpr uint32_t kCombCover = 32;   // covering blocks staged per tile
constexpr uint32_t kCombFar = 2048;   // far pairs staged per tile

template <typename YT>
__global__ void __launch_bounds__(256) bvt_combine_kernel(BvdDev g, const uint32_t* __restrict__ tile_ptr,
                                                          const uint32_t* __restrict__ tile_blk,
                                                          const uint32_t* __restrict__ farp_ptr,
                                                          const uint32_t* __restrict__ farp, BvtOut out,
                                                          uint32_t nbl, uint32_t fs0, uint32_t fs1,
                                                          YT* __restrict__ y) {
  __shared__ uint32_t s_bl[kCombCover], s_wlo[kCombCover], s_far[2 * kCombFar];
  __shared__ uint32_t s_nc;
  const BvdDims& D = g.d;
  const uint32_t B = D.block_rows, W = D.window, tid = threadIdx.x;
  const uint32_t t = blockIdx.x;
  const uint32_t c0 = t * B;
  const uint32_t q0 = tile_ptr[t], q1 = tile_ptr[t + 1];
  const uint32_t f0 = farp_ptr[t], f1 = farp_ptr[t + 1];
  const bool staged = q1 - q0 <= kCombCover && f1 - f0 <= kCombFar;
  if (staged) {
    if (tid < 32) {  // this shard's covering blocks, in block order
      const uint32_t q = q0 + tid;
      uint32_t b = 0;
      bool mine = false;
      if (q < q1) {
        b = tile_blk[q];
        mine = b >= g.block_begin && b - g.block_begin < nbl;
      }
      const uint32_t m = __ballot_sync(0xffffffffu, mine);
      if (mine) {
        const uint32_t i = __popc(m & ((1u << tid) - 1u)), bl = b - g.block_begin;
        s_bl[i] = bl;
        s_wlo[i] = g.blocks[bl].wlo;
      }
      if (tid == 0) s_nc = __popc(m);
    }
    for (uint32_t i = tid; i < 2 * (f1 - f0); i += blockDim.x) s_far[i] = farp[2 * f0 + i];
    __syncthreads();
  }
  for (uint32_t j = tid; j < B && c0 + j < D.n; j += blockDim.x) {
    const uint32_t col = c0 + j;
    double hi = 0.0, lo = 0.0;
    uint32_t p0 = 0, pe = 0;
    const uint32_t* fp;
    if (staged) {
      const uint32_t nc = s_nc;
      for (uint32_t i = 0; i < nc; ++i) {
        const uint32_t jj = col - s_wlo[i];
        if (jj < W) {
          const size_t o = (size_t)s_bl[i] * W + jj;
          dd_add(hi, lo, out.st_hi[o], (double)out.st_lo[o]);
        }
      }
      fp = s_far;
      pe = f1 - f0;
    } else {
      for (uint32_t q = q0; q < q1; ++q) {
        const uint32_t b = tile_blk[q];
        if (b < g.block_begin || b - g.block_begin >= nbl) continue;  // another shard's block
        const uint32_t bl = b - g.block_begin;
        const uint32_t jj = col - g.blocks[bl].wlo;
        if (jj < W) dd_add(hi, lo, out.st_hi[(size_t)bl * W + jj], (double)out.st_lo[(size_t)bl * W + jj]);
      }
      fp = farp;
      p0 = f0;
      pe = f1;
    }
    // far slots of this column: pairs sorted by (column, slot)
    uint32_t a = p0, e = pe;
    while (a < e) {
      const uint32_t mid = (a + e) >> 1;
      if (fp[2 * mid] < col) a = mid + 1;
      else e = mid;
    }
    for (uint32_t p = a; p < pe && fp[2 * p] == col; ++p) {
      const uint32_t slot = fp[2 * p + 1];
      if (slot >= fs0 && slot < fs1) dd_add(hi, lo, out.far_hi[slot], (double)out.far_lo[slot]);
    }
    y[col] = (YT)(hi + lo);
  }
}

}  // namespace cmvg
