// bvs_gather: y = A * x^T on the sliced layout BV-S (host/layout.hpp) -- the
// gather hot path, replacing the reference's sequential `matvec_ref_into`
// (include/cmv/ref_matvec.hpp:20-31), and
// (PR = true) the product + update of one PageRank iteration
// (pagerank.hpp:83-102).
//
// One CTA per block of B rows (reference chains never leave a block), four
// CTAs per SM (no stream staging: ~52 KB of shared memory, 64 registers):
//   1. the block's sliced stream is prefetched into L2 (TMA bulk prefetch)
//      while all threads stage the x-window x[wlo, wlo + W) and its two-level
//      double-double prefix in shared memory;
//   2. warps claim heavy rows dynamically (one warp per row, lanes stride
//      over its fixed-width codes), then take 32-unit slices round-robin (one
//      unit of <= 16 points / <= 2 intervals per lane; the transcoder already
//      dealt units into slices of near-equal work and interleaved their words
//      by lane, so a lane loads its <= 10 words with coalesced 128-B warp
//      loads straight into registers -- no row setup, no staging).  Points
//      (minus -> -x[c], residual -> +x[c]) then intervals (O(1) from the
//      prefix), delta accumulated with TwoSum compensation;
//   3. a barrier, then the reference
//      chains y_i = delta_i + y_{i-r} (ref_matvec.hpp:23-25) and the
//      coalesced store / PageRank epilogue.
#pragma once
#include <cstdint>

#include "bvd_common.cuh"

namespace cmvg {

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
  const uint8_t* push_mask;  // fused halo push (see PageRankEpi); null = none
  double* const* push_dst;
  const double* p0;          // restart distribution (start vector), global rows; null = uniform 1/n
};

constexpr uint32_t kBvsGuardWords = 64;  // zero words after the last block (lanes never read past their unit)

constexpr uint32_t kBvsSliceTab = 128;  // slice-table entries staged in shared memory

struct BvsSmem {
  uint32_t off_x, off_rows, off_ptr, off_tab, off_pref, off_misc, total;
};

__host__ __device__ inline BvsSmem bvs_smem_layout(uint32_t W, uint32_t B, uint32_t xsize) {
  BvsSmem s;
  uint32_t o = 0;
  s.off_x = o;
  o = align16(o + xw_bytes(W, xsize));
  s.off_rows = o;  // RowRec per row: delta and reference distance
  o = align16(o + B * (uint32_t)sizeof(RowRec));
  s.off_ptr = o;  // chain pointers (unbounded chains only)
  o = align16(o + B * 2);
  s.off_tab = o;
  o = align16(o + kBvsSliceTab * 8);
  s.off_pref = o;  // block-table entry of the block `ahead` blocks on (L2 prefetch)
  o = align16(o + 16);
  s.off_misc = o;  // mbarrier (16) + 16 ints + scratch (64 ints)
  o = align16(o + 16 + 64 + 64 * 4);
  s.total = o;
  return s;
}
__host__ __device__ inline BvsSmem bvs_smem_layout(const BvdDims& d, uint32_t xsize) {
  return bvs_smem_layout(d.window, d.block_rows, xsize);
}

// Compile-time shape of the specialised gather kernels (x-window W, block
// rows B, threads T); 0 = read at run time.  The default options
// (W = 1536, B = 1024, T = 256) get the specialised kernel: its shared-memory
// layout, chunking and loop bounds are constants (no address arithmetic
// rematerialised under the 64-register cap).
struct GatherShape {
  uint32_t W, B, T;
};
#ifndef CMVG_DEFAULT_W  // build-time override for A/B experiments
#define CMVG_DEFAULT_W 1536
#endif
constexpr GatherShape kGatherDefault{CMVG_DEFAULT_W, 1024, 256};

__device__ __forceinline__ uint32_t ticket_issue(int* counter) {
  return (threadIdx.x & 31u) == 0 ? (uint32_t)atomicAdd(counter, 1) : 0u;
}
__device__ __forceinline__ uint32_t ticket_take(uint32_t t) { return __shfl_sync(0xffffffffu, t, 0); }

enum BvsMisc : int { kBvsHeavyCtr = 0, kBvsSliceCtr = 1 };

// Heavy rows (more than 32 units): their points are cut into work items of
// kBvsHeavyChunk codes (the transcoder numbers them per block, header word 3
// and heavy-table word 5), taken by any warp through a ticket, lanes striding
// over the item's fixed-width codes; item 0 of a row also sums the row's
// intervals (in-window ones O(1) by their lane, the others by the whole warp,
// coalesced).  Each item's warp-reduced double-double sum goes to its slot in
// g.hpart; bvs_heavy_finish combines a row's items in item order after the
// decode barrier, so a hub row is spread over the CTA and the result does not
// depend on which warp took which item.
template <class S, class XW>
__device__ __forceinline__ void bvs_heavy(const S& src, const XW& xw, int32_t r0, uint32_t lmin, int* misc,
                                          double2* hpart) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t nh = src.w(0) >> 16;
  if (!nh) return;
  const uint32_t htab = src.w(1), hbase = src.w(2) * 32u, ibase = src.w(3);
  const uint32_t el = htab + (nh - 1u) * kBvsHeavyEntry;
  const uint32_t nitems = src.w(el + 5) + heavy_chunks(src.w(el + 1) + src.w(el + 2));
  for (;;) {
    const uint32_t item = ticket_take(ticket_issue(&misc[kBvsHeavyCtr]));
    if (item >= nitems) break;
    uint32_t lo_q = 0, hi_q = nh - 1u;  // the row: last entry whose first item <= item
    while (lo_q < hi_q) {
      const uint32_t mid = (lo_q + hi_q + 1u) >> 1;
      if (src.w(htab + mid * kBvsHeavyEntry + 5) <= item) lo_q = mid;
      else hi_q = mid - 1u;
    }
    const uint32_t e = htab + lo_q * kBvsHeavyEntry;
    const uint32_t sa = src.w(e), nm = src.w(e + 1), ns = src.w(e + 2), ni = src.w(e + 3);
    const uint32_t off0 = hbase + src.w(e + 4), j = item - src.w(e + 5);
    const uint32_t k = sa_k(sa), wp = sa_wp(sa), wl = sa_wl(sa);
    const int32_t ib = r0 + (int32_t)k - (int32_t)code_bias(wp);
    const uint32_t np = nm + ns;
    double acc = 0.0, comp = 0.0;
    const uint32_t t1 = min(np, (j + 1u) * kBvsHeavyChunk);
    for (uint32_t t = j * kBvsHeavyChunk + lane; t < t1; t += 32) {
      const double xv = xw.at(ib + (int32_t)extract_bits(src, off0 + t * wp, wp));
      tsum(acc, comp, t < nm ? -xv : xv);
    }
    if (j == 0) {
      const uint32_t ioff = off0 + np * wp;
      for (uint32_t tb = 0; tb < ni; tb += 32) {
        const uint32_t t = tb + lane;
        const bool on = t < ni;
        int32_t left = 0;
        uint32_t len = 0;
        if (on) {
          const uint32_t o = ioff + t * (wp + wl);
          left = ib + (int32_t)extract_bits(src, o, wp);
          len = extract_bits(src, o + wp, wl) + lmin;
        }
        const uint32_t a = (uint32_t)(left - (int32_t)xw.wlo);
        const bool nearw = on && a < xw.W && a + len <= xw.W;
        if (nearw) {
          double lo;
          const double hi = xw.isum_near(a, len, lo);
          tsum(acc, comp, hi);
          comp += lo;
        }
        uint32_t m = __ballot_sync(0xffffffffu, on && !nearw);
        while (m) {
          const int sl = __ffs(m) - 1;
          m &= m - 1u;
          const int32_t L = __shfl_sync(0xffffffffu, left, sl);
          const uint32_t N = __shfl_sync(0xffffffffu, len, sl);
          for (uint32_t e2 = lane; e2 < N; e2 += 32) tsum(acc, comp, xw.at(L + (int32_t)e2));
        }
      }
    }
    double hi = acc + comp, lo = comp - (hi - acc);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double uh = __shfl_down_sync(0xffffffffu, hi, o), ul = __shfl_down_sync(0xffffffffu, lo, o);
      dd_add(hi, lo, uh, ul);
    }
    if (lane == 0) hpart[ibase + item] = make_double2(hi, lo);
  }
}

// After the decode barrier: each heavy row's items, combined in item order
// (one thread per heavy row), become the row's record.  Block-uniform: only
// blocks with heavy rows take the extra barrier.
template <class S>
__device__ __forceinline__ void bvs_heavy_finish(const S& src, const double2* hpart, RowRec* s_rows, uint32_t T) {
  const uint32_t nh = src.w(0) >> 16;
  if (!nh) return;
  const uint32_t htab = src.w(1), ibase = src.w(3);
  for (uint32_t q = threadIdx.x; q < nh; q += T) {
    const uint32_t e = htab + q * kBvsHeavyEntry;
    const uint32_t sa = src.w(e), i0 = ibase + src.w(e + 5);
    const uint32_t nit = heavy_chunks(src.w(e + 1) + src.w(e + 2));
    double hi = 0.0, lo = 0.0;
    for (uint32_t i = 0; i < nit; ++i) {
      const double2 v = hpart[i0 + i];
      dd_add(hi, lo, v.x, v.y);
    }
    put_row(s_rows, sa_k(sa), hi, lo, sa_r(sa));
  }
  __syncthreads();
}

// +x, or -x for t < nm (minus codes come first): flip the sign bit when t - nm < 0
__device__ __forceinline__ double signed_term(double x, uint32_t t, uint32_t nm) {
  const uint32_t m = (t - nm) & 0x80000000u;
  return __hiloint2double(__double2hiint(x) ^ (int)m, __double2loint(x));
}

// A slice's epilogue: segmented reduction of a multi slice, then the primary
// lane writes delta_i and r_i.
__device__ __forceinline__ void bvs_slice_epilogue(uint32_t lane, uint32_t meta, uint32_t h, double hi, double lo,
                                                   RowRec* s_rows) {
  if (smeta_multi(meta)) {
    // a row's units sit in adjacent lanes starting at its primary: segmented
    // suffix reduction so the primary lane ends with the row's delta
    const uint32_t heads = __ballot_sync(0xffffffffu, uh_primary(h));
    const uint32_t above = heads & ~((2u << lane) - 1u);
    const uint32_t end = above ? (uint32_t)__ffs(above) - 2u : 31u;
    const uint32_t rounds = smeta_rounds(meta);  // ceil(log2(most units of a row)): often 1
#pragma unroll
    for (uint32_t i = 0; i < 5; ++i) {
      if (i >= rounds) break;  // warp-uniform
      const uint32_t o = 1u << i;
      const double uh = __shfl_down_sync(0xffffffffu, hi, o), ul = __shfl_down_sync(0xffffffffu, lo, o);
      if (lane + o <= end) dd_add(hi, lo, uh, ul);
    }
  }
  if (uh_primary(h)) put_row(s_rows, uh_k(h), hi, lo, uh_r(h));
}

// Slices: one unit (<= 16 points, <= 2 intervals of one row) per lane; in
// "multi" slices a row's units occupy adjacent lanes and are combined by a
// segmented warp reduction.  `bs` is the block's stream in global memory.
template <bool DYN, class XW>
__device__ __forceinline__ void bvs_slices(const uint32_t* __restrict__ bs, const XW& xw, uint32_t lmin, int* misc,
                                           RowRec* s_rows, const uint32_t* s_tab, uint32_t T) {
  constexpr bool kExact = sizeof(typename XW::value_type) == 8;  // compensated point sums for fp64 x
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t nsl = __ldg(bs) & 0xffffu;
  bool have_prev = false;
  uint32_t prev_meta = 0, prev_h = 0;
  double prev_hi = 0.0, prev_lo = 0.0;
  // static schedule: with kBvsWarps warps each takes the contiguous table
  // range the transcoder's LPT assignment gave it (header words 4..8), else
  // round-robin; no ticket round trip sits in front of a slice's loads
  // Blocks with heavy rows (DYN) take slices dynamically: a warp still busy
  // with a hub row must not hold a static share of the slices (C4's
  // power-law rows); the others use the transcoder's static LPT ranges.
  const uint32_t nwarp = T >> 5, warp = threadIdx.x >> 5;
  constexpr bool dyn = DYN;
  uint32_t s = warp, s_end = nsl, step = nwarp;
  if (dyn) {
    s = ticket_take(ticket_issue(&misc[kBvsSliceCtr]));
  } else if (nwarp == kBvsWarps) {
    const uint16_t* starts = reinterpret_cast<const uint16_t*>(bs + kBvsWarpTab);
    s = __ldg(starts + warp);
    s_end = __ldg(starts + warp + 1);
    step = 1;
  }
  while (s < s_end) {
    const uint32_t tk = dyn ? ticket_issue(&misc[kBvsSliceCtr]) : 0u;  // the next ticket, one slice ahead
    const uint32_t next = s + step;
    // slice table entry from shared memory (staged per block) when it fits:
    // header, meta and body words then come in one round of global loads
    uint32_t roff, meta;
    if (nsl <= kBvsSliceTab) {
      roff = s_tab[2 * s];
      meta = s_tab[2 * s + 1];
    } else {
      roff = __ldg(bs + kBvsHead + 2 * s);
      meta = __ldg(bs + kBvsHead + 2 * s + 1);
    }
    const uint32_t* rec = bs + roff;
    const uint32_t h = __ldg(rec + 1u + lane);
    const uint32_t* body = rec + 33u + lane;  // this lane's word q at body[32 q]
    const uint32_t mnp = smeta_np(meta), mni = smeta_ni(meta);
    double acc = 0.0, comp = 0.0;
    if (!smeta_c32(meta) && !smeta_far(meta)) {
      // near class 16 (rectangular): no per-lane counts -- pad codes read the
      // window's zero entry, empty intervals have length 0
      const uint32_t mnpw = (mnp + 1u) >> 1;
      // exactly mnpw point words (warp-uniform): a jump into the unrolled
      // loads instead of eight predicated ones; words past mnpw are never read
      uint32_t w[kBvsUnitPts / 2];
      static_assert(kBvsUnitPts / 2 <= 16, "unrolled loads");
#define CMVG_LD(q) \
  case q + 1:      \
    if (q < kBvsUnitPts / 2) w[q] = __ldg(body + (q)*32u); /* fall through */
      switch (mnpw) {
        default:
          CMVG_LD(15) CMVG_LD(14) CMVG_LD(13) CMVG_LD(12) CMVG_LD(11) CMVG_LD(10) CMVG_LD(9) CMVG_LD(8) CMVG_LD(7)
          CMVG_LD(6) CMVG_LD(5) CMVG_LD(4) CMVG_LD(3) CMVG_LD(2) CMVG_LD(1) CMVG_LD(0)
        case 0:
          break;
      }
#undef CMVG_LD
      const uint32_t wi0 = mni > 0 ? __ldg(body + mnpw * 32u) : 0u;
      const uint32_t wi1 = mni > 1 ? __ldg(body + (mnpw + 1u) * 32u) : 0u;
      if (have_prev) {  // the previous slice's epilogue while these loads are in flight
        bvs_slice_epilogue(lane, prev_meta, prev_h, prev_hi, prev_lo, s_rows);
        have_prev = false;
      }
      double acc2 = 0.0, comp2 = 0.0;
#pragma unroll
      for (uint32_t q = 0; q < kBvsUnitPts / 2; ++q) {
        if (q >= mnpw) break;  // warp-uniform
        const uint32_t v = w[q];
        const double x0 = xw.at_padded((v >> 16) & 0x7fffu), x1 = xw.at_padded(v & 0x7fffu);
        // minus codes: flip the sign bit (bit 15 of each code)
        // fp64 x: TwoSum, not plain adds: plain fp64 here measured 1.7e-11
        // relative error on C2 (rows whose copy list cancels most of the
        // reference row)
        const double t0 = __hiloint2double(__double2hiint(x0) ^ (int)(v & 0x80000000u), __double2loint(x0));
        const double t1 = __hiloint2double(__double2hiint(x1) ^ (int)((v << 16) & 0x80000000u), __double2loint(x1));
        if constexpr (kExact) {
          tsum(acc, comp, t0);
          tsum(acc2, comp2, t1);
        } else {  // fp32 x: plain fp64 sums (error ~1e-16 x cancellation, far inside the fp32 tolerance)
          acc += t0;
          acc2 += t1;
        }
      }
      tsum(acc, comp, acc2);
      comp += comp2;
      if (mni > 0) {
        double lo;
        const double hi = xw.isum_near(wi0 >> 16, wi0 & 0xffffu, lo);
        tsum(acc, comp, hi);
        comp += lo;
      }
      if (mni > 1) {
        double lo;
        const double hi = xw.isum_near(wi1 >> 16, wi1 & 0xffffu, lo);
        tsum(acc, comp, hi);
        comp += lo;
      }
    } else if (!smeta_c32(meta)) {
      // far class 16: biased 16-bit codes, bounds-checked; words loaded up front
      const uint32_t nm = uh_nm(h), np = uh_np(h), ni = uh_ni(h);
      const int32_t base = (int32_t)xw.wlo - (int32_t)kBvsBias16;
      const uint32_t npw = (np + 1u) >> 1;
      uint32_t w[kBvsUnitPts / 2];
#pragma unroll
      for (uint32_t q = 0; q < kBvsUnitPts / 2; ++q) w[q] = q < npw ? __ldg(body + q * 32u) : 0u;
      const uint32_t wi0 = ni > 0 ? __ldg(body + npw * 32u) : 0u;
      const uint32_t wi1 = ni > 1 ? __ldg(body + (npw + 1u) * 32u) : 0u;
#pragma unroll
      for (uint32_t q = 0; q < kBvsUnitPts / 2; ++q) {
        const uint32_t t = 2u * q;
        if (t >= mnp) break;  // warp-uniform
        const double x0 = t < np ? xw.at(base + (int32_t)(w[q] >> 16)) : 0.0;
        const double x1 = t + 1u < np ? xw.at(base + (int32_t)(w[q] & 0xffffu)) : 0.0;
        if constexpr (kExact) {
          tsum(acc, comp, signed_term(x0, t, nm));
          tsum(acc, comp, signed_term(x1, t + 1u, nm));
        } else {
          acc += signed_term(x0, t, nm) + signed_term(x1, t + 1u, nm);
        }
      }
#pragma unroll
      for (uint32_t u = 0; u < kBvsUnitInts; ++u) {
        if (u >= mni) break;
        const uint32_t v = u ? wi1 : wi0;
        double hi = 0.0, lo = 0.0;
        if (u < ni) hi = xw.isum(base + (int32_t)(v >> 16), (v & 0xffffu) + lmin, lo);
        tsum(acc, comp, hi);
        comp += lo;
      }
    } else {  // class 32: absolute columns, bounds-checked; 8 columns, then their 8 x loads, in flight together
      const uint32_t nm = uh_nm(h), np = uh_np(h), ni = uh_ni(h);
      for (uint32_t t0 = 0; t0 < mnp; t0 += 8) {
        uint32_t c[8];
#pragma unroll
        for (uint32_t j = 0; j < 8; ++j) c[j] = t0 + j < np ? __ldg(body + (t0 + j) * 32u) : 0u;
        double xv[8];
#pragma unroll
        for (uint32_t j = 0; j < 8; ++j) xv[j] = t0 + j < np ? xw.at((int32_t)c[j]) : 0.0;
#pragma unroll
        for (uint32_t j = 0; j < 8; ++j) {
          if constexpr (kExact) tsum(acc, comp, signed_term(xv[j], t0 + j, nm));
          else acc += signed_term(xv[j], t0 + j, nm);
        }
      }
      for (uint32_t u = 0; u < mni; ++u) {
        double hi = 0.0, lo = 0.0;
        if (u < ni)
          hi = xw.isum((int32_t)__ldg(body + (np + 2u * u) * 32u), __ldg(body + (np + 2u * u + 1u) * 32u) + lmin, lo);
        tsum(acc, comp, hi);
        comp += lo;
      }
    }
    // this slice's epilogue runs after the next slice's loads are issued (it
    // hides their latency): keep its state
    if (have_prev) bvs_slice_epilogue(lane, prev_meta, prev_h, prev_hi, prev_lo, s_rows);
    prev_hi = acc + comp;
    prev_lo = comp - (prev_hi - acc);
    prev_h = h;
    prev_meta = meta;
    have_prev = true;
    s = dyn ? ticket_take(tk) : next;
  }
  if (have_prev) bvs_slice_epilogue(lane, prev_meta, prev_h, prev_hi, prev_lo, s_rows);
}

template <typename XT, typename YT, bool PR = false, uint32_t CW = 0, uint32_t CB = 0, uint32_t CT = 0>
#ifndef CMVG_GATHER_MINB  // CTAs per SM the register budget is sized for (build-time A/B)
#define CMVG_GATHER_MINB 4
#endif
__global__ void __launch_bounds__(256, CMVG_GATHER_MINB) bvs_gather_kernel(BvdDev g, const XT* __restrict__ x, const XT* xfar,
                                                             YT* __restrict__ y, PrArgs pr) {
  extern __shared__ __align__(16) unsigned char smem[];
  const BvdDims& D = g.d;
  const uint32_t W = CW ? CW : D.window, B = CB ? CB : D.block_rows, T = CT ? CT : blockDim.x;
  const BvsSmem L = bvs_smem_layout(W, B, sizeof(XT));
  const uint32_t bl = blockIdx.x;  // index into this shard's tables
  const uint32_t b = g.block_begin + bl;
  const BvdBlockInfo bi = g.blocks[bl];
  const uint32_t r0 = b * B;
  const uint32_t nr = min(B, D.n - r0);

  int* misc = reinterpret_cast<int*>(smem + L.off_misc + 16);
  const uint32_t* bs = g.words + bi.word_offset;  // this block's stream (global; read through L1/L2)
  if (threadIdx.x == 0) {
    misc[kBvsHeavyCtr] = 0;
    misc[kBvsSliceCtr] = 0;
  }
  // L2 prefetch a launch-wide wave ahead: this CTA fetches (cp.async, no
  // register or stall) the table entry of block bl + ahead -- about the block
  // whose CTA takes this slot when this one retires -- and after its decode
  // issues bulk L2 prefetches of that block's stream and x-window, so the
  // later CTA's dependent setup loads hit L2.
  BvdBlockInfo* s_pref = reinterpret_cast<BvdBlockInfo*>(smem + L.off_pref);
  const bool ahead = g.ahead && bl + g.ahead < g.nlaunch;
  if (threadIdx.x == 32) {
    bulk_prefetch_l2(bs, bi.nwords * 4u);
    if (ahead) cp_async<16>(s_pref, g.blocks + bl + g.ahead);
  }
  uint32_t* s_tab = reinterpret_cast<uint32_t*>(smem + L.off_tab);
  // the first kBvsSliceTab table entries, staged without waiting for the
  // slice count (bounded by the block's stream length instead, which the
  // block-table entry already gave): one dependent global round trip fewer
  // at the CTA's start; used only when the block has <= kBvsSliceTab slices
  for (uint32_t i = threadIdx.x; i < 2 * kBvsSliceTab; i += T)
    if (kBvsHead + i < bi.nwords) s_tab[i] = __ldg(bs + kBvsHead + i);
  XWin<XT> xw;
  xw.carve(smem + L.off_x, W, T);
  xw.x = x;
  xw.xfar = xfar;
  xw.wlo = bi.wlo;
  XT xpre[XWin<XT>::kPre];
  xw.prefetch(D.n, xpre);
  __syncthreads();      // publishes the counters
  xw.stage(D.n, xpre);  // ends with __syncthreads

  RowRec* s_rows = reinterpret_cast<RowRec*>(smem + L.off_rows);
  const Src<false> src{bs};
  bvs_heavy(src, xw, (int32_t)r0, D.min_interval, misc, g.hpart);
  if (__ldg(bs) >> 16)  // heavy rows in this block: slices dynamically
    bvs_slices<true>(bs, xw, D.min_interval, misc, s_rows, s_tab, T);
  else
    bvs_slices<false>(bs, xw, D.min_interval, misc, s_rows, s_tab, T);
  __syncthreads();
  bvs_heavy_finish(src, g.hpart, s_rows, T);
  if (threadIdx.x == 32 && ahead) {
    cp_async_wait_all();
    const uint64_t wo = s_pref->word_offset;
    const uint32_t nw = s_pref->nwords, wl = s_pref->wlo;
    bulk_prefetch_l2(g.words + wo, nw * 4u);
    const uint32_t xe = min(wl + W, D.n);
    const uint32_t xb = ((xe > wl ? xe - wl : 0u) * (uint32_t)sizeof(XT)) & ~15u;
    if (xb && (reinterpret_cast<uintptr_t>(x) & 15u) == 0) bulk_prefetch_l2(x + wl, xb);
  }

  ChainCtx rc;
  rc.rows = s_rows;
  rc.ptr = reinterpret_cast<uint16_t*>(smem + L.off_ptr);
  rc.wscratch = misc + 16;
  rc.nr = nr;
  YT* yb = y + (r0 - g.row_begin);
  if constexpr (PR) {
    const uint32_t sh = r0 - g.row_begin;
    PageRankEpi epi;
    epi.deg = pr.deg + sh;
    epi.p_prev = pr.p_prev ? pr.p_prev + sh : nullptr;
    epi.q_next = pr.q_next + sh;
    epi.partial = pr.partial;
    epi.base = pr.alpha / (double)pr.n;
    epi.alpha_p0 = pr.alpha;
    epi.scale = 1.0 - pr.alpha;
    const double dm = pr.dmass ? *pr.dmass : pr.dmass_host;
    epi.dn = pr.uniform ? dm / (double)pr.n : 0.0;
    epi.bl = bl;
    epi.dang = 0.0;
    epi.l1 = 0.0;
    epi.push_mask = pr.push_mask ? pr.push_mask + sh : nullptr;
    epi.p0 = pr.p0 ? pr.p0 + r0 : nullptr;
    epi.push_dst = pr.push_dst;
    epi.grow0 = r0;
    chain_and_store(rc, yb, epi, D.max_depth, T);
  } else {
    PlainEpi epi;
    chain_and_store(rc, yb, epi, D.max_depth, T);
  }
}

}  // namespace cmvg
