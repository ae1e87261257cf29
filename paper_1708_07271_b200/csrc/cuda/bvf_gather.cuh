// bvf_gather: y = A * x^T on the flat term layout BV-F (host/layout.hpp) -- the
// gather hot path replacing the reference's sequential `matvec_ref_into`
// (include/cmv/ref_matvec.hpp:20-31), and
// (PR = true) the product + update of one PageRank iteration
// (pagerank.hpp:83-102).
//
// One CTA of 256 threads per block of B rows (reference chains never leave a
// block), 4 CTAs per SM at the default shape:
//   1. staging: the x-window x[wlo, wlo + W) and the block's far columns go to
//      a shared-memory table (fp64 x, default shape: one TMA bulk copy per
//      warp straight into the table, awaited on the warp's mbarrier); each x is split exactly at a block-wide grid
//      G = 2^(E - cbits) (E: the block's largest exponent) into
//      h = (x + s) - s, a multiple of G, and l = x - h (both exact), and the
//      window's exclusive prefix F = (sum h, sum l) is written after it.  Sums
//      of h are EXACT in fp64 (the transcoder bounds every partial sum below
//      2^53 G), so the differential evaluation loses nothing to cancellation
//      in the h part -- the rounding left is that of the small l sums
//      (|l| <= G/2) -- and reference chains, carries and prefix differences
//      are plain adds (no TwoSum);
//   2. terms: thread t sums chunk t of the block's flat term list (K terms,
//      coalesced word loads straight into registers), +-table[index] split as
//      above, and stores a row's differential sum when the row's last term
//      passes -- every thread has the same work whatever the row lengths;
//   3. a row cut by a chunk boundary gets the preceding chunks' tails (carry);
//   4. reference chains y_i = delta_i + y_{i-r} (ref_matvec.hpp:23-25) and the
//      coalesced store or the fused PageRank epilogue.
#pragma once
#include <cstdint>
#include <type_traits>

#include "bvs_gather.cuh"

#ifndef BVF_TMA
#define BVF_TMA 1
#endif

namespace cmvg {

struct BvfDev {
  const uint32_t* words;
  const BvfBlockInfo* blocks;
  uint32_t n, B, W, max_depth;
  uint32_t block_begin;  // first block of this launch (global numbering)
  uint32_t row_begin;    // first row of the shard (y is shard-relative)
  uint32_t nlaunch;
  uint32_t ahead;  // L2 prefetch distance in blocks (about the CTAs resident at once; 0 = none)
  const uint32_t* esc_base;  // first escape of each block of this launch (index into xe)
};

struct __align__(16) RowD {
  double hi, lo;
};

constexpr uint32_t kBvfThreads = 256;
constexpr uint32_t kBvfXPer = 8;  // window entries per thread (W <= 2048)

struct BvfSmem {
  uint32_t off_tab, off_fhi, off_flo, off_rows, off_rn, off_misc, total;
};
// The x/F table region is dead after the term loop; the pointer-jumping chain
// reuses it.  x window, far slots, zero entry and F hi are one table of
// doubles; split (fp64 x): then F lo, and row records (sum hi, lo) of 16
// bytes; plain (fp32 x): row records are the 8-byte sum.
__host__ __device__ inline BvfSmem bvf_smem_layout(uint32_t W, uint32_t B, bool split) {
  BvfSmem s;
  uint32_t o = 0;
  s.off_tab = o;  // x window, far slots, zero entry, F hi
  s.off_fhi = o + bvf_f0(W) * 8u;
  o = align16(o + (bvf_f0(W) + W + 1) * 8u);
  s.off_flo = o;  // F lo (split mode)
  o = align16(o + (split ? (W + 1) * 8u : 0u));
  s.off_rows = o;
  o = align16(o + B * (split ? 16u : 8u));
  s.off_rn = o;  // r per row, one byte each
  o = align16(o + kBvfRnWords * 8u);
  s.off_misc = o;  // warp maxima / totals / carries / epilogue scratch
  o = align16(o + 64 * 8);
  s.total = o;
  return s;
}

// reference distance of block row k (bytes in shared memory, expanded from the stream's nibbles)
__device__ __forceinline__ uint32_t bvf_r(const uint8_t* r8, uint32_t k) { return r8[k]; }
__device__ __forceinline__ uint32_t bvf_slot(uint32_t k) { return k; }

// flip the sign of v when bit 31 of m is set
__device__ __forceinline__ double flip_sign(double v, uint32_t m) {
  return __hiloint2double(__double2hiint(v) ^ (int)(m & 0x80000000u), __double2loint(v));
}

// shared-memory accesses by 32-bit shared address (the hot loop keeps one
// uniform base per table and adds the term's byte offset)
__device__ __forceinline__ double lds_f64(uint32_t a) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ float lds_f32(uint32_t a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts_f64(uint32_t a, double x) {
  asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(x) : "memory");
}
__device__ __forceinline__ void sts_f64x2(uint32_t a, double x, double y) {
  asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(a), "d"(x), "d"(y) : "memory");
}

template <typename XT, bool SPLIT, bool ESC>
struct BvfTerms {
  uint32_t tab;    // shared address: x / slots / zero / F hi, 8 bytes per term index
  uint32_t flo_b;  // shared address of F lo minus F0 * 8 (the term's byte offset indexes it)
  const XT* esc;  // x values of this chunk's escape terms, in term order (ESC; bvf_esc_gather)
  double sigma;
  uint32_t f0b;  // F0 * 8
  // one term: +-table[index] split at the block grid; bit 31 of `signw` is the
  // term's minus flag; a row end stores the row's sum at rowp and moves on
  // ev: the term's x value when it is an escape (loaded ahead, see esc_group)
  // END: the term may end a row (the high term of a word; rows have an even
  // number of terms, so the low term never does)
  template <bool END>
  __device__ __forceinline__ void term(uint32_t c, uint32_t signw, double& ah, double& al, uint32_t& rowp,
                                       XT ev = XT(0)) const {
    const uint32_t off = (c << 3) & (kBvfIdxMask << 3);
    const bool e = ESC && (c & kBvfEsc);
    double v;
    if (e) v = (double)ev;
    else v = lds_f64(tab + off);
    // the minus flag flips the sign bit of the value (and of its F lo part);
    // the split of -v is the negated split of v up to the choice of h on a
    // tie, and either choice keeps h a multiple of G and v - h exact
    const uint32_t sm = signw & 0x80000000u;
    v = __hiloint2double(__double2hiint(v) ^ (int)sm, __double2loint(v));
    if (SPLIT) {
      const double h = (v + sigma) - sigma;
      ah += h;
      al += v - h;
      if (off >= f0b && !e) {  // F term: its lo part (a predicated load)
        const double wl = lds_f64(flo_b + off);
        al += __hiloint2double(__double2hiint(wl) ^ (int)sm, __double2loint(wl));
      }
    } else {
      ah += v;
    }
    if (END && (c & kBvfEnd)) {
      if (SPLIT) {
        sts_f64x2(rowp, ah, al);
        rowp += 16;
      } else {
        sts_f64(rowp, ah);
        rowp += 8;
      }
      ah = 0.0;
      al = 0.0;
    }
  }
  __device__ __forceinline__ void word(uint32_t w, double& ah, double& al, uint32_t& rowp) const {
    term<false>(w & 0xffffu, w << 16, ah, al, rowp);
    term<true>(w >> 16, w, ah, al, rowp);
  }
  // escape blocks: 8 terms at a time, the x values of their escapes (gathered
  // ahead by bvf_esc_gather) loaded together before the sums
  __device__ __forceinline__ void esc_group(const uint32_t* w4, double& ah, double& al, uint32_t& rowp) const {
    XT ev[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint32_t c = (w4[i >> 1] >> (16 * (i & 1))) & 0xffffu;
      ev[i] = (c & kBvfEsc) ? __ldg(esc + (c & kBvfIdxMask)) : XT(0);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      term<false>(w4[i] & 0xffffu, w4[i] << 16, ah, al, rowp, ev[2 * i]);
      term<true>(w4[i] >> 16, w4[i], ah, al, rowp, ev[2 * i + 1]);
    }
  }
};

template <typename XT, bool SPLIT, bool ESC>
__device__ __forceinline__ void bvf_chunk(const BvfTerms<XT, SPLIT, ESC>& tm, const uint32_t* __restrict__ cw,
                                          uint32_t nact, uint32_t nwords, const uint32_t (&w0)[8], double& ah,
                                          double& al, uint32_t& rowp) {
  uint32_t w[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) w[i] = w0[i];
  for (uint32_t q = 8;; q += 8) {
    uint32_t nx[8];
    const bool more = q < nwords;
    if (more) {
#pragma unroll
      for (int i = 0; i < 8; ++i) nx[i] = __ldg(cw + (size_t)(q + i) * nact);
    }
    if constexpr (ESC) {
      tm.esc_group(w, ah, al, rowp);
      tm.esc_group(w + 4, ah, al, rowp);
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) tm.word(w[i], ah, al, rowp);
    }
    if (!more) break;
#pragma unroll
    for (int i = 0; i < 8; ++i) w[i] = nx[i];
  }
}

// xe[i] = x[esc[i]] for the escape terms of a launch's blocks (columns outside
// a block's x-window and far slots): one independent, fully parallel gather,
// so the term loop streams the values instead of chasing column -> x.
// L2 eviction hints (createpolicy + L2::cache_hint): the escape columns and
// xe stream through L2 once (evict_first) while the gathered x lines stay
// (evict_last) -- at C4 x (134 MB of fp32) is about the size of L2 and the
// gathers hit it repeatedly
__device__ __forceinline__ uint64_t l2_policy_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint32_t ld_hint(const uint32_t* a, uint64_t pol) {
  uint32_t v;
  asm volatile("ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ float ld_hint(const float* a, uint64_t pol) {
  float v;
  asm volatile("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ double ld_hint(const double* a, uint64_t pol) {
  double v;
  asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ void st_hint(float* a, float v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(a), "f"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_hint(double* a, double v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(a), "d"(v), "l"(pol) : "memory");
}

template <typename XT>
__global__ void __launch_bounds__(256) bvf_esc_gather(const uint32_t* __restrict__ esc, uint64_t cnt,
                                                      const XT* __restrict__ x, XT* __restrict__ xe) {
  const uint64_t step = (uint64_t)gridDim.x * blockDim.x;
  uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t pf = l2_policy_first(), pl = l2_policy_last();
  for (; i + 3 * step < cnt; i += 4 * step) {  // four independent gathers in flight per thread
    uint32_t c[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) c[k] = ld_hint(esc + i + k * step, pf);
    XT v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] = ld_hint(x + c[k], pl);
#pragma unroll
    for (int k = 0; k < 4; ++k) st_hint(xe + i + k * step, v[k], pf);
  }
  for (; i < cnt; i += step) st_hint(xe + i, ld_hint(x + ld_hint(esc + i, pf), pl), pf);
}

// CW, CB: compile-time window and block rows (0 = from BvfDev): the default
// shape gets constant loop bounds and shared-memory offsets.
template <typename XT, typename YT, bool PR, uint32_t CW = 0, uint32_t CB = 0>
__global__ void __launch_bounds__(kBvfThreads, 4)
    bvf_gather_kernel(BvfDev g, const XT* __restrict__ x, const XT* xfar, const XT* __restrict__ xe,
                      YT* __restrict__ y, PrArgs pr) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr bool kSplit = sizeof(XT) == 8;  // fp32 x: plain fp64 sums (error far inside the fp32 tolerance)
  const uint32_t W = CW ? CW : g.W, B = CB ? CB : g.B;
  const BvfSmem L = bvf_smem_layout(W, B, kSplit);
  const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
  const uint32_t bl = blockIdx.x, b = g.block_begin + bl;
  const BvfBlockInfo bi = g.blocks[bl];
  const uint32_t r0 = b * B, nr = min(B, g.n - r0);
  const uint32_t* bs = g.words + bi.word_offset;
  const uint32_t K = bi.K, nact = bi.nact, nslot = bi.nslot;
  const uint32_t F0 = bvf_f0(W);
  double* tab = reinterpret_cast<double*>(smem + L.off_tab);
  double* fhi = reinterpret_cast<double*>(smem + L.off_fhi);
  double* flo = reinterpret_cast<double*>(smem + L.off_flo);
  constexpr uint32_t RS = kSplit ? 16u : 8u;  // row record bytes
  auto put_x = [&](uint32_t j, double v) { tab[j] = v; };
  auto get_x = [&](uint32_t j) -> double { return tab[j]; };
  char* rows = reinterpret_cast<char*>(smem + L.off_rows);
  uint8_t* r8 = reinterpret_cast<uint8_t*>(smem + L.off_rn);
  double* misc = reinterpret_cast<double*>(smem + L.off_misc);
  uint32_t* misc_u = reinterpret_cast<uint32_t*>(smem + L.off_misc);

  // ---- loads: code words of this chunk, x window chunk, far slots, r
  const bool active = tid < nact;
  const uint32_t* cw = bs + bi.codes_off + tid;
  if (tid == 32) {
    // the rest of this block's terms into L2 now (the loop's later word loads
    // then hit L2); and a wave ahead, the stream, window and table entry of the
    // block whose CTA will take this slot, so its dependent setup loads hit L2
    const uint32_t cb = bi.nwords - bi.codes_off;
    if (cb > 8 * nact) bulk_prefetch_l2(bs + bi.codes_off + 8 * nact, ((cb - 8 * nact) * 4u) & ~15u);
    if (g.ahead && bl + g.ahead < g.nlaunch) {
      const BvfBlockInfo* nb = g.blocks + bl + g.ahead;
      asm volatile("prefetch.global.L2 [%0];" ::"l"(nb));
    }
  }
  if (tid == 64 && g.ahead && bl + g.ahead / 2 < g.nlaunch) {
    // half a wave ahead (its table entry was prefetched half a wave ago)
    const BvfBlockInfo nb = g.blocks[bl + g.ahead / 2];
    // its header and terms; not its escape column table (read by the
    // escape pre-gather, never by this kernel: ~1 GB per product at C4)
    if (nb.flags & kBvfFlagEsc) {
      bulk_prefetch_l2(g.words + nb.word_offset, nb.esc_off * 4u);
      bulk_prefetch_l2(g.words + nb.word_offset + nb.codes_off, (nb.nwords - nb.codes_off) * 4u);
    } else {
      bulk_prefetch_l2(g.words + nb.word_offset, nb.nwords * 4u);
    }
    const uint32_t xe = min(nb.wlo + W, g.n);
    const uint32_t xb = ((xe > nb.wlo ? xe - nb.wlo : 0u) * (uint32_t)sizeof(XT)) & ~15u;
    if (xb && (reinterpret_cast<uintptr_t>(x + nb.wlo) & 15u) == 0) bulk_prefetch_l2(x + nb.wlo, xb);
  }
  // default shape, fp64 x: each warp's 192 window entries come by one TMA bulk
  // copy straight into the table (the raw x values are its entries), issued
  // before the other loads and awaited on the warp's own mbarrier -- no
  // per-thread global loads and table stores for the window
  constexpr bool kTma = BVF_TMA && kSplit && CW == 1536;
  bool tma = false;
  const uint32_t mbar = smem_u32(misc + 48 + warp);
  if constexpr (kTma) {
    tma = !(bi.wlo & 1u) && bi.wlo + CW <= g.n && (reinterpret_cast<uintptr_t>(x) & 15u) == 0;
    if (tma) {
      if (lane == 0) bulk_load_init(mbar, smem_u32(tab + warp * 192u), x + bi.wlo + warp * 192u, 192u * 8u);
      __syncwarp();
    }
  }
  uint32_t w0[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) w0[i] = active ? __ldg(cw + (size_t)i * nact) : 0u;
  const uint32_t srow = active ? (uint32_t)reinterpret_cast<const uint16_t*>(bs)[tid] : 0u;
  const uint32_t E = CW ? (CW + kBvfThreads - 1) / kBvfThreads : (W + kBvfThreads - 1) / kBvfThreads;
  // windows of more than kBvfXPer entries per thread (W > 2048, generic shape
  // only) stage through shared memory instead of registers
  const bool wide = CW == 0 && E > kBvfXPer;
  const uint32_t j0 = tid * E;
  // a full chunk of an even count: paired 16-byte loads and stores
  const bool full = !(E & 1u) && j0 + E <= W && bi.wlo + j0 + E <= g.n && !(bi.wlo & 1u) &&
                    (reinterpret_cast<uintptr_t>(x) & (2 * sizeof(XT) - 1)) == 0;
  double xv[kBvfXPer];
  {
    using P2 = typename std::conditional<sizeof(XT) == 8, double2, float2>::type;
#pragma unroll
    for (uint32_t k = 0; k < kBvfXPer; k += 2) {
      const uint32_t j = j0 + k, c = bi.wlo + j;
      xv[k] = xv[k + 1] = 0.0;
      if (k < E && !wide && !tma) {
        if (full) {
          const P2 v2 = __ldg(reinterpret_cast<const P2*>(x + c));
          xv[k] = (double)v2.x;
          xv[k + 1] = (double)v2.y;
        } else {
          if (j < W && c < g.n) xv[k] = (double)__ldg(x + c);
          if (k + 1 < E && j + 1 < W && c + 1 < g.n) xv[k + 1] = (double)__ldg(x + c + 1);
        }
      }
    }
  }
  double fv = 0.0;
  const uint32_t far_off = bvf_far_off(nact);
  if (tid < nslot) fv = (double)__ldg(xfar + __ldg(bs + far_off + tid));
  const uint32_t rnw = tid < kBvfRnWords ? __ldg(bs + bvf_rn_off(nact) + tid) : 0u;  // stored after the loop
  if constexpr (kTma) {
    if (tma) {
      mbar_wait(mbar, 0);
#pragma unroll
      for (uint32_t k = 0; k < 6; k += 2) {
        const double2 v2 = *reinterpret_cast<const double2*>(tab + j0 + k);
        xv[k] = v2.x;
        xv[k + 1] = v2.y;
      }
    }
  }

  // ---- block exponent (finite values), non-finite flag; the x table
  uint32_t emax = 0, nonfin = 0;
  auto see = [&](double v) {
    const uint32_t e = ((uint32_t)__double2hiint(v) >> 20) & 0x7ffu;
    if (e == 0x7ffu) nonfin = 1;
    else emax = max(emax, e);
  };
  if (wide) {  // lane-consecutive (coalesced loads, conflict-free stores)
    for (uint32_t j = tid; j < W; j += kBvfThreads) {
      const uint32_t c = bi.wlo + j;
      const double v = c < g.n ? (double)__ldg(x + c) : 0.0;
      put_x(j, v);
      see(v);
    }
  }
#pragma unroll
  for (uint32_t k = 0; k < kBvfXPer; k += 2) {
    see(xv[k]);
    see(xv[k + 1]);
    const uint32_t j = j0 + k;
    if (k < E && !wide && !tma) {
      if (full) {
        *reinterpret_cast<double2*>(tab + j) = make_double2(xv[k], xv[k + 1]);
      } else {
        if (j < W) put_x(j, xv[k]);
        if (k + 1 < E && j + 1 < W) put_x(j + 1, xv[k + 1]);
      }
    }
  }
  see(fv);
  if (tid < nslot) put_x(W + tid, fv);
  const XT* xeb = xe;  // this block's escape values
  if (bi.flags & kBvfFlagEsc) {
    xeb = xe + __ldg(g.esc_base + bl);
    if (kSplit) {  // escaped columns take part in the exponent
      const uint32_t nesc = __ldg(bs + bi.esc_off + nact);
      for (uint32_t i = tid; i < nesc; i += kBvfThreads) see((double)__ldg(xeb + i));
    }
  }
  if (tid == 0) put_x(bvf_zero(W), 0.0);
  emax = __reduce_max_sync(0xffffffffu, emax);
  nonfin = __any_sync(0xffffffffu, nonfin);
  if (lane == 0) misc_u[warp] = emax | (nonfin << 16);
  __syncthreads();  // #1
  uint32_t em = 0, nf = 0;
#pragma unroll
  for (uint32_t w = 0; w < kBvfThreads / 32; ++w) {
    const uint32_t v = misc_u[w];
    em = max(em, v & 0xffffu);
    nf |= v >> 16;
  }
  // sigma = 1.5 * 2^(g + 52), g = E - cbits, E = em - 1023 + 1: h = (x + sigma) - sigma
  // rounds x to a multiple of 2^g; a non-finite block sums plainly (sigma = 0)
  double sigma = 0.0;
  if (kSplit && !nf) {
    int ef = (int)em + 1 + 52 - (int)bi.cbits;
    ef = max(ef, 1);
    sigma = __hiloint2double((ef << 20) | 0x80000, 0);
  }

  // ---- window prefix F (exclusive): F hi = sum h (exact), F lo = sum l
  {
    double sh = 0.0, sl = 0.0;
    // wide: warp w owns the window segment [w S, (w + 1) S), read lane-consecutively
    const uint32_t S = ((W + 8 * 32 - 1) / (8 * 32)) * 32, s0 = warp * S, s1 = min(W, s0 + S);
    if (wide) {
      for (uint32_t j = s0 + lane; j < s1; j += 32) {
        const double v = get_x(j);
        if (kSplit) {
          const double h = (v + sigma) - sigma;
          sh += h;
          sl += v - h;
        } else {
          sh += v;
        }
      }
    }
#pragma unroll
    for (uint32_t k = 0; k < kBvfXPer; ++k) {
      if (k < E && !wide) {
        const double v = xv[k];
        if (kSplit) {
          const double h = (v + sigma) - sigma;
          sh += h;
          sl += v - h;
        } else {
          sh += v;
        }
      }
    }
    // inclusive warp scan of the chunk totals
    double ih = sh, il = sl;
#pragma unroll
    for (uint32_t o = 1; o < 32; o <<= 1) {
      const double uh = __shfl_up_sync(0xffffffffu, ih, o);
      const double ul = kSplit ? __shfl_up_sync(0xffffffffu, il, o) : 0.0;
      if (lane >= o) {
        ih += uh;
        il += ul;
      }
    }
    if (lane == 31) {
      misc[16 + 2 * warp] = ih;
      misc[16 + 2 * warp + 1] = il;
    }
    __syncthreads();  // #2
    double bh = ih - sh, blo = il - sl;  // exclusive within the warp
    for (uint32_t w = 0; w < warp; ++w) {
      bh += misc[16 + 2 * w];
      blo += misc[16 + 2 * w + 1];
    }
    if (wide) {
      // the warp's offset (totals of the warps before it), then a warp scan per round of 32
      double wh = 0.0, wl = 0.0;
      for (uint32_t w = 0; w < warp; ++w) {
        wh += misc[16 + 2 * w];
        wl += misc[16 + 2 * w + 1];
      }
      for (uint32_t jb = s0; jb < s1; jb += 32) {
        const uint32_t j = jb + lane;
        const double v = j < s1 ? get_x(j) : 0.0;
        double h = v, l = 0.0;
        if (kSplit) {
          h = (v + sigma) - sigma;
          l = v - h;
        }
        double ih2 = h, il2 = l;
#pragma unroll
        for (uint32_t o = 1; o < 32; o <<= 1) {
          const double uh = __shfl_up_sync(0xffffffffu, ih2, o);
          const double ul = kSplit ? __shfl_up_sync(0xffffffffu, il2, o) : 0.0;
          if (lane >= o) {
            ih2 += uh;
            il2 += ul;
          }
        }
        if (j < s1) {
          fhi[j] = wh + (ih2 - h);
          if (kSplit) flo[j] = wl + (il2 - l);
        }
        if (j + 1 == W) {  // F[W]
          fhi[W] = wh + ih2;
          if (kSplit) flo[W] = wl + il2;
        }
        wh += __shfl_sync(0xffffffffu, ih2, 31);
        wl += __shfl_sync(0xffffffffu, il2, 31);
      }
    }
#pragma unroll
    for (uint32_t k = 0; k < kBvfXPer; k += 2) {
      if (wide) break;
      const uint32_t j = j0 + k;
      double h0 = bh, l0 = blo;
      if (k < E) {
        const double v = xv[k];
        if (kSplit) {
          const double h = (v + sigma) - sigma;
          bh += h;
          blo += v - h;
        } else {
          bh += v;
        }
      }
      double h1 = bh, l1 = blo;
      if (k + 1 < E) {
        const double v = xv[k + 1];
        if (kSplit) {
          const double h = (v + sigma) - sigma;
          bh += h;
          blo += v - h;
        } else {
          bh += v;
        }
      }
      if (k < E) {
        if (full) {
          *reinterpret_cast<double2*>(fhi + j) = make_double2(h0, h1);
          if (kSplit) *reinterpret_cast<double2*>(flo + j) = make_double2(l0, l1);
        } else {
          if (j < W) {
            fhi[j] = h0;
            if (kSplit) flo[j] = l0;
          }
          if (k + 1 < E && j + 1 < W) {
            fhi[j + 1] = h1;
            if (kSplit) flo[j + 1] = l1;
          }
        }
      }
    }
    if (!wide && j0 < W && j0 + E >= W) {  // the thread holding the window's last entry writes F[W]
      fhi[W] = bh;
      if (kSplit) flo[W] = blo;
    }
  }
  __syncthreads();  // #3

  // ---- terms
  double ah = 0.0, al = 0.0;
  const uint32_t rows_s = smem_u32(rows);
  uint32_t rowp = rows_s + srow * RS;
  if (active) {
    uint32_t tabc = smem_u32(tab);
    const uint32_t flob = smem_u32(flo) - F0 * 8u;
    if (bi.flags & kBvfFlagEsc) {
      // the table address and the chunk's escape pointer held in registers
      // (opaque to the compiler, which otherwise rebuilds the shared-window
      // base and a 64-bit element offset for every term)
      const XT* escp = xeb + __ldg(bs + bi.esc_off + tid);
      asm volatile("" : "+r"(tabc));
      asm volatile("" : "+l"(escp));
      BvfTerms<XT, kSplit, true> te{tabc, flob, escp, sigma, F0 * 8u};
      bvf_chunk(te, cw, nact, K / 2, w0, ah, al, rowp);
    } else {
      BvfTerms<XT, kSplit, false> tm{tabc, flob, nullptr, sigma, F0 * 8u};
      bvf_chunk(tm, cw, nact, K / 2, w0, ah, al, rowp);
    }
  }
  if (tid < kBvfRnWords) {  // r nibbles -> bytes
    uint32_t lo = 0, hi = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      lo |= ((rnw >> (4 * q)) & 15u) << (8 * q);
      hi |= ((rnw >> (4 * q + 16)) & 15u) << (8 * q);
    }
    reinterpret_cast<uint2*>(r8)[tid] = make_uint2(lo, hi);
  }
  // ---- carries: a row cut by chunk boundaries gets the tails of the chunks
  // before its end -- a segmented scan of the tails (segments start at the
  // chunks that end a row) in the warp, then across warps
  const bool has_end = active && rowp != rows_s + srow * RS;
  double sh = ah, sl = al;
  bool sf = has_end;
  if (!__all_sync(0xffffffffu, has_end || !active)) {  // a chunk inside one row: segmented scan
#pragma unroll
    for (uint32_t o = 1; o < 32; o <<= 1) {
      const double uh = __shfl_up_sync(0xffffffffu, sh, o), ul = __shfl_up_sync(0xffffffffu, sl, o);
      const bool uf = __shfl_up_sync(0xffffffffu, sf, o);
      if (lane >= o) {
        if (!sf) {
          sh += uh;
          sl += ul;
        }
        sf = sf || uf;
      }
    }
  }
  if (lane == 31) {
    misc[32 + 2 * warp] = sh;
    misc[32 + 2 * warp + 1] = sl;
    misc_u[8 + warp] = sf;
  }
  // carry into this lane's first row: the segment value of the lane before
  double ch = __shfl_up_sync(0xffffffffu, sh, 1), cl = __shfl_up_sync(0xffffffffu, sl, 1);
  const bool cf = __shfl_up_sync(0xffffffffu, sf, 1);
  if (lane == 0) ch = cl = 0.0;
  __syncthreads();  // #4
  if (has_end) {
    if (lane == 0 || !cf) {  // the segment reaches back past this warp's first lane
      for (int w = (int)warp - 1; w >= 0; --w) {
        ch += misc[32 + 2 * w];
        cl += misc[32 + 2 * w + 1];
        if (misc_u[8 + w]) break;
      }
    }
    if constexpr (kSplit) {
      double2* rr = reinterpret_cast<double2*>(rows + bvf_slot(srow) * 16u);
      double2 v = *rr;
      v.x += ch;
      v.y += cl;
      *rr = v;
    } else {
      reinterpret_cast<double*>(rows)[bvf_slot(srow)] += ch;
    }
  }
  __syncthreads();  // #5

  // ---- reference chains and the store
  auto rec = [&](uint32_t k) -> double2 {
    if constexpr (kSplit) return *reinterpret_cast<const double2*>(rows + bvf_slot(k) * 16u);
    else return make_double2(reinterpret_cast<const double*>(rows)[bvf_slot(k)], 0.0);
  };
  YT* yb = y + (r0 - g.row_begin);
  auto walk = [&](auto& epi) {
    if (g.max_depth <= 3) {
      for (uint32_t kb = tid; kb < nr; kb += kEpiPre * kBvfThreads) {
        epi.prefetch(kb, kBvfThreads, nr);
#pragma unroll
        for (uint32_t q = 0; q < kEpiPre; ++q) {
          const uint32_t k = kb + q * kBvfThreads;
          if (k >= nr) break;
          const double2 rk = rec(k);
          double hs = rk.x, ls = rk.y;
          uint32_t p = k, r = bvf_r(r8, k);
#pragma unroll
          for (int d = 0; d < 3; ++d) {
            if (r) {
              p -= r;
              const double2 rp = rec(p);
              hs += rp.x;
              ls += rp.y;
              r = bvf_r(r8, p);
            }
          }
          epi.store(yb, k, hs + ls, q);
        }
      }
    } else {
      // unbounded chains: pointer jumping, one barrier-separated level per step
      constexpr uint32_t kMaxPer = 4;  // B <= 1024 rows
      constexpr uint16_t kNone = 0xffffu;
      uint16_t* ptr = reinterpret_cast<uint16_t*>(tab);  // the table is dead after the terms
      int any = 0;
      for (uint32_t k = tid; k < nr; k += kBvfThreads) {
        const uint32_t r = bvf_r(r8, k);
        ptr[k] = r ? (uint16_t)(k - r) : kNone;
        any |= (r != 0);
      }
      any = __syncthreads_or(any);
      while (any) {
        double nh[kMaxPer], nl[kMaxPer];
        uint16_t np_[kMaxPer];
        int more = 0;
#pragma unroll
        for (uint32_t q = 0; q < kMaxPer; ++q) {
          const uint32_t k = tid + q * kBvfThreads;
          if (k < nr) {
            const uint32_t p = ptr[k];
            const double2 rk = rec(k);
            double h = rk.x, l = rk.y;
            uint16_t pn = kNone;
            if (p != kNone) {
              const double2 rp = rec(p);
              h += rp.x;
              l += rp.y;
              pn = ptr[p];
            }
            nh[q] = h;
            nl[q] = l;
            np_[q] = pn;
            more |= (pn != kNone);
          }
        }
        __syncthreads();
#pragma unroll
        for (uint32_t q = 0; q < kMaxPer; ++q) {
          const uint32_t k = tid + q * kBvfThreads;
          if (k < nr) {
            if constexpr (kSplit) *reinterpret_cast<double2*>(rows + bvf_slot(k) * 16u) = make_double2(nh[q], nl[q]);
            else reinterpret_cast<double*>(rows)[bvf_slot(k)] = nh[q];
            ptr[k] = np_[q];
          }
        }
        any = __syncthreads_or(more);
      }
      for (uint32_t kb = tid; kb < nr; kb += kEpiPre * kBvfThreads) {
        epi.prefetch(kb, kBvfThreads, nr);
#pragma unroll
        for (uint32_t q = 0; q < kEpiPre; ++q) {
          const uint32_t k = kb + q * kBvfThreads;
          if (k < nr) {
            const double2 rk = rec(k);
            epi.store(yb, k, rk.x + rk.y, q);
          }
        }
      }
    }
    epi.finish(reinterpret_cast<int*>(misc));
  };
  if constexpr (PR) {
    const uint32_t sh0 = r0 - g.row_begin;
    PageRankEpi epi;
    epi.deg = pr.deg + sh0;
    epi.p_prev = pr.p_prev ? pr.p_prev + sh0 : nullptr;
    epi.q_next = pr.q_next + sh0;
    epi.partial = pr.partial;
    epi.base = pr.alpha / (double)pr.n;
    epi.alpha_p0 = pr.alpha;
    epi.scale = 1.0 - pr.alpha;
    const double dm = pr.dmass ? *pr.dmass : pr.dmass_host;
    epi.dn = pr.uniform ? dm / (double)pr.n : 0.0;
    epi.bl = bl;
    epi.dang = 0.0;
    epi.l1 = 0.0;
    epi.push_mask = pr.push_mask ? pr.push_mask + sh0 : nullptr;
    epi.p0 = pr.p0 ? pr.p0 + r0 : nullptr;
    epi.push_dst = pr.push_dst;
    epi.grow0 = r0;
    walk(epi);
  } else {
    PlainEpi epi;
    walk(epi);
  }
}

}  // namespace cmvg
