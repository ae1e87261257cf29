// Shared device pieces of the BV-D product kernels: block staging (TMA bulk
// copy of the coded block), row setup (row bit offsets + warp rounds), code
// extraction, compensated accumulation and the reference-chain level
// scheduler.  Layout: host/layout.hpp.
#pragma once
#include <cstdint>

#include "../host/layout.hpp"
#include "ptx.cuh"
#include "xwindow.cuh"

namespace cmvg {

struct BvdDev {
  const uint32_t* words;
  const BvdBlockInfo* blocks;
  BvdDims d;
  uint32_t block_begin;       // first block of this shard
  uint32_t row_begin;         // first row of this shard
  uint32_t stream_cap_words;  // blocks with more words decode from global memory
  uint32_t pad;
};

__host__ __device__ inline uint32_t align16(uint32_t v) { return (v + 15u) & ~15u; }

// ---- coded-stream sources --------------------------------------------------
// Staged blocks are read with 32-bit shared-window addresses (LDS), large
// blocks straight from global memory.
template <bool STAGED>
struct Src;
template <>
struct Src<true> {
  uint32_t sbase;  // shared address of word 0
  __device__ __forceinline__ uint32_t w(uint32_t i) const {
    uint32_t v;
    asm("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(sbase + 4u * i));
    return v;
  }
};
template <>
struct Src<false> {
  const uint32_t* __restrict__ p;
  __device__ __forceinline__ uint32_t w(uint32_t i) const { return __ldg(p + i); }
};

template <class S>
__device__ __forceinline__ uint32_t extract_bits(const S& s, uint32_t off, uint32_t w) {
  const uint32_t wi = off >> 5, sh = off & 31u;
  const uint64_t win = (((uint64_t)s.w(wi) << 32) | s.w(wi + 1)) << sh;
  return w ? (uint32_t)(win >> (64u - w)) : 0u;
}

// ---- row setup scratch -----------------------------------------------------
// Rows with more codes than this are decoded by a whole warp (lanes stride
// over the row's fixed-width codes) instead of one lane.
constexpr uint32_t kHeavyCodes = 96;

struct RowSmem {
  uint32_t off_rowoff, off_perm, off_permi, off_permh, off_key, off_ref, off_misc, total;
};
__host__ __device__ inline RowSmem row_smem_layout(uint32_t base, uint32_t B) {
  RowSmem s;
  uint32_t o = base;
  s.off_rowoff = o;
  o = align16(o + B * 4);
  s.off_perm = o;
  o = align16(o + B * 2);
  s.off_permi = o;
  o = align16(o + B * 2);
  s.off_permh = o;
  o = align16(o + B * 2);
  s.off_key = o;
  o = align16(o + B * 2);
  s.off_ref = o;
  o = align16(o + B);
  s.off_misc = o;  // mbarrier (16) + 16 ints + 2 x 64-bin histograms + scratch (64 ints)
  o = align16(o + 16 + 64 + 128 * 4 + 64 * 4);
  s.total = o;
  return s;
}

enum MiscSlot : int {
  kNesc = 0,    // escaped rows in the block
  kNInt = 2,    // light rows with intervals
  kNPts = 3,    // light rows (point rounds)
  kRoundP = 4,  // dynamic round counters
  kRoundI = 5,
  kNHeavy = 6,  // heavy rows
  kRoundH = 7,
};

struct RowCtx {
  uint32_t* rowoff;  // bit offset of each row body
  uint16_t* perm;    // rows by point-code count desc (later: chain pointers)
  uint16_t* permi;   // light rows with intervals, by interval count desc
  uint16_t* permh;   // heavy rows (warp-cooperative)
  uint16_t* key;     // per-row sort keys
  uint8_t* ref;      // reference distance per row
  int* misc;
  int* hist;      // 2 x 64 bins
  int* wscratch;  // 64 ints
  uint64_t* bar;
  uint32_t nr, B;
};

__device__ __forceinline__ RowCtx carve_rows(unsigned char* smem, const RowSmem& L, uint32_t B, uint32_t nr) {
  RowCtx c;
  c.rowoff = reinterpret_cast<uint32_t*>(smem + L.off_rowoff);
  c.perm = reinterpret_cast<uint16_t*>(smem + L.off_perm);
  c.permi = reinterpret_cast<uint16_t*>(smem + L.off_permi);
  c.permh = reinterpret_cast<uint16_t*>(smem + L.off_permh);
  c.key = reinterpret_cast<uint16_t*>(smem + L.off_key);
  c.ref = reinterpret_cast<uint8_t*>(smem + L.off_ref);
  c.bar = reinterpret_cast<uint64_t*>(smem + L.off_misc);
  c.misc = reinterpret_cast<int*>(smem + L.off_misc + 16);
  c.hist = reinterpret_cast<int*>(smem + L.off_misc + 80);
  c.wscratch = reinterpret_cast<int*>(smem + L.off_misc + 80 + 512);
  c.B = B;
  c.nr = nr;
  return c;
}

// Thread 0 issues the TMA bulk copy of the block's coded stream; blocks
// larger than the staging cap are decoded from global memory instead.
__device__ __forceinline__ bool stage_stream_begin(const BvdDev& g, const BvdBlockInfo& bi, uint32_t* s_stream,
                                                   uint64_t* s_bar) {
  const bool staged = bi.nwords <= g.stream_cap_words;
  if (threadIdx.x == 0) {
    mbar_init(s_bar, 1);
    const uint32_t sbytes = staged ? bi.nwords * 4u : 0u;
    mbar_arrive_expect_tx(s_bar, sbytes);
    if (sbytes) bulk_g2s(s_stream, g.words + bi.word_offset, sbytes, s_bar);
  }
  if (threadIdx.x < 8) s_stream[(staged ? bi.nwords : 0u) + threadIdx.x] = 0u;
  return staged;
}

struct RowCounts {
  uint32_t nm, ns, ni;
};
template <class S>
__device__ __forceinline__ RowCounts row_counts(const S& src, uint32_t B, uint32_t h, uint32_t k, int nesc) {
  RowCounts c{hdr_nm(h), hdr_ns(h), hdr_ni(h)};
  if (hdr_escaped(h)) {  // rare: binary search of the escape table
    int lo = 0, hi = nesc - 1;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (src.w(B + 4u * mid) < k) lo = mid + 1;
      else hi = mid;
    }
    c.nm = src.w(B + 4u * lo + 1);
    c.ns = src.w(B + 4u * lo + 2);
    c.ni = src.w(B + 4u * lo + 3);
  }
  return c;
}

__device__ __forceinline__ int warp_excl_scan(int v, int& total) {
  const uint32_t lane = threadIdx.x & 31u;
  int inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int u = __shfl_up_sync(0xffffffffu, inc, o);
    if ((int)lane >= o) inc += u;
  }
  total = __shfl_sync(0xffffffffu, inc, 31);
  return inc - v;
}

// Row setup, all threads: row bit offsets (exclusive scan of body lengths),
// reference pointers, and the round permutations (counting sorts): rows by
// point-code count (perm) and rows with intervals by interval count (permi),
// both descending so the heaviest rounds are claimed first.
// Ends with __syncthreads().
template <class S>
__device__ __forceinline__ void row_setup(RowCtx& c, const S& src, int nesc, bool split_heavy = false) {
  const uint32_t T = blockDim.x, tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5, nwarps = T >> 5;
  const uint32_t B = c.B, nr = c.nr;
  const uint32_t per = (B + T - 1) >> (31 - __clz(T));  // T is a power of 2
  const uint32_t k0 = tid * per;
  int* hp = c.hist;
  int* hi = c.hist + 64;
  for (uint32_t k = tid; k < 128; k += T) c.hist[k] = 0;
  if (tid < 16) c.misc[tid] = 0;
  __syncthreads();
  const uint32_t body0 = (B + 4u * (uint32_t)nesc) * 32u;  // bodies follow headers + escape table
  uint32_t loc = 0;
  for (uint32_t j = 0; j < per; ++j) {
    const uint32_t k = k0 + j;
    if (k < nr) {
      const uint32_t h = src.w(k);
      const RowCounts rc = row_counts(src, B, h, k, nesc);
      c.rowoff[k] = loc;
      loc += (rc.nm + rc.ns + rc.ni) * hdr_wp(h) + rc.ni * hdr_wl(h);
      c.ref[k] = (uint8_t)hdr_r(h);
      const uint32_t kp = min(rc.nm + rc.ns, 63u), ki = min(rc.ni, 63u);
      const bool heavy = split_heavy && rc.nm + rc.ns + 2 * rc.ni > kHeavyCodes;
      c.key[k] = (uint16_t)((heavy ? 0x8000u : 0u) | (ki << 6) | kp);
      if (heavy) {
        c.permh[atomicAdd(&c.misc[kNHeavy], 1)] = (uint16_t)k;
      } else {
        atomicAdd(&hp[kp], 1);
        if (ki) atomicAdd(&hi[ki], 1);
      }
    }
  }
  int wtot;
  const int ex = warp_excl_scan((int)loc, wtot);
  if (lane == 0) c.wscratch[warp] = wtot;
  __syncthreads();
  for (uint32_t which = warp; which < 2; which += nwarps) {  // descending-key bin starts
    int* hb = c.hist + 64 * which;
    const int v0 = hb[63 - 2 * lane], v1 = hb[62 - 2 * lane];
    int tot;
    const int e2 = warp_excl_scan(v0 + v1, tot);
    hb[63 - 2 * lane] = e2;
    hb[62 - 2 * lane] = e2 + v0;
    if (lane == 0) c.misc[which == 1 ? kNInt : kNPts] = tot;
  }
  uint32_t wbase = 0;
  for (uint32_t w = 0; w < warp; ++w) wbase += (uint32_t)c.wscratch[w];
  const uint32_t tbase = body0 + wbase + (uint32_t)ex;
  __syncthreads();
  for (uint32_t j = 0; j < per; ++j) {
    const uint32_t k = k0 + j;
    if (k < nr) {
      c.rowoff[k] += tbase;
      const uint32_t key = c.key[k];
      if (key & 0x8000u) continue;  // heavy rows are already listed
      c.perm[atomicAdd(&hp[key & 63u], 1)] = (uint16_t)k;
      const uint32_t ki = (key >> 6) & 63u;
      if (ki) c.permi[atomicAdd(&hi[ki], 1)] = (uint16_t)k;
    }
  }
  if (tid == 0) c.misc[kNesc] = nesc;
  __syncthreads();
}

// Claim the next round of 32 rows (warp-uniform).
__device__ __forceinline__ uint32_t next_round(int* counter) {
  uint32_t rb = 0;
  if ((threadIdx.x & 31u) == 0) rb = 32u * (uint32_t)atomicAdd(counter, 1);
  return __shfl_sync(0xffffffffu, rb, 0);
}
// Split claim: issue the atomic early (lane 0), consume its result later, so
// the shared-atomic latency overlaps the current round's decode.
__device__ __forceinline__ uint32_t claim_issue(int* counter) {
  return (threadIdx.x & 31u) == 0 ? (uint32_t)atomicAdd(counter, 1) : 0u;
}
__device__ __forceinline__ uint32_t claim_take(uint32_t ticket) { return 32u * __shfl_sync(0xffffffffu, ticket, 0); }

// Compensated accumulation: TwoSum, error term into `c` (error ~ eps|sum| +
// n eps^2 sum|t|), so y_i stays accurate when the differential terms cancel.
__device__ __forceinline__ void tsum(double& s, double& c, double t) {
  const double u = s + t;
  const double bb = u - s;
  c += (s - (u - bb)) + (t - bb);
  s = u;
}

__device__ __forceinline__ void dd_add(double& hi, double& lo, double bhi, double blo) {
  const double s = hi + bhi;
  const double bb = s - hi;
  const double e = (hi - (s - bb)) + (bhi - bb) + lo + blo;
  hi = s + e;
  lo = e - (hi - s);
}

// Output stage of the gather: plain y, or the fused PageRank update
// (pagerank.hpp:83-102, Eq. 1):
//   p'_i = alpha/n + (1 - alpha) (y_i + D/n)   (D = dangling mass, kUniform;
//                                                0 for kDrop)
//   q'_i = p'_i / d_i  (0 for dangling i)
// plus per-block partials {sum_{d_i = 0} p'_i, sum |p'_i - p_i|}.
struct PlainEpi {
  template <typename YT>
  __device__ __forceinline__ void store(YT* yb, uint32_t k, double y) const {
    yb[k] = (YT)y;
  }
  __device__ __forceinline__ void finish(int*) const {}
};

struct PageRankEpi {
  const uint32_t* deg;     // out-degrees of A for this block's rows (shard-relative, offset applied)
  const double* p_prev;    // may be null
  double* q_next;          // shard-relative, offset applied
  double* partial;         // [nblocks][2]
  double base, scale, dn;  // alpha/n, 1 - alpha, D/n (or 0)
  uint32_t bl;
  double dang, l1;         // per-thread partials
  template <typename YT>
  __device__ __forceinline__ void store(YT* pb, uint32_t k, double y) {
    const double pn = base + scale * (y + dn);
    pb[k] = (YT)pn;
    const uint32_t d = deg[k];
    q_next[k] = d ? pn / (double)d : 0.0;
    if (!d) dang += pn;
    if (p_prev) l1 += fabs(pn - p_prev[k]);
  }
  __device__ __forceinline__ void finish(int* scratch) {
    // deterministic block reduction: warp sums, then warp 0 in warp order
    double a = dang, b = l1;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      a += __shfl_down_sync(0xffffffffu, a, o);
      b += __shfl_down_sync(0xffffffffu, b, o);
    }
    double* ws = reinterpret_cast<double*>(scratch);
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    __syncthreads();
    if (lane == 0) {
      ws[2 * warp] = a;
      ws[2 * warp + 1] = b;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double sa = 0.0, sb = 0.0;
      for (uint32_t w = 0; w < nw; ++w) {
        sa += ws[2 * w];
        sb += ws[2 * w + 1];
      }
      partial[2 * bl] = sa;
      partial[2 * bl + 1] = sb;
    }
  }
};

// Reference-chain resolution -- the level scheduler.  Every row holds
// (value, pointer) = (delta_i, i - r_i); each level of pointer jumping is one
// barrier-separated data-parallel step
//     value_i += value_{ptr_i};  ptr_i = ptr_{ptr_i}
// in double-double, so after ceil(log2(depth + 1)) levels value_i = y_i =
// delta_i + y_{i - r_i} (ref_matvec.hpp:23-25; the pairing differs from the
// reference's left-to-right order only below double-double resolution).
// Bounded chains (R = 3) take two levels; unbounded ones log2(depth).
// Writes y (YT) with coalesced stores.  Uses c.perm as the pointer array.
template <typename YT, class EPI = PlainEpi>
__device__ __forceinline__ void chain_and_store(double* s_yhi, float* s_ylo, RowCtx& c, YT* __restrict__ yb,
                                                EPI epi = EPI(), uint32_t max_depth = 0xffffffffu) {
  const uint32_t T = blockDim.x, tid = threadIdx.x;
  if (max_depth <= 3) {
    // Bounded chains (R <= 3): each row walks its <= 3 ancestors,
    // y_i = d_i + d_p1 + d_p2 + d_p3 accumulated with TwoSum (error terms
    // collected with the low parts), no barriers.
    for (uint32_t k = tid; k < c.nr; k += T) {
      double s = s_yhi[k], e = (double)s_ylo[k];
      uint32_t p = k, r = c.ref[k];
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        if (r) {
          p -= r;
          tsum(s, e, s_yhi[p]);
          e += (double)s_ylo[p];
          r = c.ref[p];
        }
      }
      epi.store(yb, k, s + e);
    }
    epi.finish(c.wscratch);
    return;
  }
  constexpr uint32_t kMaxPer = 4;  // rows per thread per level (block_rows / threads <= 4)
  constexpr uint16_t kNone = 0xffffu;
  uint16_t* ptr = c.perm;
  int any = 0;
  for (uint32_t k = tid; k < c.nr; k += T) {
    const uint32_t r = c.ref[k];
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
      const uint32_t k = tid + q * T;
      if (k < c.nr) {
        const uint32_t p = ptr[k];
        double h = s_yhi[k], l = s_ylo[k];
        uint16_t pn = kNone;
        if (p != kNone) {
          dd_add(h, l, s_yhi[p], s_ylo[p]);
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
      const uint32_t k = tid + q * T;
      if (k < c.nr) {
        s_yhi[k] = nh[q];
        s_ylo[k] = (float)nl[q];
        ptr[k] = np_[q];
      }
    }
    any = __syncthreads_or(more);
  }
  for (uint32_t k = tid; k < c.nr; k += T) epi.store(yb, k, s_yhi[k] + (double)s_ylo[k]);
  epi.finish(c.wscratch);
}

}  // namespace cmvg
